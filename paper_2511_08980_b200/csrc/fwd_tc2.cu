// fwd_tc2.cu -- the tensor-core forward on CTA pairs (tcgen05 cta_group::2) with two half-tile
// slots in flight (tcpair.cuh).  Same arithmetic as fwd_tc.cu (modes 1 and 2, bf16x6, the
// cancellation-free pair maps, fdepi.cuh epilogues); what changes is the schedule:
//   * a pair tile = 2 slots of CPS centres (mode 1: 16 centres x 4 columns, mode 2: 8 centres
//     x 8 pair columns); each slot is a 64-column GEMM on the pair (M = 256 over 2 SMs, each SM
//     computing its 128 output neurons for all 64 columns);
//   * per layer the leader issues slot 0's MMAs, then slot 1's, while the 16 epilogue warps of
//     each CTA process the other slot -- the MMA phase of one slot overlaps the epilogue of the
//     other (the single-CTA kernels serialise them);
//   * each CTA streams only its 128 weight rows: 192 KB per slot-layer instead of 384 KB;
//   * the six bf16x6 products are issued as four M = 256 MMAs per K step into two TMEM
//     regions, R01 = a0.[b0|b1] + a1.[b0|b1] (N = 128) and R2 = a0.b2 + a2.b0 (N = 64): on a
//     pair one MMA does twice the work of a single-CTA one for the same issue cost
//     (scripts/mma_rate.py: 128 cycles per K step and M = 128 half, against 204 for the
//     single-CTA three-range form);
//   * operand hand-off: CTA r holds the B columns [32 r, 32 r + 32) of a slot for all 256 K
//     rows, but its epilogue threads produce K rows [128 r, 128 r + 128) for all 64 columns.
//     The peer's columns are written into a local 24 KB staging block laid out exactly as the
//     peer's B rows [128 r, ...), and a dedicated exchanger warp moves it with ONE
//     cp.async.bulk shared::cta -> shared::cluster per slot-layer (complete_tx on the peer's
//     mbarrier).  Everything the tensor cores read is then written either by local generic
//     stores behind fence.proxy.async.shared::cta or by the async proxy -- no cluster-scope
//     generic-proxy fence (MEMBAR.ALL.GPU) on the path, which is what made the first pair
//     version (remote st.shared::cluster per element) slower than the single-CTA kernel;
//   * the last-layer sums over the 256 neurons are reduced across the pair through distributed
//     shared memory into the CTA that owns the centre, whose first epilogue warp runs the
//     per-centre epilogue (frame / FD, Eq. (1) terms, seeds) during the next tile's first MMA
//     phase.
// Used for 256-padded widths (C2, C4, C5); the single-CTA kernels keep C1.
#include "act.cuh"
#include "fdepi.cuh"
#include "tcmlp.cuh"
#include "tcpair.cuh"

namespace fdsdf {

template <int MODE>
struct F2Cfg {
  static constexpr int MPAD = 256;
  static constexpr int KC = 4;                          // K chunks of 64
  static constexpr int NS = 64;                         // columns per slot (pair-wide)
  static constexpr int NH = 32;                         // columns per slot per CTA
  static constexpr int CPC = MODE == 1 ? 4 : 8;         // columns per centre
  static constexpr int CPS = NS / CPC;                  // centres per slot (16 / 8)
  static constexpr int COWN = NH / CPC;                 // centres per slot owned by one CTA
  static constexpr int STAGE = 3 * 128 * 128;           // weight stage: this CTA's 128 rows
  static constexpr int NST = 2;
  static constexpr int BSLOT = KC * 3 * NH * 128;       // B block of one slot in one CTA (48 KB)
  static constexpr int STG = 2 * 3 * NH * 128;          // staging: the peer's columns, 2 K chunks
  static constexpr int NEPI = 16;
  static constexpr int XW = 2 + NEPI;                   // exchanger warps: sender, receiver
  static constexpr int NTHR = (4 + NEPI) * 32;
  static constexpr int CPT = CPS / 4;                   // centres per epilogue thread per slot
  static constexpr int NRED = 8 * CPS * 4;              // floats per (parity, slot) reduction block
  static constexpr int DSL = 3 * NS;                    // TMEM columns per slot: R01 (2 NS), R2 (NS)
  static constexpr int OFF_W = 0;
  static constexpr int OFF_B = NST * STAGE;
  static constexpr int OFF_ST = OFF_B + 2 * BSLOT;
  static constexpr int OFF_RED = OFF_ST + STG;          // float [2 par][2 slot][8 grp][CPS][4]
  static constexpr int OFF_CI = OFF_RED + 4 * NRED * 4; // mode 2: float [2 par][2 slot][CPS][16]
  static constexpr int OFF_LV = OFF_CI + (MODE == 2 ? 4 * CPS * NCINFO * 4 : 0);
  static constexpr int OFF_BAR = OFF_LV + (MODE == 2 ? 2 * CPS * NLOSS * 8 : 0);
  // wfull, wempty, wpeer [NST]; bfull, dfull [2]; rfull [4]; sready, bin [2]; sfree
  static constexpr int NBAR = 3 * NST + 2 + 2 + 4 + 2 + 2 + 1;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr uint32_t TCOLS = 512;
  static_assert(2 * DSL <= (int)TCOLS, "two slots of R01 + R2");
  static_assert(BYTES <= 232448, "shared memory per CTA");
};

int fwd_tc2_tile_centres(int mode) { return mode == 1 ? 32 : 16; }

template <int ACT, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(F2Cfg<MODE>::NTHR, 1)
    fwd_tc2_kernel(const FwdArgs a) {
  using C = F2Cfg<MODE>;
  using AF = Act<ACT>;
  constexpr int MPAD = C::MPAD, NS = C::NS, NH = C::NH, CPS = C::CPS, CPC = C::CPC, CPT = C::CPT;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw;
  sm += (1024 - (smem_u32(sm) & 1023)) & 1023;
  unsigned char* Ws = sm + C::OFF_W;
  unsigned char* Bs = sm + C::OFF_B;
  unsigned char* Stg = sm + C::OFF_ST;
  float* red0 = reinterpret_cast<float*>(sm + C::OFF_RED);
  float* cis0 = reinterpret_cast<float*>(sm + C::OFF_CI);
  double* lvs = reinterpret_cast<double*>(sm + C::OFF_LV);
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* wempty = wfull + C::NST;
  uint64_t* wpeer = wempty + C::NST;
  uint64_t* bfull = wpeer + C::NST;
  uint64_t* dfull = bfull + 2;
  uint64_t* rfull = dfull + 2;  // [par][slot]
  uint64_t* sready = rfull + 4;
  uint64_t* bin = sready + 2;
  uint64_t* sfree = bin + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sfree + 1);

  const Net& net = a.net;
  const int L = net.L;
  const int nh = L - 1;
  const int ngemm = L - 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tp::ctarank();
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (tid == 0) {
    for (int s = 0; s < C::NST; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
      mbar_init(&wpeer[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bfull[s], 2);  // one arrival per CTA of the pair: its B half is complete
      mbar_init(&dfull[s], 1);
      mbar_init(&sready[s], C::NEPI);
      mbar_init(&bin[s], 1);
    }
    for (int s = 0; s < 4; ++s) mbar_init(&rfull[s], 2 * C::NEPI);
    mbar_init(sfree, 1);
    fence_mbar_init();
  }
  if (warp == 1) tp::tmem_alloc2(tslot, C::TCOLS);
  tc::fence_before();
  tp::cluster_sync();
  tc::fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ------------------------------------------------------------------ weight producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t tile = cid; tile < a.ntiles; tile += ncl)
        for (int g = 0; g < ngemm; ++g)
          for (int slot = 0; slot < 2; ++slot)
            for (int kc = 0; kc < C::KC; ++kc, ++it) {
              const int s = (int)(it % C::NST);
              mbar_wait(&wempty[s], ((it / C::NST) & 1u) ^ 1u);
              mbar_arrive_expect_tx(&wfull[s], C::STAGE);
              bulk_g2s(Ws + s * C::STAGE, a.wimg + (((size_t)g * C::KC + kc) * 2 + rank) * C::STAGE, C::STAGE,
                       &wfull[s]);
            }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------------------------------------------------------- MMA issuer (leader)
      // the whole warp runs the issue loop (warp-uniform descriptors in uniform registers);
      // one elected lane issues each tcgen05.mma / commit
      constexpr uint32_t id2 = tc::idesc_bf16(256, 2 * NS), id1 = tc::idesc_bf16(256, NS);
      uint32_t it = 0, nb[2] = {0u, 0u};
#ifdef FDSDF_PHASE_TIMING
      long long t0 = clock64(), tb = 0, tw = 0, tspan = 0, tm;
#endif
      for (int64_t tile = cid; tile < a.ntiles; tile += ncl)
        for (int g = 0; g < ngemm; ++g)
          for (int slot = 0; slot < 2; ++slot) {
#ifdef FDSDF_PHASE_TIMING
            tm = clock64();
#endif
            tp::wait_cluster(&bfull[slot], nb[slot] & 1u);
#ifdef FDSDF_PHASE_TIMING
            const long long tstart = clock64();
            tb += tstart - tm;
#endif
            ++nb[slot];
            tc::fence_after();
            const uint32_t bslot = smem_u32(Bs + slot * C::BSLOT);
            const uint32_t d01 = tbase + slot * C::DSL, d2 = d01 + 2 * NS;
            for (int kc = 0; kc < C::KC; ++kc, ++it) {
              const int s = (int)(it % C::NST);
              const uint32_t ph = (it / C::NST) & 1u;
#ifdef FDSDF_PHASE_TIMING
              tm = clock64();
#endif
              mbar_wait(&wfull[s], ph);
              tp::wait_cluster(&wpeer[s], ph);
#ifdef FDSDF_PHASE_TIMING
              tw += clock64() - tm;
#endif
              tc::fence_after();
              const uint32_t wa = smem_u32(Ws + s * C::STAGE);
              const uint32_t ba = bslot + kc * (3 * NH * 128);
#pragma unroll
              for (int sub = 0; sub < 4; ++sub) {
                const uint64_t b01 = tc::sdesc_sw128(ba + sub * 32);            // [b0|b1], NH rows each
                const uint64_t b2 = tc::sdesc_sw128(ba + 2 * NH * 128 + sub * 32);
                const uint32_t first = (kc | sub) != 0 ? 1u : 0u;
                tp::mma2_w(d01, tc::sdesc_sw128(wa + 0 * 16384 + sub * 32), b01, id2, first);
                tp::mma2_w(d01, tc::sdesc_sw128(wa + 1 * 16384 + sub * 32), b01, id2, 1u);
                tp::mma2_w(d2, tc::sdesc_sw128(wa + 0 * 16384 + sub * 32), b2, id1, first);
                tp::mma2_w(d2, tc::sdesc_sw128(wa + 2 * 16384 + sub * 32), b01, id1, 1u);
              }
              tp::commit2_w(&wempty[s]);
            }
            tp::commit2_w(&dfull[slot]);
#ifdef FDSDF_PHASE_TIMING
            tspan += clock64() - tstart;
#endif
          }
#ifdef FDSDF_PHASE_TIMING
      if (blockIdx.x == 0 && lane == 0)
        printf("[phase] pair mma: total %lld, passes %u, wait B %.0f/pass, issue span %.0f/pass, W waits %.0f/pass\n",
               clock64() - t0, nb[0] + nb[1], (double)tb / (nb[0] + nb[1]), (double)tspan / (nb[0] + nb[1]),
               (double)tw / (nb[0] + nb[1]));
#endif
    } else if (lane == 0 && rank == 1) {
      // ---------------------------------------------------------------- stage forwarder (peer)
      uint32_t it = 0;
      const uint32_t wpeer_leader = tp::mapa(smem_u32(wpeer), 0);
      for (int64_t tile = cid; tile < a.ntiles; tile += ncl)
        for (int g = 0; g < ngemm; ++g)
          for (int slot = 0; slot < 2; ++slot)
            for (int kc = 0; kc < C::KC; ++kc, ++it) {
              const int s = (int)(it % C::NST);
              mbar_wait(&wfull[s], (it / C::NST) & 1u);
              tp::arrive_cluster(wpeer_leader + s * 8);
            }
    }
  } else if (warp == C::XW) {
    // ------------------------------------------------------------------ operand sender
    // per hand-off (tile, layer < L-2, slot), in the epilogue's order: once this CTA's B half
    // and staging block are written, send the staging block to the peer's B rows [128 rank, ..)
    if (lane == 0 && ngemm > 0) {
      const uint32_t peer_b = tp::mapa(smem_u32(Bs), rank ^ 1u) + rank * C::STG;
      const uint32_t peer_bin = tp::mapa(smem_u32(bin), rank ^ 1u);
      uint32_t ph[2] = {0u, 0u};
      for (int64_t tile = cid; tile < a.ntiles; tile += ncl)
        for (int l = 0; l < L - 2; ++l)
          for (int slot = 0; slot < 2; ++slot) {
            mbar_wait(&sready[slot], ph[slot] & 1u);
            ++ph[slot];
            tp::bulk_s2peer(peer_b + slot * C::BSLOT, Stg, C::STG, peer_bin + slot * 8);
          }
    }
  } else if (warp == C::XW + 1) {
    // ------------------------------------------------------------------ operand receiver
    // per hand-off: wait for the peer's block to land here and tell the peer at once that its
    // staging block is free; then, once this CTA's own half is written too, report this CTA's
    // B half of the slot complete to the leader's MMA thread
    if (lane == 0 && ngemm > 0) {
      const uint32_t peer_sfree = tp::mapa(smem_u32(sfree), rank ^ 1u);
      const uint32_t bfull_leader = tp::mapa(smem_u32(bfull), 0);
      uint32_t ph[2] = {0u, 0u};
#ifdef FDSDF_PHASE_TIMING
      long long t0 = clock64(), ti = 0, tr = 0, tm;
#endif
      for (int64_t tile = cid; tile < a.ntiles; tile += ncl)
        for (int l = 0; l < L - 2; ++l)
          for (int slot = 0; slot < 2; ++slot) {
#ifdef FDSDF_PHASE_TIMING
            tm = clock64();
#endif
            mbar_arrive_expect_tx(&bin[slot], C::STG);
            mbar_wait(&bin[slot], ph[slot] & 1u);
            tp::arrive_cluster(peer_sfree);
#ifdef FDSDF_PHASE_TIMING
            ti += clock64() - tm;
            tm = clock64();
#endif
            mbar_wait(&sready[slot], ph[slot] & 1u);
#ifdef FDSDF_PHASE_TIMING
            tr += clock64() - tm;
#endif
            ++ph[slot];
            tp::arrive_cluster(bfull_leader + slot * 8);
          }
#ifdef FDSDF_PHASE_TIMING
      if (blockIdx.x < 2)
        printf("[phase] pair receiver rank %u: total %lld, %u hand-offs, waiting for the peer block %.0f, then "
               "for the own half %.0f per hand-off\n",
               rank, clock64() - t0, ph[0] + ph[1], (double)ti / (ph[0] + ph[1]), (double)tr / (ph[0] + ph[1]));
#endif
    }
  } else {
    // ------------------------------------------------------------------ epilogue warps
    const int ew = warp - 2;                          // 0..15
    const int et = tid - 64;                          // 0..511
    const int q4 = warp & 3;                          // TMEM lane quarter
    const int eg = ew >> 2;                           // centre group 0..3
    const int ml = 32 * q4 + lane;                    // neuron within this CTA's half
    const int m = 128 * (int)rank + ml;               // output neuron (= next layer's K index)
    const uint32_t tl = tbase + ((uint32_t)(32 * q4) << 16);
    const float beta = net.beta;
    const float h = a.h;
    const bool step = a.step != 0;
    const uint32_t red_c[2] = {tp::mapa(smem_u32(red0), 0), tp::mapa(smem_u32(red0), 1)};
    const uint32_t rfull_c[2] = {tp::mapa(smem_u32(rfull), 0), tp::mapa(smem_u32(rfull), 1)};
    uint32_t nd[2] = {0u, 0u}, rph[4] = {0u, 0u, 0u, 0u}, nhand = 0;
    PhaseTimer ptimer;
    ptimer.start();
    double lacc[NLOSS];
#pragma unroll
    for (int q = 0; q < NLOSS; ++q) lacc[q] = 0.0;

    // this thread's stored pre-activations (kernels.cuh zf layout): float4 group g (step), the
    // centre value z (step: in group 0; eval: z only, contiguous over m)
    auto zg4 = [&](int64_t c, int l, int g) -> float4* {
      return reinterpret_cast<float4*>(a.zf + ((size_t)c * nh + l) * NCOLF * MPAD + (size_t)g * 4 * MPAD) + m;
    };
    auto zc = [&](int64_t c, int l) -> float* {
      return a.zf + ((size_t)c * nh + l) * a.zcols * MPAD + (step ? 4 * m : m);
    };
    // 8 accumulator columns [c8, c8 + 8) of a slot (pair-wide column numbers, within one owner
    // CTA's 32): R01 holds owner o's columns as [o][b0 | b1 products][32], R2 as [o][32]
    auto ld_x8 = [&](int slot, int c8, float (&v)[8]) {
      const int o = c8 / NH, lc = c8 % NH;
      const uint32_t t01 = tl + slot * C::DSL + (uint32_t)(o * 2 * NH + lc);
      const uint32_t t2 = tl + slot * C::DSL + (uint32_t)(2 * NS + o * NH + lc);
      float r1[8], r2[8];
      tc::tmem_ld8(t01, v);
      tc::tmem_ld8(t01 + NH, r1);
      tc::tmem_ld8(t2, r2);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += r1[j] + r2[j];
    };

    // per-centre epilogue of the centres this CTA owns in (tile base c0, parity par)
    auto finish = [&](int64_t c0, int par) {
      if (ew == 0) {
        for (int slot = 0; slot < 2; ++slot) {
          tp::wait_cluster(&rfull[par * 2 + slot], rph[par * 2 + slot] & 1u);
          ++rph[par * 2 + slot];
        }
        if (et < 2 * C::COWN) {
          const int slot = et / C::COWN;
          const int cl = (int)rank * C::COWN + et % C::COWN;  // centre within the slot
          const int64_t c = c0 + slot * CPS + cl;
          const bool valid = c < a.n;
          const float* red = red0 + (par * 2 + slot) * C::NRED;
          float tot[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float v = 0.f;
            for (int grp = 0; grp < 8; ++grp) v += red[(grp * CPS + cl) * 4 + j];
            tot[j] = v;
          }
          if (MODE == 1) {
            float ci[NCINFO];
            centre_frame(a, c, valid, tot[0] + net.b[L - 1][0], tot[1], tot[2], tot[3], ci);
            if (valid) {
#pragma unroll
              for (int q = 0; q < NCINFO; ++q) a.cinfo[c * NCINFO + q] = ci[q];
            }
          } else {
            const float* ci = cis0 + ((par * 2 + slot) * CPS + cl) * NCINFO;
            double lv[NLOSS];
            fd_centre(a, c, valid, tot, ci, lv);
#pragma unroll
            for (int q = 0; q < NLOSS; ++q) lvs[et * NLOSS + q] = lv[q];
          }
        }
        __syncwarp();
        if (MODE == 2 && et == 0) {  // fixed order: slot 0 centres, then slot 1
          for (int s2 = 0; s2 < 2 * C::COWN; ++s2)
#pragma unroll
            for (int q = 0; q < NLOSS; ++q) lacc[q] += lvs[s2 * NLOSS + q];
        }
      }
    };

    bool pending = false;
    int64_t pend_c0 = 0;
    int pend_par = 0, par = 0;
    for (int64_t tile = cid; tile < a.ntiles; tile += ncl, par ^= 1) {
      const int64_t c0 = tile * 2 * CPS;
      float* cisp = cis0 + par * 2 * CPS * NCINFO;
      if (MODE == 2) {  // both slots' centre info (frames) from the centre kernel
        for (int i = et; i < 2 * CPS * NCINFO; i += C::NEPI * 32) {
          const int64_t c = c0 + i / NCINFO;
          cisp[i] = c < a.n ? a.cinfo[c * NCINFO + (i % NCINFO)] : 0.f;
        }
      }
      bar_named(1, C::NEPI * 32);

      for (int l = 0; l <= L - 2; ++l) {
        const bool last = (l == L - 2);
        const int M = net.width[l + 1];
        const float om = net.omega[l];
        const bool mok = m < M;
        const float wl = (last && mok) ? net.W[L - 1][m] : 0.f;
        for (int slot = 0; slot < 2; ++slot) {
          const int64_t cs = c0 + slot * CPS;
          // the pre-activations the backward needs, stored after the hand-off below
          // (arrays indexed by the processing position jj; centre i = pos_i(jj))
          auto pos_i = [&](int jj) { return rank ? (jj + CPT / 2) % CPT : jj; };
          float zst[CPT][8];
          float z0n[CPT];
#pragma unroll
          for (int jj = 0; jj < CPT; ++jj) {
            const int64_t c = cs + eg + 4 * pos_i(jj);
            z0n[jj] = (MODE == 2 && c < a.n) ? __ldg(zc(c, l)) : 0.f;
          }
          if (l > 0) {
            ptimer.before_wait();
            mbar_wait(&dfull[slot], nd[slot] & 1u);
            ptimer.after_wait();
            ++nd[slot];
            tc::fence_after();
          }
          unsigned char* bsl = Bs + slot * C::BSLOT;
          // B of (slot, l+1): own columns into this CTA's B block, the peer's into the staging
          // block.  Of this thread's centres eg + 4i, the first CPT/2 are owned by CTA 0: the
          // locally owned ones go first, so the staging block (free once the peer has received
          // the previous hand-off) is waited for only after half of the work.  Register arrays
          // are indexed by the (unrolled) position jj, the centre is i.
#pragma unroll
          for (int jj = 0; jj < CPT; ++jj) {
            const int i = pos_i(jj);
            if (!last && jj == CPT / 2) {
              mbar_wait(sfree, (nhand & 1u) ^ 1u);
              ++nhand;
            }
            const int cl = eg + 4 * i;           // centre within the slot
            const int64_t c = cs + cl;
            const bool valid = c < a.n;
            float outv[8];
            if (MODE == 1) {
              float z = 0.f, t0 = 0.f, t1 = 0.f, t2 = 0.f;
              if (l == 0) {
                float x0 = 0.f, x1 = 0.f, x2 = 0.f;
                if (valid) {
                  x0 = a.x[c * 3 + 0];
                  x1 = a.x[c * 3 + 1];
                  x2 = a.x[c * 3 + 2];
                  if (m == 0 && !(isfinite(x0) && isfinite(x1) && isfinite(x2))) atomicOr(a.dflags, 1u);
                }
                if (mok) {
                  const float* W0 = net.W[0];
                  const float w0 = W0[m * 3 + 0], w1 = W0[m * 3 + 1], w2 = W0[m * 3 + 2];
                  z = om * (fmaf(w0, x0, fmaf(w1, x1, w2 * x2)) + net.b[0][m]);
                  t0 = om * w0;
                  t1 = om * w1;
                  t2 = om * w2;
                }
              } else {
                float v[8];
                ld_x8(slot, (cl >> 1) * 8, v);
                const int o = (cl & 1) * 4;
                if (mok) {
                  z = om * (v[o] + net.b[l][m]);
                  t0 = om * v[o + 1];
                  t1 = om * v[o + 2];
                  t2 = om * v[o + 3];
                }
              }
              zst[jj][0] = z;
              zst[jj][1] = t0;
              zst[jj][2] = t1;
              zst[jj][3] = t2;
              float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
              if (mok) {
                const typename AF::C cc = AF::centre(z, beta);
                const float s1 = AF::d1(cc, beta);
                o0 = AF::value(cc, beta);
                o1 = s1 * t0;
                o2 = s1 * t1;
                o3 = s1 * t2;
              }
              outv[0] = o0;
              outv[1] = o1;
              outv[2] = o2;
              outv[3] = o3;
            } else {
              const float* ci = cisp + (slot * CPS + cl) * NCINFO;
              float Av[4] = {0.f, 0.f, 0.f, 0.f}, Sv[4] = {0.f, 0.f, 0.f, 0.f};
              if (l == 0) {
                if (mok) {
                  const float* W0 = net.W[0];
                  const float w0 = W0[m * 3 + 0], w1 = W0[m * 3 + 1], w2 = W0[m * 3 + 2];
                  const float du = fmaf(w0, ci[4], fmaf(w1, ci[5], w2 * ci[6]));
                  const float dv = fmaf(w0, ci[7], fmaf(w1, ci[8], w2 * ci[9]));
                  const float hs = om * h;
                  Av[0] = hs * du;
                  Av[1] = hs * dv;
                  Av[2] = hs * (du + dv);
                  Av[3] = hs * (du - dv);
                }
              } else {
                float v[8];
                ld_x8(slot, cl * 8, v);
                if (mok) {
#pragma unroll
                  for (int p = 0; p < 4; ++p) {
                    Av[p] = om * v[2 * p];
                    Sv[p] = om * v[2 * p + 1];
                  }
                }
              }
              const float z0 = z0n[jj];
#pragma unroll
              for (int p = 0; p < 4; ++p) {
                zst[jj][2 * p] = Av[p];
                zst[jj][2 * p + 1] = Sv[p];
              }
#pragma unroll
              for (int p = 0; p < 8; ++p) outv[p] = 0.f;
              if (mok) {
                const typename AF::C cc = AF::centre(z0, beta);
#pragma unroll
                for (int p = 0; p < 4; ++p) AF::pair_fwd(cc, Av[p], Sv[p], beta, &outv[2 * p], &outv[2 * p + 1]);
              }
            }
            const int owner = (cl * CPC) / NH;  // CTA holding this centre's columns
            if (!last) {
              const int nl0 = (cl * CPC) % NH;
              if (owner == (int)rank) {
#pragma unroll
                for (int j = 0; j < CPC; ++j) tp::put_b_local<NH>(bsl, nl0 + j, m, outv[j]);
              } else {
#pragma unroll
                for (int j = 0; j < CPC; ++j) tp::put_b_local<NH>(Stg, nl0 + j, ml, outv[j]);
              }
            } else {
              // last layer: this warp's 32-neuron sums of w_L * (values), into the owner's block
              float pv[4];
              if (MODE == 1) {
                pv[0] = wl * outv[0];
                pv[1] = wl * outv[1];
                pv[2] = wl * outv[2];
                pv[3] = wl * outv[3];
              } else {
                pv[0] = wl * outv[1];
                pv[1] = wl * outv[3];
                pv[2] = wl * outv[5];
                pv[3] = wl * outv[7];
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float v = pv[j];
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                if (lane == 0) {
                  const int grp = (int)rank * 4 + q4;
                  tp::st_f32(red_c[owner] + (uint32_t)((((par * 2 + slot) * 8 + grp) * CPS + cl) * 4 + j) * 4, v);
                }
              }
            }
          }
          if (l > 0) ptimer.end_b();
          if (!last) {  // this warp's part of (slot, l+1)'s B half and staging block is written
            tc::fence_before();
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sready[slot]);
          } else {
            if (l > 0) tc::fence_before();
            __syncwarp();
            if (lane == 0) {  // partial sums in place (both owners)
              tp::arrive_cluster(rfull_c[0] + (par * 2 + slot) * 8);
              tp::arrive_cluster(rfull_c[1] + (par * 2 + slot) * 8);
            }
          }
#pragma unroll
          for (int jj = 0; jj < CPT; ++jj) {  // the deferred pre-activation stores
            const int64_t c = cs + eg + 4 * pos_i(jj);
            if (c < a.n) {
              if (MODE == 1) {
                if (step)
                  *zg4(c, l, 0) = make_float4(zst[jj][0], zst[jj][1], zst[jj][2], zst[jj][3]);
                else
                  *zc(c, l) = zst[jj][0];
              } else if (step) {
                *zg4(c, l, 1) = make_float4(zst[jj][0], zst[jj][1], zst[jj][2], zst[jj][3]);
                *zg4(c, l, 2) = make_float4(zst[jj][4], zst[jj][5], zst[jj][6], zst[jj][7]);
              }
            }
          }
          if (l == 0 && slot == 1 && pending) {  // previous tile's per-centre work, during this MMA phase
            finish(pend_c0, pend_par);
            pending = false;
          }
        }
      }
      pending = true;
      pend_c0 = c0;
      pend_par = par;
    }
    if (pending) finish(pend_c0, pend_par);
    ptimer.report(MODE == 1 ? "fwd_tc2 centre" : "fwd_tc2 pairs", (et == 0 || et == 480) && rank == 0);
    if (MODE == 2 && et == 0) {
#pragma unroll
      for (int q = 0; q < NLOSS; ++q) a.lossp[(size_t)blockIdx.x * NLOSS + q] = lacc[q];
    }
  }

  tc::fence_before();
  tp::cluster_sync();
  if (warp == 1) tp::tmem_dealloc2(tbase, C::TCOLS);
}

template <int ACT, int MODE>
static cudaError_t launch_fwd_tc2_t(const FwdArgs& a, int grid, cudaStream_t st) {
  using C = F2Cfg<MODE>;
  auto k = fwd_tc2_kernel<ACT, MODE>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::BYTES);
  if (e != cudaSuccess) return e;
  k<<<grid, C::NTHR, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

// grid: an even number of CTAs (clusters of 2)
cudaError_t launch_fwd_tc2(const FwdArgs& a, int mode, int grid, cudaStream_t st) {
  const int act = a.net.act;
  if (a.net.mpad != 256 || a.net.L < 3) return cudaErrorInvalidValue;
  if (act == ACT_SINE && mode == 1) return launch_fwd_tc2_t<ACT_SINE, 1>(a, grid, st);
  if (act == ACT_SINE && mode == 2) return launch_fwd_tc2_t<ACT_SINE, 2>(a, grid, st);
  if (act == ACT_SOFTPLUS && mode == 1) return launch_fwd_tc2_t<ACT_SOFTPLUS, 1>(a, grid, st);
  if (act == ACT_SOFTPLUS && mode == 2) return launch_fwd_tc2_t<ACT_SOFTPLUS, 2>(a, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace fdsdf
