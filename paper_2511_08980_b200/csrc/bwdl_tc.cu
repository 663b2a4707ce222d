// bwdl_tc.cu -- the backward through every stencil evaluation on the tensor
// cores for the networks the fused backward (bwd_tc.cu) does not cover: 512-wide layers and the
// skip layer (C3, the FD-NSH configuration of PAPER.md L117-127).  One launch per hidden layer
// l, top-down:
//   X_l = omega_l W_{l+1}^T delta_{l+1}      tcgen05 bf16x6 GEMM: A = the packed W^T image
//                                             (pack_tc_kernel, omega folded in), B = delta_{l+1}
//                                             read back from the workspace and split into bf16
//                                             pieces by two stager warps, K-chunk by K-chunk
//   delta_l, a_l = adjoint maps (act.cuh)     epilogue: thread = neuron of layer l, the same
//                                             per-neuron algebra as the FFMA kernel bwd.cu
// The top layer (l = L-2) has no GEMM: X = omega W_{L-1} * the output seeds.  Tile = 8 centres
// x 10 adjoint columns (N = 80); D = MPAD/128 M-halves x 80 TMEM columns.  The kernel writes
// delta_l (l >= 1) and the layer's activations a_l (l <= L-3; the skip input cat(a, x)/sqrt(2))
// in the layouts of the weight-gradient kernel, and per (CTA, centre group) slot the fixed-order
// sums of db_l, dW_last (top), db_last (top) and dW_0 (l = 0) for the finalize kernel.
#include <algorithm>
#include <cuda.h>  // CUtensorMap (the encode entry point is fetched from the driver at run time)

#include "act.cuh"
#include "tcmlp.cuh"
#include "tcpair.cuh"

#ifdef FDSDF_BWDL_TRACE
#define BL_TRACE(fmt, ...) \
  if (blockIdx.x < 2) printf("b%d " fmt, (int)blockIdx.x, ##__VA_ARGS__)
#else
#define BL_TRACE(...)
#endif

// 1: the producer thread bulk-prefetches the next tile's stored pre-activations into L2 while
// the current tile runs (the epilogue's loads then hit L2)
#ifndef BWDL_PF
#define BWDL_PF 0
#endif

// M-half passes per tile (single-CTA kernel): 2 = the MMAs of the second half of the output
// neurons run while the epilogue warps of the first half consume theirs (and the next tile's
// first pass overlaps the second half's epilogue); each pass re-stages the tile's delta chunks
// (L2 hits)
#ifndef BWDL_PASSES
#define BWDL_PASSES 2
#endif

// 512-wide layers on CTA pairs (tcgen05 cta_group::2, tcpair.cuh): a tile is 16 centres (MMA
// N = 160), CTA r stages the delta rows of centres [8 r, 8 r + 8) and streams only the weight
// rows of its M-halves 2 ps + r; pass ps = one M = 256 block.  Per SM that halves the shared-
// memory reads per MAC of the single-CTA form (whose N = 80 MMAs are bound by the A + B
// operand reads, not by the tensor pipe) and quarters the weight stream per centre.
#ifndef BWDL_PAIR
#define BWDL_PAIR 1
#endif

namespace fdsdf {

template <int MPAD, bool PAIR>
struct BlCfg {
  static constexpr int MH = MPAD / 128, KC = MPAD / 64;
  static constexpr int CT = 8, NT = CT * NCOLB;         // centres / B rows staged per CTA and tile
  static constexpr int CTT = PAIR ? 2 * CT : CT;        // centres per tile (both CTAs of a pair)
  static constexpr int NTT = CTT * NCOLB;               // MMA N = accumulator columns per M-half
  static constexpr int EPI0 = 4, NEPI = 16;             // warps 0..3 control, 4..19 epilogue
  static constexpr int NTHR = (EPI0 + NEPI) * 32;
  static constexpr int NSTGT = 64;                      // stager threads (warps 2, 3)
  static constexpr int NPASS = PAIR ? MH / 2 : BWDL_PASSES;  // passes per tile
  static constexpr int HPP = PAIR ? 1 : MH / NPASS;     // M-halves of this CTA per pass
  static constexpr int WPP = NEPI / NPASS;              // epilogue warps per pass
  static constexpr int EG = WPP / (4 * HPP);            // centre groups (accumulator slots per CTA)
  static constexpr int CPE = CTT / EG;                  // centres per epilogue thread
  static constexpr int WSTAGE = 16384, NWST = 6;        // weight ring: single-piece stages
  static constexpr int BPIECE = NT * 128;               // one bf16 piece of a 64-K chunk of the tile
  static constexpr int BSTAGE = 3 * BPIECE;
  static constexpr int NBST = 2;
  static constexpr int RSTAGE = NT * 64 * 4;            // raw fp32 delta of one 64-K chunk (2-D TMA box)
  static constexpr int NRST = 2;
  static constexpr int OFF_W = 0;
  static constexpr int OFF_B = NWST * WSTAGE;
  static constexpr int OFF_R = OFF_B + NBST * BSTAGE;
  static constexpr int OFF_SD = OFF_R + NRST * RSTAGE;  // float [NPASS][2][CTT][20]: seeds + x
  static constexpr int OFF_BAR = OFF_SD + NPASS * 2 * CTT * 20 * 4;
  // wfull, wempty, wpeer, bfull, bempty, rfull, rempty, dfull[NPASS], dfree[NPASS]
  static constexpr int NBAR = 3 * NWST + 2 * NBST + 2 * NRST + 2 * NPASS;
  static constexpr int BYTES = OFF_BAR + NBAR * 8 + 16 + 1024;
  static constexpr uint32_t TCOLS = NPASS * HPP * NTT <= 128 ? 128 : (NPASS * HPP * NTT <= 256 ? 256 : 512);
  static constexpr int REG_LAUNCH = 96, REG_CTL = 56, REG_EPI = 104;
  static_assert(EPI0 * REG_CTL + NEPI * REG_EPI <= (EPI0 + NEPI) * REG_LAUNCH, "setmaxnreg pool");
  static_assert(NPASS * HPP * NTT <= 512 && BYTES <= 232448, "TMEM / shared memory");
  static_assert(EG >= 1 && CTT % EG == 0, "centre groups");
  static_assert(NPASS >= 1 && WPP % 4 == 0 && (PAIR ? MH % 2 == 0 : MH % NPASS == 0), "passes");
};

#ifndef BWDL_PAIR256
#define BWDL_PAIR256 0
#endif
static constexpr bool bwdl_pair(int mpad) { return BWDL_PAIR && (mpad == 512 || (BWDL_PAIR256 && mpad == 256)); }
int bwdl_tc_tile_centres(int mpad) { return bwdl_pair(mpad) ? 16 : 8; }
int bwdl_tc_acc_slots(int mpad) {
  return mpad == 512 ? BlCfg<512, bwdl_pair(512)>::EG : BlCfg<256, bwdl_pair(256)>::EG;
}
bool bwdl_tc_supported(int mpad) { return mpad == 256 || mpad == 512; }
int bwdl_tc_grid(int nsm, int64_t ntiles, int mpad) {
  if (!bwdl_pair(mpad)) return (int)std::min<int64_t>(nsm, ntiles);
  return (int)(2 * std::min<int64_t>(nsm / 2, ntiles));  // clusters of 2, one pair tile each at most
}

template <int ACT, int MPAD, bool PAIR>
__global__ void __launch_bounds__(BlCfg<MPAD, PAIR>::NTHR, 1)
    bwdl_tc_kernel(const BwdArgs a, const int l, const __grid_constant__ CUtensorMap tmap) {
  using C = BlCfg<MPAD, PAIR>;
  using AF = Act<ACT>;
  constexpr int NTT = C::NTT, MH = C::MH, CT = C::CT, CTT = C::CTT, EG = C::EG, CPE = C::CPE;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw;
  sm += (1024 - (smem_u32(sm) & 1023)) & 1023;  // the same offset in both CTAs of a pair
  unsigned char* Ws = sm + C::OFF_W;
  unsigned char* Bs = sm + C::OFF_B;
  float* sds0 = reinterpret_cast<float*>(sm + C::OFF_SD);
  uint64_t* wfull = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* wempty = wfull + C::NWST;
  uint64_t* wpeer = wempty + C::NWST;  // pair leader: the peer's weight stage s is full
  uint64_t* bfull = wpeer + C::NWST;
  uint64_t* bempty = bfull + C::NBST;
  uint64_t* rfull = bempty + C::NBST;
  uint64_t* rempty = rfull + C::NRST;
  uint64_t* dfull = rempty + C::NRST;
  uint64_t* dfree = dfull + C::NPASS;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dfree + C::NPASS);

  const Net& net = a.net;
  const int L = net.L;
  const int nh = L - 1;
  const bool top = (l == L - 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nrows = a.n * NCOLB;
  const uint32_t rank = PAIR ? tp::ctarank() : 0u;
  const int64_t tile0 = PAIR ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int64_t tstep = PAIR ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
  constexpr int NCTA = PAIR ? 2 : 1;

  if (tid == 0) {
    for (int s = 0; s < C::NWST; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);  // pair: the leader's commit arrives in both CTAs
      mbar_init(&wpeer[s], 1);
    }
    for (int s = 0; s < C::NBST; ++s) {
      mbar_init(&bfull[s], NCTA * C::NSTGT / 32);  // pair: the stager warps of both CTAs (leader's)
      mbar_init(&bempty[s], 1);
    }
    for (int s = 0; s < C::NRST; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], C::NSTGT / 32);
    }
    for (int p = 0; p < C::NPASS; ++p) {
      mbar_init(&dfull[p], 1);
      mbar_init(&dfree[p], NCTA * C::WPP);  // pair: the pass's epilogue warps of both CTAs
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tp::tmem_alloc2(tslot, C::TCOLS);
    else tc::tmem_alloc(tslot, C::TCOLS);
  }
  tc::fence_before();
  if constexpr (PAIR) tp::cluster_sync();  // the peer's barriers exist before any remote arrive
  else __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *tslot;

  if (warp < C::EPI0) {
#ifndef BWDL_NOREG
    setmaxnreg_dec<C::REG_CTL>();
#endif
    if (!top) {
      if (warp == 0) {
        // ---------------------------------------------------------------- producer (lane 0)
        // per pass and K chunk: this CTA's delta_{l+1} rows of the tile (one 2-D TMA box into
        // the raw ring, split by the stagers), then the chunk's weight pieces of this CTA's
        // M-halves of the pass
        const unsigned char* img = a.wimg + (size_t)l * MPAD * MPAD * 2 * tc::WP;  // image g = l: omega_l W_{l+1}^T
        uint32_t it = 0, ir = 0;
        for (int64_t tile = lane == 0 ? tile0 : a.ntiles; tile < a.ntiles; tile += tstep)
          for (int ps = 0; ps < C::NPASS; ++ps)
            for (int kc = 0; kc < C::KC; ++kc) {
              if (BWDL_PF && kc == 0 && ps == 0) {  // the next tile's zf blocks (layer l) -> L2
                const int64_t nxt = tile + tstep;
                for (int cl = 0; cl < CTT && nxt < a.ntiles; ++cl) {
                  const int64_t c = nxt * CTT + cl;
                  if (c < a.n)
                    prefetch_l2_bulk(a.zf + ((size_t)c * nh + l) * NCOLF * MPAD,
                                     (uint32_t)(NCOLF * MPAD * sizeof(float)));
                }
              }
              {
                const int sr = (int)(ir % C::NRST);
                mbar_wait_backoff(&rempty[sr], ((ir / C::NRST) & 1u) ^ 1u);
                // one 2-D TMA box: 80 rows (this CTA's columns) x 64 K of delta_{l+1}; rows past
                // the end of the array are filled with zeros
                mbar_arrive_expect_tx(&rfull[sr], (uint32_t)C::RSTAGE);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                    "%3}], [%4];" ::"r"(smem_u32(sm + C::OFF_R + sr * C::RSTAGE)),
                    "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(kc * 64),
                    "r"((int)((tile * CTT + rank * CT) * NCOLB)), "r"(smem_u32(&rfull[sr]))
                    : "memory");
                ++ir;
              }
              for (int hl = 0; hl < C::HPP; ++hl) {
                const int h = PAIR ? 2 * ps + (int)rank : ps * C::HPP + hl;
                for (int p = 0; p < tc::WP; ++p, ++it) {
                  const int s = (int)(it % C::NWST);
                  mbar_wait_backoff(&wempty[s], ((it / C::NWST) & 1u) ^ 1u);
                  mbar_arrive_expect_tx(&wfull[s], C::WSTAGE);
                  bulk_g2s(Ws + s * C::WSTAGE, img + (((size_t)kc * MH + h) * tc::WP + p) * 16384, C::WSTAGE,
                           &wfull[s]);
                }
              }
            }
        if (lane == 0) BL_TRACE("[l%d] producer done\n", l);
      } else if (warp == 1 && rank == 0) {
        // ---------------------------------------------------------------- MMA issuer
        // per pass, K chunk, M-half and weight piece a_p: the products a_p b_j, j <= 2 - p
        // (bf16x6), all into the one accumulator range of the half (pair: M = 256, N = 160)
        constexpr uint32_t idesc = tc::idesc_bf16(PAIR ? 256 : 128, NTT);
        uint32_t it = 0, ib = 0, nt = 0;
#ifdef FDSDF_PHASE_TIMING
        long long t_all = clock64(), t_d = 0, t_b = 0, t_w = 0, t0;
#define BL_T(acc, stmt) t0 = clock64(); stmt; acc += clock64() - t0;
#else
#define BL_T(acc, stmt) stmt;
#endif
        for (int64_t tile = tile0; tile < a.ntiles; tile += tstep, ++nt)
          for (int ps = 0; ps < C::NPASS; ++ps) {
            // the pass's epilogue warps have read the previous tile's D of these halves
            if constexpr (PAIR) {
              BL_T(t_d, tp::wait_cluster(&dfree[ps], (nt & 1u) ^ 1u));
            } else {
              BL_T(t_d, mbar_wait_backoff(&dfree[ps], (nt & 1u) ^ 1u));
            }
            tc::fence_after();
            for (int kc = 0; kc < C::KC; ++kc, ++ib) {
              const int sb = (int)(ib % C::NBST);
              if constexpr (PAIR) {
                BL_T(t_b, tp::wait_cluster(&bfull[sb], (ib / C::NBST) & 1u));
              } else {
                BL_T(t_b, mbar_wait(&bfull[sb], (ib / C::NBST) & 1u));
              }
              tc::fence_after();
              const uint32_t bb = smem_u32(Bs + sb * C::BSTAGE);
              for (int hl = 0; hl < C::HPP; ++hl)
#pragma unroll
                for (int p = 0; p < tc::WP; ++p, ++it) {
                  const int s = (int)(it % C::NWST);
                  BL_T(t_w, mbar_wait(&wfull[s], (it / C::NWST) & 1u));
                  if constexpr (PAIR) tp::wait_cluster(&wpeer[s], (it / C::NWST) & 1u);
                  tc::fence_after();
                  const uint32_t wa = smem_u32(Ws + s * C::WSTAGE);
                  const uint32_t d = tbase + (ps * C::HPP + hl) * NTT;
#pragma unroll
                  for (int sub = 0; sub < 4; ++sub)
#pragma unroll
                    for (int j = 0; j < tc::WP - p; ++j) {
                      const uint64_t ad = tc::sdesc_sw128(wa + sub * 32);
                      const uint64_t bd = tc::sdesc_sw128(bb + j * C::BPIECE + sub * 32);
                      const uint32_t acc = (kc | p | j | sub) != 0 ? 1u : 0u;
                      if constexpr (PAIR) tp::mma2_w(d, ad, bd, idesc, acc);
                      else tc::mma_bf16_w(d, ad, bd, idesc, acc);
                    }
                  if constexpr (PAIR) tp::commit2_w(&wempty[s]);
                  else tc::mma_commit_w(&wempty[s]);
                }
              if constexpr (PAIR) tp::commit2_w(&bempty[sb]);
              else tc::mma_commit_w(&bempty[sb]);
            }
            if constexpr (PAIR) tp::commit2_w(&dfull[ps]);
            else tc::mma_commit_w(&dfull[ps]);
            if (lane == 0) BL_TRACE("[l%d] mma committed dfull tile %u pass %d\n", l, nt, ps);
          }
        if (lane == 0) BL_TRACE("[l%d] mma done\n", l);
#ifdef FDSDF_PHASE_TIMING
        if (blockIdx.x == 0 && lane == 0)
          printf("[phase] bwdl l%d mma: total %lld, wait D free %lld, wait B %lld, wait W %lld (%u tiles)\n", l,
                 clock64() - t_all, t_d, t_b, t_w, nt);
#endif
#undef BL_T
      } else if (warp == 1) {
        // ---------------------------------------------------------------- stage forwarder (pair peer)
        // the leader's MMAs read this CTA's weight stage s too: tell it when the stage is full
        if (PAIR && lane == 0) {
          const uint32_t wpeer_leader = tp::mapa(smem_u32(wpeer), 0);
          uint32_t it = 0;
          for (int64_t tile = tile0; tile < a.ntiles; tile += tstep)
            for (int q = 0; q < C::NPASS * C::KC * C::HPP * tc::WP; ++q, ++it) {
              const int s = (int)(it % C::NWST);
              mbar_wait(&wfull[s], (it / C::NWST) & 1u);
              tp::arrive_cluster(wpeer_leader + s * 8);
            }
        }
      } else {
        // ---------------------------------------------------------------- B stagers (warps 2, 3)
        // the raw fp32 rows of one 64-K chunk -> per (column n, 8 K) the exact bf16x3 split, one
        // 16-byte store per piece (K-major SW128); rows of centres past n are zeros
        const int st = tid - 64;
        const uint32_t bfull_leader = PAIR ? tp::mapa(smem_u32(bfull), 0) : 0u;
        uint32_t ib = 0;
        for (int64_t tile = tile0; tile < a.ntiles; tile += tstep)
          for (int ps = 0; ps < C::NPASS; ++ps)
            for (int kc = 0; kc < C::KC; ++kc, ++ib) {
              const int sb = (int)(ib % C::NBST), sr = (int)(ib % C::NRST);
              mbar_wait(&rfull[sr], (ib / C::NRST) & 1u);
              mbar_wait(&bempty[sb], ((ib / C::NBST) & 1u) ^ 1u);
              const float* raw = reinterpret_cast<const float*>(sm + C::OFF_R + sr * C::RSTAGE);
              unsigned char* dst = Bs + sb * C::BSTAGE;
              const int64_t cown = tile * CTT + rank * CT;  // this CTA's first centre
              const int nrow = (int)(a.n - cown <= 0 ? 0 : (a.n - cown < CT ? a.n - cown : CT)) * NCOLB;
              for (int item = st; item < C::NT * 8; item += C::NSTGT) {
                const int n = item >> 3, q = item & 7;
                float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
                if (n < nrow) {
                  const float4* src = reinterpret_cast<const float4*>(raw + n * 64 + q * 8);
                  v0 = src[0];
                  v1 = src[1];
                }
                uint32_t w[4][3];
                tc::split3x2(v0.x, v0.y, w[0]);
                tc::split3x2(v0.z, v0.w, w[1]);
                tc::split3x2(v1.x, v1.y, w[2]);
                tc::split3x2(v1.z, v1.w, w[3]);
                const uint32_t off = tc::sw128_off(n, q * 8, C::NT);
#pragma unroll
                for (int p = 0; p < tc::WP; ++p)
                  *reinterpret_cast<uint4*>(dst + p * C::BPIECE + off) = make_uint4(w[0][p], w[1][p], w[2][p], w[3][p]);
              }
              fence_proxy_async();
              __syncwarp();
              if (lane == 0) {
                if constexpr (PAIR) tp::arrive_cluster(bfull_leader + sb * 8);
                else mbar_arrive(&bfull[sb]);
                mbar_arrive(&rempty[sr]);
              }
            }
        if (lane == 0) BL_TRACE("[l%d] stager warp %d done\n", l, warp);
      }
    }
  } else {
#ifndef BWDL_NOREG
    setmaxnreg_inc<C::REG_EPI>();
#endif
    // ------------------------------------------------------------------ epilogue warps
    // pass group ps = WPP warps; in it, warp = (lane quarter q4, M-half hl, centre group eg)
    const int ew = warp - C::EPI0;
    const int ps = ew / C::WPP, et = tid - 32 * (C::EPI0 + ps * C::WPP);  // pass group, thread in it
    const int q4 = warp & 3;
    const int hl = ((ew % C::WPP) >> 2) % C::HPP;
    const int eg = ((ew % C::WPP) >> 2) / C::HPP;
    const int hh = PAIR ? 2 * ps + (int)rank : ps * C::HPP + hl;
    const int m = hh * 128 + 32 * q4 + lane;  // neuron of layer l
    const uint32_t taddr = tbase + ((uint32_t)(32 * q4) << 16) + (ps * C::HPP + hl) * NTT;
    const uint32_t dfree_leader = PAIR ? tp::mapa(smem_u32(dfree), 0) : 0u;
    const int M = net.width[l + 1];
    const bool mok = m < M;
    const bool nskip = (l + 1 == net.skip);
    const float xsc = nskip ? 0.70710678118654752f : 1.0f;  // d(layer input)/d(a): cat(a, x)/sqrt(2)
    const float beta = net.beta;
    const float h = a.h;
    // top layer: X = omega_l W_{L-1}[m] * (output seeds)
    const float wtop = (top && mok) ? net.omega[l] * net.W[L - 1][m] : 0.f;
    float r_db = 0.f, r_dWL = 0.f, r_dbL = 0.f, r_w0[3] = {0.f, 0.f, 0.f};
    uint32_t nt = 0;
    for (int64_t tile = tile0; tile < a.ntiles; tile += tstep, ++nt) {
      const int64_t c0 = tile * CTT;
      float* sds = sds0 + (ps * 2 + (nt & 1u)) * CTT * 20;
      for (int i = et; i < CTT * 20; i += C::WPP * 32) {
        const int cl = i / 20, q = i % 20;
        const int64_t c = c0 + cl;
        float v = 0.f;
        if (c < a.n && q < NSEED) v = a.seed[c * NSEED + q];
        else if (c < a.n && q >= 16 && q < 19) v = a.x[c * 3 + (q - 16)];
        sds[i] = v;
      }
      bar_named(1 + ps, C::WPP * 32);
      if (et == 0) BL_TRACE("[l%d] epilogue tile %u\n", l, nt);
      // this thread's stored forward pre-activations (z, t | A, S pairs) of centre i, loaded one
      // centre ahead of its use
      auto ldz = [&](int i, float4 (&g)[3]) {
        const int64_t c = c0 + eg + EG * i;
        g[0] = g[1] = g[2] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < CPE && c < a.n && mok) {
          const float4* zq = reinterpret_cast<const float4*>(a.zf + ((size_t)c * nh + l) * NCOLF * MPAD) + m;
          g[0] = __ldg(zq);
          g[1] = __ldg(zq + MPAD);
          g[2] = __ldg(zq + 2 * MPAD);
        }
      };
      float4 gn[3];
      ldz(0, gn);
      if (!top) {
        if (et < 32) mbar_wait(&dfull[ps], nt & 1u);
        bar_named(1 + C::NPASS + ps, C::WPP * 32);
        tc::fence_after();
      }
#pragma unroll 1
      for (int i = 0; i < CPE; ++i) {
        const int cl = eg + EG * i;
        const int64_t c = c0 + cl;
        const bool valid = c < a.n;
        const float4 g0 = gn[0], g1 = gn[1], g2 = gn[2];
        ldz(i + 1, gn);
        const float* sd = sds + cl * 20;
        const float dL[NCOLB] = {sd[0], valid ? 1.f : 0.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
        float X[NCOLB];
        if (top) {
#pragma unroll
          for (int j = 0; j < NCOLB; ++j) X[j] = wtop * dL[j];
        } else {
          tc::tmem_ld10(taddr + cl * NCOLB, X);
#pragma unroll
          for (int j = 0; j < NCOLB; ++j) X[j] *= xsc;
        }
        const float r0 = sd[5], r1 = sd[6], r2 = sd[7];
        const float dpx[4] = {sd[8], sd[11], sd[8] + sd[11], sd[8] - sd[11]};
        const float dpy[4] = {sd[9], sd[12], sd[9] + sd[12], sd[9] - sd[12]};
        const float dpz[4] = {sd[10], sd[13], sd[10] + sd[13], sd[10] - sd[13]};
        float dl[NCOLB], pv[NCOLB];
#pragma unroll
        for (int j = 0; j < NCOLB; ++j) dl[j] = pv[j] = 0.f;
        if (valid && mok) {
          const float Av[4] = {g1.x, g1.y, g2.x, g2.y}, Sv[4] = {g1.z, g1.w, g2.z, g2.w};
          const float tr = fmaf(r0, g0.y, fmaf(r1, g0.z, r2 * g0.w));
          const typename AF::C cc = AF::centre(g0.x, beta);
          float zbar = 0.f;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            float Aa, Sa, P, Dd, Z;
            AF::pair_bwd(cc, Av[p], Sv[p], beta, &Aa, &Sa, &P, &Dd, &Z);
            const float XA = X[2 + 2 * p], XS = X[3 + 2 * p];
            dl[2 + 2 * p] = fmaf(XA, P, 2.0f * XS * Dd);
            dl[3 + 2 * p] = fmaf(0.5f * XA, Dd, XS * P);
            zbar = fmaf(XA, Dd, fmaf(XS, Z, zbar));
            pv[2 + 2 * p] = Aa * xsc;
            pv[3 + 2 * p] = Sa * xsc;
            if (top) r_dWL = fmaf(dL[2 + 2 * p], Aa, fmaf(dL[3 + 2 * p], Sa, r_dWL));
          }
          const float s1 = AF::d1(cc, beta), s2 = AF::d2(cc, beta);
          dl[0] = fmaf(X[0], s1, fmaf(s2 * tr, X[1], zbar));
          dl[1] = s1 * X[1];
          pv[0] = AF::value(cc, beta) * xsc;
          pv[1] = s1 * tr * xsc;
          if (top) r_dWL = fmaf(dL[0], pv[0], fmaf(dL[1], pv[1], r_dWL));
        } else if (valid && nskip && m < M + 3) {
          // rows M .. M+2 of the skip layer's input: the x part (value x_d, tangent r_d, pair
          // odd parts h d_p, even parts 0), no delta (x is not a parameter)
          const int d = m - M;
          pv[0] = sd[16 + d] * xsc;
          pv[1] = (d == 0 ? r0 : (d == 1 ? r1 : r2)) * xsc;
#pragma unroll
          for (int p = 0; p < 4; ++p) pv[2 + 2 * p] = h * (d == 0 ? dpx[p] : (d == 1 ? dpy[p] : dpz[p])) * xsc;
        }
        if (l == 0) {  // a^{-1}: centre -> x0, tangent -> r, pairs -> h d_p (S parts 0)
          r_w0[0] = fmaf(dl[0], sd[16], fmaf(dl[1], r0, r_w0[0]));
          r_w0[1] = fmaf(dl[0], sd[17], fmaf(dl[1], r1, r_w0[1]));
          r_w0[2] = fmaf(dl[0], sd[18], fmaf(dl[1], r2, r_w0[2]));
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            r_w0[0] = fmaf(dl[2 + 2 * p], h * dpx[p], r_w0[0]);
            r_w0[1] = fmaf(dl[2 + 2 * p], h * dpy[p], r_w0[1]);
            r_w0[2] = fmaf(dl[2 + 2 * p], h * dpz[p], r_w0[2]);
          }
        }
        if (valid) {
          if (l >= 1) {
            float* dp = a.del + ((size_t)l * nrows + (size_t)c * NCOLB) * MPAD + m;
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) __stcs(dp + j * MPAD, dl[j]);
          }
          if (l <= L - 3) {
            float* ap = a.actv + ((size_t)l * nrows + (size_t)c * NCOLB) * MPAD + m;
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) __stcs(ap + j * MPAD, pv[j]);
          }
        }
        r_db += dl[0];
        if (top && m == 0) r_dbL += dL[0];
      }
      if (!top) {
        tc::fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) tp::arrive_cluster(dfree_leader + ps * 8);
          else mbar_arrive(&dfree[ps]);
        }
      }
      bar_named(1 + ps, C::WPP * 32);  // the seeds buffer of this parity is free again
    }
    if (et == 0) BL_TRACE("[l%d] epilogue done\n", l);
    // this thread's rows of its (CTA, centre group) slot: db_l, and dW_last / db_last (top) or
    // dW_0 (l = 0); the other layers' launches write the other rows.  Pair: the rows of the
    // peer's neurons in this CTA's slot are zero.
    float* bacc = a.bacc + ((size_t)blockIdx.x * EG + eg) * a.nacc;
#pragma unroll
    for (int side = 0; side < NCTA; ++side) {
      const bool own = side == 0;
      const int mm = own ? m : m + (rank == 0 ? 128 : -128);
      bacc[(size_t)l * MPAD + mm] = own ? r_db : 0.f;
      if (top) {
        bacc[(size_t)(L - 1) * MPAD + mm] = own ? r_dWL : 0.f;
        if (mm == 0) bacc[(size_t)(L - 1) * MPAD + MPAD] = own ? r_dbL : 0.f;
      }
      if (l == 0) {
        float* w0 = bacc + (size_t)(L - 1) * MPAD + MPAD + 1 + (size_t)mm * 3;
        w0[0] = own ? r_w0[0] : 0.f;
        w0[1] = own ? r_w0[1] : 0.f;
        w0[2] = own ? r_w0[2] : 0.f;
      }
    }
  }
  if (lane == 0) BL_TRACE("[l%d] warp %d at the end barrier\n", l, warp);
  __syncwarp();  // warp 0 diverged (lane 0 = the producer): reconverge before the aligned barrier
  tc::fence_before();
  if constexpr (PAIR) {
    tp::cluster_sync();  // no multicast commit / remote arrive still targets either CTA
    if (warp == 1) tp::tmem_dealloc2(tbase, C::TCOLS);
  } else {
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tbase, C::TCOLS);
  }
  if (tid == 0) BL_TRACE("[l%d] kernel end\n", l);
}

// TMA descriptor of delta_{l+1} viewed as a 2-D fp32 array [rows = n * 10][MPAD], box 80 x 64
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <int ACT, int MPAD>
static cudaError_t launch_bwdl_tc_t(const BwdArgs& a, int l, int grid, cudaStream_t st) {
  constexpr bool PAIR = bwdl_pair(MPAD);
  using C = BlCfg<MPAD, PAIR>;
  auto k = bwdl_tc_kernel<ACT, MPAD, PAIR>;
  if (PAIR && (grid & 1)) return cudaErrorInvalidValue;
  cudaError_t e = smem_attr_once<bwdl_tc_kernel<ACT, MPAD, PAIR>>(C::BYTES);
  if (e != cudaSuccess) return e;
  CUtensorMap tm{};
  if (l < a.net.L - 2) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)MPAD, (cuuint64_t)(a.n * NCOLB)};
    const cuuint64_t strides[1] = {(cuuint64_t)MPAD * sizeof(float)};
    const cuuint32_t box[2] = {64, (cuuint32_t)C::NT}, estr[2] = {1, 1};
    float* base = a.del + (size_t)(l + 1) * a.n * NCOLB * MPAD;
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if constexpr (PAIR) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::NTHR);
    cfg.dynamicSmemBytes = C::BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, a, l, tm);
  } else {
    k<<<grid, C::NTHR, C::BYTES, st>>>(a, l, tm);
    return cudaGetLastError();
  }
}

// the whole backward: one launch per hidden layer, top-down
cudaError_t launch_bwdl_tc(const BwdArgs& a, int grid, cudaStream_t st) {
  const int act = a.net.act, mp = a.net.mpad;
  for (int l = a.net.L - 2; l >= 0; --l) {
    cudaError_t e = cudaErrorInvalidValue;
#define FDSDF_CASE(A, MP) \
  if (act == A && mp == MP) e = launch_bwdl_tc_t<A, MP>(a, l, grid, st);
    FDSDF_CASE(ACT_SINE, 256)
    FDSDF_CASE(ACT_SINE, 512)
    FDSDF_CASE(ACT_SOFTPLUS, 256)
    FDSDF_CASE(ACT_SOFTPLUS, 512)
#undef FDSDF_CASE
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fdsdf
