// bwd_tc.cu -- the backward through every stencil evaluation on the tensor cores
// (bf16x6, tc.cuh / DESIGN.md §4b).  Same adjoint algebra as the FFMA
// kernel bwd.cu (act.cuh backward maps), on the warp-specialised engine of tcmlp.cuh.
//
// Tile = 8 centres x 10 adjoint columns (centre value, tangent along r = dL/dg, and the 4
// pairs (A, S)), N = 80.  Top-down over the hidden layers:
//   X_l = W_{l+1}^T delta_{l+1}           tcgen05: A operand = packed W^T (bwd image),
//                                          B operand = delta_{l+1} (bf16x3, written below)
//   delta_l = omega_l * activation-backward(z_l, X_l)    epilogue thread = neuron of layer l
// The epilogue writes delta_l and the layer inputs of every column for the weight-gradient
// contraction, the next B operand, and accumulates -- each thread for its own neuron, in
// fixed tile order -- the bias gradients, dW of the last layer (fan-out 1) and of the first
// layer (fan-in 3).
// Schedule per layer: phase A (X-independent, while the layer's MMA runs: the pair maps'
// derivative factors into spare TMEM columns, the layer's activations, sigma'(z) and
// sigma''(z) (r . t) handed to phase B, part of the NEXT tile's top layer, an L2 prefetch of
// the next layer's stored pre-activations), then phase B (with X: delta, its stores and the
// bf16x3 split into the next B operand).  X is accumulated in two TMEM ranges:
// a0.[b0|b1] + a1.[b0|b1] and a0.b2 + a2.b0.
#include "act.cuh"
#include "tcmlp.cuh"

namespace fdsdf {

// L2 prefetch of the stored forward pre-activations: 1 = one layer of one tile (8 x 12 KB bulk
// prefetches) issued one MMA pass before phase A reads it; 0 = none
#ifndef BWD_TC_PREFETCH
#define BWD_TC_PREFETCH 0
#endif
#ifndef BWD_TC_NEPI
#define BWD_TC_NEPI 16
#endif
// unroll of the per-centre loops of phases A and B: 1 keeps them rolled (the per-centre carry
// arrays then live in local memory); CPE (4) unrolls them, so the carries stay in registers and
// the loads of later centres can be hoisted
#ifndef BWD_TC_UNROLL
#define BWD_TC_UNROLL 4
#endif
constexpr int kBwdUnroll = BWD_TC_UNROLL;
// stores of delta / the layer activations (read once, by the weight-gradient kernel after the
// whole backward): 1 = streaming (st.global.cs, evict-first), 0 = default caching
#ifndef BWD_TC_STCS
#define BWD_TC_STCS 1
#endif
__device__ __forceinline__ void bwd_st(float* p, float v) {
  if (BWD_TC_STCS)
    __stcs(p, v);
  else
    *p = v;
}
// B / D column of (centre cl, adjoint column j) = 8 j + cl: the SW128 row group of column j is
// j itself, so each thread writes a centre's ten B columns at one base offset plus compile-time
// offsets j * 1024 (no per-element swizzle arithmetic)
// 1: the top layer of tile t+1 (adjoint seeds -> delta_{L-2}; needs no MMA) is computed during
// tile t's MMA phases and parked in the delta buffer, so a tile starts with a reload + split
// instead of a full epilogue pass with the tensor cores idle.
#ifndef BWD_TC_PIPE_TOP
#define BWD_TC_PIPE_TOP 1
#endif
// 1: phase A hands sigma'(z) and sigma''(z) (r . t) of each centre to phase B
// in a small per-thread array, instead of phase B reloading z, t and recomputing sincos(z)
// 1: one epilogue warp polls "D full", the others wait in a named barrier (no spinning warps
// beside the ones still in phase A)
#ifndef BWD_TC_POLL1
#define BWD_TC_POLL1 0
#endif
// back-off between the per-warp polls (ns; 0 = try_wait with a suspend-time hint only)
#ifndef BWD_TC_POLL_NS
#define BWD_TC_POLL_NS 0
#endif
// unroll of phase B's M-block loop (1: one copy of the phase-B code for both halves)
#ifndef BWD_TC_BUNROLL
#define BWD_TC_BUNROLL 1
#endif
constexpr int kBwdBUnroll = BWD_TC_BUNROLL;
#ifndef BWD_TC_CARRY
#define BWD_TC_CARRY 1
#endif
// The X GEMM accumulates in two TMEM ranges (a0.[b0|b1] + a1.[b0|b1], a0.b2 + a2.b0: four A
// reads per K step), which leaves room for a stash of the 12 derivative factors per centre
constexpr int BWD_SV = 12;  // stashed values per centre: P, Dd, Z of the 4 pairs
// TMEM stash: (MH x EG thread groups) x (centres per thread) x BWD_SV values
#define BWD_TC_STASH(MPAD) ((BWD_TC_NEPI / 4) * (8 / (BWD_TC_NEPI / (4 * ((MPAD) / 128)))) * BWD_SV)
// M-half pipelining of the 256-wide layers (tcmlp.cuh TcCfg::HP): phase B of M-half 0 runs
// while the MMAs of output half 1 are in flight, and half 1's while the next layer's first group runs
#ifndef BWD_TC_HP
#define BWD_TC_HP 0
#endif
constexpr int bwd_tc_hp(int mpad) { return (BWD_TC_HP && mpad == 256) ? 1 : 0; }
template <int MPAD>
struct BtcCfg : TcCfg<MPAD, 80, BWD_TC_NEPI, 2, BWD_TC_STASH(MPAD), 1, 0, 6, bwd_tc_hp(MPAD)> {
  using B = TcCfg<MPAD, 80, BWD_TC_NEPI, 2, BWD_TC_STASH(MPAD), 1, 0, 6, bwd_tc_hp(MPAD)>;
  static constexpr int CT = 8;                                      // centres per tile
  static constexpr int OFF_SD = B::OFF_X;                           // float [2][CT][20]: seeds + x
  static constexpr int OFF_BAR = OFF_SD + 2 * CT * 20 * 4;
  static constexpr int BYTES = OFF_BAR + tc_bars_bytes<B>() + 1024;
};

int bwd_tc_tile_centres() { return 8; }
// accumulator slots per CTA: the centre groups (EG, or NEPI / 4 under M-half pipelining)
int bwd_tc_acc_slots(int mpad) { return bwd_tc_hp(mpad) ? BWD_TC_NEPI / 4 : BWD_TC_NEPI / (4 * (mpad / 128)); }

template <int ACT, int MPAD>
__global__ void FDSDF_TC_CLUSTER __launch_bounds__(BtcCfg<MPAD>::NTHR, 1) bwd_tc_kernel(const BwdArgs a) {
  using C = BtcCfg<MPAD>;
  using AF = Act<ACT>;
  constexpr int N = C::N, MH = C::MH, CT = C::CT, EG = C::EG;
  constexpr int CPE = CT / EG;
  static_assert(CT == 8 && NCOLB == 10 && C::NSPLIT == 1 && C::RANGES == 2,
                "column permutation 8 j + cl: 8 centres x 10 columns in two accumulator ranges");
  constexpr int SV = BWD_SV;
  FDSDF_ASSERT((int)C::TCOLS >= C::MH * C::DH + C::MH * EG * CPE * SV);

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw;
  sm += (1024 - (smem_u32(sm) & 1023)) & 1023;
  unsigned char* Ws = sm + C::OFF_W;
  unsigned char* Bs = sm + C::OFF_B;
  float* sds0 = reinterpret_cast<float*>(sm + C::OFF_SD);
  const TcBars bars = tc_bars<C>(sm + C::OFF_BAR);

  const Net& net = a.net;
  const int L = net.L;
  const int nh = L - 1;
  const int ngemm = L - 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tbase = tc_setup<C>(bars);

  if (tc_is_ctl<C>(warp)) {
    // control warp group: producer (warp 0), MMA issuer (warp 1), two idle warps
    setmaxnreg_dec<C::REG_CTL>();
    if (warp == C::CTL0) {
      if (lane == 0 && ngemm > 0) tc_producer<C>(a.wimg, ngemm, 1, a.ntiles, Ws, bars);
    } else if (warp == C::CTL0 + 1) {
      if (ngemm > 0) tc_mma<C>(ngemm, a.ntiles, Ws, Bs, tbase, bars);
    }
  } else {
    setmaxnreg_inc<C::REG_EPI>();
    const int ew = warp - C::EPI0;
    const int et = tid - 32 * C::EPI0;
    const int q4 = warp & 3;
    // M-blocks (as in fwd_tc.cu): without M-half pipelining every warp owns one M-half and EG
    // centre groups split the tile; with it (C::HP) every warp walks both M-halves in turn (phase
    // B of half 0, then of half 1) and NEPI / 4 centre groups split the tile
    constexpr bool HP = C::HP;
    constexpr int NBLK = HP ? MH : 1;               // M-blocks per layer and thread
    constexpr int EGX = HP ? C::NEPI / 4 : EG;      // centre groups = accumulator slots per CTA
    constexpr int CPX = CT / EGX;                   // centres per thread and M-block
    constexpr int NIT = NBLK * CPX;                 // (M-block, centre) items per thread and layer
    static_assert(CT % EGX == 0 && NIT == CPE, "every thread handles CPE (neuron, centre) items per layer");
    const int hh0 = HP ? 0 : (ew >> 2) % MH;
    const int egx = HP ? (ew >> 2) : ew / (4 * MH);
    auto half_of = [&](int blk) { return HP ? blk : hh0; };
    auto m_of = [&](int blk) { return half_of(blk) * 128 + 32 * q4 + lane; };  // this thread's neuron
    auto taddr_of = [&](int blk) -> uint32_t {
      return tbase + ((uint32_t)(32 * q4) << 16) + half_of(blk) * C::DH;
    };
    // this thread's stash columns of M-block blk (after both halves' accumulators)
    auto tstash_of = [&](int blk) -> uint32_t {
      return tbase + ((uint32_t)(32 * q4) << 16) + C::MH * C::DH + (half_of(blk) * EGX + egx) * CPX * SV;
    };
    auto slot_of = [&](int i) { return egx + EGX * i; };  // centre slot of this thread's i-th centre
    const float beta = net.beta;
    const float h = a.h;
    const int64_t nrows = a.n * NCOLB;
    // this thread's accumulator slot (one per CTA and centre group): [L-1][MPAD] db |
    // dW_last [MPAD] | db_last [1] | dW_0 [MPAD][3]   (kernels.cuh bacc_size)
    float* bacc = a.bacc + ((size_t)blockIdx.x * EGX + egx) * a.nacc;
    float* acc_db = bacc;
    float* acc_dWL = bacc + (size_t)(L - 1) * MPAD;
    float* acc_dbL = acc_dWL + MPAD;
    float* acc_dW0 = acc_dbL + 1;
    // this thread's accumulators (its neuron of each M-block), summed over its tiles in tile
    // order and written once at the end: db per hidden layer, dW_last[m], dW_0[m][:], db_last (m == 0)
    float r_db[NBLK][MAXL];
#pragma unroll
    for (int b = 0; b < NBLK; ++b)
#pragma unroll
      for (int l = 0; l < MAXL; ++l) r_db[b][l] = 0.f;
    float r_dWL[NBLK], r_dW0[NBLK][3], r_dbtop[NBLK], r_dbL = 0.f;
#pragma unroll
    for (int b = 0; b < NBLK; ++b) r_dWL[b] = r_dbtop[b] = r_dW0[b][0] = r_dW0[b][1] = r_dW0[b][2] = 0.f;
    // += into element blk of a per-M-block register array (compile-time indices only: a runtime
    // index would move the array to local memory)
    auto addb = [&](float (&arr)[NBLK], int blk, float v) {
      if (NBLK > 1 && blk)
        arr[NBLK - 1] += v;
      else
        arr[0] += v;
    };
    uint32_t nd = 0;
    PhaseTimer ptimer;
    ptimer.start();
    // layer l of the stored forward pre-activations of tile `tile`: per centre one contiguous
    // NCOLF x MPAD block of zf (one thread issues the bulk L2 prefetches)
    auto prefetch_layer = [&](int64_t tile, int l) {
      if (BWD_TC_PREFETCH && et == 0 && tile < a.ntiles && l >= 0) {
        for (int cl = 0; cl < CT; ++cl) {
          const int64_t c = tile * CT + cl;
          if (c < a.n)
            prefetch_l2_bulk(a.zf + ((size_t)c * nh + l) * NCOLF * MPAD, (uint32_t)(NCOLF * MPAD * sizeof(float)));
        }
      }
    };

    // per-tile seeds + coordinates, double-buffered: the next tile's are copied asynchronously
    // (cp.async) while this tile runs
    auto load_seeds = [&](int64_t tile, float* dst) {
      const int64_t cb = tile * CT;
      for (int i = et; i < CT * 20; i += C::NEPI * 32) {
        const int cl = i / 20, q = i % 20;
        const int64_t c = cb + cl;
        if (tile < a.ntiles && c < a.n && q < NSEED + 3)
          cp_async4(dst + i, q < NSEED ? (const void*)(a.seed + c * NSEED + q) : (const void*)(a.x + c * 3 + (q - NSEED)));
        else
          dst[i] = 0.f;
      }
    };
    load_seeds(blockIdx.x, sds0);

    // write delta (10 columns of centre slot cl, neuron m) as the next GEMM's B operand
    auto put_b10 = [&](int m, int cl, const float (&dl)[NCOLB]) {
      FDSDF_ASSERT(cl >= 0 && cl < CT && m >= 0 && m < MPAD);
      // sw128_off(8 j + cl, m) = (m / 64) BKC + 1024 j + 128 cl + (((m % 64) / 8 ^ cl) << 4) + 2 (m % 8)
      unsigned char* bp = Bs + (m >> 6) * C::BKC + cl * 128 + ((((m & 63) >> 3) ^ cl) << 4) + ((m & 7) << 1);
      // columns j, j+1 split together (packed bf16x2 conversions on the ALU pipe instead of
      // scalar ones on the quarter-rate XU), each half stored at its own column
#pragma unroll
      for (int j = 0; j < NCOLB; j += 2) {
        uint32_t w[3];
        tc::split3x2(dl[j], dl[j + 1], w);
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          *reinterpret_cast<uint16_t*>(bp + j * 1024 + p * C::NS * 128) = (uint16_t)(w[p] & 0xFFFFu);
          *reinterpret_cast<uint16_t*>(bp + (j + 1) * 1024 + p * C::NS * 128) = (uint16_t)(w[p] >> 16);
        }
      }
    };
    // the top layer l = L-2 for centre i of M-block blk of tile tl (seeds sdsT): X = W_{L-1}^T
    // fbar-seeds, so delta_{L-2} needs no MMA.  Writes delta to a.del and accumulates db_{L-2}
    // and dW_{L-1}.
    const int ltop = L - 2;
    const bool pipe_top = BWD_TC_PIPE_TOP && ngemm > 0;
    // this thread's last-layer weights (fan-out 1), loaded once instead of per top-layer centre
    float wlast[NBLK];
#pragma unroll
    for (int b = 0; b < NBLK; ++b) wlast[b] = m_of(b) < net.width[ltop + 1] ? net.W[L - 1][m_of(b)] : 0.f;
    auto wlast_of = [&](int blk) -> float { return (NBLK > 1 && blk) ? wlast[NBLK - 1] : wlast[0]; };
    // the pair maps of a centre's 4 pairs, two pairs per packed fp32 x2 lane pair, into
    // t[5 p .. 5 p + 4] = A_a, S_a, P, Dd, Z of pair p (zero on rows past the width); every lane
    // of the warp calls this (the sine maps vote on their fast form)
    auto pair_maps = [&](const typename AF::C& cc, bool mk, const float (&A)[4], const float (&S)[4], float (&t)[20]) {
      const float2 A2[2] = {make_float2(A[0], A[1]), make_float2(A[2], A[3])};
      const float2 S2[2] = {make_float2(S[0], S[1]), make_float2(S[2], S[3])};
      float2 Aa[2], Sa[2], P[2], Dd[2], Z[2];
      AF::pairs_bwd4x2(cc, A2, S2, beta, Aa, Sa, P, Dd, Z);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        t[10 * k + 0] = mk ? Aa[k].x : 0.f;
        t[10 * k + 1] = mk ? Sa[k].x : 0.f;
        t[10 * k + 2] = mk ? P[k].x : 0.f;
        t[10 * k + 3] = mk ? Dd[k].x : 0.f;
        t[10 * k + 4] = mk ? Z[k].x : 0.f;
        t[10 * k + 5] = mk ? Aa[k].y : 0.f;
        t[10 * k + 6] = mk ? Sa[k].y : 0.f;
        t[10 * k + 7] = mk ? P[k].y : 0.f;
        t[10 * k + 8] = mk ? Dd[k].y : 0.f;
        t[10 * k + 9] = mk ? Z[k].y : 0.f;
      }
    };
    // this thread's stored pre-activations of top-layer item (blk, i) of tile tl (zero if none)
    auto top_load = [&](int64_t tl, int blk, int i, float4 (&zg)[ZG]) {
      const int m = m_of(blk);
      const int64_t c = tl * CT + slot_of(i);
#pragma unroll
      for (int g = 0; g < ZG; ++g) zg[g] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (tl >= a.ntiles || c >= a.n || m >= net.width[ltop + 1]) return;
      const float4* zq = reinterpret_cast<const float4*>(a.zf + ((size_t)c * nh + ltop) * NCOLF * MPAD) + m;
#pragma unroll
      for (int g = 0; g < ZG; ++g) zg[g] = __ldg(zq + g * MPAD);
    };
    auto top_centre = [&](int64_t tl, int blk, int i, const float* sdsT, const float4 (&zg)[ZG]) {
      const int cl = slot_of(i);
      const int64_t c = tl * CT + cl;
      if (tl >= a.ntiles || c >= a.n) return;  // warp-uniform: the pair maps below vote
      const int m = m_of(blk);
      const bool mk = m < net.width[ltop + 1];
      const float omt = net.omega[ltop];
      const float wlt = wlast_of(blk);
      FDSDF_ASSERT(c >= 0 && c < a.n);
      float zv[NCOLF];
#pragma unroll
      for (int g = 0; g < ZG; ++g) {
        const float4 v = zg[g];
        zv[4 * g] = v.x;
        zv[4 * g + 1] = v.y;
        zv[4 * g + 2] = v.z;
        zv[4 * g + 3] = v.w;
      }
      const float* sd = sdsT + cl * 20;
      const float dL[NCOLB] = {sd[0], 1.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
      const typename AF::C cc = AF::centre(zv[0], beta);
      float t[20];
      {
        const float A[4] = {zv[4], zv[5], zv[8], zv[9]}, S[4] = {zv[6], zv[7], zv[10], zv[11]};  // kernels.cuh zf
        pair_maps(cc, mk, A, S, t);
      }
      if (!mk) return;
      float dl[NCOLB], pv[NCOLB];
      float zbar = 0.f;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const float Aa = t[5 * p], Sa = t[5 * p + 1], P = t[5 * p + 2], Dd = t[5 * p + 3], Z = t[5 * p + 4];
        const float XA = wlt * dL[2 + 2 * p], XS = wlt * dL[3 + 2 * p];
        dl[2 + 2 * p] = omt * fmaf(XA, P, 2.0f * XS * Dd);
        dl[3 + 2 * p] = omt * fmaf(0.5f * XA, Dd, XS * P);
        zbar = fmaf(XA, Dd, fmaf(XS, Z, zbar));
        pv[2 + 2 * p] = Aa;
        pv[3 + 2 * p] = Sa;
      }
      const float tr = fmaf(sd[5], zv[1], fmaf(sd[6], zv[2], sd[7] * zv[3]));
      const float s1 = AF::d1(cc, beta), s2 = AF::d2(cc, beta);
      const float Xc = wlt * dL[0], Xt = wlt * dL[1];
      dl[0] = omt * fmaf(Xc, s1, fmaf(s2 * tr, Xt, zbar));
      dl[1] = omt * s1 * Xt;
      pv[0] = AF::value(cc, beta);
      pv[1] = s1 * tr;
      FDSDF_ASSERT(c >= 0 && c < a.n && ltop >= 0 && ltop < nh);
      float* dp = a.del + ((size_t)ltop * nrows + (size_t)c * NCOLB) * MPAD + m;
#pragma unroll
      for (int j = 0; j < NCOLB; ++j) bwd_st(dp + j * MPAD, dl[j]);
      float v = 0.f;
#pragma unroll
      for (int j = 0; j < NCOLB; ++j) v = fmaf(dL[j], pv[j], v);
      addb(r_dbtop, blk, dl[0]);
      addb(r_dWL, blk, v);
    };
    uint32_t spar = 0;
#ifdef FDSDF_PHASE_TIMING
    long long t_tstart = 0, t_tstart_n = 0, t_top = 0, t_pa = 0;
#endif
    const int64_t tend = tc_tile_end<C>(a.ntiles);
    // centre / layer strides of zf and of the delta / activation rows (floats): per tile one
    // 64-bit product, per centre and layer 32-bit offsets
    constexpr int ZCS_L = NCOLF * MPAD;
    const int zcs = nh * ZCS_L;
    for (int64_t tile = blockIdx.x; tile < tend; tile += gridDim.x, spar ^= 1u) {
      const int64_t c0 = tile * CT;
      const float* const zt = a.zf + (size_t)c0 * zcs;       // zf block of the tile's first centre
      const size_t drow0 = (size_t)c0 * NCOLB * MPAD;        // its first delta / activation row
      // this tile's first MMA pass reads layer L-3; the next tile's top layer (computed during
      // this tile's passes) reads layer L-2 of that tile
      if (tile == blockIdx.x) prefetch_layer(tile, L - 3);  // later tiles: during the previous tile
      prefetch_layer(tile + gridDim.x, L - 2);
      cp_async_wait_all();
      bar_named(1, C::NEPI * 32);  // this tile's seeds are in; every thread is done with the other buffer
      const float* sds = sds0 + spar * CT * 20;
      load_seeds(tile + gridDim.x, sds0 + (spar ^ 1u) * CT * 20);
      const float* sds_next = sds0 + (spar ^ 1u) * CT * 20;

#ifdef FDSDF_PHASE_TIMING
      const long long t_ts0 = clock64();
#endif
      if (pipe_top) {
        // the first GEMM's B operand: delta_{L-2} of this tile, computed during the previous
        // tile (here only for the CTA's first tile) and reloaded from a.del (this thread's
        // writes), M-block by M-block
        if (tile == blockIdx.x)
          for (int k = 0; k < NIT; ++k) {
            float4 zg[ZG];
            top_load(tile, k / CPX, k % CPX, zg);
            top_centre(tile, k / CPX, k % CPX, sds, zg);
          }
#pragma unroll
        for (int blk = 0; blk < NBLK; ++blk) {
          const int m = m_of(blk);
          const bool mt = m < net.width[ltop + 1];
          auto ldd = [&](int i, float (&d)[NCOLB]) {
            const int64_t c = c0 + slot_of(i);
            const bool ok = i < CPX && c < a.n && mt;
            const float* dp = a.del + ((size_t)ltop * nrows + (size_t)c * NCOLB) * MPAD + m;
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) d[j] = ok ? dp[j * MPAD] : 0.f;
          };
          float dn[NCOLB];
          ldd(0, dn);
#pragma unroll 1
          for (int i = 0; i < CPX; ++i) {
            float dl[NCOLB];
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) dl[j] = dn[j];
            ldd(i + 1, dn);
            put_b10(m, slot_of(i), dl);
          }
          tc_epi_arrive(bars, HP ? blk : 0);
        }
      }
#ifdef FDSDF_PHASE_TIMING
      t_tstart += clock64() - t_ts0;
      t_tstart_n += 1;
#endif

      for (int l = pipe_top ? L - 3 : L - 2; l >= 0; --l) {
        const bool top = (l == L - 2);
        const int M = net.width[l + 1];
        float s_vL[NBLK];
#pragma unroll
        for (int b = 0; b < NBLK; ++b) s_vL[b] = 0.f;
        constexpr bool CARRY = BWD_TC_CARRY;
        float c_s1[NIT], c_s2tr[NIT];  // CARRY: sigma'(z), sigma''(z) (r . t) per item of this thread
        // the next pass's phase A: layer l - 1 of this tile, or the next tile's first GEMM layer
        if (!top) prefetch_layer(l > 0 ? tile : tile + gridDim.x, l > 0 ? l - 1 : L - 3);
        // ---- phase A (X-independent, overlaps this layer's MMA): the pair maps of every
        // item of this thread -- A_a, S_a and the derivative factors P, Dd, Z -- from the
        // stored forward pre-activations, stashed in this thread's TMEM lane
        struct Zq {
          float z, t0, t1, t2, A[4], S[4];
        };
        auto ldq = [&](int k) -> Zq {
          Zq q{};
          const int blk = k / CPX, i = k % CPX;
          const int m = m_of(blk);
          const int64_t c = c0 + slot_of(i);
          if (k < NIT && c < a.n && m < M) {
            FDSDF_ASSERT(c >= 0 && c < a.n && l >= 0 && l < nh);
            const float4* zq = reinterpret_cast<const float4*>(zt + slot_of(i) * zcs + l * ZCS_L) + m;
            FDSDF_ASSERT((const float*)zq == a.zf + ((size_t)c * nh + l) * NCOLF * MPAD + 4 * m);
            const float4 g0 = __ldg(zq), g1 = __ldg(zq + MPAD), g2 = __ldg(zq + 2 * MPAD);
            q.z = g0.x;
            q.t0 = g0.y;
            q.t1 = g0.z;
            q.t2 = g0.w;
            q.A[0] = g1.x;
            q.A[1] = g1.y;
            q.S[0] = g1.z;
            q.S[1] = g1.w;
            q.A[2] = g2.x;
            q.A[3] = g2.y;
            q.S[2] = g2.z;
            q.S[3] = g2.w;
          }
          return q;
        };
        {
          Zq qn = ldq(0);
#pragma unroll kBwdUnroll
          for (int k = 0; k < NIT; ++k) {
            const Zq q = qn;
            qn = ldq(k + 1);
            const int blk = k / CPX, i = k % CPX;
            const int m = m_of(blk);
            const bool mok = m < M;
            const int cl = slot_of(i);
            const int64_t c = c0 + cl;
            const bool valid = c < a.n;
            float t[20];
#pragma unroll
            for (int j = 0; j < 20; ++j) t[j] = 0.f;
            float pv[NCOLB];
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) pv[j] = 0.f;
            float cs1 = 0.f, cs2tr = 0.f;
            typename AF::C cc{};
            if (valid) {  // every lane of the warp: the sine maps vote on their fast series form
              cc = AF::centre(q.z, beta);
              pair_maps(cc, mok, q.A, q.S, t);
            }
            if (mok && valid) {
              {  // the layer's activations (wgrad operand) are X-independent: stored here
                const float* sd = sds + cl * 20;
                const float tr = fmaf(sd[5], q.t0, fmaf(sd[6], q.t1, sd[7] * q.t2));
                pv[0] = AF::value(cc, beta);
                pv[1] = AF::d1(cc, beta) * tr;
                if (CARRY) {
                  cs1 = AF::d1(cc, beta);
                  cs2tr = AF::d2(cc, beta) * tr;
                }
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                  pv[2 + 2 * p] = t[5 * p];
                  pv[3 + 2 * p] = t[5 * p + 1];
                }
              }
            }
            if (CARRY) {
              c_s1[k] = cs1;
              c_s2tr[k] = cs2tr;
            }
            {
              if (valid && l <= L - 3) {
                FDSDF_ASSERT(c >= 0 && c < a.n && l >= 0 && l < nh);
                float* ap = a.actv + (size_t)l * nrows * MPAD + drow0 + cl * (NCOLB * MPAD) + m;
                FDSDF_ASSERT(ap == a.actv + ((size_t)l * nrows + (size_t)c * NCOLB) * MPAD + m);
#pragma unroll
                for (int j = 0; j < NCOLB; ++j) bwd_st(ap + j * MPAD, pv[j]);
              }
              if (top) {
                const float* sd = sds + cl * 20;
                const float dL[NCOLB] = {sd[0], valid ? 1.f : 0.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
                float v = 0.f;
#pragma unroll
                for (int j = 0; j < NCOLB; ++j) v = fmaf(dL[j], pv[j], v);
                addb(s_vL, blk, v);
              }
              // stash P, Dd, Z of the four pairs
              float v4[4];
#pragma unroll
              for (int kk = 0; kk < 3; ++kk) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int e = 4 * kk + j;  // (pair e / 3, factor e % 3)
                  v4[j] = t[5 * (e / 3) + 2 + e % 3];
                }
                tc::tmem_st4(tstash_of(blk) + i * SV + 4 * kk, v4);
              }
            }
          }
          tc::tmem_wait_st();
        }
#ifdef FDSDF_PHASE_TIMING
        const long long t_pa1 = clock64();
#endif
        if (pipe_top) {  // the next tile's top layer, its items spread over this tile's MMA phases
          const int g = L - 3 - l;
          if (g == 0) {
            cp_async_wait_all();
            bar_named(1, C::NEPI * 32);  // the next tile's seeds are in
          }
#pragma unroll 1
          for (int k = g; k < NIT; k += ngemm) {
            float4 zg[ZG];
            top_load(tile + gridDim.x, k / CPX, k % CPX, zg);
            top_centre(tile + gridDim.x, k / CPX, k % CPX, sds_next, zg);
          }
        }
#ifdef FDSDF_PHASE_TIMING
        t_top += clock64() - t_pa1;
#endif
        // ---- phase B (after the MMA), M-block by M-block: combine with the adjoint X
#pragma unroll kBwdBUnroll
        for (int blk = 0; blk < NBLK; ++blk) {
          const int m = m_of(blk);
          const bool mok = m < M;
          // omega_l: in the image of the GEMM that produced X (pack_tc_kernel), or (top layer
          // without an MMA) in its last-layer weight
          const float wl = (top && mok) ? wlast_of(blk) * net.omega[l] : 0.f;
          const uint32_t taddr = taddr_of(blk);
          const uint32_t tstash = tstash_of(blk);
          float s_db = 0.f, s_w0[3] = {0.f, 0.f, 0.f};
          const float db_l = r_db[blk][l];  // local-memory read issued here, consumed after phase B
          auto ldz = [&](int i, float (&z4)[4]) {
            const int64_t c = c0 + slot_of(i);
            z4[0] = z4[1] = z4[2] = z4[3] = 0.f;
            if (!CARRY && i < CPX && c < a.n && mok) {
              const float4 g0 = __ldg(reinterpret_cast<const float4*>(zt + slot_of(i) * zcs + l * ZCS_L) + m);
              z4[0] = g0.x;
              z4[1] = g0.y;
              z4[2] = g0.z;
              z4[3] = g0.w;
            }
          };
          float zn[4];
          ldz(0, zn);
          if (!top) {
            ptimer.before_wait();
            if (BWD_TC_POLL1) {  // one warp polls, the others sleep in a hardware named barrier
              if (et < 32) mbar_wait(&bars.dfull[HP ? blk : 0], nd & 1u);
              bar_named(2, C::NEPI * 32);
            } else {
              mbar_wait_sleep<BWD_TC_POLL_NS>(&bars.dfull[HP ? blk : 0], nd & 1u);
            }
            ptimer.after_wait();
            tc::fence_after();
          }
          // HP: the B rows of K half 0 may still be read by the layer's (1, 0) MMA group --
          // wait for "B free" before this M-block's first B store
          if (HP && blk == 0 && l >= 1) mbar_wait(bars.bfree, nd & 1u);
#pragma unroll
          for (int i = 0; i < CPX; ++i) {
            const int k = blk * CPX + i;
            const int cl = slot_of(i);
            const int64_t c = c0 + cl;
            const bool valid = c < a.n;
            const float zc[4] = {zn[0], zn[1], zn[2], zn[3]};
            ldz(i + 1, zn);
            const float cs1 = CARRY ? c_s1[k] : 0.f, cs2 = CARRY ? c_s2tr[k] : 0.f;
            const float* sd = sds + cl * 20;
            float X[NCOLB];
            if (top) {
              const float dL[NCOLB] = {sd[0], valid ? 1.f : 0.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
#pragma unroll
              for (int j = 0; j < NCOLB; ++j) X[j] = wl * dL[j];
            } else {  // the two accumulator ranges, columns cl + 8 j
              tc::tmem_ld10x2_stride8(taddr + cl, taddr + C::NS + cl, X);
            }
            float t[20];  // per pair: A_a, S_a, P, Dd, Z (only P, Dd, Z are stashed / used here)
            {
              float v4[4];
#pragma unroll
              for (int kk = 0; kk < 3; ++kk) {
                tc::tmem_ld4(tstash + i * SV + 4 * kk, v4);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int e = 4 * kk + j;
                  t[5 * (e / 3) + 2 + e % 3] = v4[j];
                }
              }
#pragma unroll
              for (int p = 0; p < 4; ++p) t[5 * p] = t[5 * p + 1] = 0.f;
            }
            const float r0 = sd[5], r1 = sd[6], r2 = sd[7];
            const float u0 = sd[8], u1 = sd[9], u2 = sd[10], v0 = sd[11], v1 = sd[12], v2_ = sd[13];
            float dl[NCOLB];
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) dl[j] = 0.f;
            float w0p[3] = {0.f, 0.f, 0.f};
            if (mok && valid) {
              float tr = 0.f, s1, s2tr;
              typename AF::C cc{};
              if (CARRY) {
                s1 = cs1;
                s2tr = cs2;
              } else {
                tr = fmaf(r0, zc[1], fmaf(r1, zc[2], r2 * zc[3]));
                cc = AF::centre(zc[0], beta);
                s1 = AF::d1(cc, beta);
                s2tr = AF::d2(cc, beta) * tr;
              }
              float zbar = 0.f;
#pragma unroll
              for (int p = 0; p < 4; ++p) {
                const float P = t[5 * p + 2], Dd = t[5 * p + 3], Z = t[5 * p + 4];
                const float XA = X[2 + 2 * p], XS = X[3 + 2 * p];
                const float dA = fmaf(XA, P, 2.0f * XS * Dd);
                const float dS = fmaf(0.5f * XA, Dd, XS * P);
                zbar = fmaf(XA, Dd, fmaf(XS, Z, zbar));
                dl[2 + 2 * p] = dA;
                dl[3 + 2 * p] = dS;
                if (l == 0) {  // a^{-1} of pair columns: A -> h d_p, S -> 0
                  const float dpx = p == 0 ? u0 : (p == 1 ? v0 : (p == 2 ? u0 + v0 : u0 - v0));
                  const float dpy = p == 0 ? u1 : (p == 1 ? v1 : (p == 2 ? u1 + v1 : u1 - v1));
                  const float dpz = p == 0 ? u2 : (p == 1 ? v2_ : (p == 2 ? u2 + v2_ : u2 - v2_));
                  w0p[0] = fmaf(dA, h * dpx, w0p[0]);
                  w0p[1] = fmaf(dA, h * dpy, w0p[1]);
                  w0p[2] = fmaf(dA, h * dpz, w0p[2]);
                }
              }
              const float Xc = X[0], Xt = X[1];
              const float zb = fmaf(Xc, s1, fmaf(s2tr, Xt, zbar));
              dl[0] = zb;
              dl[1] = s1 * Xt;
              if (l == 0) {  // a^{-1}: centre -> x0, tangent -> r
                w0p[0] = fmaf(dl[0], sd[16], fmaf(dl[1], r0, w0p[0]));
                w0p[1] = fmaf(dl[0], sd[17], fmaf(dl[1], r1, w0p[1]));
                w0p[2] = fmaf(dl[0], sd[18], fmaf(dl[1], r2, w0p[2]));
              }
            }
            if (valid) {
              if (l >= 1) {
                FDSDF_ASSERT(c >= 0 && c < a.n && l >= 1 && l < nh);
                float* dp = a.del + (size_t)l * nrows * MPAD + drow0 + cl * (NCOLB * MPAD) + m;
                FDSDF_ASSERT(dp == a.del + ((size_t)l * nrows + (size_t)c * NCOLB) * MPAD + m);
#pragma unroll
                for (int j = 0; j < NCOLB; ++j) bwd_st(dp + j * MPAD, dl[j]);
              }
            }
            if (l >= 1) put_b10(m, cl, dl);
            s_db += dl[0];
            if (l == 0) {
              s_w0[0] += w0p[0];
              s_w0[1] += w0p[1];
              s_w0[2] += w0p[2];
            }
          }
          if (!top) ptimer.end_b();
          if (l >= 1) {
            tc_epi_arrive(bars, HP ? blk : 0);
          } else if (!top) {
            tc::fence_before();
          }
          r_db[blk][l] = db_l + s_db;
          if (l == 0) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              if (NBLK > 1 && blk)
                r_dW0[NBLK - 1][d] += s_w0[d];
              else
                r_dW0[0][d] += s_w0[d];
            }
          }
        }  // M-block
        if (!top) ++nd;
        if (top) {
#pragma unroll
          for (int b = 0; b < NBLK; ++b) r_dWL[b] += s_vL[b];
        }
      }
      if (m_of(0) == 0) {  // bias of the last layer: sum of the centre seeds (fbar) of this group
        float v = 0.f;
        for (int i = 0; i < CPX; ++i) v += sds[slot_of(i) * 20 + 0];
        r_dbL += v;
      }
    }
    // write this thread's slots (every element of the slot is owned by exactly one thread)
#pragma unroll
    for (int b = 0; b < NBLK; ++b) {
      const int m = m_of(b);
      r_db[b][ltop] += r_dbtop[b];
      for (int l = 0; l <= L - 2; ++l) acc_db[(size_t)l * MPAD + m] = r_db[b][l];
      acc_dWL[m] = r_dWL[b];
      acc_dW0[m * 3 + 0] = r_dW0[b][0];
      acc_dW0[m * 3 + 1] = r_dW0[b][1];
      acc_dW0[m * 3 + 2] = r_dW0[b][2];
    }
    if (m_of(0) == 0) acc_dbL[0] = r_dbL;
#ifdef FDSDF_PHASE_TIMING
    if (blockIdx.x == 0 && (et == 0 || et == C::NEPI * 32 - 32))
      printf("[phase] bwd_tc (thread %d): tile-start phase %.0f cyc/tile, next-tile top work %.0f cyc/tile\n", (int)threadIdx.x,
             (double)t_tstart / t_tstart_n, (double)t_top / t_tstart_n);
#endif
    ptimer.report("bwd_tc", et == 0 || et == C::NEPI * 32 - 32);
  }

  tc_teardown<C>(tbase);
}

template <int ACT, int MPAD>
static cudaError_t launch_bwd_tc_t(const BwdArgs& a, int grid, cudaStream_t st) {
  using C = BtcCfg<MPAD>;
  auto k = bwd_tc_kernel<ACT, MPAD>;
  cudaError_t e = smem_attr_once<bwd_tc_kernel<ACT, MPAD>>(C::BYTES);
  if (e != cudaSuccess) return e;
  k<<<grid, C::NTHR, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bwd_tc(const BwdArgs& a, int grid, cudaStream_t st) {
  const int act = a.net.act, mp = a.net.mpad;
#define FDSDF_CASE(A, MP) \
  if (act == A && mp == MP) return launch_bwd_tc_t<A, MP>(a, grid, st);
  FDSDF_CASE(ACT_SINE, 128)
  FDSDF_CASE(ACT_SINE, 256)
  FDSDF_CASE(ACT_SOFTPLUS, 128)
  FDSDF_CASE(ACT_SOFTPLUS, 256)
#undef FDSDF_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fdsdf
