// fwd_tc.cu -- the forward of the FD curvature step on the 5th-generation tensor cores
// (precision scheme bf16x6, tc.cuh / DESIGN.md §4b).
//
// Two launches of one warp-specialised persistent kernel, one CTA per SM:
//   mode 1  columns (z, dz/dx, dz/dy, dz/dz) of 16 centres (forward-mode tangents give
//           g = grad f); last layer -> f, g; per centre the degenerate mask and the
//           random right-handed frame -> cinfo.
//   mode 2  the 8 pair columns (A, S) x {u, v, u+v, u-v} of 8 centres in the pair-symmetric
//           difference form (act.cuh; P:L83-91 regrouped); last layer -> S_p; per centre the
//           FD epilogue (fdepi.cuh: f_uu, f_vv, f_uv, D_FD, K_FD, Eq. (1), seeds).
// Every hidden GEMM layer is D[m][n] = sum_k W[m][k] B[k][n] with M = MPAD output neurons
// (MPAD/128 tcgen05 M-halves), N = FWD_TC_N (64) columns, K = MPAD (engine: tcmlp.cuh):
//   warp 0      one thread streams the pre-packed bf16x3 weight image through a 2-stage
//               shared-memory ring with the TMA bulk engine (cp.async.bulk + mbarrier tx);
//   warp 1      allocates TMEM; the warp runs the issue loop, one elected lane issues the
//               six bf16x6 piece products per 16-wide K step as three MMAs into three TMEM
//               ranges (tcgen05.mma kind::f16, fp32 accumulate) and commits to mbarriers;
//   warps 2..17 epilogue (16 warps): thread = output neuron (TMEM lane), reads its row of D
//               with tcgen05.ld, applies bias / omega / the activation (centre + tangents, or
//               the cancellation-free pair maps), stores the pre-activations the backward
//               needs, splits the outputs into bf16 pieces and writes them into the K-major
//               SWIZZLE_128B B operand of the next layer.  X-independent work -- the next
//               tile's layer 0, the previous tile's per-centre FD epilogue -- runs while the
//               layer's MMA is in flight.
// Layer 0 (fan-in 3) and the last layer (fan-out 1) are computed by the epilogue threads
// directly (FFMA) -- they are not contractions worth a tensor-core pass.
#include "act.cuh"
#include "fdepi.cuh"
#include "tcmlp.cuh"

namespace fdsdf {

// 1: every epilogue warp polls "D full" itself; 0: one warp polls, the others wait in a named barrier
#ifndef FWD_TC_POLLALL
#define FWD_TC_POLLALL 1
#endif
// back-off between those polls (ns; 0 = try_wait with a suspend-time hint only)
#ifndef FWD_TC_POLL_NS
#define FWD_TC_POLL_NS 0
#endif
// M-half pipelining of the 256-wide layers (tcmlp.cuh TcCfg::HP): 1 = on
#ifndef FWD_TC_HP
#define FWD_TC_HP 1
#endif
#ifndef FWD_TC_NEPI
#define FWD_TC_NEPI 16
#endif
// unroll of the per-centre epilogue loop (1 = rolled)
#ifndef FWD_TC_UNROLL
#define FWD_TC_UNROLL 2
#endif
constexpr int kFwdUnroll = FWD_TC_UNROLL;
// GEMM columns per tile (mode 1: N/4 centres, mode 2: N/8 centres); with FWD_TC_NEPI the
// epilogue warps (a multiple of 4 x M-halves whose centre groups divide the tile)
#ifndef FWD_TC_N
#define FWD_TC_N 64
#endif
// 1: layer 0 of tile t+1 (fan-in 3, no MMA) is computed in tile t's MMA phases and parked in
// spare TMEM columns, so a tile starts with a split of the parked outputs into the B operand
// instead of a full epilogue pass with the tensor cores idle
#ifndef FWD_TC_PIPE0
#define FWD_TC_PIPE0 1
#endif
constexpr bool FWD_PIPE0 = FWD_TC_PIPE0;
// tile width: FWD_TC_N columns up to 256-wide layers; 32 for 512-wide ones (C3), where a wider
// B operand (32 x 512 x 3 pieces = 96 KB) would not fit next to the weight ring
constexpr int fwd_tc_n(int mpad) { return mpad == 512 ? 32 : FWD_TC_N; }
// MN-major B operand (a thread writes a centre's 4 / 8 consecutive columns as one vector store
// per piece) wherever the tile is whole 64-column swizzle atoms: N = 64 (MPAD <= 256)
#ifndef FWD_TC_BMN
#define FWD_TC_BMN 1
#endif
constexpr int fwd_tc_bmn(int mpad) { return (FWD_TC_BMN && fwd_tc_n(mpad) % 64 == 0) ? 1 : 0; }
constexpr int fwd_tc_hp(int mpad) { return (FWD_TC_HP && mpad == 256) ? 1 : 0; }
// weight ring depth (16 KB single-piece stages): one more than the backward's 6 fits next to the
// forward's 96 KB B operand
#ifndef FWD_TC_NST
#define FWD_TC_NST 6
#endif
template <int MPAD, int MODE>
struct FtcCfg : TcCfg<MPAD, fwd_tc_n(MPAD), FWD_TC_NEPI, 3, FWD_PIPE0 ? fwd_tc_n(MPAD) * (MPAD / 128) : 0, 1,
                      fwd_tc_bmn(MPAD), FWD_TC_NST, fwd_tc_hp(MPAD)> {
  // TMEM stash (FWD_PIPE0): the next tile's layer-0 outputs, (MH x EG thread groups) x CPE x
  // columns per centre = MH x N columns
  using B = TcCfg<MPAD, fwd_tc_n(MPAD), FWD_TC_NEPI, 3, FWD_PIPE0 ? fwd_tc_n(MPAD) * (MPAD / 128) : 0, 1,
                  fwd_tc_bmn(MPAD), FWD_TC_NST, fwd_tc_hp(MPAD)>;
  static constexpr int MAXC = 16;                                   // max centres per tile
  // last-layer partial sums and the tile's centre info are double-buffered by tile parity:
  // the per-centre epilogue of tile t runs during the first MMA phase of tile t+1
  static constexpr int RED_N = B::NEPI * MAXC * 4;                  // floats per buffer
  static constexpr int CI_N = MAXC * NCINFO;                        // floats per buffer
  static constexpr int OFF_RED = B::OFF_X;                          // float [2][NEPI][MAXC][4]
  static constexpr int OFF_CI = OFF_RED + 2 * RED_N * 4;            // float [2][MAXC][16]
  static constexpr int OFF_LV = OFF_CI + 2 * CI_N * 4;              // double [MAXC][NLOSS]
  static constexpr int OFF_BAR = OFF_LV + MAXC * NLOSS * 8;         // mbarriers + TMEM slot
  static constexpr int BYTES = OFF_BAR + tc_bars_bytes<B>() + 1024; // + alignment slack
  static_assert(BYTES <= 232448, "shared memory per CTA");
};

bool tc_supported(int mpad, int skip) { return (mpad == 128 || mpad == 256) && skip < 0; }

// the tensor-core forward alone (centre + pair kernels) also covers 512-wide layers and the skip
// layer; such networks run their backward / weight gradient on the FFMA kernels
bool tc_fwd_supported(int mpad) { return mpad == 128 || mpad == 256 || mpad == 512; }

size_t tc_wimg_bytes(int mpad, int ngemm) { return (size_t)(ngemm > 0 ? ngemm : 0) * mpad * mpad * 2 * tc::WP; }

int fwd_tc_tile_centres(int mode, int mpad) { return mode == 1 ? fwd_tc_n(mpad) / 4 : fwd_tc_n(mpad) / 8; }

// ----------------------------------------------------------------------------- weight images
// image[g][kc][h][piece < WP][sw128 128 rows x 64 k]: forward A operand = omega_l W_l (rows =
// output neuron m, K = input neuron k); backward A operand = omega_{l-1} W_l^T (rows = k, K = m),
// l = g + 1.  The SIREN frequency of the layer whose pre-activation the GEMM produces (forward:
// z_l = omega_l (W_l a + b_l); backward: delta_{l-1} = omega_{l-1} (...) (W_l^T delta_l)) is folded
// into the image (one fp32 rounding of omega W, <= 2^-24 relative), so the epilogues never scale
// the accumulator; omega = 1 for softplus.
__global__ void pack_tc_kernel(const Net net, unsigned char* fimg, unsigned char* bimg) {
  const int mp = net.mpad;
  const int KC = mp / 64, MH = mp / 128;
  const int g = blockIdx.y;
  const int l = g + 1;
  const int M = net.width[l + 1];
  const int K = net.width[l] + (l == net.skip ? 3 : 0);  // fan-in: cat(a, x) at the skip layer
  const float* W = net.W[l];
  const size_t per_layer = (size_t)mp * mp * 2 * tc::WP;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < mp * mp; idx += gridDim.x * blockDim.x) {
    const int r = idx / mp, k = idx % mp;  // A-operand row r, K index k
    const int h = r >> 7, rr = r & 127, kc = k >> 6, kk = k & 63;
    const size_t off = (size_t)g * per_layer + ((size_t)kc * MH + h) * (tc::WP * 16384) + tc::sw128_off(rr, kk, 128);
    {
      const float v = (r < M && k < K) ? net.omega[l] * W[(size_t)r * K + k] : 0.f;  // forward: W[m = r][k]
      const tc::Bf3 s = tc::split3(v);
#pragma unroll
      for (int p = 0; p < tc::WP; ++p) *reinterpret_cast<__nv_bfloat16*>(fimg + off + p * 16384) = s.p[p];
    }
    if (bimg) {
      const float v = (k < M && r < K) ? net.omega[g] * W[(size_t)k * K + r] : 0.f;  // backward: W^T[k = r][m = k]
      const tc::Bf3 s = tc::split3(v);
#pragma unroll
      for (int p = 0; p < tc::WP; ++p) *reinterpret_cast<__nv_bfloat16*>(bimg + off + p * 16384) = s.p[p];
    }
  }
  (void)KC;
}

cudaError_t launch_pack_tc(const Net& net, unsigned char* fimg, unsigned char* bimg, cudaStream_t st) {
  if (net.L <= 2) return cudaSuccess;
  dim3 grid(64, net.L - 2);
  pack_tc_kernel<<<grid, 256, 0, st>>>(net, fimg, bimg);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- the kernel

template <int ACT, int MPAD, int MODE>
__global__ void FDSDF_TC_CLUSTER __launch_bounds__(FtcCfg<MPAD, MODE>::NTHR, 1) fwd_tc_kernel(const FwdArgs a) {
  using C = FtcCfg<MPAD, MODE>;
  using AF = Act<ACT>;
  constexpr int N = C::N, MH = C::MH;
  constexpr int CPC = MODE == 1 ? 4 : 8;  // columns per centre
  constexpr int CT = N / CPC;             // centres per tile
  constexpr int CPE = CT / C::EG;         // centres per epilogue thread

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw;
  sm += (1024 - (smem_u32(sm) & 1023)) & 1023;
  unsigned char* Ws = sm + C::OFF_W;
  unsigned char* Bs = sm + C::OFF_B;
  float* red0 = reinterpret_cast<float*>(sm + C::OFF_RED);
  float* cis0 = reinterpret_cast<float*>(sm + C::OFF_CI);
  double* lvs = reinterpret_cast<double*>(sm + C::OFF_LV);
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
      if (lane == 0 && ngemm > 0) tc_producer<C>(a.wimg, ngemm, 0, a.ntiles, Ws, bars);
    } else if (warp == C::CTL0 + 1) {
      if (ngemm > 0) tc_mma<C>(ngemm, a.ntiles, Ws, Bs, tbase, bars);
    }
  } else {
    setmaxnreg_inc<C::REG_EPI>();
    // ------------------------------------------------------------------ epilogue warps
    const int ew = warp - C::EPI0;  // 0 .. NEPI-1
    const int et = tid - 32 * C::EPI0;  // 0 .. NEPI*32-1
    const int q4 = warp & 3;                 // TMEM lane quarter
    // M-blocks: without M-half pipelining every warp owns one M-half and EG centre groups split
    // the tile; with it (C::HP) every warp walks both M-halves in turn (half 0, then half 1 of
    // each layer) and NEPI / 4 centre groups split the tile
    constexpr bool HP = C::HP;
    constexpr int NBLK = HP ? MH : 1;        // M-blocks per layer and thread
    constexpr int EGX = HP ? C::NEPI / 4 : C::EG;  // centre groups
    constexpr int CPX = CT / EGX;            // centres per thread and M-block
    static_assert(CT % EGX == 0, "centre groups divide the tile");
    const int hh0 = HP ? 0 : (ew >> 2) % MH;
    const int egx = HP ? (ew >> 2) : ew / (4 * MH);  // centre group
    auto half_of = [&](int blk) { return HP ? blk : hh0; };
    auto neuron = [&](int blk) { return half_of(blk) * 128 + 32 * q4 + lane; };  // output neuron of this thread
    auto taddr_of = [&](int blk) -> uint32_t {
      return tbase + ((uint32_t)(32 * q4) << 16) + half_of(blk) * C::DH;
    };
    // this thread's stash columns of M-block blk: CPX centres x CPC values (FWD_PIPE0)
    auto tstash_of = [&](int blk) -> uint32_t {
      return tbase + ((uint32_t)(32 * q4) << 16) + MH * C::DH + (half_of(blk) * EGX + egx) * CPX * CPC;
    };
    // slot of this warp's last-layer partial sums of M-block blk (finish() sums the slots)
    auto rslot = [&](int blk) { return HP ? blk * 4 + q4 : ew; };
    const float beta = net.beta;
    const float h = a.h;
    const bool step = a.step != 0;
    uint32_t nd = 0;
    PhaseTimer ptimer;
    ptimer.start();
    double lacc[NLOSS];
#pragma unroll
    for (int q = 0; q < NLOSS; ++q) lacc[q] = 0.0;

    // this thread's stored pre-activations of layer l, centre c, neuron m (kernels.cuh zf
    // layout): float4 group g (step), the centre value z (step: in group 0; eval: z only,
    // contiguous over m)
    // `zb` = the centre's block of zf (zrow(c)): one 64-bit product per centre, the rest in 32 bits
    const int zcs = nh * a.zcols * MPAD, zls = a.zcols * MPAD;  // centre / layer strides (floats)
    auto zrow = [&](int64_t c) -> float* { return a.zf + (size_t)c * zcs; };
    auto zg4 = [&](const float* zb, int64_t c, int l, int g, int m) -> float4* {
      FDSDF_ASSERT(c >= 0 && c < a.n && l >= 0 && l < nh && g >= 0 && g < ZG && a.zcols == NCOLF && m < MPAD);
      FDSDF_ASSERT(zb == a.zf + (size_t)c * zcs);
      return reinterpret_cast<float4*>(const_cast<float*>(zb) + l * zls + g * 4 * MPAD) + m;
    };
    auto zc = [&](const float* zb, int64_t c, int l, int m) -> float* {
      FDSDF_ASSERT(c >= 0 && c < a.n && l >= 0 && l < nh && m < MPAD);
      FDSDF_ASSERT(zb == a.zf + (size_t)c * zcs);
      return const_cast<float*>(zb) + l * zls + (step ? 4 * m : m);
    };
    // a centre's consecutive columns n0 .. n0+3 / n0+7 of the next B operand (K index m)
    auto put_b4 = [&](int n0, int m, const float (&v)[4]) {
      if constexpr (C::BMN) {
        tc_put_b4<C>(Bs, n0, m, v);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) tc_put_b<C>(Bs, n0 + j, m, v[j]);
      }
    };
    auto put_b8 = [&](int n0, int m, const float (&v)[8]) {
      if constexpr (C::BMN) {
        tc_put_b8<C>(Bs, n0, m, v);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) tc_put_b<C>(Bs, n0 + j, m, v[j]);
      }
    };
    // cat(a, x) / sqrt(2) at the input of the skip layer net.skip (IGR convention, SURVEY §8c
    // item 14): when layer l's outputs feed it, every output is scaled by 1/sqrt(2) and the
    // threads of rows M .. M+2 (no neuron of layer l) supply the x part (as fwd.cu does)
    constexpr float RSQ2 = 0.70710678118654752f;
    auto skip_centre = [&](int l, int m, int64_t c, bool valid, float& o0, float& o1, float& o2, float& o3) {
      if (l + 1 != net.skip) return;
      const int M = net.width[l + 1];
      if (m >= M && m < M + 3) {  // value x_d, tangents e_d
        const int d = m - M;
        o0 = valid ? a.x[c * 3 + d] : 0.f;
        o1 = d == 0 ? 1.f : 0.f;
        o2 = d == 1 ? 1.f : 0.f;
        o3 = d == 2 ? 1.f : 0.f;
      }
      o0 *= RSQ2;
      o1 *= RSQ2;
      o2 *= RSQ2;
      o3 *= RSQ2;
    };
    auto skip_pairs = [&](int l, int m, const float* ci, float (&o)[8]) {
      if (l + 1 != net.skip) return;
      const int M = net.width[l + 1];
      if (m >= M && m < M + 3) {  // odd part of x0 +- h d_p = h d_p, even part 0 (column order: see kPairCol)
        const int d = m - M;
        const float ud = ci[4 + d], vd = ci[7 + d];
        o[0] = h * ud;
        o[1] = h * vd;
        o[4] = h * (ud + vd);
        o[5] = h * (ud - vd);
        o[2] = o[3] = o[6] = o[7] = 0.f;
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) o[p] *= RSQ2;
    };
    // the pair maps of all 4 pairs of a centre (packed by two: A2[k] = (A_{2k}, A_{2k+1})) -> the
    // next layer's 8 B columns of the centre in the order A0 A1 S0 S1 A2 A3 S2 S3 (kPairCol: the
    // accumulator columns come back in that order, i.e. already packed by two); every lane calls
    // this (the sine maps vote on their fast form); rows past the width give 0
    auto pair_outputs = [&](const typename AF::C& cc, bool mok, const float2 (&A2)[2], const float2 (&S2)[2],
                            float (&o)[8]) {
      float2 Aa[2], Sa[2];
      AF::pairs_fwd4x2(cc, A2, S2, beta, Aa, Sa);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        o[4 * k] = mok ? Aa[k].x : 0.f;
        o[4 * k + 1] = mok ? Aa[k].y : 0.f;
        o[4 * k + 2] = mok ? Sa[k].x : 0.f;
        o[4 * k + 3] = mok ? Sa[k].y : 0.f;
      }
    };
    const bool pipe0 = FWD_PIPE0 && ngemm > 0;
    FDSDF_ASSERT(!FWD_PIPE0 || (MH * C::DH + MH * EGX * CPX * CPC) <= (int)C::TCOLS);
    // this thread's layer-0 weight rows and biases, one per M-block (fan-in 3; constant over the
    // kernel, loaded once instead of before every centre's layer-0 arithmetic)
    float w0r[NBLK][3], b0r[NBLK];
#pragma unroll
    for (int blk = 0; blk < NBLK; ++blk) {
      const int m = neuron(blk);
      const bool mok0 = m < net.width[1];
#pragma unroll
      for (int j = 0; j < 3; ++j) w0r[blk][j] = mok0 ? net.W[0][m * 3 + j] : 0.f;
      b0r[blk] = (MODE == 1 && mok0) ? net.b[0][m] : 0.f;
    }
    // compile-time indexed (a runtime index would put the arrays in local memory)
    auto w0of = [&](int blk, int j) -> float { return (NBLK > 1 && blk) ? w0r[NBLK - 1][j] : w0r[0][j]; };
    auto b0of = [&](int blk) -> float { return (NBLK > 1 && blk) ? b0r[NBLK - 1] : b0r[0]; };
    // layer 0 of centre i of M-block blk of tile tl (centre info cis_t): pre-activations -> zf,
    // activations -> this thread's stash columns (exactly the l == 0 arithmetic of the epilogue)
    auto layer0_centre = [&](int64_t tl, int blk, int i, const float* cis_t) {
      if (tl >= a.ntiles) return;
      const int cl = egx + EGX * i;
      const int64_t c = tl * CT + cl;
      const bool valid = c < a.n;
      const float om = net.omega[0];
      const int m = neuron(blk);
      const bool mok = m < net.width[1];
      const uint32_t tstash = tstash_of(blk);
      if (MODE == 1) {
        float z = 0.f, t0 = 0.f, t1 = 0.f, t2 = 0.f;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f;
        if (valid) {
          x0 = a.x[c * 3 + 0];
          x1 = a.x[c * 3 + 1];
          x2 = a.x[c * 3 + 2];
          if (m == 0 && !(isfinite(x0) && isfinite(x1) && isfinite(x2))) atomicOr(a.dflags, 1u);
        }
        if (mok) {
          const float w0 = w0of(blk, 0), w1 = w0of(blk, 1), w2 = w0of(blk, 2);
          z = om * (fmaf(w0, x0, fmaf(w1, x1, w2 * x2)) + b0of(blk));
          t0 = om * w0;
          t1 = om * w1;
          t2 = om * w2;
        }
        if (valid) {
          if (step)
            *zg4(zrow(c), c, 0, 0, m) = make_float4(z, t0, t1, t2);
          else
            *zc(zrow(c), c, 0, m) = z;
        }
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        if (mok) {
          const typename AF::C cc = AF::centre(z, beta);
          const float s1 = AF::d1(cc, beta);
          o[0] = AF::value(cc, beta);
          o[1] = s1 * t0;
          o[2] = s1 * t1;
          o[3] = s1 * t2;
        }
        skip_centre(0, m, c, valid, o[0], o[1], o[2], o[3]);
        tc::tmem_st4(tstash + i * CPC, o);
      } else {
        const float* ci = cis_t + cl * NCINFO;
        const float* zb = zrow(c);
        const float z0 = valid ? __ldg(zc(zb, c, 0, m)) : 0.f;
        float2 A2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, S2[2] = {A2[0], A2[0]};
        if (mok) {
          const float w0 = w0of(blk, 0), w1 = w0of(blk, 1), w2 = w0of(blk, 2);
          const float du = fmaf(w0, ci[4], fmaf(w1, ci[5], w2 * ci[6]));
          const float dv = fmaf(w0, ci[7], fmaf(w1, ci[8], w2 * ci[9]));
          const float hs = om * h;
          A2[0] = make_float2(hs * du, hs * dv);
          A2[1] = make_float2(hs * (du + dv), hs * (du - dv));
        }
        if (step && valid) {
          *zg4(zb, c, 0, 1, m) = make_float4(A2[0].x, A2[0].y, S2[0].x, S2[0].y);
          *zg4(zb, c, 0, 2, m) = make_float4(A2[1].x, A2[1].y, S2[1].x, S2[1].y);
        }
        float o[8];
        pair_outputs(AF::centre(z0, beta), mok, A2, S2, o);
        skip_pairs(0, m, ci, o);
        float o4[4] = {o[0], o[1], o[2], o[3]};
        tc::tmem_st4(tstash + i * CPC, o4);
        o4[0] = o[4];
        o4[1] = o[5];
        o4[2] = o[6];
        o4[3] = o[7];
        tc::tmem_st4(tstash + i * CPC + 4, o4);
      }
    };
    // the MMA phases of a tile that also run the next tile's layer 0 (mode 2: from layer 2 on,
    // once warp 2's copy of the next tile's centre info has landed)
    const int l0first = (MODE == 2 && ngemm >= 2) ? 2 : 1;

    // per-centre epilogue of a finished tile (warp 2 only: et < CT <= 16): mode 1 -> f, g, mask,
    // frame, cinfo; mode 2 -> FD entries, D, K, Eq. (1) terms, seeds, and the fixed-order
    // fp64 accumulation of the tile's loss terms
    auto finish = [&](int64_t fc0, const float* red, float* cis) {
      if (et < CT) {
        const int cl = et;
        const int64_t c = fc0 + cl;
        const bool valid = c < a.n;
        float tot[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float v = 0.f;
          if (HP) {  // slots blk * 4 + q4: every one holds a partial sum of every centre
            for (int w = 0; w < 4 * MH; ++w) v += red[(w * C::MAXC + cl) * 4 + j];
          } else {
            for (int w = 0; w < C::NEPI; ++w)
              if ((w / (4 * MH)) == (cl % C::EG)) v += red[(w * C::MAXC + cl) * 4 + j];
          }
          tot[j] = v;
        }
        if (MODE == 1) {
          float* ci = cis + cl * NCINFO;
          centre_frame(a, c, valid, tot[0] + net.b[L - 1][0], tot[1], tot[2], tot[3], ci);
          if (valid) {
#pragma unroll
            for (int q = 0; q < NCINFO; ++q) a.cinfo[c * NCINFO + q] = ci[q];
          }
        } else {
          double lv[NLOSS];
          fd_centre(a, c, valid, tot, cis + cl * NCINFO, lv);
#pragma unroll
          for (int q = 0; q < NLOSS; ++q) lvs[cl * NLOSS + q] = lv[q];
        }
      }
      __syncwarp();
      if (MODE == 2 && et == 0) {  // fixed-order tile reduction of the loss terms
        for (int s2 = 0; s2 < CT; ++s2)
#pragma unroll
          for (int q = 0; q < NLOSS; ++q) lacc[q] += lvs[s2 * NLOSS + q];
      }
    };
    bool pending = false;
    int64_t pend_c0 = 0;
    const float* pend_red = nullptr;
    float* pend_cis = nullptr;
    uint32_t tpar = 0;

    // mode 2: the tile's centre info (f, g, frame, mask) from mode 1.  The first tile's is
    // loaded here; every later one is copied asynchronously (cp.async, warp 2) into the other
    // buffer right after that buffer's deferred per-centre epilogue
    auto load_cinfo = [&](int64_t tile, float* dst, int t0, int nt) {
      const int64_t cb = tile * CT;
      for (int i = t0; i < CT * NCINFO; i += nt) {
        const int64_t c = cb + i / NCINFO;
        if (tile < a.ntiles && c < a.n)
          cp_async4(dst + i, a.cinfo + c * NCINFO + (i % NCINFO));
        else
          dst[i] = 0.f;
      }
    };
    if (MODE == 2) load_cinfo(blockIdx.x, cis0, et, C::NEPI * 32);
    const int64_t tend = tc_tile_end<C>(a.ntiles);
    for (int64_t tile = blockIdx.x; tile < tend; tile += gridDim.x, tpar ^= 1u) {
      const int64_t c0 = tile * CT;
      float* const zt = zrow(c0);  // the tile's first centre's block of zf
      float* red = red0 + tpar * C::RED_N;
      float* cis = cis0 + tpar * C::CI_N;
      if (MODE == 2) {
        cp_async_wait_all();
        bar_named(1, C::NEPI * 32);
      }

      for (int l = 0; l <= L - 2; ++l) {
        const bool last = (l == L - 2);
        const int M = net.width[l + 1];
        const float om = net.omega[l];
        // last layer: sum over this warp's 32 neurons of w_L[m] * out_j, one slot per centre
        auto reduce4 = [&](int blk, int cl, float wl, float p0, float p1, float p2, float p3) {
          float pv[4] = {wl * p0, wl * p1, wl * p2, wl * p3};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float v = pv[j];
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            if (lane == 0) red[(rslot(blk) * C::MAXC + cl) * 4 + j] = v;
          }
        };
        if (l == 0 && pipe0) {
          // B operand of layer 1 from the parked layer-0 outputs (computed here only for the
          // CTA's first tile), M-block by M-block
          if (tile == blockIdx.x) {
            for (int blk = 0; blk < NBLK; ++blk)
              for (int i = 0; i < CPX; ++i) layer0_centre(tile, blk, i, cis);
            tc::tmem_wait_st();
          }
#pragma unroll
          for (int blk = 0; blk < NBLK; ++blk) {
            const int m = neuron(blk);
            const uint32_t tstash = tstash_of(blk);
#pragma unroll 1
            for (int i = 0; i < CPX; ++i) {
              const int cl = egx + EGX * i;
              if constexpr (CPC == 4) {
                float o4[4];
                tc::tmem_ld4(tstash + i * CPC, o4);
                put_b4(cl * CPC, m, o4);
              } else {
                float o8[8];
                tc::tmem_ld8(tstash + i * CPC, o8);
                put_b8(cl * CPC, m, o8);
              }
            }
            tc_epi_arrive(bars, HP ? blk : 0);
          }
        } else {
          if (pipe0 && l >= l0first) {  // the next tile's layer 0, spread over this tile's MMA phases
            if (MODE == 2 && l == l0first) {
              if (ew == 0) cp_async_wait_all();
              bar_named(1, C::NEPI * 32);  // the next tile's centre info is in
            }
#pragma unroll 1
            for (int k = l - l0first; k < NBLK * CPX; k += L - 1 - l0first)
              layer0_centre(tile + gridDim.x, k / CPX, k % CPX, cis0 + (tpar ^ 1u) * C::CI_N);
            tc::tmem_wait_st();
          }
#pragma unroll 1
          for (int blk = 0; blk < NBLK; ++blk) {
            const int m = neuron(blk);
            const bool mok = m < M;
            const float wl = (last && mok) ? net.W[L - 1][m] : 0.f;
            // omega_l b_l (the image carries omega_l W_l), once per layer and M-block
            const float bias_l = (MODE == 1 && l > 0 && mok) ? om * net.b[l][m] : 0.f;
            const uint32_t taddr = taddr_of(blk);
            // mode 2: the centre pre-activation of this neuron at centre slot cl (prefetched one
            // centre ahead; this thread's first centre before the MMA wait)
            auto ldz = [&](int cl) -> float {
              const int64_t c = c0 + cl;
              return (MODE == 2 && cl < CT && c < a.n) ? __ldg(zc(zt + cl * zcs, c, l, m)) : 0.f;
            };
            float z0n = ldz(egx);  // mode 2: prefetched one centre ahead (the first before the MMA wait)
            if (l > 0) {
              ptimer.before_wait();
              // one warp polls the mbarrier, the others sleep in a hardware named barrier (no
              // spin instructions competing with the MMA warp for issue slots)
              if (FWD_TC_POLLALL) {  // every warp waits for itself (no wait for the slowest warp)
                mbar_wait_sleep<FWD_TC_POLL_NS>(&bars.dfull[HP ? blk : 0], nd & 1u);
              } else {
                if (ew == 0) mbar_wait(&bars.dfull[HP ? blk : 0], nd & 1u);
                bar_named(2, C::NEPI * 32);
              }
              ptimer.after_wait();
              tc::fence_after();
            }
            // HP: the B rows of K half 0 may still be read by the layer's (1, 0) MMA group --
            // wait for "B free" before this M-block's first B store
            bool need_free = HP && blk == 0 && l > 0 && !last;
            // cc0: mode 2, the centre terms sigma(z0), sigma'(z0) of the centre (two centres' sincos
            // evaluated together, packed)
            // mode 1, per centre: the accumulator -> z, tangents (-> zf), then (with the centre
            // terms of two centres evaluated together, packed) the outputs -> next B / last layer
            struct M1 {
              float z, t0, t1, t2;
            };
            auto m1_pre = [&](const int cl) -> M1 {
              const int64_t c = c0 + cl;
              const bool valid = c < a.n;
              M1 q{0.f, 0.f, 0.f, 0.f};
              if (l == 0) {
                float x0 = 0.f, x1 = 0.f, x2 = 0.f;
                if (valid) {
                  x0 = a.x[c * 3 + 0];
                  x1 = a.x[c * 3 + 1];
                  x2 = a.x[c * 3 + 2];
                  if (m == 0 && !(isfinite(x0) && isfinite(x1) && isfinite(x2))) atomicOr(a.dflags, 1u);
                }
                if (mok) {
                  const float w0 = w0of(blk, 0), w1 = w0of(blk, 1), w2 = w0of(blk, 2);
                  q.z = om * (fmaf(w0, x0, fmaf(w1, x1, w2 * x2)) + b0of(blk));
                  q.t0 = om * w0;
                  q.t1 = om * w1;
                  q.t2 = om * w2;
                }
              } else {
                float v[4];
                tc_ld_sum4<C>(taddr, cl * 4, v);  // centre cl's 4 columns
                if (mok) {
                  q.z = v[0] + bias_l;
                  q.t0 = v[1];
                  q.t1 = v[2];
                  q.t2 = v[3];
                }
              }
              if (valid) {
                if (step)
                  *zg4(zt + cl * zcs, c, l, 0, m) = make_float4(q.z, q.t0, q.t1, q.t2);
                else
                  *zc(zt + cl * zcs, c, l, m) = q.z;
              }
              return q;
            };
            auto m1_post = [&](const int cl, const typename AF::C& cc, const M1& q) {
              const int64_t c = c0 + cl;
              const bool valid = c < a.n;
              float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
              if (mok) {
                const float s1 = AF::d1(cc, beta);
                o0 = AF::value(cc, beta);
                o1 = s1 * q.t0;
                o2 = s1 * q.t1;
                o3 = s1 * q.t2;
              }
              skip_centre(l, m, c, valid, o0, o1, o2, o3);
              if (last) {
                reduce4(blk, cl, wl, o0, o1, o2, o3);
              } else {
                const float o4[4] = {o0, o1, o2, o3};
                if (need_free) {
                  mbar_wait(bars.bfree, nd & 1u);
                  need_free = false;
                }
                put_b4(cl * 4, m, o4);
              }
            };
            // mode 2, per centre; cc0 = the centre terms sigma(z0), sigma'(z0) of the centre
            auto centre_body = [&](const int cl, const typename AF::C& cc0) {
              const int64_t c = c0 + cl;
              const bool valid = c < a.n;
              if constexpr (MODE == 2) {
                const float* ci = cis + cl * NCINFO;
                float2 A2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)}, S2[2] = {A2[0], A2[0]};
                if (l == 0) {
                  if (mok) {
                    const float w0 = w0of(blk, 0), w1 = w0of(blk, 1), w2 = w0of(blk, 2);
                    const float du = fmaf(w0, ci[4], fmaf(w1, ci[5], w2 * ci[6]));
                    const float dv = fmaf(w0, ci[7], fmaf(w1, ci[8], w2 * ci[9]));
                    const float hs = om * h;
                    A2[0] = make_float2(hs * du, hs * dv);
                    A2[1] = make_float2(hs * (du + dv), hs * (du - dv));
                  }
                } else {
                  float v[8];
                  tc_ld_sum8<C>(taddr, cl * 8, v);  // columns A0 A1 S0 S1 A2 A3 S2 S3 (kPairCol)
                  if (mok) {
                    A2[0] = make_float2(v[0], v[1]);
                    S2[0] = make_float2(v[2], v[3]);
                    A2[1] = make_float2(v[4], v[5]);
                    S2[1] = make_float2(v[6], v[7]);
                  }
                }
                if (step && valid) {
                  float* zb = zt + cl * zcs;
                  *zg4(zb, c, l, 1, m) = make_float4(A2[0].x, A2[0].y, S2[0].x, S2[0].y);
                  *zg4(zb, c, l, 2, m) = make_float4(A2[1].x, A2[1].y, S2[1].x, S2[1].y);
                }
                float o[8];
                pair_outputs(cc0, mok, A2, S2, o);
                skip_pairs(l, m, ci, o);
                if (last) {
                  reduce4(blk, cl, wl, o[2], o[3], o[6], o[7]);
                } else {
                  if (need_free) {
                    mbar_wait(bars.bfree, nd & 1u);
                    need_free = false;
                  }
                  put_b8(cl * 8, m, o);
                }
              }
            };
            {
              if constexpr (MODE == 1) {
#pragma unroll kFwdUnroll
                for (int i = 0; i < CPX; i += 2) {
                  static_assert(CPX % 2 == 0, "centres of a thread and M-block come in pairs");
                  const int cla = egx + EGX * i, clb = egx + EGX * (i + 1);  // centre slots in the tile
                  const M1 qa = m1_pre(cla), qb = m1_pre(clb);
                  typename AF::C cc[2];
                  AF::centre2(qa.z, qb.z, beta, cc[0], cc[1]);
                  m1_post(cla, cc[0], qa);
                  m1_post(clb, cc[1], qb);
                }
              } else {  // (packing two centres' sincos here measured 1-2% slower)
#pragma unroll kFwdUnroll
                for (int i = 0; i < CPX; ++i) {
                  const int cl = egx + EGX * i;  // centre slot in the tile
                  const float z0 = z0n;
                  z0n = ldz(cl + EGX);
                  centre_body(cl, AF::centre(z0, beta));
                }
              }
            }
            if (l > 0) ptimer.end_b();
            if (!last) {  // this M-block's rows of the next B operand (this warp's part): hand to the MMA
              tc_epi_arrive(bars, HP ? blk : 0);
            } else if (l > 0) {
              tc::fence_before();
            }
          }  // M-block
        }
        if (l > 0) ++nd;
        if (l == 0 && pending) {  // the previous tile's per-centre work, overlapping the MMA phase
          if (ew == 0) finish(pend_c0, pend_red, pend_cis);
          pending = false;
        }
        if (l == 0 && MODE == 2 && ew == 0)  // next tile's centre info into the buffer just freed
          load_cinfo(tile + gridDim.x, cis0 + (tpar ^ 1u) * C::CI_N, lane, 32);
      }

      bar_named(1, C::NEPI * 32);  // this tile's last-layer partial sums are complete
      pending = true;
      pend_c0 = c0;
      pend_red = red;
      pend_cis = cis;
    }
    if (pending && ew == 0) finish(pend_c0, pend_red, pend_cis);
    if (MODE == 2 && et == 0) {
#pragma unroll
      for (int q = 0; q < NLOSS; ++q) a.lossp[(size_t)blockIdx.x * NLOSS + q] = lacc[q];
    }
    ptimer.report(MODE == 1 ? "fwd_tc centre" : "fwd_tc pairs", et == 0 || et == C::NEPI * 32 - 32);
  }

  tc_teardown<C>(tbase);
}

// ----------------------------------------------------------------------------- host launch
template <int ACT, int MPAD, int MODE>
static cudaError_t launch_fwd_tc_t(const FwdArgs& a, int grid, cudaStream_t st) {
  using C = FtcCfg<MPAD, MODE>;
  auto k = fwd_tc_kernel<ACT, MPAD, MODE>;
  cudaError_t e = smem_attr_once<fwd_tc_kernel<ACT, MPAD, MODE>>(C::BYTES);
  if (e != cudaSuccess) return e;
  k<<<grid, C::NTHR, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fwd_tc(const FwdArgs& a, int mode, int grid, cudaStream_t st) {
  const int act = a.net.act, mp = a.net.mpad;
#define FDSDF_CASE(A, MP, MO) \
  if (act == A && mp == MP && mode == MO) return launch_fwd_tc_t<A, MP, MO>(a, grid, st);
  FDSDF_CASE(ACT_SINE, 128, 1)
  FDSDF_CASE(ACT_SINE, 128, 2)
  FDSDF_CASE(ACT_SINE, 256, 1)
  FDSDF_CASE(ACT_SINE, 256, 2)
  FDSDF_CASE(ACT_SOFTPLUS, 128, 1)
  FDSDF_CASE(ACT_SOFTPLUS, 128, 2)
  FDSDF_CASE(ACT_SOFTPLUS, 256, 1)
  FDSDF_CASE(ACT_SOFTPLUS, 256, 2)
  FDSDF_CASE(ACT_SINE, 512, 1)
  FDSDF_CASE(ACT_SINE, 512, 2)
  FDSDF_CASE(ACT_SOFTPLUS, 512, 1)
  FDSDF_CASE(ACT_SOFTPLUS, 512, 2)
#undef FDSDF_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fdsdf
