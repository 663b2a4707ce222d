// bwd.cu -- backward through every stencil evaluation.
//
// Per tile of CG centres, 10 adjoint columns per centre: the centre value, the tangent along
// r = d loss/d g (the eikonal and the live |g|^p denominator need only the directional
// derivative r.g, whose weight gradient is that of one forward-mode tangent column), and the
// (A, S) pairs of act.cuh.  Top-down over the hidden layers:
//   X = W_{l+1}^T delta_{l+1}         (column GEMM, W streamed by TMA, tile.cuh)
//   delta_l = omega_l * activation-backward(z_l, X)         (cancellation-free, act.cuh)
// The kernel writes delta_l and the layer inputs (post-activations) of every GEMM layer for
// the split-K weight-gradient kernel, and accumulates per CTA (fixed tile order) the bias
// gradients, dW of the first layer (fan-in 3) and dW of the last layer (fan-out 1).
#include "act.cuh"
#include "tile.cuh"

namespace fdsdf {

template <int MPAD>
struct BwdSmem {
  using T = TileCfg<MPAD, 8192, 3>;
  static constexpr int ACT8 = MPAD * T::NC;
  static constexpr int ACT2 = MPAD * T::CG * 2;
  static constexpr int WST = T::NSTG * T::SLAB;
  static constexpr int RED = MPAD * T::CG;
  static constexpr int SEEDS = T::CG * 20;
  static constexpr size_t BYTES = (size_t)(ACT8 + ACT2 + WST + RED + SEEDS) * 4 + 2 * T::NSTG * 8 + 64;
};

template <int ACT, int MPAD>
__global__ void __launch_bounds__(NTH, 2) bwd_kernel(const BwdArgs a) {
  using S = BwdSmem<MPAD>;
  using T = typename S::T;
  using AF = Act<ACT>;
  constexpr int RG = T::RG, CG = T::CG, NC = T::NC;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* act8 = reinterpret_cast<float*>(smem_raw);
  float* act2 = act8 + S::ACT8;
  float* wst = act2 + S::ACT2;
  float* red = wst + S::WST;
  float* sseed = red + S::RED;  // [CG][20]: seeds(16) + x(3)
  uint64_t* full = reinterpret_cast<uint64_t*>(sseed + S::SEEDS);
  uint64_t* empty = full + T::NSTG;

  const Net& net = a.net;
  const int L = net.L;
  const int nh = L - 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < T::NSTG; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // weight stream: W_{l+1} for l = L-3 .. 0, i.e. GEMM layers L-2 .. 1
  WStream<T> ws;
  ws.layers = net.Wb;
  ws.L = L;
  ws.backward = 1;
  ws.per_tile = (uint32_t)(L - 2) * T::NCHUNK;
  ws.total = (L > 2 && blockIdx.x < a.ntiles)
                 ? (uint32_t)((a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * ws.per_tile
                 : 0u;
  ws.wst = wst;
  ws.full = full;
  ws.empty = empty;
  if (tid == 0) ws.prologue();

  const int wr = warp % T::RGW, wc = warp / T::RGW;
  const int rg = wr * 8 + (lane & 7);
  const int cg = wc * 4 + (lane >> 3);
  const float beta = net.beta;
  const float h = a.h;
  const float isq2 = 0.70710678118654752f;
  const int64_t nrows = a.n * NCOLB;
  float* bacc = a.bacc + (size_t)blockIdx.x * a.nacc;
  float* acc_db = bacc;                               // [L-1][MPAD]
  float* acc_dWL = bacc + (size_t)(L - 1) * MPAD;     // [MPAD]
  float* acc_dbL = acc_dWL + MPAD;                    // [1]
  float* acc_dW0 = acc_dbL + 1;                       // [MPAD][3]
  for (int64_t i = tid; i < a.nacc; i += NCT) bacc[i] = 0.f;
  bar_compute(NCT);

  uint32_t it = 0;
  float acc[8][8];
  float acc2[8][2];

  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t c0 = tile * CG;
    if (tid < CG) {
      const int64_t c = c0 + tid;
      float* sd = sseed + tid * 20;
      if (c < a.n) {
        for (int q = 0; q < NSEED; ++q) sd[q] = a.seed[c * NSEED + q];
        for (int d = 0; d < 3; ++d) sd[16 + d] = a.x[c * 3 + d];
      } else {
        for (int q = 0; q < 20; ++q) sd[q] = 0.f;
      }
    }
    bar_compute(NCT);

    const int64_t c = c0 + cg;
    const bool valid = c < a.n;
    const float* sd = sseed + cg * 20;
    // delta of the output layer per column: (c, t, A_u, S_u, A_v, S_v, A_p, S_p, A_q, S_q)
    const float dL[10] = {sd[0], valid ? 1.f : 0.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
    const float r0 = sd[5], r1 = sd[6], r2 = sd[7];
    // layer-0 inputs a^{-1} per column and coordinate: x0, r, h*d_p, 0
    const float u0 = sd[8], u1 = sd[9], u2 = sd[10], v0 = sd[11], v1 = sd[12], v2 = sd[13];

    for (int l = L - 2; l >= 0; --l) {
      const bool top = (l == L - 2);
      if (!top) {
        tile_gemm<T, true>(acc, acc2, act8, act2, ws, it, rg, cg, tid);
        bar_compute(NCT);
        // park X = W^T delta in shared memory (own positions) to free registers
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int m = tile_row<MPAD>(rg, i);
          *reinterpret_cast<float4*>(act8 + act_idx<NC>(m, cg * 8)) =
              make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
          *reinterpret_cast<float4*>(act8 + act_idx<NC>(m, cg * 8 + 4)) =
              make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
          *reinterpret_cast<float2*>(act2 + m * (CG * 2) + cg * 2) = make_float2(acc2[i][0], acc2[i][1]);
        }
      }
      const float om = net.omega[l];
      const int M = net.width[l + 1];
      const bool nskip = (l + 1 == net.skip);
      const float xsc = nskip ? isq2 : 1.0f;       // d(layer input)/d(a): cat(a,x)/sqrt(2)
      const float* __restrict__ Wlast = net.W[L - 1];
      const bool store_del = (l >= 1) && (l <= L - 2) && valid;
      const bool store_act = (l <= L - 3) && valid;
      float* delp = a.del + (size_t)l * nrows * MPAD + (size_t)c * NCOLB * MPAD;
      float* actp = a.actv + (size_t)l * nrows * MPAD + (size_t)c * NCOLB * MPAD;
      // this (centre, layer)'s stored pre-activations: float4 groups per neuron (kernels.cuh)
      const float4* zq = reinterpret_cast<const float4*>(a.zf + ((size_t)c * nh + l) * NCOLF * MPAD);

      float w0s[2][4][3];  // dW_0 partials (l == 0), parked after the epilogue barrier
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) w0s[q][j][0] = w0s[q][j][1] = w0s[q][j][2] = 0.f;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int mb = tile_row<MPAD>(rg, q * 4);
        float zc[4], tr[4];
        {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 g0 = valid ? zq[mb + j] : make_float4(0.f, 0.f, 0.f, 0.f);  // (z, t0, t1, t2)
            zc[j] = g0.x;
            tr[j] = fmaf(r0, g0.y, fmaf(r1, g0.z, r2 * g0.w));
          }
        }
        typename AF::C cc[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) cc[j] = AF::centre(zc[j], beta);
        float zbar[4] = {0.f, 0.f, 0.f, 0.f};
        float vL[4] = {0.f, 0.f, 0.f, 0.f};          // dW_last partial (top layer only)
        float w0p[4][3];                              // dW_0 partial (l == 0 only)
#pragma unroll
        for (int j = 0; j < 4; ++j) w0p[j][0] = w0p[j][1] = w0p[j][2] = 0.f;
        float wl[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) wl[j] = (top && mb + j < M) ? Wlast[mb + j] : 0.f;

        // ---------------------------------------------------------------- 4 pairs
#pragma unroll 1
        for (int p = 0; p < 4; ++p) {
          float Av[4], Sv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {  // (A_p, S_p): half (p & 1) of group 1 + p / 2
            // group 1 + p / 2 = (A_{2k}, A_{2k+1}, S_{2k}, S_{2k+1}), k = p / 2 (kernels.cuh)
            const float4 g = valid ? zq[(1 + (p >> 1)) * MPAD + mb + j] : make_float4(0.f, 0.f, 0.f, 0.f);
            Av[j] = (p & 1) ? g.y : g.x;
            Sv[j] = (p & 1) ? g.w : g.z;
          }
          // offset d_p (for the skip x-part and layer-0 weight gradient)
          const float dpx = p == 0 ? u0 : (p == 1 ? v0 : (p == 2 ? u0 + v0 : u0 - v0));
          const float dpy = p == 0 ? u1 : (p == 1 ? v1 : (p == 2 ? u1 + v1 : u1 - v1));
          const float dpz = p == 0 ? u2 : (p == 1 ? v2 : (p == 2 ? u2 + v2 : u2 - v2));
          float dA[4], dS[4], pA[4], pS[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int m = mb + j;
            float XA, XS;
            if (top) {
              XA = wl[j] * dL[2 + 2 * p];
              XS = wl[j] * dL[3 + 2 * p];
            } else {
              const float2 x2 = *reinterpret_cast<const float2*>(act8 + act_idx<NC>(m, cg * 8 + 2 * p));
              XA = x2.x * xsc;
              XS = x2.y * xsc;
            }
            dA[j] = dS[j] = pA[j] = pS[j] = 0.f;
            if (m < M) {
              float Aa, Sa, P, Dd, Z;
              AF::pair_bwd(cc[j], Av[j], Sv[j], beta, &Aa, &Sa, &P, &Dd, &Z);
              dA[j] = om * fmaf(XA, P, 2.0f * XS * Dd);
              dS[j] = om * fmaf(0.5f * XA, Dd, XS * P);
              zbar[j] = fmaf(XA, Dd, fmaf(XS, Z, zbar[j]));
              pA[j] = Aa * xsc;
              pS[j] = Sa * xsc;
              if (top) vL[j] = fmaf(dL[2 + 2 * p], Aa, fmaf(dL[3 + 2 * p], Sa, vL[j]));
            } else if (nskip && m < M + 3) {
              const int d = m - M;
              pA[j] = h * (d == 0 ? dpx : (d == 1 ? dpy : dpz)) * xsc;
            }
            if (l == 0) {  // a^{-1} of pair columns: A -> h d_p, S -> 0
              w0p[j][0] = fmaf(dA[j], h * dpx, w0p[j][0]);
              w0p[j][1] = fmaf(dA[j], h * dpy, w0p[j][1]);
              w0p[j][2] = fmaf(dA[j], h * dpz, w0p[j][2]);
            }
          }
          if (store_del) {
            *reinterpret_cast<float4*>(delp + (2 + 2 * p) * MPAD + mb) = make_float4(dA[0], dA[1], dA[2], dA[3]);
            *reinterpret_cast<float4*>(delp + (3 + 2 * p) * MPAD + mb) = make_float4(dS[0], dS[1], dS[2], dS[3]);
          }
          if (store_act) {
            *reinterpret_cast<float4*>(actp + (2 + 2 * p) * MPAD + mb) = make_float4(pA[0], pA[1], pA[2], pA[3]);
            *reinterpret_cast<float4*>(actp + (3 + 2 * p) * MPAD + mb) = make_float4(pS[0], pS[1], pS[2], pS[3]);
          }
          if (l >= 1) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<float2*>(act8 + act_idx<NC>(mb + j, cg * 8 + 2 * p)) = make_float2(dA[j], dS[j]);
          }
        }

        // ---------------------------------------------------------------- centre + tangent
        float dc[4], dt[4], pc[4], pt[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int m = mb + j;
          float Xc, Xt;
          if (top) {
            Xc = wl[j] * dL[0];
            Xt = wl[j] * dL[1];
          } else {
            const float2 x2 = *reinterpret_cast<const float2*>(act2 + m * (CG * 2) + cg * 2);
            Xc = x2.x * xsc;
            Xt = x2.y * xsc;
          }
          dc[j] = dt[j] = pc[j] = pt[j] = 0.f;
          if (m < M) {
            const float s1 = AF::d1(cc[j], beta), s2 = AF::d2(cc[j], beta);
            const float zb = fmaf(Xc, s1, fmaf(s2 * tr[j], Xt, zbar[j]));
            dc[j] = om * zb;
            dt[j] = om * s1 * Xt;
            pc[j] = AF::value(cc[j], beta) * xsc;
            pt[j] = s1 * tr[j] * xsc;
            if (top) vL[j] = fmaf(dL[0], pc[j], fmaf(dL[1], pt[j], vL[j]));
          } else if (nskip && m < M + 3) {
            const int d = m - M;
            pc[j] = sd[16 + d] * xsc;
            pt[j] = (d == 0 ? r0 : (d == 1 ? r1 : r2)) * xsc;
          }
          if (l == 0) {  // a^{-1}: centre -> x0, tangent -> r
            w0p[j][0] = fmaf(dc[j], sd[16], fmaf(dt[j], r0, w0p[j][0]));
            w0p[j][1] = fmaf(dc[j], sd[17], fmaf(dt[j], r1, w0p[j][1]));
            w0p[j][2] = fmaf(dc[j], sd[18], fmaf(dt[j], r2, w0p[j][2]));
          }
        }
        if (store_del) {
          *reinterpret_cast<float4*>(delp + 0 * MPAD + mb) = make_float4(dc[0], dc[1], dc[2], dc[3]);
          *reinterpret_cast<float4*>(delp + 1 * MPAD + mb) = make_float4(dt[0], dt[1], dt[2], dt[3]);
        }
        if (store_act) {
          *reinterpret_cast<float4*>(actp + 0 * MPAD + mb) = make_float4(pc[0], pc[1], pc[2], pc[3]);
          *reinterpret_cast<float4*>(actp + 1 * MPAD + mb) = make_float4(pt[0], pt[1], pt[2], pt[3]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<float2*>(act2 + (mb + j) * (CG * 2) + cg * 2) = make_float2(dc[j], dt[j]);
        if (top) {
#pragma unroll
          for (int j = 0; j < 4; ++j) red[(mb + j) * CG + cg] = vL[j];
        }
        if (l == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int d = 0; d < 3; ++d) w0s[q][j][d] = w0p[j][d];
        }
      }
      bar_compute(NCT);
      if (l == 0) {  // act8 is dead now: dW_0 scratch [m][cg][3]
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int d = 0; d < 3; ++d)
              act8[((tile_row<MPAD>(rg, q * 4) + j) * CG + cg) * 3 + d] = w0s[q][j][d];
        bar_compute(NCT);
      }

      // ---------------------------------------------------------- fixed-order CTA reductions
      for (int m = tid; m < M; m += NCT) {
        float s = 0.f;
        for (int g = 0; g < CG; ++g) s += act2[m * (CG * 2) + g * 2];
        acc_db[(size_t)l * MPAD + m] += s;
        if (top) {
          float v = 0.f;
          for (int g = 0; g < CG; ++g) v += red[m * CG + g];
          acc_dWL[m] += v;
        }
        if (l == 0) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            float v = 0.f;
            for (int g = 0; g < CG; ++g) v += act8[(m * CG + g) * 3 + d];
            acc_dW0[m * 3 + d] += v;
          }
        }
      }
      if (top && tid == NCT - 1) {
        float v = 0.f;
        for (int g = 0; g < CG; ++g) v += sseed[g * 20 + 0];
        acc_dbL[0] += v;
      }
      if (l == 0) bar_compute(NCT);  // act8 scratch read before the next tile overwrites it
    }
  }
}

template <int ACT, int MPAD>
static cudaError_t launch_bwd_t(const BwdArgs& a, int grid, cudaStream_t st) {
  const size_t smem = BwdSmem<MPAD>::BYTES;
  cudaError_t e = smem_attr_once<bwd_kernel<ACT, MPAD>>((int)smem);
  if (e != cudaSuccess) return e;
  bwd_kernel<ACT, MPAD><<<grid, NTH, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bwd(const BwdArgs& a, int grid, cudaStream_t st) {
  const int act = a.net.act, mp = a.net.mpad;
#define FDSDF_CASE(A, M) \
  if (act == A && mp == M) return launch_bwd_t<A, M>(a, grid, st);
  FDSDF_CASE(ACT_SINE, 64)
  FDSDF_CASE(ACT_SINE, 128)
  FDSDF_CASE(ACT_SINE, 256)
  FDSDF_CASE(ACT_SINE, 512)
  FDSDF_CASE(ACT_SOFTPLUS, 64)
  FDSDF_CASE(ACT_SOFTPLUS, 128)
  FDSDF_CASE(ACT_SOFTPLUS, 256)
  FDSDF_CASE(ACT_SOFTPLUS, 512)
#undef FDSDF_CASE
  return cudaErrorInvalidValue;
}

int bwd_tile_centres(int mpad) { return NCT / (mpad / 8); }

size_t bwd_smem_bytes(int mpad) {
  switch (mpad) {
    case 64: return BwdSmem<64>::BYTES;
    case 128: return BwdSmem<128>::BYTES;
    case 256: return BwdSmem<256>::BYTES;
    default: return BwdSmem<512>::BYTES;
  }
}

}  // namespace fdsdf
