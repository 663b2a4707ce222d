// fwd.cu -- fused stencil-MLP forward + FD epilogue.
//
// One persistent CTA per (SM, slot) walks a static list of tiles of TILE = 2*CG centres.
//   phase 1: columns (f, d/dx, d/dy, d/dz) of every centre through all layers (forward-mode
//            tangents give g = grad f); then per centre: mask, right-handed random
//            frame (u, v).
//   phase 2: for each half of the tile, the 8 pair columns (A, S) x {u, v, u+v, u-v}
//            (act.cuh) through all layers; then the FD epilogue per centre: f_uu, f_vv, f_uv
//            (P:L83-91), D_FD, K_FD, the Eq. (1) terms
//             with a fixed-order fp64 tile reduction, and the backward seeds.
// Layer weights stream through shared memory with the TMA bulk engine (tile.cuh); all
// activations of the tile stay in shared memory.  In step mode the pre-activations of every
// stored column are written to the workspace for the backward kernel.
#include "act.cuh"
#include "fdepi.cuh"
#include "tile.cuh"

namespace fdsdf {

template <int MPAD>
struct FwdSmem {
  using T = TileCfg<MPAD, 16384, 3>;
  static constexpr int TILE = 2 * T::CG;
  static constexpr int ACT = MPAD * T::NC;
  static constexpr int WST = T::NSTG * T::SLAB;
  static constexpr int RED = T::RGW * T::NC;
  static constexpr int CINFO = TILE * 16;
  static constexpr size_t BYTES =
      (size_t)(ACT + WST + RED + CINFO) * 4 + (size_t)TILE * NLOSS * 8 + 2 * T::NSTG * 8 + 64;
};

template <int ACT, int MPAD>
__global__ void __launch_bounds__(NTH, 2) fwd_kernel(const FwdArgs a) {
  using S = FwdSmem<MPAD>;
  using T = typename S::T;
  using AF = Act<ACT>;
  constexpr int TILE = S::TILE;
  constexpr int RG = T::RG, CG = T::CG, NC = T::NC;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* act = reinterpret_cast<float*>(smem_raw);
  float* wst = act + S::ACT;
  float* red = wst + S::WST;
  float* cinfo = red + S::RED;
  double* lossv = reinterpret_cast<double*>(cinfo + S::CINFO);
  uint64_t* full = reinterpret_cast<uint64_t*>(lossv + TILE * NLOSS);
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
  WStream<T> ws;
  ws.layers = net.Wt;
  ws.L = L;
  ws.backward = 0;
  ws.per_tile = 3u * (uint32_t)(L - 2) * T::NCHUNK;
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
  const bool step = a.step != 0;
  const int zcols = step ? NCOLF : 1;
  float* zbase = step ? a.zf : a.zf + (size_t)blockIdx.x * TILE * nh * MPAD;
  const float isq2 = 0.70710678118654752f;
  uint32_t it = 0;
  double lacc[NLOSS];
#pragma unroll
  for (int q = 0; q < NLOSS; ++q) lacc[q] = 0.0;

  // stored pre-activations of layer l for tile slot / centre c: step -> float4 group g of
  // neuron m (kernels.cuh zf layout); eval scratch -> the centre values, [MPAD]
  auto zg4 = [&](int64_t c, int l, int g, int m) -> float4* {
    return reinterpret_cast<float4*>(zbase + ((c * nh + l) * zcols + 4 * g) * (int64_t)MPAD) + m;
  };
  auto zev = [&](int slot, int l) -> float* { return zbase + ((int64_t)slot * nh + l) * (int64_t)MPAD; };

  float acc[8][8];
  float acc2[8][2];

  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t c0 = tile * TILE;

    // ============================================================== phase 1: f and grad f
    for (int l = 0; l <= L - 2; ++l) {
      if (l > 0) {
        tile_gemm<T, false>(acc, acc2, act, nullptr, ws, it, rg, cg, tid);
        bar_compute(NCT);  // every thread is done reading act
      }
      const float om = net.omega[l];
      const int M = net.width[l + 1];
      const bool last = (l == L - 2);
      const bool nskip = (l + 1 == net.skip);
      const float osc = nskip ? isq2 : 1.0f;
      const float* __restrict__ bl = net.b[l];
      const float* __restrict__ Wl = net.W[l];
      const float* __restrict__ Wlast = net.W[L - 1];
      float part[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) part[j] = 0.f;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int slot = 2 * cg + e;
        const int64_t c = c0 + slot;
        const bool valid = c < a.n;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f;
        if (l == 0 || nskip) {
          if (valid) {
            x0 = a.x[c * 3 + 0];
            x1 = a.x[c * 3 + 1];
            x2 = a.x[c * 3 + 2];
            if (l == 0 && rg == 0 && !(isfinite(x0) && isfinite(x1) && isfinite(x2)))
              atomicOr(a.dflags, 1u);
          }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float zv[4], tv[4][3];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int i = q * 4 + j;
            const int m = tile_row<MPAD>(rg, i);
            float z = 0.f, t0 = 0.f, t1 = 0.f, t2 = 0.f;
            if (m < M) {
              if (l == 0) {
                const float w0 = Wl[m * 3 + 0], w1 = Wl[m * 3 + 1], w2 = Wl[m * 3 + 2];
                z = om * (fmaf(w0, x0, fmaf(w1, x1, w2 * x2)) + bl[m]);
                t0 = om * w0;
                t1 = om * w1;
                t2 = om * w2;
              } else {
                z = om * (acc[i][4 * e + 0] + bl[m]);
                t0 = om * acc[i][4 * e + 1];
                t1 = om * acc[i][4 * e + 2];
                t2 = om * acc[i][4 * e + 3];
              }
            }
            zv[j] = z;
            tv[j][0] = t0;
            tv[j][1] = t1;
            tv[j][2] = t2;
          }
          const int mb = tile_row<MPAD>(rg, q * 4);
          if (valid) {
            if (step) {
#pragma unroll
              for (int j = 0; j < 4; ++j) *zg4(c, l, 0, mb + j) = make_float4(zv[j], tv[j][0], tv[j][1], tv[j][2]);
            } else {
              *reinterpret_cast<float4*>(zev(slot, l) + mb) = make_float4(zv[0], zv[1], zv[2], zv[3]);
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int i = q * 4 + j;
            const int m = mb + j;
            float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
            if (m < M) {
              const typename AF::C cc = AF::centre(zv[j], beta);
              const float s1 = AF::d1(cc, beta);
              o0 = AF::value(cc, beta);
              o1 = s1 * tv[j][0];
              o2 = s1 * tv[j][1];
              o3 = s1 * tv[j][2];
            } else if (nskip && m < M + 3) {  // x-part of cat(a, x)
              const int d = m - M;
              o0 = d == 0 ? x0 : (d == 1 ? x1 : x2);
              o1 = d == 0 ? 1.f : 0.f;
              o2 = d == 1 ? 1.f : 0.f;
              o3 = d == 2 ? 1.f : 0.f;
            }
            if (last) {
              const float wl = (m < M) ? Wlast[m] : 0.f;
              part[4 * e + 0] = fmaf(wl, o0, part[4 * e + 0]);
              part[4 * e + 1] = fmaf(wl, o1, part[4 * e + 1]);
              part[4 * e + 2] = fmaf(wl, o2, part[4 * e + 2]);
              part[4 * e + 3] = fmaf(wl, o3, part[4 * e + 3]);
            } else {
              *reinterpret_cast<float4*>(act + act_idx<NC>(m, cg * 8 + 4 * e)) =
                  make_float4(o0 * osc, o1 * osc, o2 * osc, o3 * osc);
            }
          }
        }
      }
      if (last) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float v = part[j];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          part[j] = v;
        }
        if ((lane & 7) == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j) red[wr * NC + cg * 8 + j] = part[j];
        }
      }
      bar_compute(NCT);
    }

    // -------------------------------------------------------------- per centre: g -> frame
    if (tid < TILE) {
      const int slot = tid;
      const int64_t c = c0 + slot;
      const int col = (slot >> 1) * 8 + (slot & 1) * 4;
      float tot[4];
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        float v = 0.f;
        for (int w = 0; w < T::RGW; ++w) v += red[w * NC + col + d];
        tot[d] = v;
      }
      const float f = tot[0] + net.b[L - 1][0];
      centre_frame(a, c, c < a.n, f, tot[1], tot[2], tot[3], cinfo + slot * 16);
    }
    bar_compute(NCT);

    // ============================================================== phase 2: 4 stencil pairs
    for (int half = 0; half < 2; ++half) {
      const int slot = half * CG + cg;
      const int64_t c = c0 + slot;
      const bool valid = c < a.n;
      const float* ci = cinfo + slot * 16;
      for (int l = 0; l <= L - 2; ++l) {
        // prefetch the centre pre-activations of this layer (written in phase 1)
        float zpre[8];
        if (step) {
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int j = 0; j < 4; ++j) zpre[4 * q + j] = valid ? zg4(c, l, 0, tile_row<MPAD>(rg, 4 * q) + j)->x : 0.f;
        } else {
          const float4 z0 = valid ? *reinterpret_cast<const float4*>(zev(slot, l) + tile_row<MPAD>(rg, 0))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          const float4 z1 = valid ? *reinterpret_cast<const float4*>(zev(slot, l) + tile_row<MPAD>(rg, 4))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
          zpre[0] = z0.x; zpre[1] = z0.y; zpre[2] = z0.z; zpre[3] = z0.w;
          zpre[4] = z1.x; zpre[5] = z1.y; zpre[6] = z1.z; zpre[7] = z1.w;
        }
        if (l > 0) {
          tile_gemm<T, false>(acc, acc2, act, nullptr, ws, it, rg, cg, tid);
          bar_compute(NCT);
        }
        const float om = net.omega[l];
        const int M = net.width[l + 1];
        const bool last = (l == L - 2);
        const bool nskip = (l + 1 == net.skip);
        const float osc = nskip ? isq2 : 1.0f;
        const float* __restrict__ Wl = net.W[l];
        const float* __restrict__ Wlast = net.W[L - 1];
        const float u0 = ci[4], u1 = ci[5], u2 = ci[6], v0 = ci[7], v1 = ci[8], v2 = ci[9];
        float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          float Av[4][4], Sv[4][4];  // [row j][pair]
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int i = q * 4 + j;
            const int m = tile_row<MPAD>(rg, i);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              Av[j][p] = 0.f;
              Sv[j][p] = 0.f;
            }
            if (m < M) {
              if (l == 0) {
                const float w0 = Wl[m * 3 + 0], w1 = Wl[m * 3 + 1], w2 = Wl[m * 3 + 2];
                const float du = fmaf(w0, u0, fmaf(w1, u1, w2 * u2));
                const float dv = fmaf(w0, v0, fmaf(w1, v1, w2 * v2));
                const float hs = om * h;
                Av[j][0] = hs * du;
                Av[j][1] = hs * dv;
                Av[j][2] = hs * (du + dv);
                Av[j][3] = hs * (du - dv);
              } else {
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                  Av[j][p] = om * acc[i][2 * p];
                  Sv[j][p] = om * acc[i][2 * p + 1];
                }
              }
            }
          }
          const int mb = tile_row<MPAD>(rg, q * 4);
          if (step && valid) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              *zg4(c, l, 1, mb + j) = make_float4(Av[j][0], Av[j][1], Sv[j][0], Sv[j][1]);
              *zg4(c, l, 2, mb + j) = make_float4(Av[j][2], Av[j][3], Sv[j][2], Sv[j][3]);
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int m = mb + j;
            float o[8];
#pragma unroll
            for (int p = 0; p < 8; ++p) o[p] = 0.f;
            if (m < M) {
              const typename AF::C cc = AF::centre(zpre[q * 4 + j], beta);
#pragma unroll
              for (int p = 0; p < 4; ++p) AF::pair_fwd(cc, Av[j][p], Sv[j][p], beta, &o[2 * p], &o[2 * p + 1]);
            } else if (nskip && m < M + 3) {  // x-part: odd part = offset, even part = 0
              const int d = m - M;
              const float ud = d == 0 ? u0 : (d == 1 ? u1 : u2);
              const float vd = d == 0 ? v0 : (d == 1 ? v1 : v2);
              o[0] = h * ud;
              o[2] = h * vd;
              o[4] = h * (ud + vd);
              o[6] = h * (ud - vd);
            }
            if (last) {
              const float wl = (m < M) ? Wlast[m] : 0.f;
#pragma unroll
              for (int p = 0; p < 4; ++p) part[p] = fmaf(wl, o[2 * p + 1], part[p]);
            } else {
              *reinterpret_cast<float4*>(act + act_idx<NC>(m, cg * 8)) =
                  make_float4(o[0] * osc, o[1] * osc, o[2] * osc, o[3] * osc);
              *reinterpret_cast<float4*>(act + act_idx<NC>(m, cg * 8 + 4)) =
                  make_float4(o[4] * osc, o[5] * osc, o[6] * osc, o[7] * osc);
            }
          }
        }
        if (last) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            float v = part[p];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            part[p] = v;
          }
          if ((lane & 7) == 0) {
#pragma unroll
            for (int p = 0; p < 4; ++p) red[wr * NC + cg * 8 + p] = part[p];
          }
        }
        bar_compute(NCT);
      }

      // ------------------------------------------------------------ FD epilogue per centre
      if (tid < CG) {
        const int slot2 = half * CG + tid;
        const int64_t cc = c0 + slot2;
        const bool valid2 = cc < a.n;
        float Ssum[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          float v = 0.f;
          for (int w = 0; w < T::RGW; ++w) v += red[w * NC + tid * 8 + p];
          Ssum[p] = v;
        }
        double lv[NLOSS];
        fd_centre(a, cc, valid2, Ssum, cinfo + slot2 * 16, lv);
#pragma unroll
        for (int q = 0; q < NLOSS; ++q) lossv[slot2 * NLOSS + q] = lv[q];
      }
      bar_compute(NCT);
    }
    // fixed-order tile reduction of the loss terms
    if (tid == 0) {
      for (int s = 0; s < TILE; ++s)
#pragma unroll
        for (int q = 0; q < NLOSS; ++q) lacc[q] += lossv[s * NLOSS + q];
    }
  }
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NLOSS; ++q) a.lossp[(size_t)blockIdx.x * NLOSS + q] = lacc[q];
  }
}

// ----------------------------------------------------------------------------- host launch

template <int ACT, int MPAD>
static cudaError_t launch_fwd_t(const FwdArgs& a, int grid, cudaStream_t st) {
  const size_t smem = FwdSmem<MPAD>::BYTES;
  cudaError_t e = smem_attr_once<fwd_kernel<ACT, MPAD>>((int)smem);
  if (e != cudaSuccess) return e;
  fwd_kernel<ACT, MPAD><<<grid, NTH, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fwd(const FwdArgs& a, int grid, cudaStream_t st) {
  const int act = a.net.act, mp = a.net.mpad;
#define FDSDF_CASE(A, M) \
  if (act == A && mp == M) return launch_fwd_t<A, M>(a, grid, st);
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

int fwd_tile_centres(int mpad) { return 2 * (NCT / (mpad / 8)); }

size_t fwd_smem_bytes(int mpad) {
  switch (mpad) {
    case 64: return FwdSmem<64>::BYTES;
    case 128: return FwdSmem<128>::BYTES;
    case 256: return FwdSmem<256>::BYTES;
    default: return FwdSmem<512>::BYTES;
  }
}

}  // namespace fdsdf
