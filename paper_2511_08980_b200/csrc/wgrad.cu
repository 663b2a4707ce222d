// wgrad.cu -- weight packing, split-K weight-gradient contraction and the fixed-order final
// reduction.
//
//   dW_l[m][k] = sum_j delta_l[j][m] * a_{l-1}[j][k]     j over (centre, column): 10 per centre
// Each CTA owns a BMxBM block of dW_l and a contiguous j-range (split-K); its partial is written
// (not atomically added) and `finalize_kernel` sums the partials of every element in split
// order, so results are bitwise reproducible.
#include "common.cuh"
#include "kernels.cuh"

namespace fdsdf {

// ----------------------------------------------------------------------------- pack
// Wt[l][k][m] = W_l[m][k], Wb[l][m][k] = W_l[m][k], zero padded to [mpad][mpad], GEMM layers.
__global__ void pack_kernel(const Net net, float* wt, float* wb) {
  const int mp = net.mpad;
  const int l = blockIdx.y + 1;
  const int M = net.width[l + 1];
  const int K = net.width[l] + (l == net.skip ? 3 : 0);
  const float* W = net.W[l];
  float* t = wt + (size_t)(l - 1) * mp * mp;
  float* b = wb + (size_t)(l - 1) * mp * mp;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < mp * mp; idx += gridDim.x * blockDim.x) {
    const int r = idx / mp, cidx = idx % mp;
    // wb: row r = m, col = k
    b[idx] = (r < M && cidx < K) ? W[(size_t)r * K + cidx] : 0.f;
    // wt: row r = k, col = m
    t[idx] = (cidx < M && r < K) ? W[(size_t)cidx * K + r] : 0.f;
  }
}

cudaError_t launch_pack(const Net& net, float* wt, float* wb, cudaStream_t st) {
  if (net.L <= 2) return cudaSuccess;
  dim3 grid(64, net.L - 2);
  pack_kernel<<<grid, 256, 0, st>>>(net, wt, wb);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- split-K wgrad
template <int BM>
struct WgCfg {
  static constexpr int TT = BM / 16;     // thread tile (TT x TT), 16x16 threads
  static constexpr int JC = 16;          // j rows per stage
  static constexpr int NST = 3;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int BM>
__global__ void __launch_bounds__(256, 2) wgrad_kernel(const WgradArgs a) {
  using C = WgCfg<BM>;
  constexpr int TT = C::TT, JC = C::JC, NST = C::NST;
  __shared__ __align__(16) float Ds[NST][JC][BM];
  __shared__ __align__(16) float As[NST][JC][BM];
  const int mp = a.mpad;
  const int nb = mp / BM;
  const int bm = blockIdx.x / nb, bk = blockIdx.x % nb;
  const int split = blockIdx.y;
  const int layer = a.first_layer + blockIdx.z;       // GEMM layer l: delta_l, a_{l-1}
  const float* D = a.del + (size_t)layer * a.stride_layer;
  const float* A = a.actv + (size_t)(layer - 1) * a.stride_layer;
  const int64_t per = ((a.rows + a.nsplit - 1) / a.nsplit + JC - 1) / JC * JC;
  const int64_t j0 = (int64_t)split * per;
  const int64_t j1 = min(a.rows, j0 + per);
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  float acc[TT][TT];
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < TT; ++j) acc[i][j] = 0.f;

  const int nstage_iters = j1 > j0 ? (int)((j1 - j0 + JC - 1) / JC) : 0;
  // loader: JC*BM/4 float4 per matrix per stage
  constexpr int NV = JC * BM / 4;
  auto load = [&](int stg, int64_t jb) {
    for (int v = tid; v < NV; v += 256) {
      const int jj = v / (BM / 4), cc = (v % (BM / 4)) * 4;
      const int64_t j = jb + jj;
      const bool ok = j < j1;
      const int64_t jr = ok ? j : j0;
      cp_async16(&Ds[stg][jj][cc], D + jr * mp + bm * BM + cc, ok);
      cp_async16(&As[stg][jj][cc], A + jr * mp + bk * BM + cc, ok);
    }
  };
#pragma unroll
  for (int s = 0; s < NST - 1; ++s) {
    if (s < nstage_iters) load(s, j0 + (int64_t)s * JC);
    cp_async_commit();
  }
  constexpr int H = BM / 2;  // rows {ty*TT/2 + i} and {H + ty*TT/2 + i}
  for (int itn = 0; itn < nstage_iters; ++itn) {
    cp_async_wait<NST - 2>();
    __syncthreads();
    {
      const int nx = itn + NST - 1;
      if (nx < nstage_iters) load(nx % NST, j0 + (int64_t)nx * JC);
      cp_async_commit();
    }
    const int s = itn % NST;
#pragma unroll
    for (int jj = 0; jj < JC; ++jj) {
      float dv[TT], av[TT];
#pragma unroll
      for (int i = 0; i < TT / 2; ++i) {
        dv[i] = Ds[s][jj][ty * (TT / 2) + i];
        dv[TT / 2 + i] = Ds[s][jj][H + ty * (TT / 2) + i];
        av[i] = As[s][jj][tx * (TT / 2) + i];
        av[TT / 2 + i] = As[s][jj][H + tx * (TT / 2) + i];
      }
#pragma unroll
      for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TT; ++j) acc[i][j] = fmaf(dv[i], av[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();
  float* out = a.part + ((size_t)blockIdx.z * a.nsplit + split) * mp * mp;
#pragma unroll
  for (int i = 0; i < TT; ++i) {
    const int m = bm * BM + (i < TT / 2 ? ty * (TT / 2) + i : H + ty * (TT / 2) + i - TT / 2);
#pragma unroll
    for (int j = 0; j < TT; ++j) {
      const int k = bk * BM + (j < TT / 2 ? tx * (TT / 2) + j : H + tx * (TT / 2) + j - TT / 2);
      out[(size_t)m * mp + k] = acc[i][j];
    }
  }
}

cudaError_t launch_wgrad(const WgradArgs& a, int nglayers, cudaStream_t st) {
  if (nglayers <= 0) return cudaSuccess;
  const int BM = a.mpad >= 128 ? 128 : 64;
  const int nb = a.mpad / BM;
  dim3 grid(nb * nb, a.nsplit, nglayers);
  if (BM == 128)
    wgrad_kernel<128><<<grid, 256, 0, st>>>(a);
  else
    wgrad_kernel<64><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- finalize
// sum_{s < n} p[s * stride] in the fixed order s = 0, 1, ..., with 8 loads in flight
__device__ __forceinline__ float sum_strided(const float* __restrict__ p, int64_t stride, int n) {
  float v = 0.f;
  int s = 0;
  for (; s + 8 <= n; s += 8) {
    float t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = __ldg(p + (size_t)(s + q) * stride);
#pragma unroll
    for (int q = 0; q < 8; ++q) v += t[q];
  }
  for (; s < n; ++s) v += __ldg(p + (size_t)s * stride);
  return v;
}

// grid.y = layer (0..L-1), plus one extra block row for the loss.
__global__ void finalize_kernel(const FinArgs a) {
  const Net& net = a.net;
  const int L = net.L, mp = net.mpad;
  const int l = blockIdx.y;
  if (l == L) {  // loss: fixed-order sum over forward CTAs
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double s[NLOSS];
      for (int q = 0; q < NLOSS; ++q) s[q] = 0.0;
      for (int c = 0; c < a.nfcta; ++c)
        for (int q = 0; q < NLOSS; ++q) s[q] += a.lossp[(size_t)c * NLOSS + q];
      const LossCfg& ls = a.ls;
      const double dm = s[0] * ls.inv_ns, dnm = s[1] * ls.inv_nu, eik = s[2] * ls.inv_n, fd = s[3] * ls.inv_n;
      const double tot = (double)ls.w_dm * dm + (double)ls.lambda_dnm * dnm + (double)ls.lambda_eik * eik +
                         (double)ls.lambda_fd * fd;
      a.loss[0] = dm;
      a.loss[1] = dnm;
      a.loss[2] = eik;
      a.loss[3] = fd;
      a.loss[4] = tot;
      a.loss[5] = s[4];
      a.loss[6] = 0.0;
      a.loss[7] = 0.0;
      unsigned fl = 0;
      if (!isfinite(tot)) fl |= 2u;
      if (a.n_local > 0 && s[4] >= (double)a.n_local) fl |= 4u;
      if (fl) atomicOr(a.dflags, fl);
    }
    return;
  }
  const int M = net.width[l + 1];
  const int K = net.width[l] + (l == net.skip ? 3 : 0);
  // flat offsets: recomputed from the widths (W_l then b_l per layer)
  int64_t off = 0;
  for (int q = 0; q < l; ++q) {
    const int Mq = net.width[q + 1], Kq = net.width[q] + (q == net.skip ? 3 : 0);
    off += (int64_t)Mq * Kq + Mq;
  }
  float* gW = a.grad + off;
  float* gb = gW + (int64_t)M * K;
  const int64_t nW = (int64_t)M * K;
  const int64_t oWL = (int64_t)(L - 1) * mp, obL = oWL + mp, oW0 = obL + 1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nW + M;
       idx += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (idx < nW) {
      const int m = (int)(idx / K), k = (int)(idx % K);
      if (l == L - 1) {
        v = sum_strided(a.bacc + oWL + k, a.nacc, a.nbcta);
      } else if (l == 0) {
        v = sum_strided(a.bacc + oW0 + m * 3 + k, a.nacc, a.nbcta);
      } else {
        const float* p = a.part + (size_t)(l - 1) * a.nsplit * mp * mp + (size_t)m * mp + k;
        v = sum_strided(p, (int64_t)mp * mp, a.nsplit);
      }
      if (a.accumulate) v += gW[idx];
      gW[idx] = v;
    } else {
      const int m = (int)(idx - nW);
      if (l == L - 1) {
        v = sum_strided(a.bacc + obL, a.nacc, a.nbcta);
      } else {
        v = sum_strided(a.bacc + (size_t)l * mp + m, a.nacc, a.nbcta);
      }
      if (a.accumulate) v += gb[m];
      gb[m] = v;
    }
  }
}

cudaError_t launch_finalize(const FinArgs& a, cudaStream_t st) {
  const int mp = a.net.mpad;
  dim3 grid(std::max(64, (mp * mp + mp + 255) / 256), a.net.L + 1);
  finalize_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

__global__ void add_kernel(float* y, const float* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

cudaError_t launch_add_inplace(float* y, const float* x, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>(1184, (n + 255) / 256);
  add_kernel<<<grid, 256, 0, st>>>(y, x, n);
  return cudaGetLastError();
}

}  // namespace fdsdf
