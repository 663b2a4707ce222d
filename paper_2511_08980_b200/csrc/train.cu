// train.cu -- the steps around fdsdf_step that make a full training iteration (SURVEY §8f
// NEXT-1; §4 "Datasets" P:L150 and "Methods and Setup" P:L153):
//
//   fdsdf_sample  per-iteration batch: n_pick of the n_pool surface samples WITHOUT
//                 replacement ("we sample 30k surface points; 20k are used per iteration",
//                 P:L150) followed by n_uniform fresh points uniform in the bounding box
//                 ("with 20k off-surface samples drawn uniformly in the bounding box").
//   fdsdf_adam    the Adam update ("Adam optimizer (5e-5)"; standard bias-corrected
//                 form), applied on the stream after the (allreduced) gradient.
//
// Both are counter-based, hence deterministic and shard-independent:
//   * subset: row j < n_pick takes pool index pi(j), pi a keyed pseudo-random permutation of
//     [0, n_pool): a 4-round balanced Feistel network on 2b bits (b = ceil(bits(n_pool-1)/2))
//     with round function mix64(key + (r+1)*gamma + R) & mask, cycle-walked into [0, n_pool);
//     key = mix64(seed ^ ((iteration + 1) * gamma2)).  Distinct j give distinct indices.
//   * box point j, coordinate d: U = (mix64(seed2 + ((iteration*n_uniform + j)*3 + d + 1) *
//     gamma) >> 11) * 2^-53, x = half * (2U - 1) in fp64, rounded to fp32; seed2 = mix64(~seed).
// The oracle (oracle/train_oracle.py) implements the same generators independently.
#include <algorithm>
#include <cmath>

#include "../../include/fdsdf.h"
#include "kernels.cuh"

namespace fdsdf {

namespace {
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kGamma2 = 0xD1B54A32D192ED03ull;

__host__ __device__ __forceinline__ uint64_t mix64_t(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t feistel(uint64_t x, uint64_t key, int b) {
  const uint64_t mask = (b >= 32) ? 0xFFFFFFFFull : ((1ull << b) - 1ull);
  uint64_t L = x >> b, R = x & mask;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint64_t nl = R;
    R = L ^ (mix64_t(key + (uint64_t)(r + 1) * kGamma + R) & mask);
    L = nl;
  }
  return (L << b) | R;
}

__global__ void sample_kernel(const float* __restrict__ pool, int64_t n_pool, int64_t n_pick, float half,
                              int64_t n_uniform, uint64_t seed, int64_t iteration, int b, float* __restrict__ out) {
  const uint64_t key = mix64_t(seed ^ ((uint64_t)(iteration + 1) * kGamma2));
  const uint64_t seed2 = mix64_t(~seed);
  const int64_t total = n_pick + n_uniform;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
    if (j < n_pick) {
      uint64_t x = (uint64_t)j;
      do {
        x = feistel(x, key, b);
      } while (x >= (uint64_t)n_pool);
      out[j * 3 + 0] = pool[x * 3 + 0];
      out[j * 3 + 1] = pool[x * 3 + 1];
      out[j * 3 + 2] = pool[x * 3 + 2];
    } else {
      const uint64_t ju = (uint64_t)(j - n_pick);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const uint64_t k = mix64_t(seed2 + (((uint64_t)iteration * (uint64_t)n_uniform + ju) * 3ull + d + 1ull) * kGamma);
        const double U = (double)(k >> 11) * 0x1.0p-53;
        out[j * 3 + d] = (float)((double)half * (2.0 * U - 1.0));
      }
    }
  }
}

// Adam (bias-corrected); c1 = lr / (1 - beta1^t), c2 = 1 / (1 - beta2^t) precomputed in fp64
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, int64_t n, float b1, float b2, float eps, double c1, double c2,
                            unsigned* dflags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    if (!isfinite(gi)) {  // non-finite gradient: leave this parameter untouched, flag it
      atomicOr(dflags, 8u);
      continue;
    }
    const float mi = fmaf(b1, m[i], (1.0f - b1) * gi);
    const float vi = fmaf(b2, v[i], (1.0f - b2) * gi * gi);
    m[i] = mi;
    v[i] = vi;
    const double vh = (double)vi * c2;
    p[i] = (float)((double)p[i] - c1 * (double)mi / (sqrt(vh) + (double)eps));
  }
}

}  // namespace

int feistel_half_bits(int64_t n_pool) {
  int bits = 1;
  while (bits < 62 && ((n_pool - 1) >> bits) > 0) ++bits;
  return (bits + 1) / 2;
}

cudaError_t launch_sample(const float* pool, int64_t n_pool, int64_t n_pick, float half, int64_t n_uniform,
                          uint64_t seed, int64_t iteration, float* out, cudaStream_t st) {
  const int64_t total = n_pick + n_uniform;
  const int grid = (int)std::min<int64_t>(1184, (total + 255) / 256);
  sample_kernel<<<grid, 256, 0, st>>>(pool, n_pool, n_pick, half, n_uniform, seed, iteration,
                                      feistel_half_bits(n_pool), out);
  return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                        float eps, int64_t t, unsigned* dflags, cudaStream_t st) {
  const double c1 = (double)lr / (1.0 - std::pow((double)b1, (double)t));
  const double c2 = 1.0 / (1.0 - std::pow((double)b2, (double)t));
  const int grid = (int)std::min<int64_t>(1184, (n + 255) / 256);
  adam_kernel<<<grid, 256, 0, st>>>(p, g, m, v, n, b1, b2, eps, c1, c2, dflags);
  return cudaGetLastError();
}

}  // namespace fdsdf

// ----------------------------------------------------------------------------- Hessian mode
// fdsdf_eval_hessian: the world-axis Hessian as three GIVEN-frame stencil
// passes with (u, v) = (e_a, e_b); these two kernels set the frames and scatter the pass's
// (f_uu, f_uv, f_vv) into H = (H_xx, H_xy, H_xz, H_yy, H_yz, H_zz).
namespace fdsdf {
__global__ void axis_frames_kernel(float* frames, int64_t n, int a, int b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 6; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % 6);
    frames[i] = (k < 3 ? (k == a) : (k - 3 == b)) ? 1.f : 0.f;
  }
}

// pass 0 (e_x, e_y): xx, xy, yy;  pass 1 (e_x, e_z): xz, zz;  pass 2 (e_y, e_z): yz
__global__ void hess_scatter_kernel(const float* __restrict__ t, float* __restrict__ H, int64_t n, int pass) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float fuu = t[i * 3 + 0], fuv = t[i * 3 + 1], fvv = t[i * 3 + 2];
    if (pass == 0) {
      H[i * 6 + 0] = fuu;
      H[i * 6 + 1] = fuv;
      H[i * 6 + 3] = fvv;
    } else if (pass == 1) {
      H[i * 6 + 2] = fuv;
      H[i * 6 + 5] = fvv;
    } else {
      H[i * 6 + 4] = fuv;
    }
  }
}

static int ew_grid(int64_t work) { return (int)std::min<int64_t>(std::max<int64_t>((work + 255) / 256, 1), 4096); }

cudaError_t launch_axis_frames(float* frames, int64_t n, int a, int b, cudaStream_t st) {
  axis_frames_kernel<<<ew_grid(n * 6), 256, 0, st>>>(frames, n, a, b);
  return cudaGetLastError();
}

// the (u, v) fields [4, 10) of the 16-float centre info of every row (fdepi.cuh layout)
__global__ void cinfo_axis_frames_kernel(float* cinfo, int64_t n, int a, int b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * 6; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % 6);
    cinfo[(i / 6) * 16 + 4 + k] = (k < 3 ? (k == a) : (k - 3 == b)) ? 1.f : 0.f;
  }
}

cudaError_t launch_cinfo_axis_frames(float* cinfo, int64_t n, int a, int b, cudaStream_t st) {
  cinfo_axis_frames_kernel<<<ew_grid(n * 6), 256, 0, st>>>(cinfo, n, a, b);
  return cudaGetLastError();
}

cudaError_t launch_hess_scatter(const float* t, float* H, int64_t n, int pass, cudaStream_t st) {
  hess_scatter_kernel<<<ew_grid(n), 256, 0, st>>>(t, H, n, pass);
  return cudaGetLastError();
}
}  // namespace fdsdf
