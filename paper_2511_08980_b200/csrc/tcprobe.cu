// tcprobe.cu -- self-test of the tcgen05 bf16x6 contraction core (tc.cuh) on a plain GEMM.
//
//   D[m][n] = sum_k W[m][k] * B[n][k]        (W: [M][K] row-major, B: [N][K] row-major)
//
// One CTA, synchronous K loop: the 256 threads split each K chunk of W and B into bf16
// pieces and store them in the K-major SWIZZLE_128B layout, one thread issues the
// (M/128) x 4 x nprod tcgen05.mma per chunk, tcgen05.commit signals an mbarrier, and at the
// end every warp reads its TMEM lane quarter with tcgen05.ld.  It exercises exactly the
// descriptors, instruction descriptor, swizzle and TMEM mapping of the production kernels,
// so a layout error shows up here as a wrong GEMM rather than as a wrong curvature.
#include "../../include/fdsdf.h"
#include "tc.cuh"

namespace fdsdf {

__global__ void __launch_bounds__(256, 1) tcprobe_kernel(const float* __restrict__ W, const float* __restrict__ B,
                                                         float* __restrict__ D, int M, int N, int K, int nprod,
                                                         int mn) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // carve: A pieces [3][M x 128 B], B pieces [3][N x 128 B], mbarrier, tmem slot
  unsigned char* base = smem_raw;
  {
    const uint32_t a = smem_u32(base);
    base += (1024 - (a & 1023)) & 1023;
  }
  // MN-major: N may be a partial swizzle atom (N % 64 != 0): the B pieces take whole 64-column atoms
  const int NA = mn ? (N + 63) / 64 * 64 : N;
  unsigned char* As = base;
  unsigned char* Bs = As + 3 * M * 128;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bs + 3 * NA * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int MH = M / 128;
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(MH * N)) ncols <<= 1;

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, ncols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t idesc = mn ? tc::idesc_bf16(128, N, 1, 1) : tc::idesc_bf16(128, N);
  // MN-major strides: atoms along MN are 1024 B apart, along K (M/64)*1024 resp. (N/64)*1024
  const uint32_t a_mn = 1024, a_k = (uint32_t)(M / 64) * 1024, b_mn = 1024, b_k = (uint32_t)(NA / 64) * 1024;
  const int q0 = nprod == 1 ? 5 : (nprod == 3 ? 3 : 0);

  for (int kc = 0; kc < K / 64; ++kc) {
    // stage chunk kc: element (r, k) of the chunk, split into 3 pieces
    for (int i = tid; i < M * 64; i += 256) {
      const int r = i >> 6, k = i & 63;
      const tc::Bf3 s = tc::split3(W[(size_t)r * K + kc * 64 + k]);
      const uint32_t o = mn ? tc::sw128mn_off(r, k, M) : tc::sw128_off(r, k, M);
#pragma unroll
      for (int p = 0; p < 3; ++p) *reinterpret_cast<__nv_bfloat16*>(As + p * M * 128 + o) = s.p[p];
    }
    for (int i = tid; i < N * 64; i += 256) {
      const int r = i >> 6, k = i & 63;
      const tc::Bf3 s = tc::split3(B[(size_t)r * K + kc * 64 + k]);
      const uint32_t o = mn ? tc::sw128mn_off(r, k, NA) : tc::sw128_off(r, k, N);
#pragma unroll
      for (int p = 0; p < 3; ++p) *reinterpret_cast<__nv_bfloat16*>(Bs + p * NA * 128 + o) = s.p[p];
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      for (int s = 0; s < 4; ++s)
        for (int h = 0; h < MH; ++h)
          for (int q = q0; q < 6; ++q) {
            uint64_t ad, bd;
            if (!mn) {
              ad = tc::sdesc_sw128(smem_u32(As + tc::prod_a(q) * M * 128 + h * 128 * 128 + s * 32));
              bd = tc::sdesc_sw128(smem_u32(Bs + tc::prod_b(q) * NA * 128 + s * 32));
            } else {
              // K step s = 16 K = 2 atoms along K; M-half h = 2 atoms along M
              const uint32_t aa = smem_u32(As + tc::prod_a(q) * M * 128 + 2 * s * a_k + 2 * h * a_mn);
              const uint32_t bb = smem_u32(Bs + tc::prod_b(q) * NA * 128 + 2 * s * b_k);
              ad = tc::sdesc_sw128_mn(aa, a_mn, a_k);
              bd = tc::sdesc_sw128_mn(bb, b_mn, b_k);
            }
            tc::mma_bf16(tbase + h * N, ad, bd, idesc, (kc | s | (q - q0)) != 0 ? 1u : 0u);
          }
      tc::mma_commit(bar);
    }
    mbar_wait(bar, kc & 1);
    tc::fence_after();
  }
  // epilogue: warp w reads lane quarter w%4 of M-halves h = w/4, w/4 + 2, ...
  for (int h = warp >> 2; h < MH; h += 2) {
    const int m = h * 128 + 32 * (warp & 3) + (tid & 31);
    for (int n0 = 0; n0 < N; n0 += 8) {
      float v[8];
      tc::tmem_ld8(tbase + tc::tmem_lane_base(warp) + h * N + n0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) D[(size_t)m * N + n0 + j] = v[j];
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, ncols);
}

}  // namespace fdsdf

extern "C" fdsdf_status fdsdf_selftest_mma(const float* d_W, const float* d_B, float* d_D, int M, int N, int K,
                                           int nprod, int mn_major, void* stream) {
  using namespace fdsdf;
  if (!d_W || !d_B || !d_D) return FDSDF_E_INVALID;
  if (M < 128 || M > 256 || M % 128 || N < 16 || N > 256 || N % 16 || K < 64 || K % 64) return FDSDF_E_INVALID;
  if (nprod != 1 && nprod != 3 && nprod != 6) return FDSDF_E_INVALID;
  if (mn_major < 0 || mn_major > 1) return FDSDF_E_INVALID;
  const size_t smem = 3 * (size_t)(M + (N + 63) / 64 * 64) * 128 + 64 + 1024;
  cudaError_t e = cudaFuncSetAttribute(tcprobe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return FDSDF_E_CUDA;
  tcprobe_kernel<<<1, 256, smem, (cudaStream_t)stream>>>(d_W, d_B, d_D, M, N, K, nprod, mn_major);
  return cudaGetLastError() == cudaSuccess ? FDSDF_OK : FDSDF_E_CUDA;
}

// ----------------------------------------------------------------------------- CTA-pair probe
// D[256][N] = W[256][K] . B[N][K]^T on a CTA pair (cluster of 2, tcgen05 cta_group::2):
// CTA r stages W rows [128 r, 128 r + 128) and B rows [N/2 r, N/2 (r + 1)) (bf16x3 pieces,
// K-major SW128) at the SAME shared-memory offsets; the leader (rank 0) issues M = 256 MMAs
// that read both CTAs' operands; the commit is multicast to both CTAs' mbarriers; each CTA
// reads its own 128 TMEM lanes (rows 128 r ..) back.  Validates the pair mechanics used by the
// pair-tiled kernels.
namespace fdsdf {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    tcprobe2_kernel(const float* __restrict__ W, const float* __restrict__ B, float* __restrict__ D, int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw;
  base += (1024 - (smem_u32(base) & 1023)) & 1023;
  const int NH = N / 2;
  unsigned char* As = base;                 // [3][128 rows x 128 B]
  unsigned char* Bs = As + 3 * 128 * 128;   // [3][NH rows x 128 B]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bs + 3 * NH * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_ctarank();
  uint32_t ncols = 32;
  while (ncols < (uint32_t)N) ncols <<= 1;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::fence_before();
  cluster_sync_all();
  tc::fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t idesc = tc::idesc_bf16(256, N);
  for (int kc = 0; kc < K / 64; ++kc) {
    for (int i = tid; i < 128 * 64; i += 256) {
      const int r = i >> 6, k = i & 63;
      const tc::Bf3 s = tc::split3(W[(size_t)(128 * rank + r) * K + kc * 64 + k]);
      const uint32_t o = tc::sw128_off(r, k, 128);
#pragma unroll
      for (int p = 0; p < 3; ++p) *reinterpret_cast<__nv_bfloat16*>(As + p * 128 * 128 + o) = s.p[p];
    }
    for (int i = tid; i < NH * 64; i += 256) {
      const int r = i >> 6, k = i & 63;
      const tc::Bf3 s = tc::split3(B[(size_t)(NH * rank + r) * K + kc * 64 + k]);
      const uint32_t o = tc::sw128_off(r, k, NH);
#pragma unroll
      for (int p = 0; p < 3; ++p) *reinterpret_cast<__nv_bfloat16*>(Bs + p * NH * 128 + o) = s.p[p];
    }
    fence_proxy_async();
    tc::fence_before();
    cluster_sync_all();  // both CTAs' operands of this chunk are in place
    if (rank == 0 && tid == 0) {
      tc::fence_after();
      for (int s = 0; s < 4; ++s)
        for (int q = 0; q < 6; ++q) {
          const uint64_t ad = tc::sdesc_sw128(smem_u32(As + tc::prod_a(q) * 128 * 128 + s * 32));
          const uint64_t bd = tc::sdesc_sw128(smem_u32(Bs + tc::prod_b(q) * NH * 128 + s * 32));
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
              "l"(ad), "l"(bd), "r"(idesc), "r"((kc | s | q) != 0 ? 1u : 0u)
              : "memory");
        }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(bar)),
          "h"((uint16_t)3)
          : "memory");
    }
    mbar_wait(bar, kc & 1);
    tc::fence_after();
  }
  if (warp < 4) {
    const int m = 128 * (int)rank + 32 * warp + (tid & 31);
    for (int n0 = 0; n0 < N; n0 += 8) {
      float v[8];
      tc::tmem_ld8(tbase + tc::tmem_lane_base(warp) + n0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) D[(size_t)m * N + n0 + j] = v[j];
    }
  }
  tc::fence_before();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(ncols) : "memory");
}

}  // namespace fdsdf

extern "C" fdsdf_status fdsdf_selftest_mma_pair(const float* d_W, const float* d_B, float* d_D, int N, int K,
                                                void* stream) {
  using namespace fdsdf;
  if (!d_W || !d_B || !d_D) return FDSDF_E_INVALID;
  if (N < 32 || N > 256 || N % 32 || K < 64 || K % 64) return FDSDF_E_INVALID;
  const size_t smem = 3 * (size_t)(128 + N / 2) * 128 + 64 + 1024;
  cudaError_t e = cudaFuncSetAttribute(tcprobe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return FDSDF_E_CUDA;
  tcprobe2_kernel<<<2, 256, smem, (cudaStream_t)stream>>>(d_W, d_B, d_D, N, K);
  return cudaGetLastError() == cudaSuccess ? FDSDF_OK : FDSDF_E_CUDA;
}

// ----------------------------------------------------------------------------- MMA issue rate
// Diagnostic (not part of include/fdsdf.h; called by scripts/mma_rate.py): cycles per 16-wide
// K step of one CTA issuing the six bf16x6 piece products back to back in different shapes,
//   mode 0: six MMAs a_i . b_j, N = n each, one accumulator range
//   mode 1: a0 . [b0|b1|b2] (3n), a1 . [b0|b1] (2n), a2 . b0 (n)      -> three ranges
//   mode 2: a0 . [b0|b1] (2n), a1 . [b0|b1] (2n), a0 . b2 (n), a2 . b0 (n) -> two ranges
//   mode 3: one MMA a0 . b0 (N = n) per K step (reference rate)
// Operands are zero; the timing does not depend on the values.
namespace fdsdf {
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int mode, int n, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw;
  base += (1024 - (smem_u32(base) & 1023)) & 1023;
  unsigned char* As = base;                    // 3 pieces x [128 rows x 128 B]
  unsigned char* Bs = As + 3 * 16384;          // 3 pieces x [n rows x 128 B]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bs + 3 * n * 128 + 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (3 * 16384 + 3 * n * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(As)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, 512);
  fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t d = *tslot;
  if (tid == 32) {
    const uint32_t a = smem_u32(As), b = smem_u32(Bs);
    const uint32_t i1 = tc::idesc_bf16(128, n), i2 = tc::idesc_bf16(128, 2 * n), i3 = tc::idesc_bf16(128, 3 * n);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int sub = 0; sub < 4; ++sub) {
        auto A = [&](int p) { return tc::sdesc_sw128(a + p * 16384 + sub * 32); };
        auto B = [&](int p) { return tc::sdesc_sw128(b + p * n * 128 + sub * 32); };
        if (mode == 0) {
#pragma unroll
          for (int q = 0; q < 6; ++q) tc::mma_bf16(d, A(tc::prod_a(q)), B(tc::prod_b(q)), i1, 1u);
        } else if (mode == 1) {
          tc::mma_bf16(d, A(0), B(0), i3, 1u);
          tc::mma_bf16(d, A(1), B(0), i2, 1u);
          tc::mma_bf16(d, A(2), B(0), i1, 1u);
        } else if (mode == 2) {
          tc::mma_bf16(d, A(0), B(0), i2, 1u);
          tc::mma_bf16(d, A(1), B(0), i2, 1u);
          tc::mma_bf16(d, A(0), B(2), i1, 1u);
          tc::mma_bf16(d, A(2), B(0), i1, 1u);
        } else {
          tc::mma_bf16(d, A(0), B(0), i1, 1u);
        }
      }
    tc::mma_commit(bar);
    mbar_wait(bar, 0);
    out[0] = clock64() - t0;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(d, 512);
}
}  // namespace fdsdf

extern "C" int fdsdf_probe_mma_rate(int mode, int n, int iters, long long* d_out) {
  const int bytes = 3 * 16384 + 3 * n * 128 + 2048 + 64;
  auto k = fdsdf::mma_rate_kernel;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return 1;
  k<<<1, 128, bytes>>>(mode, n, iters, d_out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 2;
}

// ----------------------------------------------------------------------------- TMEM load rate
// Diagnostic: `nw` warps each issue `iters` x (tcgen05.ld 32x32b.x`W` + wait::ld) on their lane
// quarter; returns the CTA's cycles.  Bytes moved = nw * iters * 32 lanes * W * 4.
namespace fdsdf {
template <int W>
__global__ void tmem_rate_kernel(int iters, long long* out, float* sink) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc(&tslot, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t t = tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (warp >> 2) * 32;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[8];
    if (W == 8) {
      tc::tmem_ld8(t + (it & 7) * 8, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j];
    } else {
      float w[16];
      tc::tmem_ld16(t + (it & 1) * 16, w);
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += w[j];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[0] = clock64() - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tslot, 512);
}
}  // namespace fdsdf

extern "C" int fdsdf_probe_tmem_rate(int width, int nwarps, int iters, long long* d_out, float* d_sink) {
  if (width == 8)
    fdsdf::tmem_rate_kernel<8><<<1, nwarps * 32>>>(iters, d_out, d_sink);
  else
    fdsdf::tmem_rate_kernel<16><<<1, nwarps * 32>>>(iters, d_out, d_sink);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 2;
}

// ----------------------------------------------------------------------------- pair MMA rate
// Diagnostic: the same issue shapes on a CTA pair (tcgen05 cta_group::2, M = 256): `n` is the
// pair-wide N of one operand piece (each CTA holds n/2 columns of it).
//   mode 0: six MMAs a_i . b_j (N = n);  mode 1: three MMAs a_p . [b0|b1|b2] (N = 3n, 9
//   products);  mode 2: a0.[b0|b1], a1.[b0|b1] (2n), a0.b2, a2.b0 (n);  mode 3: one MMA (N = n)
namespace fdsdf {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_rate2_kernel(int mode, int n, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw;
  base += (1024 - (smem_u32(base) & 1023)) & 1023;
  const int nh = n / 2;
  unsigned char* As = base;
  unsigned char* Bs = As + 3 * 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Bs + 3 * nh * 128 + 1024);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < (3 * 16384 + 3 * nh * 128) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(As)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();
  tc::fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc::fence_after();
  const uint32_t d = *tslot;
  auto mma2 = [&](uint64_t ad, uint64_t bd, uint32_t id) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(ad), "l"(bd), "r"(id), "r"(1u)
        : "memory");
  };
  if (tid == 32 && rank == 0) {
    const uint32_t a = smem_u32(As), b = smem_u32(Bs);
    const uint32_t i1 = tc::idesc_bf16(256, n), i2 = tc::idesc_bf16(256, 2 * n), i3 = tc::idesc_bf16(256, 3 * n);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int sub = 0; sub < 4; ++sub) {
        auto A = [&](int p) { return tc::sdesc_sw128(a + p * 16384 + sub * 32); };
        auto B = [&](int p) { return tc::sdesc_sw128(b + p * nh * 128 + sub * 32); };
        if (mode == 0) {
#pragma unroll
          for (int q = 0; q < 6; ++q) mma2(A(tc::prod_a(q)), B(tc::prod_b(q)), i1);
        } else if (mode == 1) {
          mma2(A(0), B(0), i3);
          mma2(A(1), B(0), i3);
          mma2(A(2), B(0), i3);
        } else if (mode == 2) {
          mma2(A(0), B(0), i2);
          mma2(A(1), B(0), i2);
          mma2(A(0), B(2), i1);
          mma2(A(2), B(0), i1);
        } else {
          mma2(A(0), B(0), i1);
        }
      }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
    mbar_wait(bar, 0);
    out[0] = clock64() - t0;
  } else if (tid == 32) {
    mbar_wait(bar, 0);
  }
  tc::fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(d), "r"(512) : "memory");
}
}  // namespace fdsdf

extern "C" int fdsdf_probe_mma_rate2(int mode, int n, int iters, long long* d_out) {
  const int bytes = 3 * 16384 + 3 * (n / 2) * 128 + 2048 + 64;
  auto k = fdsdf::mma_rate2_kernel;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return 1;
  k<<<2, 128, bytes>>>(mode, n, iters, d_out);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 2;
}
