// common.cuh -- device helpers for the fdsdf sm_100a kernels.
//
//  * mbarrier / cp.async.bulk (TMA bulk-copy engine) PTX wrappers used to stream layer
//    weights into shared memory (BASELINE north_star (a));
//  * accurate fp32 elementary functions for the cancellation-free activation identities
//    (DESIGN.md §4): range-reduced sincos (Cody-Waite, 3-part pi/2 with FMA) and the
//    logistic / expm1 / log1p helpers of the softplus identities.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace fdsdf {

// Debug builds (-DFDSDF_DEBUG_ASSERT, scripts/build_variant.py): device-side bounds checks of
// the computed shared-memory, TMEM-column and global indices of the tensor kernels (the
// stand-in for compute-sanitizer memcheck, which this GPU pool does not allow).  No-op otherwise.
#ifdef FDSDF_DEBUG_ASSERT
#define FDSDF_ASSERT(cond)                                                                       \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("FDSDF_ASSERT failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x, #cond);                                                           \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define FDSDF_ASSERT(cond) ((void)0)
#endif

// ----------------------------------------------------------------------------- PTX: mbarrier + bulk copy

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// try_wait with a suspend-time hint: the waiting thread is suspended in hardware until the
// phase completes (or the hint, in ns, elapses) instead of spinning on issue slots that the
// compute warps of the same scheduler need
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}

// poll with a fixed __nanosleep between polls (ns > 0): for many warps waiting on the same
// phase, so their polls do not take the issue slots of the warps still working
template <int NS>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  if (NS <= 0) {
    mbar_wait(bar, parity);
    return;
  }
  while (!mbar_try_wait(bar, parity)) __nanosleep(NS);
}

// the same with a __nanosleep back-off between polls: for the long waits of the single-thread
// roles (producer, MMA issuer), whose polling shares a scheduler with epilogue warps
#ifndef FDSDF_WAIT_BACKOFF_NS
#define FDSDF_WAIT_BACKOFF_NS 0
#endif
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  if (FDSDF_WAIT_BACKOFF_NS == 0) {
    mbar_wait(bar, parity);
    return;
  }
  while (!mbar_try_wait_sleep(bar, parity)) __nanosleep(FDSDF_WAIT_BACKOFF_NS);
}

// 1-D bulk copy global -> shared through the TMA engine, completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk prefetch of [ptr, ptr + bytes) into L2 (bytes a multiple of 16); no completion tracking
__device__ __forceinline__ void prefetch_l2_bulk(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// 4-byte asynchronous global -> shared copy (LDGSTS) and its completion wait
__device__ __forceinline__ void cp_async4(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// named barrier `id` over `nthreads` threads (a multiple of 32)
__device__ __forceinline__ void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// named barrier over the compute warps only (the producer warp never joins)
__device__ __forceinline__ void bar_compute(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// ----------------------------------------------------------------------------- launch helpers
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel K, device): the attribute
// persists on the device, and setting it before every launch cost a driver call per launch on the
// step's host-side enqueue path
template <auto K>
inline cudaError_t smem_attr_once(int bytes) {
  static unsigned long long done = 0;  // bit d: set on device d
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done |= bit;
  return e;
}

// ----------------------------------------------------------------------------- packed fp32 x2
// sm_100 FFMA2 / FADD2 / FMUL2: two independent fp32 lanes per instruction, each rounded exactly
// as the scalar instruction would (so a packed evaluation is bitwise the scalar one); half the
// issue slots of the scalar form for the pair maps, which run two pairs per lane pair
__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

// ----------------------------------------------------------------------------- accurate fp32 math

// sin and cos of x, |x| up to ~1e5, error ~1-2 ulp (relative for small |x|).
// Cody-Waite reduction by pi/2 with FMA, minimax polynomials on [-pi/4, pi/4].
__device__ __forceinline__ void sincos_acc(float x, float* s, float* c) {
  const float k = rintf(x * 0.636619772367581343f);
  float r = fmaf(-k, 1.5707963705062866f, x);
  r = fmaf(-k, -4.371138828673793e-08f, r);
  r = fmaf(-k, -1.7763568394002505e-15f, r);
  const int q = static_cast<int>(k);
  const float z = r * r;
  float ps = fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f);
  ps = fmaf(ps * z, r, r);
  float pc = fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z, 4.166664568298827e-2f);
  pc = fmaf(pc * z, z, fmaf(-0.5f, z, 1.0f));
  float sv = (q & 1) ? pc : ps;
  float cv = (q & 1) ? ps : pc;
  if (q & 2) sv = -sv;
  if ((q + 1) & 2) cv = -cv;
  *s = sv;
  *c = cv;
}

// sincos_acc of two arguments at once (packed fp32 x2 for the reduction and the polynomials:
// per lane exactly the scalar arithmetic, so bitwise sincos_acc of each)
__device__ __forceinline__ void sincos_acc2(float2 x, float2* s, float2* c) {
  const float2 kx = mul2(x, f2s(0.636619772367581343f));
  const float2 k = make_float2(rintf(kx.x), rintf(kx.y));
  const float2 nk = make_float2(-k.x, -k.y);
  float2 r = fma2(nk, f2s(1.5707963705062866f), x);
  r = fma2(nk, f2s(-4.371138828673793e-08f), r);
  r = fma2(nk, f2s(-1.7763568394002505e-15f), r);
  const float2 z = mul2(r, r);
  float2 ps = fma2(fma2(f2s(-1.9515295891e-4f), z, f2s(8.3321608736e-3f)), z, f2s(-1.6666654611e-1f));
  ps = fma2(mul2(ps, z), r, r);
  float2 pc = fma2(fma2(f2s(2.443315711809948e-5f), z, f2s(-1.388731625493765e-3f)), z, f2s(4.166664568298827e-2f));
  pc = fma2(mul2(pc, z), z, fma2(f2s(-0.5f), z, f2s(1.0f)));
  const int qa = static_cast<int>(k.x), qb = static_cast<int>(k.y);
  float sa = (qa & 1) ? pc.x : ps.x, ca = (qa & 1) ? ps.x : pc.x;
  float sb = (qb & 1) ? pc.y : ps.y, cb = (qb & 1) ? ps.y : pc.y;
  if (qa & 2) sa = -sa;
  if ((qa + 1) & 2) ca = -ca;
  if (qb & 2) sb = -sb;
  if ((qb + 1) & 2) cb = -cb;
  *s = make_float2(sa, sb);
  *c = make_float2(ca, cb);
}

// sincos for the small arguments of the pair maps (A/2, S/4): most are below 2^-4, where a
// short Taylor polynomial is exact to fp32 rounding; |x| <= pi/4 needs no range reduction
// (k = 0, r = x: the sincos_acc polynomial alone); larger |x| (rare) take the full path.
__device__ __forceinline__ void sincos_small(float x, float* s, float* c) {
  if (fabsf(x) <= 0.0625f) {
    // |x| <= 2^-4: Taylor to x^5 / x^6; truncation <= x^7/5040 < 1e-12 |x|, below fp32 rounding
    const float z = x * x;
    *s = fmaf(-x * z, fmaf(z, -8.3333333333e-3f, 1.6666666667e-1f), x);
    *c = fmaf(z, fmaf(z, fmaf(z, -1.3888888889e-3f, 4.1666666667e-2f), -0.5f), 1.0f);
  } else if (fabsf(x) <= 0.78539816339744831f) {
    const float z = x * x;
    float ps = fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f);
    ps = fmaf(ps * z, x, x);
    float pc = fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z, 4.166664568298827e-2f);
    pc = fmaf(pc * z, z, fmaf(-0.5f, z, 1.0f));
    *s = ps;
    *c = pc;
  } else {
    sincos_acc(x, s, c);
  }
}

// logistic s(t) = 1/(1+exp(-t)), accurate, saturating without NaN
__device__ __forceinline__ float logistic_acc(float t) { return 1.0f / (1.0f + expf(-t)); }

// exact softplus log(1+exp(t)) without threshold
__device__ __forceinline__ float softplus_acc(float t) { return fmaxf(t, 0.0f) + log1pf(expf(-fabsf(t))); }

}  // namespace fdsdf
