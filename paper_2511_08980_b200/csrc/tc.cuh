// tc.cuh -- tcgen05 (5th-generation tensor core) building blocks for the sm_100a contractions.
//
// Precision scheme "bf16x6": every fp32 operand x is split EXACTLY into three
// bf16 pieces x = x0 + x1 + x2 (x0 = rn(x), x1 = rn(x - x0), x2 = rn(x - x0 - x1); each
// residual is exactly representable, so the three pieces carry all 24 bits of x).  A product
// sum_k a_k b_k is formed from the six piece products with i + j <= 2,
//     a2 b0 + a1 b1 + a0 b2 + a1 b0 + a0 b1 + a0 b0,
// all accumulated in fp32 in tensor memory.  The dropped terms (a1 b2, a2 b1, a2 b2) are
// <= 2^-25 |a b|, below fp32 rounding, so the contraction is fp32-accurate while running on
// the bf16 tensor pipe (6 bf16 MMAs = the cost of 3 tf32 MMAs).  Plain bf16/tf32 fails the
// BASELINE tolerances and is never used.
//
// Operand layout: K-major, 128-byte swizzled bf16 tiles (the canonical UMMA SWIZZLE_128B
// K-major layout): a tile of R rows and K columns is stored as K/64 column chunks of
// R x 128 B; row r of a chunk sits at (r/8)*1024 + (r%8)*128 and its 16-byte pieces are
// XOR-permuted by r%8.  Descriptor: SBO = 1024 B (8-row group stride), LBO unused,
// layout SWIZZLE_128B; the K sub-step of 16 elements advances the start address by 32 B.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"

namespace fdsdf {
namespace tc {

// ----------------------------------------------------------------------------- bf16 x3 split
struct Bf3 {
  __nv_bfloat16 p[3];
};

__device__ __forceinline__ Bf3 split3(float x) {
  Bf3 o;
  o.p[0] = __float2bfloat16_rn(x);
  float r = x - __bfloat162float(o.p[0]);
  o.p[1] = __float2bfloat16_rn(r);
  r = r - __bfloat162float(o.p[1]);
  o.p[2] = __float2bfloat16_rn(r);
  return o;
}

// the same exact split for two values at once, as packed bf16x2 words (lo half = x, hi = y):
// cvt.rn.bf16x2.f32 runs on the ALU pipe, the scalar conversion on the quarter-rate XU
__device__ __forceinline__ void split3x2(float x, float y, uint32_t (&w)[3]) {
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const __nv_bfloat162 b = __floats2bfloat162_rn(x, y);
    const uint32_t u = *reinterpret_cast<const uint32_t*>(&b);
    w[p] = u;
    // (x, y) -= the two pieces, one packed fp32 x2 subtraction (exact: each residual fits fp32)
    const float2 r = add2(make_float2(x, y), make_float2(-__uint_as_float(u << 16), -__uint_as_float(u & 0xFFFF0000u)));
    x = r.x;
    y = r.y;
  }
}

// byte offset of element (r, k) in a K-major SWIZZLE_128B bf16 tile with R rows
__host__ __device__ __forceinline__ uint32_t sw128_off(int r, int k, int R) {
  const int kc = k >> 6, kk = k & 63;
  return (uint32_t)(kc * R * 128 + (r >> 3) * 1024 + (r & 7) * 128 + ((((kk >> 3) ^ (r & 7))) << 4) +
                    ((kk & 7) << 1));
}

// ----------------------------------------------------------------------------- descriptors
// shared-memory matrix descriptor (sm_100 UMMA layout): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 [46,48), layout type [61,64) (2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// MN-major SWIZZLE_128B bf16 tile, `mn` = extent along M/N (multiple of 64): swizzle atoms of
// 64 MN-elements (one 128-byte row) x 8 K-rows, atoms ordered MN-fastest; byte offset of
// element (r = MN index, k = K index)
__host__ __device__ __forceinline__ uint32_t sw128mn_off(int r, int k, int mn) {
  const int ma = r >> 6, ka = k >> 3, k8 = k & 7, r64 = r & 63;
  return (uint32_t)((ka * (mn >> 6) + ma) * 1024 + k8 * 128 + ((((r64 >> 3) ^ k8)) << 4) + ((r64 & 7) << 1));
}

// MN-major SWIZZLE_128B descriptor: lbo = byte stride between atoms along MN, sbo = along K
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor, kind::f16: D f32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
// both K-major (bits 15, 16 = 0), N>>3 [17,23), M>>4 [24,29)
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn = 0, int b_mn = 0) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ----------------------------------------------------------------------------- tcgen05 PTX
__device__ __forceinline__ void mma_bf16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// warp-collective forms: executed by a whole warp with warp-uniform operands (which then stay
// in uniform registers: no per-lane waterfall around each issue), one elected lane issues
__device__ __forceinline__ void mma_bf16_w(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// arrive (once) on an mbarrier when every previously issued tcgen05.mma of this thread is done
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// one full warp: allocate ncols TMEM columns (power of two >= 32), base address -> *dst
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// warp-collective: thread t of warp w reads lane 32*(w%4)+t, 8 consecutive fp32 columns
// starting at column `col` (taddr must carry the warp's lane base in bits 16..31).
// The load and its wait are one asm statement so no use of v can be scheduled before the wait.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
      : "r"(taddr)
      : "memory");
  v[0] = __uint_as_float(r0);
  v[1] = __uint_as_float(r1);
  v[2] = __uint_as_float(r2);
  v[3] = __uint_as_float(r3);
  v[4] = __uint_as_float(r4);
  v[5] = __uint_as_float(r5);
  v[6] = __uint_as_float(r6);
  v[7] = __uint_as_float(r7);
}

// x2 / x16 variants of tmem_ld8
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float (&v)[2]) {
  uint32_t r0, r1;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r0), "=r"(r1)
      : "r"(taddr)
      : "memory");
  v[0] = __uint_as_float(r0);
  v[1] = __uint_as_float(r1);
}


// columns ta + 8 j and tb + 8 j, j = 0..9, summed pairwise (two accumulator ranges), one wait
__device__ __forceinline__ void tmem_ld10x2_stride8(uint32_t ta, uint32_t tb, float (&v)[10]) {
  uint32_t r[20];
#define FDSDF_LD1(i, t) "tcgen05.ld.sync.aligned.32x32b.x1.b32 {%" #i "}, [%" #t "];\n\t"
  asm volatile(FDSDF_LD1(0, 20) FDSDF_LD1(1, 21) FDSDF_LD1(2, 22) FDSDF_LD1(3, 23) FDSDF_LD1(4, 24)
                   FDSDF_LD1(5, 25) FDSDF_LD1(6, 26) FDSDF_LD1(7, 27) FDSDF_LD1(8, 28) FDSDF_LD1(9, 29)
                       FDSDF_LD1(10, 30) FDSDF_LD1(11, 31) FDSDF_LD1(12, 32) FDSDF_LD1(13, 33) FDSDF_LD1(14, 34)
                           FDSDF_LD1(15, 35) FDSDF_LD1(16, 36) FDSDF_LD1(17, 37) FDSDF_LD1(18, 38)
                               FDSDF_LD1(19, 39) "tcgen05.wait::ld.sync.aligned;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19])
               : "r"(ta), "r"(ta + 8), "r"(ta + 16), "r"(ta + 24), "r"(ta + 32), "r"(ta + 40), "r"(ta + 48),
                 "r"(ta + 56), "r"(ta + 64), "r"(ta + 72), "r"(tb), "r"(tb + 8), "r"(tb + 16), "r"(tb + 24),
                 "r"(tb + 32), "r"(tb + 40), "r"(tb + 48), "r"(tb + 56), "r"(tb + 64), "r"(tb + 72)
               : "memory");
#undef FDSDF_LD1
#pragma unroll
  for (int j = 0; j < 10; ++j) v[j] = __uint_as_float(r[j]) + __uint_as_float(r[10 + j]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const float (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__float_as_uint(v[0])),
               "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3]))
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r0, r1, r2, r3;
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
      : "r"(taddr)
      : "memory");
  v[0] = __uint_as_float(r0);
  v[1] = __uint_as_float(r1);
  v[2] = __uint_as_float(r2);
  v[3] = __uint_as_float(r3);
}




// 10 consecutive columns as five 2-column loads, one wait
__device__ __forceinline__ void tmem_ld10(uint32_t ta, float (&v)[10]) {
  uint32_t r[10];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%10];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%2,%3}, [%11];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%4,%5}, [%12];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%6,%7}, [%13];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x2.b32 {%8,%9}, [%14];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9])
      : "r"(ta), "r"(ta + 2), "r"(ta + 4), "r"(ta + 6), "r"(ta + 8)
      : "memory");
#pragma unroll
  for (int j = 0; j < 10; ++j) v[j] = __uint_as_float(r[j]);
}

// three 8-column loads (the three accumulator ranges of one column group), one wait
__device__ __forceinline__ void tmem_ld8x3(uint32_t ta, uint32_t tb, uint32_t tc_, float (&a)[8], float (&b)[8],
                                           float (&c)[8]) {
  uint32_t r[24];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%24];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%25];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [%26];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23])
      : "r"(ta), "r"(tb), "r"(tc_)
      : "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = __uint_as_float(r[j]);
    b[j] = __uint_as_float(r[8 + j]);
    c[j] = __uint_as_float(r[16 + j]);
  }
}

// three 4-column loads (the three accumulator ranges of one column group), one wait
__device__ __forceinline__ void tmem_ld4x3(uint32_t ta, uint32_t tb, uint32_t tc_, float (&a)[4], float (&b)[4],
                                           float (&c)[4]) {
  uint32_t r[12];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%12];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [%13];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [%14];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
      : "r"(ta), "r"(tb), "r"(tc_)
      : "memory");
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a[j] = __uint_as_float(r[j]);
    b[j] = __uint_as_float(r[4 + j]);
    c[j] = __uint_as_float(r[8 + j]);
  }
}

__device__ __forceinline__ uint32_t tmem_lane_base(int warp) { return (uint32_t)(32 * (warp & 3)) << 16; }

// the packed weight images hold WP = 3 exact bf16 pieces per weight (48 KB per (K chunk,
// M-half) stage)
constexpr int WP = 3;
// the six piece products (i, j), i + j <= 2, smallest first
__host__ __device__ constexpr int prod_a(int q) { return q == 0 ? 2 : (q == 1 || q == 3) ? 1 : 0; }
__host__ __device__ constexpr int prod_b(int q) { return q == 2 ? 2 : (q == 1 || q == 4) ? 1 : 0; }

}  // namespace tc
}  // namespace fdsdf
