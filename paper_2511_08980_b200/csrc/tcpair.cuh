// tcpair.cuh -- CTA-pair (cluster of 2, tcgen05 cta_group::2) building blocks of the
// pair-tiled tensor-core kernels (fwd_tc2.cu, bwd_tc2.cu).
//
// A pair tile is split into two half-tile SLOTS that are pipelined against each other: while
// the tensor cores run layer l of one slot, the epilogue warps of both CTAs work on the other
// slot.  Per CTA (rank r of the pair):
//   * weights: only W rows [128 r, 128 r + 128) (its M-half) are streamed -- half the per-SM
//     weight traffic of the single-CTA kernels, which is what makes a second slot affordable;
//   * B operand of each slot: its half of the slot's columns ([NS/2 r, NS/2 (r+1))), all K;
//   * TMEM: D rows [128 r, ..) of both slots (one accumulator range each);
//   * the leader (r = 0) issues `tcgen05.mma.cta_group::2` (M = 256); commits are multicast
//     to both CTAs' mbarriers; the peer forwards its weight-stage completion to the leader.
// Epilogue threads own one output neuron (TMEM lane) of their CTA and write every B element
// into the CTA that holds its column (st.shared::cluster), then arrive on the leader's "B full"
// barrier with cluster-scope release.
#pragma once
#include "tc.cuh"

namespace fdsdf {
namespace tp {

__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of local shared address `saddr` in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_u16(uint32_t caddr, uint16_t v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(caddr), "h"(v) : "memory");
}
__device__ __forceinline__ void st_f32(uint32_t caddr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(caddr), "f"(v) : "memory");
}
// arrive on an mbarrier of any CTA of the cluster (release at cluster scope)
__device__ __forceinline__ void arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// wait (acquire at cluster scope) on a local mbarrier that receives remote arrivals
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}
// generic-proxy writes to shared memory of either CTA of the pair -> visible to the async proxy
// (the tensor cores).  Compiles to MEMBAR.ALL.GPU + FENCE.VIEW.ASYNC: it also waits for this
// thread's outstanding GLOBAL stores, so issue those after it.
__device__ __forceinline__ void fence_proxy_async_cluster() {
  asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
}

// bulk copy of `bytes` from this CTA's shared memory to shared::cluster address `dst` (a peer
// CTA), completing `bytes` of transaction count on the mbarrier at shared::cluster `mbar` (in
// the destination CTA).  Async proxy end to end: the source needs fence.proxy.async.shared::cta
// after its generic writes, the destination's readers only the mbarrier.
__device__ __forceinline__ void bulk_s2peer(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst),
               "r"(smem_u32(src)), "r"(bytes), "r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mma2(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// warp-collective forms: the whole warp executes them with warp-uniform operands (kept in
// uniform registers -- no per-lane waterfall around the issue), one elected lane issues
__device__ __forceinline__ void mma2_w(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit2_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// arrive once on the mbarrier at this shared offset in BOTH CTAs when the issued MMAs are done
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// write v split into 3 bf16 pieces at B element (local column nl of the owner CTA, K index k):
// per slot the B block is [K chunk kc][piece][NH rows][128 B] (SW128 K-major rows)
template <int NH>
__device__ __forceinline__ void put_b(uint32_t bslot_caddr, int nl, int k, float v) {
  const tc::Bf3 s = tc::split3(v);
  const uint32_t off = (uint32_t)((k >> 6) * (3 * NH * 128)) + tc::sw128_off(nl, k & 63, NH);
#pragma unroll
  for (int p = 0; p < 3; ++p) st_u16(bslot_caddr + p * NH * 128 + off, __bfloat16_as_ushort(s.p[p]));
}
// the same into this CTA's own shared memory (plain st.shared)
template <int NH>
__device__ __forceinline__ void put_b_local(unsigned char* bslot, int nl, int k, float v) {
  const tc::Bf3 s = tc::split3(v);
  const uint32_t off = (uint32_t)((k >> 6) * (3 * NH * 128)) + tc::sw128_off(nl, k & 63, NH);
#pragma unroll
  for (int p = 0; p < 3; ++p) *reinterpret_cast<__nv_bfloat16*>(bslot + p * NH * 128 + off) = s.p[p];
}

}  // namespace tp
}  // namespace fdsdf
