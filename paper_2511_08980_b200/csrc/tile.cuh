// tile.cuh -- the per-CTA column-GEMM core shared by the forward and backward kernels.
//
// A CTA holds a tile of activation columns in shared memory, act[k][col] (k = input neuron,
// fp32, 16-byte chunks XOR-swizzled by (k>>2)&7 so both the GEMM reads and the epilogue
// writes are bank-conflict free).  Layer weights are streamed through an NSTG-deep ring of
// KC-row slabs filled by the TMA bulk-copy engine (cp.async.bulk + mbarrier complete_tx);
// thread 0 issues each slab one slab ahead of use, the slab is released by one mbarrier
// arrive per warp.  Each of the 256 threads owns an 8-row x 8-column register tile:
// rows {rg*4+j, RG*4+rg*4+j | j<4}, columns = the 8 columns of centre-group cg.
// out[m][col] = sum_k Wslab[k][m] * act[k][col]: the slab is [k][m] (m contiguous), i.e. the
// packed forward weight is W^T and the packed backward weight is W itself.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace fdsdf {

template <int MPAD_, int SLAB_BYTES, int NSTG_>
struct TileCfg {
  static constexpr int MPAD = MPAD_;
  static constexpr int RG = MPAD / 8;        // row groups
  static constexpr int CG = NCT / RG;        // centre groups (8 columns each)
  static constexpr int RGW = RG / 8;         // warps along rows
  static constexpr int NC = CG * 8;          // columns of act
  static constexpr int KC = SLAB_BYTES / (4 * MPAD);  // weight rows per slab
  static constexpr int NSTG = NSTG_;
  static constexpr int SLAB = KC * MPAD;     // floats per slab
  static constexpr int NCHUNK = MPAD / KC;   // slabs per layer
};

__device__ __forceinline__ int swz(int k) { return (k >> 2) & 7; }

// index of act[k][col] (col in [0, NC)), swizzled 16-byte chunks
template <int NC>
__device__ __forceinline__ int act_idx(int k, int col) {
  return k * NC + ((((col >> 2) ^ swz(k))) << 2) + (col & 3);
}

template <int MPAD>
__device__ __forceinline__ int tile_row(int rg, int i) {
  return (i < 4) ? rg * 4 + i : (MPAD / 2) + rg * 4 + (i - 4);
}

// The weight stream of one CTA: `per_tile` slabs per tile, the layer sequence repeating
// every (L-2) layers, forward (layers 1..L-2) or backward (layers L-2..1).
template <class T>
struct WStream {
  const float* const* layers;
  int L;
  int backward;
  uint32_t per_tile;
  uint32_t total;
  float* wst;
  uint64_t* full;
  uint64_t* empty;

  __device__ __forceinline__ void issue(uint32_t it) const {
    if (it >= total) return;
    const uint32_t w = it % per_tile;
    const int ls = (int)(w / T::NCHUNK) % (L - 2);
    const int ch = (int)(w % T::NCHUNK);
    const int l = backward ? (L - 2 - ls) : (1 + ls);
    const int s = (int)(it % T::NSTG);
    const uint32_t par = (it / T::NSTG) & 1u;
    mbar_wait(&empty[s], par ^ 1u);
    mbar_arrive_expect_tx(&full[s], T::SLAB * 4);
    bulk_g2s(wst + s * T::SLAB, layers[l] + (size_t)ch * T::SLAB, T::SLAB * 4, &full[s]);
  }
  // prologue: slabs 0 .. NSTG-3 (thread 0 only)
  __device__ __forceinline__ void prologue() const {
    for (uint32_t i = 0; i + 2 < (uint32_t)T::NSTG; ++i) issue(i);
  }
};

// One layer of the column GEMM: acc[i][j] = sum_k slab(k, row_i) * act[k][cg*8 + j]
// (+ optional second column group act2[k][cg*2 + j2] into acc2).
template <class T, bool TWO>
__device__ __forceinline__ void tile_gemm(float (&acc)[8][8], float (&acc2)[8][2], const float* __restrict__ act,
                                          const float* __restrict__ act2, const WStream<T>& ws, uint32_t& it,
                                          int rg, int cg, int tid) {
  constexpr int MPAD = T::MPAD;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    acc2[i][0] = 0.f;
    acc2[i][1] = 0.f;
  }
  const int c0 = 2 * cg, c1 = 2 * cg + 1;
#pragma unroll 1
  for (int ch = 0; ch < T::NCHUNK; ++ch, ++it) {
    if (tid == 0) ws.issue(it + T::NSTG - 2);
    const int s = (int)(it % T::NSTG);
    const uint32_t par = (it / T::NSTG) & 1u;
    mbar_wait(&ws.full[s], par);
    const float* w = ws.wst + s * T::SLAB;
#pragma unroll
    for (int kk = 0; kk < T::KC; ++kk) {
      const int k = ch * T::KC + kk;
      const float4 w0 = *reinterpret_cast<const float4*>(w + kk * MPAD + rg * 4);
      const float4 w1 = *reinterpret_cast<const float4*>(w + kk * MPAD + MPAD / 2 + rg * 4);
      const int sw = swz(k);
      const float* ar = act + k * T::NC;
      const float4 a0 = *reinterpret_cast<const float4*>(ar + ((c0 ^ sw) << 2));
      const float4 a1 = *reinterpret_cast<const float4*>(ar + ((c1 ^ sw) << 2));
      const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(wv[i], av[j], acc[i][j]);
      if (TWO) {
        const float2 b = *reinterpret_cast<const float2*>(act2 + k * (T::CG * 2) + cg * 2);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc2[i][0] = fmaf(wv[i], b.x, acc2[i][0]);
          acc2[i][1] = fmaf(wv[i], b.y, acc2[i][1]);
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&ws.empty[s]);
  }
}

}  // namespace fdsdf
