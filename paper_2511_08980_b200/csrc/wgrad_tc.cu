// wgrad_tc.cu -- the weight-gradient contraction on the tensor cores (
// bf16x6, tc.cuh / DESIGN.md §4b):
//
//   dW_l[m][k] = sum_j delta_l[j][m] * a_{l-1}[j][k]     j over (centre, column): 10 per centre
//
// Split-K: CTA (s, b, l) owns a contiguous j-range of GEMM layer l and computes output block b
// (BW x BW, BW = min(MPAD, 256): the whole layer for MPAD <= 256, one of four 256 x 256 blocks
// for MPAD = 512) into TMEM (M = BW rows in 128-row halves, N = BW), then writes its part of the
// split's partial (never atomically added); finalize_kernel sums the partials in split order, so
// the result is bitwise reproducible. The blocks of one split are adjacent in the grid, so they
// run together and read the same delta / a rows through L2.
//   warp 0      TMEM owner + MMA issuer (one thread): per 32-wide j chunk, 2 K-steps x
//               M-halves x 6 piece products, tcgen05.mma kind::f16 with BOTH operands
//               MN-major (delta and a are stored j-major, m / k contiguous);
//   warps 1..16 stagers: read the fp32 chunk of delta_l and a_{l-1} (float4, coalesced), split
//               every value into 3 bf16 pieces and store them in the MN-major SWIZZLE_128B
//               layout of a 2-deep ring (8-byte st.shared per piece); after the last chunk of
//               a layer they read the accumulator back (tcgen05.ld) and write the partial.
#include "kernels.cuh"
#include "tc.cuh"

namespace fdsdf {

// stage depth along j and ring depth (the ring holds NST * JC / 16 K steps: 2 x 32 or 4 x 16)
#ifndef WGRAD_TC_JC
#define WGRAD_TC_JC 32
#endif
#ifndef WGRAD_TC_NST
#define WGRAD_TC_NST 2
#endif
// NPROD: bf16 piece products per MAC -- 6 = bf16x6 (fp32-accurate, the default);
// 3 = a0 b0 + a0 b1 + a1 b0 (FDSDF_CREATE_WGRAD_BF16X3: each product to ~3 * 2^-16 relative; the
// third pieces are neither split nor stored)
template <int MPAD>
struct WtcCfg {
  static constexpr int BW = MPAD > 256 ? 256 : MPAD;  // output block edge
  static constexpr int NB = MPAD / BW;              // blocks per edge
  static constexpr int JC = WGRAD_TC_JC;            // j per stage (JC / 8 swizzle atoms along K)
  static constexpr int MH = BW / 128;
  static constexpr int PIECE = BW * JC * 2;         // one bf16 piece of one operand chunk
  static constexpr int OPER = 3 * PIECE;            // one operand chunk (3 pieces)
  static constexpr int STAGE = 2 * OPER;            // delta chunk + a chunk
  static constexpr int NST = WGRAD_TC_NST;
  static constexpr int KSTRIDE = (BW / 64) * 1024;  // byte stride between swizzle atoms along K
  static constexpr int NSTG = 16;                   // stager warps
  static constexpr int NTHR = (1 + NSTG) * 32;
  static constexpr int OFF_BAR = NST * STAGE;
  static constexpr int BYTES = OFF_BAR + 64 + 1024;
  static constexpr uint32_t TCOLS = MH * BW <= 128 ? 128 : (MH * BW <= 256 ? 256 : 512);
};

bool wgrad_tc_supported(int mpad) { return mpad == 128 || mpad == 256 || mpad == 512; }

// one split per SM-sized slice of the grid: about nsm CTAs per layer in all
int wgrad_tc_splits(int nsm, int64_t rows, int mpad) {
  const int64_t chunks = (rows + 31) / 32;
  const int nb2 = mpad > 256 ? (mpad / 256) * (mpad / 256) : 1;
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, nsm / nb2), chunks));
}

template <int MPAD, int NPROD>
__global__ void __launch_bounds__(WtcCfg<MPAD>::NTHR, 1) wgrad_tc_kernel(const WgradArgs a) {
  static_assert(NPROD == 6 || NPROD == 3, "bf16x6 or the three leading products");
  using C = WtcCfg<MPAD>;
  constexpr int Q0 = 6 - NPROD;       // products q0..5 of tc::prod_a / prod_b (smallest first)
  constexpr int NPC = NPROD == 6 ? 3 : 2;  // pieces staged per operand
  constexpr int JC = C::JC, MH = C::MH, NST = C::NST, BW = C::BW, NB = C::NB;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw;
  sm += (1024 - (smem_u32(sm) & 1023)) & 1023;
  uint64_t* sfull = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* sempty = sfull + NST;
  uint64_t* dfull = sempty + NST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dfull + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&sfull[s], C::NSTG);
      mbar_init(&sempty[s], 1);
    }
    mbar_init(dfull, 1);
    fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tslot, C::TCOLS);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = *tslot;

  const int split = blockIdx.x / (NB * NB);
  const int bm = (blockIdx.x % (NB * NB)) / NB, bn = blockIdx.x % NB;  // output block rows / cols
  const int64_t per = ((a.rows + a.nsplit - 1) / a.nsplit + JC - 1) / JC * JC;
  const int64_t j0 = (int64_t)split * per;
  const int64_t j1 = min(a.rows, j0 + per);
  const int nchunk = j1 > j0 ? (int)((j1 - j0 + JC - 1) / JC) : 0;
  const int li = blockIdx.y;  // GEMM layer first_layer + li

  if (warp == 0) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(128, BW, 1, 1);
      uint32_t it = 0;
      {
        for (int ch = 0; ch < nchunk; ++ch, ++it) {
          const int s = (int)(it % NST);
          mbar_wait(&sfull[s], (it / NST) & 1u);
          tc::fence_after();
          const uint32_t da = smem_u32(sm + s * C::STAGE);
          const uint32_t aa = da + C::OPER;
#pragma unroll
          for (int ks = 0; ks < JC / 16; ++ks)
#pragma unroll
            for (int h = 0; h < MH; ++h)
#pragma unroll
              for (int q = Q0; q < 6; ++q) {
                const uint64_t ad = tc::sdesc_sw128_mn(da + tc::prod_a(q) * C::PIECE + ks * 2 * C::KSTRIDE +
                                                           h * 2 * 1024,
                                                       1024, C::KSTRIDE);
                const uint64_t bd =
                    tc::sdesc_sw128_mn(aa + tc::prod_b(q) * C::PIECE + ks * 2 * C::KSTRIDE, 1024, C::KSTRIDE);
                tc::mma_bf16(tbase + h * BW, ad, bd, idesc, (ch | ks | (q - Q0)) != 0 ? 1u : 0u);
              }
          tc::mma_commit(&sempty[s]);
        }
        tc::mma_commit(dfull);
      }
    }
  } else {
    // ------------------------------------------------------------------ stagers + readback
    const int sw = warp - 1;        // 0 .. NSTG-1
    const int st = tid - 32;        // 0 .. NSTG*32-1
    uint32_t it = 0;
    constexpr int QUADS = BW / 4;  // float4 per j row of the block
    {
      const int layer = a.first_layer + li;
      const float* D = a.del + (size_t)layer * a.stride_layer + bm * BW;
      const float* A = a.actv + (size_t)(layer - 1) * a.stride_layer + bn * BW;
      // the chunk's float4 loads of delta and a, issued one chunk ahead of their split (the
      // global-load latency of chunk ch+1 overlaps the split and stores of chunk ch)
      constexpr int NIT = JC * QUADS / (C::NSTG * 32);
      auto load_chunk = [&](int ch, float4 (&dv)[NIT], float4 (&av)[NIT]) {
        const int64_t jb = j0 + (int64_t)ch * JC;
#pragma unroll
        for (int q = 0; q < NIT; ++q) {
          const int item = st + q * C::NSTG * 32;
          const int jj = item / QUADS, r = (item % QUADS) * 4;
          const int64_t j = jb + jj;
          dv[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          av[q] = dv[q];
          if (ch < nchunk && j < j1) {
            FDSDF_ASSERT(j >= 0 && j < a.rows && r + 4 <= BW && layer >= 1);
            dv[q] = __ldg(reinterpret_cast<const float4*>(D + j * MPAD + r));
            av[q] = __ldg(reinterpret_cast<const float4*>(A + j * MPAD + r));
          }
        }
      };
      float4 dv[NIT], av[NIT];
      load_chunk(0, dv, av);
      for (int ch = 0; ch < nchunk; ++ch, ++it) {
        const int s = (int)(it % NST);
        float4 dn[NIT], an[NIT];
        load_chunk(ch + 1, dn, an);
        mbar_wait(&sempty[s], ((it / NST) & 1u) ^ 1u);
        unsigned char* dst = sm + s * C::STAGE;
#pragma unroll
        for (int q = 0; q < NIT; ++q) {
          const int item = st + q * C::NSTG * 32;
          const int jj = item / QUADS, r = (item % QUADS) * 4;
          const uint32_t off = tc::sw128mn_off(r, jj, BW);
          FDSDF_ASSERT(off + 8 <= (uint32_t)C::PIECE);
          uint32_t d01[3], d23[3], a01[3], a23[3];
          tc::split3x2(dv[q].x, dv[q].y, d01);
          tc::split3x2(dv[q].z, dv[q].w, d23);
          tc::split3x2(av[q].x, av[q].y, a01);
          tc::split3x2(av[q].z, av[q].w, a23);
#pragma unroll
          for (int p = 0; p < NPC; ++p) {
            *reinterpret_cast<uint2*>(dst + p * C::PIECE + off) = make_uint2(d01[p], d23[p]);
            *reinterpret_cast<uint2*>(dst + C::OPER + p * C::PIECE + off) = make_uint2(a01[p], a23[p]);
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfull[s]);
#pragma unroll
        for (int q = 0; q < NIT; ++q) {
          dv[q] = dn[q];
          av[q] = an[q];
        }
      }
      // readback of this layer's partial: warp sw -> lane quarter (warp % 4), halves (sw / 4) + 4i
      mbar_wait(dfull, 0u);
      tc::fence_after();
      float* out = a.part + ((size_t)li * a.nsplit + split) * MPAD * MPAD;
      for (int h = sw >> 2; h < MH; h += C::NSTG / 4) {
        const int q4 = (warp & 3);
        const int m = bm * BW + h * 128 + 32 * q4 + lane;
        const uint32_t taddr = tbase + ((uint32_t)(32 * q4) << 16) + h * BW;
        float* row = out + (size_t)m * MPAD + bn * BW;
#pragma unroll 1
        for (int k0 = 0; k0 < BW; k0 += 16) {
          float v[16];
          tc::tmem_ld16(taddr + k0, v);
          if (nchunk == 0) {  // empty j-range: the accumulator was never written
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = 0.f;
          }
#pragma unroll
          for (int q = 0; q < 16; q += 4)
            *reinterpret_cast<float4*>(row + k0 + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
        }
      }
      tc::fence_before();
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, C::TCOLS);
}

template <int MPAD, int NPROD>
static cudaError_t launch_wgrad_tc_t(const WgradArgs& a, int nglayers, cudaStream_t st) {
  using C = WtcCfg<MPAD>;
  cudaError_t e = smem_attr_once<wgrad_tc_kernel<MPAD, NPROD>>(C::BYTES);
  if (e != cudaSuccess) return e;
  wgrad_tc_kernel<MPAD, NPROD><<<dim3(a.nsplit * C::NB * C::NB, nglayers), C::NTHR, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

template <int NPROD>
static cudaError_t launch_wgrad_tc_p(const WgradArgs& a, int nglayers, cudaStream_t st) {
  if (a.mpad == 512) return launch_wgrad_tc_t<512, NPROD>(a, nglayers, st);
  if (a.mpad == 256) return launch_wgrad_tc_t<256, NPROD>(a, nglayers, st);
  if (a.mpad == 128) return launch_wgrad_tc_t<128, NPROD>(a, nglayers, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_wgrad_tc(const WgradArgs& a, int nglayers, bool bf16x3, cudaStream_t st) {
  if (nglayers <= 0) return cudaSuccess;
  return bf16x3 ? launch_wgrad_tc_p<3>(a, nglayers, st) : launch_wgrad_tc_p<6>(a, nglayers, st);
}

}  // namespace fdsdf
