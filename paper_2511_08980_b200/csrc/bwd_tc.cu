// bwd_tc.cu -- the backward through every stencil evaluation on the tensor cores
// (bf16x6, tc.cuh / DESIGN.md §4b).  Same adjoint algebra as the FFMA
// kernel bwd.cu (act.cuh backward maps), on the warp-specialised engine of tcmlp.cuh.
//
// Tile = 8 centres x 10 adjoint columns (centre value, tangent along r = dL/dg, and the 4
// pairs (A, S)), N = 80.  Top-down over the hidden layers:
//   X_l = W_{l+1}^T delta_{l+1}           tcgen05: A operand = packed W^T (bwd image),
//                                          B operand = delta_{l+1} (bf16x3, written below)
//   delta_l = omega_l * activation-backward(z_l, X_l)    epilogue thread = neuron of layer l
// The epilogue writes delta_l and the layer inputs of every column for the weight-gradient
// contraction, the next B operand, and accumulates -- each thread for its own neuron, in
// fixed tile order -- the bias gradients, dW of the last layer (fan-out 1) and of the first
// layer (fan-in 3).
#include "act.cuh"
#include "tcmlp.cuh"

namespace fdsdf {

#ifndef BWD_TC_PREFETCH
#define BWD_TC_PREFETCH 0
#endif
#ifndef BWD_TC_WPK
#define BWD_TC_WPK 3
#endif
#ifndef BWD_TC_NEPI
#define BWD_TC_NEPI 16
#endif
template <int MPAD>
struct BtcCfg : TcCfg<MPAD, 80, BWD_TC_NEPI, 1, (BWD_TC_NEPI / 4) * (8 / (BWD_TC_NEPI / (4 * (MPAD / 128)))) * 20, 1,
                      BWD_TC_WPK> {
  // one accumulator range (6 MMAs per K step) leaves TMEM for the phase-A stash:
  // (MH x EG thread groups) x (centres per thread) x 20 values
  using B = TcCfg<MPAD, 80, BWD_TC_NEPI, 1, (BWD_TC_NEPI / 4) * (8 / (BWD_TC_NEPI / (4 * (MPAD / 128)))) * 20, 1,
                  BWD_TC_WPK>;
  static constexpr int CT = 8;                                      // centres per tile
  static constexpr int OFF_SD = B::OFF_X;                           // float [2][CT][20]: seeds + x
  static constexpr int OFF_BAR = OFF_SD + 2 * CT * 20 * 4;
  static constexpr int BYTES = OFF_BAR + tc_bars_bytes<B>() + 1024;
};

int bwd_tc_tile_centres() { return 8; }
int bwd_tc_acc_slots(int mpad) { return BWD_TC_NEPI / (4 * (mpad / 128)); }  // accumulator slots per CTA (EG)

template <int ACT, int MPAD>
__global__ void __launch_bounds__(BtcCfg<MPAD>::NTHR, 1) bwd_tc_kernel(const BwdArgs a) {
  using C = BtcCfg<MPAD>;
  using AF = Act<ACT>;
  constexpr int N = C::N, MH = C::MH, CT = C::CT, EG = C::EG;
  constexpr int CPE = CT / EG;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw;
  sm += (1024 - (smem_u32(sm) & 1023)) & 1023;
  unsigned char* Ws = sm + C::OFF_W;
  unsigned char* Bs = sm + C::OFF_B;
  float* sds0 = reinterpret_cast<float*>(sm + C::OFF_SD);
  const TcBars bars = tc_bars<C>(sm + C::OFF_BAR);

  const Net& net = a.net;
  const int L = net.L;
  const int nh = L - 1;
  const int ngemm = L - 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tbase = tc_setup<C>(bars);

  if (warp == 0) {
    if (lane == 0 && ngemm > 0) tc_producer<C>(a.wimg, ngemm, 1, a.ntiles, Ws, bars);
  } else if (warp == 1) {
    if (lane == 0 && ngemm > 0) tc_mma<C>(ngemm, a.ntiles, Ws, Bs, tbase, bars);
  } else {
    const int ew = warp - 2;
    const int et = tid - 64;
    const int q4 = warp & 3;
    const int hh = (ew >> 2) % MH;
    const int eg = ew / (4 * MH);
    const int m = hh * 128 + 32 * q4 + lane;
    const uint32_t taddr = tbase + ((uint32_t)(32 * q4) << 16) + hh * C::DH;
    // this thread group's stash columns (after both halves' accumulators)
    const uint32_t tstash = tbase + ((uint32_t)(32 * q4) << 16) + C::MH * C::DH + (hh * EG + eg) * CPE * 20;
    const float beta = net.beta;
    const float h = a.h;
    const int64_t nrows = a.n * NCOLB;
    // this thread's accumulator slot (one per CTA and centre group): [L-1][MPAD] db |
    // dW_last [MPAD] | db_last [1] | dW_0 [MPAD][3]   (kernels.cuh bacc_size)
    float* bacc = a.bacc + ((size_t)blockIdx.x * EG + eg) * a.nacc;
    float* acc_db = bacc;
    float* acc_dWL = bacc + (size_t)(L - 1) * MPAD;
    float* acc_dbL = acc_dWL + MPAD;
    float* acc_dW0 = acc_dbL + 1;
    // this thread's accumulators (its neuron m), summed over its tiles in tile order and
    // written once at the end: db per hidden layer, dW_last[m], dW_0[m][:], db_last (m == 0)
    float r_db[MAXL];
#pragma unroll
    for (int l = 0; l < MAXL; ++l) r_db[l] = 0.f;
    float r_dWL = 0.f, r_dbL = 0.f, r_dW0[3] = {0.f, 0.f, 0.f};
    uint32_t nd = 0;
    PhaseTimer ptimer;
    ptimer.start();
    // the stored forward pre-activations of a tile are one contiguous block of zf
    auto prefetch_tile = [&](int64_t tile) {
      if (et == 0 && tile < a.ntiles) {
        const int64_t cb = tile * CT, ce = min(cb + CT, a.n);
        const size_t per = (size_t)nh * NCOLF * MPAD * sizeof(float);
        const char* p0 = reinterpret_cast<const char*>(a.zf) + (size_t)cb * per;
        for (size_t off = 0; off < (size_t)(ce - cb) * per; off += 65536)
          prefetch_l2_bulk(p0 + off, (uint32_t)min((size_t)65536, (size_t)(ce - cb) * per - off));
      }
    };
    if (BWD_TC_PREFETCH) prefetch_tile(blockIdx.x);

    // per-tile seeds + coordinates, double-buffered: the next tile's are copied asynchronously
    // (cp.async) while this tile runs
    auto load_seeds = [&](int64_t tile, float* dst) {
      const int64_t cb = tile * CT;
      for (int i = et; i < CT * 20; i += C::NEPI * 32) {
        const int cl = i / 20, q = i % 20;
        const int64_t c = cb + cl;
        if (tile < a.ntiles && c < a.n && q < NSEED + 3)
          cp_async4(dst + i, q < NSEED ? (const void*)(a.seed + c * NSEED + q) : (const void*)(a.x + c * 3 + (q - NSEED)));
        else
          dst[i] = 0.f;
      }
    };
    load_seeds(blockIdx.x, sds0);
    uint32_t spar = 0;
    for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, spar ^= 1u) {
      const int64_t c0 = tile * CT;
      if (BWD_TC_PREFETCH) prefetch_tile(tile + gridDim.x);
      cp_async_wait_all();
      bar_named(1, C::NEPI * 32);  // this tile's seeds are in; every thread is done with the other buffer
      const float* sds = sds0 + spar * CT * 20;
      load_seeds(tile + gridDim.x, sds0 + (spar ^ 1u) * CT * 20);

      for (int l = L - 2; l >= 0; --l) {
        const bool top = (l == L - 2);
        const int M = net.width[l + 1];
        const float om = net.omega[l];
        const bool mok = m < M;
        const float wl = (top && mok) ? net.W[L - 1][m] : 0.f;
        float s_db = 0.f, s_vL = 0.f, s_w0[3] = {0.f, 0.f, 0.f};
        // ---- phase A (X-independent, overlaps this layer's MMA): the pair maps of every
        // centre of this thread -- A_a, S_a and the derivative factors P, Dd, Z -- from the
        // stored forward pre-activations, stashed in this thread's TMEM lane
        struct Zq {
          float z, t0, t1, t2, A[4], S[4];
        };
        auto ldq = [&](int i) -> Zq {
          Zq q{};
          const int64_t c = c0 + eg + EG * i;
          if (i < CPE && c < a.n && mok) {
            const float* zq = a.zf + ((size_t)c * nh + l) * NCOLF * MPAD + m;
            q.z = __ldg(zq);
            q.t0 = __ldg(zq + 1 * MPAD);
            q.t1 = __ldg(zq + 2 * MPAD);
            q.t2 = __ldg(zq + 3 * MPAD);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              q.A[p] = __ldg(zq + (4 + 2 * p) * MPAD);
              q.S[p] = __ldg(zq + (5 + 2 * p) * MPAD);
            }
          }
          return q;
        };
        {
          Zq qn = ldq(0);
#pragma unroll 1
          for (int i = 0; i < CPE; ++i) {
            const Zq q = qn;
            qn = ldq(i + 1);
            float v16[16], v4[4];
#pragma unroll
            for (int j = 0; j < 16; ++j) v16[j] = 0.f;
            v4[0] = v4[1] = v4[2] = v4[3] = 0.f;
            if (mok && c0 + eg + EG * i < a.n) {
              const typename AF::C cc = AF::centre(q.z, beta);
              float t[20];
#pragma unroll
              for (int p = 0; p < 4; ++p)
                AF::pair_bwd(cc, q.A[p], q.S[p], beta, &t[5 * p], &t[5 * p + 1], &t[5 * p + 2], &t[5 * p + 3],
                             &t[5 * p + 4]);
#pragma unroll
              for (int j = 0; j < 16; ++j) v16[j] = t[j];
#pragma unroll
              for (int j = 0; j < 4; ++j) v4[j] = t[16 + j];
            }
            tc::tmem_st16(tstash + i * 20, v16);
            tc::tmem_st4(tstash + i * 20 + 16, v4);
          }
          tc::tmem_wait_st();
        }
        // ---- phase B (after the MMA): combine with the adjoint X
        auto ldz = [&](int i, float (&z4)[4]) {
          const int64_t c = c0 + eg + EG * i;
          z4[0] = z4[1] = z4[2] = z4[3] = 0.f;
          if (i < CPE && c < a.n && mok) {
            const float* zq = a.zf + ((size_t)c * nh + l) * NCOLF * MPAD + m;
            z4[0] = __ldg(zq);
            z4[1] = __ldg(zq + 1 * MPAD);
            z4[2] = __ldg(zq + 2 * MPAD);
            z4[3] = __ldg(zq + 3 * MPAD);
          }
        };
        float zn[4];
        ldz(0, zn);
        if (!top) {
          ptimer.before_wait();
          mbar_wait(bars.dfull, nd & 1u);
          ptimer.after_wait();
          ++nd;
          tc::fence_after();
        }
#pragma unroll 1
        for (int i = 0; i < CPE; ++i) {
          const int cl = eg + EG * i;
          const int64_t c = c0 + cl;
          const bool valid = c < a.n;
          const float zc[4] = {zn[0], zn[1], zn[2], zn[3]};
          ldz(i + 1, zn);
          const float* sd = sds + cl * 20;
          float X[NCOLB];
          if (top) {
            const float dL[NCOLB] = {sd[0], valid ? 1.f : 0.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) X[j] = wl * dL[j];
          } else {
            float v8[8], v2[2];
            tc_ld_sum8<C>(taddr, cl * NCOLB, v8);
            tc_ld_sum2<C>(taddr, cl * NCOLB + 8, v2);
#pragma unroll
            for (int j = 0; j < 8; ++j) X[j] = v8[j];
            X[8] = v2[0];
            X[9] = v2[1];
          }
          float t[20];
          {
            float v16[16], v4[4];
            tc::tmem_ld16(tstash + i * 20, v16);
            tc::tmem_ld4(tstash + i * 20 + 16, v4);
#pragma unroll
            for (int j = 0; j < 16; ++j) t[j] = v16[j];
#pragma unroll
            for (int j = 0; j < 4; ++j) t[16 + j] = v4[j];
          }
          const float r0 = sd[5], r1 = sd[6], r2 = sd[7];
          const float u0 = sd[8], u1 = sd[9], u2 = sd[10], v0 = sd[11], v1 = sd[12], v2_ = sd[13];
          float dl[NCOLB], pv[NCOLB];
#pragma unroll
          for (int j = 0; j < NCOLB; ++j) dl[j] = pv[j] = 0.f;
          float w0p[3] = {0.f, 0.f, 0.f};
          if (mok && valid) {
            const float tr = fmaf(r0, zc[1], fmaf(r1, zc[2], r2 * zc[3]));
            const typename AF::C cc = AF::centre(zc[0], beta);
            float zbar = 0.f;
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const float Aa = t[5 * p], Sa = t[5 * p + 1], P = t[5 * p + 2], Dd = t[5 * p + 3], Z = t[5 * p + 4];
              const float XA = X[2 + 2 * p], XS = X[3 + 2 * p];
              const float dA = om * fmaf(XA, P, 2.0f * XS * Dd);
              const float dS = om * fmaf(0.5f * XA, Dd, XS * P);
              zbar = fmaf(XA, Dd, fmaf(XS, Z, zbar));
              dl[2 + 2 * p] = dA;
              dl[3 + 2 * p] = dS;
              pv[2 + 2 * p] = Aa;
              pv[3 + 2 * p] = Sa;
              if (l == 0) {  // a^{-1} of pair columns: A -> h d_p, S -> 0
                const float dpx = p == 0 ? u0 : (p == 1 ? v0 : (p == 2 ? u0 + v0 : u0 - v0));
                const float dpy = p == 0 ? u1 : (p == 1 ? v1 : (p == 2 ? u1 + v1 : u1 - v1));
                const float dpz = p == 0 ? u2 : (p == 1 ? v2_ : (p == 2 ? u2 + v2_ : u2 - v2_));
                w0p[0] = fmaf(dA, h * dpx, w0p[0]);
                w0p[1] = fmaf(dA, h * dpy, w0p[1]);
                w0p[2] = fmaf(dA, h * dpz, w0p[2]);
              }
            }
            const float s1 = AF::d1(cc, beta), s2 = AF::d2(cc, beta);
            const float Xc = X[0], Xt = X[1];
            const float zb = fmaf(Xc, s1, fmaf(s2 * tr, Xt, zbar));
            dl[0] = om * zb;
            dl[1] = om * s1 * Xt;
            pv[0] = AF::value(cc, beta);
            pv[1] = s1 * tr;
            if (l == 0) {  // a^{-1}: centre -> x0, tangent -> r
              w0p[0] = fmaf(dl[0], sd[16], fmaf(dl[1], r0, w0p[0]));
              w0p[1] = fmaf(dl[0], sd[17], fmaf(dl[1], r1, w0p[1]));
              w0p[2] = fmaf(dl[0], sd[18], fmaf(dl[1], r2, w0p[2]));
            }
          }
          if (valid) {
            if (l >= 1) {
              float* dp = a.del + ((size_t)l * nrows + (size_t)c * NCOLB) * MPAD + m;
#pragma unroll
              for (int j = 0; j < NCOLB; ++j) dp[j * MPAD] = dl[j];
            }
            if (l <= L - 3) {
              float* ap = a.actv + ((size_t)l * nrows + (size_t)c * NCOLB) * MPAD + m;
#pragma unroll
              for (int j = 0; j < NCOLB; ++j) ap[j * MPAD] = pv[j];
            }
          }
          if (l >= 1) {
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) tc_put_b<C>(Bs, cl * NCOLB + j, m, dl[j]);
          }
          s_db += dl[0];
          if (top) {
            const float dL[NCOLB] = {sd[0], valid ? 1.f : 0.f, 0.f, sd[1], 0.f, sd[2], 0.f, sd[3], 0.f, sd[4]};
            float v = 0.f;
#pragma unroll
            for (int j = 0; j < NCOLB; ++j) v = fmaf(dL[j], pv[j], v);
            s_vL += v;
          }
          if (l == 0) {
            s_w0[0] += w0p[0];
            s_w0[1] += w0p[1];
            s_w0[2] += w0p[2];
          }
        }
        if (l >= 1) {
          tc_epi_arrive(bars);
        } else if (!top) {
          tc::fence_before();
        }
        r_db[l] += s_db;
        if (top) r_dWL += s_vL;
        if (l == 0) {
          r_dW0[0] += s_w0[0];
          r_dW0[1] += s_w0[1];
          r_dW0[2] += s_w0[2];
        }
      }
      if (m == 0) {  // bias of the last layer: sum of the centre seeds (fbar) of this group
        float v = 0.f;
        for (int i = 0; i < CPE; ++i) v += sds[(eg + EG * i) * 20 + 0];
        r_dbL += v;
      }
    }
    // write this thread's slots (every element of the slot is owned by exactly one thread)
    for (int l = 0; l <= L - 2; ++l) acc_db[(size_t)l * MPAD + m] = r_db[l];
    acc_dWL[m] = r_dWL;
    acc_dW0[m * 3 + 0] = r_dW0[0];
    acc_dW0[m * 3 + 1] = r_dW0[1];
    acc_dW0[m * 3 + 2] = r_dW0[2];
    if (m == 0) acc_dbL[0] = r_dbL;
    ptimer.report("bwd_tc", et == 0);
  }
  tc_teardown<C>(tbase);
}

template <int ACT, int MPAD>
static cudaError_t launch_bwd_tc_t(const BwdArgs& a, int grid, cudaStream_t st) {
  using C = BtcCfg<MPAD>;
  auto k = bwd_tc_kernel<ACT, MPAD>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::BYTES);
  if (e != cudaSuccess) return e;
  k<<<grid, C::NTHR, C::BYTES, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bwd_tc(const BwdArgs& a, int grid, cudaStream_t st) {
  const int act = a.net.act, mp = a.net.mpad;
#define FDSDF_CASE(A, MP) \
  if (act == A && mp == MP) return launch_bwd_tc_t<A, MP>(a, grid, st);
  FDSDF_CASE(ACT_SINE, 128)
  FDSDF_CASE(ACT_SINE, 256)
  FDSDF_CASE(ACT_SOFTPLUS, 128)
  FDSDF_CASE(ACT_SOFTPLUS, 256)
#undef FDSDF_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fdsdf
