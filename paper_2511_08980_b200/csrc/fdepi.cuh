// fdepi.cuh -- per-centre pieces shared by the FFMA (fwd.cu) and tensor-core (fwd_tc.cu)
// forward kernels, so both compute bit-identical epilogues:
//   * centre_frame: degenerate mask m = [|g| >= eps] and the uniformly random
//     right-handed tangent frame (u, v) of n = g/|g| (reading 6);
//   * fd_centre: f_uu, f_vv, f_uv (§3.1) from the pair sums S_p, D_FD,
//     K_FD (P:L112 with the §3.4 replacement P:L131), the per-centre Eq. (1) terms
//      and the backward seeds.
#pragma once
#include "kernels.cuh"

namespace fdsdf {

__device__ __forceinline__ double sgn_d(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// x^p for an integer p >= 0 (the |g|^p denominator, P:L112 p = 4) by repeated squaring
__device__ __forceinline__ double ipow_d(double x, int p) {
  double r = 1.0;
  while (p > 0) {
    if (p & 1) r *= x;
    x *= x;
    p >>= 1;
  }
  return r;
}

// cinfo layout per centre (16 floats): f, g0, g1, g2, u0, u1, u2, v0, v1, v2, mask, 0...
constexpr int NCINFO = 16;

// Mask + frame of centre c (global row c, valid = c < n); writes ci[0..15] and the optional
// eval outputs.  Frames: GIVEN mode copies d_frames_in; RANDOM mode draws theta from the
// counter-based SplitMix64 of (seed, global index) and rotates the Duff et al. ONB.
__device__ __forceinline__ void centre_frame(const FwdArgs& a, int64_t c, bool valid, float f, float g0, float g1,
                                             float g2, float* ci) {
  const double gnd = sqrt((double)g0 * g0 + (double)g1 * g1 + (double)g2 * g2);
  const bool msk = valid && (gnd >= (double)a.ls.eps_grad);
  float u[3] = {0.f, 0.f, 0.f}, v[3] = {0.f, 0.f, 0.f};
  if (valid && a.frame_given) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      u[d] = a.frames_in[c * 6 + d];
      v[d] = a.frames_in[c * 6 + 3 + d];
    }
  } else if (msk) {
    // branchless right-handed ONB of n (Duff et al. 2017), s = +1 for n_z >= 0 (incl. -0)
    const double nx = g0 / gnd, ny = g1 / gnd, nz = g2 / gnd;
    const double s = (nz >= 0.0) ? 1.0 : -1.0;
    const double aa = -1.0 / (s + nz);
    const double bb = nx * ny * aa;
    const double b1[3] = {1.0 + s * nx * nx * aa, s * bb, -s * nx};
    const double b2[3] = {bb, s + ny * ny * aa, -ny};
    const uint64_t gidx = (uint64_t)(a.index_offset + c);
    const uint64_t k = mix64(a.frame_seed + (gidx + 1ull) * 0x9E3779B97F4A7C15ull) >> 11;
    const double th = 6.283185307179586 * ((double)k * 0x1.0p-53);
    double st, ct;
    sincos(th, &st, &ct);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      u[d] = (float)(ct * b1[d] + st * b2[d]);
      v[d] = (float)(-st * b1[d] + ct * b2[d]);
    }
  }
  ci[0] = f;
  ci[1] = g0;
  ci[2] = g1;
  ci[3] = g2;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    ci[4 + d] = u[d];
    ci[7 + d] = v[d];
  }
  ci[10] = msk ? 1.f : 0.f;
#pragma unroll
  for (int q = 11; q < NCINFO; ++q) ci[q] = 0.f;
  if (valid) {
    if (a.out_f) a.out_f[c] = f;
    if (a.out_g) {
      a.out_g[c * 3 + 0] = g0;
      a.out_g[c * 3 + 1] = g1;
      a.out_g[c * 3 + 2] = g2;
    }
    if (a.out_mask) a.out_mask[c] = msk ? 1 : 0;
    if (a.out_frames) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        a.out_frames[c * 6 + d] = u[d];
        a.out_frames[c * 6 + 3 + d] = v[d];
      }
    }
  }
}

// FD epilogue of centre cc from its output pair sums Ssum = (S_u, S_v, S_{u+v}, S_{u-v}) and
// its cinfo cj.  Writes the eval outputs, the backward seeds (step mode) and lv[NLOSS].
__device__ __forceinline__ void fd_centre(const FwdArgs& a, int64_t cc, bool valid2, const float (&Ssum)[4],
                                          const float* cj, double (&lv)[NLOSS]) {
  const float ih2 = 1.0f / (a.h * a.h);
  const float f = cj[0], g0 = cj[1], g1 = cj[2], g2 = cj[3];
  const bool msk = cj[10] != 0.f;
  const float fuu = Ssum[0] * ih2;
  const float fvv = Ssum[1] * ih2;
  const float fuv = (Ssum[2] - Ssum[3]) * (0.25f * ih2);
  const double D = (double)fuu * fvv - (double)fuv * fuv;
  const double gn = sqrt((double)g0 * g0 + (double)g1 * g1 + (double)g2 * g2);
  const bool surf = cc < a.n_surface;
  const LossCfg& ls = a.ls;
  bool den_live = false;
  double den = 1.0;
  if (ls.denom == 2 || (ls.denom == 0 && !surf)) {
    den = ipow_d(gn, ls.denom_pow);
    den_live = true;
  }
  if (!msk) {
    den = 1.0;
    den_live = false;
  }
  const double K = msk ? D / den : 0.0;
  const double Q = (ls.kind == 0) ? K : D;
  const double af = fabs((double)f);
  lv[0] = (valid2 && surf) ? af : 0.0;
  lv[1] = (valid2 && !surf) ? exp(-(double)ls.alpha * af) : 0.0;
  lv[2] = valid2 ? (gn - 1.0) * (gn - 1.0) : 0.0;
  lv[3] = (valid2 && msk) ? (ls.fd_form == 0 ? fabs(Q) : Q * Q) : 0.0;
  lv[4] = (valid2 && !msk) ? 1.0 : 0.0;
  lv[5] = 0.0;
  if (!valid2) return;
  if (a.out_hess) {
    a.out_hess[cc * 3 + 0] = fuu;
    a.out_hess[cc * 3 + 1] = fuv;
    a.out_hess[cc * 3 + 2] = fvv;
  }
  if (a.out_K) a.out_K[cc] = (float)K;
  if (a.out_D) a.out_D[cc] = (float)D;
  if (a.step) {
    const double sf = sgn_d(f);
    const double fbar = surf ? (double)ls.w_dm * sf * ls.inv_ns
                             : (double)ls.lambda_dnm * (-(double)ls.alpha) * sf * exp(-(double)ls.alpha * af) *
                                   ls.inv_nu;
    const double gQ = msk ? (double)ls.lambda_fd * ls.inv_n * (ls.fd_form == 0 ? sgn_d(Q) : 2.0 * Q) : 0.0;
    const double gD = (ls.kind == 0) ? gQ / den : gQ;
    double cr = gn > 0.0 ? 2.0 * (double)ls.lambda_eik * ls.inv_n * (gn - 1.0) / gn : 0.0;
    if (ls.kind == 0 && den_live && gn > 0.0) cr += -(double)ls.denom_pow * gQ * Q / (gn * gn);
    float* sd = a.seed + cc * NSEED;
    const double ih2d = (double)ih2;
    sd[0] = (float)fbar;
    sd[1] = (float)(gD * fvv * ih2d);
    sd[2] = (float)(gD * fuu * ih2d);
    sd[3] = (float)(-0.5 * gD * fuv * ih2d);
    sd[4] = (float)(0.5 * gD * fuv * ih2d);
    sd[5] = (float)(cr * g0);
    sd[6] = (float)(cr * g1);
    sd[7] = (float)(cr * g2);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      sd[8 + d] = cj[4 + d];
      sd[11 + d] = cj[7 + d];
    }
    sd[14] = 0.f;
    sd[15] = 0.f;
  }
}

}  // namespace fdsdf
