// act.cuh -- cancellation-free activation maps of the pair-symmetric difference form.
//
// The stencil of PAPER.md L83-91 consists of the centre x0 and four symmetric pairs
// x0 +- h*d_p with d_p in {u, v, u+v, u-v}:
//     f_uu = S_u / h^2,  f_vv = S_v / h^2,  f_uv = (S_{u+v} - S_{u-v}) / (4 h^2),
// where S_p = f(x0 + h d_p) + f(x0 - h d_p) - 2 f(x0).  (f_pp - f_pm - f_mp + f_mm
// regroups as S_{u+v} - S_{u-v}.)  Instead of the 8 absolute values the kernels carry, per
// pair and per neuron, the odd part A = (z+ - z-)/2 and the even part S = z+ + z- - 2 z0 of
// the pre-activations, through every layer:
//     A^{l+1} = W A_a^l,  S^{l+1} = W S_a^l          (no bias: it cancels exactly)
//     A_a = (sigma(y+A) - sigma(y-A))/2,  S_a = sigma(y+A) + sigma(y-A) - 2 sigma(z),
//     y = z + S/2,  z = the centre pre-activation.
// Both maps are evaluated with identities that contain no difference of nearly equal
// numbers, so S (an O(h^2) quantity) is carried with fp32 RELATIVE precision and the
// final S_p^L is obtained without the 1/h^2 cancellation of the printed formula
// (DESIGN.md §4 derives every identity below).  Mathematically the result is identical
// to evaluating f at the 9 stencil points.
//
// Backward: with adjoints (Xa, Xs) of (A_a, S_a),
//     A_bar = Xa P + 2 Xs Dd,   S_bar = Xa Dd / 2 + Xs P,   z_bar += Xa Dd + Xs Z,
// where P = dA_a/dA = dS_a/dS, Dd = dA_a/dz = 2 dA_a/dS = dS_a/dA / 2, Z = dS_a/dz.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

// 1: the sine pair maps take the fast series form when the whole warp's arguments are small
#ifndef FDSDF_PAIR_FAST
#define FDSDF_PAIR_FAST 1
#endif

namespace fdsdf {

template <int ACT>
struct Act;

// ----------------------------------------------------------------------------- SIREN: sigma = sin
template <>
struct Act<ACT_SINE> {
  struct C {
    float sz, cz;
  };
  __device__ __forceinline__ static C centre(float z, float /*beta*/) {
    C c;
    sincos_acc(z, &c.sz, &c.cz);
    return c;
  }
  // the centre terms of two centres at once (packed sincos: bitwise centre() of each)
  __device__ __forceinline__ static void centre2(float za, float zb, float /*beta*/, C& ca, C& cb) {
    float2 sv, cv;
    sincos_acc2(make_float2(za, zb), &sv, &cv);
    ca.sz = sv.x;
    ca.cz = cv.x;
    cb.sz = sv.y;
    cb.cz = cv.y;
  }
  __device__ __forceinline__ static float value(const C& c, float) { return c.sz; }
  __device__ __forceinline__ static float d1(const C& c, float) { return c.cz; }
  __device__ __forceinline__ static float d2(const C& c, float) { return -c.sz; }

  // shared part of forward / backward: sin/cos of y = z + S/2 and of A
  struct P2 {
    float sy, cy, sA, cA, s2A, dys, dyc;
  };
  __device__ __forceinline__ static P2 pre(const C& c, float A, float S) {
    P2 p;
    float sh, ch, ss, cs;
    sincos_small(0.5f * A, &sh, &ch);
    sincos_small(0.25f * S, &ss, &cs);
    p.sA = 2.0f * sh * ch;
    p.s2A = sh * sh;
    p.cA = fmaf(-2.0f, p.s2A, 1.0f);
    const float sS2 = 2.0f * ss * cs;  // sin(S/2)
    const float s2S = ss * ss;         // sin^2(S/4)
    p.dys = fmaf(sS2, c.cz, -2.0f * s2S * c.sz);   // sin y - sin z
    p.dyc = fmaf(-sS2, c.sz, -2.0f * s2S * c.cz);  // cos y - cos z
    p.sy = c.sz + p.dys;
    p.cy = c.cz + p.dyc;
    return p;
  }
  __device__ __forceinline__ static void pair_fwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa) {
    const P2 p = pre(c, A, S);
    *Aa = p.cy * p.sA;                           // (sin(y+A) - sin(y-A))/2
    *Sa = fmaf(-4.0f * p.sy, p.s2A, 2.0f * p.dys);  // sin(y+A)+sin(y-A)-2 sin z
  }

  // Fast form of pre() for |A| <= FAST_A and |S| <= FAST_S (the whole warp, chosen per centre
  // by pairs_fwd4 / pairs_bwd4 with a vote, so there is no divergent branch): sin A and
  // sin^2(A/2), sin(S/2) and sin^2(S/4) straight from their Taylor series in A^2 and (S/2)^2 --
  // no half-angle sincos, no range tests.  Truncation (first omitted term) relative to the
  // value: sin A  A^10/11! <= 2.4e-11, sin^2(A/2)  A^10/(2 * 12!/...) <= 4e-12, sin(S/2) (S/2)^8/9!
  // <= 2e-14, sin^2(S/4) (S/2)^6/20160 <= 2e-10 -- all below fp32 rounding, and every series
  // keeps the RELATIVE precision of the small quantities.
  static constexpr float FAST_A = 0.5f, FAST_S = 0.25f;
  __device__ __forceinline__ static P2 pre_fast(const C& c, float A, float S) {
    P2 p;
    const float a2 = A * A;
    float q = fmaf(a2, 2.7557319224e-6f, -1.9841269841e-4f);  // sin A = A (1 - A^2/6 + ... + A^8/9!)
    q = fmaf(a2, q, 8.3333333333e-3f);
    q = fmaf(a2, q, -1.6666666667e-1f);
    p.sA = fmaf(A * a2, q, A);
    float r = fmaf(a2, 1.3778659612e-7f, -1.2400793651e-5f);  // sin^2(A/2) = A^2/4 - A^4/48 + ... + A^10/7257600
    r = fmaf(a2, r, 6.9444444444e-4f);
    r = fmaf(a2, r, -2.0833333333e-2f);
    r = fmaf(a2, r, 0.25f);
    p.s2A = a2 * r;
    p.cA = fmaf(-2.0f, p.s2A, 1.0f);
    const float y = 0.5f * S, y2 = y * y;
    float t = fmaf(y2, -1.9841269841e-4f, 8.3333333333e-3f);  // sin y, y = S/2
    t = fmaf(y2, t, -1.6666666667e-1f);
    const float sS2 = fmaf(y * y2, t, y);
    float w = fmaf(y2, 6.9444444444e-4f, -2.0833333333e-2f);  // sin^2(y/2) = y^2/4 - y^4/48 + y^6/1440
    w = fmaf(y2, w, 0.25f);
    const float s2S = y2 * w;
    p.dys = fmaf(sS2, c.cz, -2.0f * s2S * c.sz);   // sin y - sin z
    p.dyc = fmaf(-sS2, c.sz, -2.0f * s2S * c.cz);  // cos y - cos z
    p.sy = c.sz + p.dys;
    p.cy = c.cz + p.dyc;
    return p;
  }
  // all 4 pairs of a centre: o[2p] = A_a, o[2p+1] = S_a (warp-uniform choice of the fast form)
  __device__ __forceinline__ static void pairs_fwd4(const C& c, const float (&A)[4], const float (&S)[4], float beta,
                                                    float (&o)[8]) {
    const float mA = fmaxf(fmaxf(fabsf(A[0]), fabsf(A[1])), fmaxf(fabsf(A[2]), fabsf(A[3])));
    const float mS = fmaxf(fmaxf(fabsf(S[0]), fabsf(S[1])), fmaxf(fabsf(S[2]), fabsf(S[3])));
    if (FDSDF_PAIR_FAST && __all_sync(0xffffffffu, mA <= FAST_A && mS <= FAST_S)) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const P2 p = pre_fast(c, A[q], S[q]);
        o[2 * q] = p.cy * p.sA;
        o[2 * q + 1] = fmaf(-4.0f * p.sy, p.s2A, 2.0f * p.dys);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) pair_fwd(c, A[q], S[q], beta, &o[2 * q], &o[2 * q + 1]);
    }
  }
  __device__ __forceinline__ static void pair_bwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa, float* P, float* Dd, float* Z) {
    const P2 p = pre(c, A, S);
    bwd_from(p, Aa, Sa, P, Dd, Z);
  }
  __device__ __forceinline__ static void bwd_from(const P2& p, float* Aa, float* Sa, float* P, float* Dd, float* Z) {
    *Aa = p.cy * p.sA;
    *Sa = fmaf(-4.0f * p.sy, p.s2A, 2.0f * p.dys);
    *P = p.cy * p.cA;
    *Dd = -p.sy * p.sA;
    *Z = fmaf(-4.0f * p.cy, p.s2A, 2.0f * p.dyc);
  }
  // pre_fast on two pairs at once (packed fp32 x2: per lane exactly the scalar arithmetic)
  struct P2x2 {
    float2 sy, cy, sA, cA, s2A, dys, dyc;
  };
  __device__ __forceinline__ static P2x2 pre_fast2(const C& c, float2 A, float2 S) {
    P2x2 p;
    const float2 a2 = mul2(A, A);
    float2 q = fma2(a2, f2s(2.7557319224e-6f), f2s(-1.9841269841e-4f));
    q = fma2(a2, q, f2s(8.3333333333e-3f));
    q = fma2(a2, q, f2s(-1.6666666667e-1f));
    p.sA = fma2(mul2(A, a2), q, A);
    float2 r = fma2(a2, f2s(1.3778659612e-7f), f2s(-1.2400793651e-5f));
    r = fma2(a2, r, f2s(6.9444444444e-4f));
    r = fma2(a2, r, f2s(-2.0833333333e-2f));
    r = fma2(a2, r, f2s(0.25f));
    p.s2A = mul2(a2, r);
    p.cA = fma2(f2s(-2.0f), p.s2A, f2s(1.0f));
    const float2 y = mul2(f2s(0.5f), S), y2 = mul2(y, y);
    float2 t = fma2(y2, f2s(-1.9841269841e-4f), f2s(8.3333333333e-3f));
    t = fma2(y2, t, f2s(-1.6666666667e-1f));
    const float2 sS2 = fma2(mul2(y, y2), t, y);
    float2 w = fma2(y2, f2s(6.9444444444e-4f), f2s(-2.0833333333e-2f));
    w = fma2(y2, w, f2s(0.25f));
    const float2 s2S = mul2(y2, w);
    // (-2 s2S) sz = s2S (-2 sz) and (-sS2) sz = sS2 (-sz) exactly (power-of-two / sign scalings)
    p.dys = fma2(sS2, f2s(c.cz), mul2(s2S, f2s(-2.0f * c.sz)));
    p.dyc = fma2(sS2, f2s(-c.sz), mul2(s2S, f2s(-2.0f * c.cz)));
    p.sy = add2(f2s(c.sz), p.dys);
    p.cy = add2(f2s(c.cz), p.dyc);
    return p;
  }
  __device__ __forceinline__ static bool fast_ok(const float2 (&A)[2], const float2 (&S)[2]) {
    const float mA = fmaxf(fmaxf(fabsf(A[0].x), fabsf(A[0].y)), fmaxf(fabsf(A[1].x), fabsf(A[1].y)));
    const float mS = fmaxf(fmaxf(fabsf(S[0].x), fabsf(S[0].y)), fmaxf(fabsf(S[1].x), fabsf(S[1].y)));
    return FDSDF_PAIR_FAST && __all_sync(0xffffffffu, mA <= FAST_A && mS <= FAST_S);
  }
  // all 4 pairs of a centre, packed by two: A[k] = (A_{2k}, A_{2k+1}), S[k] likewise; out the same
  // packing of A_a, S_a (warp-uniform choice of the fast form; every lane of the warp calls this)
  __device__ __forceinline__ static void pairs_fwd4x2(const C& c, const float2 (&A)[2], const float2 (&S)[2],
                                                      float beta, float2 (&Aa)[2], float2 (&Sa)[2]) {
    if (fast_ok(A, S)) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const P2x2 p = pre_fast2(c, A[k], S[k]);
        Aa[k] = mul2(p.cy, p.sA);
        Sa[k] = fma2(mul2(f2s(-4.0f), p.sy), p.s2A, mul2(f2s(2.0f), p.dys));
      }
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        pair_fwd(c, A[k].x, S[k].x, beta, &Aa[k].x, &Sa[k].x);
        pair_fwd(c, A[k].y, S[k].y, beta, &Aa[k].y, &Sa[k].y);
      }
    }
  }
  // + the derivative factors P, Dd, Z (same packing)
  __device__ __forceinline__ static void pairs_bwd4x2(const C& c, const float2 (&A)[2], const float2 (&S)[2],
                                                      float beta, float2 (&Aa)[2], float2 (&Sa)[2], float2 (&P)[2],
                                                      float2 (&Dd)[2], float2 (&Z)[2]) {
    if (fast_ok(A, S)) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const P2x2 p = pre_fast2(c, A[k], S[k]);
        Aa[k] = mul2(p.cy, p.sA);
        Sa[k] = fma2(mul2(f2s(-4.0f), p.sy), p.s2A, mul2(f2s(2.0f), p.dys));
        P[k] = mul2(p.cy, p.cA);
        Dd[k] = mul2(make_float2(-p.sy.x, -p.sy.y), p.sA);
        Z[k] = fma2(mul2(f2s(-4.0f), p.cy), p.s2A, mul2(f2s(2.0f), p.dyc));
      }
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        pair_bwd(c, A[k].x, S[k].x, beta, &Aa[k].x, &Sa[k].x, &P[k].x, &Dd[k].x, &Z[k].x);
        pair_bwd(c, A[k].y, S[k].y, beta, &Aa[k].y, &Sa[k].y, &P[k].y, &Dd[k].y, &Z[k].y);
      }
    }
  }
  // all 4 pairs of a centre: t[5p .. 5p+4] = A_a, S_a, P, Dd, Z (warp-uniform fast form);
  // `all` = every lane of the warp calls this (else the general form, no vote)
  __device__ __forceinline__ static void pairs_bwd4(const C& c, const float (&A)[4], const float (&S)[4], float beta,
                                                    float (&t)[20]) {
    const float mA = fmaxf(fmaxf(fabsf(A[0]), fabsf(A[1])), fmaxf(fabsf(A[2]), fabsf(A[3])));
    const float mS = fmaxf(fmaxf(fabsf(S[0]), fabsf(S[1])), fmaxf(fabsf(S[2]), fabsf(S[3])));
    if (FDSDF_PAIR_FAST && __all_sync(0xffffffffu, mA <= FAST_A && mS <= FAST_S)) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        bwd_from(pre_fast(c, A[q], S[q]), &t[5 * q], &t[5 * q + 1], &t[5 * q + 2], &t[5 * q + 3], &t[5 * q + 4]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        pair_bwd(c, A[q], S[q], beta, &t[5 * q], &t[5 * q + 1], &t[5 * q + 2], &t[5 * q + 3], &t[5 * q + 4]);
    }
  }
};

// ----------------------------------------------------------------------------- softplus_beta
// sigma(z) = sp(beta z)/beta, sp(t) = log(1 + e^t); s(t) = logistic.
template <>
struct Act<ACT_SOFTPLUS> {
  // s(t) and 1 - s(t) = s(-t) from ONE exponential: e = exp(-|t|) <= 1, r = 1 / (1 + e);
  // the larger of the two is r, the smaller e r (both with fp32 relative precision)
  __device__ __forceinline__ static void logistic2(float t, float* s, float* sm) {
    const float e = expf(-fabsf(t));
    const float r = __fdividef(1.0f, 1.0f + e);
    const float lo = e * r;
    *s = t >= 0.0f ? r : lo;
    *sm = t >= 0.0f ? lo : r;
  }
  struct C {
    float t, s0, s0m;  // beta z, s(t), 1 - s(t)
  };
  __device__ __forceinline__ static C centre(float z, float beta) {
    C c;
    c.t = beta * z;
    logistic2(c.t, &c.s0, &c.s0m);
    return c;
  }
  __device__ __forceinline__ static void centre2(float za, float zb, float beta, C& ca, C& cb) {
    ca = centre(za, beta);
    cb = centre(zb, beta);
  }
  __device__ __forceinline__ static float value(const C& c, float beta) { return softplus_acc(c.t) / beta; }
  __device__ __forceinline__ static float d1(const C& c, float) { return c.s0; }
  __device__ __forceinline__ static float d2(const C& c, float beta) { return beta * c.s0 * c.s0m; }

  struct P2 {
    float sy, sym, ps, ea, ema, ima, E, em_d;
  };
  __device__ __forceinline__ static P2 pre(const C& c, float A, float S, float beta) {
    P2 p;
    const float a = beta * A;
    const float d = 0.5f * beta * S;
    const float ty = c.t + d;
    logistic2(ty, &p.sy, &p.sym);          // s(ty), 1 - s(ty)
    p.ps = p.sy * p.sym;                   // s(ty)(1 - s(ty))
    p.ea = expm1f(a);                      // e^a - 1
    p.ima = __fdividef(1.0f, 1.0f + p.ea); // e^-a
    p.ema = -p.ea * p.ima;                 // e^-a - 1
    p.E = p.ea * (-p.ema);                 // e^a - 2 + e^-a = 4 sinh^2(a/2) >= 0
    p.em_d = expm1f(d);
    return p;
  }
  __device__ __forceinline__ static void fwd_from(const C& c, const P2& p, float beta, float* Aa, float* Sa) {
    const float ib = 1.0f / beta;
    // sp(ty+a) - sp(ty-a) = log((1 + s ea) / (1 + s ema)) = log1p(s (ea - ema) / (1 + s ema)),
    // 1 + s ema = (1 - s) + s e^-a  (sums of positive terms only)
    *Aa = 0.5f * ib * log1pf(p.sy * (p.ea - p.ema) / fmaf(p.sy, p.ima, p.sym));
    // sp(ty+a)+sp(ty-a)-2sp(ty) = log1p(s(1-s) E);  sp(ty)-sp(t) = log1p(s0 expm1(d))
    *Sa = ib * (log1pf(p.ps * p.E) + 2.0f * log1pf(c.s0 * p.em_d));
  }
  __device__ __forceinline__ static void pair_fwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa) {
    const P2 p = pre(c, A, S, beta);
    fwd_from(c, p, beta, Aa, Sa);
  }
  __device__ __forceinline__ static void pairs_fwd4(const C& c, const float (&A)[4], const float (&S)[4], float beta,
                                                    float (&o)[8]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) pair_fwd(c, A[q], S[q], beta, &o[2 * q], &o[2 * q + 1]);
  }
  __device__ __forceinline__ static void pairs_bwd4(const C& c, const float (&A)[4], const float (&S)[4], float beta,
                                                    float (&t)[20]) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      pair_bwd(c, A[q], S[q], beta, &t[5 * q], &t[5 * q + 1], &t[5 * q + 2], &t[5 * q + 3], &t[5 * q + 4]);
  }
  // the packed-by-two interface of the sine maps (scalar arithmetic here)
  __device__ __forceinline__ static void pairs_fwd4x2(const C& c, const float2 (&A)[2], const float2 (&S)[2],
                                                      float beta, float2 (&Aa)[2], float2 (&Sa)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      pair_fwd(c, A[k].x, S[k].x, beta, &Aa[k].x, &Sa[k].x);
      pair_fwd(c, A[k].y, S[k].y, beta, &Aa[k].y, &Sa[k].y);
    }
  }
  __device__ __forceinline__ static void pairs_bwd4x2(const C& c, const float2 (&A)[2], const float2 (&S)[2],
                                                      float beta, float2 (&Aa)[2], float2 (&Sa)[2], float2 (&P)[2],
                                                      float2 (&Dd)[2], float2 (&Z)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      pair_bwd(c, A[k].x, S[k].x, beta, &Aa[k].x, &Sa[k].x, &P[k].x, &Dd[k].x, &Z[k].x);
      pair_bwd(c, A[k].y, S[k].y, beta, &Aa[k].y, &Sa[k].y, &P[k].y, &Dd[k].y, &Z[k].y);
    }
  }
  __device__ __forceinline__ static void pair_bwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa, float* P, float* Dd, float* Z) {
    const P2 p = pre(c, A, S, beta);
    fwd_from(c, p, beta, Aa, Sa);
    const float den = __fdividef(1.0f, fmaf(p.ps, p.E, 1.0f));
    const float one_m_2s = p.sym - p.sy;                              // 1 - 2 s(ty)
    const float even = p.E * p.ps * one_m_2s * den;                   // s(ty+a)+s(ty-a)-2s(ty)
    const float odd = (p.ea - p.ema) * p.ps * den;                    // s(ty+a)-s(ty-a)
    *P = 0.5f * (2.0f * p.sy + even);
    *Dd = 0.5f * odd;
    // s(ty) - s(t) = -s(ty)(1-s(t)) expm1(-d),  expm1(-d) = -expm1(d) / (1 + expm1(d))
    const float dsy = p.sy * c.s0m * (p.em_d / (1.0f + p.em_d));
    *Z = even + 2.0f * dsy;
  }
};

}  // namespace fdsdf
