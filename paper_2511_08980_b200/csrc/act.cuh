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
  __device__ __forceinline__ static void pair_bwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa, float* P, float* Dd, float* Z) {
    const P2 p = pre(c, A, S);
    *Aa = p.cy * p.sA;
    *Sa = fmaf(-4.0f * p.sy, p.s2A, 2.0f * p.dys);
    *P = p.cy * p.cA;
    *Dd = -p.sy * p.sA;
    *Z = fmaf(-4.0f * p.cy, p.s2A, 2.0f * p.dyc);
  }
};

// ----------------------------------------------------------------------------- softplus_beta
// sigma(z) = sp(beta z)/beta, sp(t) = log(1 + e^t); s(t) = logistic.
template <>
struct Act<ACT_SOFTPLUS> {
  struct C {
    float t, s0, s0m;  // beta z, s(t), 1 - s(t)
  };
  __device__ __forceinline__ static C centre(float z, float beta) {
    C c;
    c.t = beta * z;
    c.s0 = logistic_acc(c.t);
    c.s0m = logistic_acc(-c.t);
    return c;
  }
  __device__ __forceinline__ static float value(const C& c, float beta) { return softplus_acc(c.t) / beta; }
  __device__ __forceinline__ static float d1(const C& c, float) { return c.s0; }
  __device__ __forceinline__ static float d2(const C& c, float beta) { return beta * c.s0 * c.s0m; }

  struct P2 {
    float sy, ps, ea, ema, E, em_d;
  };
  __device__ __forceinline__ static P2 pre(const C& c, float A, float S, float beta) {
    P2 p;
    const float a = beta * A;
    const float d = 0.5f * beta * S;
    const float ty = c.t + d;
    p.sy = logistic_acc(ty);
    p.ps = p.sy * logistic_acc(-ty);       // s(ty)(1 - s(ty))
    p.ea = expm1f(a);                      // e^a - 1
    p.ema = -p.ea / (1.0f + p.ea);         // e^-a - 1
    p.E = p.ea * (-p.ema);                 // e^a - 2 + e^-a = 4 sinh^2(a/2) >= 0
    p.em_d = expm1f(d);
    return p;
  }
  __device__ __forceinline__ static void fwd_from(const C& c, const P2& p, float beta, float* Aa, float* Sa) {
    const float ib = 1.0f / beta;
    // sp(ty+a) - sp(ty-a) = log1p(s ea) - log1p(s ema)       (terms of opposite sign)
    *Aa = 0.5f * ib * (log1pf(p.sy * p.ea) - log1pf(p.sy * p.ema));
    // sp(ty+a)+sp(ty-a)-2sp(ty) = log1p(s(1-s) E);  sp(ty)-sp(t) = log1p(s0 expm1(d))
    *Sa = ib * (log1pf(p.ps * p.E) + 2.0f * log1pf(c.s0 * p.em_d));
  }
  __device__ __forceinline__ static void pair_fwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa) {
    const P2 p = pre(c, A, S, beta);
    fwd_from(c, p, beta, Aa, Sa);
  }
  __device__ __forceinline__ static void pair_bwd(const C& c, float A, float S, float beta, float* Aa,
                                                  float* Sa, float* P, float* Dd, float* Z) {
    const P2 p = pre(c, A, S, beta);
    fwd_from(c, p, beta, Aa, Sa);
    const float den = 1.0f / fmaf(p.ps, p.E, 1.0f);
    const float one_m_2s = -tanhf(0.5f * (c.t + 0.5f * beta * S));  // 1 - 2 s(ty)
    const float even = p.E * p.ps * one_m_2s * den;                   // s(ty+a)+s(ty-a)-2s(ty)
    const float odd = (p.ea - p.ema) * p.ps * den;                    // s(ty+a)-s(ty-a)
    *P = 0.5f * (2.0f * p.sy + even);
    *Dd = 0.5f * odd;
    // s(ty) - s(t) = -s(ty)(1-s(t)) expm1(-d)
    const float dsy = -p.sy * c.s0m * expm1f(-0.5f * beta * S);
    *Z = even + 2.0f * dsy;
  }
};

}  // namespace fdsdf
