// Device-side SDF evaluation for sm_100a: FP32 CUDA-core math with analytic
// derivatives (SQ / PSQ / half-space / booleans) and compact forward-mode jets
// (XPSQ), plus the smooth operators of §II-A.
//
// Citations: P:n = PAPER.md line n.  Derivative structure: DESIGN.md §5
// (SURVEY Appendix A).  This file shares no code with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "cm_internal.h"

namespace cmd {
using namespace cmi;

// Code-size control.  In the fused one-kernel manifold design the XPSQ
// evaluators had to stay out of line (inlined, its four phases overflowed the
// instruction cache).  The per-phase kernels hold one evaluation instance
// each, so the constant-schedule evaluator is inlined there (the call ABI
// spilled ~10% of the trace kernel's instructions to local memory; inlining:
// C5 +6%, C4 +23%); the varying-schedule jets stay out of line.
#ifndef CM_XPSQ_NOINLINE
#define CM_XPSQ_NOINLINE 1
#endif
#ifndef CM_XPSQ_CULL
#define CM_XPSQ_CULL 1   // skip XPSQ union operands with provably negligible weight (eval_shape)
#endif
#ifndef CM_XPSQ_INLINE_MAX_O
#define CM_XPSQ_INLINE_MAX_O 2   // constant-schedule XPSQ inlined up to this order
#endif
#ifndef CM_SQ_SHARED_W
#define CM_SQ_SHARED_W 1      // SQ weights from the LSE exponentials (fewer MUFU ops)
#endif
#ifndef CM_SOFTCLIP_FAST
#define CM_SOFTCLIP_FAST 0    // softclip interior shortcut: measured C5 -1.5%, C4 -1.7% (r02j sweep)
#endif
#ifndef CM_LEAF_LAZY_R
#define CM_LEAF_LAZY_R 0      // (retired by the 128-bit leaf loads) leaf rotation loaded only for rotated leaves: C5 -1.7%, C4 -1.2% (r02j)
#endif
#ifndef CM_XPSQ_TSPACE
#define CM_XPSQ_TSPACE 1      // curved roots outside the band: Newton-polished in t (near-straight splines)
#endif
#ifndef CM_SOFTCLIP_ACCURATE
#define CM_SOFTCLIP_ACCURATE 1
#endif
#ifndef CM_SHAPE_NOINLINE
#define CM_SHAPE_NOINLINE 0
#endif
#if CM_XPSQ_NOINLINE
#define CM_XINL __noinline__
#else
#define CM_XINL __forceinline__
#endif
#if CM_SHAPE_NOINLINE
#define CM_SINL __noinline__
#else
#define CM_SINL
#endif

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;
constexpr float SQ_GUARD = 1e-12f;  // |u|^p = exp(p log(u^2 + g)/2)

// MUFU approximations (ex2/lg2/rcp .approx: rel. error ~2^-22)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpa(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- §II-A smooth operators --------------------------------------
// sigma(x) = 1 / (1 + e^-x)
__device__ __forceinline__ float sigm(float x) { return rcpa(1.f + ex2(-x * LOG2E)); }
// s+(x; tau) = tau log(1 + e^(x/tau)) = max(x,0) + tau log(1 + e^(-|x|/tau))
__device__ __forceinline__ float softplus(float x, float tau, float itau) {
  return fmaxf(x, 0.f) + (tau * LN2) * lg2(1.f + ex2(-fabsf(x) * (itau * LOG2E)));
}
// soft clip = lo + s+(x - lo) - s+(x - hi)  (two softplus)
__device__ __forceinline__ float softclip(float x, float lo, float hi, float tau, float itau) {
  return lo + softplus(x - lo, tau, itau) - softplus(x - hi, tau, itau);
}
// d softclip / dx = sigma((x-lo)/tau) - sigma((x-hi)/tau)
__device__ __forceinline__ float softclip_d(float x, float lo, float hi, float itau) {
  return sigm((x - lo) * itau) - sigm((x - hi) * itau);
}
// s+(x; tau) and sigma(x / tau) from one exponential e = exp(-|x|/tau):
// s+ = max(x, 0) + tau log(1 + e), sigma = 1/(1+e) (x >= 0) or e/(1+e)
// (e and r = 1/(1+e) are returned too: sigma (1 - sigma) = e r^2 without
// the cancellation of 1 - sigma)
__device__ __forceinline__ void softplus_sig(float x, float tau, float itau, float& sp, float& sg, float& e, float& r) {
  e = ex2(-fabsf(x) * (itau * LOG2E));
  sp = fmaxf(x, 0.f) + (tau * LN2) * lg2(1.f + e);
  r = rcpa(1.f + e);
  sg = x >= 0.f ? r : e * r;
}
// softclip value with its first and second derivatives (two exponentials)
__device__ __forceinline__ void softclip_12(float x, float lo, float hi, float tau, float itau, float& v, float& d1,
                                            float& d2) {
  // interior: both exponentials are below 2^-144 and flush to 0 (ftz), so the
  // general path below returns exactly lo + (x - lo), 1, 0 -- skip its 6 MUFU ops
  if (CM_SOFTCLIP_FAST && (x - lo) * itau > 100.f && (hi - x) * itau > 100.f) {
    v = lo + (x - lo);
    d1 = 1.f;
    d2 = 0.f;
    return;
  }
  float sp1, s1, e1, r1, sp2, s2, e2, r2;
  softplus_sig(x - lo, tau, itau, sp1, s1, e1, r1);
  softplus_sig(x - hi, tau, itau, sp2, s2, e2, r2);
  v = lo + sp1 - sp2;
#if CM_SOFTCLIP_ACCURATE
  // above hi both sigmas are ~1: their difference is (e2 - e1) r1 r2
  d1 = x >= hi ? (e2 - e1) * r1 * r2 : s1 - s2;
  d2 = (e1 * r1 * r1 - e2 * r2 * r2) * itau;
#else
  d1 = s1 - s2;
  d2 = (s1 * (1.f - s1) - s2 * (1.f - s2)) * itau;
#endif
}

// cube root from the MUFU log / exp plus one Newton step (rel. error ~1e-7)
__device__ __forceinline__ float cbrt_fast(float x) {
  const float ax = fabsf(x);
  float y = ex2(lg2(ax) * (1.f / 3.f));          // ax = 0 -> 0
  if (y > 0.f && y < INFINITY) y = fmaf(1.f / 3.f, fmaf(ax, rcpa(y * y), -y), y);
  return copysignf(y, x);
}
// atan2(y, x) for y >= 0 (result in [0, pi]): octant reduction and an odd
// degree-15 polynomial on [0, 1] (abs. error ~1.2e-7)
__device__ __forceinline__ float atan2_pos(float y, float x) {
  const float ax = fabsf(x);
  const float mx = fmaxf(ax, y), mn = fminf(ax, y);
  const float a = mx > 0.f ? mn * rcpa(mx) : 0.f;
  const float t = a * a;
  float r = -0.004054551012814045f;
  r = fmaf(r, t, 0.02186291106045246f);
  r = fmaf(r, t, -0.055912282317876816f);
  r = fmaf(r, t, 0.09642196446657181f);
  r = fmaf(r, t, -0.1390863060951233f);
  r = fmaf(r, t, 0.19946566224098206f);
  r = fmaf(r, t, -0.33329862356185913f);
  r = fmaf(r, t, 0.9999993443489075f);
  r *= a;
  if (y > ax) r = 1.5707963267948966f - r;
  if (x < 0.f) r = 3.141592653589793f - r;
  return r;
}

// ---- results ---------------------------------------------------------------
// packed symmetric 3x3: xx, xy, xz, yy, yz, zz
template <int O> struct Res {
  float v;
  float g[3];
  float h[6];
};

__device__ __forceinline__ constexpr int hidx3(int i, int j) {
  return i <= j ? (i == 0 ? j : (i == 1 ? 2 + j : 5)) : (j == 0 ? i : (j == 1 ? 2 + i : 5));
}

// ---- rigid transforms -------------------------------------------------------
__device__ __forceinline__ void quat_to_R(const float* q, float* R) {
  float n = rsqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  float w = q[0] * n, x = q[1] * n, y = q[2] * n, z = q[3] * n;
  R[0] = 1.f - 2.f * (y * y + z * z); R[1] = 2.f * (x * y - w * z);       R[2] = 2.f * (x * z + w * y);
  R[3] = 2.f * (x * y + w * z);       R[4] = 1.f - 2.f * (x * x + z * z); R[5] = 2.f * (y * z - w * x);
  R[6] = 2.f * (x * z - w * y);       R[7] = 2.f * (y * z + w * x);       R[8] = 1.f - 2.f * (x * x + y * y);
}
// y = R^T (x - t)
__device__ __forceinline__ void to_local(const float* R, const float* t, const float* x, float* y) {
  float d0 = x[0] - t[0], d1 = x[1] - t[1], d2 = x[2] - t[2];
  y[0] = R[0] * d0 + R[3] * d1 + R[6] * d2;
  y[1] = R[1] * d0 + R[4] * d1 + R[7] * d2;
  y[2] = R[2] * d0 + R[5] * d1 + R[8] * d2;
}
__device__ __forceinline__ void rot_vec(const float* R, const float* a, float* b) {
  b[0] = R[0] * a[0] + R[1] * a[1] + R[2] * a[2];
  b[1] = R[3] * a[0] + R[4] * a[1] + R[5] * a[2];
  b[2] = R[6] * a[0] + R[7] * a[1] + R[8] * a[2];
}
// H_w = R H R^T (packed in, packed out)
__device__ __forceinline__ void rot_sym(const float* R, const float* h, float* o) {
  float H[3][3] = {{h[0], h[1], h[2]}, {h[1], h[3], h[4]}, {h[2], h[4], h[5]}};
  float M[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) M[i][j] = R[i * 3 + 0] * H[0][j] + R[i * 3 + 1] * H[1][j] + R[i * 3 + 2] * H[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j)
      o[hidx3(i, j)] = M[i][0] * R[j * 3 + 0] + M[i][1] * R[j * 3 + 1] + M[i][2] * R[j * 3 + 2];
}

// ---- streaming LSE with derivatives (Eq. (2)-(4)) ---------
// psi = tau log sum exp(v_i / tau),  grad = sum w g_i,
// hess = sum w (H_i + g_i g_i^T / tau) - grad grad^T / tau
template <int O> struct Acc {
  float m, S;
  float G[3];
  float H[6];
};
template <int O> __device__ __forceinline__ void acc_init(Acc<O>& a) {
  a.m = -INFINITY;
  a.S = 0.f;
#pragma unroll
  for (int i = 0; i < 3; ++i) a.G[i] = 0.f;
#pragma unroll
  for (int k = 0; k < 6; ++k) a.H[k] = 0.f;
}
// fold s * r into the accumulator (itl = log2(e) / tau, itau = 1 / tau)
template <int O> __device__ __forceinline__ void acc_fold(Acc<O>& a, float s, const Res<O>& r, float itl,
                                                          float itau) {
  float v = s * r.v;
  float dm = v - a.m;
  bool up = dm > 0.f;
  float e = ex2(-fabsf(dm) * itl);
  float cs = up ? e : 1.f;
  float cn = up ? 1.f : e;
  a.m = up ? v : a.m;
  a.S = fmaf(a.S, cs, cn);
  if constexpr (O >= 1) {
    float g[3] = {s * r.g[0], s * r.g[1], s * r.g[2]};
#pragma unroll
    for (int i = 0; i < 3; ++i) a.G[i] = fmaf(a.G[i], cs, cn * g[i]);
    if constexpr (O >= 2) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j) {
          int k = hidx3(i, j);
          a.H[k] = fmaf(a.H[k], cs, cn * fmaf(g[i] * g[j], itau, s * r.h[k]));
        }
    }
  }
}
template <int O> __device__ __forceinline__ void acc_final(const Acc<O>& a, float s, float tau, float itau,
                                                           Res<O>& r) {
  r.v = s * fmaf(tau * LN2, lg2(a.S), a.m);
  if constexpr (O >= 1) {
    float iS = rcpa(a.S);
    float g[3] = {a.G[0] * iS, a.G[1] * iS, a.G[2] * iS};
#pragma unroll
    for (int i = 0; i < 3; ++i) r.g[i] = s * g[i];
    if constexpr (O >= 2) {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j) {
          int k = hidx3(i, j);
          r.h[k] = s * fmaf(-g[i] * g[j], itau, a.H[k] * iS);
        }
    }
  }
}

// ---- superquadric, analytic value / gradient / Hessian ----------------------
// Eq. (1) with u_i = y_i / a_i, q_i = u_i^2 + g:
//   A_i = q_i^(1/eps2) (i = 0, 1), S = A_0 + A_1, B = S^(eps2/eps1),
//   C = q_2^(1/eps1), f = B + C;  phi = |y| (1 - f^(-eps1/2))  (reading #2).
// Everything in the log2 domain so that large exponents (eps -> 0.1) cannot
// overflow; beta = B/f, gamma = C/f, w_i = A_i/S are bounded ratios.
// grad L = grad f / f = 2 p1 (beta w0 s0, beta w1 s1, gamma s2),
//   s_i = u_i / (a_i q_i), c_i = d s_i / d y_i = (1 - 2 u_i^2/q_i) / (a_i^2 q_i),
// F2 = hess f / f: F2_ij (i,j < 2) = 2 p1 beta [2 (p1 - p2) w_i w_j s_i s_j
//   + delta_ij w_i (2 p2 s_i^2 + c_i)], F2_22 = 2 p1 gamma (2 p1 s2^2 + c2);
// grad phi = (1-h) yh + k r h L;
// hess phi = (1-h)(I - yh yh^T)/r + k h (yh L^T + L yh^T) + k r h (F2 - (1+k) L L^T)
template <int O, class SP> __device__ __forceinline__ void sq_eval(const SP& Lf, const float* y, Res<O>& r) {
  const float ia0 = Lf.ia[0], ia1 = Lf.ia[1], ia2 = Lf.ia[2];
  const float p1 = Lf.p1, p2 = Lf.p2, m = Lf.m, k = Lf.k;
  float u0 = y[0] * ia0, u1 = y[1] * ia1, u2 = y[2] * ia2;
  float q0 = fmaf(u0, u0, SQ_GUARD), q1 = fmaf(u1, u1, SQ_GUARD), q2 = fmaf(u2, u2, SQ_GUARD);
  float la0 = p2 * lg2(q0), la1 = p2 * lg2(q1), l3 = p1 * lg2(q2);
  // log-sum-exp in base 2; e = 2^-|difference| also gives both weights
  // (w_big = 1/(1+e), w_small = e/(1+e)) without two more exponentials
  const float eS = ex2(-fabsf(la0 - la1));
  float lS = fmaxf(la0, la1) + lg2(1.f + eS);
  float lB = m * lS;
  const float ef = ex2(-fabsf(lB - l3));
  float lf = fmaxf(lB, l3) + lg2(1.f + ef);
  float h = ex2(-k * lf);
  float rr = fmaf(y[0], y[0], fmaf(y[1], y[1], y[2] * y[2]));
  float ir = rsqrtf(fmaxf(rr, 1e-30f));
  float rad = rr * ir;
  float omh = 1.f - h;
  r.v = rad * omh;
  if constexpr (O >= 1) {
#if CM_SQ_SHARED_W
    const float rS = rcpa(1.f + eS), rf = rcpa(1.f + ef);
    const bool a0big = la0 >= la1, bbig = lB >= l3;
    float w0 = a0big ? rS : eS * rS, w1 = a0big ? eS * rS : rS;   // A_i / S
    float be = bbig ? rf : ef * rf, ga = bbig ? ef * rf : rf;      // B / f, C / f
    const float r01 = rcpa(q0 * q1);   // q >= 1e-12: the product stays normal
    float iq0 = q1 * r01, iq1 = q0 * r01, iq2 = rcpa(q2);
#else
    float w0 = ex2(la0 - lS), w1 = ex2(la1 - lS);
    float be = ex2(lB - lf), ga = ex2(l3 - lf);
    float iq0 = rcpa(q0), iq1 = rcpa(q1), iq2 = rcpa(q2);
#endif
    float s0 = u0 * ia0 * iq0, s1 = u1 * ia1 * iq1, s2 = u2 * ia2 * iq2;
    float tp1 = 2.f * p1;
    float L0 = tp1 * be * w0 * s0, L1 = tp1 * be * w1 * s1, L2 = tp1 * ga * s2;
    float yh0 = y[0] * ir, yh1 = y[1] * ir, yh2 = y[2] * ir;
    float kh = k * h, krh = kh * rad;
    r.g[0] = fmaf(omh, yh0, krh * L0);
    r.g[1] = fmaf(omh, yh1, krh * L1);
    r.g[2] = fmaf(omh, yh2, krh * L2);
    if constexpr (O >= 2) {
      float c0 = (1.f - 2.f * u0 * u0 * iq0) * ia0 * ia0 * iq0;
      float c1 = (1.f - 2.f * u1 * u1 * iq1) * ia1 * ia1 * iq1;
      float c2 = (1.f - 2.f * u2 * u2 * iq2) * ia2 * ia2 * iq2;
      float tb = tp1 * be, dp = 2.f * (p1 - p2);
      float ws0 = w0 * s0, ws1 = w1 * s1;
      float F00 = tb * fmaf(dp * ws0, ws0, w0 * fmaf(2.f * p2 * s0, s0, c0));
      float F01 = tb * dp * ws0 * ws1;
      float F11 = tb * fmaf(dp * ws1, ws1, w1 * fmaf(2.f * p2 * s1, s1, c1));
      float F22 = tp1 * ga * fmaf(tp1 * s2, s2, c2);
      float a1 = omh * ir;          // (1-h)/r
      float opk = 1.f + k;
      float yh[3] = {yh0, yh1, yh2}, Lv[3] = {L0, L1, L2};
      float F[6] = {F00, F01, 0.f, F11, 0.f, F22};
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j) {
          int q = hidx3(i, j);
          float v = a1 * ((i == j ? 1.f : 0.f) - yh[i] * yh[j]);
          v = fmaf(kh, fmaf(yh[i], Lv[j], Lv[i] * yh[j]), v);
          v = fmaf(krh, fmaf(-opk * Lv[i], Lv[j], F[q]), v);
          r.h[q] = v;
        }
    }
  }
}

// plane value n.y + h (gradient n, Hessian 0)
template <int O> __device__ __forceinline__ void plane_eval(const float* pl, const float* y, Res<O>& r) {
  r.v = fmaf(pl[0], y[0], fmaf(pl[1], y[1], fmaf(pl[2], y[2], pl[3])));
  if constexpr (O >= 1) {
    r.g[0] = pl[0]; r.g[1] = pl[1]; r.g[2] = pl[2];
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < 6; ++k) r.h[k] = 0.f;
  }
}

// ============================================================================
// Compact forward-mode jets for the XPSQ: Jet<NV, O> carries the value, NV
// first and NV(NV+1)/2 second partials (O = 0/1/2).
// ============================================================================
template <int NV, int O> struct Jet {
  static constexpr int NH = NV * (NV + 1) / 2;
  float v;
  float g[NV];
  float h[NH];
};
template <int NV> __device__ __forceinline__ constexpr int jhi(int k) {
  return NV == 3 ? (k < 3 ? 0 : (k < 5 ? 1 : 2)) : (k < 2 ? 0 : 1);
}
template <int NV> __device__ __forceinline__ constexpr int jhj(int k) {
  return NV == 3 ? (k < 3 ? k : (k < 5 ? k - 2 : 2)) : (k < 2 ? k : 1);
}

#define JT template <int NV, int O>
#define JJ Jet<NV, O>

JT __device__ __forceinline__ JJ jconst(float c) {
  JJ r;
  r.v = c;
#pragma unroll
  for (int i = 0; i < NV; ++i) r.g[i] = 0.f;
#pragma unroll
  for (int k = 0; k < JJ::NH; ++k) r.h[k] = 0.f;
  return r;
}
JT __device__ __forceinline__ JJ jvar(float c, int i) {
  JJ r = jconst<NV, O>(c);
  r.g[i] = 1.f;
  return r;
}
JT __device__ __forceinline__ JJ operator+(const JJ& a, const JJ& b) {
  JJ r;
  r.v = a.v + b.v;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = a.g[i] + b.g[i];
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) r.h[k] = a.h[k] + b.h[k];
  }
  return r;
}
JT __device__ __forceinline__ JJ operator-(const JJ& a, const JJ& b) {
  JJ r;
  r.v = a.v - b.v;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = a.g[i] - b.g[i];
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) r.h[k] = a.h[k] - b.h[k];
  }
  return r;
}
JT __device__ __forceinline__ JJ operator-(const JJ& a) {
  JJ r;
  r.v = -a.v;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = -a.g[i];
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) r.h[k] = -a.h[k];
  }
  return r;
}
JT __device__ __forceinline__ JJ operator*(const JJ& a, float s) {
  JJ r;
  r.v = a.v * s;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = a.g[i] * s;
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) r.h[k] = a.h[k] * s;
  }
  return r;
}
JT __device__ __forceinline__ JJ operator*(float s, const JJ& a) { return a * s; }
JT __device__ __forceinline__ JJ operator+(const JJ& a, float s) {
  JJ r = a;
  r.v = a.v + s;
  return r;
}
JT __device__ __forceinline__ JJ operator+(float s, const JJ& a) { return a + s; }
JT __device__ __forceinline__ JJ operator-(const JJ& a, float s) { return a + (-s); }
JT __device__ __forceinline__ JJ operator-(float s, const JJ& a) { return (-a) + s; }
JT __device__ __forceinline__ JJ operator*(const JJ& a, const JJ& b) {
  JJ r;
  r.v = a.v * b.v;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = fmaf(a.g[i], b.v, a.v * b.g[i]);
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) {
      const int i = jhi<NV>(k), j = jhj<NV>(k);
      r.h[k] = fmaf(a.h[k], b.v, fmaf(a.v, b.h[k], fmaf(a.g[i], b.g[j], a.g[j] * b.g[i])));
    }
  }
  return r;
}
// unary chain: value f, first derivative f1, second derivative f2
JT __device__ __forceinline__ JJ jchain(const JJ& a, float f, float f1, float f2) {
  JJ r;
  r.v = f;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = f1 * a.g[i];
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) {
      const int i = jhi<NV>(k), j = jhj<NV>(k);
      r.h[k] = fmaf(f1, a.h[k], f2 * a.g[i] * a.g[j]);
    }
  }
  return r;
}
// binary chain F(a, b)
JT __device__ __forceinline__ JJ jchain2(const JJ& a, const JJ& b, float f, float fa, float fb, float faa, float fab,
                                         float fbb) {
  JJ r;
  r.v = f;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < NV; ++i) r.g[i] = fmaf(fa, a.g[i], fb * b.g[i]);
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int k = 0; k < JJ::NH; ++k) {
      const int i = jhi<NV>(k), j = jhj<NV>(k);
      float v = fmaf(fa, a.h[k], fb * b.h[k]);
      v = fmaf(faa, a.g[i] * a.g[j], v);
      v = fmaf(fbb, b.g[i] * b.g[j], v);
      v = fmaf(fab, fmaf(a.g[i], b.g[j], a.g[j] * b.g[i]), v);
      r.h[k] = v;
    }
  }
  return r;
}
JT __device__ __forceinline__ JJ jinv(const JJ& a) {
  float f = 1.f / a.v;
  return jchain(a, f, -f * f, 2.f * f * f * f);
}
JT __device__ __forceinline__ JJ operator/(const JJ& a, const JJ& b) { return a * jinv(b); }
JT __device__ __forceinline__ JJ jex2(const JJ& a) {
  float f = ex2(a.v);
  return jchain(a, f, f * LN2, f * (LN2 * LN2));
}
JT __device__ __forceinline__ JJ jlg2(const JJ& a) {
  float iv = 1.f / a.v;
  return jchain(a, lg2(a.v), iv * (1.f / LN2), -iv * iv * (1.f / LN2));
}
JT __device__ __forceinline__ JJ jsqrt(const JJ& a) {
  float f = sqrtf(fmaxf(a.v, 0.f));
  float fg = fmaxf(f, 1e-20f);
  float f1 = 0.5f / fg;
  return jchain(a, f, f1, -f1 / (2.f * fg * fg));
}
JT __device__ __forceinline__ JJ jrsqrt(const JJ& a) {
  float f = rsqrtf(a.v);
  float f3 = f * f * f;
  return jchain(a, f, -0.5f * f3, 0.75f * f3 * f * f);
}
// real cube root (sign-preserving); derivatives guarded at 0 (the literal
// formula's cusp, reading #15; excluded from parity)
JT __device__ __forceinline__ JJ jcbrt(const JJ& a) {
  float f = cbrtf(a.v);
  float f2g = fmaxf(f * f, 1e-30f);
  float f1 = 1.f / (3.f * f2g);
  float f2 = -2.f * f1 / (3.f * (fabsf(a.v) > 1e-30f ? a.v : 1e-30f));
  return jchain(a, f, f1, f2);
}
JT __device__ __forceinline__ JJ jcos(const JJ& a) {
  float s, c;
  sincosf(a.v, &s, &c);
  return jchain(a, c, -s, -c);
}
JT __device__ __forceinline__ JJ jatan2(const JJ& y, const JJ& x) {
  float r2 = fmaf(x.v, x.v, y.v * y.v);
  float ir2 = 1.f / r2, ir4 = ir2 * ir2;
  return jchain2(y, x, atan2f(y.v, x.v), x.v * ir2, -y.v * ir2, -2.f * x.v * y.v * ir4,
                 (y.v * y.v - x.v * x.v) * ir4, 2.f * x.v * y.v * ir4);
}
// sigma(a) with derivatives s(1-s), s(1-s)(1-2s)
JT __device__ __forceinline__ JJ jsigm(const JJ& a) {
  float s = sigm(a.v);
  float d = s * (1.f - s);
  return jchain(a, s, d, d * (1.f - 2.f * s));
}
// s+(a; tau): derivative sigma(a/tau), second sigma(1-sigma)/tau
JT __device__ __forceinline__ JJ jsoftplus(const JJ& a, float tau, float itau) {
  float s = sigm(a.v * itau);
  return jchain(a, softplus(a.v, tau, itau), s, s * (1.f - s) * itau);
}
JT __device__ __forceinline__ JJ jsoftclip(const JJ& a, float lo, float hi, float tau, float itau) {
  float s1 = sigm((a.v - lo) * itau), s2 = sigm((a.v - hi) * itau);
  return jchain(a, softclip(a.v, lo, hi, tau, itau), s1 - s2, (s1 * (1.f - s1) - s2 * (1.f - s2)) * itau);
}
// log2(2^a + 2^b) = max + log2(1 + 2^-(|a-b|))
JT __device__ __forceinline__ JJ jlse2(const JJ& a, const JJ& b) {
  float d = a.v - b.v;
  float e = ex2(-fabsf(d));
  float f = fmaxf(a.v, b.v) + lg2(1.f + e);
  // weights wa = 2^a / (2^a + 2^b), wb = 1 - wa, each formed directly: the
  // small one multiplies huge derivatives of the other operand (e.g. an SQ
  // coordinate near its axis plane), so 1 - wa would cancel catastrophically
  const float ir = rcpa(1.f + e);
  const float wa = d > 0.f ? ir : e * ir;
  const float wb = d > 0.f ? e * ir : ir;
  float c = LN2 * wa * wb;
  return jchain2(a, b, f, wa, wb, c, -c, c);
}
#undef JT
#undef JJ

template <int O> using J3 = Jet<3, O>;
template <int O> using J2 = Jet<2, O>;

// scalar-or-jet helpers for schedule parameters (float when constant)
template <int O> __device__ __forceinline__ J3<O> lift(float x) { return jconst<3, O>(x); }

// SQ radial distance on jets (same log2-domain formulas as sq_eval);
// parameters are jets only when the XPSQ schedules vary along t.
template <int O, class S>
__device__ __forceinline__ J3<O> sq_jet(const J3<O>* y, const S& p1, const S& p2, const S& m, const S& k,
                                        const S* ia) {
  J3<O> u0 = y[0] * ia[0], u1 = y[1] * ia[1], u2 = y[2] * ia[2];
  J3<O> q0 = u0 * u0 + SQ_GUARD, q1 = u1 * u1 + SQ_GUARD, q2 = u2 * u2 + SQ_GUARD;
  J3<O> la0 = jlg2(q0) * p2, la1 = jlg2(q1) * p2, l3 = jlg2(q2) * p1;
  J3<O> lS = jlse2(la0, la1);
  J3<O> lB = lS * m;
  J3<O> lf = jlse2(lB, l3);
  J3<O> h = jex2(-(lf * k));
  J3<O> rad = jsqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
  return rad * (1.f - h);
}

// direct LSE_tau over n jets (n <= 9), sign s: s * LSE(s * x)
template <int O> __device__ __forceinline__ J3<O> lse_jets(const J3<O>* x, int n, float s, float tau) {
  float m = s * x[0].v;
  for (int i = 1; i < n; ++i) m = fmaxf(m, s * x[i].v);
  float itl = LOG2E / tau;
  J3<O> S = jconst<3, O>(0.f);
  for (int i = 0; i < n; ++i) S = S + jex2((x[i] * s - m) * itl);
  J3<O> L = jlg2(S) * (tau * LN2) + m;
  return L * s;
}

// soft Cardano (Eq. (6)) with implicit derivatives, defined below
template <int O>
__device__ __forceinline__ bool soft_cardano_implicit(float P, float Q, float b3, const SmoothDev& sp, J2<O>* t,
                                                      float* tb3 = nullptr);

// Roots t_k(w) of the projection with their gradient and Hessian
// with respect to w = y - p1 (packed xx, xy, xz, yy, yz, zz).  Returns true
// when the three roots are bitwise identical (point / straight splines, or
// the curved case in the one-real-root regime): then the three PSQ terms
// coincide and -LSE(-phi, -phi, -phi) = phi - tau ln 3 exactly, so one PSQ
// evaluation suffices.
//
// Curved splines outside the soft-Cardano band (|Delta| > 46 tau_Delta:
// the other branch's gate weight sigma(-|Delta|/tau) < 1e-20 is skipped,
// reading #34, and s+(Delta) < tau e^-46 leaves P and the discriminant
// unchanged in FP32) are the exact roots of the cubic g(t) = c3 t^3 + c2 t^2
// + c1 t + c0, c1 = 2 A.w - B.B, c0 = B.w.  There the Cardano / trigonometric
// value is polished by Newton steps on g in t (for nearly straight splines
// the depressed coefficients grow like (|B| / |A|)^2 and (|B| / |A|)^3, so
// the FP32 Cardano / trigonometric values and t = s - b/3 cancel digits)
// and differentiated implicitly: g_t dt + (B + 2 A t) dw = 0,
//   t_i = -(B_i + 2 A_i t) / g_t,
//   t_ij = -(g_tt t_i t_j + 2 A_i t_j + 2 A_j t_i) / g_t.
// Inside the band both branches are blended literally (soft_cardano_implicit).
template <int O>
__device__ __forceinline__ void xpsq_t_implicit(const Xpsq& X, const SmoothDev& sp, const float* w, float t,
                                                int newton, float* tv, float* tg, float* th) {
  const float c1 = fmaf(2.f * X.A[0], w[0], fmaf(2.f * X.A[1], w[1], fmaf(2.f * X.A[2], w[2], -X.BB)));
  const float c0 = fmaf(X.B[0], w[0], fmaf(X.B[1], w[1], X.B[2] * w[2]));
  // one Newton step always, a second for nearly straight splines (newton = 2)
  float g = fmaf(fmaf(fmaf(X.c3, t, X.c2), t, c1), t, c0);
  float r = rcpa(fmaf(fmaf(3.f * X.c3, t, 2.f * X.c2), t, c1));
  t = fmaf(-g, r, t);
  if (newton > 1) {
    g = fmaf(fmaf(fmaf(X.c3, t, X.c2), t, c1), t, c0);
    r = rcpa(fmaf(fmaf(3.f * X.c3, t, 2.f * X.c2), t, c1));
    t = fmaf(-g, r, t);
  }
  float v, d1, d2;
  softclip_12(t, 0.f, 1.f, sp.tau_clip_t, sp.i_clip_t, v, d1, d2);
  *tv = v;
  if constexpr (O >= 1) {
    float ti[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      ti[i] = -fmaf(2.f * X.A[i], t, X.B[i]) * r;
      tg[i] = d1 * ti[i];
    }
    if constexpr (O >= 2) {
      const float gtt = fmaf(6.f * X.c3, t, 2.f * X.c2);
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int i = jhi<3>(q), j = jhj<3>(q);
        const float tij = -fmaf(gtt * ti[i], ti[j], 2.f * fmaf(X.A[i], ti[j], X.A[j] * ti[i])) * r;
        th[q] = fmaf(d2 * ti[i], ti[j], d1 * tij);
      }
    }
  }
}

// The curved spline's rarer regimes (inline by default): three real roots
// (Delta > 46 tau_Delta) and the soft-Cardano band (both branches,
// P:113-124).  Returns true when the three roots are identical.
#ifndef CM_XPSQ_RARE_NOINLINE
#define CM_XPSQ_RARE_NOINLINE 0   // out of line: C5 -19% (its array arguments live in local memory), r02l
#endif
template <int O>
__device__
#if CM_XPSQ_RARE_NOINLINE
__noinline__
#else
__forceinline__
#endif
bool xpsq_root_t_rare(const Xpsq& X, const SmoothDev& sp, const float* w, float Pv, float Qv, float Delta, int newton,
                      float* tv, float (*tg)[3], float (*th)[6]) {
  if (CM_XPSQ_TSPACE && Delta * sp.i_delta > 46.f) {
    // three real roots: trigonometric form, k = 0, 1, 2
    const float rho = sqrtf(fmaxf(-Pv * (1.f / 3.f), 0.f));
    const float th3 = atan2_pos(sqrtf(Delta * (1.f / 108.f)), -0.5f * Qv) * (1.f / 3.f);
    float sn3, cs3;
    __sincosf(th3, &sn3, &cs3);
    const float ck[3] = {cs3, fmaf(-0.8660254037844386f, sn3, -0.5f * cs3),
                         fmaf(0.8660254037844386f, sn3, -0.5f * cs3)};
#pragma unroll 1
    for (int k = 0; k < 3; ++k) xpsq_t_implicit<O>(X, sp, w, 2.f * rho * ck[k] - X.b3, newton, &tv[k], tg[k], th[k]);
    return false;
  }
  constexpr int OC = O;
  J2<OC> t2[3];
  const bool single = soft_cardano_implicit<OC>(Pv, Qv, X.b3, sp, t2);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    tv[k] = t2[k].v;
    if constexpr (O >= 1) {
#pragma unroll
      for (int i = 0; i < 3; ++i) tg[k][i] = fmaf(t2[k].g[0], X.gP[i], t2[k].g[1] * X.gQ[i]);
    }
    if constexpr (O >= 2) {
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const int i = jhi<3>(q), j = jhj<3>(q);
        float v = t2[k].h[0] * X.gP[i] * X.gP[j];
        v = fmaf(t2[k].h[1], fmaf(X.gP[i], X.gQ[j], X.gQ[i] * X.gP[j]), v);
        th[k][q] = fmaf(t2[k].h[2], X.gQ[i] * X.gQ[j], v);
      }
    }
  }
  return single;
}

template <int O>
__device__ __forceinline__ bool xpsq_root_t(const Xpsq& X, const SmoothDev& sp, const float* w, float* tv, float (*tg)[3],
                                            float (*th)[6]) {
  // (when the three roots are identical only entry 0 is written)
  const float tc = sp.tau_clip_t, itc = sp.i_clip_t;
  if (X.cls == 1) {
    const float s = X.Bn[0] * w[0] + X.Bn[1] * w[1] + X.Bn[2] * w[2];
    float v, d1, d2;
    softclip_12(s, 0.f, 1.f, tc, itc, v, d1, d2);
    tv[0] = v;
#pragma unroll
    for (int i = 0; i < 3; ++i) tg[0][i] = d1 * X.Bn[i];
#pragma unroll
    for (int q = 0; q < 6; ++q) th[0][q] = d2 * X.Bn[jhi<3>(q)] * X.Bn[jhj<3>(q)];
    return true;
  }
  if (X.cls == 2) {
    const float Pv = X.gP[0] * w[0] + X.gP[1] * w[1] + X.gP[2] * w[2] + X.P0;
    const float Qv = X.gQ[0] * w[0] + X.gQ[1] * w[1] + X.gQ[2] * w[2] + X.Q0;
    const float Delta = -(4.f * Pv * Pv * Pv + 27.f * Qv * Qv);
    // Newton steps: one always (s = u - P/(3u) and 2 rho cos(.) cancel
    // digits when |P| is large, e.g. A nearly perpendicular to B with
    // |A| << |B|), two when t = s - b/3 cancels digits too (|b/3| > 4)
    const int newton = fabsf(X.b3) > 4.f ? 2 : 1;
    if (CM_XPSQ_TSPACE && Delta * sp.i_delta < -46.f) {
      // one real root: Cardano in its cancellation-free form
      const float sD = sqrtf(-Delta * (1.f / 108.f));
      const float u = cbrt_fast(Qv >= 0.f ? -0.5f * Qv - sD : -0.5f * Qv + sD);
      const float s = fabsf(u) > 1e-30f ? u - Pv * rcpa(3.f * u) : u;
      xpsq_t_implicit<O>(X, sp, w, s - X.b3, newton, &tv[0], tg[0], th[0]);
      return true;
    }
    return xpsq_root_t_rare<O>(X, sp, w, Pv, Qv, Delta, newton, tv, tg, th);
  }
  // point spline: t = 1/2, no derivatives
  tv[0] = 0.5f;
#pragma unroll
  for (int i = 0; i < 3; ++i) tg[0][i] = 0.f;
#pragma unroll
  for (int q = 0; q < 6; ++q) th[0][q] = 0.f;
  return true;
}

// XPSQ leaf in its local frame
template <int O> __device__ CM_XINL void xpsq_eval(const Xpsq& X, const SmoothDev& sp, const float* y, Res<O>& out) {
  float w[3] = {y[0] - X.p1[0], y[1] - X.p1[1], y[2] - X.p1[2]};
  J3<O> tk[3];
  {
    float tv[3], tg[3][3], th[3][6];
    if (xpsq_root_t<O>(X, sp, w, tv, tg, th)) {   // identical roots: entry 0 only
#pragma unroll
      for (int k = 1; k < 3; ++k) {
        tv[k] = tv[0];
#pragma unroll
        for (int i = 0; i < 3; ++i) tg[k][i] = tg[0][i];
#pragma unroll
        for (int q = 0; q < 6; ++q) th[k][q] = th[0][q];
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      tk[k].v = tv[k];
#pragma unroll
      for (int i = 0; i < 3; ++i) tk[k].g[i] = tg[k][i];
#pragma unroll
      for (int q = 0; q < 6; ++q) tk[k].h[q] = th[k][q];
    }
  }
  J3<O> yj[3] = {jvar<3, O>(y[0], 0), jvar<3, O>(y[1], 1), jvar<3, O>(y[2], 2)};
  J3<O> phis[3];
  const float tmin = sp.tau_min;
#pragma unroll 1
  for (int k = 0; k < 3; ++k) {
    const J3<O>& t = tk[k];
    J3<O> tt = t * t;
    J3<O> dx[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) dx[i] = yj[i] - (t * X.B[i] + tt * X.A[i] + X.p1[i]);
    J3<O> yk[3];
    if (X.frenet) {
      J3<O> pd[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) pd[i] = t * (2.f * X.A[i]) + X.B[i];
      J3<O> inv = jrsqrt(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
      J3<O> T[3] = {pd[0] * inv, pd[1] * inv, pd[2] * inv};
      const float* b = X.bhat;
      J3<O> N[3] = {T[2] * b[1] - T[1] * b[2], T[0] * b[2] - T[2] * b[0], T[1] * b[0] - T[0] * b[1]};
      yk[0] = T[0] * dx[0] + T[1] * dx[1] + T[2] * dx[2];
      yk[1] = N[0] * dx[0] + N[1] * dx[1] + N[2] * dx[2];
      yk[2] = dx[0] * b[0] + dx[1] * b[1] + dx[2] * b[2];
    } else {
      const float* R = X.R0;
#pragma unroll
      for (int i = 0; i < 3; ++i) yk[i] = dx[0] * R[0 * 3 + i] + dx[1] * R[1 * 3 + i] + dx[2] * R[2 * 3 + i];
    }
    J3<O> ops[1 + CM_MAX_PLANES];
    if (X.varying) {
      J3<O> e1 = t * X.deps[0] + X.eps0[0], e2 = t * X.deps[1] + X.eps0[1];
      J3<O> ip1 = jinv(e1), ip2 = jinv(e2);
      J3<O> m = e2 * ip1, kk = e1 * 0.5f;
      J3<O> ia[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) ia[i] = jinv(t * X.da[i] + X.a0[i]);
      ops[0] = sq_jet<O>(yk, ip1, ip2, m, kk, ia);
      for (int j = 0; j < X.n_planes; ++j) {
        J3<O> nv[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) nv[i] = t * X.dpl[j][i] + X.pl0[j][i];
        J3<O> in = jrsqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
        ops[1 + j] = (nv[0] * yk[0] + nv[1] * yk[1] + nv[2] * yk[2]) * in + (t * X.dpl[j][3] + X.pl0[j][3]);
      }
    } else {
      float e1 = X.eps0[0], e2 = X.eps0[1];
      float ia[3] = {1.f / X.a0[0], 1.f / X.a0[1], 1.f / X.a0[2]};
      ops[0] = sq_jet<O, float>(yk, 1.f / e1, 1.f / e2, e2 / e1, 0.5f * e1, ia);
      for (int j = 0; j < X.n_planes; ++j)
        ops[1 + j] = yk[0] * X.pl0[j][0] + yk[1] * X.pl0[j][1] + yk[2] * X.pl0[j][2] + X.pl0[j][3];
    }
    phis[k] = X.n_planes > 0 ? lse_jets<O>(ops, 1 + X.n_planes, 1.f, tmin) : ops[0];
  }
  // smooth minimum of the three PSQ SDFs
  J3<O> phi = lse_jets<O>(phis, 3, -1.f, tmin);
  out.v = phi.v;
  if constexpr (O >= 1) {
#pragma unroll
    for (int i = 0; i < 3; ++i) out.g[i] = phi.g[i];
  }
  if constexpr (O >= 2) {
#pragma unroll
    for (int q = 0; q < 6; ++q) out.h[q] = phi.h[q];
  }
}

// ---- XPSQ, analytic fast path (constant schedules) ---------------------------
// phi_k(x) = psi(y_k(x, t_k(x))) with y = R(t)^T (x - p(t));
// psi = PSQ at the root's pose, t_k from soft Cardano (2-variable jets
// in (P, Q), chained to x).  With G = grad_y psi, H = hess_y psi, y_t = dy/dt:
//   grad phi = R G + (G . y_t) grad t
//   hess phi = M^T H M + (R'G) grad t^T + grad t (R'G)^T
//              + (G . y_tt) grad t grad t^T + (G . y_t) hess t,
//   M_i = R_col_i + (y_t)_i grad t,
//   y_t  = (T'.d - T.p', N'.d - N.p', -b.p'),  d = x - p(t),
//   y_tt = (T''.d - 2T'.p' - T.p'', N''.d - 2N'.p' - N.p'', -b.p''),
// Frenet frame of the quadratic (constant binormal b):
//   T' = (p'' - T (T.p''))/|p'|,  T'' = (-2 T' (T.p'') - T (T'.p''))/|p'|,
//   N = b x T, N' = b x T', N'' = b x T''.
struct XsqParams {
  float ia[3];
  float p1, p2, m, k;
};

// Soft Cardano with implicit derivatives (same function as soft_cardano; far
// less code than the jets).  Each branch returns roots of a modified
// depressed cubic F(s) = s^3 + Pt s + Q = 0 whose discriminant is the
// projected one (reading #10):
//   negative:  Pt = cbrt(W),       W = P^3 + s+(Delta)/4            (one root)
//   positive:  Pt = -3 cbrt(V),    V = Q^2/4 + s+(Delta)/108        (three roots)
// so with a, b in {P, Q}:  s_a = -(Pt_a s + Q_a)/F_s,  F_s = 3 s^2 + Pt,
//   s_ab = -(6 s s_a s_b + Pt_b s_a + Pt_a s_b + Pt_ab s)/F_s.
// The values use the cancellation-free forms of soft_cardano.
template <int O>
__device__ __forceinline__ bool soft_cardano_implicit(float P, float Q, float b3, const SmoothDev& sp, J2<O>* t,
                                                      float* tb3) {
  const float td = sp.tau_delta, itd = sp.i_delta;
  const float tc = sp.tau_clip_t, itc = sp.i_clip_t;
  const float P2 = P * P, P3 = P2 * P;
  const float Delta = -(4.f * P3 + 27.f * Q * Q);
  const float Dl[2] = {-12.f * P2, -54.f * Q};          // dDelta/d(P, Q)
  const float Dll[3] = {-24.f * P, 0.f, -54.f};         // PP, PQ, QQ
  // one exponential e = exp(-|Delta|/tau) gives both gates sigma(+-Delta/tau),
  // s+'(Delta) = sigma(Delta/tau) and s+(+-Delta) = max(+-Delta, 0) + tau log(1+e)
  const float eD = ex2(-fabsf(Delta) * (itd * LOG2E));
  const float rD = rcpa(1.f + eD);
  const float wp = Delta >= 0.f ? rD : eD * rD, wn = Delta >= 0.f ? eD * rD : rD;
  // tau log(1 + e): log1p form below 1e-2 (1 + e rounds e away in FP32, and
  // the projected discriminants s+(+-Delta) below enter square / cube roots
  // whose derivatives need them to full relative precision)
  const float lgD = td * (eD < 1e-2f ? eD * fmaf(-eD, fmaf(-eD, 1.f / 3.f, 0.5f), 1.f) : LN2 * lg2(1.f + eD));
  // blend weights and their derivatives; sigma (1 - sigma) = wn wp and
  // 1 - 2 sigma = wn - wp with both weights formed directly (1 - wn rounds
  // the smaller weight away: 20% off at |Delta| = 17 tau in FP32)
  const float ww = wn * wp;
  const float sp1 = wp;                                 // s+'(Delta)
  const float sp2 = ww * itd;                           // s+''(Delta)
  const float spD = fmaxf(Delta, 0.f) + lgD;           // s+(Delta)
  const float dwn = -ww * itd, dwp = ww * itd;
  const float ddwn = ww * (wp - wn) * itd * itd;
  const float ddwp = ww * (wn - wp) * itd * itd;
  // derivatives of the modified coefficient and of the root
  auto root_derivs = [&](float s, float Pt, const float* Pa, const float* Pab, float* sa, float* sab) {
    const float Fs = fmaf(3.f * s, s, Pt);
    const float iF = rcpa(Fs);
    sa[0] = -(Pa[0] * s) * iF;
    sa[1] = -(fmaf(Pa[1], s, 1.f)) * iF;
    if constexpr (O >= 2) {
      sab[0] = -(6.f * s * sa[0] * sa[0] + 2.f * Pa[0] * sa[0] + Pab[0] * s) * iF;
      sab[1] = -(6.f * s * sa[0] * sa[1] + Pa[1] * sa[0] + Pa[0] * sa[1] + Pab[1] * s) * iF;
      sab[2] = -(6.f * s * sa[1] * sa[1] + 2.f * Pa[1] * sa[1] + Pab[2] * s) * iF;
    }
  };
  // soft clip of s - b/3 into (0, 1) with derivatives
  float clip_d1 = 0.f;   // the last clip's derivative (d t / d b3 = -wn c1- - wp c1+, optional output)
  auto clip = [&](float s, const float* sa, const float* sab, float& v, float* va, float* vab) {
    const float x = s - b3;
    float c1, c2;
    softclip_12(x, 0.f, 1.f, tc, itc, v, c1, c2);
    clip_d1 = c1;
    va[0] = c1 * sa[0];
    va[1] = c1 * sa[1];
    if constexpr (O >= 2) {
      vab[0] = fmaf(c2 * sa[0], sa[0], c1 * sab[0]);
      vab[1] = fmaf(c2 * sa[0], sa[1], c1 * sab[1]);
      vab[2] = fmaf(c2 * sa[1], sa[1], c1 * sab[2]);
    }
  };
  float tm = 0.f, tma[2] = {0.f, 0.f}, tmab[3] = {0.f, 0.f, 0.f};
  float tp[3] = {0.f, 0.f, 0.f}, tpa[3][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}}, tpab[3][3] = {};
  constexpr float W_SKIP = 1e-20f;   // negligible branches are skipped (reading #34)
  const bool use_n = wn > W_SKIP, use_p = wp > W_SKIP;
  if (use_n) {
    // W = P^3 + s+(Delta)/4; above Delta = 0 its two terms cancel (P^3 ~
    // -s+(Delta)/4 near the cusp, reading #15): there the identity s+(Delta)
    // = Delta + s+(-Delta), Delta = -(4 P^3 + 27 Q^2), gives the
    // cancellation-free W = (s+(-Delta) - 27 Q^2) / 4
    const float W = Delta > 0.f ? 0.25f * fmaf(-27.f * Q, Q, lgD) : fmaf(0.25f, spD, P3);
    const float Pm = cbrt_fast(W);
    // Cardano's cancellation-free form: u = cbrt(-Q/2 - sign(Q) sqrt(D)), v = -Pm/(3u)
    const float D = (fmaxf(-Delta, 0.f) + lgD) * (1.f / 108.f);   // s+(-Delta) / 108
    const float sD = sqrtf(D);
    const float u = cbrt_fast(Q >= 0.f ? -0.5f * Q - sD : -0.5f * Q + sD);
    const float s = fabsf(u) > 1e-30f ? u - Pm * rcpa(3.f * u) : u;
    float sa[2] = {0.f, 0.f}, sab[3] = {0.f, 0.f, 0.f};
    if constexpr (O >= 1) {
      // dW/dP = 3 P^2 (1 - s+') = 3 P^2 wn, dW/dQ = -13.5 Q wp (1 - wp
      // formed as wn: no cancellation where the negative branch is weak)
      const float Wa[2] = {3.f * P2 * wn, 0.25f * sp1 * Dl[1]};
      const float ip2 = rcpa(fmaxf(3.f * Pm * Pm, 1e-30f));   // guarded at the cusp (reading #15)
      const float Pa[2] = {Wa[0] * ip2, Wa[1] * ip2};
      float Pab[3] = {0.f, 0.f, 0.f};
      if constexpr (O >= 2) {
        const float Wab[3] = {fmaf(6.f * P, wn, 0.25f * sp2 * Dl[0] * Dl[0]),   // 6P + s+' Delta_PP/4 = 6 P wn
                              0.25f * sp2 * Dl[0] * Dl[1], 0.25f * fmaf(sp2 * Dl[1], Dl[1], sp1 * Dll[2])};
        const float den = 3.f * Pm * Pm * Pm;
        const float c = 2.f * ip2 * rcpa(fabsf(den) > 1e-30f ? den : copysignf(1e-30f, den));
        Pab[0] = fmaf(-c, Wa[0] * Wa[0], Wab[0] * ip2);
        Pab[1] = fmaf(-c, Wa[0] * Wa[1], Wab[1] * ip2);
        Pab[2] = fmaf(-c, Wa[1] * Wa[1], Wab[2] * ip2);
      }
      root_derivs(s, Pm, Pa, Pab, sa, sab);
    }
    clip(s, sa, sab, tm, tma, tmab);
    if (tb3) tb3[0] = tb3[1] = tb3[2] = -wn * clip_d1;
  }
  if (use_p) {
    // trigonometric form: with X = -Q/2, Y = sqrt(D), D = s+(Delta)/108,
    // z = X + iY = sqrt(V) e^(i th), V = X^2 + Y^2, the roots are
    // s_k = w_k + conj(w_k), w_k = z^(1/3) e^(2 pi i k/3) = rho e^(i phi_k).
    // Derivatives straight from the cube roots (no implicit 1/F'(s), which
    // is 0/0 when two roots nearly coincide at a small positive weight):
    //   ds_k = (2/3) Re(E_k dz),  E_k = w_k / z = V^(-1/3) e^(i(phi_k - th)),
    //   d2s_k = 2 Re((-2/9) F_k dz dz + (1/3) E_k d2z),  F_k = w_k / z^2,
    //   dX = -dQ/2, dY = s+'(Delta) dDelta / (216 Y),
    //   d2Y = (s+'' dDelta dDelta + s+' d2Delta) / (216 Y) - (s+' / Y)^2 dDelta dDelta / (46656 Y)
    const float D = spD * (1.f / 108.f);
    const float V = fmaf(0.25f * Q, Q, D);
    const float rho = ex2(lg2(V) * (1.f / 6.f));
    const float Y = sqrtf(D);
    const float th3 = atan2_pos(Y, -0.5f * Q) * (1.f / 3.f);
    float sn3, cs3;
    __sincosf(th3, &sn3, &cs3);
    const float ck1 = fmaf(-0.8660254037844386f, sn3, -0.5f * cs3), ck2 = fmaf(0.8660254037844386f, sn3, -0.5f * cs3);
    constexpr float C120 = -0.5f, S120 = 0.8660254037844386f;   // e^(2 pi i / 3)
    float Ya[2] = {0.f, 0.f}, Yab[3] = {0.f, 0.f, 0.f}, e_re = 0.f, e_im = 0.f, f_re = 0.f, f_im = 0.f;
    if constexpr (O >= 1) {
      const float iY = rsqrtf(fmaxf(D, 1e-37f));
      const float A1 = sp1 * iY;                               // s+'(Delta) / Y
      Ya[0] = A1 * Dl[0] * (1.f / 216.f);
      Ya[1] = A1 * Dl[1] * (1.f / 216.f);
      const float iV13 = rcpa(fmaxf(rho * rho, 1e-30f));      // V^(-1/3)
      float s2, c2;
      __sincosf(2.f * th3, &s2, &c2);                          // E_0 phase -2 th / 3
      e_re = iV13 * c2;
      e_im = -iV13 * s2;
      if constexpr (O >= 2) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int i = q == 2 ? 1 : 0, j = q == 0 ? 0 : 1;
          Yab[q] = fmaf(fmaf(sp2 * Dl[i], Dl[j], sp1 * Dll[q]), iY * (1.f / 216.f),
                        -A1 * A1 * iY * Dl[i] * Dl[j] * (1.f / 46656.f));
        }
        float s5, c5;
        __sincosf(5.f * th3, &s5, &c5);                        // F_0 phase -5 th / 3
        const float iV56 = iV13 * rsqrtf(fmaxf(V, 1e-30f));     // V^(-5/6)
        f_re = iV56 * c5;
        f_im = -iV56 * s5;
      }
    }
    const float Xa[2] = {0.f, -0.5f};
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      const float s = 2.f * rho * (k == 0 ? cs3 : (k == 1 ? ck1 : ck2));
      float sa[2] = {0.f, 0.f}, sab[3] = {0.f, 0.f, 0.f};
      if constexpr (O >= 1) {
#pragma unroll
        for (int i = 0; i < 2; ++i) sa[i] = (2.f / 3.f) * fmaf(e_re, Xa[i], -e_im * Ya[i]);
        if constexpr (O >= 2) {
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int i = q == 2 ? 1 : 0, j = q == 0 ? 0 : 1;
            const float zz_re = fmaf(Xa[i], Xa[j], -Ya[i] * Ya[j]), zz_im = fmaf(Xa[i], Ya[j], Ya[i] * Xa[j]);
            const float fz = fmaf(f_re, zz_re, -f_im * zz_im);
            sab[q] = 2.f * fmaf(-2.f / 9.f, fz, (-1.f / 3.f) * e_im * Yab[q]);
          }
        }
      }
      float v, va[2], vab[3];
      clip(s, sa, sab, v, va, vab);
      if (tb3) tb3[k] = (use_n ? tb3[k] : 0.f) - wp * clip_d1;
      tp[k] = v;
      tpa[k][0] = va[0]; tpa[k][1] = va[1];
      if constexpr (O >= 2) { tpab[k][0] = vab[0]; tpab[k][1] = vab[1]; tpab[k][2] = vab[2]; }
      // next root: E_k and F_k turn by e^(2 pi i / 3)
      const float er = e_re, fr = f_re;
      e_re = fmaf(er, C120, -e_im * S120);
      e_im = fmaf(er, S120, e_im * C120);
      f_re = fmaf(fr, C120, -f_im * S120);
      f_im = fmaf(fr, S120, f_im * C120);
    }
  }
  // blend t_k = wn t- + wp t+_k (product rule)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float a = use_n ? 1.f : 0.f, b = use_p ? 1.f : 0.f;
    t[k].v = a * wn * tm + b * wp * tp[k];
    if constexpr (O >= 1) {
#pragma unroll
      for (int i = 0; i < 2; ++i)
        t[k].g[i] = a * fmaf(dwn * Dl[i], tm, wn * tma[i]) + b * fmaf(dwp * Dl[i], tp[k], wp * tpa[k][i]);
    }
    if constexpr (O >= 2) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int i = q == 2 ? 1 : 0, j = q == 0 ? 0 : 1;
        const float wnab = fmaf(ddwn * Dl[i], Dl[j], dwn * Dll[q]);
        const float wpab = fmaf(ddwp * Dl[i], Dl[j], dwp * Dll[q]);
        const float hn = wnab * tm + dwn * Dl[i] * tma[j] + dwn * Dl[j] * tma[i] + wn * tmab[q];
        const float hp = wpab * tp[k] + dwp * Dl[i] * tpa[k][j] + dwp * Dl[j] * tpa[k][i] + wp * tpab[k][q];
        t[k].h[q] = a * hn + b * hp;
      }
    }
  }
  return !use_p;
}

template <int O>
__device__ __forceinline__ void xpsq_eval_fast_body(const Xpsq& X, const SmoothDev& sp, const float* y, Res<O>& out) {
  const float tau = sp.tau_min, itau = sp.i_min, itl = LOG2E * itau;
  const float w[3] = {y[0] - X.p1[0], y[1] - X.p1[1], y[2] - X.p1[2]};
  float tv[3], tg[3][3], th[3][6];
  const bool single = xpsq_root_t<O>(X, sp, w, tv, tg, th);
  XsqParams sq;
#pragma unroll
  for (int i = 0; i < 3; ++i) sq.ia[i] = X.sq_ia[i];
  sq.p1 = X.sq_p1;
  sq.p2 = X.sq_p2;
  sq.m = X.sq_m;
  sq.k = X.sq_k;
  const float* b = X.frenet ? X.bhat : nullptr;
  Acc<O> acc;
  acc_init(acc);
  const int n_roots = single ? 1 : 3;
#pragma unroll 1
  for (int k = 0; k < n_roots; ++k) {
    const float t = tv[k];
    float pd[3], d[3], T[3], N[3], bb[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      pd[i] = fmaf(2.f * X.A[i], t, X.B[i]);
      d[i] = y[i] - fmaf(fmaf(X.A[i], t, X.B[i]), t, X.p1[i]);
    }
    float Tp[3] = {0.f, 0.f, 0.f}, Np[3] = {0.f, 0.f, 0.f}, Tpp[3] = {0.f, 0.f, 0.f}, Npp[3] = {0.f, 0.f, 0.f};
    if (b) {
      const float in = rsqrtf(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
#pragma unroll
      for (int i = 0; i < 3; ++i) { T[i] = pd[i] * in; bb[i] = b[i]; }
      N[0] = bb[1] * T[2] - bb[2] * T[1]; N[1] = bb[2] * T[0] - bb[0] * T[2]; N[2] = bb[0] * T[1] - bb[1] * T[0];
      if constexpr (O >= 1) {
        const float pdd[3] = {2.f * X.A[0], 2.f * X.A[1], 2.f * X.A[2]};
        const float tp = T[0] * pdd[0] + T[1] * pdd[1] + T[2] * pdd[2];
#pragma unroll
        for (int i = 0; i < 3; ++i) Tp[i] = (pdd[i] - T[i] * tp) * in;
        Np[0] = bb[1] * Tp[2] - bb[2] * Tp[1]; Np[1] = bb[2] * Tp[0] - bb[0] * Tp[2]; Np[2] = bb[0] * Tp[1] - bb[1] * Tp[0];
        if constexpr (O >= 2) {
          const float tpp = Tp[0] * pdd[0] + Tp[1] * pdd[1] + Tp[2] * pdd[2];
#pragma unroll
          for (int i = 0; i < 3; ++i) Tpp[i] = (-2.f * Tp[i] * tp - T[i] * tpp) * in;
          Npp[0] = bb[1] * Tpp[2] - bb[2] * Tpp[1]; Npp[1] = bb[2] * Tpp[0] - bb[0] * Tpp[2];
          Npp[2] = bb[0] * Tpp[1] - bb[1] * Tpp[0];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i) { T[i] = X.R0[i * 3 + 0]; N[i] = X.R0[i * 3 + 1]; bb[i] = X.R0[i * 3 + 2]; }
    }
    const float yk[3] = {T[0] * d[0] + T[1] * d[1] + T[2] * d[2], N[0] * d[0] + N[1] * d[1] + N[2] * d[2],
                         bb[0] * d[0] + bb[1] * d[1] + bb[2] * d[2]};
    // PSQ at the root: SQ intersected with the cross-section planes
    Res<O> r;
    sq_eval<O>(sq, yk, r);
    if (X.n_planes > 0) {
      Acc<O> a;
      acc_init(a);
      acc_fold(a, 1.f, r, itl, itau);
      for (int j = 0; j < X.n_planes; ++j) {
        Res<O> pr;
        plane_eval<O>(X.pl0[j], yk, pr);
        acc_fold(a, 1.f, pr, itl, itau);
      }
      acc_final(a, 1.f, tau, itau, r);
    }
    Res<O> rk;
    rk.v = r.v;
    if constexpr (O >= 1) {
      const float* G = r.g;
      // y_t, s = G . y_t
      const float yt[3] = {(Tp[0] * d[0] + Tp[1] * d[1] + Tp[2] * d[2]) - (T[0] * pd[0] + T[1] * pd[1] + T[2] * pd[2]),
                           (Np[0] * d[0] + Np[1] * d[1] + Np[2] * d[2]) - (N[0] * pd[0] + N[1] * pd[1] + N[2] * pd[2]),
                           -(bb[0] * pd[0] + bb[1] * pd[1] + bb[2] * pd[2])};
      const float s = G[0] * yt[0] + G[1] * yt[1] + G[2] * yt[2];
#pragma unroll
      for (int a = 0; a < 3; ++a) rk.g[a] = fmaf(s, tg[k][a], T[a] * G[0] + N[a] * G[1] + bb[a] * G[2]);
      if constexpr (O >= 2) {
        const float pdd[3] = {2.f * X.A[0], 2.f * X.A[1], 2.f * X.A[2]};
        const float ytt[3] = {(Tpp[0] * d[0] + Tpp[1] * d[1] + Tpp[2] * d[2]) -
                                  2.f * (Tp[0] * pd[0] + Tp[1] * pd[1] + Tp[2] * pd[2]) -
                                  (T[0] * pdd[0] + T[1] * pdd[1] + T[2] * pdd[2]),
                              (Npp[0] * d[0] + Npp[1] * d[1] + Npp[2] * d[2]) -
                                  2.f * (Np[0] * pd[0] + Np[1] * pd[1] + Np[2] * pd[2]) -
                                  (N[0] * pdd[0] + N[1] * pdd[1] + N[2] * pdd[2]),
                              -(bb[0] * pdd[0] + bb[1] * pdd[1] + bb[2] * pdd[2])};
        const float sg = G[0] * ytt[0] + G[1] * ytt[1] + G[2] * ytt[2];
        float RpG[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) RpG[a] = Tp[a] * G[0] + Np[a] * G[1];
        // M_i = col_i + yt_i grad t
        float M[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          M[0][a] = fmaf(yt[0], tg[k][a], T[a]);
          M[1][a] = fmaf(yt[1], tg[k][a], N[a]);
          M[2][a] = fmaf(yt[2], tg[k][a], bb[a]);
        }
        const float Hm[3][3] = {{r.h[0], r.h[1], r.h[2]}, {r.h[1], r.h[3], r.h[4]}, {r.h[2], r.h[4], r.h[5]}};
        float HM[3][3];   // HM[i][b] = sum_j H_ij M_j,b
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int c = 0; c < 3; ++c) HM[i][c] = Hm[i][0] * M[0][c] + Hm[i][1] * M[1][c] + Hm[i][2] * M[2][c];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const int a = jhi<3>(q), c = jhj<3>(q);
          float v = M[0][a] * HM[0][c] + M[1][a] * HM[1][c] + M[2][a] * HM[2][c];
          v = fmaf(RpG[a], tg[k][c], fmaf(RpG[c], tg[k][a], v));
          v = fmaf(sg * tg[k][a], tg[k][c], v);
          rk.h[q] = fmaf(s, th[k][q], v);
        }
      }
    }
    if (single) {   // three identical terms: -LSE(-phi x 3) = phi - tau ln 3
      out = rk;
      out.v = fmaf(-tau, 1.0986122886681098f, rk.v);
      return;
    }
    acc_fold(acc, -1.f, rk, itl, itau);   // smooth minimum over the roots
  }
  acc_final(acc, -1.f, tau, itau, out);
}
// out-of-line instance, used above CM_XPSQ_INLINE_MAX_O
template <int O> __device__ CM_XINL void xpsq_eval_fast(const Xpsq& X, const SmoothDev& sp, const float* y, Res<O>& out) {
  xpsq_eval_fast_body<O>(X, sp, y, out);
}

// ---- leaf dispatch ---------------------------------------------------------
// XP: 0 no XPSQ leaves, 1 constant-schedule XPSQ (analytic fast path),
// 2 any XPSQ (jets when the schedules vary along t); XINL: constant-schedule
// XPSQ inlined up to order CM_XPSQ_INLINE_MAX_O (manifold kernels) or always
// out of line (sdf_eval: one kernel for all leaf kinds, measured faster so)
// a leaf's frame, kind and SQ constants in registers: six 128-bit loads
// (cm_internal.h Leaf layout)
struct LeafRegs {
  float R[9], t[3];
  int kind, n_planes, rot_identity, xidx;
  float ia[3], p1, p2, m, k;
};
#ifndef CM_LEAF_VEC
#define CM_LEAF_VEC 0   // explicit __ldg 128-bit leaf loads: SDF +1.3%, manifold C5 -1.5% / C4 -2.5% against the
                        // compiler's own merging of the aligned fields (r02z4); cm_kernels_sdf.cu sets it
#endif
__device__ __forceinline__ void ld_leaf(const Leaf* lp, LeafRegs& o) {
#if CM_LEAF_VEC
  const float4* q = reinterpret_cast<const float4*>(lp);
  const float4 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  const int4 d = __ldg(reinterpret_cast<const int4*>(q + 3));
  const float4 e = __ldg(q + 4), f = __ldg(q + 5);
  o.R[0] = a.x; o.R[1] = a.y; o.R[2] = a.z; o.R[3] = a.w;
  o.R[4] = b.x; o.R[5] = b.y; o.R[6] = b.z; o.R[7] = b.w;
  o.R[8] = c.x; o.t[0] = c.y; o.t[1] = c.z; o.t[2] = c.w;
  o.kind = d.x; o.n_planes = d.y; o.rot_identity = d.z; o.xidx = d.w;
  o.ia[0] = e.x; o.ia[1] = e.y; o.ia[2] = e.z; o.p1 = e.w;
  o.p2 = f.x; o.m = f.y; o.k = f.z;
#else
  const Leaf& L = *lp;
#pragma unroll
  for (int i = 0; i < 9; ++i) o.R[i] = L.R[i];
  o.t[0] = L.t[0]; o.t[1] = L.t[1]; o.t[2] = L.t[2];
  o.kind = L.kind; o.n_planes = L.n_planes; o.rot_identity = L.rot_identity; o.xidx = L.xidx;
  o.ia[0] = L.ia[0]; o.ia[1] = L.ia[1]; o.ia[2] = L.ia[2];
  o.p1 = L.p1; o.p2 = L.p2; o.m = L.m; o.k = L.k;
#endif
}
__device__ __forceinline__ void ld_plane(const float* pl, float* o) {
#if CM_LEAF_VEC
  const float4 v = __ldg(reinterpret_cast<const float4*>(pl));
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
#else
  o[0] = pl[0]; o[1] = pl[1]; o[2] = pl[2]; o[3] = pl[3];
#endif
}

template <int O, int XP, bool XINL = true>
__device__ __forceinline__ void leaf_eval(const SceneDev& S, int li, const float* x, Res<O>& r) {
  LeafRegs L;
  ld_leaf(S.leaves + li, L);
  const float* lplanes = &S.leaves[li].planes[0][0];
  float y[3];
  const float* t = L.t;
  const bool ident = L.rot_identity != 0;
  const float* R = L.R;
  if (ident) {
    y[0] = x[0] - t[0]; y[1] = x[1] - t[1]; y[2] = x[2] - t[2];
  } else {
    to_local(R, t, x, y);
  }
  Res<O> l;
  const int kind = L.kind;
  if (kind == LK_SQ) {
    sq_eval<O>(L, y, l);
    const int np = L.n_planes;
    if (np > 0) {
      // PSQ: smooth intersection Eq. (3) with the half-spaces
      const float tau = S.sp.tau_min, itau = S.sp.i_min, itl = LOG2E * itau;
      Acc<O> a;
      acc_init(a);
      acc_fold(a, 1.f, l, itl, itau);
      for (int j = 0; j < np; ++j) {
        Res<O> p;
        float pl[4];
        ld_plane(lplanes + 4 * j, pl);
        plane_eval<O>(pl, y, p);
        acc_fold(a, 1.f, p, itl, itau);
      }
      acc_final(a, 1.f, tau, itau, l);
    }
  } else if (XP > 0 && kind == LK_XPSQ) {
    const Xpsq& X = S.xpsq[L.xidx];
    if constexpr (XP == 2) {
      if (X.varying) xpsq_eval<O>(X, S.sp, y, l);   // schedules vary along t: jets
      else xpsq_eval_fast<O>(X, S.sp, y, l);
    } else if constexpr (XINL && O <= CM_XPSQ_INLINE_MAX_O) {
      xpsq_eval_fast_body<O>(X, S.sp, y, l);
    } else {
      xpsq_eval_fast<O>(X, S.sp, y, l);
    }
  } else {
    float pl[4];
    ld_plane(lplanes, pl);
    plane_eval<O>(pl, y, l);
  }
  r.v = l.v;
  if constexpr (O >= 1) {
    if (ident) {
#pragma unroll
      for (int i = 0; i < 3; ++i) r.g[i] = l.g[i];
    } else {
      rot_vec(R, l.g, r.g);
    }
  }
  if constexpr (O >= 2) {
    if (ident) {
#pragma unroll
      for (int k = 0; k < 6; ++k) r.h[k] = l.h[k];
    } else {
      rot_sym(R, l.h, r.h);
    }
  }
}

// ---- shape program interpreter ----------------------------------------------
template <int O>
__device__ __forceinline__ void fold_level(Acc<O>& a0, Acc<O>& a1, Acc<O>& a2, int lvl, float s, const Res<O>& r,
                                           float itl, float itau) {
  if (lvl == 0) acc_fold(a0, s, r, itl, itau);
  else if (lvl == 1) acc_fold(a1, s, r, itl, itau);
  else acc_fold(a2, s, r, itl, itau);
}

// phi, grad, hess of shape `sh` at the body-frame point x
// FLAT: every boolean node of the shape sits at the root (nesting depth <= 1),
// so one accumulator level suffices (fewer live registers)
template <int O, int XP, bool FLAT, bool XINL, bool CULL>
__device__ __forceinline__ void eval_prog(const SceneDev& S, const ShapeRec& sh, const float* x, Res<O>& out);

// SINGLE: the shape is one leaf (no program loop compiled); CULL: XPSQ union
// operands with provably negligible weight are skipped (class-4 shapes only:
// the check costs the other XPSQ kernels registers)
template <int O, int XP, bool FLAT = false, bool XINL = true, bool CULL = false, bool SINGLE = false>
__device__ CM_SINL void eval_shape(const SceneDev& S, const ShapeRec& sh, const float* x, Res<O>& out) {
  if (SINGLE || sh.prog_len == 1) {  // single leaf: no accumulator needed
    leaf_eval<O, XP, XINL>(S, S.prog[sh.prog_begin].idx, x, out);
    return;
  }
  if constexpr (!SINGLE) eval_prog<O, XP, FLAT, XINL, CULL>(S, sh, x, out);
}

template <int O, int XP, bool FLAT, bool XINL, bool CULL>
__device__ __forceinline__ void eval_prog(const SceneDev& S, const ShapeRec& sh, const float* x, Res<O>& out) {
  const float tau = S.sp.tau_min, itau = S.sp.i_min, itl = LOG2E * itau;
  Acc<O> a0, a1, a2;
  int lvl = -1;
  const Instr* prog = S.prog + sh.prog_begin;
  for (int pc = 0; pc < sh.prog_len; ++pc) {
    const Instr in = prog[pc];
    if (in.op == OP_BEGIN) {
      ++lvl;
      if (FLAT || lvl == 0) acc_init(a0);
      else if (lvl == 1) acc_init(a1);
      else acc_init(a2);
      continue;
    }
    Res<O> r;
    if (in.op == OP_LEAF) {
      if constexpr (CULL && XP > 0 && CM_XPSQ_CULL) {
        // an XPSQ operand of a union whose weight is provably below 2^-66
        // against the operands folded so far adds nothing representable to
        // the value or its derivatives: skipped (Leaf::cull bound)
        if (in.child_sign < 0.f) {
          const float m = (FLAT || lvl == 0) ? a0.m : (lvl == 1 ? a1.m : a2.m);
          const Leaf& Lc = S.leaves[in.idx];
          if (m > -INFINITY && Lc.kind == LK_XPSQ) {
            const float dx = x[0] - Lc.cull[0], dy = x[1] - Lc.cull[1], dz = x[2] - Lc.cull[2];
            const float lb = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) - Lc.cull[3];
            if ((-lb - m) * itl < -66.f) continue;
          }
        }
      }
      leaf_eval<O, XP, XINL>(S, in.idx, x, r);
    } else {
      if (FLAT || lvl == 0) acc_final(a0, in.out_sign, tau, itau, r);
      else if (lvl == 1) acc_final(a1, in.out_sign, tau, itau, r);
      else acc_final(a2, in.out_sign, tau, itau, r);
      --lvl;
    }
    if (lvl < 0) out = r;
    else if (FLAT) acc_fold(a0, in.child_sign, r, itl, itau);
    else fold_level(a0, a1, a2, lvl, in.child_sign, r, itl, itau);
  }
}

}  // namespace cmd
