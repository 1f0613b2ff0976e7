// Shape-parameter derivatives of the SDF: d phi / d
// (a, eps, planes, XPSQ control points) of every leaf kind and the chain
// through boolean trees.  Shared by sdf_param_grad (cm_kernels_sdf.cu) and
// the manifold's parameter VJP (cm_kernels_manifold.cu).
#pragma once
#include "cm_device.cuh"
#include "cm_internal.h"

namespace cmd {
using namespace cmi;

// ============================================================================
// shape-parameter derivatives
// ============================================================================

// d phi / d (a_x, a_y, a_z, eps1, eps2) of the SQ radial distance, from the
// same log2-domain quantities as sq_eval (cm_device.cuh): with
// lf = log2 f, h = 2^(-k lf), phi = r (1 - h):
//   d phi = r h ln2 d(k lf),  d lf = beta d lB + gamma d l3,  lB = m lS,
//   d lS = w0 d la0 + w1 d la1,  d la_i / d a_i = p2 d log2 q_i / d a_i,
//   d log2 q_i / d a_i = -2 u_i^2 / (a_i q_i ln2)
//   eps1: d lB = -p1 lB, d l3 = -p1 l3, d k = 1/2;  eps2: d la_i = -p2 la_i,
//   d lB = p1 lS + m d lS
__device__ __forceinline__ float sq_param_grad_p(const float* ia, float p1, float p2, float m, float k,
                                                 const float* y, float* o) {
  const float ia0 = ia[0], ia1 = ia[1], ia2 = ia[2];
  const float u0 = y[0] * ia0, u1 = y[1] * ia1, u2 = y[2] * ia2;
  const float q0 = fmaf(u0, u0, SQ_GUARD), q1 = fmaf(u1, u1, SQ_GUARD), q2 = fmaf(u2, u2, SQ_GUARD);
  const float lq0 = lg2(q0), lq1 = lg2(q1), lq2 = lg2(q2);
  const float la0 = p2 * lq0, la1 = p2 * lq1, l3 = p1 * lq2;
  const float lS = fmaxf(la0, la1) + lg2(1.f + ex2(-fabsf(la0 - la1)));
  const float lB = m * lS;
  const float lf = fmaxf(lB, l3) + lg2(1.f + ex2(-fabsf(lB - l3)));
  const float h = ex2(-k * lf);
  const float rr = fmaf(y[0], y[0], fmaf(y[1], y[1], y[2] * y[2]));
  const float rad = rr * rsqrtf(fmaxf(rr, 1e-30f));
  const float w0 = ex2(la0 - lS), w1 = ex2(la1 - lS), be = ex2(lB - lf), ga = ex2(l3 - lf);
  const float c = rad * h * LN2;   // d phi = c d(k lf)
  const float dq0 = -2.f * u0 * u0 * ia0 * rcpa(q0) * LOG2E;   // d log2 q_i / d a_i (a_i = 1/ia_i)
  const float dq1 = -2.f * u1 * u1 * ia1 * rcpa(q1) * LOG2E;
  const float dq2 = -2.f * u2 * u2 * ia2 * rcpa(q2) * LOG2E;
  o[0] = c * k * be * m * w0 * p2 * dq0;
  o[1] = c * k * be * m * w1 * p2 * dq1;
  o[2] = c * k * ga * p1 * dq2;
  o[3] = c * fmaf(0.5f, lf, -k * p1 * (be * lB + ga * l3));
  const float dlS2 = -p2 * (w0 * la0 + w1 * la1);
  o[4] = c * k * be * fmaf(m, dlS2, p1 * lS);
  return rad * (1.f - h);
}
__device__ __forceinline__ float sq_param_grad(const Leaf& L, const float* y, float* o) {
  return sq_param_grad_p(L.ia, L.p1, L.p2, L.m, L.k, y, o);
}

// XPSQ cross-section parameters (f4): at each projection root t_k (which does
// not depend on a, eps or the planes) the PSQ of the root's local point y_k;
// phi = -tau LSE(-phi_k / tau) over the roots (one root when they coincide),
// so d phi = sum_k u_k d PSQ_k, u = softmax(-phi / tau).  Constant
// schedules: one slot per cross-section parameter.  Varying schedules
// (linear in t, reading #8): the cross-section at t_k is (1 - t_k) theta_0 +
// t_k theta_1, so slot s (the t = 0 value) takes (1 - t_k) and slot M + s
// (the t = 1 value) takes t_k of root k's derivative, M = 5 + 4 n_planes.
// Plane normals are renormalised in the XPSQ: n = v / |v| gives
// d/dv = (I - n n^T) y_k w_j / |v| (|v| = 1 for the constant schedule's
// unit normal)
// ---- XPSQ control points (f4): d t_k / d(A, B, w) of the
// projection roots.  Outside the soft-Cardano band the roots are exact roots
// of g(t) = (w - B t - A t^2).(B + 2 A t) (reading #43):
//   dt_raw = -(g_A dA + g_B dB + g_w dw) / g_t,  g_A = 2t (w - p) - t^2 p',
//   g_B = (w - p) - t p',  g_w = p',  g_t = 2 A.(w - p) - |p'|^2,
// then the soft clip's derivative; inside the band the literal blend through
// (P, Q, b): P = c1/c3 - b^2/3, Q = 2b^3/27 - b c1/(3 c3) + c0/c3, b = c2/c3
// with c3 = -2 A.A, c2 = -3 A.B, c1 = 2 A.w - B.B, c0 = B.w.  Straight
// splines: t = softclip(B.w / B.B) with B the chord; points: t = 1/2.
__device__ __forceinline__ void xpsq_root_dtheta(const Xpsq& X, const SmoothDev& sp, const float* w,
                                                 float (*dtA)[3], float (*dtB)[3], float (*dtw)[3]) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int m = 0; m < 3; ++m) dtA[k][m] = dtB[k][m] = dtw[k][m] = 0.f;
  if (X.cls == 0) return;
  if (X.cls == 1) {
    const float BB = X.B[0] * X.B[0] + X.B[1] * X.B[1] + X.B[2] * X.B[2];
    const float iBB = 1.f / BB;
    const float sv = (X.B[0] * w[0] + X.B[1] * w[1] + X.B[2] * w[2]) * iBB;
    float v, d1, d2;
    softclip_12(sv, 0.f, 1.f, sp.tau_clip_t, sp.i_clip_t, v, d1, d2);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        dtw[k][m] = d1 * X.B[m] * iBB;
        dtB[k][m] = d1 * (w[m] - 2.f * sv * X.B[m]) * iBB;
      }
    return;
  }
  const float Pv = X.gP[0] * w[0] + X.gP[1] * w[1] + X.gP[2] * w[2] + X.P0;
  const float Qv = X.gQ[0] * w[0] + X.gQ[1] * w[1] + X.gQ[2] * w[2] + X.Q0;
  const float Delta = -(4.f * Pv * Pv * Pv + 27.f * Qv * Qv);
  const int newton = fabsf(X.b3) > 4.f ? 2 : 1;
  const float c1 = fmaf(2.f * X.A[0], w[0], fmaf(2.f * X.A[1], w[1], fmaf(2.f * X.A[2], w[2], -X.BB)));
  const float c0 = fmaf(X.B[0], w[0], fmaf(X.B[1], w[1], X.B[2] * w[2]));
  // the exact-root regimes: implicit derivative of g at the polished root
  auto implicit = [&](float t, int k) {
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
    float pd[3], dm[3];
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      pd[m] = fmaf(2.f * X.A[m], t, X.B[m]);
      dm[m] = w[m] - fmaf(fmaf(X.A[m], t, X.B[m]), t, 0.f);
    }
    const float gt = 2.f * (X.A[0] * dm[0] + X.A[1] * dm[1] + X.A[2] * dm[2]) -
                     (pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
    const float c = -d1 / gt;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      dtA[k][m] = c * fmaf(2.f * t, dm[m], -t * t * pd[m]);
      dtB[k][m] = c * fmaf(-t, pd[m], dm[m]);
      dtw[k][m] = c * pd[m];
    }
  };
  if (Delta * sp.i_delta < -46.f) {   // one real root
    const float sD = sqrtf(-Delta * (1.f / 108.f));
    const float u = cbrt_fast(Qv >= 0.f ? -0.5f * Qv - sD : -0.5f * Qv + sD);
    const float sr = fabsf(u) > 1e-30f ? u - Pv * rcpa(3.f * u) : u;
    implicit(sr - X.b3, 0);
    return;
  }
  if (Delta * sp.i_delta > 46.f) {    // three real roots
    const float rho = sqrtf(fmaxf(-Pv * (1.f / 3.f), 0.f));
    const float th3 = atan2_pos(sqrtf(Delta * (1.f / 108.f)), -0.5f * Qv) * (1.f / 3.f);
    float sn3, cs3;
    __sincosf(th3, &sn3, &cs3);
    const float ck[3] = {cs3, fmaf(-0.8660254037844386f, sn3, -0.5f * cs3),
                         fmaf(0.8660254037844386f, sn3, -0.5f * cs3)};
#pragma unroll 1
    for (int k = 0; k < 3; ++k) implicit(2.f * rho * ck[k] - X.b3, k);
    return;
  }
  // the band: the literal blend through (P, Q, b)
  J2<1> t2[3];
  float tb3[3] = {0.f, 0.f, 0.f};
  soft_cardano_implicit<1>(Pv, Qv, X.b3, sp, t2, tb3);
  const float b = 3.f * X.b3, ic3 = 1.f / X.c3;
  const float cc = c1 * ic3, dd = c0 * ic3;
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int which = 0; which < 3; ++which) {   // A_m, B_m, w_m
      const float dc3 = which == 0 ? -4.f * X.A[m] : 0.f;
      const float dc2 = which == 0 ? -3.f * X.B[m] : (which == 1 ? -3.f * X.A[m] : 0.f);
      const float dc1 = which == 0 ? 2.f * w[m] : (which == 1 ? -2.f * X.B[m] : 2.f * X.A[m]);
      const float dc0 = which == 0 ? 0.f : (which == 1 ? w[m] : X.B[m]);
      const float db = (dc2 - b * dc3) * ic3;
      const float dcc = (dc1 - cc * dc3) * ic3;
      const float ddd = (dc0 - dd * dc3) * ic3;
      const float dP = fmaf(-(2.f / 3.f) * b, db, dcc);
      const float dQ = fmaf((2.f / 9.f) * b * b - cc * (1.f / 3.f), db, fmaf(-b * (1.f / 3.f), dcc, ddd));
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float v = fmaf(t2[k].g[0], dP, fmaf(t2[k].g[1], dQ, tb3[k] * db * (1.f / 3.f)));
        if (which == 0) dtA[k][m] = v;
        else if (which == 1) dtB[k][m] = v;
        else dtw[k][m] = v;
      }
    }
}

// d y / d(A, B, w) of the cross-section coordinates y = R(t)^T d at a fixed
// t (d = w - B t - A t^2; the frame R = [T, b x T, b]: the Frenet frame of
// p' = B + 2 A t with b = B x A / |B x A|, or the constant frame from T0 =
// (A + B) / |A + B| (B / |B| for straight splines) and the up hint by
// Gram-Schmidt), and y_t = d y / d t; out [3 (A, B, w)][3 m][3 y]
__device__ __forceinline__ void xpsq_dy_dtheta(const Xpsq& X, float t, const float* d, const float* T, const float* N,
                                               const float* bb, float (*out)[3][3], float* yt) {
  float pd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) pd[i] = fmaf(2.f * X.A[i], t, X.B[i]);
  // frame derivatives dT[which][m][i], db[which][m][i] (N = b x T)
  float dT[3][3][3] = {}, dbv[3][3][3] = {};
  if (X.cls == 2 && X.frenet) {
    const float ip = rsqrtf(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
    const float bxa[3] = {X.B[1] * X.A[2] - X.B[2] * X.A[1], X.B[2] * X.A[0] - X.B[0] * X.A[2],
                          X.B[0] * X.A[1] - X.B[1] * X.A[0]};
    const float ib = rsqrtf(bxa[0] * bxa[0] + bxa[1] * bxa[1] + bxa[2] * bxa[2]);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      // dp'/dA_m = 2t e_m, dp'/dB_m = e_m;  d(BxA)/dA_m = B x e_m, d(BxA)/dB_m = e_m x A
      const float e[3] = {m == 0 ? 1.f : 0.f, m == 1 ? 1.f : 0.f, m == 2 ? 1.f : 0.f};
      const float cA[3] = {X.B[1] * e[2] - X.B[2] * e[1], X.B[2] * e[0] - X.B[0] * e[2], X.B[0] * e[1] - X.B[1] * e[0]};
      const float cB[3] = {e[1] * X.A[2] - e[2] * X.A[1], e[2] * X.A[0] - e[0] * X.A[2], e[0] * X.A[1] - e[1] * X.A[0]};
      const float Tm = T[m];
      const float bA = bb[0] * cA[0] + bb[1] * cA[1] + bb[2] * cA[2];
      const float bB = bb[0] * cB[0] + bb[1] * cB[1] + bb[2] * cB[2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float proj = (e[i] - T[i] * Tm) * ip;   // (I - T T^T) e_m / |p'|
        dT[0][m][i] = 2.f * t * proj;
        dT[1][m][i] = proj;
        dbv[0][m][i] = (cA[i] - bb[i] * bA) * ib;
        dbv[1][m][i] = (cB[i] - bb[i] * bB) * ib;
      }
    }
  } else if (X.cls >= 1) {
    // constant frame: T0 from A + B (curved, A || B) or the chord B (straight)
    float T0r[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) T0r[i] = X.cls == 1 ? X.B[i] : X.A[i] + X.B[i];
    const float i0 = rsqrtf(T0r[0] * T0r[0] + T0r[1] * T0r[1] + T0r[2] * T0r[2]);
    const float ut = X.up[0] * T[0] + X.up[1] * T[1] + X.up[2] * T[2];
    float v[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) v[i] = X.up[i] - ut * T[i];
    const float iv = rsqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      float dT0[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) dT0[i] = ((i == m ? 1.f : 0.f) - T[i] * T[m]) * i0;   // d T0 / d(T0r)_m
      const float udT = X.up[0] * dT0[0] + X.up[1] * dT0[1] + X.up[2] * dT0[2];
      float dv[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) dv[i] = -udT * T[i] - ut * dT0[i];
      const float bdv = bb[0] * dv[0] + bb[1] * dv[1] + bb[2] * dv[2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float db = (dv[i] - bb[i] * bdv) * iv;
        // T0r = A + B (curved) or B (straight: the chord; A = 0)
        dT[1][m][i] = dT0[i];
        dbv[1][m][i] = db;
        if (X.cls == 2) { dT[0][m][i] = dT0[i]; dbv[0][m][i] = db; }
      }
    }
  }
  const float tt = t * t;
#pragma unroll
  for (int which = 0; which < 3; ++which)
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      // d d / d theta at fixed t: A_m -> -t^2 e_m, B_m -> -t e_m, w_m -> e_m
      const float sd = which == 0 ? -tt : (which == 1 ? -t : 1.f);
      const float* dTm = dT[which][m];
      const float* dbm = dbv[which][m];
      // dN = db x T + b x dT
      const float dN[3] = {dbm[1] * T[2] - dbm[2] * T[1] + bb[1] * dTm[2] - bb[2] * dTm[1],
                           dbm[2] * T[0] - dbm[0] * T[2] + bb[2] * dTm[0] - bb[0] * dTm[2],
                           dbm[0] * T[1] - dbm[1] * T[0] + bb[0] * dTm[1] - bb[1] * dTm[0]};
      out[which][m][0] = dTm[0] * d[0] + dTm[1] * d[1] + dTm[2] * d[2] + sd * T[m];
      out[which][m][1] = dN[0] * d[0] + dN[1] * d[1] + dN[2] * d[2] + sd * N[m];
      out[which][m][2] = dbm[0] * d[0] + dbm[1] * d[1] + dbm[2] * d[2] + sd * bb[m];
    }
  // y_t: Frenet T' = (p'' - T (T.p'')) / |p'|, N' = b x T'; constant frames: -R^T p'
  if (X.cls == 2 && X.frenet) {
    const float ip = rsqrtf(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
    const float tp = 2.f * (T[0] * X.A[0] + T[1] * X.A[1] + T[2] * X.A[2]);
    float Tp[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) Tp[i] = (2.f * X.A[i] - T[i] * tp) * ip;
    const float Np[3] = {bb[1] * Tp[2] - bb[2] * Tp[1], bb[2] * Tp[0] - bb[0] * Tp[2], bb[0] * Tp[1] - bb[1] * Tp[0]};
    yt[0] = (Tp[0] * d[0] + Tp[1] * d[1] + Tp[2] * d[2]) - (T[0] * pd[0] + T[1] * pd[1] + T[2] * pd[2]);
    yt[1] = (Np[0] * d[0] + Np[1] * d[1] + Np[2] * d[2]) - (N[0] * pd[0] + N[1] * pd[1] + N[2] * pd[2]);
  } else {
    yt[0] = -(T[0] * pd[0] + T[1] * pd[1] + T[2] * pd[2]);
    yt[1] = -(N[0] * pd[0] + N[1] * pd[1] + N[2] * pd[2]);
  }
  yt[2] = -(bb[0] * pd[0] + bb[1] * pd[1] + bb[2] * pd[2]);
}

template <class Emit>
__device__ __forceinline__ void xpsq_param_grad(const SceneDev& S, const Xpsq& X, const float* y, float scale,
                                                Emit emit) {
  const float w[3] = {y[0] - X.p1[0], y[1] - X.p1[1], y[2] - X.p1[2]};
  float tv[3], tg[3][3], th[3][6];
  const bool single = xpsq_root_t<0>(X, S.sp, w, tv, tg, th);
  const int nr = single ? 1 : 3, np = X.n_planes;
  const bool vary = X.varying != 0;
  const float itl = LOG2E * S.sp.i_min, tau = S.sp.tau_min;
  float g5[3][5], wsq[3], phk[3], yk[3][3], wpl[3][CM_MAX_PLANES];
  // the plane j at root parameter t: unit normal n, 1 / |v|, offset h
  auto plane_at = [&](int j, float t, float* n, float& iv, float& h) {
    if (vary) {
      float v[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) v[i] = fmaf(t, X.dpl[j][i], X.pl0[j][i]);
      iv = rsqrtf(fmaf(v[0], v[0], fmaf(v[1], v[1], v[2] * v[2])));
#pragma unroll
      for (int i = 0; i < 3; ++i) n[i] = v[i] * iv;
      h = fmaf(t, X.dpl[j][3], X.pl0[j][3]);
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i) n[i] = X.pl0[j][i];
      iv = 1.f;
      h = X.pl0[j][3];
    }
  };
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (k >= nr) break;
    const float t = tv[k];
    float pd[3], d[3], T[3], N[3], bb[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      pd[i] = fmaf(2.f * X.A[i], t, X.B[i]);
      d[i] = y[i] - fmaf(fmaf(X.A[i], t, X.B[i]), t, X.p1[i]);
    }
    if (X.frenet) {
      const float in = rsqrtf(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
#pragma unroll
      for (int i = 0; i < 3; ++i) { T[i] = pd[i] * in; bb[i] = X.bhat[i]; }
      N[0] = bb[1] * T[2] - bb[2] * T[1]; N[1] = bb[2] * T[0] - bb[0] * T[2]; N[2] = bb[0] * T[1] - bb[1] * T[0];
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i) { T[i] = X.R0[i * 3 + 0]; N[i] = X.R0[i * 3 + 1]; bb[i] = X.R0[i * 3 + 2]; }
    }
    yk[k][0] = T[0] * d[0] + T[1] * d[1] + T[2] * d[2];
    yk[k][1] = N[0] * d[0] + N[1] * d[1] + N[2] * d[2];
    yk[k][2] = bb[0] * d[0] + bb[1] * d[1] + bb[2] * d[2];
    float phs;
    if (vary) {   // the SQ constants of the cross-section at t_k
      float ia[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) ia[i] = 1.f / fmaf(t, X.da[i], X.a0[i]);
      const float e1 = fmaf(t, X.deps[0], X.eps0[0]), e2 = fmaf(t, X.deps[1], X.eps0[1]);
      const float ie1 = 1.f / e1;
      phs = sq_param_grad_p(ia, ie1, 1.f / e2, e2 * ie1, 0.5f * e1, yk[k], g5[k]);
    } else {
      phs = sq_param_grad_p(X.sq_ia, X.sq_p1, X.sq_p2, X.sq_m, X.sq_k, yk[k], g5[k]);
    }
    float mx = phs;
    float pv[CM_MAX_PLANES];
    for (int j = 0; j < np; ++j) {
      float n[3], iv, h;
      plane_at(j, t, n, iv, h);
      pv[j] = fmaf(n[0], yk[k][0], fmaf(n[1], yk[k][1], fmaf(n[2], yk[k][2], h)));
      mx = fmaxf(mx, pv[j]);
    }
    float Z = ex2((phs - mx) * itl);
    wsq[k] = Z;
    for (int j = 0; j < np; ++j) {
      wpl[k][j] = ex2((pv[j] - mx) * itl);
      Z += wpl[k][j];
    }
    const float iZ = rcpa(Z);
    wsq[k] *= iZ;
    for (int j = 0; j < np; ++j) wpl[k][j] *= iZ;
    phk[k] = fmaf(tau * LN2, lg2(Z), mx);   // PSQ = tau log sum exp(v / tau)
  }
  float u[3] = {1.f, 0.f, 0.f};
  if (!single) {   // softmax(-phi_k / tau)
    const float mn = fminf(phk[0], fminf(phk[1], phk[2]));
    float Zu = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) { u[k] = ex2((mn - phk[k]) * itl); Zu += u[k]; }
    const float iZu = rcpa(Zu);
#pragma unroll
    for (int k = 0; k < 3; ++k) u[k] *= iZu;
  }
  const int M = 5 + 4 * np;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    float v0 = 0.f, v1 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (k < nr) {
        const float c = u[k] * wsq[k] * g5[k][q];
        v0 = fmaf(c, 1.f - tv[k], v0);
        v1 = fmaf(c, tv[k], v1);
      }
    if (vary) {
      emit(q, scale * v0);
      emit(M + q, scale * v1);
    } else {
      emit(q, scale * (v0 + v1));
    }
  }
  for (int j = 0; j < np; ++j) {
    float dn0[3] = {0.f, 0.f, 0.f}, dn1[3] = {0.f, 0.f, 0.f}, dh0 = 0.f, dh1 = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k >= nr) break;
      float n[3], iv, h;
      plane_at(j, tv[k], n, iv, h);
      const float c = u[k] * wpl[k][j];
      const float ny = n[0] * yk[k][0] + n[1] * yk[k][1] + n[2] * yk[k][2];
      const float a1 = tv[k], a0 = 1.f - a1;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float g = c * iv * (yk[k][i] - ny * n[i]);
        dn0[i] = fmaf(a0, g, dn0[i]);
        dn1[i] = fmaf(a1, g, dn1[i]);
      }
      dh0 = fmaf(a0, c, dh0);
      dh1 = fmaf(a1, c, dh1);
    }
    if (vary) {
      emit(5 + 4 * j, scale * dn0[0]); emit(6 + 4 * j, scale * dn0[1]); emit(7 + 4 * j, scale * dn0[2]);
      emit(8 + 4 * j, scale * dh0);
      emit(M + 5 + 4 * j, scale * dn1[0]); emit(M + 6 + 4 * j, scale * dn1[1]); emit(M + 7 + 4 * j, scale * dn1[2]);
      emit(M + 8 + 4 * j, scale * dh1);
    } else {
      emit(5 + 4 * j, scale * (dn0[0] + dn1[0])); emit(6 + 4 * j, scale * (dn0[1] + dn1[1]));
      emit(7 + 4 * j, scale * (dn0[2] + dn1[2])); emit(8 + 4 * j, scale * (dh0 + dh1));
    }
  }
  // control points p1, p2, p3 (slots base .. base + 8): through the roots,
  // the frame and p(t) of every root's PSQ, weighted by the smooth minimum
  // (DESIGN.md §2 f4; the oracle seeds the control points)
  float dtA[3][3], dtB[3][3], dtw[3][3];
  xpsq_root_dtheta(X, S.sp, w, dtA, dtB, dtw);
  float dph[3][3] = {};   // [A, B, w][m]
#pragma unroll 1
  for (int k = 0; k < nr; ++k) {
    const float t = tv[k];
    float pd[3], d[3], T[3], N[3], bb[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      pd[i] = fmaf(2.f * X.A[i], t, X.B[i]);
      d[i] = y[i] - fmaf(fmaf(X.A[i], t, X.B[i]), t, X.p1[i]);
    }
    if (X.frenet) {
      const float in = rsqrtf(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
#pragma unroll
      for (int i = 0; i < 3; ++i) { T[i] = pd[i] * in; bb[i] = X.bhat[i]; }
      N[0] = bb[1] * T[2] - bb[2] * T[1]; N[1] = bb[2] * T[0] - bb[0] * T[2]; N[2] = bb[0] * T[1] - bb[1] * T[0];
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i) { T[i] = X.R0[i * 3 + 0]; N[i] = X.R0[i * 3 + 1]; bb[i] = X.R0[i * 3 + 2]; }
    }
    // G = grad_y of the PSQ at y_k; S_t = its derivative along t through the
    // schedules (varying only)
    XsqParams q;
    if (vary) {
#pragma unroll
      for (int i = 0; i < 3; ++i) q.ia[i] = 1.f / fmaf(t, X.da[i], X.a0[i]);
      const float e1 = fmaf(t, X.deps[0], X.eps0[0]), e2 = fmaf(t, X.deps[1], X.eps0[1]);
      q.p1 = 1.f / e1; q.p2 = 1.f / e2; q.m = e2 / e1; q.k = 0.5f * e1;
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i) q.ia[i] = X.sq_ia[i];
      q.p1 = X.sq_p1; q.p2 = X.sq_p2; q.m = X.sq_m; q.k = X.sq_k;
    }
    Res<1> rs;
    sq_eval<1>(q, yk[k], rs);
    float G[3] = {wsq[k] * rs.g[0], wsq[k] * rs.g[1], wsq[k] * rs.g[2]};
    float St = 0.f;
    if (vary) {
      St = wsq[k] * (g5[k][0] * X.da[0] + g5[k][1] * X.da[1] + g5[k][2] * X.da[2] + g5[k][3] * X.deps[0] +
                     g5[k][4] * X.deps[1]);
    }
    for (int j = 0; j < np; ++j) {
      float n[3], iv, h;
      plane_at(j, t, n, iv, h);
#pragma unroll
      for (int i = 0; i < 3; ++i) G[i] = fmaf(wpl[k][j], n[i], G[i]);
      if (vary) {   // d(n.y + h)/dt = ((I - n n^T) dpl / |v|).y + dh
        const float nd = n[0] * X.dpl[j][0] + n[1] * X.dpl[j][1] + n[2] * X.dpl[j][2];
        float dn = 0.f;
#pragma unroll
        for (int i = 0; i < 3; ++i) dn = fmaf((X.dpl[j][i] - n[i] * nd) * iv, yk[k][i], dn);
        St = fmaf(wpl[k][j], dn + X.dpl[j][3], St);
      }
    }
    float dyt[3][3][3], yt[3];
    xpsq_dy_dtheta(X, t, d, T, N, bb, dyt, yt);
    const float Gyt = G[0] * yt[0] + G[1] * yt[1] + G[2] * yt[2] + St;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const float dts[3] = {dtA[k][m], dtB[k][m], dtw[k][m]};
#pragma unroll
      for (int which = 0; which < 3; ++which) {
        const float v = G[0] * dyt[which][m][0] + G[1] * dyt[which][m][1] + G[2] * dyt[which][m][2] + Gyt * dts[which];
        dph[which][m] = fmaf(u[k], v, dph[which][m]);
      }
    }
  }
  const int base = (vary ? 2 : 1) * M;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    if (X.cls == 1) {   // straight: the chord B = p3 - p1 (A = 0), w = x - p1
      emit(base + m, scale * (-dph[1][m] - dph[2][m]));
      emit(base + 3 + m, 0.f);
      emit(base + 6 + m, scale * dph[1][m]);
    } else {            // A = p1 - 2 p2 + p3, B = 2 (p2 - p1), w = x - p1
      emit(base + m, scale * (dph[0][m] - 2.f * dph[1][m] - dph[2][m]));
      emit(base + 3 + m, scale * (-2.f * dph[0][m] + 2.f * dph[1][m]));
      emit(base + 6 + m, scale * dph[0][m]);
    }
  }
}

// parameters of leaf li at the shape-frame point x, scaled by d phi_shape /
// d phi_leaf; emit(k, value) is called for k = 0 .. count-1
template <class Emit>
__device__ __forceinline__ void leaf_param_grad(const SceneDev& S, int li, const float* x, float scale, Emit emit) {
  const Leaf& L = S.leaves[li];
  float y[3];
  const float t[3] = {L.t[0], L.t[1], L.t[2]};
  float R[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = L.R[i];
  to_local(R, t, x, y);
  if (L.kind == LK_XPSQ) {
    xpsq_param_grad(S, S.xpsq[L.xidx], y, scale, emit);
    return;
  }
  if (L.kind == LK_HALFSPACE) {   // phi = n.y + h
    emit(0, scale * y[0]); emit(1, scale * y[1]); emit(2, scale * y[2]); emit(3, scale);
    return;
  }
  // SQ, or PSQ = LSE_tau_min(phi_SQ, n_j . y + h_j): weights of the terms
  float g5[5];
  const float phs = sq_param_grad(L, y, g5);
  const int np = L.n_planes;
  float wsq = 1.f;
  float mx = phs, Z = 1.f;
  const float itl = LOG2E * S.sp.i_min;
  if (np > 0) {
    for (int j = 0; j < np; ++j) {
      const float* pl = L.planes[j];
      mx = fmaxf(mx, fmaf(pl[0], y[0], fmaf(pl[1], y[1], fmaf(pl[2], y[2], pl[3]))));
    }
    Z = ex2((phs - mx) * itl);
    wsq = Z;
    for (int j = 0; j < np; ++j) {
      const float* pl = L.planes[j];
      Z += ex2((fmaf(pl[0], y[0], fmaf(pl[1], y[1], fmaf(pl[2], y[2], pl[3]))) - mx) * itl);
    }
    wsq *= rcpa(Z);
  }
#pragma unroll
  for (int q = 0; q < 5; ++q) emit(q, scale * wsq * g5[q]);
  for (int j = 0; j < np; ++j) {
    const float* pl = L.planes[j];
    const float wj = ex2((fmaf(pl[0], y[0], fmaf(pl[1], y[1], fmaf(pl[2], y[2], pl[3]))) - mx) * itl) * rcpa(Z);
    const float sw = scale * wj;
    emit(5 + 4 * j, sw * y[0]); emit(6 + 4 * j, sw * y[1]); emit(7 + 4 * j, sw * y[2]); emit(8 + 4 * j, sw);
  }
}

__device__ __forceinline__ int leaf_param_count(const SceneDev& S, const Leaf& L) {
  if (L.kind == LK_HALFSPACE) return 4;
  if (L.kind != LK_XPSQ) return 5 + 4 * L.n_planes;
  const Xpsq& X = S.xpsq[L.xidx];
  return (X.varying ? 2 : 1) * (5 + 4 * X.n_planes) + 9;   // + control points
}


// d phi / d (every parameter of shape sh) at the shape-frame point y:
// emit(k, value) for k = 0 .. count - 1 (the cm_param_layout order); returns
// the count.  Boolean trees (Eqs. (2)-(4), postfix program, nesting <=
// CM_MAX_DEPTH, <= kParamMaxNodes boolean nodes): node N: phi_N = s_N tau
// log sum_c exp(s_c phi_c / tau), so d phi_N / d phi_c = s_N s_c
// softmax_N(c) and d phi / d phi_leaf is the product of these factors over
// the leaf's ancestors.  Pass 1: every node's accumulator (max m, sum Z),
// its signs and its folded value s_c phi_N; pass 2: the factors down the
// tree, one leaf parameter block at a time (leaves in program = pre-order).
template <class Emit>
__device__ __forceinline__ int shape_param_grad(const SceneDev& S, const ShapeRec& sh, const float* y, Emit emit) {
  int kbase = 0;
  auto emitk = [&](int k, float v) { emit(kbase + k, v); };
  const Instr* prog = S.prog + sh.prog_begin;
  if (sh.prog_len == 1) {
    leaf_param_grad(S, prog[0].idx, y, 1.f, emitk);
    kbase += leaf_param_count(S, S.leaves[prog[0].idx]);
  } else {
    const float tau = S.sp.tau_min, itl = LOG2E * S.sp.i_min;
    float nm[kParamMaxNodes], nz[kParamMaxNodes], nfv[kParamMaxNodes], nos[kParamMaxNodes], ncs[kParamMaxNodes];
    int stk[CM_MAX_DEPTH + 1];
    float am[CM_MAX_DEPTH + 1], az[CM_MAX_DEPTH + 1];
    int lvl = -1, nn = 0;
    for (int pc = 0; pc < sh.prog_len; ++pc) {
      const Instr in = prog[pc];
      if (in.op == OP_BEGIN) {
        ++lvl;
        stk[lvl] = nn++;
        am[lvl] = -INFINITY;
        az[lvl] = 0.f;
        continue;
      }
      float v;
      if (in.op == OP_LEAF) {
        Res<0> r;
        leaf_eval<0, 2, false>(S, in.idx, y, r);
        v = in.child_sign * r.v;
      } else {   // OP_END: node value from its accumulator, folded into the parent
        const int k = stk[lvl];
        nm[k] = am[lvl];
        nz[k] = az[lvl];
        nos[k] = in.out_sign;
        ncs[k] = in.child_sign;
        v = in.child_sign * (in.out_sign * fmaf(tau * LN2, lg2(az[lvl]), am[lvl]));
        nfv[k] = v;
        --lvl;
      }
      if (lvl >= 0) {
        if (v > am[lvl]) { az[lvl] = fmaf(az[lvl], ex2((am[lvl] - v) * itl), 1.f); am[lvl] = v; }
        else az[lvl] += ex2((v - am[lvl]) * itl);
      }
    }
    float fac[CM_MAX_DEPTH + 1];
    lvl = -1;
    nn = 0;
    for (int pc = 0; pc < sh.prog_len; ++pc) {
      const Instr in = prog[pc];
      if (in.op == OP_BEGIN) {
        const int k = nn++;
        if (lvl < 0) {
          fac[0] = 1.f;
        } else {   // d phi_parent / d phi_k = s_parent s_k softmax_parent(k)
          const int p = stk[lvl];
          fac[lvl + 1] = fac[lvl] * nos[p] * ncs[k] * ex2((nfv[k] - nm[p]) * itl) * rcpa(nz[p]);
        }
        stk[++lvl] = k;
        continue;
      }
      if (in.op == OP_END) { --lvl; continue; }
      const int k = stk[lvl];
      Res<0> r;
      leaf_eval<0, 2, false>(S, in.idx, y, r);
      const float sc = fac[lvl] * nos[k] * in.child_sign * ex2((in.child_sign * r.v - nm[k]) * itl) * rcpa(nz[k]);
      leaf_param_grad(S, in.idx, y, sc, emitk);
      kbase += leaf_param_count(S, S.leaves[in.idx]);
    }
  }
  return kbase;
}

}  // namespace cmd
