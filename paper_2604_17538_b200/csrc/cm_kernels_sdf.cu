// sm_100a kernel of the sdf_eval path (arXiv 2604.17538 §II-B, Eq. (1)-(6)):
//   k_sdf_eval  batched SDF value / gradient / Hessian (+ pose derivatives),
//               one thread per point, one instantiation per SDF class.
// FP32 CUDA-core math (not a dense contraction: no tensor cores), MUFU
// ex2/lg2/rcp in the log domain, field-major coalesced stores.
// The manifold kernels are in cm_kernels_manifold.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#ifndef CM_LEAF_VEC
#define CM_LEAF_VEC 1   // explicit 128-bit leaf loads in this unit (SDF +1.3%, r02z4)
#endif
#include "cm_device.cuh"
#include "cm_internal.h"
#include "cm_launch.h"

using namespace cmi;
using namespace cmd;

using cml::check_launch;
using cml::num_sms;

// ============================================================================
// sdf_eval
// ============================================================================
#ifndef CM_SDF_MINB
#define CM_SDF_MINB 3   // 80 registers: +2% on the SDF workload over 1 and 2
#endif
#ifndef CM_SDF_XINL
#define CM_SDF_XINL true    // constant-schedule XPSQ evaluator inlined in sdf_eval: +6.5% over out of line (r02r)
#endif
#ifndef CM_SDF_MINB_XP
#define CM_SDF_MINB_XP 2   // the XPSQ classes (1, 2, 4): 128 registers, SDF +1.8% over 80 (r02m)
#endif
template <int O, int XP, bool PG, bool PH>
__global__ void __launch_bounds__(256, (XP == 1 || XP == 2 || XP == 4) ? CM_SDF_MINB_XP : CM_SDF_MINB) k_sdf_eval(SceneDev S, const int32_t* __restrict__ shape_ids,
                                                  const float* __restrict__ poses, const float* __restrict__ points,
                                                  int64_t B, int64_t P, float* __restrict__ d,
                                                  float* __restrict__ grad, float* __restrict__ hess,
                                                  float* __restrict__ dpose, float* __restrict__ d2pose,
                                                  float* __restrict__ dxdpose, int xp_filter, int own_invalid) {
  const int64_t N = B * P;
  const bool n32 = N <= 0x7fffffff;   // 32-bit index arithmetic (no 64-bit division)
  // (warps walking 32-point segments with the class decided once per warp
  // measured -7.5% on the SDF workload, r02r)
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = n32 ? (int64_t)((uint32_t)n / (uint32_t)P) : n / P;
    const int sid = __ldg(shape_ids + b);
    // the class byte first: points of other classes are skipped without
    // loading their 64-B shape record
    const int cls = (unsigned)sid < (unsigned)S.n_shapes ? (int)__ldg(S.shape_cls + sid) : -1;
    if (cls >= 0 && xp_filter >= 0 && cls != xp_filter) continue;
    if (cls < 0) {
      // invalid shape id (or a shape without an SDF): NaN outputs, written and
      // counted once per point by the first class instantiation launched
      if (own_invalid) {
        const float qn = __int_as_float(0x7fc00000);
        d[n] = qn;
        if (grad) for (int k = 0; k < 3; ++k) grad[k * N + n] = qn;
        if (hess) for (int k = 0; k < 6; ++k) hess[k * N + n] = qn;
        if (dpose) for (int k = 0; k < 6; ++k) dpose[k * N + n] = qn;
        if (d2pose) for (int k = 0; k < 21; ++k) d2pose[k * N + n] = qn;
        if (dxdpose) for (int k = 0; k < 18; ++k) dxdpose[k * N + n] = qn;
        atomicAdd(S.err, 1u);
      }
      continue;
    }
    const ShapeRec sh = S.shapes[sid];
    const float4 pa = __ldg(reinterpret_cast<const float4*>(poses) + 2 * b);
    const float4 pb = __ldg(reinterpret_cast<const float4*>(poses) + 2 * b + 1);
    const float t[3] = {pa.x, pa.y, pa.z};
    const float q[4] = {pa.w, pb.x, pb.y, pb.z};
    float R[9];
    quat_to_R(q, R);
    const float x[3] = {__ldg(points + 3 * n), __ldg(points + 3 * n + 1), __ldg(points + 3 * n + 2)};
    float y[3];
    to_local(R, t, x, y);
    Res<O> r;
    // class 4 (XPSQ operands of boolean trees): provably negligible union
    // operands culled, as in the manifold kernels (cm_device.cuh eval_prog)
    eval_shape<O, XP == 3 ? 0 : (XP == 4 ? 1 : XP), XP == 0, CM_SDF_XINL, XP == 4>(S, sh, y, r);
    d[n] = r.v;
    if constexpr (O >= 1) {
      float g[3];
      rot_vec(R, r.g, g);
      if (grad) {
        grad[n] = g[0]; grad[N + n] = g[1]; grad[2 * N + n] = g[2];
      }
      const float rv[3] = {x[0] - t[0], x[1] - t[1], x[2] - t[2]};
      if constexpr (PG) {
        // d phi / d(dt, dtheta) = (-g, g x r)
        dpose[n] = -g[0]; dpose[N + n] = -g[1]; dpose[2 * N + n] = -g[2];
        dpose[3 * N + n] = g[1] * rv[2] - g[2] * rv[1];
        dpose[4 * N + n] = g[2] * rv[0] - g[0] * rv[2];
        dpose[5 * N + n] = g[0] * rv[1] - g[1] * rv[0];
      }
      if constexpr (O >= 2) {
        float h[6];
        rot_sym(R, r.h, h);
        if (hess) {
#pragma unroll
          for (int k = 0; k < 6; ++k) hess[k * N + n] = h[k];
        }
        if constexpr (PH) {
          const float H[3][3] = {{h[0], h[1], h[2]}, {h[1], h[3], h[4]}, {h[2], h[4], h[5]}};
          // K = [r]x, HK = H [r]x, G = [g]x
          const float K[3][3] = {{0.f, -rv[2], rv[1]}, {rv[2], 0.f, -rv[0]}, {-rv[1], rv[0], 0.f}};
          const float G[3][3] = {{0.f, -g[2], g[1]}, {g[2], 0.f, -g[0]}, {-g[1], g[0], 0.f}};
          float HK[3][3], KHK[3][3];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) HK[i][j] = H[i][0] * K[0][j] + H[i][1] * K[1][j] + H[i][2] * K[2][j];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) KHK[i][j] = K[i][0] * HK[0][j] + K[i][1] * HK[1][j] + K[i][2] * HK[2][j];
          const float gr = g[0] * rv[0] + g[1] * rv[1] + g[2] * rv[2];
          // 6x6: tt = H; t-theta = -H[r]x + [g]x; theta-theta =
          // -[r]x H [r]x + (g r^T + r g^T)/2 - (g.r) I
          float M6[6][6];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              M6[i][j] = H[i][j];
              M6[i][3 + j] = -HK[i][j] + G[i][j];
              M6[3 + i][3 + j] = -KHK[i][j] + 0.5f * (g[i] * rv[j] + rv[i] * g[j]) - (i == j ? gr : 0.f);
            }
          int kk = 0;
#pragma unroll
          for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = i; j < 6; ++j) d2pose[(kk++) * N + n] = M6[i][j];
          // d grad / d pose = [-H, H[r]x - [g]x]
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              dxdpose[(i * 6 + j) * N + n] = -H[i][j];
              dxdpose[(i * 6 + 3 + j) * N + n] = HK[i][j] - G[i][j];
            }
        }
      }
    }
  }
}

template <int O, int XP, bool PG, bool PH>
static int launch_sdf_t(const SceneDev& s, int xp_filter, int own, const int32_t* ids, const float* poses, const float* pts,
                        int64_t B, int64_t P, float* d, float* g, float* h, float* dp, float* d2p, float* dxp,
                        cudaStream_t st) {
  const int threads = 256;
  int64_t N = B * P;
  int64_t blocks = (N + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_sdf_eval<O, XP, PG, PH><<<(unsigned)blocks, threads, 0, st>>>(s, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp,
                                                                   xp_filter, own);
  return check_launch("k_sdf_eval");
}

template <int XP>
static int dispatch_sdf(const SceneDev& s, int xp_filter, int own, const int32_t* ids, const float* poses, const float* pts,
                        int64_t B, int64_t P, uint32_t flags, float* d, float* g, float* h, float* dp, float* d2p,
                        float* dxp, cudaStream_t st) {
  const bool PG = flags & CM_SDF_POSE_GRAD, PH = flags & CM_SDF_POSE_HESS;
  const int O = (flags & (CM_SDF_HESS | CM_SDF_POSE_HESS)) ? 2 : ((flags & (CM_SDF_GRAD | CM_SDF_POSE_GRAD)) ? 1 : 0);
  if (O == 0) return launch_sdf_t<0, XP, false, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  if (O == 1) {
    if (PG) return launch_sdf_t<1, XP, true, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
    return launch_sdf_t<1, XP, false, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  }
  if (PG && PH) return launch_sdf_t<2, XP, true, true>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  if (PG) return launch_sdf_t<2, XP, true, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  if (PH) return launch_sdf_t<2, XP, false, true>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  return launch_sdf_t<2, XP, false, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
}

namespace cml {

int launch_sdf_eval(const SceneDev& s, int class_mask, const int32_t* ids, const float* poses, const float* pts,
                    int64_t B, int64_t P, uint32_t flags, float* d, float* g, float* h, float* dp, float* d2p,
                    float* dxp, void* const* streams, int n_streams) {
  // class_mask bit c: the scene has SDF shapes of class c (0 SQ family, 1
  // constant-schedule XPSQ, 2 varying-schedule XPSQ); one instantiation per
  // present class, each filtering its own shapes when several are present;
  // the j-th present class runs on streams[j % n_streams] (concurrent classes
  // fill each other's wave tails)
  const bool multi = (class_mask & (class_mask - 1)) != 0;
  int rc = CM_OK, j = 0;
  auto next = [&]() { return (cudaStream_t)streams[(j++) % n_streams]; };
  const int first = class_mask ? __builtin_ctz(class_mask) : 0;   // owns invalid shape ids
  if (class_mask & 1)
    rc = dispatch_sdf<0>(s, multi ? 0 : -1, first == 0, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next());
  if (!rc && (class_mask & 2))
    rc = dispatch_sdf<1>(s, multi ? 1 : -1, first == 1, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next());
  if (!rc && (class_mask & 4))
    rc = dispatch_sdf<2>(s, multi ? 2 : -1, first == 2, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next());
  // nested SQ-family shapes: general interpreter, no XPSQ code
  if (!rc && (class_mask & 8))
    rc = dispatch_sdf<3>(s, multi ? 3 : -1, first == 3, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next());
  // constant-schedule XPSQ inside boolean trees
  if (!rc && (class_mask & 16))
    rc = dispatch_sdf<4>(s, multi ? 4 : -1, first == 4, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next());
  return rc;
}

}  // namespace cml

// ============================================================================
// shape-parameter derivatives
// ============================================================================
namespace {

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

// one thread per point; shapes are single leaves or boolean trees of up to
// kParamMaxNodes nodes (SQ family or XPSQ leaves).
// J[k * N + n]; vjp[poff[shape] + k] += w[n] J[k, n] (warp-reduced when the
// warp's points share one shape, else per-lane atomics)
__global__ void __launch_bounds__(256) k_sdf_param_grad(SceneDev S, const int32_t* __restrict__ shape_ids,
                                                        const float* __restrict__ poses,
                                                        const float* __restrict__ points, int64_t B, int64_t P,
                                                        int32_t pmax, float* __restrict__ J,
                                                        const float* __restrict__ w, float* __restrict__ vjp,
                                                        const int64_t* __restrict__ poff) {
  const int64_t N = B * P;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // every lane of a warp runs the same number of iterations (warp reductions)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < N; base += stride) {
    const int64_t n = base + lane;
    const bool valid = n < N;
    const int64_t b = valid ? n / P : 0;
    const int sid = valid ? __ldg(shape_ids + b) : -1;
    const int sid0 = __shfl_sync(0xffffffffu, sid, 0);
    const bool uni = __all_sync(0xffffffffu, valid && sid == sid0);
    if (!valid) continue;
    if ((unsigned)sid >= (unsigned)S.n_shapes || !S.shapes[sid].has_sdf) {
      // invalid shape id: NaN rows of J, no VJP contribution, counted (a warp
      // is uniform only if all its lanes take this branch: no shuffles skipped)
      if (J)
        for (int k = 0; k < pmax; ++k) J[(int64_t)k * N + n] = __int_as_float(0x7fc00000);
      atomicAdd(S.err, 1u);
      continue;
    }
    const ShapeRec sh = S.shapes[sid];
    const float4 pa = __ldg(reinterpret_cast<const float4*>(poses) + 2 * b);
    const float4 pb = __ldg(reinterpret_cast<const float4*>(poses) + 2 * b + 1);
    const float t[3] = {pa.x, pa.y, pa.z};
    const float q[4] = {pa.w, pb.x, pb.y, pb.z};
    float R[9];
    quat_to_R(q, R);
    const float x[3] = {__ldg(points + 3 * n), __ldg(points + 3 * n + 1), __ldg(points + 3 * n + 2)};
    float y[3];
    to_local(R, t, x, y);
    const float wn = vjp ? __ldg(w + n) : 0.f;
    const int64_t off = vjp ? __ldg(poff + sid) : 0;
    int kbase = 0;
    auto emit = [&](int k, float v) {
      const int kk = kbase + k;
      if (J && kk < pmax) J[(int64_t)kk * N + n] = v;
      if (vjp) {
        float s = wn * v;
        if (uni) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) atomicAdd(vjp + off + kk, s);
        } else {
          atomicAdd(vjp + off + kk, s);
        }
      }
    };
    const Instr* prog = S.prog + sh.prog_begin;
    if (sh.prog_len == 1) {
      leaf_param_grad(S, prog[0].idx, y, 1.f, emit);
      kbase += leaf_param_count(S, S.leaves[prog[0].idx]);
    } else {
      // boolean tree (Eqs. (2)-(4), postfix program, nesting <= CM_MAX_DEPTH):
      // node N: phi_N = s_N tau log sum_c exp(s_c phi_c / tau), so
      // d phi_N / d phi_c = s_N s_c softmax_N(c) and d phi / d phi_leaf is the
      // product of these factors over the leaf's ancestors.
      // Pass 1: every node's accumulator (max m, sum Z), its signs and its
      // folded value s_c phi_N; pass 2: the factors down the tree, one leaf
      // parameter block at a time (leaves in program = pre-order).
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
        leaf_param_grad(S, in.idx, y, sc, emit);
        kbase += leaf_param_count(S, S.leaves[in.idx]);
      }
    }
    if (J)
      for (int kk = kbase; kk < pmax; ++kk) J[(int64_t)kk * N + n] = 0.f;
  }
}


// ---- node-pose derivatives (f4, reading #47) --------------------------------
// d phi / d twist of node k (in its parent frame P, x_shape = RP x_P + tP):
// phi depends on the node's pose only through the node's own SDF phi_k, which
// the twist moves rigidly about the node origin tk (in P), so
//   d phi / d dt = -f_k gP,  d phi / d dtheta = f_k gP x (xP - tk),
// f_k = d phi / d phi_k (through the enclosing LSEs, Eqs. (2)-(4)),
// gP = RP^T grad phi_k(x), xP = RP^T (x - tP).
template <class Emit>
__device__ __forceinline__ void node_twist(const NodeFrame& nf, const float* y, float fac, const float* g,
                                           Emit emit) {
  float gP[3], xr[3];
  const float d[3] = {y[0] - nf.tP[0], y[1] - nf.tP[1], y[2] - nf.tP[2]};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    gP[i] = nf.RP[i] * g[0] + nf.RP[3 + i] * g[1] + nf.RP[6 + i] * g[2];
    xr[i] = nf.RP[i] * d[0] + nf.RP[3 + i] * d[1] + nf.RP[6 + i] * d[2] - nf.tk[i];
  }
  const int b = 6 * nf.node;
  emit(b + 0, -fac * gP[0]);
  emit(b + 1, -fac * gP[1]);
  emit(b + 2, -fac * gP[2]);
  emit(b + 3, fac * (gP[1] * xr[2] - gP[2] * xr[1]));
  emit(b + 4, fac * (gP[2] * xr[0] - gP[0] * xr[2]));
  emit(b + 5, fac * (gP[0] * xr[1] - gP[1] * xr[0]));
}

// one thread per point (the layout of k_sdf_param_grad): pass 1 evaluates the
// shape program at order 1 keeping every boolean node's accumulator (max,
// sum), its folded value and the gradient of its own value; pass 2 walks the
// program again with the factors d phi / d phi_node down the tree and emits
// each node's six slots (boolean nodes at their BEGIN, leaves with their
// order-1 evaluation)
__global__ void __launch_bounds__(256) k_sdf_node_pose_grad(SceneDev S, const int32_t* __restrict__ shape_ids,
                                                            const float* __restrict__ poses,
                                                            const float* __restrict__ points, int64_t B, int64_t P,
                                                            int32_t nmax, float* __restrict__ J,
                                                            const float* __restrict__ w, float* __restrict__ vjp,
                                                            const int64_t* __restrict__ noff) {
  const int64_t N = B * P;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < N; base += stride) {
    const int64_t n = base + lane;
    const bool valid = n < N;
    const int64_t b = valid ? n / P : 0;
    const int sid = valid ? __ldg(shape_ids + b) : -1;
    const int sid0 = __shfl_sync(0xffffffffu, sid, 0);
    const bool uni = __all_sync(0xffffffffu, valid && sid == sid0);
    if (!valid) continue;
    if ((unsigned)sid >= (unsigned)S.n_shapes || !S.shapes[sid].has_sdf) {
      if (J)
        for (int k = 0; k < nmax; ++k) J[(int64_t)k * N + n] = __int_as_float(0x7fc00000);
      atomicAdd(S.err, 1u);
      continue;
    }
    const ShapeRec sh = S.shapes[sid];
    const float4 pa = __ldg(reinterpret_cast<const float4*>(poses) + 2 * b);
    const float4 pb = __ldg(reinterpret_cast<const float4*>(poses) + 2 * b + 1);
    const float t[3] = {pa.x, pa.y, pa.z};
    const float q[4] = {pa.w, pb.x, pb.y, pb.z};
    float R[9];
    quat_to_R(q, R);
    const float x[3] = {__ldg(points + 3 * n), __ldg(points + 3 * n + 1), __ldg(points + 3 * n + 2)};
    float y[3];
    to_local(R, t, x, y);
    const float wn = vjp ? __ldg(w + n) : 0.f;
    const int64_t off = vjp ? __ldg(noff + sid) : 0;
    // slots of nodes the program does not reach stay zero
    if (J)
      for (int k = 0; k < nmax; ++k) J[(int64_t)k * N + n] = 0.f;
    auto emit = [&](int kk, float v) {
      if (J && kk < nmax) J[(int64_t)kk * N + n] = v;
      if (vjp) {
        float s = wn * v;
        if (uni) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) atomicAdd(vjp + off + kk, s);
        } else {
          atomicAdd(vjp + off + kk, s);
        }
      }
    };
    const Instr* prog = S.prog + sh.prog_begin;
    const NodeFrame* nfr = S.op_frames + sh.prog_begin;
    if (sh.prog_len == 1) {
      Res<1> r;
      leaf_eval<1, 2, false>(S, prog[0].idx, y, r);
      node_twist(nfr[0], y, 1.f, r.g, emit);
      continue;
    }
    const float tau = S.sp.tau_min, itau = S.sp.i_min, itl = LOG2E * itau;
    float nm[kParamMaxNodes], nz[kParamMaxNodes], nfv[kParamMaxNodes], nos[kParamMaxNodes], ncs[kParamMaxNodes];
    float ng[kParamMaxNodes][3];
    int stk[CM_MAX_DEPTH + 1];
    Acc<1> acc[CM_MAX_DEPTH + 1];
    int lvl = -1, nn = 0;
    for (int pc = 0; pc < sh.prog_len; ++pc) {   // pass 1: node accumulators and gradients
      const Instr in = prog[pc];
      if (in.op == OP_BEGIN) {
        ++lvl;
        stk[lvl] = nn++;
        acc_init(acc[lvl]);
        continue;
      }
      Res<1> r;
      if (in.op == OP_LEAF) {
        leaf_eval<1, 2, false>(S, in.idx, y, r);
      } else {   // OP_END: the node's own value and gradient
        const int k = stk[lvl];
        nm[k] = acc[lvl].m;
        nz[k] = acc[lvl].S;
        nos[k] = in.out_sign;
        ncs[k] = in.child_sign;
        acc_final(acc[lvl], in.out_sign, tau, itau, r);
        nfv[k] = in.child_sign * r.v;
#pragma unroll
        for (int i = 0; i < 3; ++i) ng[k][i] = r.g[i];
        --lvl;
      }
      if (lvl >= 0) acc_fold(acc[lvl], in.child_sign, r, itl, itau);
    }
    float fac[CM_MAX_DEPTH + 1];
    lvl = -1;
    nn = 0;
    for (int pc = 0; pc < sh.prog_len; ++pc) {   // pass 2: factors down the tree, six slots per node
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
        node_twist(nfr[pc], y, fac[lvl], ng[k], emit);
        continue;
      }
      if (in.op == OP_END) { --lvl; continue; }
      const int k = stk[lvl];
      Res<1> r;
      leaf_eval<1, 2, false>(S, in.idx, y, r);
      const float sc = fac[lvl] * nos[k] * in.child_sign * ex2((in.child_sign * r.v - nm[k]) * itl) * rcpa(nz[k]);
      node_twist(nfr[pc], y, sc, r.g, emit);
    }
  }
}

}  // namespace

namespace cml {

int launch_sdf_node_pose_grad(const SceneDev& s, const int32_t* ids, const float* poses, const float* pts, int64_t B,
                              int64_t P, int32_t nmax, float* J, const float* w, float* vjp, const int64_t* noff,
                              void* stream) {
  const int threads = 256;
  const int64_t N = B * P;
  int64_t blocks = (N + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_sdf_node_pose_grad<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(s, ids, poses, pts, B, P, nmax, J, w,
                                                                               vjp, noff);
  return check_launch("k_sdf_node_pose_grad");
}

int launch_sdf_param_grad(const SceneDev& s, const int32_t* ids, const float* poses, const float* pts, int64_t B,
                          int64_t P, int32_t pmax, float* J, const float* w, float* vjp, const int64_t* poff,
                          void* stream) {
  const int threads = 256;
  const int64_t N = B * P;
  int64_t blocks = (N + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_sdf_param_grad<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(s, ids, poses, pts, B, P, pmax, J, w, vjp,
                                                                           poff);
  return check_launch("k_sdf_param_grad");
}

}  // namespace cml
