// sm_100a kernel of the sdf_eval path (arXiv 2604.17538 §II-B, Eq. (1)-(6)):
//   k_sdf_eval  batched SDF value / gradient / Hessian (+ pose derivatives),
//               one thread per point, one instantiation per SDF class.
// FP32 CUDA-core math (not a dense contraction: no tensor cores), MUFU
// ex2/lg2/rcp in the log domain, field-major coalesced stores.
// The manifold kernels are in cm_kernels_manifold.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

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
template <int O, int XP, bool PG, bool PH>
__global__ void __launch_bounds__(256) k_sdf_eval(SceneDev S, const int32_t* __restrict__ shape_ids,
                                                  const float* __restrict__ poses, const float* __restrict__ points,
                                                  int64_t B, int64_t P, float* __restrict__ d,
                                                  float* __restrict__ grad, float* __restrict__ hess,
                                                  float* __restrict__ dpose, float* __restrict__ d2pose,
                                                  float* __restrict__ dxdpose, int xp_filter) {
  const int64_t N = B * P;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N; n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = n / P;
    const ShapeRec sh = S.shapes[__ldg(shape_ids + b)];
    if (xp_filter >= 0 && sh.uses_xpsq != xp_filter) continue;
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
    eval_shape<O, XP == 3 ? 0 : XP, XP == 0, false>(S, sh, y, r);
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
static int launch_sdf_t(const SceneDev& s, int xp_filter, const int32_t* ids, const float* poses, const float* pts,
                        int64_t B, int64_t P, float* d, float* g, float* h, float* dp, float* d2p, float* dxp,
                        cudaStream_t st) {
  const int threads = 256;
  int64_t N = B * P;
  int64_t blocks = (N + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_sdf_eval<O, XP, PG, PH><<<(unsigned)blocks, threads, 0, st>>>(s, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp,
                                                                   xp_filter);
  return check_launch("k_sdf_eval");
}

template <int XP>
static int dispatch_sdf(const SceneDev& s, int xp_filter, const int32_t* ids, const float* poses, const float* pts,
                        int64_t B, int64_t P, uint32_t flags, float* d, float* g, float* h, float* dp, float* d2p,
                        float* dxp, cudaStream_t st) {
  const bool PG = flags & CM_SDF_POSE_GRAD, PH = flags & CM_SDF_POSE_HESS;
  const int O = (flags & (CM_SDF_HESS | CM_SDF_POSE_HESS)) ? 2 : ((flags & (CM_SDF_GRAD | CM_SDF_POSE_GRAD)) ? 1 : 0);
  if (O == 0) return launch_sdf_t<0, XP, false, false>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  if (O == 1) {
    if (PG) return launch_sdf_t<1, XP, true, false>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
    return launch_sdf_t<1, XP, false, false>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  }
  if (PG && PH) return launch_sdf_t<2, XP, true, true>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  if (PG) return launch_sdf_t<2, XP, true, false>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  if (PH) return launch_sdf_t<2, XP, false, true>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
  return launch_sdf_t<2, XP, false, false>(s, xp_filter, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st);
}

namespace cml {

int launch_sdf_eval(const SceneDev& s, int class_mask, const int32_t* ids, const float* poses, const float* pts,
                    int64_t B, int64_t P, uint32_t flags, float* d, float* g, float* h, float* dp, float* d2p,
                    float* dxp, void* stream) {
  // class_mask bit c: the scene has SDF shapes of class c (0 SQ family, 1
  // constant-schedule XPSQ, 2 varying-schedule XPSQ); one instantiation per
  // present class, each filtering its own shapes when several are present
  cudaStream_t st = (cudaStream_t)stream;
  const bool multi = (class_mask & (class_mask - 1)) != 0;
  int rc = CM_OK;
  if (class_mask & 1) rc = dispatch_sdf<0>(s, multi ? 0 : -1, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, st);
  if (!rc && (class_mask & 2))
    rc = dispatch_sdf<1>(s, multi ? 1 : -1, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, st);
  if (!rc && (class_mask & 4))
    rc = dispatch_sdf<2>(s, multi ? 2 : -1, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, st);
  // nested SQ-family shapes: general interpreter, no XPSQ code
  if (!rc && (class_mask & 8))
    rc = dispatch_sdf<3>(s, multi ? 3 : -1, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, st);
  return rc;
}

}  // namespace cml
