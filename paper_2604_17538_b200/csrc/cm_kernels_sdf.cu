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
#include "cm_param.cuh"
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
#ifndef CM_SDF_CHUNK
#define CM_SDF_CHUNK 1024   // points per work item of the dynamic (multi-class) sdf_eval schedule
#endif
#ifndef CM_SDF_THREADS
#define CM_SDF_THREADS 64   // threads per sdf_eval block (the grid keeps 148 x 16 x 256 threads): 64 +4.8% on
                            // the SDF workload over 256 (a block holds its SM slots until its slowest warp ends)
#endif
template <int O, int XP, bool PG, bool PH, bool DYN>
__global__ void __launch_bounds__(CM_SDF_THREADS, ((XP == 1 || XP == 2 || XP == 4) ? CM_SDF_MINB_XP : CM_SDF_MINB) * (256 / CM_SDF_THREADS)) k_sdf_eval(SceneDev S, const int32_t* __restrict__ shape_ids,
                                                  const float* __restrict__ poses, const float* __restrict__ points,
                                                  int64_t B, int64_t P, float* __restrict__ d,
                                                  float* __restrict__ grad, float* __restrict__ hess,
                                                  float* __restrict__ dpose, float* __restrict__ d2pose,
                                                  float* __restrict__ dxdpose, int xp_filter, int own_invalid,
                                                  unsigned long long* __restrict__ ctr) {
  const int64_t N = B * P;
  const bool n32 = N <= 0x7fffffff;   // 32-bit index arithmetic (no 64-bit division)
  // (warps walking 32-point segments with the class decided once per warp
  // measured -7.5% on the SDF workload, r02r)
  // work (DYN, the scene's multi-class launches): chunks of CM_SDF_CHUNK
  // points per warp taken from a device counter, so that warps whose chunks
  // hold few points of this class take more of them (the static walk leaves
  // warps idle behind the slowest of their block; r02zk); otherwise the
  // thread-level grid-stride walk (a separate instantiation: a warp
  // reconvergence point at every iteration costs the static walk 10%)
  const int lane = threadIdx.x & 31;
  int64_t cb = 0, ce = 0;   // DYN: the warp's current chunk [cb, ce) (warp-uniform)
  int64_t n = DYN ? 0 : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (;; n += DYN ? 0 : stride) {
    if constexpr (DYN) {
      if (cb >= ce) {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(ctr, (unsigned long long)CM_SDF_CHUNK);
        cb = (int64_t)__shfl_sync(0xffffffffu, b0, 0);
        ce = cb + CM_SDF_CHUNK;
        if (cb >= N) break;
        if (ce > N) ce = N;
      }
      n = cb + lane;
      cb += 32;
      if (n >= ce) continue;
    } else {
      if (n >= N) break;
    }
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
                        cudaStream_t st, unsigned long long* ctr) {
  const int threads = CM_SDF_THREADS;
  int64_t N = B * P;
  int64_t blocks = (N + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16 * (256 / CM_SDF_THREADS);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (ctr) {
    if (cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st) != cudaSuccess) return CM_ERR_CUDA;
    k_sdf_eval<O, XP, PG, PH, true><<<(unsigned)blocks, threads, 0, st>>>(s, ids, poses, pts, B, P, d, g, h, dp, d2p,
                                                                          dxp, xp_filter, own, ctr);
  } else {
    k_sdf_eval<O, XP, PG, PH, false><<<(unsigned)blocks, threads, 0, st>>>(s, ids, poses, pts, B, P, d, g, h, dp, d2p,
                                                                           dxp, xp_filter, own, nullptr);
  }
  return check_launch("k_sdf_eval");
}

template <int XP>
static int dispatch_sdf(const SceneDev& s, int xp_filter, int own, const int32_t* ids, const float* poses, const float* pts,
                        int64_t B, int64_t P, uint32_t flags, float* d, float* g, float* h, float* dp, float* d2p,
                        float* dxp, cudaStream_t st, unsigned long long* ctr) {
  const bool PG = flags & CM_SDF_POSE_GRAD, PH = flags & CM_SDF_POSE_HESS;
  const int O = (flags & (CM_SDF_HESS | CM_SDF_POSE_HESS)) ? 2 : ((flags & (CM_SDF_GRAD | CM_SDF_POSE_GRAD)) ? 1 : 0);
  if (O == 0) return launch_sdf_t<0, XP, false, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
  if (O == 1) {
    if (PG) return launch_sdf_t<1, XP, true, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
    return launch_sdf_t<1, XP, false, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
  }
  if (PG && PH) return launch_sdf_t<2, XP, true, true>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
  if (PG) return launch_sdf_t<2, XP, true, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
  if (PH) return launch_sdf_t<2, XP, false, true>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
  return launch_sdf_t<2, XP, false, false>(s, xp_filter, own, ids, poses, pts, B, P, d, g, h, dp, d2p, dxp, st, ctr);
}

namespace cml {

int launch_sdf_eval(const SceneDev& s, int class_mask, const int32_t* ids, const float* poses, const float* pts,
                    int64_t B, int64_t P, uint32_t flags, float* d, float* g, float* h, float* dp, float* d2p,
                    float* dxp, void* const* streams, int n_streams, unsigned long long* ctrs) {
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
    rc = dispatch_sdf<0>(s, multi ? 0 : -1, first == 0, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next(),
                         ctrs ? ctrs + 0 : nullptr);
  if (!rc && (class_mask & 2))
    rc = dispatch_sdf<1>(s, multi ? 1 : -1, first == 1, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next(),
                         ctrs ? ctrs + 1 : nullptr);
  if (!rc && (class_mask & 4))
    rc = dispatch_sdf<2>(s, multi ? 2 : -1, first == 2, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next(),
                         ctrs ? ctrs + 2 : nullptr);
  // nested SQ-family shapes: general interpreter, no XPSQ code
  if (!rc && (class_mask & 8))
    rc = dispatch_sdf<3>(s, multi ? 3 : -1, first == 3, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next(),
                         ctrs ? ctrs + 3 : nullptr);
  // constant-schedule XPSQ inside boolean trees
  if (!rc && (class_mask & 16))
    rc = dispatch_sdf<4>(s, multi ? 4 : -1, first == 4, ids, poses, pts, B, P, flags, d, g, h, dp, d2p, dxp, next(),
                         ctrs ? ctrs + 4 : nullptr);
  return rc;
}

}  // namespace cml

namespace {

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
    auto emit = [&](int kk, float v) {
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
    const int kcount = shape_param_grad(S, sh, y, emit);
    if (J)
      for (int kk = kcount; kk < pmax; ++kk) J[(int64_t)kk * N + n] = 0.f;
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
