// sm_100a support kernels of the manifold path (arXiv 2604.17538 §II-C):
//   k_face_counts + cub exclusive scan   per-pair output offsets
//   k_expand_jacobian                    fused 3x12 J from the compact (W, q)
//                                        form
// plus the launch bookkeeping shared by the kernel translation units
// (launch counter, last CUDA error, SM count).
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cub/device/device_scan.cuh>

#include "cm_internal.h"
#include "cm_launch.h"

using namespace cmi;

namespace {
std::atomic<int64_t> g_launches{0};
thread_local char g_cuda_msg[256];
}  // namespace

namespace cml {
void count_launch() { g_launches.fetch_add(1); }
void set_error(const char* msg) { snprintf(g_cuda_msg, sizeof(g_cuda_msg), "%s", msg); }
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  g_launches.fetch_add(1);
  if (e != cudaSuccess) {
    snprintf(g_cuda_msg, sizeof(g_cuda_msg), "%s: %s", what, cudaGetErrorString(e));
    return CM_ERR_CUDA;
  }
  return CM_OK;
}
int num_sms() {   // of the current device (cached per device)
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int n = cache[dev];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev] = n;
  }
  return n;
}

// ---- offsets: exclusive scan of F(shapeA) over the pairs ---------------------
// (a pair whose shape ids are out of range gets no rows and is counted in
// the scene's error word)
__global__ void k_face_counts(const ShapeRec* __restrict__ shapes, int32_t n_shapes, unsigned int* err,
                              const int32_t* __restrict__ pairs, int64_t n, uint32_t flags, int64_t* __restrict__ cnt) {
  const bool full = flags & CM_FULL_MODE, two = flags & CM_TWO_SIDED;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int ia = __ldg(pairs + 5 * i + 3), ib = __ldg(pairs + 5 * i + 4);
    if ((unsigned)ia >= (unsigned)n_shapes || (unsigned)ib >= (unsigned)n_shapes) {
      cnt[i] = 0;
      atomicAdd(err, 1u);
      continue;
    }
    const ShapeRec a = shapes[ia];
    int64_t c = full ? (int64_t)a.V + a.E : (int64_t)a.F;
    if (two) {
      const ShapeRec b = shapes[ib];
      c += full ? (int64_t)b.V + b.E : (int64_t)b.F;
    }
    cnt[i] = c;
  }
}

int64_t offsets_workspace(int64_t n_pairs) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)n_pairs);
  return (int64_t)bytes + 256;
}

int launch_offsets(const SceneDev& s, const int32_t* pairs, int64_t n_pairs, uint32_t flags, int64_t* offsets,
                   void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t blocks = (n_pairs + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) return CM_OK;
  k_face_counts<<<(unsigned)blocks, 256, 0, st>>>(s.shapes, s.n_shapes, s.err, pairs, n_pairs, flags, offsets);
  int rc = check_launch("k_face_counts");
  if (rc) return rc;
  size_t bytes = (size_t)ws_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(ws, bytes, offsets, offsets, (int)n_pairs, st);
  g_launches.fetch_add(1);
  if (e != cudaSuccess) {
    snprintf(g_cuda_msg, sizeof(g_cuda_msg), "offsets scan: %s", cudaGetErrorString(e));
    return CM_ERR_CUDA;
  }
  return CM_OK;
}

// ---- J expansion (App. A.7): J = [W I, -[q - W tA]x, -W I, [q - W tB]x] ------
__global__ void k_expand_jacobian(const ShapeRec* __restrict__ shapes, int32_t n_shapes,
                                  const int32_t* __restrict__ pairs, int64_t n_pairs,
                                  const int64_t* __restrict__ offsets, const float* __restrict__ poses, int64_t n_env,
                                  int32_t n_slot, const float* __restrict__ W, const float* __restrict__ q, int64_t C,
                                  float* __restrict__ J, uint32_t flags) {
  const bool full = flags & CM_FULL_MODE, two = flags & CM_TWO_SIDED;
  for (int64_t pi = blockIdx.x; pi < n_pairs; pi += gridDim.x) {
    const int32_t* pr = pairs + 5 * pi;
    // invalid records (counted by the offsets / manifold kernels): no J
    if ((unsigned)pr[3] >= (unsigned)n_shapes || (unsigned)pr[4] >= (unsigned)n_shapes ||
        (int64_t)(unsigned)pr[0] >= n_env || (unsigned)pr[1] >= (unsigned)n_slot || (unsigned)pr[2] >= (unsigned)n_slot)
      continue;
    const float* pa = poses + 8 * ((int64_t)pr[0] * n_slot + pr[1]);
    const float* pb = poses + 8 * ((int64_t)pr[0] * n_slot + pr[2]);
    int64_t off = offsets[pi];
    for (int side = 0; side < (two ? 2 : 1); ++side) {
      const ShapeRec sh = shapes[pr[3 + side]];
      const int nf = full ? sh.V + sh.E : sh.F;
      // side 1 samples B against A: its contact velocity is v_B - v_A, i.e.
      // J = -[W I, -[q - W tA]x, -W I, [q - W tB]x] in the pair's (A, B) order
      const float sg = side ? -1.f : 1.f;
      for (int f = threadIdx.x; f < nf; f += blockDim.x) {
        const int64_t c = off + f;
        const float w = W[c];
        const float qa[3] = {q[c] - w * pa[0], q[C + c] - w * pa[1], q[2 * C + c] - w * pa[2]};
        const float qb[3] = {q[c] - w * pb[0], q[C + c] - w * pb[1], q[2 * C + c] - w * pb[2]};
        const float Ka[3][3] = {{0.f, -qa[2], qa[1]}, {qa[2], 0.f, -qa[0]}, {-qa[1], qa[0], 0.f}};
        const float Kb[3][3] = {{0.f, -qb[2], qb[1]}, {qb[2], 0.f, -qb[0]}, {-qb[1], qb[0], 0.f}};
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            J[(r * 12 + k) * C + c] = sg * (r == k ? w : 0.f);
            J[(r * 12 + 3 + k) * C + c] = -sg * Ka[r][k];
            J[(r * 12 + 6 + k) * C + c] = sg * (r == k ? -w : 0.f);
            J[(r * 12 + 9 + k) * C + c] = sg * Kb[r][k];
          }
      }
      off += nf;
    }
  }
}

int launch_expand(const int32_t* pairs, int64_t n_pairs, const int64_t* offsets, const SceneDev& s,
                  const float* poses, int64_t n_env, int32_t n_slot, const float* W, const float* q, int64_t C,
                  float* J, uint32_t flags, void* stream) {
  int64_t grid = n_pairs < 65535 ? n_pairs : 65535;
  if (grid < 1) return CM_OK;
  k_expand_jacobian<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(s.shapes, s.n_shapes, pairs, n_pairs, offsets,
                                                                       poses, n_env, n_slot, W, q, C, J, flags);
  return check_launch("k_expand_jacobian");
}

// ---- pair-level reductions (SURVEY §8(b) optional outputs; §8(f) f4 VJP) ----
// One warp per pair (grid-stride), lanes over the pair's rows, shuffles for
// the reductions:
//   pair_depth = -tau LSE(-depth / tau) over the pair's contacts (smooth
//                minimum, the fusion's own depth operator, reading #25)
//   pair_W     = sum W
//   g_pose     = sum_rows (w_depth ddepth[:, row] + sum_k w_normal[k, row] dnormal[k, :, row])
//                (the vector-Jacobian product of the depths and normals with
//                respect to q = (dt_A, dtheta_A, dt_B, dtheta_B))
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(256) k_pair_reduce(const ShapeRec* __restrict__ shapes, int32_t n_shapes,
                                                     const int32_t* __restrict__ pairs, int64_t n_pairs,
                                                     const int64_t* __restrict__ offsets, uint32_t flags,
                                                     cm_manifold_out o, int64_t C, const float* __restrict__ w_depth,
                                                     const float* __restrict__ w_normal, float tau, float* pair_depth,
                                                     float* pair_W, float* g_pose) {
  const bool full = flags & CM_FULL_MODE, two = flags & CM_TWO_SIDED;
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float itl = 1.4426950408889634f / tau;
  for (int64_t pi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; pi < n_pairs; pi += warps) {
    const int ia = __ldg(pairs + 5 * pi + 3), ib = __ldg(pairs + 5 * pi + 4);
    int64_t n = 0;
    if ((unsigned)ia < (unsigned)n_shapes && (unsigned)ib < (unsigned)n_shapes) {
      const ShapeRec a = shapes[ia];
      n = full ? (int64_t)a.V + a.E : (int64_t)a.F;
      if (two) {
        const ShapeRec b = shapes[ib];
        n += full ? (int64_t)b.V + b.E : (int64_t)b.F;
      }
    }
    const int64_t r0 = __ldg(offsets + pi);
    if (pair_depth) {
      float m = -INFINITY;
      for (int64_t r = lane; r < n; r += 32) m = fmaxf(m, -o.depth[r0 + r]);
      m = warp_max(m);
      float z = 0.f;
      for (int64_t r = lane; r < n; r += 32) z += exp2f((-o.depth[r0 + r] - m) * itl);
      z = warp_sum(z);
      if (lane == 0) pair_depth[pi] = n > 0 ? -(m + tau * logf(z)) : __int_as_float(0x7fc00000);
    }
    if (pair_W) {
      float w = 0.f;
      for (int64_t r = lane; r < n; r += 32) w += o.W[r0 + r];
      w = warp_sum(w);
      if (lane == 0) pair_W[pi] = w;
    }
    if (g_pose) {
      float g[12];
#pragma unroll
      for (int j = 0; j < 12; ++j) g[j] = 0.f;
      for (int64_t r = lane; r < n; r += 32) {
        const int64_t c = r0 + r;
        const float wd = w_depth ? w_depth[c] : 0.f;
        const float wn[3] = {w_normal ? w_normal[c] : 0.f, w_normal ? w_normal[C + c] : 0.f,
                             w_normal ? w_normal[2 * C + c] : 0.f};
#pragma unroll
        for (int j = 0; j < 12; ++j) {
          float v = wd * o.ddepth[(int64_t)j * C + c];
#pragma unroll
          for (int k = 0; k < 3; ++k) v = fmaf(wn[k], o.dnormal[(int64_t)(k * 12 + j) * C + c], v);
          g[j] += v;
        }
      }
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        const float v = warp_sum(g[j]);
        if (lane == 0) g_pose[12 * pi + j] = v;
      }
    }
  }
}

int launch_pair_reduce(const SceneDev& s, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                       uint32_t flags, const cm_manifold_out* out, int64_t C, const float* w_depth,
                       const float* w_normal, float* pair_depth, float* pair_W, float* g_pose, void* stream) {
  int64_t blocks = (n_pairs * 32 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) return CM_OK;
  k_pair_reduce<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(s.shapes, s.n_shapes, pairs, n_pairs, offsets,
                                                                      flags, *out, C, w_depth, w_normal,
                                                                      s.sp.tau_min, pair_depth, pair_W, g_pose);
  return check_launch("k_pair_reduce");
}

const char* last_cuda_error() { return g_cuda_msg; }
int64_t launch_count() { return g_launches.load(); }

}  // namespace cml
