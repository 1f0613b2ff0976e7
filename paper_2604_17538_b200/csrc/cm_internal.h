// Internal layouts shared by the host library (cm_host.cpp) and the sm_100a
// kernels (cm_kernels_*.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>

#include "xpsq_cm.h"

namespace cmi {

// ---- shape program ---------------------------------------------------------
// A shape's SDF tree is flattened into a postfix-like program evaluated with a
// small stack of streaming LSE accumulators (one per open boolean node):
//   BEGIN        open an accumulator
//   LEAF k       evaluate leaf k, fold child_sign * result into the top
//   END          close the top: out_sign * LSE(...), fold child_sign * it
// Union: children -1, out -1 (-LSE(-phi), Eq. (2)); intersection +1, +1
// (Eq. (3)); subtraction (+1, -1), out +1 (Eq. (4)).
enum { OP_LEAF = 0, OP_BEGIN = 1, OP_END = 2 };
struct alignas(16) Instr {   // one 128-bit load per instruction
  int32_t op;
  int32_t idx;
  float child_sign;
  float out_sign;
};

enum { LK_HALFSPACE = 0, LK_SQ = 1, LK_XPSQ = 3 };

// Leaf record (SQ / PSQ / half-space; XPSQ points into Xpsq[xidx]).
// Frame: x_body = R y + t (composed down the tree on the host in FP64).
// 16-B aligned, field groups on 16-B boundaries: the kernels load a leaf with
// six 128-bit loads (cm_device.cuh ld_leaf) instead of 23 scalar ones.
struct alignas(16) Leaf {
  float R[9];
  float t[3];
  int32_t kind;
  int32_t n_planes;
  int32_t rot_identity;
  int32_t xidx;
  float ia[3];            // 1 / a
  float p1, p2, m, k;     // 1/eps1, 1/eps2, eps2/eps1, eps1/2
  float pad0;
  float planes[CM_MAX_PLANES][4];
  // XPSQ leaves: phi >= |x - cull[0..2]| - cull[3] for x in the shape frame
  // (the spline lies in its control points' hull: bounding sphere of their
  // box; |y| - |a|_max bounds the radial SQ distance; PSQ >= SQ; the 3-root
  // smooth minimum >= min - tau ln 3), used to skip leaves whose union
  // weight is below 2^-66
  float cull[4];
};
static_assert(sizeof(Leaf) % 16 == 0 && offsetof(Leaf, planes) == 96, "Leaf: 128-bit load layout");

// XPSQ static data: p(t) = p1 + B t + A t^2 (A := 0, B := p3 - p1
// for the snapped straight class), projection cubic constants in the affine form
//   P = gP . w + P0,  Q = gQ . w + Q0,  w = y - p1
// (c3, c2 depend only on the spline; c1, c0 are affine in w), b3 = b/3.
// 16-B aligned with the fields the projection and the evaluation read
// together in 16-B groups (the compiler merges them into 128-bit loads)
struct alignas(16) Xpsq {
  float p1[3], P0;
  float gP[3], Q0;
  float gQ[3], b3;
  float A[3], c3;         // the cubic in t: c3 t^3 + c2 t^2 + (2 A.w - BB) t + B.w
  float B[3], c2;
  float Bn[3], BB;        // straight class: t = softclip(Bn . w)
  float bhat[3];          // Frenet binormal (constant for a quadratic)
  int32_t cls;            // 0 point, 1 straight, 2 curve
  int32_t frenet;
  int32_t varying;        // schedules differ between the endpoints
  int32_t n_planes;
  int32_t pad0;
  float sq_ia[3], sq_p1;  // SQ constants of the t = 0 schedule
  float sq_p2, sq_m, sq_k, pad1;
  float R0[9];            // constant frame (straight / point / A || B)
  float up[3];            // the up hint (control-point derivatives of the constant frame, f4)
  float eps0[2], deps[2];
  float a0[3], pad2;
  float da[3], pad3;
  float pl0[CM_MAX_PLANES][4], dpl[CM_MAX_PLANES][4];
};
static_assert(sizeof(Xpsq) % 16 == 0 && offsetof(Xpsq, pl0) % 16 == 0 && offsetof(Xpsq, sq_ia) % 16 == 0,
              "Xpsq: 128-bit load layout");

struct ShapeRec {
  int32_t prog_begin, prog_len;
  // SDF class (one kernel instantiation each): 0 SQ family with nesting depth
  // <= 1, 1 a lone constant-schedule XPSQ, 2 varying-schedule XPSQ, 3 SQ
  // family with nested booleans, 4 constant-schedule XPSQ in a boolean tree
  int32_t has_sdf, uses_xpsq;
  int32_t V, E, F;
  int32_t v_off, e_off, f_off;   // into verts (x3), edges (x2), faces / face_edges (x3)
  int32_t pad;
};

struct SmoothDev {
  float tau_cmp, tau_min, tau_clip_alpha, tau_clip_t, tau_delta;
  int32_t iters;
  float i_cmp, i_min, i_clip_alpha, i_clip_t, i_delta;   // reciprocals (host-computed)
};

// everything a kernel needs to evaluate any shape of the scene
// node-pose derivatives (f4, reading #47): per program op (BEGIN / LEAF; END
// unused) the node's index in its shape description, the composed frame of
// its parent in the shape frame (x_shape = RP x_parent + tP) and the node's
// own pose translation tk (in the parent frame)
struct alignas(16) NodeFrame {
  float RP[9];
  float tP[3];
  float tk[3];
  int32_t node;
};
static_assert(sizeof(NodeFrame) == 64, "NodeFrame: 64 B");

struct SceneDev {
  const Instr* prog;
  const NodeFrame* op_frames; // parallel to prog
  const Leaf* leaves;
  const Xpsq* xpsq;
  const ShapeRec* shapes;
  const float* verts;         // sampled-surface vertices, 4 floats each (x, y, z, 0)
  const int32_t* edges;
  const float* edge_geom;     // per edge 8 floats: x_I[3], L, e_t[3] (unit, local), 0
  const int32_t* faces;
  const int32_t* face_edges;
  SmoothDev sp;
  int32_t n_shapes;
  unsigned int* err;          // device counter of invalid pair records / shape ids (cm_scene_error_count)
  const int8_t* shape_cls;    // per shape: its SDF class (ShapeRec::uses_xpsq), -1 without an SDF
  int32_t n_leaves, n_xpsq;   // sizes of leaves[] and xpsq[] (shared-memory staging)
  const float4* bounds;       // broad phase (f2): [2 s] sampled-vertex sphere (c, r), [2 s + 1] SDF bound (c, rho)
};

// manifold chunk scratch: the units of one chunk keep their candidate state
// in a global slot each; the scene allocates kChunkUnits slots (capped at
// kScratchCapBytes) at creation (CM_CHUNK_UNITS overrides the unit count)
constexpr int64_t kChunkUnits = 262144;   // C5 +5%, C4 +2% over 32768 (r02q sweep; 4-7 GB of scratch)
#ifndef CM_N_AUX_STREAMS
#define CM_N_AUX_STREAMS 2
#endif
constexpr int kManifoldStreams = CM_N_AUX_STREAMS;   // chunks alternate between the scene's aux streams
constexpr int64_t kScratchCapBytes = 8192ll << 20;

// shape-parameter derivatives (f4): boolean nodes of one shape the
// parameter kernel tracks per point (shapes with more report count -1)
constexpr int kParamMaxNodes = 16;

}  // namespace cmi

// launchers implemented in cm_kernels_*.cu
namespace cml {
int launch_sdf_eval(const cmi::SceneDev& s, int class_mask, const int32_t* shape_ids, const float* poses,
                    const float* points, int64_t B, int64_t P, uint32_t flags, float* d, float* grad, float* hess,
                    float* dpose, float* d2pose, float* dxdpose, void* const* streams, int n_streams,
                    unsigned long long* ctrs = nullptr);
int launch_manifold(const cmi::SceneDev& s, int class_mask, int max_V, int max_E, const int32_t* pairs,
                    int64_t n_pairs, const int64_t* offsets, const float* poses, int64_t n_env, int32_t n_slot,
                    uint32_t flags,
                    const cm_manifold_out* out, int64_t C, float* scratch, int64_t scratch_floats,
                    void* const* streams, int n_streams);
int launch_offsets(const cmi::SceneDev& s, const int32_t* pairs, int64_t n_pairs, uint32_t flags, int64_t* offsets,
                   void* ws, int64_t ws_bytes, void* stream);
int64_t offsets_workspace(int64_t n_pairs);
int launch_expand(const int32_t* pairs, int64_t n_pairs, const int64_t* offsets, const cmi::SceneDev& s,
                  const float* poses, int64_t n_env, int32_t n_slot, const float* W, const float* q, int64_t C,
                  float* J, uint32_t flags, void* stream);
int64_t manifold_slot_floats(int V, int E, int tier);
int launch_pair_reduce(const cmi::SceneDev& s, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                       uint32_t flags, const cm_manifold_out* out, int64_t C, const float* w_depth,
                       const float* w_normal, float* pair_depth, float* pair_W, float* g_pose, void* stream);
int launch_manifold_param_vjp(const cmi::SceneDev& s, int max_V, int max_E, int pmax, const int32_t* pairs,
                              int64_t n_pairs, const int64_t* offsets, const float* poses, int64_t n_env,
                              int32_t n_slot, uint32_t mode, const float* w, float* vjp, const int64_t* poff,
                              void* stream);
int launch_sdf_node_pose_grad(const cmi::SceneDev& s, const int32_t* ids, const float* poses, const float* pts,
                              int64_t B, int64_t P, int32_t nmax, float* J, const float* w, float* vjp,
                              const int64_t* noff, void* stream);
int launch_sdf_param_grad(const cmi::SceneDev& s, const int32_t* ids, const float* poses, const float* pts, int64_t B,
                          int64_t P, int32_t pmax, float* J, const float* w, float* vjp, const int64_t* poff,
                          void* stream);
const char* last_cuda_error();
int64_t launch_count();
}  // namespace cml
