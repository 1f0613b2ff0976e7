/*
 * xpsq_cm.h — C ABI of the B200 (sm_100a) XPSQ SDF + smooth contact-manifold
 * library (arXiv 2604.17538, "XPSQ analytical SDF primitives and smooth
 * one-shot contact manifolds").
 *
 * Citations: P:n = PAPER.md line n (section / equation named in brackets).
 *
 * Two compute entry points follow the paper's statement of the problem:
 *   cm_sdf_eval         sdf_eval(prims, poses, points) -> d, grad d, hess d
 *                       (+ derivatives with respect to the poses)
 *                       [§II-B, Eq. (1)-(6), P:52-126]
 *   cm_contact_manifold contact_manifold(pairs, poses) -> points, normals,
 *                       depths, Jacobians (+ pose derivatives)
 *                       [§II-C, P:129-163]
 *
 * Conventions
 *   - Ownership: the scene (shape library, sampled-surface topology, device
 *     copies) is owned by the library behind the opaque cm_scene handle and is
 *     immutable after creation.  Every batch input and output of a compute
 *     call is a CALLER-OWNED DEVICE pointer (e.g. a torch tensor's data_ptr());
 *     compute calls perform no allocation and no host<->device copy.
 *   - Streams: compute calls take a cudaStream_t (passed as void*) and return
 *     as soon as the work is enqueued; NULL means the legacy default stream.
 *   - Errors: every function returns 0 (CM_OK) or a negative cm_status; the
 *     message of the last failure on the calling thread is cm_last_error().
 *     No C++ exception crosses the ABI.  Non-finite per-element inputs
 *     propagate NaN into that element's outputs and do not fail the call.
 *   - Poses: 8 floats per body: t = (x, y, z), unit quaternion q = (w, x, y, z)
 *     (normalised by the library), 1 pad float.  A point x_local of a body is
 *     at R(q) x_local + t in the world.
 *   - Pose derivatives use world-frame left perturbations (twists): for a body
 *     with pose (R, t), R <- exp([dtheta]x) R and t <- t + dt, coordinates
 *     ordered (dt_x, dt_y, dt_z, dtheta_x, dtheta_y, dtheta_z).
 *   - Sign convention: phi < 0 inside, > 0 outside ("gamma = [[d < 0]]").
 *   - Thread safety: calls on distinct streams may run concurrently.
 *     cm_contact_manifold uses the scene's chunk scratch (allocated at scene
 *     creation): concurrent manifold calls on ONE scene are enqueued under a
 *     per-scene lock and serialised on the device through the scene's two
 *     internal streams (forked from and joined back into the caller's stream
 *     with events, so stream capture into a CUDA graph works); calls on
 *     distinct scenes run concurrently.
 */
#ifndef XPSQ_CM_H
#define XPSQ_CM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CM_ABI_VERSION 6
#define CM_MAX_PLANES 8      /* half-spaces per PSQ / XPSQ cross-section      */
#define CM_MAX_CHILDREN 32   /* children per boolean node                     */
#define CM_MAX_DEPTH 3       /* nesting of boolean nodes in one shape         */

typedef enum cm_status {
  CM_OK = 0,
  CM_ERR_INVALID = -1,     /* bad argument, NULL pointer, bad index          */
  CM_ERR_NONFINITE = -2,   /* non-finite shape parameter                     */
  CM_ERR_UNSUPPORTED = -3, /* unsupported kind / depth / size                */
  CM_ERR_ARITY = -4,       /* boolean arity (subtraction 2, others >= 2)     */
  CM_ERR_EMPTY = -5,       /* empty input where one is required              */
  CM_ERR_CUDA = -6,        /* CUDA runtime error (message has the detail)    */
  CM_ERR_OOM = -7          /* device allocation failed at scene creation     */
} cm_status;

/* SDF node kinds.  Leaves: HALFSPACE phi = y.n + h; SQ radial
 * distance from the inside-outside function of Eq. (1); PSQ = smooth
 * intersection (Eq. (3)) of an SQ and N half-spaces; XPSQ = a PSQ swept
 * along a quadratic spline (Eq. (5)).  Operators (Eq. (2)-(4),
 * P:78-83): UNION -LSE(-phi_i), INTERSECTION LSE(phi_i) (n-ary, one LSE),
 * SUBTRACTION LSE(phi_1, -phi_2) (binary). */
typedef enum cm_node_type {
  CM_HALFSPACE = 0,
  CM_SQ = 1,
  CM_PSQ = 2,
  CM_XPSQ = 3,
  CM_UNION = 10,
  CM_INTERSECTION = 11,
  CM_SUBTRACTION = 12
} cm_node_type;

/* One node of a shape's SDF tree; node 0 is the root.  Every node carries a
 * pose relative to its parent (the root's is relative to the body frame).
 * Leaf parameters ([e] = endpoint 0/1 of the XPSQ schedules; SQ, PSQ
 * and HALFSPACE use endpoint 0 only):
 *   eps[e] = (eps1, eps2) in [0.1, 2]; a[e] = (a_x, a_y, a_z) > 0;
 *   planes[e][j] = (n_x, n_y, n_z, h), |n| = 1, inside where n.y + h <= 0;
 *   HALFSPACE uses planes[0][0];
 *   XPSQ: ctrl = p1, p2, p3 (Eq. (5)); up = up hint for straight/point
 *   splines (the frame of a curved spline is its Frenet frame). */
typedef struct cm_node {
  int32_t type;                       /* cm_node_type                          */
  int32_t n_children;                 /* operators only                        */
  int32_t children[CM_MAX_CHILDREN];  /* node indices (> own index)            */
  int32_t n_planes;                   /* PSQ / XPSQ (HALFSPACE: 1)             */
  float pose[7];                      /* t(3), q(w,x,y,z) in the parent frame  */
  float eps[2][2];
  float a[2][3];
  float planes[2][CM_MAX_PLANES][4];
  float ctrl[9];
  float up[3];
} cm_node;

/* A shape: optional SDF (n_nodes > 0) and optional sampled surface (the
 * paper's mesh side): local-frame vertices [V,3] and triangles [F,3]
 * (int32 vertex indices).  Host pointers, copied at scene creation.  With
 * n_faces == 0 and sample_res > 0 the library tessellates the shape's single
 * SQ / PSQ / XPSQ node itself (cm_tessellate, placed by the node's pose):
 * SURVEY §8(b) `sample_res`. */
typedef struct cm_shape_desc {
  int32_t n_nodes;
  const cm_node* nodes;
  int32_t n_vertices;
  const float* vertices;
  int32_t n_faces;
  const int32_t* faces;
  int32_t sample_res;
} cm_shape_desc;

/* Library-side sampled surface of one SQ / PSQ / XPSQ node in its own frame
 * (host; SURVEY §8(b) sample_res): SQ a cube-sphere with res x res
 * cells per face on the parametric surface of Eq. (1) (V = 6 res^2 + 2,
 * F = 12 res^2); PSQ the same with the vertices outside each plane pulled
 * radially onto it (planes must keep the centre inside: h < 0); XPSQ a tube
 * of 2 res + 1 rings x 4 res points on the t = 0 cross-section along the
 * spline (Eq. (5)) plus two end caps (V = 4 res (2 res + 1) + 2).  Endpoint-0
 * schedules.  n_vertices / n_faces (host) receive the counts; vertices
 * [3V] and faces [3F] (host) are filled when both are non-NULL (size them by
 * a first call with NULL).  CM_ERR_INVALID (bad node / res outside
 * [1, 256]), CM_ERR_UNSUPPORTED (half-space, boolean node, point spline). */
int cm_tessellate(const cm_node* node, int32_t res, float* vertices, int32_t* faces, int32_t* n_vertices,
                  int32_t* n_faces);

/* Temperatures of the smooth operators (§II-A; one generic tau in
 * the paper, five named ones here — DESIGN.md reading #1), all > 0:
 *   tau_cmp         gamma gate and sphere-trace gate
 *   tau_min         boolean LSE, XPSQ smooth-min, depth softmax
 *   tau_clip_alpha  soft clip of traced edge parameters
 *   tau_clip_t      soft clip of the spline roots
 *   tau_delta       soft Cardano discriminant gate
 *   trace_iters     sphere-trace iterations per edge corner (3)      */
typedef struct cm_smooth_params {
  float tau_cmp, tau_min, tau_clip_alpha, tau_clip_t, tau_delta;
  int32_t trace_iters;
} cm_smooth_params;

typedef struct cm_scene cm_scene;

int cm_version(void);
const char* cm_last_error(void);

/* Validates and packs the shapes, builds each sampled surface's unique edges
 * (sorted vertex pairs) and face->edge incidence, copies everything to
 * device `device`.  Errors: CM_ERR_INVALID (bad index, degenerate edge,
 * |n| != 1), CM_ERR_NONFINITE, CM_ERR_ARITY, CM_ERR_UNSUPPORTED (depth >
 * CM_MAX_DEPTH, > CM_MAX_PLANES), CM_ERR_OOM, CM_ERR_CUDA. */
int cm_scene_create(const cm_shape_desc* shapes, int32_t n_shapes, const cm_smooth_params* sp, int device,
                    cm_scene** out);
int cm_scene_destroy(cm_scene* scene);

/* V, E, F of shape `shape`'s sampled surface (0 if it has none). */
int cm_shape_counts(const cm_scene* scene, int32_t shape, int32_t* V, int32_t* E, int32_t* F);
/* Host copy of the topology the library built: edges [E,2] (lower index
 * first), face_edges [F,3] (edges (i0,i1), (i1,i2), (i2,i0)). */
int cm_shape_topology(const cm_scene* scene, int32_t shape, int32_t* edges, int32_t* face_edges);

/* ---- sdf_eval --------------------------------------------------------------
 * For batch item b in [0,B): shape shape_ids[b] placed at poses[b*8 .. +8];
 * for its P query points n = b*P + j (world, points[n*3 .. +3]) computes the
 * outputs selected by `flags` (SoA, N = B*P, field-major):
 *   d[N]         phi (CM_SDF_VALUE)
 *   grad[3*N]    d phi / d x                            (CM_SDF_GRAD)
 *   hess[6*N]    xx, xy, xz, yy, yz, zz                 (CM_SDF_HESS)
 *   dpose[6*N]   d phi / d(dt, dtheta)                  (CM_SDF_POSE_GRAD)
 *   d2pose[21*N] packed upper triangle of the 6x6 pose Hessian, row-major
 *                                                       (CM_SDF_POSE_HESS)
 *   dxdpose[18*N] [i*6+j] = d (grad_i) / d pose_j       (CM_SDF_POSE_HESS)
 * Unselected outputs may be NULL.  All pointers are device pointers. */
#define CM_SDF_VALUE 1u
#define CM_SDF_GRAD 2u
#define CM_SDF_HESS 4u
#define CM_SDF_POSE_GRAD 8u
#define CM_SDF_POSE_HESS 16u
int cm_sdf_eval(const cm_scene* scene, const int32_t* shape_ids, const float* poses, const float* points, int64_t B,
                int64_t P, uint32_t flags, float* d, float* grad, float* hess, float* dpose, float* d2pose,
                float* dxdpose, void* stream);

/* ---- shape-parameter derivatives ------------------------
 * Parameters of shape s, in the order of its SDF nodes (pre-order, as given
 * to cm_scene_create), endpoint-0 values: half-space (n_x, n_y, n_z, h); SQ
 * (a_x, a_y, a_z, eps1, eps2); PSQ as SQ then (n_x, n_y, n_z, h) per plane;
 * XPSQ with constant schedules as PSQ (its cross-section; each parameter
 * moves both endpoint values, normals renormalised as in the XPSQ); XPSQ
 * with varying schedules: the PSQ slots of the t = 0 endpoint, then those of
 * the t = 1 endpoint (schedules linear in t, P:108 / reading #8); every XPSQ
 * then the 9 control-point slots p1, p2, p3 (Eq. (5): through the
 * projection roots, the frame and p(t); within the spline's static class --
 * a straight spline's p2 has no effect, its chord is p1 -> p3); boolean nodes have none (a PSQ's raw plane
 * normal is the parameter: no renormalisation).  counts[s] (host,
 * [n_shapes]) = the count, 0 without an SDF, -1 when the shape has more
 * than 16 boolean nodes, or leaves whose node indices are not in
 * depth-first (pre-order) order (not parametrised);
 * booleans nested up to CM_MAX_DEPTH are parametrised (chain rule through
 * every enclosing LSE, Eqs. (2)-(4)); offsets (host, [n_shapes + 1]) = prefix sums of
 * max(count, 0) (the layout of the vjp vector).  Either may be NULL. */
int cm_param_layout(const cm_scene* scene, int32_t* counts, int64_t* offsets);
/* For each point n (layout of cm_sdf_eval): J[k*N + n] = d phi(n) / d param k
 * of point n's shape for k < pmax (zero beyond the shape's count), and
 * vjp[offsets[s] + k] += sum over the points n of shape s of w[n] J[k, n]
 * (device, accumulated: zero it first; FP32 atomics, warp-reduced when a
 * warp's points share one shape, so the summation order is not fixed).
 * J or vjp may be NULL (not both; vjp needs w).  CM_ERR_UNSUPPORTED when any
 * SDF shape of the scene has count -1. */
int cm_sdf_param_grad(const cm_scene* scene, const int32_t* shape_ids, const float* poses, const float* points,
                      int64_t B, int64_t P, int32_t pmax, float* J, const float* w, float* vjp, void* stream);

/* ---- node-pose derivatives (DESIGN reading #47) ----------
 * Node poses as shape parameters (fitting needs d/d shape; the paper
 * defines no parametrisation): six slots per SDF node of shape s, for the
 * nodes in the order of its description (every boolean node and leaf, the
 * root included; a node unreachable from the root has zero slots' values):
 * the twist (dt_x, dt_y, dt_z, dtheta_x, dtheta_y, dtheta_z) of the node's
 * pose (R, t) in its PARENT's frame (the root's: the body frame) with the
 * body poses' convention, R <- exp([dtheta]x) R and t <- t + dt, where
 * x_parent = R x_node + t.  counts[s] (host, [n_shapes]) = 6 x the shape's
 * node count, 0 without an SDF, -1 with more than 16 boolean nodes (not
 * parametrised); offsets (host, [n_shapes + 1]) = prefix sums of
 * max(count, 0).  Either may be NULL. */
int cm_node_pose_layout(const cm_scene* scene, int32_t* counts, int64_t* offsets);
/* For each point n (layout of cm_sdf_eval): J[k*N + n] = d phi(n) / d slot k
 * of point n's shape for k < nmax (zero beyond 6 x its node count), and
 * vjp[offsets[s] + k] += sum over the points n of shape s of w[n] J[k, n]
 * (device, accumulated: zero it first; FP32 atomics, warp-reduced when a
 * warp's points share one shape: the summation order is not fixed).  J or
 * vjp may be NULL (not both; vjp needs w).  Invalid shape ids: NaN rows,
 * counted in cm_scene_error_count.  CM_ERR_UNSUPPORTED when any SDF shape of
 * the scene has count -1. */
int cm_sdf_node_pose_grad(const cm_scene* scene, const int32_t* shape_ids, const float* poses, const float* points,
                          int64_t B, int64_t P, int32_t nmax, float* J, const float* w, float* vjp, void* stream);

/* ---- contact manifold ------------------------------------------------------
 * pairs[5*i ..]: {env, slotA, slotB, shapeA (sampled surface), shapeB (SDF)}
 * (device int32); poses [n_env, n_slot, 8] (device).  One-sided reduced
 * manifold: one fused contact per face of shapeA's surface.
 * Contacts of pair i occupy rows [offsets[i], offsets[i] + F(shapeA_i)) of
 * every output array (offsets: device int64, e.g. from cm_manifold_offsets);
 * n_contacts = C, the total (cm_manifold_size), is the stride of the fields.
 * Outputs (device, field-major SoA over C contacts; a field is written iff its
 * tier is selected, lower-tier fields are always written):
 *   tier 0: point[3C] (sum z_i p_i, reporting only), normal[3C] (raw
 *           fused sum z_i gamma_i n_i), depth[C] (smooth min of the
 *           candidate depths), dom[C] (argmax z_i gamma_i, int8)
 *   tier 1: W[C] = sum z_i gamma_i and q[3C] = sum z_i gamma_i p_i: the fused
 *           3x12 contact Jacobian sum z_i gamma_i J_i is exactly
 *           [W I, -[q - W tA]x, -W I, [q - W tB]x] (cm_expand_jacobian)
 *   tier 2: ddepth[12C] and dnormal[36C] ([i*12+j] = d n_i / d q_j): the
 *           derivatives with respect to q = (dt_A, dtheta_A, dt_B, dtheta_B)
 *   tier 3: d2depth[78C]: the second derivatives d^2 depth / dq_i dq_j, packed
 *           upper triangle i <= j in row order ((0,0), (0,1), .., (0,11),
 *           (1,1), ..), field k at d2depth[k*C + row] (
 *           P:8 motivates Hessians for second-order control).  Full mode:
 *           of the candidate's phi. */
#define CM_TIER0 0u
#define CM_TIER1 1u
#define CM_TIER2 2u
#define CM_TIER3 3u
#define CM_TIER_MASK 3u
/* CM_FULL_MODE: one contact per vertex and per edge of the sampled
 * surface (V + E rows, vertices first, then edges in cm_shape_topology order)
 * instead of one fused contact per face.  Row i is candidate i itself: point,
 * raw normal grad phi, depth phi, W = gamma = sigma(-phi/tau_cmp), q = gamma p
 * (J = gamma J_i), dom = 0 vertex / 1 edge point; tier-2 derivatives of
 * phi and grad phi.
 * CM_TWO_SIDED: the manifold of A sampled against B's SDF followed by
 * the manifold of B sampled against A's SDF (both shapes of every pair need an
 * SDF and a sampled surface); derivative columns of both halves are in the
 * pair's own order (t_A, theta_A, t_B, theta_B). */
#define CM_FULL_MODE 4u
#define CM_TWO_SIDED 8u
/* CM_BROAD_PHASE ("utilizing [a broad phase] to filter
 * edges prior to passing them to the edge-SDF routine"): a (pair, side) whose
 * certified bound lb = |c_A - c_B| - r_A - rho_B on every candidate depth
 * exceeds 40 tau_cmp (every gate below e^-40) skips the traces, evaluations
 * and fusion.  (c_A, r_A): the sampled vertices' bounding sphere; phi_B >=
 * |x - c_B| - rho_B from the SDF tree (shapes containing an unbounded
 * half-space operand are never culled).  Its rows: point = the face centroid
 * (full mode: the vertex / edge midpoint), depth = lb - tau_min ln 6 (full
 * mode: lb), a certified lower bound of the fused depth; normal, W, q and
 * every derivative 0; dom = -2.  Kept pairs are bit-identical to the call
 * without the flag (reading #46). */
#define CM_BROAD_PHASE 16u

typedef struct cm_manifold_out {
  float* point;
  float* normal;
  float* depth;
  float* W;
  float* q;
  float* ddepth;
  float* dnormal;
  int8_t* dom;
  float* d2depth;   /* tier 3 only (may be NULL below tier 3) */
} cm_manifold_out;

/* Number of contacts of a pair list given on the HOST (pairs_host [n,5]) for
 * the mode bits of `flags` (CM_FULL_MODE, CM_TWO_SIDED); also validates that
 * every pair's sampled shape has a surface and its SDF shape an SDF (both, on
 * both shapes, with CM_TWO_SIDED) -> CM_ERR_INVALID otherwise. */
int cm_manifold_size(const cm_scene* scene, const int32_t* pairs_host, int64_t n_pairs, uint32_t flags,
                     int64_t* n_contacts);
/* Device exclusive scan of the per-pair contact counts (same mode bits) ->
 * offsets[n_pairs] (device int64).  Uses `workspace` of
 * cm_manifold_offsets_workspace() bytes (device, caller-owned). */
int64_t cm_manifold_offsets_workspace(int64_t n_pairs);
int cm_manifold_offsets(const cm_scene* scene, const int32_t* pairs, int64_t n_pairs, uint32_t flags, int64_t* offsets,
                        void* workspace, int64_t workspace_bytes, void* stream);
int cm_contact_manifold(const cm_scene* scene, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                        const float* poses, int64_t n_env, int32_t n_slot, uint32_t flags,
                        const cm_manifold_out* out, int64_t n_contacts, void* stream);

/* Expands the compact Jacobian: J[36*C] ([r*12+c], device) from W, q and the
 * pairs' poses, for the layout of the same mode bits (`flags`).  Rows of the
 * transposed half of CM_TWO_SIDED carry the opposite sign (their contact
 * velocity is v_B - v_A). */
int cm_expand_jacobian(const cm_scene* scene, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                       const float* poses, int64_t n_env, int32_t n_slot, uint32_t flags, const float* W,
                       const float* q, int64_t n_contacts, float* J, void* stream);

/* Shape-parameter vector-Jacobian product of the manifold depths (SURVEY
 * §8f row f4 "reverse-mode VJPs"; DESIGN reading #48): vjp[po[s] + k] +=
 * sum over the rows r of every pair whose SDF shape is s of
 * w_depth[r] d depth_r / d theta_k, theta = the parameters of shape s in the
 * cm_param_layout order (po its offsets).  Everything the manifold derives
 * from phi_s is differentiated: the candidate values, the sphere-trace
 * iterates and soft clips, the edge points and the face softmax
 * (P:158-161); the sampled surface is data.  pairs / offsets / poses /
 * n_env / n_slot as for cm_contact_manifold with the same flags (reduced or
 * CM_FULL_MODE: the rows' candidate depths; CM_TWO_SIDED: each half with
 * respect to its own SDF shape, B then A; CM_BROAD_PHASE: culled rows add
 * nothing); CM_ERR_UNSUPPORTED when a shape is not parametrised or with more
 * than 16 trace iterations.  w_depth [C] and vjp (accumulated: zero it
 * first; FP32 atomics, order not fixed) are device pointers.  Invalid pair
 * records are skipped (counted by cm_contact_manifold's validation rules). */
int cm_manifold_param_vjp(const cm_scene* scene, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                          const float* poses, int64_t n_env, int32_t n_slot, uint32_t flags, const float* w_depth,
                          float* vjp, void* stream);

/* Pair-level reductions of a manifold computed with the same mode bits
 * (`flags`; rows of pair i at [offsets[i], offsets[i] + its contact count)),
 * one warp per pair with shuffle reductions (SURVEY §8(b) optional outputs,
 * §8(f) f4 reverse mode).  Every output is device [n_pairs] (g_pose
 * [12 * n_pairs]) and may be NULL:
 *   pair_depth[i] = -tau_min log sum exp(-depth / tau_min) over the pair's
 *                   contacts (the smooth minimum of the fusion, P:161 and
 *                   DESIGN.md reading #25); NaN for a pair without contacts
 *   pair_W[i]     = sum of W (needs tier >= 1 outputs)
 *   g_pose[12 i + j] = sum over the pair's rows of w_depth[row] ddepth[j, row]
 *                   + sum_k w_normal[k, row] dnormal[k*12 + j, row]: the
 *                   vector-Jacobian product of the depths and raw normals with
 *                   respect to q = (dt_A, dtheta_A, dt_B, dtheta_B) (needs
 *                   tier-2 outputs; w_depth [C] and w_normal [3C] device, either
 *                   may be NULL).
 * Errors: CM_ERR_INVALID (NULL where an output needs it), CM_ERR_CUDA. */
int cm_manifold_pair_reduce(const cm_scene* scene, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                            uint32_t flags, const cm_manifold_out* out, int64_t n_contacts, const float* w_depth,
                            const float* w_normal, float* pair_depth, float* pair_W, float* g_pose, void* stream);

/* Number of kernel launches the library issued since scene creation (all
 * scenes, this process) — instrumentation for bench.py's gpu_launches. */
int64_t cm_launch_count(void);

/* Invalid batch records the device saw since scene creation (or the last
 * reset): pair records whose shape ids are out of [0, n_shapes) (those pairs
 * get no rows from cm_manifold_offsets), whose env / slot indices are out of
 * [0, n_env) / [0, n_slot) or whose shapes lack the sampled surface / SDF
 * (their rows are filled with NaN, dom = -1), and sdf_eval / param_grad
 * shape ids that are out of range or name a shape without an SDF (their
 * outputs are NaN).  Invalid indices are never dereferenced.  Synchronises
 * the device; reset != 0 zeroes the counter. */
int cm_scene_error_count(const cm_scene* scene, int64_t* count, int reset);

#ifdef __cplusplus
}
#endif
#endif /* XPSQ_CM_H */
