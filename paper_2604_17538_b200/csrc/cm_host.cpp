// Host side of the C ABI (include/xpsq_cm.h): validation, static packing of
// the shape library (flattened SDF programs, leaf parameters, XPSQ static
// data, sampled-surface topology), device residency, argument checks and
// kernel dispatch.  No compute of the hot path runs here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges around the C-ABI compute calls

#include "cm_internal.h"
#include "xpsq_cm.h"

using namespace cmi;

namespace {
// NVTX range of one C-ABI call (visible in Nsight Systems / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct Frame {
  double R[9], t[3];
};

void quat_R(const float* q, double* R) {
  double n = std::sqrt((double)q[0] * q[0] + (double)q[1] * q[1] + (double)q[2] * q[2] + (double)q[3] * q[3]);
  double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

Frame compose(const Frame& p, const float* pose7) {
  Frame c, r;
  quat_R(pose7 + 3, c.R);
  for (int i = 0; i < 3; ++i) c.t[i] = pose7[i];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.R[i * 3 + j] = p.R[i * 3 + 0] * c.R[0 * 3 + j] + p.R[i * 3 + 1] * c.R[1 * 3 + j] + p.R[i * 3 + 2] * c.R[2 * 3 + j];
  for (int i = 0; i < 3; ++i)
    r.t[i] = p.R[i * 3 + 0] * c.t[0] + p.R[i * 3 + 1] * c.t[1] + p.R[i * 3 + 2] * c.t[2] + p.t[i];
  return r;
}

double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
void cross3(const double* a, const double* b, double* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0];
}
void unit3(double* v) {
  double n = std::sqrt(dot3(v, v));
  for (int i = 0; i < 3; ++i) v[i] /= n;
}

bool finite_all(const float* p, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

// XPSQ classification thresholds (reading #14; the same rule is
// written independently in the oracle)
constexpr double X_EPS_POINT = 1e-6, X_EPS_LINE = 1e-4, X_EPS_FRAME = 1e-3;

Xpsq pack_xpsq(const cm_node& n) {
  Xpsq X;
  std::memset(&X, 0, sizeof(X));
  double p1[3], p2[3], p3[3], A[3], B[3];
  for (int i = 0; i < 3; ++i) { p1[i] = n.ctrl[i]; p2[i] = n.ctrl[3 + i]; p3[i] = n.ctrl[6 + i]; }
  for (int i = 0; i < 3; ++i) { A[i] = p1[i] - 2 * p2[i] + p3[i]; B[i] = 2 * (p2[i] - p1[i]); }
  double nA = std::sqrt(dot3(A, A)), nB = std::sqrt(dot3(B, B));
  double T0[3] = {1, 0, 0};
  if (nA < X_EPS_POINT && nB < X_EPS_POINT) {
    X.cls = 0;
  } else if (nA < X_EPS_LINE * nB) {
    // straight: the chord p1 -> p3 (B := A + B = p3 - p1, A := 0; both end
    // points kept, within |A|/4 of the spline)
    X.cls = 1;
    for (int i = 0; i < 3; ++i) { B[i] += A[i]; A[i] = 0; T0[i] = B[i]; }
  } else {
    X.cls = 2;
    for (int i = 0; i < 3; ++i) T0[i] = A[i] + B[i];
    if (std::sqrt(dot3(T0, T0)) < X_EPS_POINT)
      for (int i = 0; i < 3; ++i) T0[i] = nB > X_EPS_POINT ? B[i] : A[i];
  }
  double bxa[3];
  cross3(B, A, bxa);
  X.frenet = (X.cls == 2 && std::sqrt(dot3(bxa, bxa)) >= X_EPS_FRAME * nA * nB) ? 1 : 0;
  double bh[3];
  if (X.frenet) {
    for (int i = 0; i < 3; ++i) bh[i] = bxa[i];
    unit3(bh);
  } else {
    double up[3] = {n.up[0], n.up[1], n.up[2]};
    if (X.cls == 0) {
      unit3(up);
      double e[3] = {1, 0, 0};
      double c = dot3(e, up);
      if (std::fabs(c) > 0.9) { e[0] = 0; e[1] = 1; c = dot3(e, up); }
      for (int i = 0; i < 3; ++i) T0[i] = e[i] - c * up[i];
      unit3(T0);
    } else {
      unit3(T0);
      double c = dot3(up, T0);
      for (int i = 0; i < 3; ++i) up[i] -= c * T0[i];
      unit3(up);
    }
    for (int i = 0; i < 3; ++i) bh[i] = up[i];
    double N[3];
    cross3(bh, T0, N);
    for (int i = 0; i < 3; ++i) {
      X.R0[i * 3 + 0] = (float)T0[i];
      X.R0[i * 3 + 1] = (float)N[i];
      X.R0[i * 3 + 2] = (float)bh[i];
    }
  }
  for (int i = 0; i < 3; ++i) {
    X.p1[i] = (float)p1[i]; X.A[i] = (float)A[i]; X.B[i] = (float)B[i]; X.bhat[i] = (float)bh[i];
    X.up[i] = n.up[i];
  }
  double BB = dot3(B, B);
  if (X.cls == 1)
    for (int i = 0; i < 3; ++i) X.Bn[i] = (float)(B[i] / BB);
  if (X.cls == 2) {
    // cubic of P:112: c3 t^3 + c2 t^2 + c1 t + c0, c3 = -2 A.A, c2 = -3 A.B,
    // c1 = 2 A.w - B.B, c0 = B.w; monic b = c2/c3; depressed P, Q affine in w
    double c3 = -2 * dot3(A, A), c2 = -3 * dot3(A, B), b = c2 / c3;
    for (int i = 0; i < 3; ++i) {
      X.gP[i] = (float)(2 * A[i] / c3);
      X.gQ[i] = (float)((B[i] - (2 * b / 3) * A[i]) / c3);
    }
    X.c3 = (float)c3;
    X.c2 = (float)c2;
    X.BB = (float)BB;
    X.P0 = (float)(-BB / c3 - b * b / 3);
    X.Q0 = (float)(2 * b * b * b / 27 + (b / 3) * BB / c3);
    X.b3 = (float)(b / 3);
  }
  X.n_planes = n.n_planes;
  bool varying = false;
  for (int i = 0; i < 2; ++i) {
    X.eps0[i] = n.eps[0][i];
    X.deps[i] = n.eps[1][i] - n.eps[0][i];
    varying |= X.deps[i] != 0.f;
  }
  for (int i = 0; i < 3; ++i) {
    X.a0[i] = n.a[0][i];
    X.da[i] = n.a[1][i] - n.a[0][i];
    varying |= X.da[i] != 0.f;
  }
  for (int i = 0; i < 3; ++i) X.sq_ia[i] = (float)(1.0 / n.a[0][i]);
  X.sq_p1 = (float)(1.0 / n.eps[0][0]);
  X.sq_p2 = (float)(1.0 / n.eps[0][1]);
  X.sq_m = (float)((double)n.eps[0][1] / n.eps[0][0]);
  X.sq_k = (float)(0.5 * n.eps[0][0]);
  for (int j = 0; j < n.n_planes; ++j)
    for (int i = 0; i < 4; ++i) {
      X.pl0[j][i] = n.planes[0][j][i];
      X.dpl[j][i] = n.planes[1][j][i] - n.planes[0][j][i];
      varying |= X.dpl[j][i] != 0.f;
    }
  X.varying = varying ? 1 : 0;
  return X;
}

// ---- broad-phase bounds (f2, reading #46) ------------------------
// phi >= |x - c| - r over the whole space (r = +inf: unbounded below), in the
// body frame, from the SDF tree with node frames composed on the way down
struct HBound {
  double c[3];
  double r;
};
HBound tree_bound(const cm_shape_desc& d, int k, const Frame& parent, double tau_min) {
  const cm_node& n = d.nodes[k];
  const Frame fr = compose(parent, n.pose);
  HBound b;
  b.r = INFINITY;
  for (int i = 0; i < 3; ++i) b.c[i] = fr.t[i];
  if (n.type == CM_HALFSPACE) return b;
  if (n.type == CM_SQ || n.type == CM_PSQ) {   // inside the box |y_i| <= a_i; PSQ >= SQ
    b.r = std::sqrt((double)n.a[0][0] * n.a[0][0] + (double)n.a[0][1] * n.a[0][1] + (double)n.a[0][2] * n.a[0][2]);
    return b;
  }
  if (n.type == CM_XPSQ) {   // the spline in its control points' box; three-root smooth min >= min - tau ln 3
    double mid[3], half2 = 0.0, am = 0.0;
    for (int i = 0; i < 3; ++i) {
      const double lo = std::min({(double)n.ctrl[i], (double)n.ctrl[3 + i], (double)n.ctrl[6 + i]});
      const double hi = std::max({(double)n.ctrl[i], (double)n.ctrl[3 + i], (double)n.ctrl[6 + i]});
      mid[i] = 0.5 * (lo + hi);
      half2 += 0.25 * (hi - lo) * (hi - lo);
    }
    for (int e = 0; e < 2; ++e)
      am = std::max(am, std::sqrt((double)n.a[e][0] * n.a[e][0] + (double)n.a[e][1] * n.a[e][1] +
                                  (double)n.a[e][2] * n.a[e][2]));
    for (int i = 0; i < 3; ++i)
      b.c[i] = fr.R[i * 3 + 0] * mid[0] + fr.R[i * 3 + 1] * mid[1] + fr.R[i * 3 + 2] * mid[2] + fr.t[i];
    b.r = std::sqrt(half2) + am + tau_min * std::log(3.0);
    return b;
  }
  std::vector<HBound> kids;
  for (int c = 0; c < n.n_children; ++c) kids.push_back(tree_bound(d, n.children[c], fr, tau_min));
  if (n.type == CM_SUBTRACTION) return kids[0];             // LSE(phi1, -phi2) >= phi1
  if (n.type == CM_INTERSECTION) {                          // LSE(phi_i) >= each phi_i
    for (const HBound& x : kids) if (x.r < b.r) b = x;
    return b;
  }
  // union: -LSE(-phi_i) >= min phi_i - tau ln n
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (const HBound& x : kids) {
    if (!(x.r < INFINITY)) return b;
    for (int i = 0; i < 3; ++i) { lo[i] = std::min(lo[i], x.c[i]); hi[i] = std::max(hi[i], x.c[i]); }
  }
  for (int i = 0; i < 3; ++i) b.c[i] = 0.5 * (lo[i] + hi[i]);
  double r = 0.0;
  for (const HBound& x : kids) {
    const double dx = x.c[0] - b.c[0], dy = x.c[1] - b.c[1], dz = x.c[2] - b.c[2];
    r = std::max(r, std::sqrt(dx * dx + dy * dy + dz * dz) + x.r);
  }
  b.r = r + tau_min * std::log((double)kids.size());
  return b;
}

template <class T> T* dev_copy(const std::vector<T>& v, int& rc) {
  if (v.empty()) return nullptr;
  T* p = nullptr;
  cudaError_t e = cudaMalloc(&p, v.size() * sizeof(T));
  if (e != cudaSuccess) {
    rc = CM_ERR_OOM;
    g_err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
    return nullptr;
  }
  e = cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    rc = CM_ERR_CUDA;
    g_err = std::string("cudaMemcpy: ") + cudaGetErrorString(e);
  }
  return p;
}
}  // namespace

struct cm_scene {
  int device = 0;
  SceneDev dev;
  std::vector<ShapeRec> shapes;
  std::vector<std::vector<int32_t>> edges, face_edges;
  int max_V = 0, max_E = 0, max_F = 0;
  std::vector<int32_t> param_count;    // per shape (f4), -1: not parametrised
  std::vector<int64_t> param_off;      // prefix sums of max(count, 0)
  int64_t* param_off_dev = nullptr;
  std::vector<int32_t> pose_count;     // per shape: 6 x its SDF nodes (f4 node poses), -1: not parametrised
  std::vector<int64_t> pose_off;       // prefix sums of max(count, 0)
  int64_t* pose_off_dev = nullptr;
  int class_mask = 0;  // bit c: SDF shapes of class c (0 SQ family, 1 XPSQ, 2 varying-schedule XPSQ)
  std::vector<void*> allocs;
  float* scratch = nullptr;
  int64_t scratch_floats = 0;
  // manifold calls share the scratch: a call enqueues under `mu` and forks
  // onto the scene's aux streams, which serialise calls on the device
  std::mutex mu;
  cudaStream_t aux[cmi::kManifoldStreams] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[cmi::kManifoldStreams] = {};
  int64_t manifold_calls = 0;   // under mu
  unsigned long long last_capture_id = 0;   // capture of the last manifold call (0: none)
  int last_tier = -1;                        // tier of the last manifold call (its scratch layout)
  unsigned long long* sdf_ctr = nullptr;     // multi-class sdf_eval: per-class work counters
};

// aux streams used per manifold call (CM_MANIFOLD_STREAMS=1 serialises the
// chunks on one stream; experiments only)
static int n_aux_streams() {
  static const int n = [] {
    const char* e = std::getenv("CM_MANIFOLD_STREAMS");
    int v = e ? std::atoi(e) : cmi::kManifoldStreams;
    return std::min(std::max(v, 1), cmi::kManifoldStreams);
  }();
  return n;
}

// sdf_eval with several SDF classes runs the class kernels concurrently on
// the scene's streams (CM_SDF_CONCURRENT=0: in order on the caller's stream;
// experiments only)
static bool sdf_concurrent() {
  static const bool on = [] {
    const char* e = std::getenv("CM_SDF_CONCURRENT");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

#ifndef CM_SDF_DYNAMIC
#define CM_SDF_DYNAMIC 0   // multi-class sdf_eval: dynamic per-warp work from device counters on the aux
                           // streams (SDF +3.6% at 256 threads, +4.1% at 64; static at 64 threads +4.8%: r02zk3)
#endif

// makes the scene's device current for a call and restores the caller's
// device afterwards (compute calls must not depend on, or change,
// the caller's current device)
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

extern "C" {

int cm_version(void) { return CM_ABI_VERSION; }
const char* cm_last_error(void) { return g_err.c_str(); }

int cm_scene_create(const cm_shape_desc* shapes, int32_t n_shapes, const cm_smooth_params* sp, int device,
                    cm_scene** out) {
  if (!shapes || !sp || !out || n_shapes <= 0) return fail(CM_ERR_INVALID, "cm_scene_create: bad arguments");
  *out = nullptr;
  const float taus[5] = {sp->tau_cmp, sp->tau_min, sp->tau_clip_alpha, sp->tau_clip_t, sp->tau_delta};
  for (float t : taus)
    if (!(t > 0.f) || !std::isfinite(t)) return fail(CM_ERR_INVALID, "smooth params: every tau must be > 0 (S:28)");
  if (sp->trace_iters < 0 || sp->trace_iters > 64) return fail(CM_ERR_INVALID, "trace_iters out of range");

  std::vector<Instr> prog;
  std::vector<NodeFrame> op_frames;   // parallel to prog (node-pose derivatives, f4)
  std::vector<Leaf> leaves;
  std::vector<Xpsq> xps;
  std::vector<ShapeRec> recs(n_shapes);
  std::vector<float> verts;
  std::vector<int32_t> edges_all, faces_all, fe_all;
  std::vector<float> edge_geom;   // x_I, L, e_t (computed in FP64 from the FP32 vertices)
  cm_scene* sc = new cm_scene;
  sc->device = device;
  sc->param_count.assign(n_shapes, 0);
  sc->pose_count.assign(n_shapes, 0);
  sc->edges.resize(n_shapes);
  sc->face_edges.resize(n_shapes);

  std::vector<std::vector<float>> tess_v(n_shapes);
  std::vector<std::vector<int32_t>> tess_f(n_shapes);
  for (int s = 0; s < n_shapes; ++s) {
    cm_shape_desc dloc = shapes[s];
    if (dloc.n_faces == 0 && dloc.sample_res > 0) {
      // library-side sampled surface (SURVEY §8(b) sample_res): the single
      // SQ / PSQ / XPSQ node tessellated in its frame, placed by its pose
      if (dloc.n_nodes != 1 || !dloc.nodes) {
        delete sc;
        return fail(CM_ERR_UNSUPPORTED, "shape " + std::to_string(s) + ": sample_res needs a single SQ / PSQ / XPSQ node");
      }
      int32_t nv = 0, nf = 0;
      int trc = cm_tessellate(dloc.nodes, dloc.sample_res, nullptr, nullptr, &nv, &nf);
      if (trc == CM_OK) {
        tess_v[s].resize(3 * (size_t)nv);
        tess_f[s].resize(3 * (size_t)nf);
        trc = cm_tessellate(dloc.nodes, dloc.sample_res, tess_v[s].data(), tess_f[s].data(), &nv, &nf);
      }
      if (trc != CM_OK) {
        delete sc;
        return fail(trc, "shape " + std::to_string(s) + ": cannot tessellate this node (cm_tessellate)");
      }
      double q[4] = {dloc.nodes[0].pose[3], dloc.nodes[0].pose[4], dloc.nodes[0].pose[5], dloc.nodes[0].pose[6]};
      const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      for (double& c : q) c /= qn;
      const double w = q[0], x = q[1], y = q[2], z = q[3];
      const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                           2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                           2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
      for (int32_t v = 0; v < nv; ++v) {
        const double p[3] = {tess_v[s][3 * v], tess_v[s][3 * v + 1], tess_v[s][3 * v + 2]};
        for (int i = 0; i < 3; ++i)
          tess_v[s][3 * v + i] = (float)(R[3 * i] * p[0] + R[3 * i + 1] * p[1] + R[3 * i + 2] * p[2] + dloc.nodes[0].pose[i]);
      }
      dloc.n_vertices = nv;
      dloc.vertices = tess_v[s].data();
      dloc.n_faces = nf;
      dloc.faces = tess_f[s].data();
    }
    const cm_shape_desc& d = dloc;
    ShapeRec& r = recs[s];
    std::memset(&r, 0, sizeof(r));
    r.prog_begin = (int32_t)prog.size();
    if (d.n_nodes > 0) {
      if (!d.nodes) { delete sc; return fail(CM_ERR_INVALID, "shape " + std::to_string(s) + ": nodes is NULL"); }
      // validate nodes
      for (int k = 0; k < d.n_nodes; ++k) {
        const cm_node& n = d.nodes[k];
        std::string w = "shape " + std::to_string(s) + " node " + std::to_string(k) + ": ";
        if (!finite_all(n.pose, 7) || !finite_all(&n.eps[0][0], 4) || !finite_all(&n.a[0][0], 6) ||
            !finite_all(&n.planes[0][0][0], 2 * CM_MAX_PLANES * 4) || !finite_all(n.ctrl, 9) || !finite_all(n.up, 3)) {
          delete sc;
          return fail(CM_ERR_NONFINITE, w + "non-finite parameter");
        }
        const bool leaf = n.type <= CM_XPSQ;
        if (leaf) {
          if (n.type < 0) { delete sc; return fail(CM_ERR_UNSUPPORTED, w + "unknown node type"); }
          int np = n.type == CM_HALFSPACE ? 1 : (n.type == CM_SQ ? 0 : n.n_planes);
          if (np < 0 || np > CM_MAX_PLANES) { delete sc; return fail(CM_ERR_UNSUPPORTED, w + "too many planes"); }
          int ends = n.type == CM_XPSQ ? 2 : 1;
          for (int e = 0; e < ends; ++e)
            for (int j = 0; j < np; ++j) {
              const float* pl = n.planes[e][j];
              double nn = std::sqrt((double)pl[0] * pl[0] + (double)pl[1] * pl[1] + (double)pl[2] * pl[2]);
              if (std::fabs(nn - 1.0) > 1e-5) { delete sc; return fail(CM_ERR_INVALID, w + "plane normal not unit (S:172)"); }
            }
          if (n.type != CM_HALFSPACE)
            for (int e = 0; e < ends; ++e) {
              for (int i = 0; i < 2; ++i)
                if (n.eps[e][i] < 0.1f - 1e-6f || n.eps[e][i] > 2.0f + 1e-6f) {
                  delete sc;
                  return fail(CM_ERR_INVALID, w + "eps outside [0.1, 2] (S:177)");
                }
              for (int i = 0; i < 3; ++i)
                if (!(n.a[e][i] > 0.f)) { delete sc; return fail(CM_ERR_INVALID, w + "scale a must be > 0"); }
            }
        } else {
          if (n.type != CM_UNION && n.type != CM_INTERSECTION && n.type != CM_SUBTRACTION) {
            delete sc;
            return fail(CM_ERR_UNSUPPORTED, w + "unknown node type");
          }
          if (n.type == CM_SUBTRACTION ? n.n_children != 2 : (n.n_children < 2 || n.n_children > CM_MAX_CHILDREN)) {
            delete sc;
            return fail(CM_ERR_ARITY, w + "arity (subtraction 2, union/intersection >= 2) (S:184)");
          }
          for (int c = 0; c < n.n_children; ++c)
            if (n.children[c] <= k || n.children[c] >= d.n_nodes) {
              delete sc;
              return fail(CM_ERR_INVALID, w + "child index must point to a later node");
            }
        }
      }
      // flatten: depth-first emission with composed frames
      int xclass = 0;
      int max_depth = 0;
      struct Item { int node; float child_sign; Frame parent; int depth; };
      std::string err;
      std::vector<int> leaf_nodes;   // node index of each emitted leaf (program order)
      std::function<bool(int, float, const Frame&, int)> emit;
      auto op_frame = [&](int k, const Frame& parent) {
        NodeFrame nf;
        std::memset(&nf, 0, sizeof(nf));
        for (int i = 0; i < 9; ++i) nf.RP[i] = (float)parent.R[i];
        for (int i = 0; i < 3; ++i) { nf.tP[i] = (float)parent.t[i]; nf.tk[i] = d.nodes[k].pose[i]; }
        nf.node = k;
        return nf;
      };
      emit = [&](int k, float cs, const Frame& parent, int depth) -> bool {
        const cm_node& n = d.nodes[k];
        Frame fr = compose(parent, n.pose);
        if (n.type <= CM_XPSQ) {
          Leaf L;
          std::memset(&L, 0, sizeof(L));
          bool ident = true;
          for (int i = 0; i < 9; ++i) {
            L.R[i] = (float)fr.R[i];
            ident &= L.R[i] == ((i % 4 == 0) ? 1.f : 0.f);
          }
          for (int i = 0; i < 3; ++i) L.t[i] = (float)fr.t[i];
          L.rot_identity = ident ? 1 : 0;
          L.n_planes = n.type == CM_PSQ ? n.n_planes : (n.type == CM_HALFSPACE ? 1 : 0);
          for (int j = 0; j < L.n_planes && n.type != CM_XPSQ; ++j)
            for (int i = 0; i < 4; ++i) L.planes[j][i] = n.planes[0][j][i];
          if (n.type == CM_HALFSPACE) {
            L.kind = LK_HALFSPACE;
          } else if (n.type == CM_XPSQ) {
            L.kind = LK_XPSQ;
            L.n_planes = 0;
            L.xidx = (int32_t)xps.size();
            xps.push_back(pack_xpsq(n));
            {   // culling sphere in the shape frame (see Leaf::cull)
              double lo[3], hi[3];
              for (int i = 0; i < 3; ++i) {
                lo[i] = std::min({(double)n.ctrl[i], (double)n.ctrl[3 + i], (double)n.ctrl[6 + i]});
                hi[i] = std::max({(double)n.ctrl[i], (double)n.ctrl[3 + i], (double)n.ctrl[6 + i]});
              }
              double cl[3], rho = 0.0, amax = 0.0;
              for (int i = 0; i < 3; ++i) {
                cl[i] = 0.5 * (lo[i] + hi[i]);
                rho += 0.25 * (hi[i] - lo[i]) * (hi[i] - lo[i]);
              }
              for (int e = 0; e < 2; ++e)
                amax = std::max(amax, std::sqrt((double)n.a[e][0] * n.a[e][0] + (double)n.a[e][1] * n.a[e][1] +
                                                (double)n.a[e][2] * n.a[e][2]));
              for (int i = 0; i < 3; ++i)   // node frame -> shape frame (x = R y + t)
                L.cull[i] = (float)(fr.R[i * 3 + 0] * cl[0] + fr.R[i * 3 + 1] * cl[1] + fr.R[i * 3 + 2] * cl[2] + fr.t[i]);
              L.cull[3] = (float)((std::sqrt(rho) + amax + sp->tau_min * std::log(3.0)) * (1.0 + 1e-5) + 1e-7);
            }
            xclass = std::max(xclass, xps.back().varying ? 2 : 1);
          } else {
            L.kind = LK_SQ;
            double e1 = n.eps[0][0], e2 = n.eps[0][1];
            for (int i = 0; i < 3; ++i) L.ia[i] = (float)(1.0 / n.a[0][i]);
            L.p1 = (float)(1.0 / e1);
            L.p2 = (float)(1.0 / e2);
            L.m = (float)(e2 / e1);
            L.k = (float)(0.5 * e1);
          }
          prog.push_back(Instr{OP_LEAF, (int32_t)leaves.size(), cs, 1.f});
          op_frames.push_back(op_frame(k, parent));
          leaves.push_back(L);
          leaf_nodes.push_back(k);
          return true;
        }
        if (depth >= CM_MAX_DEPTH) {
          err = "boolean nesting deeper than CM_MAX_DEPTH";
          return false;
        }
        max_depth = std::max(max_depth, depth + 1);
        prog.push_back(Instr{OP_BEGIN, 0, 0.f, 0.f});
        op_frames.push_back(op_frame(k, parent));
        for (int c = 0; c < n.n_children; ++c) {
          float s2 = n.type == CM_UNION ? -1.f : (n.type == CM_INTERSECTION ? 1.f : (c == 0 ? 1.f : -1.f));
          if (!emit(n.children[c], s2, fr, depth + 1)) return false;
        }
        prog.push_back(Instr{OP_END, 0, cs, n.type == CM_UNION ? -1.f : 1.f});
        op_frames.push_back(op_frame(k, parent));
        return true;
      };
      Frame id;
      for (int i = 0; i < 9; ++i) id.R[i] = (i % 4 == 0) ? 1.0 : 0.0;
      id.t[0] = id.t[1] = id.t[2] = 0.0;
      if (!emit(0, 1.f, id, 0)) { delete sc; return fail(CM_ERR_UNSUPPORTED, "shape " + std::to_string(s) + ": " + err); }
      r.has_sdf = 1;
      // classes: 0 SQ family (booleans at most one level deep), 3 deeper SQ
      // family, 1 a lone constant-schedule XPSQ, 4 constant-schedule XPSQ in
      // a boolean tree, 2 varying-schedule XPSQ
      r.uses_xpsq = xclass == 0 ? (max_depth > 1 ? 3 : 0) : (xclass == 1 && max_depth >= 1 ? 4 : xclass);
      sc->class_mask |= 1 << r.uses_xpsq;
      // shape-parameter count (f4): leaves in pre-order, a varying-schedule
      // XPSQ with both endpoints' slots; trees of more than kParamMaxNodes
      // boolean nodes or node lists whose leaves are not in depth-first
      // order are not parametrised (-1)
      int pc = 0, n_bool = 0;
      for (int k = 0; k < d.n_nodes; ++k) {
        const int ty = d.nodes[k].type;
        if (ty == CM_HALFSPACE) pc += 4;
        else if (ty == CM_SQ) pc += 5;
        else if (ty == CM_PSQ) pc += 5 + 4 * d.nodes[k].n_planes;
        else if (ty == CM_XPSQ) pc += (pack_xpsq(d.nodes[k]).varying ? 2 : 1) * (5 + 4 * d.nodes[k].n_planes) + 9;
        else ++n_bool;
      }
      if (n_bool > cmi::kParamMaxNodes) pc = -1;   // large trees
      // the kernel lays the parameters out in program order: it must be the
      // node-index order the layout promises (true for pre-order node lists)
      if (!std::is_sorted(leaf_nodes.begin(), leaf_nodes.end())) pc = -1;
      sc->param_count[s] = pc;
      // node poses: six slots per node (the kernel writes them by the node
      // index of each op, so any node order is parametrised)
      sc->pose_count[s] = n_bool > cmi::kParamMaxNodes ? -1 : 6 * d.n_nodes;
    }
    r.prog_len = (int32_t)prog.size() - r.prog_begin;

    // sampled surface + topology: unique sorted edges,
    // face_edges for (i0,i1), (i1,i2), (i2,i0)
    if (d.n_faces > 0) {
      if (!d.vertices || !d.faces || d.n_vertices < 3) {
        delete sc;
        return fail(CM_ERR_INVALID, "shape " + std::to_string(s) + ": mesh arrays");
      }
      if (!finite_all(d.vertices, 3 * d.n_vertices)) { delete sc; return fail(CM_ERR_NONFINITE, "mesh vertex"); }
      const int V = d.n_vertices, F = d.n_faces;
      std::vector<std::tuple<int, int, int>> keys;   // (lo, hi, face*3 + k)
      keys.reserve(3 * F);
      for (int f = 0; f < F; ++f)
        for (int k = 0; k < 3; ++k) {
          int a = d.faces[3 * f + k], b = d.faces[3 * f + (k + 1) % 3];
          if (a < 0 || b < 0 || a >= V || b >= V || a == b) {
            delete sc;
            return fail(CM_ERR_INVALID, "shape " + std::to_string(s) + ": bad or degenerate face " + std::to_string(f));
          }
          keys.emplace_back(std::min(a, b), std::max(a, b), 3 * f + k);
        }
      std::sort(keys.begin(), keys.end());
      std::vector<int32_t>& eg = sc->edges[s];
      std::vector<int32_t>& fe = sc->face_edges[s];
      fe.assign(3 * F, -1);
      int E = 0;
      for (size_t i = 0; i < keys.size(); ++i) {
        if (i == 0 || std::get<0>(keys[i]) != std::get<0>(keys[i - 1]) || std::get<1>(keys[i]) != std::get<1>(keys[i - 1])) {
          int a = std::get<0>(keys[i]), b = std::get<1>(keys[i]);
          const float* va = d.vertices + 3 * a;
          const float* vb = d.vertices + 3 * b;
          if (va[0] == vb[0] && va[1] == vb[1] && va[2] == vb[2]) {
            delete sc;
            return fail(CM_ERR_INVALID, "degenerate (zero-length) edge (S:455)");
          }
          eg.push_back(a);
          eg.push_back(b);
          ++E;
        }
        fe[std::get<2>(keys[i])] = E - 1;
      }
      r.V = V; r.E = E; r.F = F;
      r.v_off = (int32_t)(verts.size() / 4);
      r.e_off = (int32_t)(edges_all.size() / 2);
      r.f_off = (int32_t)(faces_all.size() / 3);
      for (int v = 0; v < V; ++v) {   // padded to 16 B: one 128-bit load per vertex
        verts.insert(verts.end(), d.vertices + 3 * v, d.vertices + 3 * v + 3);
        verts.push_back(0.f);
      }
      edges_all.insert(edges_all.end(), eg.begin(), eg.end());
      for (int k = 0; k < E; ++k) {
        const float* xa = d.vertices + 3 * eg[2 * k];
        const float* xb = d.vertices + 3 * eg[2 * k + 1];
        const double dl[3] = {(double)xb[0] - xa[0], (double)xb[1] - xa[1], (double)xb[2] - xa[2]};
        const double L = std::sqrt(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
        const float g8[8] = {xa[0], xa[1], xa[2], (float)L, (float)(dl[0] / L), (float)(dl[1] / L), (float)(dl[2] / L), 0.f};
        edge_geom.insert(edge_geom.end(), g8, g8 + 8);
      }
      faces_all.insert(faces_all.end(), d.faces, d.faces + 3 * F);
      fe_all.insert(fe_all.end(), fe.begin(), fe.end());
      sc->max_V = std::max(sc->max_V, V);
      sc->max_E = std::max(sc->max_E, E);
      sc->max_F = std::max(sc->max_F, F);
    }
  }
  sc->shapes = recs;
  // broad-phase bounds per shape (f2): float, rounded outward
  std::vector<float4> bounds(2 * (size_t)n_shapes);
  for (int s = 0; s < n_shapes; ++s) {
    cm_shape_desc dloc = shapes[s];
    if (!tess_f[s].empty()) {   // the library-side tessellation
      dloc.n_vertices = (int32_t)(tess_v[s].size() / 3);
      dloc.vertices = tess_v[s].data();
      dloc.n_faces = (int32_t)(tess_f[s].size() / 3);
      dloc.faces = tess_f[s].data();
    }
    const cm_shape_desc& d = dloc;
    float4 mb = make_float4(0.f, 0.f, 0.f, -1.f), sb = make_float4(0.f, 0.f, 0.f, INFINITY);
    if (d.n_faces > 0) {
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY}, c[3], r = 0.0;
      for (int v = 0; v < d.n_vertices; ++v)
        for (int i = 0; i < 3; ++i) { lo[i] = std::min(lo[i], (double)d.vertices[3 * v + i]); hi[i] = std::max(hi[i], (double)d.vertices[3 * v + i]); }
      for (int i = 0; i < 3; ++i) c[i] = 0.5 * (lo[i] + hi[i]);
      for (int v = 0; v < d.n_vertices; ++v) {
        const double dx = d.vertices[3 * v] - c[0], dy = d.vertices[3 * v + 1] - c[1], dz = d.vertices[3 * v + 2] - c[2];
        r = std::max(r, std::sqrt(dx * dx + dy * dy + dz * dz));
      }
      mb = make_float4((float)c[0], (float)c[1], (float)c[2], (float)(r * (1.0 + 1e-6) + 1e-7));
    }
    if (d.n_nodes > 0) {
      Frame id;
      for (int i = 0; i < 9; ++i) id.R[i] = (i % 4 == 0) ? 1.0 : 0.0;
      id.t[0] = id.t[1] = id.t[2] = 0.0;
      const HBound hb = tree_bound(d, 0, id, sp->tau_min);
      if (hb.r < INFINITY)
        sb = make_float4((float)hb.c[0], (float)hb.c[1], (float)hb.c[2], (float)(hb.r * (1.0 + 1e-6) + 1e-7));
    }
    bounds[2 * s] = mb;
    bounds[2 * s + 1] = sb;
  }

  int prev_dev = -1;
  cudaGetDevice(&prev_dev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete sc; return fail(CM_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)); }
  struct RestoreDev {
    int d;
    ~RestoreDev() { if (d >= 0) cudaSetDevice(d); }
  } restore_dev{prev_dev};
  int rc = CM_OK;
  SceneDev& D = sc->dev;
  std::memset(&D, 0, sizeof(D));
  D.prog = dev_copy(prog, rc);
  D.op_frames = dev_copy(op_frames, rc);
  if (D.op_frames) sc->allocs.push_back(const_cast<NodeFrame*>(D.op_frames));
  D.leaves = dev_copy(leaves, rc);
  D.xpsq = dev_copy(xps, rc);
  D.shapes = dev_copy(recs, rc);
  {   // compact per-shape SDF class (sdf_eval's class kernels skip foreign points on one byte)
    std::vector<int8_t> cls(n_shapes);
    for (int s = 0; s < n_shapes; ++s) cls[s] = recs[s].has_sdf ? (int8_t)recs[s].uses_xpsq : (int8_t)-1;
    D.shape_cls = dev_copy(cls, rc);
    if (D.shape_cls) sc->allocs.push_back(const_cast<int8_t*>(D.shape_cls));
  }
  D.verts = dev_copy(verts, rc);
  D.edges = dev_copy(edges_all, rc);
  D.edge_geom = dev_copy(edge_geom, rc);
  D.bounds = dev_copy(bounds, rc);
  D.faces = dev_copy(faces_all, rc);
  D.face_edges = dev_copy(fe_all, rc);
  for (const void* p : {(const void*)D.prog, (const void*)D.leaves, (const void*)D.xpsq, (const void*)D.shapes,
                        (const void*)D.verts, (const void*)D.edges, (const void*)D.faces, (const void*)D.face_edges,
                        (const void*)D.edge_geom, (const void*)D.bounds})
    if (p) sc->allocs.push_back(const_cast<void*>(p));
  sc->param_off.assign(n_shapes + 1, 0);
  for (int s = 0; s < n_shapes; ++s) sc->param_off[s + 1] = sc->param_off[s] + std::max(sc->param_count[s], 0);
  sc->param_off_dev = dev_copy(sc->param_off, rc);
  if (sc->param_off_dev) sc->allocs.push_back(sc->param_off_dev);
  sc->pose_off.assign(n_shapes + 1, 0);
  for (int s = 0; s < n_shapes; ++s) sc->pose_off[s + 1] = sc->pose_off[s] + std::max(sc->pose_count[s], 0);
  sc->pose_off_dev = dev_copy(sc->pose_off, rc);
  if (sc->pose_off_dev) sc->allocs.push_back(sc->pose_off_dev);
  {   // work counters of the multi-class sdf_eval schedule (one per SDF class)
    std::vector<unsigned long long> zc(8, 0ull);
    sc->sdf_ctr = dev_copy(zc, rc);
    if (sc->sdf_ctr) sc->allocs.push_back(sc->sdf_ctr);
  }
  {   // error word of the device-side record validation (cm_scene_error_count)
    std::vector<unsigned int> zero(4, 0u);
    D.err = dev_copy(zero, rc);
    if (D.err) sc->allocs.push_back(D.err);
  }
  D.sp = SmoothDev{sp->tau_cmp, sp->tau_min, sp->tau_clip_alpha, sp->tau_clip_t, sp->tau_delta, sp->trace_iters,
                   (float)(1.0 / sp->tau_cmp), (float)(1.0 / sp->tau_min), (float)(1.0 / sp->tau_clip_alpha),
                   (float)(1.0 / sp->tau_clip_t), (float)(1.0 / sp->tau_delta)};
  D.n_shapes = n_shapes;
  D.n_leaves = (int32_t)leaves.size();
  D.n_xpsq = (int32_t)xps.size();
  // chunk scratch of the manifold kernels (one candidate-state slot per unit)
  if (rc == CM_OK && sc->max_F > 0) {
    const int64_t slot = cml::manifold_slot_floats(sc->max_V, sc->max_E, 2);
    int64_t units = cmi::kChunkUnits;
    if (const char* env = std::getenv("CM_CHUNK_UNITS")) units = std::max<int64_t>(1, std::atoll(env));
    units = std::min<int64_t>(units, std::max<int64_t>(1, cmi::kScratchCapBytes / (slot * 4)));
    units = std::max<int64_t>(units, cmi::kManifoldStreams);
    sc->scratch_floats = slot * units;
    e = cudaMalloc(&sc->scratch, sc->scratch_floats * sizeof(float));
    if (e != cudaSuccess) { rc = CM_ERR_OOM; g_err = "scratch allocation failed"; }
    else sc->allocs.push_back(sc->scratch);
  }
  // aux streams: manifold chunks, and the class kernels of sdf_eval when the
  // scene holds several SDF classes
  if (rc == CM_OK && (sc->max_F > 0 || (sc->class_mask & (sc->class_mask - 1)) != 0)) {
    for (int i = 0; rc == CM_OK && i < cmi::kManifoldStreams; ++i) {
      if (cudaStreamCreateWithFlags(&sc->aux[i], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&sc->ev_join[i], cudaEventDisableTiming) != cudaSuccess) {
        rc = CM_ERR_CUDA; g_err = "aux stream creation failed";
      }
    }
    if (rc == CM_OK && cudaEventCreateWithFlags(&sc->ev_fork, cudaEventDisableTiming) != cudaSuccess) {
      rc = CM_ERR_CUDA; g_err = "aux event creation failed";
    }
  }
  if (rc != CM_OK) {
    cm_scene_destroy(sc);
    return rc;
  }
  *out = sc;
  return CM_OK;
}

int cm_scene_destroy(cm_scene* sc) {
  if (!sc) return CM_OK;
  DeviceGuard device_guard(sc->device);
  for (int i = 0; i < cmi::kManifoldStreams; ++i) {
    if (sc->aux[i]) cudaStreamDestroy(sc->aux[i]);
    if (sc->ev_join[i]) cudaEventDestroy(sc->ev_join[i]);
  }
  if (sc->ev_fork) cudaEventDestroy(sc->ev_fork);
  for (void* p : sc->allocs) cudaFree(p);
  delete sc;
  return CM_OK;
}

int cm_shape_counts(const cm_scene* sc, int32_t s, int32_t* V, int32_t* E, int32_t* F) {
  if (!sc || s < 0 || s >= (int)sc->shapes.size() || !V || !E || !F) return fail(CM_ERR_INVALID, "cm_shape_counts");
  *V = sc->shapes[s].V; *E = sc->shapes[s].E; *F = sc->shapes[s].F;
  return CM_OK;
}

int cm_shape_topology(const cm_scene* sc, int32_t s, int32_t* edges, int32_t* face_edges) {
  if (!sc || s < 0 || s >= (int)sc->shapes.size()) return fail(CM_ERR_INVALID, "cm_shape_topology");
  if (edges) std::memcpy(edges, sc->edges[s].data(), sc->edges[s].size() * sizeof(int32_t));
  if (face_edges) std::memcpy(face_edges, sc->face_edges[s].data(), sc->face_edges[s].size() * sizeof(int32_t));
  return CM_OK;
}

int cm_sdf_eval(const cm_scene* sc, const int32_t* ids, const float* poses, const float* points, int64_t B, int64_t P,
                uint32_t flags, float* d, float* grad, float* hess, float* dpose, float* d2pose, float* dxdpose,
                void* stream) {
  NvtxRange nvtx_range("cm_sdf_eval");
  if (!sc) return fail(CM_ERR_INVALID, "cm_sdf_eval: NULL scene");
  DeviceGuard device_guard(sc->device);
  if (B < 0 || P < 0) return fail(CM_ERR_INVALID, "cm_sdf_eval: negative size");
  if (B == 0 || P == 0) return CM_OK;   // empty batch: nothing to launch
  if (!ids || !poses || !points || !d) return fail(CM_ERR_INVALID, "cm_sdf_eval: NULL argument");
  if (((uintptr_t)poses & 15) != 0) return fail(CM_ERR_INVALID, "cm_sdf_eval: poses must be 16-byte aligned");
  if ((flags & CM_SDF_GRAD) && !grad) return fail(CM_ERR_INVALID, "cm_sdf_eval: grad is NULL");
  if ((flags & CM_SDF_HESS) && !hess) return fail(CM_ERR_INVALID, "cm_sdf_eval: hess is NULL");
  if ((flags & CM_SDF_POSE_GRAD) && !dpose) return fail(CM_ERR_INVALID, "cm_sdf_eval: dpose is NULL");
  if ((flags & CM_SDF_POSE_HESS) && (!d2pose || !dxdpose)) return fail(CM_ERR_INVALID, "cm_sdf_eval: d2pose/dxdpose NULL");
  grad = (flags & CM_SDF_GRAD) ? grad : nullptr;
  hess = (flags & CM_SDF_HESS) ? hess : nullptr;
  const int cm = sc->class_mask;
  if ((cm & (cm - 1)) == 0 || !sdf_concurrent()) {   // one SDF class: one kernel on the caller's stream
    void* st1[1] = {stream};
    const int rc = cml::launch_sdf_eval(sc->dev, cm, ids, poses, points, B, P, flags, d, grad, hess, dpose, d2pose,
                                        dxdpose, st1, 1);
    if (rc) return fail(rc, cml::last_cuda_error());
    return CM_OK;
  }
  // several classes: fork onto the scene's aux streams (the caller's stream
  // and the aux streams each run one class kernel concurrently), then join
  cm_scene* ms = const_cast<cm_scene*>(sc);   // internal scheduling state only
  std::lock_guard<std::mutex> lock(ms->mu);
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaEventRecord(ms->ev_fork, st) != cudaSuccess) return fail(CM_ERR_CUDA, "cm_sdf_eval: event record");
  // (dynamic schedule: class c's kernel takes its work from device counter
  // c; its launches stay on one aux stream, so the counter's reset and uses
  // are stream-ordered across calls)
  void* sts[1 + cmi::kManifoldStreams] = {stream};
  for (int i = 0; i < cmi::kManifoldStreams; ++i) {
    cudaStreamWaitEvent(ms->aux[i], ms->ev_fork, 0);
    sts[1 + i] = ms->aux[i];
  }
  const int rc = CM_SDF_DYNAMIC
                     ? cml::launch_sdf_eval(sc->dev, cm, ids, poses, points, B, P, flags, d, grad, hess, dpose, d2pose,
                                            dxdpose, sts + 1, cmi::kManifoldStreams, ms->sdf_ctr)
                     : cml::launch_sdf_eval(sc->dev, cm, ids, poses, points, B, P, flags, d, grad, hess, dpose, d2pose,
                                            dxdpose, sts, 1 + cmi::kManifoldStreams);
  for (int i = 0; i < cmi::kManifoldStreams; ++i) {
    cudaEventRecord(ms->ev_join[i], ms->aux[i]);
    cudaStreamWaitEvent(st, ms->ev_join[i], 0);
  }
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_param_layout(const cm_scene* sc, int32_t* counts, int64_t* offsets) {
  if (!sc) return fail(CM_ERR_INVALID, "cm_param_layout: NULL scene");
  const int ns = (int)sc->param_count.size();
  for (int s = 0; s < ns; ++s) {
    if (counts) counts[s] = sc->param_count[s];
    if (offsets) offsets[s] = sc->param_off[s];
  }
  if (offsets) offsets[ns] = sc->param_off[ns];
  return CM_OK;
}

int cm_sdf_param_grad(const cm_scene* sc, const int32_t* ids, const float* poses, const float* points, int64_t B,
                      int64_t P, int32_t pmax, float* J, const float* w, float* vjp, void* stream) {
  NvtxRange nvtx_range("cm_sdf_param_grad");
  if (!sc) return fail(CM_ERR_INVALID, "cm_sdf_param_grad: NULL scene");
  DeviceGuard device_guard(sc->device);
  if (B < 0 || P < 0 || pmax < 0) return fail(CM_ERR_INVALID, "cm_sdf_param_grad: negative size");
  if (B == 0 || P == 0) return CM_OK;
  if (!ids || !poses || !points || (!J && !vjp) || (vjp && !w))
    return fail(CM_ERR_INVALID, "cm_sdf_param_grad: NULL argument");
  if (((uintptr_t)poses & 15) != 0) return fail(CM_ERR_INVALID, "cm_sdf_param_grad: poses must be 16-byte aligned");
  for (size_t s = 0; s < sc->param_count.size(); ++s)
    if (sc->param_count[s] < 0)
      return fail(CM_ERR_UNSUPPORTED, "cm_sdf_param_grad: shape " + std::to_string(s) +
                                           " has more than 16 boolean nodes or leaves out of depth-first order (not parametrised)");
  int rc = cml::launch_sdf_param_grad(sc->dev, ids, poses, points, B, P, pmax, J, w, vjp, sc->param_off_dev, stream);
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_node_pose_layout(const cm_scene* sc, int32_t* counts, int64_t* offsets) {
  if (!sc) return fail(CM_ERR_INVALID, "cm_node_pose_layout: NULL scene");
  const int ns = (int)sc->pose_count.size();
  for (int s = 0; s < ns; ++s) {
    if (counts) counts[s] = sc->pose_count[s];
    if (offsets) offsets[s] = sc->pose_off[s];
  }
  if (offsets) offsets[ns] = sc->pose_off[ns];
  return CM_OK;
}

int cm_sdf_node_pose_grad(const cm_scene* sc, const int32_t* ids, const float* poses, const float* points, int64_t B,
                          int64_t P, int32_t nmax, float* J, const float* w, float* vjp, void* stream) {
  NvtxRange nvtx_range("cm_sdf_node_pose_grad");
  if (!sc) return fail(CM_ERR_INVALID, "cm_sdf_node_pose_grad: NULL scene");
  DeviceGuard device_guard(sc->device);
  if (B < 0 || P < 0 || nmax < 0) return fail(CM_ERR_INVALID, "cm_sdf_node_pose_grad: negative size");
  if (B == 0 || P == 0) return CM_OK;
  if (!ids || !poses || !points || (!J && !vjp) || (vjp && !w))
    return fail(CM_ERR_INVALID, "cm_sdf_node_pose_grad: NULL argument");
  if (((uintptr_t)poses & 15) != 0) return fail(CM_ERR_INVALID, "cm_sdf_node_pose_grad: poses must be 16-byte aligned");
  for (size_t s = 0; s < sc->pose_count.size(); ++s)
    if (sc->pose_count[s] < 0)
      return fail(CM_ERR_UNSUPPORTED, "cm_sdf_node_pose_grad: shape " + std::to_string(s) +
                                           " has more than 16 boolean nodes (not parametrised)");
  int rc = cml::launch_sdf_node_pose_grad(sc->dev, ids, poses, points, B, P, nmax, J, w, vjp, sc->pose_off_dev, stream);
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_manifold_param_vjp(const cm_scene* sc, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                          const float* poses, int64_t n_env, int32_t n_slot, uint32_t flags, const float* w_depth,
                          float* vjp, void* stream) {
  NvtxRange nvtx_range("cm_manifold_param_vjp");
  if (!sc) return fail(CM_ERR_INVALID, "cm_manifold_param_vjp: NULL scene");
  DeviceGuard device_guard(sc->device);
  if (n_pairs < 0 || n_env < 0 || n_slot < 0) return fail(CM_ERR_INVALID, "cm_manifold_param_vjp: negative size");
  if (n_pairs == 0) return CM_OK;
  if (!pairs || !offsets || !poses || !w_depth || !vjp) return fail(CM_ERR_INVALID, "cm_manifold_param_vjp: NULL argument");
  if (((uintptr_t)poses & 15) != 0) return fail(CM_ERR_INVALID, "cm_manifold_param_vjp: poses must be 16-byte aligned");
  int pmax = 0;
  for (size_t s = 0; s < sc->param_count.size(); ++s) {
    if (sc->param_count[s] < 0 && sc->shapes[s].has_sdf)
      return fail(CM_ERR_UNSUPPORTED, "cm_manifold_param_vjp: shape " + std::to_string(s) + " is not parametrised");
    pmax = std::max(pmax, sc->param_count[s]);
  }
  int rc = cml::launch_manifold_param_vjp(sc->dev, sc->max_V, sc->max_E, pmax, pairs, n_pairs, offsets, poses, n_env,
                                          n_slot, flags & (CM_FULL_MODE | CM_TWO_SIDED | CM_BROAD_PHASE), w_depth, vjp,
                                          sc->param_off_dev, stream);
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_manifold_size(const cm_scene* sc, const int32_t* pairs, int64_t n_pairs, uint32_t flags, int64_t* n) {
  if (!sc || (!pairs && n_pairs > 0) || !n) return fail(CM_ERR_INVALID, "cm_manifold_size");
  const bool full = flags & CM_FULL_MODE, two = flags & CM_TWO_SIDED;
  const int ns = (int)sc->shapes.size();   // (CM_BROAD_PHASE does not change the row count)
  int64_t c = 0;
  for (int64_t i = 0; i < n_pairs; ++i) {
    const int a = pairs[5 * i + 3], b = pairs[5 * i + 4];
    if (a < 0 || a >= ns || b < 0 || b >= ns) return fail(CM_ERR_INVALID, "cm_manifold_size: bad shape id");
    for (int side = 0; side < (two ? 2 : 1); ++side) {
      const ShapeRec& sa = sc->shapes[side ? b : a];
      const ShapeRec& sb = sc->shapes[side ? a : b];
      if (sa.F == 0) return fail(CM_ERR_INVALID, "cm_manifold_size: sampled shape has no surface");
      if (!sb.has_sdf) return fail(CM_ERR_INVALID, "cm_manifold_size: SDF shape has no SDF");
      c += full ? (int64_t)sa.V + sa.E : (int64_t)sa.F;
    }
  }
  *n = c;
  return CM_OK;
}

int64_t cm_manifold_offsets_workspace(int64_t n_pairs) { return cml::offsets_workspace(n_pairs); }

int cm_manifold_offsets(const cm_scene* sc, const int32_t* pairs, int64_t n_pairs, uint32_t flags, int64_t* offsets,
                        void* ws, int64_t ws_bytes, void* stream) {
  NvtxRange nvtx_range("cm_manifold_offsets");
  if (!sc) return fail(CM_ERR_INVALID, "cm_manifold_offsets: NULL scene");
  DeviceGuard device_guard(sc->device);
  if (n_pairs == 0) return CM_OK;
  if (!pairs || !offsets || !ws) return fail(CM_ERR_INVALID, "cm_manifold_offsets: NULL argument");
  if (n_pairs > (int64_t)0x7fffffff) return fail(CM_ERR_UNSUPPORTED, "cm_manifold_offsets: too many pairs");
  if (ws_bytes < cml::offsets_workspace(n_pairs)) return fail(CM_ERR_INVALID, "cm_manifold_offsets: workspace too small");
  int rc = cml::launch_offsets(sc->dev, pairs, n_pairs, flags, offsets, ws, ws_bytes, stream);
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_contact_manifold(const cm_scene* sc, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                        const float* poses, int64_t n_env, int32_t n_slot, uint32_t flags, const cm_manifold_out* out,
                        int64_t n_contacts, void* stream) {
  NvtxRange nvtx_range("cm_contact_manifold");
  if (!sc || !out) return fail(CM_ERR_INVALID, "cm_contact_manifold: NULL argument");
  DeviceGuard device_guard(sc->device);
  if (n_pairs < 0 || n_env < 0 || n_slot <= 0 || n_contacts < 0) return fail(CM_ERR_INVALID, "cm_contact_manifold: sizes");
  if (n_pairs == 0) return CM_OK;   // empty batch: nothing to launch
  if (!pairs || !offsets || !poses) return fail(CM_ERR_INVALID, "cm_contact_manifold: NULL argument");
  const unsigned tier = flags & CM_TIER_MASK;
  if (tier > 3) return fail(CM_ERR_INVALID, "cm_contact_manifold: tier");
  if (!out->point || !out->normal || !out->depth || !out->dom) return fail(CM_ERR_INVALID, "tier-0 outputs are NULL");
  if (tier >= 1 && (!out->W || !out->q)) return fail(CM_ERR_INVALID, "tier-1 outputs are NULL");
  if (tier >= 2 && (!out->ddepth || !out->dnormal)) return fail(CM_ERR_INVALID, "tier-2 outputs are NULL");
  if (tier >= 3 && !out->d2depth) return fail(CM_ERR_INVALID, "tier-3 output d2depth is NULL");
  if (sc->max_F == 0) return fail(CM_ERR_INVALID, "scene has no sampled surface");
  cm_scene* ms = const_cast<cm_scene*>(sc);   // internal scheduling state only
  std::lock_guard<std::mutex> lock(ms->mu);
  cudaStream_t st = (cudaStream_t)stream;
  // fork: the aux streams wait for the caller's prior work and, when the
  // previous manifold call on this scene used another tier, for every aux
  // stream's part of that call (its join events): how a call splits the
  // scratch between the streams depends on its tier, so calls of different
  // tiers must never overlap on the device, whichever streams they were
  // issued from; calls of the same tier give each aux stream the same
  // scratch region, already ordered by that stream.  join: the caller's
  // stream waits for every chunk
  if (cudaEventRecord(ms->ev_fork, st) != cudaSuccess) return fail(CM_ERR_CUDA, "cm_contact_manifold: event record");
  // (under stream capture only join events recorded by the same capture can
  // be waited on: a captured graph's calls are ordered by its own edges)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  unsigned long long cap_id = 0;
  if (cudaStreamGetCaptureInfo(st, &cap, &cap_id) != cudaSuccess) return fail(CM_ERR_CUDA, "cm_contact_manifold: capture info");
  if (cap != cudaStreamCaptureStatusActive) cap_id = 0;
  const int tier_now = (int)(flags & CM_TIER_MASK);
#ifndef CM_FORK_SERIALIZE
#define CM_FORK_SERIALIZE 1
#endif
  const bool wait_prev = CM_FORK_SERIALIZE && ms->manifold_calls > 0 && ms->last_capture_id == cap_id &&
                         ms->last_tier != tier_now;
  void* aux[cmi::kManifoldStreams];
  for (int i = 0; i < cmi::kManifoldStreams; ++i) {
    cudaStreamWaitEvent(ms->aux[i], ms->ev_fork, 0);
    if (wait_prev)
      for (int j = 0; j < cmi::kManifoldStreams; ++j)
        if (j != i) cudaStreamWaitEvent(ms->aux[i], ms->ev_join[j], 0);
    aux[i] = ms->aux[i];
  }
  ++ms->manifold_calls;
  ms->last_capture_id = cap_id;
  ms->last_tier = tier_now;
  int rc = cml::launch_manifold(sc->dev, sc->class_mask, sc->max_V, sc->max_E, pairs, n_pairs, offsets, poses, n_env, n_slot,
                                flags, out, n_contacts, sc->scratch, sc->scratch_floats, aux, n_aux_streams());
  for (int i = 0; i < cmi::kManifoldStreams; ++i) {
    cudaEventRecord(ms->ev_join[i], ms->aux[i]);
    cudaStreamWaitEvent(st, ms->ev_join[i], 0);
  }
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_expand_jacobian(const cm_scene* sc, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                       const float* poses, int64_t n_env, int32_t n_slot, uint32_t flags, const float* W,
                       const float* q, int64_t n_contacts, float* J, void* stream) {
  NvtxRange nvtx_range("cm_expand_jacobian");
  if (!sc || !pairs || !offsets || !poses || !W || !q || !J) return fail(CM_ERR_INVALID, "cm_expand_jacobian");
  DeviceGuard device_guard(sc->device);
  int rc = cml::launch_expand(pairs, n_pairs, offsets, sc->dev, poses, n_env, n_slot, W, q, n_contacts, J, flags, stream);
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int cm_manifold_pair_reduce(const cm_scene* sc, const int32_t* pairs, int64_t n_pairs, const int64_t* offsets,
                            uint32_t flags, const cm_manifold_out* out, int64_t n_contacts, const float* w_depth,
                            const float* w_normal, float* pair_depth, float* pair_W, float* g_pose, void* stream) {
  NvtxRange nvtx_range("cm_manifold_pair_reduce");
  if (!sc || !out) return fail(CM_ERR_INVALID, "cm_manifold_pair_reduce: NULL argument");
  DeviceGuard device_guard(sc->device);
  if (n_pairs < 0 || n_contacts < 0) return fail(CM_ERR_INVALID, "cm_manifold_pair_reduce: sizes");
  if (n_pairs == 0) return CM_OK;
  if (!pairs || !offsets) return fail(CM_ERR_INVALID, "cm_manifold_pair_reduce: NULL argument");
  if (pair_depth && !out->depth) return fail(CM_ERR_INVALID, "cm_manifold_pair_reduce: pair_depth needs out->depth");
  if (pair_W && !out->W) return fail(CM_ERR_INVALID, "cm_manifold_pair_reduce: pair_W needs out->W (tier >= 1)");
  if (g_pose && (!out->ddepth || !out->dnormal || (!w_depth && !w_normal)))
    return fail(CM_ERR_INVALID, "cm_manifold_pair_reduce: g_pose needs tier-2 outputs and w_depth or w_normal");
  int rc = cml::launch_pair_reduce(sc->dev, pairs, n_pairs, offsets, flags, out, n_contacts, w_depth, w_normal,
                                   pair_depth, pair_W, g_pose, stream);
  if (rc) return fail(rc, cml::last_cuda_error());
  return CM_OK;
}

int64_t cm_launch_count(void) { return cml::launch_count(); }

int cm_scene_error_count(const cm_scene* sc, int64_t* count, int reset) {
  if (!sc || !count) return fail(CM_ERR_INVALID, "cm_scene_error_count: NULL argument");
  DeviceGuard device_guard(sc->device);
  unsigned int v = 0;
  cudaError_t e = cudaMemcpy(&v, sc->dev.err, sizeof(v), cudaMemcpyDeviceToHost);   // synchronises the device
  if (e != cudaSuccess) return fail(CM_ERR_CUDA, std::string("cm_scene_error_count: ") + cudaGetErrorString(e));
  *count = (int64_t)v;
  if (reset && cudaMemset(sc->dev.err, 0, sizeof(unsigned int)) != cudaSuccess)
    return fail(CM_ERR_CUDA, "cm_scene_error_count: reset");
  return CM_OK;
}

}  // extern "C"
