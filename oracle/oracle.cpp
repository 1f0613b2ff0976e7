// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, FP64 CPU implementation of what the hot path computes
// (arXiv 2604.17538, §II).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  The
// product path (paper_2604_17538_b200/) never includes, links or calls it, and
// this file includes no header of the product path.
//
// Every derivative comes from generic forward-mode jets (Dual<T,N>, nested for
// second order); no hand-derived derivative chain appears here, so the
// oracle's derivatives are independent of the CUDA kernels' analytic ones.
//
// Citations: P:n = /root/reference/PAPER.md line n (section / equation named);
// S:n = SPEC.md line n.  "Reading #k" = DESIGN.md §3 row k (the readings of
// the paper where it is silent, ambiguous or garbled).
//
// Parity pins: see tests/test_oracle_*.py.  Functions with no independent pin
// are marked "parity unpinned" below and in DESIGN.md.
// ============================================================================
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <map>
#include <utility>
#include <algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

// ---------------------------------------------------------------------------
// Forward-mode jets.  Dual<T,N>: value v and N partials, each of type T.
// Dual<Dual<double,3>,3> carries value, gradient and Hessian.
// ---------------------------------------------------------------------------
template <class T, int N> struct Dual {
  T v;
  T d[N];
  Dual() : v(0.0) { for (int i = 0; i < N; ++i) d[i] = T(0.0); }
  Dual(double c) : v(c) { for (int i = 0; i < N; ++i) d[i] = T(0.0); }
  explicit Dual(const T& c, bool) : v(c) { for (int i = 0; i < N; ++i) d[i] = T(0.0); }
};

inline double val(double x) { return x; }
template <class T, int N> inline double val(const Dual<T, N>& x) { return val(x.v); }

// lift a plain constant into any jet type
template <class T> struct Lift { static T from(double c) { return T(c); } };

#define ORC_BIN(OP)                                                                   \
  template <class T, int N> Dual<T, N> operator OP(const Dual<T, N>& a, double b) {   \
    Dual<T, N> r = a; r.v = a.v OP b; return r; }
ORC_BIN(+)
ORC_BIN(-)
#undef ORC_BIN
template <class T, int N> Dual<T, N> operator+(double a, const Dual<T, N>& b) { return b + a; }
template <class T, int N> Dual<T, N> operator-(double a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a - b.v; for (int i = 0; i < N; ++i) r.d[i] = -b.d[i]; return r; }
template <class T, int N> Dual<T, N> operator-(const Dual<T, N>& a) {
  Dual<T, N> r; r.v = -a.v; for (int i = 0; i < N; ++i) r.d[i] = -a.d[i]; return r; }
template <class T, int N> Dual<T, N> operator+(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v + b.v; for (int i = 0; i < N; ++i) r.d[i] = a.d[i] + b.d[i]; return r; }
template <class T, int N> Dual<T, N> operator-(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v - b.v; for (int i = 0; i < N; ++i) r.d[i] = a.d[i] - b.d[i]; return r; }
template <class T, int N> Dual<T, N> operator*(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v * b.v;
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
  return r; }
template <class T, int N> Dual<T, N> operator*(const Dual<T, N>& a, double b) {
  Dual<T, N> r; r.v = a.v * b; for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b; return r; }
template <class T, int N> Dual<T, N> operator*(double a, const Dual<T, N>& b) { return b * a; }
template <class T, int N> Dual<T, N> operator/(const Dual<T, N>& a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a.v / b.v;
  for (int i = 0; i < N; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) / b.v;
  return r; }
template <class T, int N> Dual<T, N> operator/(const Dual<T, N>& a, double b) {
  Dual<T, N> r; r.v = a.v / b; for (int i = 0; i < N; ++i) r.d[i] = a.d[i] / b; return r; }
template <class T, int N> Dual<T, N> operator/(double a, const Dual<T, N>& b) {
  Dual<T, N> r; r.v = a / b.v;
  for (int i = 0; i < N; ++i) r.d[i] = -(r.v * b.d[i]) / b.v;
  return r; }
template <class T, int N, class U> Dual<T, N>& operator+=(Dual<T, N>& a, const U& b) { a = a + b; return a; }
template <class T, int N, class U> Dual<T, N>& operator-=(Dual<T, N>& a, const U& b) { a = a - b; return a; }
template <class T, int N, class U> Dual<T, N>& operator*=(Dual<T, N>& a, const U& b) { a = a * b; return a; }

// chain rule: value f, derivative fp (both of type T) applied to a's partials
template <class T, int N> Dual<T, N> chain(const Dual<T, N>& a, const T& f, const T& fp) {
  Dual<T, N> r; r.v = f; for (int i = 0; i < N; ++i) r.d[i] = fp * a.d[i]; return r; }

using std::exp; using std::log; using std::log1p; using std::sqrt; using std::cbrt;
using std::sin; using std::cos; using std::atan2;

template <class T, int N> Dual<T, N> exp(const Dual<T, N>& a) { T e = exp(a.v); return chain(a, e, e); }
template <class T, int N> Dual<T, N> log(const Dual<T, N>& a) { return chain(a, T(log(a.v)), T(1.0 / a.v)); }
template <class T, int N> Dual<T, N> log1p(const Dual<T, N>& a) { return chain(a, T(log1p(a.v)), T(1.0 / (1.0 + a.v))); }
template <class T, int N> Dual<T, N> sqrt(const Dual<T, N>& a) { T s = sqrt(a.v); return chain(a, s, T(0.5 / s)); }
template <class T, int N> Dual<T, N> cbrt(const Dual<T, N>& a) { T c = cbrt(a.v); return chain(a, c, T(1.0 / (3.0 * c * c))); }
template <class T, int N> Dual<T, N> sin(const Dual<T, N>& a) { return chain(a, T(sin(a.v)), T(cos(a.v))); }
template <class T, int N> Dual<T, N> cos(const Dual<T, N>& a) { return chain(a, T(cos(a.v)), T(-sin(a.v))); }
template <class T, int N> Dual<T, N> atan2(const Dual<T, N>& y, const Dual<T, N>& x) {
  Dual<T, N> r; r.v = atan2(y.v, x.v);
  T den = x.v * x.v + y.v * y.v;
  for (int i = 0; i < N; ++i) r.d[i] = (x.v * y.d[i] - y.v * x.d[i]) / den;
  return r; }

template <class T> T sq(const T& x) { return x * x; }

// ---------------------------------------------------------------------------
// Small vector helpers (templated on the scalar type)
// ---------------------------------------------------------------------------
template <class T> struct V3 { T x[3]; };
template <class T> T dot3(const T* a, const T* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
template <class T> void cross3(const T* a, const T* b, T* r) {
  r[0] = a[1] * b[2] - a[2] * b[1];
  r[1] = a[2] * b[0] - a[0] * b[2];
  r[2] = a[0] * b[1] - a[1] * b[0]; }

// ---------------------------------------------------------------------------
// Smooth parameters (Reading #1: five named temperatures; P:42-44 give one
// generic tau).
// ---------------------------------------------------------------------------
struct Smooth {
  double tau_cmp, tau_min, tau_clip_alpha, tau_clip_t, tau_delta;
  int trace_iters;
};

// ---------------------------------------------------------------------------
// §II-A smooth operators
// ---------------------------------------------------------------------------
// sigma(x) = 1/(1+exp(-x)); branch only selects the overflow-safe form
template <class T> T sigmoid(const T& x) {
  if (val(x) >= 0) return 1.0 / (1.0 + exp(-x));
  T e = exp(x);
  return e / (1.0 + e);
}
// s+(x) = tau log(1 + exp(x/tau)); two algebraically equal branches
template <class T> T softplus(const T& x, double tau) {
  if (val(x) > 0) return x + tau * log1p(exp(-x / tau));
  return tau * log1p(exp(x / tau));
}
// soft clip from two softplus: lo + s+(x-lo) - s+(x-hi)
template <class T> T softclip(const T& x, double lo, double hi, double tau) {
  return lo + softplus(x - lo, tau) - softplus(x - hi, tau);
}
// LSE(x) = tau log sum exp(x_i/tau), evaluated with the max shift
template <class T> T lse(const T* x, int n, double tau) {
  int im = 0;
  for (int i = 1; i < n; ++i) if (val(x[i]) > val(x[im])) im = i;
  T m = x[im];
  T s = T(0.0);
  for (int i = 0; i < n; ++i) s = s + exp((x[i] - m) / tau);
  return m + tau * log(s);
}
// s_argmax(x)_i = exp(x_i/tau) / sum_j exp(x_j/tau)
template <class T> void softargmax(const T* x, int n, double tau, T* out) {
  int im = 0;
  for (int i = 1; i < n; ++i) if (val(x[i]) > val(x[im])) im = i;
  T m = x[im];
  T s = T(0.0);
  for (int i = 0; i < n; ++i) { out[i] = exp((x[i] - m) / tau); s = s + out[i]; }
  for (int i = 0; i < n; ++i) out[i] = out[i] / s;
}

// ---------------------------------------------------------------------------
// Geometry records (oracle's own layout; filled by oracle/oracle.py)
// ---------------------------------------------------------------------------
enum { K_HALFSPACE = 0, K_SQ = 1, K_PSQ = 2, K_XPSQ = 3, K_UNION = 10, K_INTER = 11, K_SUB = 12 };
constexpr int MAXP = 8;       // planes per PSQ
constexpr int MAXC = 32;      // children per operator
constexpr int NI = 3 + MAXC;  // ints per node: type, n_children, n_planes, children[32]
constexpr int NF = 93;        // floats per node (see oracle.py)

struct Node {
  int type, n_children, n_planes;
  int child[MAXC];
  double t[3], R[9];       // pose relative to parent: x_parent = R x_child + t
  double eps[2][2];        // [endpoint][eps1, eps2]
  double a[2][3];          // [endpoint][a_x, a_y, a_z]
  double pl[2][MAXP][4];   // [endpoint][plane][n_x, n_y, n_z, h]
  double ctrl[9];          // XPSQ control points p1, p2, p3
  double up[3];            // XPSQ up hint
  // XPSQ static data (Reading #7/#14)
  int xcls;                // 0 point, 1 line, 2 curve
  int frenet;              // 1: Frenet frame with constant binormal
  double A[3], B[3], bhat[3], R0[9];
};

struct Mesh {
  int V = 0, F = 0, E = 0;
  std::vector<double> v;        // V x 3 local vertices
  std::vector<int> f;           // F x 3
  std::vector<int> e;           // E x 2  (lower index first)
  std::vector<int> fe;          // F x 3  edge ids of (i0,i1),(i1,i2),(i2,i0)
};

struct Shape {
  std::vector<Node> nodes;  // node 0 = root (empty => no SDF)
  Mesh mesh;
};

struct Scene {
  std::vector<Shape> shapes;
  Smooth sp;
};

// unit quaternion (w,x,y,z) -> rotation matrix (row-major), after normalising
static void quat_to_R(const double* q, double* R) {
  double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

static void normalize3(double* v) {
  double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  v[0] /= n; v[1] /= n; v[2] /= n;
}

// static XPSQ classification (Reading #7, #14): point / line / curve;
// Frenet frame when the spline is genuinely curved, else a constant frame
// built from the up hint by Gram-Schmidt.
constexpr double XPSQ_EPS_POINT = 1e-6;   // |A|,|B| below this: point spline
constexpr double XPSQ_EPS_LINE = 1e-4;    // |A| < 1e-4 |B|: snapped straight
constexpr double XPSQ_EPS_FRAME = 1e-3;   // |BxA| < 1e-3 |A||B|: constant frame

static void xpsq_static(Node& n) {
  const double* p1 = n.ctrl; const double* p2 = n.ctrl + 3; const double* p3 = n.ctrl + 6;
  for (int i = 0; i < 3; ++i) { n.A[i] = p1[i] - 2 * p2[i] + p3[i]; n.B[i] = 2 * (p2[i] - p1[i]); }
  double nA = std::sqrt(dot3(n.A, n.A)), nB = std::sqrt(dot3(n.B, n.B));
  double T0[3];
  if (nA < XPSQ_EPS_POINT && nB < XPSQ_EPS_POINT) {
    n.xcls = 0; T0[0] = 1; T0[1] = 0; T0[2] = 0;
  } else if (nA < XPSQ_EPS_LINE * nB) {
    // straight: the segment p1 -> p3 (the chord B := p3 - p1 = A + B, A := 0;
    // it keeps both end points and lies within |A|/4 of the spline)
    n.xcls = 1; for (int i = 0; i < 3; ++i) { n.B[i] += n.A[i]; n.A[i] = 0.0; T0[i] = n.B[i]; }
  } else {
    n.xcls = 2;
    for (int i = 0; i < 3; ++i) T0[i] = n.A[i] + n.B[i];
    if (std::sqrt(dot3(T0, T0)) < XPSQ_EPS_POINT) for (int i = 0; i < 3; ++i) T0[i] = nB > XPSQ_EPS_POINT ? n.B[i] : n.A[i];
  }
  double bxa[3]; cross3(n.B, n.A, bxa);
  n.frenet = (n.xcls == 2 && std::sqrt(dot3(bxa, bxa)) >= XPSQ_EPS_FRAME * nA * nB) ? 1 : 0;
  if (n.frenet) {
    for (int i = 0; i < 3; ++i) n.bhat[i] = bxa[i];
    normalize3(n.bhat);
  } else {
    normalize3(T0);
    double b[3] = {n.up[0], n.up[1], n.up[2]};
    if (n.xcls == 0) {
      // point spline: b = up, T0 = e_x made orthogonal to b
      normalize3(b);
      double e[3] = {1, 0, 0};
      double c = dot3(e, b);
      if (std::fabs(c) > 0.9) { e[0] = 0; e[1] = 1; c = dot3(e, b); }
      for (int i = 0; i < 3; ++i) T0[i] = e[i] - c * b[i];
      normalize3(T0);
    } else {
      double c = dot3(b, T0);
      for (int i = 0; i < 3; ++i) b[i] -= c * T0[i];
      normalize3(b);
    }
    for (int i = 0; i < 3; ++i) n.bhat[i] = b[i];
    double N[3]; cross3(n.bhat, T0, N);
    // R0 = [T0, N, b] as columns (row-major storage)
    for (int i = 0; i < 3; ++i) { n.R0[i * 3 + 0] = T0[i]; n.R0[i * 3 + 1] = N[i]; n.R0[i * 3 + 2] = n.bhat[i]; }
  }
}

// ---------------------------------------------------------------------------
// Leaf SDFs in the leaf's local frame
// ---------------------------------------------------------------------------
constexpr double SQ_GUARD = 1e-12;  // |u|^p = exp(p log(u^2 + g)/2)

// Half-space phi_N = x . n + h
template <class T> T halfspace_phi(const T* y, const T* nrm, const T& h) {
  return y[0] * nrm[0] + y[1] * nrm[1] + y[2] * nrm[2] + h;
}

// SQ inside-outside function, Eq. (1), with even powers
// (x/a)^(2/e) = ((x/a)^2)^(1/e) and the guard of S:261.
template <class T> T sq_f(const T* y, const T& e1, const T& e2, const T* a) {
  T u0 = y[0] / a[0], u1 = y[1] / a[1], u2 = y[2] / a[2];
  T A0 = exp(log(u0 * u0 + SQ_GUARD) / e2);
  T A1 = exp(log(u1 * u1 + SQ_GUARD) / e2);
  T C = exp(log(u2 * u2 + SQ_GUARD) / e1);
  return exp((e2 / e1) * log(A0 + A1)) + C;
}

// SQ radial distance phi = |y| (1 - f^(-e1/2))  (Reading #2, P:72 garbled)
template <class T> T sq_phi(const T* y, const T& e1, const T& e2, const T* a) {
  T f = sq_f(y, e1, e2, a);
  T r = sqrt(y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
  return r * (1.0 - exp(-(e1 / 2.0) * log(f)));
}

// PSQ: smooth intersection Eq. (3) of an SQ and N half-spaces
template <class T> T psq_phi(const T* y, const T& e1, const T& e2, const T* a,
                             int np, const T (*pl)[4], double tau_min) {
  T ops[1 + MAXP];
  ops[0] = sq_phi(y, e1, e2, a);
  for (int i = 0; i < np; ++i) ops[1 + i] = halfspace_phi(y, pl[i], pl[i][3]);
  if (np == 0) return ops[0];
  return lse(ops, 1 + np, tau_min);
}

// ---------------------------------------------------------------------------
// XPSQ: projection onto the quadratic spline by the cubic of
// P:112, soft Cardano (Eq. (6)), three PSQs, smooth minimum.
// ---------------------------------------------------------------------------
// Eq. (5): p(t) = (1-t)^2 p1 + 2t(1-t) p2 + t^2 p3 = p1 + B t + A t^2
// stationarity (x - p(t)) . p'(t) = 0 gives c3 t^3 + c2 t^2 + c1 t + c0 = 0
//   c3 = -2 A.A, c2 = -3 A.B, c1 = 2 A.w - B.B, c0 = B.w, w = x - p1
//
// Soft Cardano, literal (Reading #9, #10, #11, #12, #13):
//   depressed cubic s^3 + P s + Q = 0 with t = s - b/3,
//   Delta = -(4P^3 + 27Q^2); Delta- = -s+(-Delta), Delta+ = s+(Delta);
//   t-  = Cardano real root with Delta- substituted,
//   t+k = trigonometric form with Delta+ substituted, k = 0, 1, 2;
//   both soft-clipped to (0,1);  t*_k = sig(-Delta/tau) t- + sig(Delta/tau) t+_k
// The spline's static data as a type S: double (the node's own values) or a
// jet type when the control points are seeded (shape parameters, f4): p1, A,
// B, the Frenet binormal and the constant frame, by the rule of xpsq_static
// (the class, frenet flag and snap decided on the values).
template <class S> struct XS { S p1[3], A[3], B[3], bhat[3], R0[9]; };
static XS<double> xs_plain(const Node& n) {
  XS<double> x;
  for (int i = 0; i < 3; ++i) { x.p1[i] = n.ctrl[i]; x.A[i] = n.A[i]; x.B[i] = n.B[i]; x.bhat[i] = n.bhat[i]; }
  for (int i = 0; i < 9; ++i) x.R0[i] = n.R0[i];
  return x;
}
template <class S> void normalize3t(S* v) {
  S nn = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  for (int i = 0; i < 3; ++i) v[i] = v[i] / nn;
}
template <class S> XS<S> xs_seeded(const Node& n, const S* ctrl) {
  XS<S> x;
  const S* p1 = ctrl; const S* p2 = ctrl + 3; const S* p3 = ctrl + 6;
  for (int i = 0; i < 3; ++i) { x.p1[i] = p1[i]; x.A[i] = p1[i] - 2.0 * p2[i] + p3[i]; x.B[i] = 2.0 * (p2[i] - p1[i]); }
  S T0[3];
  if (n.xcls == 0) {
    for (int i = 0; i < 3; ++i) T0[i] = S(0.0);
  } else if (n.xcls == 1) {
    for (int i = 0; i < 3; ++i) { x.B[i] = x.B[i] + x.A[i]; x.A[i] = S(0.0); T0[i] = x.B[i]; }
  } else {
    for (int i = 0; i < 3; ++i) T0[i] = x.A[i] + x.B[i];
    double t0v[3] = {val(T0[0]), val(T0[1]), val(T0[2])};
    if (std::sqrt(dot3(t0v, t0v)) < XPSQ_EPS_POINT) {
      double nB = std::sqrt(dot3(n.B, n.B));
      for (int i = 0; i < 3; ++i) T0[i] = nB > XPSQ_EPS_POINT ? x.B[i] : x.A[i];
    }
  }
  if (n.frenet) {
    cross3(x.B, x.A, x.bhat);
    normalize3t(x.bhat);
    for (int i = 0; i < 9; ++i) x.R0[i] = S(n.R0[i]);
    return x;
  }
  S b[3] = {S(n.up[0]), S(n.up[1]), S(n.up[2])};
  if (n.xcls == 0) {   // point spline: the frame from the up hint only
    for (int i = 0; i < 3; ++i) x.bhat[i] = S(n.bhat[i]);
    for (int i = 0; i < 9; ++i) x.R0[i] = S(n.R0[i]);
    return x;
  }
  normalize3t(T0);
  S c = b[0] * T0[0] + b[1] * T0[1] + b[2] * T0[2];
  for (int i = 0; i < 3; ++i) b[i] = b[i] - c * T0[i];
  normalize3t(b);
  for (int i = 0; i < 3; ++i) x.bhat[i] = b[i];
  S N[3]; cross3(x.bhat, T0, N);
  for (int i = 0; i < 3; ++i) { x.R0[i * 3 + 0] = T0[i]; x.R0[i * 3 + 1] = N[i]; x.R0[i * 3 + 2] = x.bhat[i]; }
  return x;
}
template <class T> T as_t(double v) { return T(v); }
template <class T> T as_t(const T& v) { return v; }

template <class T, class S> void xpsq_roots(const Node& n, const XS<S>& xs, const T* y, const Smooth& sp, T* tk,
                                            double* delta_out, double* wneg_out) {
  const S* p1 = xs.p1;
  T w[3] = {y[0] - p1[0], y[1] - p1[1], y[2] - p1[2]};
  if (delta_out) *delta_out = 0.0;
  if (wneg_out) *wneg_out = 0.0;
  if (n.xcls == 0) {  // point spline: any t projects to the same point
    for (int k = 0; k < 3; ++k) tk[k] = T(0.5);
    return;
  }
  const S* A = xs.A; const S* B = xs.B;
  T Bw = w[0] * B[0] + w[1] * B[1] + w[2] * B[2];
  S BB = dot3(B, B);
  if (n.xcls == 1) {  // straight spline: the cubic degenerates to B.w - t B.B = 0
    T t = softclip(Bw / BB, 0.0, 1.0, sp.tau_clip_t);
    for (int k = 0; k < 3; ++k) tk[k] = t;
    return;
  }
  S c3 = -2.0 * dot3(A, A);
  S c2 = -3.0 * dot3(A, B);
  T c1 = 2.0 * (w[0] * A[0] + w[1] * A[1] + w[2] * A[2]) - BB;
  T c0 = Bw;
  S b = c2 / c3;
  T c = c1 / c3, d = c0 / c3;
  T P = c - b * b / 3.0;
  T Q = 2.0 * b * b * b / 27.0 - b * c / 3.0 + d;
  T Delta = -(4.0 * P * P * P + 27.0 * Q * Q);
  T Dm = -softplus(-Delta, sp.tau_delta);
  T Dp = softplus(Delta, sp.tau_delta);
  T wneg = sigmoid(-Delta / sp.tau_delta);
  T wpos = sigmoid(Delta / sp.tau_delta);
  if (delta_out) *delta_out = val(Delta);
  if (wneg_out) *wneg_out = val(wneg);
  T tm = T(0.0), tp[3] = {T(0.0), T(0.0), T(0.0)};
  // A branch whose weight is below 1e-200 is skipped (reading #34):
  // its value contribution is < 1e-200 and its derivative contributions are
  // O(sqrt(weight)) (the branch's degenerate square / cube roots scale like
  // the projected discriminant s+(-|Delta|) ~ tau * weight), i.e. zero at FP64
  // resolution, while evaluating it literally would form 0 * inf in the jets
  // once s+ underflows (|Delta|/tau > ~740).
  const double W_SKIP = 1e-200;
  if (val(wneg) > W_SKIP) {
    T D = -Dm / 108.0;
    T sD = sqrt(D);
    // Cardano s = cbrt(-Q/2 + sqrt(D)) + cbrt(-Q/2 - sqrt(D)), evaluated in
    // its cancellation-free form (reading #37): u = the term whose
    // radicand does not cancel, v = cbrt(Q^2/4 - D) / u (the product of the two
    // cube roots), with Q^2/4 - D = -(P^3 + s+(Delta)/4)/27 (exact identity,
    // since -Delta- = s+(-Delta) = -Delta + s+(Delta) and -Delta = 4P^3 + 27Q^2).
    // Term-by-term evaluation loses every digit of the smaller radicand when
    // |P|^3 << Q^2 and returns non-finite derivatives (radicand rounded to 0).
    T u = val(Q) >= 0.0 ? cbrt(-Q / 2.0 - sD) : cbrt(-Q / 2.0 + sD);
    T prod = cbrt(-(P * P * P + softplus(Delta, sp.tau_delta) / 4.0) / 27.0);
    T s = val(u) != 0.0 ? u + prod / u : u;
    tm = softclip(s - b / 3.0, 0.0, 1.0, sp.tau_clip_t);
  }
  if (val(wpos) > W_SKIP) {
    T rho = exp(log(Q * Q / 4.0 + Dp / 108.0) / 6.0);
    T th = atan2(sqrt(Dp / 108.0), -Q / 2.0);
    for (int k = 0; k < 3; ++k) {
      T s = 2.0 * rho * cos((th + 2.0 * M_PI * k) / 3.0);
      tp[k] = softclip(s - b / 3.0, 0.0, 1.0, sp.tau_clip_t);
    }
  }
  for (int k = 0; k < 3; ++k) {
    if (val(wneg) > W_SKIP && val(wpos) > W_SKIP) tk[k] = wneg * tm + wpos * tp[k];
    else if (val(wneg) > W_SKIP) tk[k] = wneg * tm;
    else tk[k] = wpos * tp[k];
  }
}

// moving frame R(t) ("e.g. the Frenet frame"; Reading #7), row-major,
// columns [T, bhat x T, bhat]
template <class T, class S> void xpsq_frame(const Node& n, const XS<S>& xs, const T& t, T* R) {
  if (!n.frenet) { for (int i = 0; i < 9; ++i) R[i] = as_t<T>(xs.R0[i]); return; }
  T pd[3];
  for (int i = 0; i < 3; ++i) pd[i] = xs.B[i] + 2.0 * xs.A[i] * t;
  T nn = sqrt(pd[0] * pd[0] + pd[1] * pd[1] + pd[2] * pd[2]);
  T Tt[3] = {pd[0] / nn, pd[1] / nn, pd[2] / nn};
  T bh[3] = {as_t<T>(xs.bhat[0]), as_t<T>(xs.bhat[1]), as_t<T>(xs.bhat[2])};
  T N[3]; cross3(bh, Tt, N);
  for (int i = 0; i < 3; ++i) { R[i * 3 + 0] = Tt[i]; R[i * 3 + 1] = N[i]; R[i * 3 + 2] = bh[i]; }
}

template <class T> T lerp(double a, double b, const T& t) { return a + (b - a) * t; }

template <class T> T pval(double v, int node, int slot);
extern thread_local int g_seed_node, g_seed_slot;
// an XPSQ's schedules differ between its endpoints (any of eps, a, planes)
static bool xpsq_varying(const Node& n) {
  bool cst = n.eps[0][0] == n.eps[1][0] && n.eps[0][1] == n.eps[1][1];
  for (int i = 0; i < 3; ++i) cst = cst && n.a[0][i] == n.a[1][i];
  for (int j = 0; j < n.n_planes; ++j) for (int i = 0; i < 4; ++i) cst = cst && n.pl[0][j][i] == n.pl[1][j][i];
  return !cst;
}
template <class T, class S>
T xpsq_phi_s(const Node& n, const XS<S>& xs, const T* y, const Smooth& sp, int idx);
template <class T> T xpsq_phi(const Node& n, const T* y, const Smooth& sp, int idx = -1) {
  // control points seeded (f4 shape parameters: slots base .. base + 8 after
  // the cross-section's, base = (varying ? 2 : 1) (5 + 4 n_planes)): the
  // spline's static data as jets
  const int base = (xpsq_varying(n) ? 2 : 1) * (5 + 4 * n.n_planes);
  if (idx >= 0 && idx == g_seed_node && g_seed_slot >= base && g_seed_slot < base + 9) {
    T c[9];
    for (int i = 0; i < 9; ++i) c[i] = pval<T>(n.ctrl[i], idx, base + i);
    return xpsq_phi_s(n, xs_seeded<T>(n, c), y, sp, idx);
  }
  return xpsq_phi_s(n, xs_plain(n), y, sp, idx);
}
template <class T, class S>
T xpsq_phi_s(const Node& n, const XS<S>& xs, const T* y, const Smooth& sp, int idx) {
  T tk[3];
  xpsq_roots(n, xs, y, sp, tk, nullptr, nullptr);
  T phis[3];
  for (int k = 0; k < 3; ++k) {
    const T& t = tk[k];
    // PSQ pose at the root: translation p(t) (Eq. (5)), rotation R(t)
    T pt[3];
    for (int i = 0; i < 3; ++i) pt[i] = xs.p1[i] + xs.B[i] * t + xs.A[i] * (t * t);
    T R[9];
    xpsq_frame(n, xs, t, R);
    T dx[3] = {y[0] - pt[0], y[1] - pt[1], y[2] - pt[2]};
    T yk[3];
    for (int i = 0; i < 3; ++i) yk[i] = R[0 * 3 + i] * dx[0] + R[1 * 3 + i] * dx[1] + R[2 * 3 + i] * dx[2];
    // schedules eps(t), a(t), P(t): linear between endpoint values, plane
    // normals renormalised (Reading #8)
    // (shape-parameter seeds, f4: with constant schedules one slot moves
    // both endpoint values; with varying schedules slot s is the t = 0 value
    // and slot M + s the t = 1 value, M = 5 + 4 n_planes)
    const int M = 5 + 4 * n.n_planes;
    const bool vary = xpsq_varying(n);
    auto L2 = [&](double v0, double v1, int slot) {
      if (idx != g_seed_node) return lerp(v0, v1, t);          // (no seed: the literal schedule)
      const T a0 = pval<T>(v0, idx, slot), a1 = pval<T>(v1, idx, vary ? M + slot : slot);
      return a0 + (a1 - a0) * t;
    };
    T e1 = L2(n.eps[0][0], n.eps[1][0], 3);
    T e2 = L2(n.eps[0][1], n.eps[1][1], 4);
    T a[3];
    for (int i = 0; i < 3; ++i) a[i] = L2(n.a[0][i], n.a[1][i], i);
    T pl[MAXP][4];
    for (int j = 0; j < n.n_planes; ++j) {
      T nv[3];
      for (int i = 0; i < 3; ++i) nv[i] = L2(n.pl[0][j][i], n.pl[1][j][i], 5 + 4 * j + i);
      T nn = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
      for (int i = 0; i < 3; ++i) pl[j][i] = nv[i] / nn;
      pl[j][3] = L2(n.pl[0][j][3], n.pl[1][j][3], 8 + 4 * j);
    }
    phis[k] = psq_phi(yk, e1, e2, a, n.n_planes, pl, sp.tau_min);
  }
  // smooth minimum of the three PSQ SDFs
  T neg[3] = {-phis[0], -phis[1], -phis[2]};
  return -lse(neg, 3, sp.tau_min);
}

// ---------------------------------------------------------------------------
// Shape-parameter seeding: the parameter (node, slot) named
// by the calling thread's g_seed carries the derivative direction of a
// Dual<double,1>; every other jet type ignores it.  Slots per node:
// half-space (n_x, n_y, n_z, h); SQ (a_x, a_y, a_z, eps1, eps2); PSQ as SQ
// then (n_x, n_y, n_z, h) per plane.
// ---------------------------------------------------------------------------
thread_local int g_seed_node = -1, g_seed_slot = -1;
// manifold shape-parameter derivatives (f4, reading #48): with this flag set
// the manifold's pose jets are not seeded and the shape parameter named by
// g_seed takes their component 0 (the first-order q-jet D12 and the nested
// candidate jet N12 = Dual<D3, 12>), so ddepth[., 0] = d depth / d param
thread_local bool g_param_comp0 = false;
thread_local int g_param_shape = -1;   // the seeded parameters' shape (its SDF sides only)
template <class T> struct Seeder { static void apply(T&) {} };
template <> struct Seeder<Dual<double, 1>> { static void apply(Dual<double, 1>& x) { x.d[0] = 1.0; } };
template <> struct Seeder<Dual<double, 12>> {
  static void apply(Dual<double, 12>& x) { if (g_param_comp0) x.d[0] = 1.0; }
};
template <> struct Seeder<Dual<Dual<double, 3>, 12>> {
  static void apply(Dual<Dual<double, 3>, 12>& x) { if (g_param_comp0) x.d[0].v = 1.0; }
};
template <class T> T pval(double v, int node, int slot) {
  T x(v);
  if (node == g_seed_node && slot == g_seed_slot) Seeder<T>::apply(x);
  return x;
}

// ---------------------------------------------------------------------------
// Composite tree (Eqs. (2)-(4); n-ary single LSE, Reading #5;
// subtraction LSE([phi1, -phi2]), Reading #4).  Each node has a pose relative
// to its parent; y is in the parent frame.
// ---------------------------------------------------------------------------
// Node-pose seeding (node poses; DESIGN reading #47): the
// twist (dt, dtheta) of node g_pose_node's pose in its parent frame, slots
// 0-2 dt, 3-5 dtheta, with the body poses' convention (reading #28):
// R <- exp([dtheta]x) R, t <- t + dt, where x_parent = R x_node + t.
thread_local int g_pose_node = -1, g_pose_slot = -1;
template <class T> T pose_seed(int idx, int slot) {
  T x(0.0);
  if (idx == g_pose_node && slot == g_pose_slot) Seeder<T>::apply(x);
  return x;
}
template <class T> void perturbed_pose(const double* R, const double* t, const T* dt, const T* w, T* Rp, T* tp);

template <class T> T node_phi(const Shape& sh, int idx, const T* yparent, const Smooth& sp) {
  const Node& n = sh.nodes[idx];
  T y[3];
  if (idx == g_pose_node) {   // the seeded node: its perturbed pose
    T dt[3], w[3], Rp[9], tp[3];
    for (int i = 0; i < 3; ++i) { dt[i] = pose_seed<T>(idx, i); w[i] = pose_seed<T>(idx, 3 + i); }
    perturbed_pose(n.R, n.t, dt, w, Rp, tp);
    T dx[3] = {yparent[0] - tp[0], yparent[1] - tp[1], yparent[2] - tp[2]};
    for (int i = 0; i < 3; ++i) y[i] = Rp[0 * 3 + i] * dx[0] + Rp[1 * 3 + i] * dx[1] + Rp[2 * 3 + i] * dx[2];
  } else {
    T dx[3] = {yparent[0] - n.t[0], yparent[1] - n.t[1], yparent[2] - n.t[2]};
    for (int i = 0; i < 3; ++i) y[i] = n.R[0 * 3 + i] * dx[0] + n.R[1 * 3 + i] * dx[1] + n.R[2 * 3 + i] * dx[2];
  }
  switch (n.type) {
    case K_HALFSPACE: {
      T nv[3] = {pval<T>(n.pl[0][0][0], idx, 0), pval<T>(n.pl[0][0][1], idx, 1), pval<T>(n.pl[0][0][2], idx, 2)};
      return halfspace_phi(y, nv, pval<T>(n.pl[0][0][3], idx, 3));
    }
    case K_SQ: case K_PSQ: {
      T a[3] = {pval<T>(n.a[0][0], idx, 0), pval<T>(n.a[0][1], idx, 1), pval<T>(n.a[0][2], idx, 2)};
      T pl[MAXP][4];
      int np = n.type == K_SQ ? 0 : n.n_planes;
      for (int j = 0; j < np; ++j) for (int i = 0; i < 4; ++i) pl[j][i] = pval<T>(n.pl[0][j][i], idx, 5 + 4 * j + i);
      return psq_phi(y, pval<T>(n.eps[0][0], idx, 3), pval<T>(n.eps[0][1], idx, 4), a, np, pl, sp.tau_min);
    }
    case K_XPSQ:
      return xpsq_phi(n, y, sp, idx);
    default: {
      std::vector<T> ops(n.n_children);
      for (int c = 0; c < n.n_children; ++c) ops[c] = node_phi(sh, n.child[c], y, sp);
      if (n.type == K_UNION) {                       // Eq. (2): -LSE(-phi)
        for (auto& o : ops) o = -o;
        return -lse(ops.data(), n.n_children, sp.tau_min);
      }
      if (n.type == K_INTER)                         // Eq. (3): LSE(phi)
        return lse(ops.data(), n.n_children, sp.tau_min);
      ops[1] = -ops[1];                              // Eq. (4): LSE(phi1, -phi2)
      return lse(ops.data(), 2, sp.tau_min);
    }
  }
}

// SDF of a shape placed with rotation R and translation t (body pose) at the
// world point x: phi(R^T (x - t))
template <class T> T shape_phi_world(const Shape& sh, const T* R, const T* t, const T* x, const Smooth& sp) {
  T dx[3] = {x[0] - t[0], x[1] - t[1], x[2] - t[2]};
  T y[3];
  for (int i = 0; i < 3; ++i) y[i] = R[0 * 3 + i] * dx[0] + R[1 * 3 + i] * dx[1] + R[2 * 3 + i] * dx[2];
  return node_phi(sh, 0, y, sp);
}

// ---------------------------------------------------------------------------
// Mesh topology: unique edges keyed by the
// sorted vertex pair; face_edges in the order (i0,i1), (i1,i2), (i2,i0).
// ---------------------------------------------------------------------------
static void build_topology(Mesh& m) {
  std::map<std::pair<int, int>, int> key;
  m.e.clear(); m.fe.assign(3 * m.F, -1);
  for (int f = 0; f < m.F; ++f) {
    for (int k = 0; k < 3; ++k) {
      int a = m.f[3 * f + k], b = m.f[3 * f + (k + 1) % 3];
      std::pair<int, int> p(std::min(a, b), std::max(a, b));
      auto it = key.find(p);
      int id;
      if (it == key.end()) { id = (int)(m.e.size() / 2); key[p] = id; m.e.push_back(p.first); m.e.push_back(p.second); }
      else id = it->second;
      m.fe[3 * f + k] = id;
    }
  }
  m.E = (int)(m.e.size() / 2);
}

// ---------------------------------------------------------------------------
// Perturbed poses: world-frame left perturbation R <- exp([w]x) R, t <- t + dt
// (Reading #28); exp truncated after the quadratic term, exact to second
// order at w = 0 (all that first and second derivatives need).
// ---------------------------------------------------------------------------
template <class T> void perturbed_pose(const double* R, const double* t, const T* dt, const T* w, T* Rp, T* tp) {
  T W[9] = {T(0.0), -w[2], w[1], w[2], T(0.0), -w[0], -w[1], w[0], T(0.0)};
  T W2[9];
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j)
    W2[i * 3 + j] = W[i * 3 + 0] * W[0 * 3 + j] + W[i * 3 + 1] * W[1 * 3 + j] + W[i * 3 + 2] * W[2 * 3 + j];
  T E[9];
  for (int i = 0; i < 9; ++i) E[i] = W[i] + 0.5 * W2[i];
  for (int i = 0; i < 3; ++i) E[i * 3 + i] = E[i * 3 + i] + 1.0;
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j)
    Rp[i * 3 + j] = E[i * 3 + 0] * R[0 * 3 + j] + E[i * 3 + 1] * R[1 * 3 + j] + E[i * 3 + 2] * R[2 * 3 + j];
  for (int i = 0; i < 3; ++i) tp[i] = t[i] + dt[i];
}

using D3 = Dual<double, 3>;
using H3 = Dual<D3, 3>;
using D6 = Dual<double, 6>;
using D12 = Dual<double, 12>;
using N12 = Dual<D3, 12>;

}  // namespace orc

using namespace orc;

// ============================================================================
// extern "C" interface (test infrastructure)
// ============================================================================
extern "C" {

int ora_version(void) { return 1; }

void* ora_scene_create(int n_shapes, const int* node_counts, const int* node_ints, const float* node_floats,
                       const int* mesh_vcounts, const float* mesh_v, const int* mesh_fcounts, const int* mesh_f,
                       const double* smooth, int trace_iters) {
  Scene* sc = new Scene;
  sc->sp = Smooth{smooth[0], smooth[1], smooth[2], smooth[3], smooth[4], trace_iters};
  sc->shapes.resize(n_shapes);
  int ni = 0, vi = 0, fi = 0;
  for (int s = 0; s < n_shapes; ++s) {
    Shape& sh = sc->shapes[s];
    sh.nodes.resize(node_counts[s]);
    for (int k = 0; k < node_counts[s]; ++k, ++ni) {
      Node& n = sh.nodes[k];
      const int* I = node_ints + (size_t)ni * NI;
      const float* Fv = node_floats + (size_t)ni * NF;
      n.type = I[0]; n.n_children = I[1]; n.n_planes = I[2];
      for (int c = 0; c < MAXC; ++c) n.child[c] = I[3 + c];
      for (int i = 0; i < 3; ++i) n.t[i] = Fv[i];
      double q[4] = {Fv[3], Fv[4], Fv[5], Fv[6]};
      quat_to_R(q, n.R);
      int o = 7;
      for (int e = 0; e < 2; ++e) for (int i = 0; i < 2; ++i) n.eps[e][i] = Fv[o++];
      for (int e = 0; e < 2; ++e) for (int i = 0; i < 3; ++i) n.a[e][i] = Fv[o++];
      for (int e = 0; e < 2; ++e) for (int j = 0; j < MAXP; ++j) for (int i = 0; i < 4; ++i) n.pl[e][j][i] = Fv[o++];
      for (int i = 0; i < 9; ++i) n.ctrl[i] = Fv[o++];
      for (int i = 0; i < 3; ++i) n.up[i] = Fv[o++];
      if (n.type == K_XPSQ) xpsq_static(n);
    }
    Mesh& m = sh.mesh;
    m.V = mesh_vcounts[s]; m.F = mesh_fcounts[s];
    m.v.resize(3 * m.V); m.f.resize(3 * m.F);
    for (int i = 0; i < 3 * m.V; ++i) m.v[i] = mesh_v[3 * vi + i];
    for (int i = 0; i < 3 * m.F; ++i) m.f[i] = mesh_f[3 * fi + i];
    vi += m.V; fi += m.F;
    if (m.F > 0) build_topology(m);
  }
  return sc;
}

void ora_scene_destroy(void* s) { delete (Scene*)s; }

int ora_mesh_counts(void* s, int shape, int* V, int* E, int* F) {
  Scene* sc = (Scene*)s;
  const Mesh& m = sc->shapes[shape].mesh;
  *V = m.V; *E = m.E; *F = m.F;
  return 0;
}
int ora_mesh_topology(void* s, int shape, int* edges, int* face_edges) {
  Scene* sc = (Scene*)s;
  const Mesh& m = sc->shapes[shape].mesh;
  std::memcpy(edges, m.e.data(), sizeof(int) * 2 * m.E);
  std::memcpy(face_edges, m.fe.data(), sizeof(int) * 3 * m.F);
  return 0;
}

// ---- unit entry points (pins) ----------------------------------------------
double ora_sigmoid(double x) { return sigmoid(x); }
double ora_softplus(double x, double tau) { return softplus(x, tau); }
double ora_softclip(double x, double lo, double hi, double tau) { return softclip(x, lo, hi, tau); }
double ora_lse(const double* x, int n, double tau) { return lse(x, n, tau); }
void ora_softargmax(const double* x, int n, double tau, double* out) { softargmax(x, n, tau, out); }
double ora_sq_f(const double* y, double e1, double e2, const double* a) { return sq_f(y, e1, e2, a); }
double ora_sq_phi(const double* y, double e1, double e2, const double* a) { return sq_phi(y, e1, e2, a); }

// XPSQ projection internals for node `node` of shape `shape`: t*, Delta, w_neg
void ora_xpsq_roots(void* s, int shape, int node, const double* y, double* t, double* delta, double* wneg) {
  Scene* sc = (Scene*)s;
  const Node& nd = sc->shapes[shape].nodes[node];
  xpsq_roots(nd, xs_plain(nd), y, sc->sp, t, delta, wneg);
}
// moving frame of an XPSQ node at parameter t (row-major 3x3)
void ora_xpsq_frame(void* s, int shape, int node, double t, double* R) {
  Scene* sc = (Scene*)s;
  const Node& nd = sc->shapes[shape].nodes[node];
  xpsq_frame(nd, xs_plain(nd), t, R);
}
int ora_xpsq_class(void* s, int shape, int node) {
  Scene* sc = (Scene*)s;
  const Node& n = sc->shapes[shape].nodes[node];
  return n.xcls * 10 + n.frenet;
}

// ---- sdf_eval ----------------------------------------------------------------
// For batch item b (shape_ids[b], pose poses[b] = t(3), q(w,x,y,z), pad) and
// its P points (world), computes d, grad (3), hess (6: xx,xy,xz,yy,yz,zz),
// and, if want_pose, dpose (6: d/dt, d/dtheta), d2pose (21: packed upper 6x6,
// row-major), dxdpose (18: [i*6+j] = d(grad_i)/d(pose_j)).  Output layout:
// point-major (n = b*P + j), field-minor.
int ora_sdf_eval(void* s, const int* shape_ids, const double* poses, const double* points, long B, long P,
                 int want_pose, double* d, double* g, double* h, double* dpose, double* d2pose, double* dxdpose) {
  Scene* sc = (Scene*)s;
  const Smooth& sp = sc->sp;
  long total = B * P;
#pragma omp parallel for schedule(dynamic, 16)
  for (long n = 0; n < total; ++n) {
    long b = n / P;
    const Shape& sh = sc->shapes[shape_ids[b]];
    const double* pz = poses + 8 * b;
    double R[9], t[3] = {pz[0], pz[1], pz[2]};
    double q[4] = {pz[3], pz[4], pz[5], pz[6]};
    quat_to_R(q, R);
    // value, gradient, Hessian: hyper-dual jet in the world point
    H3 X[3];
    for (int i = 0; i < 3; ++i) {
      X[i] = H3(0.0);
      X[i].v.v = points[3 * n + i];
      X[i].v.d[i] = 1.0;
      X[i].d[i].v = 1.0;
    }
    H3 Rj[9], tj[3];
    for (int i = 0; i < 9; ++i) Rj[i] = H3(R[i]);
    for (int i = 0; i < 3; ++i) tj[i] = H3(t[i]);
    H3 phi = shape_phi_world(sh, Rj, tj, X, sp);
    d[n] = phi.v.v;
    for (int i = 0; i < 3; ++i) g[3 * n + i] = phi.v.d[i];
    const int hi[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    for (int k = 0; k < 6; ++k) h[6 * n + k] = phi.d[hi[k][0]].d[hi[k][1]];
    if (want_pose) {
      // second order in the 6 pose seeds
      using P6 = Dual<D6, 6>;
      P6 dt[3], w[3], Rp[9], tp[3], Xp[3];
      for (int i = 0; i < 3; ++i) {
        dt[i] = P6(0.0); dt[i].v.d[i] = 1.0; dt[i].d[i].v = 1.0;
        w[i] = P6(0.0); w[i].v.d[3 + i] = 1.0; w[i].d[3 + i].v = 1.0;
        Xp[i] = P6(points[3 * n + i]);
      }
      perturbed_pose(R, t, dt, w, Rp, tp);
      P6 ph = shape_phi_world(sh, Rp, tp, Xp, sp);
      for (int j = 0; j < 6; ++j) dpose[6 * n + j] = ph.v.d[j];
      int k = 0;
      for (int i = 0; i < 6; ++i) for (int j = i; j < 6; ++j) d2pose[21 * n + k++] = ph.d[i].d[j];
      // mixed: outer pose seeds, inner point seeds
      using M6 = Dual<D3, 6>;
      M6 dtm[3], wm[3], Rm[9], tm[3], Xm[3];
      for (int i = 0; i < 3; ++i) {
        dtm[i] = M6(0.0); dtm[i].d[i].v = 1.0;
        wm[i] = M6(0.0); wm[i].d[3 + i].v = 1.0;
        Xm[i] = M6(0.0); Xm[i].v.v = points[3 * n + i]; Xm[i].v.d[i] = 1.0;
      }
      perturbed_pose(R, t, dtm, wm, Rm, tm);
      M6 pm = shape_phi_world(sh, Rm, tm, Xm, sp);
      for (int i = 0; i < 3; ++i) for (int j = 0; j < 6; ++j) dxdpose[18 * n + i * 6 + j] = pm.d[j].d[i];
    }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Broad phase ("utilizing [a broad phase] to filter
// edges prior to passing them to the edge-SDF routine"; DESIGN.md reading
// #46).  A pair is culled when a certified lower bound of the SDF over every
// candidate of the sampled surface exceeds M = 40 tau_cmp (every gate
// sigma(-d/tau_cmp) is then below e^-40): every candidate lies in the convex
// hull of the sampled vertices, inside their bounding sphere (c_A, r_A), and
// phi_B(x) >= |x - c_B| - rho_B, so d_i >= |c_A - c_B| - r_A - rho_B =: lb.
// Bounds of phi_B, in the node frames composed down the tree:
//   SQ / PSQ: the SQ lies in the box |y_i| <= a_i (eps <= 2) and the radial
//     distance is |y| minus the surface radius along the ray, so phi >= |y| -
//     |a|_2 (PSQ = LSE(SQ, planes) >= SQ);
//   XPSQ: the spline lies in its control points' box; phi >= |x - c| - (half
//     the box diagonal + max_e |a_e|_2 + tau_min ln 3) (three-root smooth min
//     >= min - tau ln 3);
//   half-space: unbounded below (no bound);
//   union: -LSE(-phi_i) >= min_i phi_i - tau_min ln n >= |x - c| - max_i(|c_i
//     - c| + rho_i) - tau_min ln n;  intersection LSE(phi_i) >= any phi_i: the
//     child with the smallest radius;  subtraction LSE(phi_1, -phi_2) >= phi_1.
// A culled pair's rows: point = the face centroid (full mode: the vertex /
// edge midpoint), depth = lb - tau_min ln 6 (full mode: lb), a certified lower
// bound of the fused depth; normal, W, q, derivatives, J, z, gamma = 0;
// dcand = lb; dom = -2.
// ---------------------------------------------------------------------------
struct OBound { double c[3]; double rho; };   // rho = +inf: no bound

static OBound node_bound(const Shape& sh, int idx, const double* Rp, const double* tp, double tau_min) {
  const Node& n = sh.nodes[idx];
  double R[9], t[3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) R[i * 3 + j] = Rp[i * 3 + 0] * n.R[0 * 3 + j] + Rp[i * 3 + 1] * n.R[1 * 3 + j] + Rp[i * 3 + 2] * n.R[2 * 3 + j];
  for (int i = 0; i < 3; ++i) t[i] = Rp[i * 3 + 0] * n.t[0] + Rp[i * 3 + 1] * n.t[1] + Rp[i * 3 + 2] * n.t[2] + tp[i];
  OBound b;
  b.rho = INFINITY;
  for (int i = 0; i < 3; ++i) b.c[i] = t[i];
  switch (n.type) {
    case K_HALFSPACE: return b;
    case K_SQ: case K_PSQ:
      b.rho = std::sqrt(dot3(n.a[0], n.a[0]));
      return b;
    case K_XPSQ: {
      double lo[3], hi[3], cl[3], h2 = 0.0;
      for (int i = 0; i < 3; ++i) {
        lo[i] = std::min({n.ctrl[i], n.ctrl[3 + i], n.ctrl[6 + i]});
        hi[i] = std::max({n.ctrl[i], n.ctrl[3 + i], n.ctrl[6 + i]});
        cl[i] = 0.5 * (lo[i] + hi[i]);
        h2 += 0.25 * (hi[i] - lo[i]) * (hi[i] - lo[i]);
      }
      const double am = std::max(std::sqrt(dot3(n.a[0], n.a[0])), std::sqrt(dot3(n.a[1], n.a[1])));
      for (int i = 0; i < 3; ++i) b.c[i] = R[i * 3 + 0] * cl[0] + R[i * 3 + 1] * cl[1] + R[i * 3 + 2] * cl[2] + t[i];
      b.rho = std::sqrt(h2) + am + tau_min * std::log(3.0);
      return b;
    }
    default: break;
  }
  std::vector<OBound> ch;
  for (int c = 0; c < n.n_children; ++c) ch.push_back(node_bound(sh, n.child[c], R, t, tau_min));
  if (n.type == K_SUB) return ch[0];
  if (n.type == K_INTER) {
    for (const OBound& x : ch) if (x.rho < b.rho) b = x;
    return b;
  }
  // union
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (const OBound& x : ch) {
    if (!(x.rho < INFINITY)) return b;   // an unbounded operand
    for (int i = 0; i < 3; ++i) { lo[i] = std::min(lo[i], x.c[i]); hi[i] = std::max(hi[i], x.c[i]); }
  }
  for (int i = 0; i < 3; ++i) b.c[i] = 0.5 * (lo[i] + hi[i]);
  double r = 0.0;
  for (const OBound& x : ch) {
    const double d[3] = {x.c[0] - b.c[0], x.c[1] - b.c[1], x.c[2] - b.c[2]};
    r = std::max(r, std::sqrt(dot3(d, d)) + x.rho);
  }
  b.rho = r + tau_min * std::log((double)ch.size());
  return b;
}

static OBound shape_bound(const Shape& sh, double tau_min) {
  OBound b;
  b.rho = INFINITY;
  b.c[0] = b.c[1] = b.c[2] = 0.0;
  if (sh.nodes.empty()) return b;
  const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
  return node_bound(sh, 0, I, z, tau_min);
}

static OBound mesh_sphere(const Mesh& m) {
  OBound b;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int k = 0; k < m.V; ++k)
    for (int i = 0; i < 3; ++i) { lo[i] = std::min(lo[i], m.v[3 * k + i]); hi[i] = std::max(hi[i], m.v[3 * k + i]); }
  for (int i = 0; i < 3; ++i) b.c[i] = 0.5 * (lo[i] + hi[i]);
  double r = 0.0;
  for (int k = 0; k < m.V; ++k) {
    const double d[3] = {m.v[3 * k] - b.c[0], m.v[3 * k + 1] - b.c[1], m.v[3 * k + 2] - b.c[2]};
    r = std::max(r, std::sqrt(dot3(d, d)));
  }
  b.rho = r;
  return b;
}


// ---- contact manifold -------------------------------------------
// Reduced manifold: shape A (pairs[5i+3]) is the sampled mesh, shape B
// (pairs[5i+4]) the SDF.  mode bit 4: full mode (one contact
// per vertex, then per edge in sorted-(lo,hi) order: point, raw normal, depth
// phi, W = gamma, q = gamma p, dom = 0 vertex / 1 edge); mode bit 8:
// two-sided (then B sampled against A's SDF; derivative columns stay in
// the pair's (A, B) order, J rows of that half are v_B - v_A).  pairs[i] = {env, slotA, slotB, shapeA,
// shapeB}; poses[(env*n_slot + slot)*8 + ...] = t(3), q(w,x,y,z), pad.
// Contacts of pair i occupy rows [off_i, off_i + F_A) in input pair order.
// Per contact c (row-major arrays):
//   point[3], normal[3] (raw fused, Reading #24), depth, W, qv[3] (compact J),
//   ddepth[12], dnormal[36] ([i*12+j] = d n_i / d q_j), dom (int),
//   J[36] (literal sum_i z_i gamma_i J_i, [r*12+c]), z[6], dcand[6], gam[6].
// q = (dt_A, dtheta_A, dt_B, dtheta_B), world-frame left twists (Reading #28).
// broad-phase bounds (f2): out4 = (c_x, c_y, c_z, rho); rho = inf without a bound
void ora_shape_bound(void* s, int shape, double* out4) {
  Scene* sc = (Scene*)s;
  const OBound b = shape_bound(sc->shapes[shape], sc->sp.tau_min);
  for (int i = 0; i < 3; ++i) out4[i] = b.c[i];
  out4[3] = b.rho;
}
void ora_mesh_sphere(void* s, int shape, double* out4) {
  Scene* sc = (Scene*)s;
  const OBound b = mesh_sphere(sc->shapes[shape].mesh);
  for (int i = 0; i < 3; ++i) out4[i] = b.c[i];
  out4[3] = b.rho;
}

int ora_contact_manifold(void* s, const int* pairs, long n_pairs, const double* poses, long n_env, int n_slot,
                         double* point, double* normal, double* depth, double* W, double* qv, double* ddepth,
                         double* dnormal, int* dom, double* J, double* zout, double* dcand, double* gout,
                         int mode, int n_threads) {
  Scene* sc = (Scene*)s;
  const Smooth sp = sc->sp;
  (void)n_env;
  const bool full = (mode & 4) != 0, two = (mode & 8) != 0, broad = (mode & 16) != 0;
  auto count = [&](int shape) { const Mesh& m = sc->shapes[shape].mesh; return full ? (long)m.V + m.E : (long)m.F; };
  std::vector<long> off(n_pairs + 1, 0);
  for (long i = 0; i < n_pairs; ++i)
    off[i + 1] = off[i] + count(pairs[5 * i + 3]) + (two ? count(pairs[5 * i + 4]) : 0);
  // broad-phase bounds per shape (f2)
  std::vector<OBound> sdfb(sc->shapes.size()), meshb(sc->shapes.size());
  if (broad)
    for (size_t k = 0; k < sc->shapes.size(); ++k) {
      sdfb[k] = shape_bound(sc->shapes[k], sp.tau_min);
      if (sc->shapes[k].mesh.V > 0) meshb[k] = mesh_sphere(sc->shapes[k].mesh);
    }
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (long pi = 0; pi < n_pairs; ++pi) {
   long row0 = off[pi];
   for (int side = 0; side < (two ? 2 : 1); ++side) {
    // (shape-parameter mode: a side whose SDF shape is not the seeded one
    // evaluates without the seed)
    struct SeedSuspend {
      int saved = -2;
      ~SeedSuspend() { if (saved != -2) g_seed_node = saved; }
    } seed_suspend;
    if (g_param_comp0 && pairs[5 * pi + 4 - side] != g_param_shape) {
      seed_suspend.saved = g_seed_node;
      g_seed_node = -1;
    }
    // "A" below is the sampled body of this side, "B" the SDF body
    const int* pr = pairs + 5 * pi;
    const Shape& SA = sc->shapes[pr[3 + side]];
    const Shape& SB = sc->shapes[pr[4 - side]];
    const Mesh& m = SA.mesh;
    const double* pa = poses + 8 * ((long)pr[0] * n_slot + pr[1 + side]);
    const double* pb = poses + 8 * ((long)pr[0] * n_slot + pr[2 - side]);
    double RA[9], RB[9], tA[3] = {pa[0], pa[1], pa[2]}, tB[3] = {pb[0], pb[1], pb[2]};
    double qa[4] = {pa[3], pa[4], pa[5], pa[6]}, qb[4] = {pb[3], pb[4], pb[5], pb[6]};
    quat_to_R(qa, RA); quat_to_R(qb, RB);
    if (broad) {
      const OBound& bA = meshb[pr[3 + side]];
      const OBound& bB = sdfb[pr[4 - side]];
      double cA[3], cB[3];
      for (int i = 0; i < 3; ++i) {
        cA[i] = RA[i * 3 + 0] * bA.c[0] + RA[i * 3 + 1] * bA.c[1] + RA[i * 3 + 2] * bA.c[2] + tA[i];
        cB[i] = RB[i * 3 + 0] * bB.c[0] + RB[i * 3 + 1] * bB.c[1] + RB[i * 3 + 2] * bB.c[2] + tB[i];
      }
      const double dc[3] = {cA[0] - cB[0], cA[1] - cB[1], cA[2] - cB[2]};
      const double lb = std::sqrt(dot3(dc, dc)) - bA.rho - bB.rho;
      if (lb > 40.0 * sp.tau_cmp) {   // culled: no candidate can carry a gate above e^-40
        const long nr = full ? (long)m.V + m.E : (long)m.F;
        for (long k = 0; k < nr; ++k) {
          const long c = row0 + k;
          double loc[3] = {0, 0, 0};
          if (!full) {
            for (int a = 0; a < 3; ++a)
              for (int i = 0; i < 3; ++i) loc[i] += m.v[3 * m.f[3 * k + a] + i] / 3.0;
          } else if (k < m.V) {
            for (int i = 0; i < 3; ++i) loc[i] = m.v[3 * k + i];
          } else {
            // edges in sorted (lo, hi) order after the vertices
            std::vector<std::pair<int, int>> es(m.E);
            for (int e = 0; e < m.E; ++e) es[e] = std::make_pair(m.e[2 * e], m.e[2 * e + 1]);
            std::sort(es.begin(), es.end());
            const auto& ee = es[k - m.V];
            for (int i = 0; i < 3; ++i) loc[i] = 0.5 * (m.v[3 * ee.first + i] + m.v[3 * ee.second + i]);
          }
          for (int a = 0; a < 3; ++a) {
            point[3 * c + a] = RA[a * 3 + 0] * loc[0] + RA[a * 3 + 1] * loc[1] + RA[a * 3 + 2] * loc[2] + tA[a];
            normal[3 * c + a] = 0.0;
            qv[3 * c + a] = 0.0;
            for (int j = 0; j < 12; ++j) dnormal[36 * c + a * 12 + j] = 0.0;
          }
          depth[c] = full ? lb : lb - sp.tau_min * std::log(6.0);
          W[c] = 0.0;
          dom[c] = -2;
          for (int j = 0; j < 12; ++j) ddepth[12 * c + j] = 0.0;
          for (int j = 0; j < 36; ++j) J[36 * c + j] = 0.0;
          for (int i = 0; i < 6; ++i) { zout[6 * c + i] = 0.0; dcand[6 * c + i] = lb; gout[6 * c + i] = 0.0; }
        }
        row0 += nr;
        continue;
      }
    }

    // q-jet poses (first order, 12 seeds): q = (dt, dtheta) of the pair's
    // first body, then of its second body, whichever plays the sampled role
    const int sA = side ? 6 : 0, sB = side ? 0 : 6;
    D12 dtA[3], wA[3], dtB[3], wB[3];
    for (int i = 0; i < 3; ++i) {
      dtA[i] = D12(0.0); wA[i] = D12(0.0); dtB[i] = D12(0.0); wB[i] = D12(0.0);
      if (g_param_comp0) continue;   // (shape-parameter mode: component 0 carries the parameter)
      dtA[i].d[sA + i] = 1.0;
      wA[i].d[sA + 3 + i] = 1.0;
      dtB[i].d[sB + i] = 1.0;
      wB[i].d[sB + 3 + i] = 1.0;
    }
    // J_i rows are v_sampled - v_sdf; written in the pair's (A, B) columns
    const double sg = side ? -1.0 : 1.0;
    const double* tP = side ? tB : tA;   // the pair's first body translation
    const double* tQ = side ? tA : tB;   // the pair's second body translation
    D12 RAq[9], tAq[3], RBq[9], tBq[3];
    perturbed_pose(RA, tA, dtA, wA, RAq, tAq);
    perturbed_pose(RB, tB, dtB, wB, RBq, tBq);
    // the same poses lifted to the nested type (inner jet = world point)
    N12 RBn[9], tBn[3];
    auto lift = [](const D12& a) { N12 r(0.0); r.v.v = a.v; for (int j = 0; j < 12; ++j) r.d[j].v = a.d[j]; return r; };
    for (int i = 0; i < 9; ++i) RBn[i] = lift(RBq[i]);
    for (int i = 0; i < 3; ++i) tBn[i] = lift(tBq[i]);

    // world position of a local point of A as a q-jet
    auto world_of = [&](const double* v, D12* p) {
      for (int i = 0; i < 3; ++i) p[i] = RAq[i * 3 + 0] * v[0] + RAq[i * 3 + 1] * v[1] + RAq[i * 3 + 2] * v[2] + tAq[i];
    };
    auto phi1 = [&](const D12* p) { return shape_phi_world(SB, RBq, tBq, p, sp); };
    // second-order candidate evaluation: d, n = grad phi (world), both q-jets
    auto cand = [&](const D12* p, D12& dd, D12* nn) {
      N12 X[3];
      for (int i = 0; i < 3; ++i) {
        X[i] = N12(0.0);
        X[i].v.v = p[i].v; X[i].v.d[i] = 1.0;
        for (int j = 0; j < 12; ++j) X[i].d[j].v = p[i].d[j];
      }
      N12 ph = shape_phi_world(SB, RBn, tBn, X, sp);
      dd = D12(0.0); dd.v = ph.v.v;
      for (int j = 0; j < 12; ++j) dd.d[j] = ph.d[j].v;
      for (int i = 0; i < 3; ++i) {
        nn[i] = D12(0.0); nn[i].v = ph.v.d[i];
        for (int j = 0; j < 12; ++j) nn[i].d[j] = ph.d[j].d[i];
      }
    };

    // vertices: position, depth, normal
    std::vector<D12> vp(3 * m.V), vd(m.V), vn(3 * m.V);
    for (int k = 0; k < m.V; ++k) {
      world_of(&m.v[3 * k], &vp[3 * k]);
      cand(&vp[3 * k], vd[k], &vn[3 * k]);
    }
    // edges: sphere trace both corners (Fig. 2), 3 gated steps
    // each (Reading #19, #20), soft clip to the edge (Reading #21), midpoint
    std::vector<D12> ep(3 * m.E), ed(m.E), en(3 * m.E);
    for (int e = 0; e < m.E; ++e) {
      const double* vI = &m.v[3 * m.e[2 * e]];
      const double* vII = &m.v[3 * m.e[2 * e + 1]];
      double dl[3] = {vII[0] - vI[0], vII[1] - vI[1], vII[2] - vI[2]};
      double L = std::sqrt(dot3(dl, dl));
      double etl[3] = {dl[0] / L, dl[1] / L, dl[2] / L};
      D12 pI[3], et[3];
      world_of(vI, pI);
      for (int i = 0; i < 3; ++i) et[i] = RAq[i * 3 + 0] * etl[0] + RAq[i * 3 + 1] * etl[1] + RAq[i * 3 + 2] * etl[2];
      D12 alpha(0.0), beta(L);
      for (int it = 0; it < sp.trace_iters; ++it) {
        D12 x[3];
        for (int i = 0; i < 3; ++i) x[i] = pI[i] + alpha * et[i];
        D12 ph = phi1(x);
        alpha = alpha + sigmoid(ph / sp.tau_cmp) * ph;
      }
      for (int it = 0; it < sp.trace_iters; ++it) {
        D12 x[3];
        for (int i = 0; i < 3; ++i) x[i] = pI[i] + beta * et[i];
        D12 ph = phi1(x);
        beta = beta - sigmoid(ph / sp.tau_cmp) * ph;
      }
      D12 at = softclip(alpha, 0.0, L, sp.tau_clip_alpha);
      D12 bt = softclip(beta, 0.0, L, sp.tau_clip_alpha);
      D12 ab = 0.5 * (at + bt);
      for (int i = 0; i < 3; ++i) ep[3 * e + i] = pI[i] + ab * et[i];
      cand(&ep[3 * e], ed[e], &en[3 * e]);
    }
    if (full) {
      // one contact per vertex, then per edge in sorted (lo, hi) order
      std::vector<int> eo(m.E);
      for (int e = 0; e < m.E; ++e) eo[e] = e;
      std::sort(eo.begin(), eo.end(), [&](int a, int b) {
        return std::make_pair(m.e[2 * a], m.e[2 * a + 1]) < std::make_pair(m.e[2 * b], m.e[2 * b + 1]); });
      for (int k = 0; k < m.V + m.E; ++k) {
        const bool isv = k < m.V;
        const int id = isv ? k : eo[k - m.V];
        const D12* P = isv ? &vp[3 * id] : &ep[3 * id];
        const D12* N = isv ? &vn[3 * id] : &en[3 * id];
        const D12& dk = isv ? vd[id] : ed[id];
        const long c = row0 + k;
        const double gam = val(sigmoid(-dk / sp.tau_cmp));
        for (int a = 0; a < 3; ++a) {
          point[3 * c + a] = P[a].v;
          normal[3 * c + a] = N[a].v;
          qv[3 * c + a] = gam * P[a].v;
          for (int j = 0; j < 12; ++j) dnormal[36 * c + a * 12 + j] = N[a].d[j];
        }
        depth[c] = dk.v; W[c] = gam; dom[c] = isv ? 0 : 1;
        for (int j = 0; j < 12; ++j) ddepth[12 * c + j] = dk.d[j];
        double ra[3], rb[3];
        for (int a = 0; a < 3; ++a) { ra[a] = P[a].v - tP[a]; rb[a] = P[a].v - tQ[a]; }
        double Ka[9] = {0, -ra[2], ra[1], ra[2], 0, -ra[0], -ra[1], ra[0], 0};
        double Kb[9] = {0, -rb[2], rb[1], rb[2], 0, -rb[0], -rb[1], rb[0], 0};
        for (int a = 0; a < 36; ++a) J[36 * c + a] = 0.0;
        for (int r = 0; r < 3; ++r) {
          J[36 * c + r * 12 + r] += sg * gam;
          J[36 * c + r * 12 + 6 + r] -= sg * gam;
          for (int k2 = 0; k2 < 3; ++k2) {
            J[36 * c + r * 12 + 3 + k2] -= sg * gam * Ka[r * 3 + k2];
            J[36 * c + r * 12 + 9 + k2] += sg * gam * Kb[r * 3 + k2];
          }
        }
        for (int i = 0; i < 6; ++i) { zout[6 * c + i] = 0.0; dcand[6 * c + i] = dk.v; gout[6 * c + i] = gam; }
      }
      row0 += m.V + m.E;
      continue;
    }
    // per-face fusion
    for (int f = 0; f < m.F; ++f) {
      long c = row0 + f;
      const D12* P6[6]; D12 dd[6]; const D12* N6[6];
      for (int k = 0; k < 3; ++k) {
        int vi = m.f[3 * f + k];
        P6[k] = &vp[3 * vi]; dd[k] = vd[vi]; N6[k] = &vn[3 * vi];
        int ei = m.fe[3 * f + k];
        P6[3 + k] = &ep[3 * ei]; dd[3 + k] = ed[ei]; N6[3 + k] = &en[3 * ei];
      }
      D12 negd[6], z[6], gam[6];
      for (int i = 0; i < 6; ++i) negd[i] = -dd[i];
      softargmax(negd, 6, sp.tau_min, z);                   // z = s_argmax(-d)
      for (int i = 0; i < 6; ++i) gam[i] = sigmoid(-dd[i] / sp.tau_cmp);  // [[d < 0]]
      D12 n3[3] = {D12(0.0), D12(0.0), D12(0.0)}, Wf(0.0), q3[3] = {D12(0.0), D12(0.0), D12(0.0)};
      D12 pt3[3] = {D12(0.0), D12(0.0), D12(0.0)};
      for (int i = 0; i < 6; ++i) {
        D12 zg = z[i] * gam[i];
        for (int k = 0; k < 3; ++k) {
          n3[k] = n3[k] + zg * N6[i][k];                     // n = sum z gamma n_i
          q3[k] = q3[k] + zg * P6[i][k];
          pt3[k] = pt3[k] + z[i] * P6[i][k];                 // reporting only
        }
        Wf = Wf + zg;
      }
      D12 dep = -lse(negd, 6, sp.tau_min);                 // smooth min (Reading #25)
      // dominant candidate: argmax z_i gamma_i, lowest index on exact ties.
      // z_i and gamma_i both decrease strictly with d_i, so this is argmin d_i;
      // taken on d so it stays defined when the weights underflow (reading #32)
      int im = 0;
      for (int i = 1; i < 6; ++i) if (val(dd[i]) < val(dd[im])) im = i;
      // literal fused contact Jacobian J = sum z_i gamma_i J_i, J_i = [I, -[p-tA]x, -I, [p-tB]x]
      // (in the pair's (A, B) columns; the transposed side has the opposite sign)
      double Jc[36] = {0};
      for (int i = 0; i < 6; ++i) {
        double zg = sg * val(z[i]) * val(gam[i]);
        double ra[3], rb[3];
        for (int k = 0; k < 3; ++k) { ra[k] = P6[i][k].v - tP[k]; rb[k] = P6[i][k].v - tQ[k]; }
        double Ka[9] = {0, -ra[2], ra[1], ra[2], 0, -ra[0], -ra[1], ra[0], 0};
        double Kb[9] = {0, -rb[2], rb[1], rb[2], 0, -rb[0], -rb[1], rb[0], 0};
        for (int r = 0; r < 3; ++r) {
          Jc[r * 12 + r] += zg;
          Jc[r * 12 + 6 + r] -= zg;
          for (int k = 0; k < 3; ++k) {
            Jc[r * 12 + 3 + k] -= zg * Ka[r * 3 + k];
            Jc[r * 12 + 9 + k] += zg * Kb[r * 3 + k];
          }
        }
      }
      for (int k = 0; k < 3; ++k) {
        point[3 * c + k] = pt3[k].v;
        normal[3 * c + k] = n3[k].v;
        qv[3 * c + k] = q3[k].v;
        for (int j = 0; j < 12; ++j) dnormal[36 * c + k * 12 + j] = n3[k].d[j];
      }
      depth[c] = dep.v; W[c] = Wf.v; dom[c] = im;
      for (int j = 0; j < 12; ++j) ddepth[12 * c + j] = dep.d[j];
      for (int k = 0; k < 36; ++k) J[36 * c + k] = Jc[k];
      for (int i = 0; i < 6; ++i) { zout[6 * c + i] = z[i].v; dcand[6 * c + i] = dd[i].v; gout[6 * c + i] = gam[i].v; }
    }
    row0 += m.F;
   }
  }
  return 0;
}

// ---- shape-parameter derivatives of sdf_eval ----------
// Parameters of a shape: its nodes in index (pre-order) order, slots per node
// as for pval above; an XPSQ node with constant schedules has the PSQ slots
// (each moves both endpoint values; the plane normal is renormalised as in
// xpsq_phi); with varying schedules the PSQ slots of the t = 0 endpoint, then
// those of the t = 1 endpoint (the schedules are linear in t, reading #8).
// J[n * pmax + k] = d phi(point n) / d param k of the point's shape, zero
// beyond the shape's count; one Dual<double,1> evaluation per parameter.
static int node_param_count(const Node& n) {
  if (n.type == K_HALFSPACE) return 4;
  if (n.type == K_SQ) return 5;
  if (n.type == K_PSQ) return 5 + 4 * n.n_planes;
  if (n.type == K_XPSQ) return (xpsq_varying(n) ? 2 : 1) * (5 + 4 * n.n_planes) + 9;   // + control points p1, p2, p3
  return 0;
}
int ora_shape_param_count(void* s, int shape) {
  Scene* sc = (Scene*)s;
  const Shape& sh = sc->shapes[shape];
  int c = 0;
  for (const Node& n : sh.nodes) c += node_param_count(n);
  return c;
}
int ora_sdf_param_grad(void* s, const int* shape_ids, const double* poses, const double* points, long B, long P,
                       int pmax, double* J) {
  Scene* sc = (Scene*)s;
  const Smooth& sp = sc->sp;
  long total = B * P;
#pragma omp parallel for schedule(dynamic, 16)
  for (long n = 0; n < total; ++n) {
    const long b = n / P;
    const Shape& sh = sc->shapes[shape_ids[b]];
    const double* pz = poses + 8 * b;
    double R[9], t[3] = {pz[0], pz[1], pz[2]};
    double q[4] = {pz[3], pz[4], pz[5], pz[6]};
    quat_to_R(q, R);
    using D1 = Dual<double, 1>;
    D1 X[3], Rj[9], tj[3];
    for (int i = 0; i < 3; ++i) { X[i] = D1(points[3 * n + i]); tj[i] = D1(t[i]); }
    for (int i = 0; i < 9; ++i) Rj[i] = D1(R[i]);
    int k = 0;
    for (int ni = 0; ni < (int)sh.nodes.size(); ++ni) {
      const Node& nd = sh.nodes[ni];
      const int cnt = node_param_count(nd);
      for (int slot = 0; slot < cnt && k < pmax; ++slot, ++k) {
        g_seed_node = ni;
        g_seed_slot = slot;
        J[n * pmax + k] = shape_phi_world(sh, Rj, tj, X, sp).d[0];
      }
    }
    g_seed_node = g_seed_slot = -1;
    for (; k < pmax; ++k) J[n * pmax + k] = 0.0;
  }
  return 0;
}

// ---- node-pose derivatives of sdf_eval ---------------
// J[n * nmax + 6 k + j] = d phi(point n) / d twist j of node k of the point's
// shape (nodes in index order, every node incl. boolean ones and the root;
// twist in the node's parent frame, slots dt_x, dt_y, dt_z, dtheta_x,
// dtheta_y, dtheta_z, the convention of pose_seed above), zero beyond
// 6 x the shape's node count; one Dual<double,1> evaluation per slot.
int ora_sdf_node_pose_grad(void* s, const int* shape_ids, const double* poses, const double* points, long B, long P,
                           int nmax, double* J) {
  Scene* sc = (Scene*)s;
  const Smooth& sp = sc->sp;
  long total = B * P;
#pragma omp parallel for schedule(dynamic, 16)
  for (long n = 0; n < total; ++n) {
    const long b = n / P;
    const Shape& sh = sc->shapes[shape_ids[b]];
    const double* pz = poses + 8 * b;
    double R[9], t[3] = {pz[0], pz[1], pz[2]};
    double q[4] = {pz[3], pz[4], pz[5], pz[6]};
    quat_to_R(q, R);
    using D1 = Dual<double, 1>;
    D1 X[3], Rj[9], tj[3];
    for (int i = 0; i < 3; ++i) { X[i] = D1(points[3 * n + i]); tj[i] = D1(t[i]); }
    for (int i = 0; i < 9; ++i) Rj[i] = D1(R[i]);
    int k = 0;
    for (int ni = 0; ni < (int)sh.nodes.size(); ++ni)
      for (int slot = 0; slot < 6 && k < nmax; ++slot, ++k) {
        g_pose_node = ni;
        g_pose_slot = slot;
        J[n * nmax + k] = shape_phi_world(sh, Rj, tj, X, sp).d[0];
      }
    g_pose_node = g_pose_slot = -1;
    for (; k < nmax; ++k) J[n * nmax + k] = 0.0;
  }
  return 0;
}
int ora_shape_node_count(void* s, int shape) { return (int)((Scene*)s)->shapes[shape].nodes.size(); }

// ---- shape-parameter derivatives of the manifold depth (
// reading #48) -----------------------------------------------------------
// Jd[row * pmax + k] = d depth(row) / d parameter k of the pair's SDF shape B
// (the layout of ora_sdf_param_grad), one-sided modes (reduced or full): the
// literal manifold of ora_contact_manifold with the parameter seeded in
// component 0 of its jets (g_param_comp0), one evaluation per pair and slot.
int ora_manifold_param_jac(void* s, const int* pairs, long n_pairs, const double* poses, long n_env, int n_slot,
                           int mode, int pmax, double* Jd) {
  Scene* sc = (Scene*)s;
  const bool full = (mode & 4) != 0, two = (mode & 8) != 0;
  auto count = [&](int shape) { const Mesh& m = sc->shapes[shape].mesh; return full ? (long)m.V + m.E : (long)m.F; };
  std::vector<long> off(n_pairs + 1, 0);
  for (long i = 0; i < n_pairs; ++i)
    off[i + 1] = off[i] + count(pairs[5 * i + 3]) + (two ? count(pairs[5 * i + 4]) : 0);
#pragma omp parallel for schedule(dynamic, 1)
  for (long pi = 0; pi < n_pairs; ++pi) {
    const long nr = off[pi + 1] - off[pi];
    std::vector<double> pt(3 * nr), nm(3 * nr), dp(nr), W(nr), q(3 * nr), dd(12 * nr), dn(36 * nr), J(36 * nr),
        z(6 * nr), dc(6 * nr), g(6 * nr);
    std::vector<int> dom(nr);
    for (long r = 0; r < nr; ++r)
      for (int k = 0; k < pmax; ++k) Jd[(off[pi] + r) * pmax + k] = 0.0;
    // rows of side 0 (SDF shape B) then side 1 (SDF shape A, two-sided)
    const long n0 = count(pairs[5 * pi + 3]);
    for (int side = 0; side < (two ? 2 : 1); ++side) {
      const int shp = pairs[5 * pi + 4 - side];
      if (side == 1 && shp == pairs[5 * pi + 4]) continue;   // (A == B: done with side 0)
      const Shape& SB = sc->shapes[shp];
      int k = 0;
      for (int ni = 0; ni < (int)SB.nodes.size(); ++ni) {
        const int cnt = node_param_count(SB.nodes[ni]);
        for (int slot = 0; slot < cnt && k < pmax; ++slot, ++k) {
          g_seed_node = ni;
          g_seed_slot = slot;
          g_param_comp0 = true;
          g_param_shape = shp;
          // (nested inside this parallel loop the manifold's own loop runs on
          // this thread, which holds the thread-local seeds)
          ora_contact_manifold(s, pairs + 5 * pi, 1, poses, n_env, n_slot, pt.data(), nm.data(), dp.data(), W.data(),
                               q.data(), dd.data(), dn.data(), dom.data(), J.data(), z.data(), dc.data(), g.data(),
                               mode, 0);
          g_param_comp0 = false;
          g_param_shape = -1;
          for (long r = 0; r < nr; ++r) {
            const int row_shape = r < n0 ? pairs[5 * pi + 4] : pairs[5 * pi + 3];
            if (row_shape == shp) Jd[(off[pi] + r) * pmax + k] = dd[12 * r + 0];
          }
        }
      }
    }
    g_seed_node = g_seed_slot = -1;
  }
  return 0;
}

// ---- second-order manifold derivatives (P:8 motivates
// Hessians for second-order control) ----------------------------------------
// The same manifold as ora_contact_manifold (reduced or full mode, one- or
// two-sided), recomputed with second-order q-jets Dual<Dual<double,12>,12>:
// d2depth[78 c + k] = d^2 depth / dq_i dq_j for the packed upper triangle
// i <= j of the pair-ordered q = (dt_A, dtheta_A, dt_B, dtheta_B) (k runs over
// (0,0), (0,1), .., (0,11), (1,1), ..).  In full mode the depth of a row is
// the candidate's phi.  Every step is the literal one of ora_contact_manifold
// on the second-order jet type (no derivative is hand-derived here).
using Q2 = Dual<D12, 12>;
int ora_manifold_d2depth(void* s, const int* pairs, long n_pairs, const double* poses, long n_env, int n_slot,
                         double* d2depth, int mode, int n_threads) {
  Scene* sc = (Scene*)s;
  const Smooth sp = sc->sp;
  (void)n_env;
  const bool full = (mode & 4) != 0, two = (mode & 8) != 0;
  auto count = [&](int shape) { const Mesh& m = sc->shapes[shape].mesh; return full ? (long)m.V + m.E : (long)m.F; };
  std::vector<long> off(n_pairs + 1, 0);
  for (long i = 0; i < n_pairs; ++i)
    off[i + 1] = off[i] + count(pairs[5 * i + 3]) + (two ? count(pairs[5 * i + 4]) : 0);
  auto store = [&](long c, const Q2& x) {
    int k = 0;
    for (int i = 0; i < 12; ++i)
      for (int j = i; j < 12; ++j) d2depth[78 * c + (k++)] = x.d[i].d[j];
  };
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (long pi = 0; pi < n_pairs; ++pi) {
   long row0 = off[pi];
   for (int side = 0; side < (two ? 2 : 1); ++side) {
    const int* pr = pairs + 5 * pi;
    const Shape& SA = sc->shapes[pr[3 + side]];
    const Shape& SB = sc->shapes[pr[4 - side]];
    const Mesh& m = SA.mesh;
    const double* pa = poses + 8 * ((long)pr[0] * n_slot + pr[1 + side]);
    const double* pb = poses + 8 * ((long)pr[0] * n_slot + pr[2 - side]);
    double RA[9], RB[9], tA[3] = {pa[0], pa[1], pa[2]}, tB[3] = {pb[0], pb[1], pb[2]};
    double qa[4] = {pa[3], pa[4], pa[5], pa[6]}, qb[4] = {pb[3], pb[4], pb[5], pb[6]};
    quat_to_R(qa, RA); quat_to_R(qb, RB);
    // second-order seeds: q_k carries d/dq_k at both jet levels
    const int sA = side ? 6 : 0, sB = side ? 0 : 6;
    auto seed = [](int k) { Q2 x(0.0); x.v.d[k] = 1.0; x.d[k].v = 1.0; return x; };
    Q2 dtA[3], wA[3], dtB[3], wB[3];
    for (int i = 0; i < 3; ++i) {
      dtA[i] = seed(sA + i); wA[i] = seed(sA + 3 + i);
      dtB[i] = seed(sB + i); wB[i] = seed(sB + 3 + i);
    }
    Q2 RAq[9], tAq[3], RBq[9], tBq[3];
    perturbed_pose(RA, tA, dtA, wA, RAq, tAq);
    perturbed_pose(RB, tB, dtB, wB, RBq, tBq);
    auto world_of = [&](const double* v, Q2* p) {
      for (int i = 0; i < 3; ++i) p[i] = RAq[i * 3 + 0] * v[0] + RAq[i * 3 + 1] * v[1] + RAq[i * 3 + 2] * v[2] + tAq[i];
    };
    auto phi = [&](const Q2* p) { return shape_phi_world(SB, RBq, tBq, p, sp); };
    std::vector<Q2> vd(m.V), ed(m.E);
    for (int k = 0; k < m.V; ++k) {
      Q2 p[3];
      world_of(&m.v[3 * k], p);
      vd[k] = phi(p);
    }
    for (int e = 0; e < m.E; ++e) {   // trace both corners, clip, midpoint
      const double* vI = &m.v[3 * m.e[2 * e]];
      const double* vII = &m.v[3 * m.e[2 * e + 1]];
      double dl[3] = {vII[0] - vI[0], vII[1] - vI[1], vII[2] - vI[2]};
      double L = std::sqrt(dot3(dl, dl));
      double etl[3] = {dl[0] / L, dl[1] / L, dl[2] / L};
      Q2 pI[3], et[3];
      world_of(vI, pI);
      for (int i = 0; i < 3; ++i) et[i] = RAq[i * 3 + 0] * etl[0] + RAq[i * 3 + 1] * etl[1] + RAq[i * 3 + 2] * etl[2];
      Q2 alpha(0.0), beta(L);
      for (int it = 0; it < sp.trace_iters; ++it) {
        Q2 x[3];
        for (int i = 0; i < 3; ++i) x[i] = pI[i] + alpha * et[i];
        Q2 ph = phi(x);
        alpha = alpha + sigmoid(ph / sp.tau_cmp) * ph;
      }
      for (int it = 0; it < sp.trace_iters; ++it) {
        Q2 x[3];
        for (int i = 0; i < 3; ++i) x[i] = pI[i] + beta * et[i];
        Q2 ph = phi(x);
        beta = beta - sigmoid(ph / sp.tau_cmp) * ph;
      }
      Q2 ab = 0.5 * (softclip(alpha, 0.0, L, sp.tau_clip_alpha) + softclip(beta, 0.0, L, sp.tau_clip_alpha));
      Q2 x[3];
      for (int i = 0; i < 3; ++i) x[i] = pI[i] + ab * et[i];
      ed[e] = phi(x);
    }
    if (full) {
      std::vector<int> eo(m.E);
      for (int e = 0; e < m.E; ++e) eo[e] = e;
      std::sort(eo.begin(), eo.end(), [&](int a, int b) {
        return std::make_pair(m.e[2 * a], m.e[2 * a + 1]) < std::make_pair(m.e[2 * b], m.e[2 * b + 1]); });
      for (int k = 0; k < m.V + m.E; ++k) store(row0 + k, k < m.V ? vd[k] : ed[eo[k - m.V]]);
      row0 += m.V + m.E;
      continue;
    }
    for (int f = 0; f < m.F; ++f) {   // smooth-min depth of the face's 6 candidates
      Q2 negd[6];
      for (int k = 0; k < 3; ++k) {
        negd[k] = -vd[m.f[3 * f + k]];
        negd[3 + k] = -ed[m.fe[3 * f + k]];
      }
      store(row0 + f, -lse(negd, 6, sp.tau_min));
    }
    row0 += m.F;
   }
  }
  return 0;
}

int ora_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

}  // extern "C"
