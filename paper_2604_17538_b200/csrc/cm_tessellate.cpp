// Library-side sampled surfaces (`sample_res` gives the
// tessellation of the analytic kinds used as the sampled side, "sample
// points on one shape's surface").  Host code, FP64, rounded once to FP32.
//   SQ    cube-sphere topology, res x res cells per cube face, placed on the
//         superellipsoid by its parametric form (Eq. (1))
//           x = a1 C(eta)^e1 C(w)^e2, y = a2 C(eta)^e1 S(w)^e2, z = a3 S(eta)^e1
//         with (eta, w) the latitude / longitude of the tangent-warped cube
//         direction: V = 6 res^2 + 2, F = 12 res^2
//   PSQ   the SQ surface with every vertex outside a plane pulled radially
//         (towards the centre, inside every plane) onto it (star-shaped)
//   XPSQ  a tube around the quadratic spline (Eq. (5)): 2 res + 1
//         rings of 4 res points on the t = 0 cross-section superellipse
//         (a_y, a_z, exponent eps2) in the spline's frame (Frenet binormal
//         B x A, or the up hint for a straight spline), two end-cap centres:
//         V = (2 res + 1) 4 res + 2
// The vertex and face orders are those of the Python synthetic generators
// (synth.sq_mesh / psq_mesh / xpsq_mesh), which the tests compare against.
#include <array>
#include <cmath>
#include <map>
#include <tuple>
#include <vector>

#include "xpsq_cm.h"

namespace {

using V3 = std::array<double, 3>;

double spow(double x, double e) { return x == 0.0 ? 0.0 : std::copysign(std::pow(std::fabs(x), e), x); }

// closed triangulated cube [-1,1]^3, k x k cells per face, outward winding
void cube_grid(int k, std::vector<V3>& V, std::vector<int32_t>& F) {
  std::map<std::tuple<int, int, int>, int> key;
  auto vid = [&](int ix, int iy, int iz) {
    auto t = std::make_tuple(ix, iy, iz);
    auto it = key.find(t);
    if (it != key.end()) return it->second;
    const int id = (int)V.size();
    key.emplace(t, id);
    V.push_back({2.0 * ix / k - 1.0, 2.0 * iy / k - 1.0, 2.0 * iz / k - 1.0});
    return id;
  };
  for (int axis = 0; axis < 3; ++axis)
    for (int side : {0, k}) {
      const int u_ax = axis == 0 ? 1 : 0, v_ax = axis == 2 ? 1 : 2;
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
          int q[4];
          const int dd[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
          for (int c = 0; c < 4; ++c) {
            int cc[3] = {0, 0, 0};
            cc[axis] = side;
            cc[u_ax] = i + dd[c][0];
            cc[v_ax] = j + dd[c][1];
            q[c] = vid(cc[0], cc[1], cc[2]);
          }
          const V3 &p0 = V[q[0]], &p1 = V[q[1]], &p2 = V[q[2]];
          const double e1[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
          const double e2[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
          const double nrm[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                                 e1[0] * e2[1] - e1[1] * e2[0]};
          const double outward = side == k ? 1.0 : -1.0;
          if (nrm[axis] * outward < 0) std::swap(q[0], q[3]), std::swap(q[1], q[2]);
          const int tri[6] = {q[0], q[1], q[2], q[0], q[2], q[3]};
          F.insert(F.end(), tri, tri + 6);
        }
    }
}

void sq_surface(const cm_node& n, int k, std::vector<V3>& V, std::vector<int32_t>& F) {
  cube_grid(k, V, F);
  const double e1 = n.eps[0][0], e2 = n.eps[0][1];
  const double pi4 = std::atan(1.0);
  for (V3& v : V) {
    double w[3], d[3];
    for (int i = 0; i < 3; ++i) w[i] = std::tan(v[i] * pi4);
    const double nw = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    for (int i = 0; i < 3; ++i) d[i] = w[i] / nw;
    const double eta = std::asin(std::fmin(std::fmax(d[2], -1.0), 1.0));
    const double om = std::atan2(d[1], d[0]);
    const double ce = spow(std::cos(eta), e1);
    v = {n.a[0][0] * ce * spow(std::cos(om), e2), n.a[0][1] * ce * spow(std::sin(om), e2),
         n.a[0][2] * spow(std::sin(eta), e1)};
  }
}

bool xpsq_surface(const cm_node& n, int res, std::vector<V3>& V, std::vector<int32_t>& F) {
  double p[3][3];
  for (int r = 0; r < 3; ++r)
    for (int i = 0; i < 3; ++i) p[r][i] = n.ctrl[3 * r + i];
  double A[3], B[3];
  for (int i = 0; i < 3; ++i) { A[i] = p[0][i] - 2 * p[1][i] + p[2][i]; B[i] = 2 * (p[1][i] - p[0][i]); }
  const double nB = std::sqrt(B[0] * B[0] + B[1] * B[1] + B[2] * B[2]);
  if (!(nB > 1e-9)) return false;   // a point spline has no tube
  double b[3] = {B[1] * A[2] - B[2] * A[1], B[2] * A[0] - B[0] * A[2], B[0] * A[1] - B[1] * A[0]};
  double nb = std::sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
  if (nb < 1e-9 * nB * nB) {   // straight: binormal from the up hint (Gram-Schmidt against the chord)
    double T[3] = {B[0] / nB, B[1] / nB, B[2] / nB};
    const double ut = n.up[0] * T[0] + n.up[1] * T[1] + n.up[2] * T[2];
    for (int i = 0; i < 3; ++i) b[i] = n.up[i] - ut * T[i];
    nb = std::sqrt(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
    if (!(nb > 1e-9)) return false;
  }
  for (int i = 0; i < 3; ++i) b[i] /= nb;
  const int nt = 2 * res + 1, nth = 4 * res;
  const double pi = 4.0 * std::atan(1.0);
  const double ay = n.a[0][1], az = n.a[0][2], e2 = n.eps[0][1];
  for (int it = 0; it < nt; ++it) {
    const double t = (double)it / (nt - 1);
    double pt[3], T[3];
    for (int i = 0; i < 3; ++i) { pt[i] = p[0][i] + B[i] * t + A[i] * t * t; T[i] = B[i] + 2 * A[i] * t; }
    const double nT = std::sqrt(T[0] * T[0] + T[1] * T[1] + T[2] * T[2]);
    for (int i = 0; i < 3; ++i) T[i] /= nT;
    const double N[3] = {b[1] * T[2] - b[2] * T[1], b[2] * T[0] - b[0] * T[2], b[0] * T[1] - b[1] * T[0]};
    for (int j = 0; j < nth; ++j) {
      const double w = 2 * pi * j / nth;
      const double cy = ay * spow(std::cos(w), e2), cz = az * spow(std::sin(w), e2);
      V.push_back({pt[0] + cy * N[0] + cz * b[0], pt[1] + cy * N[1] + cz * b[1], pt[2] + cy * N[2] + cz * b[2]});
    }
  }
  V.push_back({p[0][0] - n.a[0][0] * B[0] / nB, p[0][1] - n.a[0][0] * B[1] / nB, p[0][2] - n.a[0][0] * B[2] / nB});
  double Te[3], pe[3];
  for (int i = 0; i < 3; ++i) { Te[i] = B[i] + 2 * A[i]; pe[i] = p[0][i] + B[i] + A[i]; }
  const double nTe = std::sqrt(Te[0] * Te[0] + Te[1] * Te[1] + Te[2] * Te[2]);
  V.push_back({pe[0] + n.a[0][0] * Te[0] / nTe, pe[1] + n.a[0][0] * Te[1] / nTe, pe[2] + n.a[0][0] * Te[2] / nTe});
  const int nv = (int)V.size();
  for (int i = 0; i < nt - 1; ++i)
    for (int j = 0; j < nth; ++j) {
      const int a0 = i * nth + j, a1 = i * nth + (j + 1) % nth, b0 = a0 + nth, b1 = a1 + nth;
      const int tri[6] = {a0, b0, b1, a0, b1, a1};
      F.insert(F.end(), tri, tri + 6);
    }
  for (int j = 0; j < nth; ++j) {
    const int o = (nt - 1) * nth;
    const int tri[6] = {nv - 2, (j + 1) % nth, j, nv - 1, o + j, o + (j + 1) % nth};
    F.insert(F.end(), tri, tri + 6);
  }
  return true;
}

}  // namespace

extern "C" int cm_tessellate(const cm_node* node, int32_t res, float* vertices, int32_t* faces, int32_t* n_vertices,
                             int32_t* n_faces) {
  if (!node || !n_vertices || !n_faces || res < 1 || res > 256) return CM_ERR_INVALID;
  const cm_node& n = *node;
  std::vector<V3> V;
  std::vector<int32_t> F;
  if (n.type == CM_SQ || n.type == CM_PSQ) {
    for (int i = 0; i < 3; ++i)
      if (!(n.a[0][i] > 0.f)) return CM_ERR_INVALID;
    if (!(n.eps[0][0] > 0.f) || !(n.eps[0][1] > 0.f)) return CM_ERR_INVALID;
    sq_surface(n, res, V, F);
    if (n.type == CM_PSQ) {
      if (n.n_planes < 0 || n.n_planes > CM_MAX_PLANES) return CM_ERR_INVALID;
      for (int j = 0; j < n.n_planes; ++j) {
        double nv[3] = {n.planes[0][j][0], n.planes[0][j][1], n.planes[0][j][2]};
        const double nn = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
        const double h = n.planes[0][j][3];
        if (!(nn > 0.0) || !(h < 0.0)) return CM_ERR_INVALID;   // the centre must be inside the plane
        for (int i = 0; i < 3; ++i) nv[i] /= nn;
        for (V3& v : V) {
          const double s = v[0] * nv[0] + v[1] * nv[1] + v[2] * nv[2];
          if (s + h > 0) {
            const double f = -h / s;
            for (int i = 0; i < 3; ++i) v[i] *= f;
          }
        }
      }
    }
  } else if (n.type == CM_XPSQ) {
    if (!(n.a[0][0] > 0.f) || !(n.a[0][1] > 0.f) || !(n.a[0][2] > 0.f) || !(n.eps[0][1] > 0.f)) return CM_ERR_INVALID;
    if (!xpsq_surface(n, res, V, F)) return CM_ERR_UNSUPPORTED;
  } else {
    return CM_ERR_UNSUPPORTED;   // half-spaces and boolean nodes have no closed sampled surface here
  }
  *n_vertices = (int32_t)V.size();
  *n_faces = (int32_t)(F.size() / 3);
  if (vertices && faces) {
    for (size_t v = 0; v < V.size(); ++v)
      for (int i = 0; i < 3; ++i) vertices[3 * v + i] = (float)V[v][i];
    for (size_t k = 0; k < F.size(); ++k) faces[k] = F[k];
  }
  return CM_OK;
}
