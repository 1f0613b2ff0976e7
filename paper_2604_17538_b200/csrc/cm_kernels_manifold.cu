// sm_100a kernels of the hot path (arXiv 2604.17538):
//   k_sdf_eval          batched SDF value / gradient / Hessian (+ pose
//                       derivatives) — §II-B, Eq. (1)-(6)
//   k_contact_manifold  one CTA per (env, pair): sampled-surface vertices ->
//                       sphere-traced edge points -> 6 candidates per face ->
//                       softmax fusion -> SoA stores — §II-C
//   k_face_counts / cub scan, k_expand_jacobian   (offsets, J expansion)
//
// Hot-path design: FP32 CUDA-core math (no tensor cores: the
// path is not a dense contraction), MUFU ex2/lg2/rcp in the log domain,
// pair-local candidate state in shared memory, field-major coalesced stores.
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
// contact manifold
// ============================================================================
// Per-pair candidate storage (field-major, stride = V or E):
//   vertex fields: xb[3] (B-local), pw[3] (world), d, n[3] (world grad phi),
//                  H[6] (world, tier 2)
//   edge fields during the trace: aI, aII, daI[12], daII[12] (tier 2);
//   after the midpoint phase:     pw[3], d, n[3], H[6], dab[12] (tier 2)
__host__ __device__ constexpr int vfields(int tier) { return tier >= 2 ? 16 : 10; }
__host__ __device__ constexpr int efields(int tier) { return tier >= 2 ? 26 : 7; }
enum { VX = 0, VP = 3, VD = 6, VN = 7, VH = 10 };
enum { EA = 0, EB = 1, EDA = 2, EDB = 14 };             // trace layout
enum { EP = 0, ED = 3, EN = 4, EH = 7, EDAB = 13 };     // midpoint layout

struct PairFrame {
  float RA[9], tA[3], RB[9], tB[3];
  float Rrel[9], trel[3];   // x_B = Rrel v_A + trel
};

__device__ __forceinline__ void pair_frame(const float* pa, const float* pb, PairFrame& F) {
  float qa[4] = {pa[3], pa[4], pa[5], pa[6]}, qb[4] = {pb[3], pb[4], pb[5], pb[6]};
  quat_to_R(qa, F.RA);
  quat_to_R(qb, F.RB);
#pragma unroll
  for (int i = 0; i < 3; ++i) { F.tA[i] = pa[i]; F.tB[i] = pb[i]; }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      F.Rrel[i * 3 + j] = F.RB[0 * 3 + i] * F.RA[0 * 3 + j] + F.RB[1 * 3 + i] * F.RA[1 * 3 + j] +
                          F.RB[2 * 3 + i] * F.RA[2 * 3 + j];
  float dt[3] = {F.tA[0] - F.tB[0], F.tA[1] - F.tB[1], F.tA[2] - F.tB[2]};
#pragma unroll
  for (int i = 0; i < 3; ++i) F.trel[i] = F.RB[0 * 3 + i] * dt[0] + F.RB[1 * 3 + i] * dt[1] + F.RB[2 * 3 + i] * dt[2];
}

// g^T J(p) for J(p) = [I, -[p - tA]x, -I, [p - tB]x]: the A blocks
// (t_A: g, theta_A: (p - tA) x g) and theta_B: g x (p - tB).  The t_B block is
// exactly -(t_A block) and is reconstructed at store time.
__device__ __forceinline__ void gJ(const float* g, const float* p, const PairFrame& F, float* o /*9*/) {
  const float ra[3] = {p[0] - F.tA[0], p[1] - F.tA[1], p[2] - F.tA[2]};
  const float rb[3] = {p[0] - F.tB[0], p[1] - F.tB[1], p[2] - F.tB[2]};
  o[0] = g[0]; o[1] = g[1]; o[2] = g[2];
  o[3] = ra[1] * g[2] - ra[2] * g[1];
  o[4] = ra[2] * g[0] - ra[0] * g[2];
  o[5] = ra[0] * g[1] - ra[1] * g[0];
  o[6] = g[1] * rb[2] - g[2] * rb[1];
  o[7] = g[2] * rb[0] - g[0] * rb[2];
  o[8] = g[0] * rb[1] - g[1] * rb[0];
}

// derivative slots: 9 independent components (tA, thetaA, thetaB); tB = -tA
constexpr int NDQ = 9;

// Full mode (V + E contacts): candidate i is its own contact.
//   point p, normal n = grad phi (raw), depth d, W = gamma, q = gamma p (so the
//   compact J = gamma J_i, the single-candidate case of P:161), dom = kind
//   (0 vertex, 1 edge point); tier 2: d d / dq = g^T J(p) (+ (g.e_t) d alpha_bar),
//   d n / dq = [H, -H[p - tA]x, (-H), H[p - tB]x - [n]x] (+ H e_t d alpha_bar^T).
template <int TIER>
__device__ __forceinline__ void store_candidate(const cm_manifold_out& out, int64_t C, int64_t c, const float* p,
                                                const float* n, float d, const float* h, const float* ew,
                                                const float* dab, const PairFrame& F, int kind, float itcmp, int cTA,
                                                int cRA, int cTB, int cRB) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    out.point[a * C + c] = p[a];
    out.normal[a * C + c] = n[a];
  }
  out.depth[c] = d;
  out.dom[c] = (int8_t)kind;
  if constexpr (TIER >= 1) {
    const float gam = sigm(-d * itcmp);
    out.W[c] = gam;
#pragma unroll
    for (int a = 0; a < 3; ++a) out.q[a * C + c] = gam * p[a];
  }
  if constexpr (TIER >= 2) {
    float dd[NDQ];
    gJ(n, p, F, dd);
    const float H[3][3] = {{h[0], h[1], h[2]}, {h[1], h[3], h[4]}, {h[2], h[4], h[5]}};
    float he[3] = {0.f, 0.f, 0.f};
    if (ew) {
      const float ge = n[0] * ew[0] + n[1] * ew[1] + n[2] * ew[2];
#pragma unroll
      for (int k = 0; k < NDQ; ++k) dd[k] = fmaf(ge, dab[k], dd[k]);
#pragma unroll
      for (int a = 0; a < 3; ++a) he[a] = H[a][0] * ew[0] + H[a][1] * ew[1] + H[a][2] * ew[2];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      out.ddepth[(cTA + k) * C + c] = dd[k];
      out.ddepth[(cRA + k) * C + c] = dd[3 + k];
      out.ddepth[(cTB + k) * C + c] = -dd[k];
      out.ddepth[(cRB + k) * C + c] = dd[6 + k];
    }
    const float ra[3] = {p[0] - F.tA[0], p[1] - F.tA[1], p[2] - F.tA[2]};
    const float rb[3] = {p[0] - F.tB[0], p[1] - F.tB[1], p[2] - F.tB[2]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float nk[3] = {a == 0 ? 0.f : (a == 1 ? n[2] : -n[1]), a == 0 ? -n[2] : (a == 1 ? 0.f : n[0]),
                           a == 0 ? n[1] : (a == 1 ? -n[0] : 0.f)};
      float row[NDQ] = {H[a][0], H[a][1], H[a][2],
                        -(H[a][1] * ra[2] - H[a][2] * ra[1]), -(H[a][2] * ra[0] - H[a][0] * ra[2]),
                        -(H[a][0] * ra[1] - H[a][1] * ra[0]),
                        (H[a][1] * rb[2] - H[a][2] * rb[1]) - nk[0], (H[a][2] * rb[0] - H[a][0] * rb[2]) - nk[1],
                        (H[a][0] * rb[1] - H[a][1] * rb[0]) - nk[2]};
      if (ew) {
#pragma unroll
        for (int k = 0; k < NDQ; ++k) row[k] = fmaf(he[a], dab[k], row[k]);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        out.dnormal[(a * 12 + cTA + k) * C + c] = row[k];
        out.dnormal[(a * 12 + cRA + k) * C + c] = row[3 + k];
        out.dnormal[(a * 12 + cTB + k) * C + c] = -row[k];
        out.dnormal[(a * 12 + cRB + k) * C + c] = row[6 + k];
      }
    }
  }
}

// optional per-phase cycle accounting (tools/phase_timing.py; off in the product build)
#ifndef CM_PHASE_TIMING
#define CM_PHASE_TIMING 0
#endif
#if CM_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[4][5];
extern "C" int cm_debug_phase_cycles(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles));
}
#endif

#ifndef CM_MANIFOLD_THREADS
#define CM_MANIFOLD_THREADS 128
#endif
#ifndef CM_MANIFOLD_MINBLOCKS_FLAT
#define CM_MANIFOLD_MINBLOCKS_FLAT 3
#endif
#ifndef CM_MANIFOLD_MINBLOCKS
#define CM_MANIFOLD_MINBLOCKS 2
#endif
// CLS: SDF class (cm_internal.h ShapeRec); XPM: XPSQ mode of leaf_eval;
// flat SQ-family shapes get a tighter register budget (3 CTAs / SM)
template <int CLS> struct ClsTraits {
  static constexpr int XPM = CLS == 3 ? 0 : CLS;
  static constexpr bool FLAT = CLS == 0;
};
template <int TIER, int XP, int MB>
__global__ void __launch_bounds__(CM_MANIFOLD_THREADS, MB) k_contact_manifold(SceneDev S, const int32_t* __restrict__ pairs,
                                                          int64_t n_pairs, const int64_t* __restrict__ offsets,
                                                          const float* __restrict__ poses, int32_t n_slot,
                                                          cm_manifold_out out, int64_t C, int xp_filter,
                                                          float* __restrict__ scratch, int64_t scratch_floats,
                                                          uint32_t mode) {
  extern __shared__ float smem[];
  const bool full = (mode & CM_FULL_MODE) != 0;        // one contact per vertex and per edge
  const bool two = (mode & CM_TWO_SIDED) != 0;         // roles transposed as a second manifold
  constexpr int OV = TIER >= 2 ? 2 : 1;   // order at vertices / midpoints
  constexpr int OT = TIER >= 2 ? 1 : 0;   // order inside the trace
  const SmoothDev sp = S.sp;
  const float tcmp = sp.tau_cmp, itcmp = 1.f / tcmp;
  const float tmin = sp.tau_min, itmin = 1.f / tmin;
  const float tca = sp.tau_clip_alpha, itca = 1.f / tca;
  float* st = scratch ? scratch + (int64_t)blockIdx.x * scratch_floats : smem;
  __shared__ PairFrame Fs;
  __shared__ ShapeRec SA, SB;
  __shared__ int64_t s_off;

#if CM_PHASE_TIMING
  long long t_mark = 0;
#define CM_PT(k)                                                                             \
  if (threadIdx.x == 0) {                                                                    \
    long long t_now = clock64();                                                             \
    if (k > 0 || t_mark) atomicAdd(&g_phase_cycles[XP][k > 0 ? k - 1 : 4], (unsigned long long)(t_now - t_mark)); \
    t_mark = t_now;                                                                          \
  }
#else
#define CM_PT(k)
#endif
  const int64_t n_units = two ? 2 * n_pairs : n_pairs;
  for (int64_t un = blockIdx.x; un < n_units; un += gridDim.x) {
    const int64_t pi = two ? un >> 1 : un;
    const int side = two ? (int)(un & 1) : 0;         // 1: B sampled against A's SDF
    const int32_t* pr = pairs + 5 * pi;
    const int env = __ldg(pr + 0);
    const int slA = __ldg(pr + 1 + side), slB = __ldg(pr + 2 - side);
    const int shA = __ldg(pr + 3 + side), shB = __ldg(pr + 4 - side);
    const ShapeRec sa = S.shapes[shA];
    const ShapeRec sb = S.shapes[shB];
    if (xp_filter >= 0 && sb.uses_xpsq != xp_filter) continue;   // uniform across the CTA
    if (!sb.has_sdf || sa.F == 0) continue;                      // rejected by cm_manifold_size
    // output columns of the (t_A, theta_A, t_B, theta_B) blocks in the pair's
    // own (A, B) order: the transposed side writes its blocks swapped
    const int cTA = side ? 6 : 0, cRA = side ? 9 : 3, cTB = side ? 0 : 6, cRB = side ? 3 : 9;
    __syncthreads();   // previous pair's readers of Fs / st are done
    if (threadIdx.x == 0) {
      float pa[8], pb[8];
      const float* a = poses + 8 * ((int64_t)env * n_slot + slA);
      const float* b = poses + 8 * ((int64_t)env * n_slot + slB);
#pragma unroll
      for (int i = 0; i < 8; ++i) { pa[i] = __ldg(a + i); pb[i] = __ldg(b + i); }
      pair_frame(pa, pb, Fs);
      SA = sa;
      SB = sb;
      int64_t o = __ldg(offsets + pi);
      if (side) {
        const ShapeRec s0 = S.shapes[__ldg(pr + 3)];
        o += full ? (int64_t)s0.V + s0.E : (int64_t)s0.F;
      }
      s_off = o;
    }
    __syncthreads();
    CM_PT(0);
    const PairFrame& F = Fs;
    const int V = sa.V, E = sa.E, NF = sa.F;
    float* sv = st;                                   // vertex block
    float* se = st + (int64_t)vfields(TIER) * V;      // edge block
    const float* lv = S.verts + 3 * (int64_t)sa.v_off;
    const int32_t* ed = S.edges + 2 * (int64_t)sa.e_off;

    // ---- phase 1: vertices: phi, n (and H) of B -------------
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      const float x[3] = {__ldg(lv + 3 * v), __ldg(lv + 3 * v + 1), __ldg(lv + 3 * v + 2)};
      float xb[3], pw[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        xb[i] = F.Rrel[i * 3] * x[0] + F.Rrel[i * 3 + 1] * x[1] + F.Rrel[i * 3 + 2] * x[2] + F.trel[i];
        pw[i] = F.RA[i * 3] * x[0] + F.RA[i * 3 + 1] * x[1] + F.RA[i * 3 + 2] * x[2] + F.tA[i];
      }
      Res<OV> r;
      eval_shape<OV, ClsTraits<XP>::XPM, ClsTraits<XP>::FLAT>(S, SB, xb, r);
      float n[3];
      rot_vec(F.RB, r.g, n);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        sv[(VX + i) * V + v] = xb[i];
        sv[(VP + i) * V + v] = pw[i];
        sv[(VN + i) * V + v] = n[i];
      }
      sv[VD * V + v] = r.v;
      float h[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if constexpr (TIER >= 2) {
        rot_sym(F.RB, r.h, h);
#pragma unroll
        for (int k = 0; k < 6; ++k) sv[(VH + k) * V + v] = h[k];
      }
      if (full)
        store_candidate<TIER>(out, C, s_off + v, pw, n, r.v, h, nullptr, nullptr, F, 0, itcmp, cTA, cRA, cTB, cRB);
    }
    __syncthreads();
    CM_PT(1);

    // ---- phase 2: sphere traces (Fig. 2), 2 per edge -------------
    for (int j = threadIdx.x; j < 2 * E; j += blockDim.x) {
      const int e = j < E ? j : j - E;
      const int dir = j < E ? 0 : 1;     // 0: from v_I along +e_t; 1: from v_II along -e_t
      const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
      const float dl[3] = {__ldg(lv + 3 * vII) - __ldg(lv + 3 * vI), __ldg(lv + 3 * vII + 1) - __ldg(lv + 3 * vI + 1),
                           __ldg(lv + 3 * vII + 2) - __ldg(lv + 3 * vI + 2)};
      const float L = sqrtf(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
      const float iL = 1.f / L;
      const float el[3] = {dl[0] * iL, dl[1] * iL, dl[2] * iL};
      float eb[3], ew[3];
      rot_vec(F.Rrel, el, eb);
      rot_vec(F.RA, el, ew);
      const float xI[3] = {sv[(VX + 0) * V + vI], sv[(VX + 1) * V + vI], sv[(VX + 2) * V + vI]};
      const float pI[3] = {sv[(VP + 0) * V + vI], sv[(VP + 1) * V + vI], sv[(VP + 2) * V + vI]};
      const int v0 = dir ? vII : vI;
      float al = dir ? L : 0.f;
      const float sgn = dir ? -1.f : 1.f;
      float da[NDQ];
#pragma unroll
      for (int k = 0; k < NDQ; ++k) da[k] = 0.f;
      for (int it = 0; it < sp.iters; ++it) {
        float phi, g[3];
        if (it == 0) {   // the corner itself: reuse the vertex evaluation (reading #22)
          phi = sv[VD * V + v0];
          g[0] = sv[(VN + 0) * V + v0]; g[1] = sv[(VN + 1) * V + v0]; g[2] = sv[(VN + 2) * V + v0];
        } else {
          const float xb[3] = {fmaf(al, eb[0], xI[0]), fmaf(al, eb[1], xI[1]), fmaf(al, eb[2], xI[2])};
          Res<OT> r;
          eval_shape<OT, ClsTraits<XP>::XPM, ClsTraits<XP>::FLAT>(S, SB, xb, r);
          phi = r.v;
          if constexpr (TIER >= 2) rot_vec(F.RB, r.g, g);
        }
        // gated step G(phi) = sigma(phi / tau) phi  (reading #20)
        const float s = sigm(phi * itcmp);
        if constexpr (TIER >= 2) {
          // d alpha_{k+1} = d alpha_k + sgn G'(phi) [g^T J(p) dq + (g.e_t) d alpha_k]
          const float Gp = fmaf(phi * s * (1.f - s), itcmp, s);
          const float p[3] = {fmaf(al, ew[0], pI[0]), fmaf(al, ew[1], pI[1]), fmaf(al, ew[2], pI[2])};
          float gj[NDQ];
          gJ(g, p, F, gj);
          const float ge = g[0] * ew[0] + g[1] * ew[1] + g[2] * ew[2];
          const float c = sgn * Gp;
#pragma unroll
          for (int k = 0; k < NDQ; ++k) da[k] = fmaf(c, fmaf(ge, da[k], gj[k]), da[k]);
        }
        al = fmaf(sgn * s, phi, al);
      }
      // soft clip to the edge (reading #21)
      const float at = softclip(al, 0.f, L, tca, itca);
      se[(dir ? EB : EA) * E + e] = at;
      if constexpr (TIER >= 2) {
        const float cd = softclip_d(al, 0.f, L, itca);
        const int base = dir ? EDB : EDA;
#pragma unroll
        for (int k = 0; k < NDQ; ++k) se[(base + k) * E + e] = cd * da[k];
      }
    }
    __syncthreads();
    CM_PT(2);

    // ---- phase 3: edge midpoints p_e = (p_I + p_II)/2 ----------------
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
      const float dl[3] = {__ldg(lv + 3 * vII) - __ldg(lv + 3 * vI), __ldg(lv + 3 * vII + 1) - __ldg(lv + 3 * vI + 1),
                           __ldg(lv + 3 * vII + 2) - __ldg(lv + 3 * vI + 2)};
      const float iL = rsqrtf(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
      const float el[3] = {dl[0] * iL, dl[1] * iL, dl[2] * iL};
      float eb[3], ew[3];
      rot_vec(F.Rrel, el, eb);
      rot_vec(F.RA, el, ew);
      const float ab = 0.5f * (se[EA * E + e] + se[EB * E + e]);
      float dab[NDQ];
      if constexpr (TIER >= 2) {
#pragma unroll
        for (int k = 0; k < NDQ; ++k) dab[k] = 0.5f * (se[(EDA + k) * E + e] + se[(EDB + k) * E + e]);
      }
      float xb[3], pw[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        xb[i] = fmaf(ab, eb[i], sv[(VX + i) * V + vI]);
        pw[i] = fmaf(ab, ew[i], sv[(VP + i) * V + vI]);
      }
      Res<OV> r;
      eval_shape<OV, ClsTraits<XP>::XPM, ClsTraits<XP>::FLAT>(S, SB, xb, r);
      float n[3];
      rot_vec(F.RB, r.g, n);
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        se[(EP + i) * E + e] = pw[i];
        se[(EN + i) * E + e] = n[i];
      }
      se[ED * E + e] = r.v;
      float h[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if constexpr (TIER >= 2) {
        rot_sym(F.RB, r.h, h);
#pragma unroll
        for (int k = 0; k < 6; ++k) se[(EH + k) * E + e] = h[k];
#pragma unroll
        for (int k = 0; k < NDQ; ++k) se[(EDAB + k) * E + e] = dab[k];
      }
      if (full)
        store_candidate<TIER>(out, C, s_off + V + e, pw, n, r.v, h, ew, dab, F, 1, itcmp, cTA, cRA, cTB, cRB);
    }
    __syncthreads();
    CM_PT(3);
    if (full) continue;   // full mode: every candidate was written above

    // ---- phase 4: per-face fusion -------------------------------
    const int64_t off = s_off;
    const int32_t* fv = S.faces + 3 * (int64_t)sa.f_off;
    const int32_t* fe = S.face_edges + 3 * (int64_t)sa.f_off;
    const float itlm = LOG2E * itmin;
    for (int f = threadIdx.x; f < NF; f += blockDim.x) {
      int cv[3], ce[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) { cv[k] = __ldg(fv + 3 * f + k); ce[k] = __ldg(fe + 3 * f + k); }
      // candidate depths d_i; order [v_i0, v_i1, v_i2, e(i0,i1), e(i1,i2), e(i2,i0)]
      float dc[6];
#pragma unroll
      for (int k = 0; k < 3; ++k) { dc[k] = sv[VD * V + cv[k]]; dc[3 + k] = se[ED * E + ce[k]]; }
      float dm = dc[0];
#pragma unroll
      for (int i = 1; i < 6; ++i) dm = fminf(dm, dc[i]);
      float z[6], Z = 0.f;
#pragma unroll
      for (int i = 0; i < 6; ++i) { z[i] = ex2((dm - dc[i]) * itlm); Z += z[i]; }
      const float iZ = 1.f / Z;
      float zg[6];
      float Wf = 0.f;
      int dom = 0;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        z[i] *= iZ;                                   // z = s_argmax(-d)
        const float gam = sigm(-dc[i] * itcmp);        // gamma = [[d < 0]]
        zg[i] = z[i] * gam;
        Wf += zg[i];
        // dominant candidate argmax z_i gamma_i = argmin d_i (both factors
        // decrease with d_i); taken on d so it survives weight underflow
        if (dc[i] < dc[dom]) dom = i;
      }
      const float depth = fmaf(-tmin * LN2, lg2(Z), dm);   // smooth min (reading #25)
      float nrm[3] = {0.f, 0.f, 0.f}, qv[3] = {0.f, 0.f, 0.f}, pt[3] = {0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const bool isv = i < 3;
        const int id = isv ? cv[i] : ce[i - 3];
        const float* bp = isv ? sv + VP * V + id : se + EP * E + id;
        const float* bn = isv ? sv + VN * V + id : se + EN * E + id;
        const int sd = isv ? V : E;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const float p = bp[a * sd], nn = bn[a * sd];
          nrm[a] = fmaf(zg[i], nn, nrm[a]);
          qv[a] = fmaf(zg[i], p, qv[a]);
          pt[a] = fmaf(z[i], p, pt[a]);
        }
      }
      const int64_t c = off + f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        out.point[a * C + c] = pt[a];
        out.normal[a * C + c] = nrm[a];
      }
      out.depth[c] = depth;
      out.dom[c] = (int8_t)dom;
      if constexpr (TIER >= 1) {
        out.W[c] = Wf;
#pragma unroll
        for (int a = 0; a < 3; ++a) out.q[a * C + c] = qv[a];
      }
      if constexpr (TIER >= 2) {
        // Tier-2 derivatives in one pass over the 6 candidates.
        // With g_i = n_i, r = p - t:  d d_i = [g, p x g - tA x g, -(p x g) + tB x g]
        //   (+ (g.e_t) d alpha_bar for edge points),
        //   d depth = sum z_i d d_i,
        //   d n = sum_i c_i n_i (x) d d_i + itmin nbar (x) d depth + sum_i zg_i d n_i,
        //   c_i = zg_i (-1/tau_min - (1 - gamma_i)/tau_cmp),
        //   d n_i = [H, -H[p - tA]x, H[p - tB]x - [n]x] (+ H e_t (x) d alpha_bar).
        // The sums collapse to a few moments of the candidates:
        //   K = sum c n n^T, L = sum c n (p x n)^T, Hb = sum zg H, M = sum zg H[p]x
        //   -> d n = [K + Hb, L + K[tA]x + Hb[tA]x - M, -L - K[tB]x + M - Hb[tB]x - [nbar]x]
        //          + itmin nbar (x) d depth + sum_edges (c ge n + zg H e_t) (x) d alpha_bar
        float Sg[3] = {0.f, 0.f, 0.f}, Spg[3] = {0.f, 0.f, 0.f}, Se[NDQ];
        float K[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, Hb[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float Lm[9], Mm[9], dnE[3][NDQ];
#pragma unroll
        for (int k = 0; k < 9; ++k) { Se[k] = 0.f; Lm[k] = 0.f; Mm[k] = 0.f; }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int k = 0; k < NDQ; ++k) dnE[a][k] = 0.f;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const bool isv = i < 3;
          const int id = isv ? cv[i] : ce[i - 3];
          const float* bp = isv ? sv + VP * V + id : se + EP * E + id;
          const float* bn = isv ? sv + VN * V + id : se + EN * E + id;
          const float* bh = isv ? sv + VH * V + id : se + EH * E + id;
          const int sd = isv ? V : E;
          const float p[3] = {bp[0], bp[sd], bp[2 * sd]};
          const float n[3] = {bn[0], bn[sd], bn[2 * sd]};
          const float h[6] = {bh[0], bh[sd], bh[2 * sd], bh[3 * sd], bh[4 * sd], bh[5 * sd]};
          const float gam = sigm(-dc[i] * itcmp);
          const float w = zg[i];
          const float ci = w * (-itmin - (1.f - gam) * itcmp);
          const float pxn[3] = {p[1] * n[2] - p[2] * n[1], p[2] * n[0] - p[0] * n[2], p[0] * n[1] - p[1] * n[0]};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            Sg[a] = fmaf(z[i], n[a], Sg[a]);
            Spg[a] = fmaf(z[i], pxn[a], Spg[a]);
          }
          const float cn[3] = {ci * n[0], ci * n[1], ci * n[2]};
          K[0] = fmaf(cn[0], n[0], K[0]); K[1] = fmaf(cn[0], n[1], K[1]); K[2] = fmaf(cn[0], n[2], K[2]);
          K[3] = fmaf(cn[1], n[1], K[3]); K[4] = fmaf(cn[1], n[2], K[4]); K[5] = fmaf(cn[2], n[2], K[5]);
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) Lm[a * 3 + b] = fmaf(cn[a], pxn[b], Lm[a * 3 + b]);
#pragma unroll
          for (int k = 0; k < 6; ++k) Hb[k] = fmaf(w, h[k], Hb[k]);
          const float H[3][3] = {{h[0], h[1], h[2]}, {h[1], h[3], h[4]}, {h[2], h[4], h[5]}};
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            // (H [p]x) row a
            Mm[a * 3 + 0] = fmaf(w, H[a][1] * p[2] - H[a][2] * p[1], Mm[a * 3 + 0]);
            Mm[a * 3 + 1] = fmaf(w, H[a][2] * p[0] - H[a][0] * p[2], Mm[a * 3 + 1]);
            Mm[a * 3 + 2] = fmaf(w, H[a][0] * p[1] - H[a][1] * p[0], Mm[a * 3 + 2]);
          }
          if (!isv) {
            // sliding along the edge: e_t (world, unit) and d alpha_bar
            const int vI = __ldg(ed + 2 * id), vII = __ldg(ed + 2 * id + 1);
            float ew[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) ew[a] = sv[(VP + a) * V + vII] - sv[(VP + a) * V + vI];
            const float il = rsqrtf(ew[0] * ew[0] + ew[1] * ew[1] + ew[2] * ew[2]);
#pragma unroll
            for (int a = 0; a < 3; ++a) ew[a] *= il;
            const float ge = n[0] * ew[0] + n[1] * ew[1] + n[2] * ew[2];
            float u[3];   // c ge n + zg H e_t
#pragma unroll
            for (int a = 0; a < 3; ++a) u[a] = fmaf(ci * ge, n[a], w * (H[a][0] * ew[0] + H[a][1] * ew[1] + H[a][2] * ew[2]));
            const float zge = z[i] * ge;
#pragma unroll
            for (int k = 0; k < NDQ; ++k) {
              const float dk = se[(EDAB + k) * E + id];
              Se[k] = fmaf(zge, dk, Se[k]);
#pragma unroll
              for (int a = 0; a < 3; ++a) dnE[a][k] = fmaf(u[a], dk, dnE[a][k]);
            }
          }
        }
        // d depth = [Sg, Spg - tA x Sg, -Spg + tB x Sg] + Se
        const float* tA = F.tA;
        const float* tB = F.tB;
        float dd[NDQ];
        dd[0] = Sg[0] + Se[0]; dd[1] = Sg[1] + Se[1]; dd[2] = Sg[2] + Se[2];
        dd[3] = Spg[0] - (tA[1] * Sg[2] - tA[2] * Sg[1]) + Se[3];
        dd[4] = Spg[1] - (tA[2] * Sg[0] - tA[0] * Sg[2]) + Se[4];
        dd[5] = Spg[2] - (tA[0] * Sg[1] - tA[1] * Sg[0]) + Se[5];
        dd[6] = -Spg[0] + (tB[1] * Sg[2] - tB[2] * Sg[1]) + Se[6];
        dd[7] = -Spg[1] + (tB[2] * Sg[0] - tB[0] * Sg[2]) + Se[7];
        dd[8] = -Spg[2] + (tB[0] * Sg[1] - tB[1] * Sg[0]) + Se[8];
        // d n rows
        const float Ks[3][3] = {{K[0], K[1], K[2]}, {K[1], K[3], K[4]}, {K[2], K[4], K[5]}};
        const float Hs[3][3] = {{Hb[0], Hb[1], Hb[2]}, {Hb[1], Hb[3], Hb[4]}, {Hb[2], Hb[4], Hb[5]}};
        float dn[3][NDQ];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const float KH[3] = {Ks[a][0] + Hs[a][0], Ks[a][1] + Hs[a][1], Ks[a][2] + Hs[a][2]};
          // (X [t]x) row a for X = K + Hb, t = tA and tB
          const float xA[3] = {KH[1] * tA[2] - KH[2] * tA[1], KH[2] * tA[0] - KH[0] * tA[2], KH[0] * tA[1] - KH[1] * tA[0]};
          const float KtB[3] = {Ks[a][1] * tB[2] - Ks[a][2] * tB[1], Ks[a][2] * tB[0] - Ks[a][0] * tB[2],
                                Ks[a][0] * tB[1] - Ks[a][1] * tB[0]};
          const float HtB[3] = {Hs[a][1] * tB[2] - Hs[a][2] * tB[1], Hs[a][2] * tB[0] - Hs[a][0] * tB[2],
                                Hs[a][0] * tB[1] - Hs[a][1] * tB[0]};
          // [nbar]x row a
          const float nk[3] = {a == 0 ? 0.f : (a == 1 ? nrm[2] : -nrm[1]), a == 0 ? -nrm[2] : (a == 1 ? 0.f : nrm[0]),
                               a == 0 ? nrm[1] : (a == 1 ? -nrm[0] : 0.f)};
          const float nb = nrm[a] * itmin;
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            dn[a][b] = KH[b] + nb * dd[b] + dnE[a][b];
            dn[a][3 + b] = Lm[a * 3 + b] + xA[b] - Mm[a * 3 + b] + nb * dd[3 + b] + dnE[a][3 + b];
            dn[a][6 + b] = -Lm[a * 3 + b] - KtB[b] + Mm[a * 3 + b] - HtB[b] - nk[b] + nb * dd[6 + b] + dnE[a][6 + b];
          }
        }
        // store: q order (tA 0-2, thetaA 3-5, tB 6-8 = -tA, thetaB 9-11)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          out.ddepth[(cTA + k) * C + c] = dd[k];
          out.ddepth[(cRA + k) * C + c] = dd[3 + k];
          out.ddepth[(cTB + k) * C + c] = -dd[k];
          out.ddepth[(cRB + k) * C + c] = dd[6 + k];
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            out.dnormal[(a * 12 + cTA + k) * C + c] = dn[a][k];
            out.dnormal[(a * 12 + cRA + k) * C + c] = dn[a][3 + k];
            out.dnormal[(a * 12 + cTB + k) * C + c] = -dn[a][k];
            out.dnormal[(a * 12 + cRB + k) * C + c] = dn[a][6 + k];
          }
      }
    }
#if CM_PHASE_TIMING
    __syncthreads();
#endif
    CM_PT(4);
  }
}

namespace cml {

int64_t manifold_smem_floats(int V, int E, int tier) {
  return (int64_t)vfields(tier) * V + (int64_t)efields(tier) * E;
}

int manifold_max_smem_bytes() {
  static int m = 0;
  if (!m) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&m, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (m <= 0) m = 227 * 1024;
  }
  return m;
}

template <int TIER, int XP, int MB>
static int launch_manifold_v(const SceneDev& s, int xp_filter, bool use_smem, int64_t need, const int32_t* pairs,
                             int64_t n_pairs, const int64_t* offsets, const float* poses, int32_t n_slot,
                             const cm_manifold_out* out, int64_t C, float* scratch, int64_t scratch_floats,
                             cudaStream_t st, uint32_t mode) {
  const int threads = CM_MANIFOLD_THREADS;
  int smem = use_smem ? (int)need : 0;
  auto kern = k_contact_manifold<TIER, XP, MB>;
  static int configured = 0;
  if (smem > configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured = smem;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (!use_smem) {
    if (scratch == nullptr) {
      set_error("manifold: surface too large for shared memory and no scratch");
      return CM_ERR_UNSUPPORTED;
    }
    int64_t slots = scratch_floats / (need / 4);
    if (grid > slots) grid = slots;
    if (grid < 1) {
      set_error("manifold: scratch too small");
      return CM_ERR_UNSUPPORTED;
    }
  }
  const int64_t n_units = (mode & CM_TWO_SIDED) ? 2 * n_pairs : n_pairs;
  if (grid > n_units) grid = n_units;
  if (grid < 1) return CM_OK;
  kern<<<(unsigned)grid, threads, smem, st>>>(s, pairs, n_pairs, offsets, poses, n_slot, *out, C, xp_filter,
                                              use_smem ? nullptr : scratch, use_smem ? 0 : need / 4, mode);
  return check_launch("k_contact_manifold");
}

template <int TIER, int XP>
static int launch_manifold_t(const SceneDev& s, int xp_filter, int max_V, int max_E, const int32_t* pairs,
                             int64_t n_pairs, const int64_t* offsets, const float* poses, int32_t n_slot,
                             const cm_manifold_out* out, int64_t C, float* scratch, int64_t scratch_floats,
                             cudaStream_t st, uint32_t mode) {
  const int64_t need = manifold_smem_floats(max_V, max_E, TIER) * 4;
  const int static_smem = (int)(sizeof(PairFrame) + 2 * sizeof(ShapeRec));
  const bool use_smem = need <= kSmemBudget && need + static_smem + 1024 <= manifold_max_smem_bytes();
  // flat SQ-family SDFs: a 3-CTA/SM register budget pays off only when three
  // pairs' state also fits in shared memory (else the tighter budget just spills)
  if constexpr (XP == 0) {
    const bool hi = !use_smem || 3 * (need + static_smem + 1024) <= 228 * 1024;
    if (hi)
      return launch_manifold_v<TIER, XP, CM_MANIFOLD_MINBLOCKS_FLAT>(s, xp_filter, use_smem, need, pairs, n_pairs,
                                                                     offsets, poses, n_slot, out, C, scratch,
                                                                     scratch_floats, st, mode);
  }
  return launch_manifold_v<TIER, XP, CM_MANIFOLD_MINBLOCKS>(s, xp_filter, use_smem, need, pairs, n_pairs, offsets,
                                                            poses, n_slot, out, C, scratch, scratch_floats, st, mode);
}

int launch_manifold(const SceneDev& s, int class_mask, int max_V, int max_E, const int32_t* pairs,
                    int64_t n_pairs, const int64_t* offsets, const float* poses, int32_t n_slot, uint32_t flags,
                    const cm_manifold_out* out, int64_t C, float* scratch, int64_t scratch_floats, void* stream) {
  // class_mask bit c: SDF shapes of class c present (0 SQ family, 1 constant
  // schedule XPSQ, 2 varying-schedule XPSQ).  One instantiation per present
  // class; with several classes each kernel skips the other classes' pairs.
  cudaStream_t st = (cudaStream_t)stream;
  const int tier = (int)(flags & CM_TIER_MASK);
  const bool multi = (class_mask & (class_mask - 1)) != 0;
#define CM_L(T, X) launch_manifold_t<T, X>(s, multi ? X : -1, max_V, max_E, pairs, n_pairs, offsets, poses, n_slot, \
                                           out, C, scratch, scratch_floats, st, flags & (CM_FULL_MODE | CM_TWO_SIDED))
#define CM_T(X) (tier >= 2 ? CM_L(2, X) : (tier == 1 ? CM_L(1, X) : CM_L(0, X)))
  int rc = CM_OK;
  if (class_mask & 1) rc = CM_T(0);
  if (!rc && (class_mask & 2)) rc = CM_T(1);
  if (!rc && (class_mask & 4)) rc = CM_T(2);
  if (!rc && (class_mask & 8)) rc = CM_T(3);
#undef CM_T
#undef CM_L
  return rc;
}

}  // namespace cml
