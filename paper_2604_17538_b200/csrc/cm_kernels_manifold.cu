// sm_100a kernels of the contact-manifold hot path (arXiv 2604.17538 §II-C,
// P:129-163).  One unit = one (env, pair[, side]) manifold.  A call runs over
// chunks of units; per chunk and per SDF class four kernels run in stream
// order, each one CTA per unit:
//   k_mf_vertices  phi, n (, H) of B at A's sampled vertices
//   k_mf_traces    2 gated sphere traces per edge (+ d alpha / dq)
//   k_mf_midpoints phi, n (, H) of B at the edge points p_e
//   k_mf_faces     per-face softmax fusion of the 6 candidates
// Candidate state lives in a per-chunk global scratch slot (L2 resident for
// the chunk sizes used).  Splitting the phases into kernels removes the
// per-pair CTA barriers and keeps a single SDF-evaluation instance per kernel
// in the instruction cache (the fused one-CTA-per-pair kernel
// was instruction-fetch and barrier bound).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>

#include "cm_device.cuh"
#include "cm_internal.h"
#include "cm_param.cuh"
#include "cm_launch.h"

using namespace cmi;
using namespace cmd;

using cml::check_launch;
using cml::num_sms;

// CM_DEBUG_BOUNDS=1 builds (tests only: tools/build_variant.py dbg
// -DCM_DEBUG_BOUNDS=1) assert every gathered index and output row against
// its bounds -- the stand-in for compute-sanitizer, which is closed on this
// pool
#ifndef CM_DEBUG_BOUNDS
#define CM_DEBUG_BOUNDS 0
#endif
#if CM_DEBUG_BOUNDS
#include <cassert>
#define CM_ASSERT(c) assert(c)
#else
#define CM_ASSERT(c) ((void)0)
#endif

// ============================================================================
// per-unit scratch slot: one 16-B aligned record per candidate (vertex records
// first, then edge records), loaded and stored with 128-bit accesses
//   vertex record:               d, n[3] (world grad phi) | H[6] (world), pad[2]
//                                (tier 2: 12 floats, else 4)
//   edge record after traces:    a_I, da_I[9], a_II, da_II[9] (tier 2: 20 floats;
//                                else a_I, a_II in 8)
//   edge record after midpoint:  a_bar, d, n[3], H[6], da_bar[9] (else a_bar, d, n[3])
// tier 3 adds the second derivatives over the 9 independent coordinates
// z = (t_A, theta_A, theta_B) (t_B = -t_A by translation invariance), packed
// upper 9x9 (45): vertex record + d2d[45] at 12 (60 floats); per trace
// direction a, da[9], d2a[45] (56 floats each, a_II record at 56); after the
// midpoint d2d[45] at 20 (edge record 112 floats).
// ============================================================================
__host__ __device__ constexpr int vrec(int tier) { return tier >= 3 ? 60 : (tier >= 2 ? 12 : 4); }
__host__ __device__ constexpr int erec(int tier) { return tier >= 3 ? 112 : (tier >= 2 ? 20 : 8); }
__host__ __device__ constexpr int trace_b(int tier) { return tier >= 3 ? 56 : (tier >= 2 ? 10 : 1); }   // a_II offset
enum { VD2 = 12, TD2 = 10, MD2 = 20 };                    // tier-3 offsets of the 45 second derivatives
enum { VD = 0, VN = 1, VH = 4 };
enum { MAB = 0, MD = 1, MN = 2, MH = 5, MDAB = 11 };       // midpoint layout

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
// Ampere-style asynchronous 16-B copies global -> shared (per thread)
__device__ __forceinline__ void cp_async16(float* dst_smem, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// 45 floats from a 16-B aligned address (11 x 128-bit + 1)
__device__ __forceinline__ void ld45(const float* p, float* o) {
#pragma unroll
  for (int q = 0; q < 11; ++q) {
    const float4 v = ld4(p + 4 * q);
    o[4 * q] = v.x; o[4 * q + 1] = v.y; o[4 * q + 2] = v.z; o[4 * q + 3] = v.w;
  }
  o[44] = p[44];
}
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}

// ---- TMA bulk copies (cp.async.bulk global -> shared, mbarrier completion)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// bulk prefetch of `bytes` (multiple of 16, 16-B aligned) into L2 (no
// destination, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16-B aligned ends)
// by the calling thread; completion is counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
      ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

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
constexpr int N45 = 45;   // packed upper 9x9
__host__ __device__ constexpr int p9(int i, int j) { return i * 9 - i * (i - 1) / 2 + (j - i); }   // i <= j

// ---- tier 3: second derivatives over z = (t_A, theta_A, theta_B) ----------
// A material point p of the sampled body A, evaluated in the SDF of B (world
// gradient g, Hessian H), under world-frame left twists of A and B (B's
// translation held: its derivatives are minus t_A's):
//   w(z) = exp(-[th_B]x)(exp([th_A]x)(p - t_A) + t_A + dt_A - t_B) + t_B,
//   d^2 phi = J^T H J + G,  J = [I, -[r_A]x, [r_B]x]  (r_X = p - t_X),
//   G: (t_A, th_B) = -[g]x;  (th_A, th_A) = sym(g r_A^T) - (g.r_A) I;
//      (th_A, th_B) = -g r_A^T + (g.r_A) I;  (th_B, th_B) = sym(g r_B^T) - (g.r_B) I;
//   (the second-order terms of exp and of the cross terms -th_B x (dt_A + th_A x r_A)).
__device__ __forceinline__ void d2_point(const float* g, const float* h6, const float* p, const float* tA,
                                         const float* tB, float* o /*45*/) {
  const float ra[3] = {p[0] - tA[0], p[1] - tA[1], p[2] - tA[2]};
  const float rb[3] = {p[0] - tB[0], p[1] - tB[1], p[2] - tB[2]};
  const float H[3][3] = {{h6[0], h6[1], h6[2]}, {h6[1], h6[3], h6[4]}, {h6[2], h6[4], h6[5]}};
  // J (3 x 9): t_A -> e_a;  th_A -> e_a x r_A;  th_B -> r_B x e_b
  const float J[3][9] = {{1.f, 0.f, 0.f, 0.f, ra[2], -ra[1], 0.f, -rb[2], rb[1]},
                         {0.f, 1.f, 0.f, -ra[2], 0.f, ra[0], rb[2], 0.f, -rb[0]},
                         {0.f, 0.f, 1.f, ra[1], -ra[0], 0.f, -rb[1], rb[0], 0.f}};
  float HJ[3][9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int c = 0; c < 9; ++c) HJ[i][c] = H[i][0] * J[0][c] + H[i][1] * J[1][c] + H[i][2] * J[2][c];
  const float gra = g[0] * ra[0] + g[1] * ra[1] + g[2] * ra[2];
  const float grb = g[0] * rb[0] + g[1] * rb[1] + g[2] * rb[2];
#pragma unroll
  for (int c1 = 0; c1 < 9; ++c1)
#pragma unroll
    for (int c2 = c1; c2 < 9; ++c2) {
      float v = J[0][c1] * HJ[0][c2] + J[1][c1] * HJ[1][c2] + J[2][c1] * HJ[2][c2];
      if (c1 < 3 && c2 >= 6) {                     // (t_A a, th_B b): eps_abk g_k
        const int a = c1, b = c2 - 6;
        v += (a == b) ? 0.f : ((b == (a + 1) % 3) ? g[(a + 2) % 3] : -g[(a + 1) % 3]);
      } else if (c1 >= 3 && c1 < 6 && c2 < 6) {   // (th_A a, th_A b)
        const int a = c1 - 3, b = c2 - 3;
        v += 0.5f * (g[a] * ra[b] + g[b] * ra[a]) - (a == b ? gra : 0.f);
      } else if (c1 >= 3 && c1 < 6 && c2 >= 6) {  // (th_A a, th_B b)
        const int a = c1 - 3, b = c2 - 6;
        v += -g[a] * ra[b] + (a == b ? gra : 0.f);
      } else if (c1 >= 6) {                        // (th_B a, th_B b)
        const int a = c1 - 6, b = c2 - 6;
        v += 0.5f * (g[a] * rb[b] + g[b] * rb[a]) - (a == b ? grb : 0.f);
      }
      o[p9(c1, c2)] = v;
    }
}
// for a point sliding along the edge direction e_t (world): phi_za (9) =
// J^T H e_t + (0, e_t x g, g x e_t) and phi_aa = e_t^T H e_t
__device__ __forceinline__ void d2_alpha(const float* g, const float* h6, const float* p, const float* ew,
                                         const float* tA, const float* tB, float* fza, float& faa) {
  const float ra[3] = {p[0] - tA[0], p[1] - tA[1], p[2] - tA[2]};
  const float rb[3] = {p[0] - tB[0], p[1] - tB[1], p[2] - tB[2]};
  const float He[3] = {h6[0] * ew[0] + h6[1] * ew[1] + h6[2] * ew[2], h6[1] * ew[0] + h6[3] * ew[1] + h6[4] * ew[2],
                       h6[2] * ew[0] + h6[4] * ew[1] + h6[5] * ew[2]};
  const float exg[3] = {ew[1] * g[2] - ew[2] * g[1], ew[2] * g[0] - ew[0] * g[2], ew[0] * g[1] - ew[1] * g[0]};
  fza[0] = He[0]; fza[1] = He[1]; fza[2] = He[2];
  fza[3] = ra[1] * He[2] - ra[2] * He[1] + exg[0];    // (r_A x He) + e_t x g
  fza[4] = ra[2] * He[0] - ra[0] * He[2] + exg[1];
  fza[5] = ra[0] * He[1] - ra[1] * He[0] + exg[2];
  fza[6] = He[1] * rb[2] - He[2] * rb[1] - exg[0];    // (He x r_B) + g x e_t
  fza[7] = He[2] * rb[0] - He[0] * rb[2] - exg[1];
  fza[8] = He[0] * rb[1] - He[1] * rb[0] - exg[2];
  faa = ew[0] * He[0] + ew[1] * He[1] + ew[2] * He[2];
}
// total second derivative along alpha(z): D2 = fzz + fza da^T + da fza^T + faa da da^T + fa d2a
__device__ __forceinline__ void d2_total(float* fzz, const float* fza, float faa, float fa, const float* da,
                                         const float* d2a) {
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) {
      const int k = p9(i, j);
      fzz[k] = fmaf(fa, d2a[k], fmaf(faa * da[i], da[j], fmaf(fza[i], da[j], fmaf(da[i], fza[j], fzz[k]))));
    }
}
// 9x9 (z) -> packed 12x12 in the pair's column order: local coordinates
// (t_s, th_s, t_f, th_f) of the side map to z with t_f = -t_s; the
// transposed side (side 1) lists the pair's B block first
template <int SIDE>
__device__ __forceinline__ void store_d2_t(float* out, int64_t C, int64_t c, const float* h45) {
  int k = 0;
#pragma unroll
  for (int i = 0; i < 12; ++i)
#pragma unroll
    for (int j = i; j < 12; ++j, ++k) {
      const int li = SIDE ? (i + 6) % 12 : i, lj = SIDE ? (j + 6) % 12 : j;
      const int ui = li < 6 ? li : (li < 9 ? li - 6 : li - 3), uj = lj < 6 ? lj : (lj < 9 ? lj - 6 : lj - 3);
      const float si = (li >= 6 && li < 9) ? -1.f : 1.f, sj = (lj >= 6 && lj < 9) ? -1.f : 1.f;
      const int a = ui < uj ? ui : uj, b = ui < uj ? uj : ui;
      out[(int64_t)k * C + c] = si * sj * h45[p9(a, b)];
    }
}
__device__ __forceinline__ void store_d2(float* out, int64_t C, int64_t c, const float* h45, int side) {
  if (side) store_d2_t<1>(out, C, c, h45);
  else store_d2_t<0>(out, C, c, h45);
}

// Full mode (V + E contacts): candidate i is its own contact.
//   point p, normal n = grad phi (raw), depth d, W = gamma, q = gamma p (so the
//   compact J = gamma J_i, the single-candidate case of P:161), dom = kind
//   (0 vertex, 1 edge point); tier 2: d d / dq = g^T J(p) (+ (g.e_t) d alpha_bar),
//   d n / dq = [H, -H[p - tA]x, (-H), H[p - tB]x - [n]x] (+ H e_t d alpha_bar^T).
template <int TIER>
__device__ __forceinline__ void store_candidate(const cm_manifold_out& out, int64_t C, int64_t c, const float* p,
                                                const float* n, float d, const float* h, const float* ew,
                                                const float* dab, const PairFrame& F, int kind, float itcmp, int cTA,
                                                int cRA, int cTB, int cRB, const float* d2 = nullptr, int side = 0) {
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
  if constexpr (TIER >= 3) store_d2(out.d2depth, C, c, d2, side);
}

// ============================================================================
// unit set-up shared by the four kernels
// ============================================================================
struct MfArgs {
  SceneDev S;
  const int32_t* pairs;
  int64_t n_pairs;
  int64_t unit0;             // first unit of this chunk
  const int64_t* offsets;
  const float* poses;
  int64_t n_env;
  int32_t n_slot;
  cm_manifold_out out;
  int64_t C;
  float* scratch;            // chunk scratch, one slot of `slot` floats per unit
  int64_t slot;
  uint32_t mode;
  struct UnitCtx* ctx;       // per-unit set-up of the chunk (k_mf_units)
  int* cls_count;            // [CM_N_CLASSES] valid units of the chunk per SDF class
  int* cls_list;             // [CM_N_CLASSES][chunk] their unit indices
  int64_t chunk;             // list stride
  int64_t nb;                // units of this chunk
};

struct alignas(16) UnitCtx {
  PairFrame F;
  ShapeRec SA, SB;
  int64_t off;               // first output row of this unit
  int side;
  int valid;                 // the unit has a manifold (SDF side and a surface)
  int cls;                   // SDF class of the unit's SDF shape
  int bad;                   // invalid record with output rows (filled with NaN)
  int culled;                // broad phase (f2): certified inactive, rows written by k_mf_culled
  float lb;                  // its certified lower bound on every candidate depth
};
static_assert(sizeof(UnitCtx) % 16 == 0, "UnitCtx is copied as float4");

// threads per unit CTA: 64 for large batches (lane use on V = 56..98 meshes);
// small batches get up to CM_MF_MAX_THREADS so the SMs still fill
#define CM_N_CLASSES 5   // SDF classes (cm_internal.h ShapeRec::uses_xpsq)
#define CM_N_LISTS 6     // + the broad phase's culled units (list CM_N_CLASSES)
#ifndef CM_MF_STAGE_MID
#define CM_MF_STAGE_MID 0   // TMA-staged trace records in the midpoint kernel: C5 -7%, C4 -0.5% (r02i sweep)
#endif
#ifndef CM_TRACE6
#define CM_TRACE6 1         // 6-component trace derivative recursion (tiers 0-2)
#endif
#ifndef CM_MF_FACE_L1PF
#define CM_MF_FACE_L1PF 1   // face kernel: L1 prefetch of the unit's records at the start (C5 +1.5%, r02zz3);
                            // 2: also the mesh's vertex and edge-geometry tables
#endif
#ifndef CM_MF_TRACE_L1PF
#define CM_MF_TRACE_L1PF 0   // trace kernel: L1 prefetch of the unit's vertex records at the start (no gain: r02zz7)
#endif
#ifndef CM_MF_TABLE_L1PF
#define CM_MF_TABLE_L1PF 0   // vertex / midpoint kernels: L1 prefetch of the mesh's vertex / edge tables (C5 -0.3%: r02zz8)
#endif
#ifndef CM_MF_MID_L1PF
#define CM_MF_MID_L1PF 1   // midpoint kernel: L1 prefetch of the unit's trace records at the start
#endif
#ifndef CM_TRACE_PAIRED
#define CM_TRACE_PAIRED 0   // tiers 0-2: both traces of an edge on adjacent lanes, one averaged record
                            // (-18 KB DRAM per C5 pair, bitwise equal; C5 -1.3%, C4 0, C3 +0.3%: r02zf)
#endif
#define CM_PAIRED_REC (CM_TRACE_PAIRED && CM_TRACE6)   // (the paired traces are the 6-component kernel's)
#ifndef CM_MF_MID_PREFETCH
#define CM_MF_MID_PREFETCH 0   // tier-2 midpoint kernel: next trace record by cp.async into shared memory:
                               // bitwise equal, C5 -4.5%, C4 -2.3% (r02z9)
#endif
#ifndef CM_MF_FUSE_EDGES
#define CM_MF_FUSE_EDGES 0  // traces + midpoints in one kernel, one thread per edge (tiers 0-2): bitwise equal,
                            // C5 -19%, C4 -47% (XPSQ classes: instruction-cache stalls; r02z2)
#endif
#ifndef CM_MF_EDGE_SMEM
#define CM_MF_EDGE_SMEM 0   // the edge kernel parks the first trace's result in shared memory
#endif
#ifndef CM_MF_REG_E_XP0
#define CM_MF_REG_E_XP0 0   // register cap of the SQ-family edge kernel (0: the trace / midpoint budget)
#endif
#ifndef CM_MF_REG_E_XP1
#define CM_MF_REG_E_XP1 0   // register cap of the order-2 XPSQ edge kernels (0: the midpoint budget)
#endif
#ifndef CM_MF_THREADS
#define CM_MF_THREADS 64
#endif
#define CM_MF_MAX_THREADS 256
// minimum resident 256-thread blocks per SM, i.e. register budgets of
// 65536 / (256 MINB): 128 registers except the order-2 XPSQ evaluations
// (measured on C5 / C4 / C3); flat SQ-family class: 80
#ifndef CM_MF_MINB_V
#define CM_MF_MINB_V 2
#endif
#ifndef CM_MF_MINB_T
#define CM_MF_MINB_T 2
#endif
#ifndef CM_MF_MINB_M
#define CM_MF_MINB_M 2
#endif
#ifndef CM_MF_MINB_V_XP0
#define CM_MF_MINB_V_XP0 3
#endif
#ifndef CM_MF_MINB_M_XP0
#define CM_MF_MINB_M_XP0 3
#endif
#ifndef CM_MF_MINB_T_XP0
#define CM_MF_MINB_T_XP0 3
#endif
#ifndef CM_MF_MINB_V_XP1
#define CM_MF_MINB_V_XP1 1
#endif
#ifndef CM_MF_MINB_M_XP1
#define CM_MF_MINB_M_XP1 1
#endif
template <int TIER, int XP> struct MinB {
  // tier 3 (second derivatives) carries 45-component arrays: full register file
  static constexpr int VERTICES = TIER >= 3 ? 1 : ((XP == 1 || XP == 4) ? CM_MF_MINB_V_XP1 : (XP == 0 ? CM_MF_MINB_V_XP0 : CM_MF_MINB_V));
  static constexpr int TRACES = TIER >= 3 ? 1 : (XP == 0 ? CM_MF_MINB_T_XP0 : CM_MF_MINB_T);
  static constexpr int MIDPOINTS = TIER >= 3 ? 1 : ((XP == 1 || XP == 4) ? CM_MF_MINB_M_XP1 : (XP == 0 ? CM_MF_MINB_M_XP0 : CM_MF_MINB_M));
};
// per-thread register caps (__maxnreg__) equivalent to MINB resident
// 256-thread blocks: 3 -> 80, 2 -> 128, 1 -> 255; CM_MF_REG_XP1 overrides the
// order-2 XPSQ kernels (vertices, midpoints)
__host__ __device__ constexpr int regs_of(int minb) { return minb >= 3 ? 80 : (minb == 2 ? 128 : 255); }
#ifndef CM_MF_REG_XP1
#define CM_MF_REG_XP1 168   // measured: C5 +1%, C4 +5% over 255 (144 and 128 lose)
#endif
#ifndef CM_MF_REG_T_XP1
#define CM_MF_REG_T_XP1 0
#endif
#ifndef CM_MF_REG_T3
#define CM_MF_REG_T3 0   // register cap of the tier-3 kernels (0: 255)
#endif
template <int TIER, int XP> struct RegCap {
  static constexpr int VERTICES = (TIER >= 3 && CM_MF_REG_T3) ? CM_MF_REG_T3 : ((TIER == 2 && (XP == 1 || XP == 4) && CM_MF_REG_XP1) ? CM_MF_REG_XP1 : regs_of(MinB<TIER, XP>::VERTICES));
  static constexpr int TRACES = (TIER >= 3 && CM_MF_REG_T3) ? CM_MF_REG_T3 : ((TIER == 2 && (XP == 1 || XP == 4) && CM_MF_REG_T_XP1) ? CM_MF_REG_T_XP1 : regs_of(MinB<TIER, XP>::TRACES));
  static constexpr int MIDPOINTS = (TIER >= 3 && CM_MF_REG_T3) ? CM_MF_REG_T3 : ((TIER == 2 && (XP == 1 || XP == 4) && CM_MF_REG_XP1) ? CM_MF_REG_XP1 : regs_of(MinB<TIER, XP>::MIDPOINTS));
};
#ifndef CM_MF_FACE_MINB
#define CM_MF_FACE_MINB 2   // face kernel: <= 128 registers
#endif

// the set-up of unit un: pair, side, shapes, frame and first output row
__device__ __forceinline__ void unit_resolve(const MfArgs& a, int64_t un, UnitCtx& U) {
  const bool full = (a.mode & CM_FULL_MODE) != 0;
  const bool two = (a.mode & CM_TWO_SIDED) != 0;
  const int64_t pi = two ? un >> 1 : un;
  const int side = two ? (int)(un & 1) : 0;          // 1: B sampled against A's SDF
  const int32_t* pr = a.pairs + 5 * pi;
  const int env = __ldg(pr + 0);
  const int slA = __ldg(pr + 1 + side), slB = __ldg(pr + 2 - side);
  const int shA = __ldg(pr + 3 + side), shB = __ldg(pr + 4 - side);
  U.valid = 0;
  U.cls = -1;
  U.bad = 0;
  U.culled = 0;
  U.lb = 0.f;
  // record validation: out-of-range shape ids (the offsets kernel gave the
  // pair no rows), env or slot indices (its rows are filled with NaN by
  // k_mf_units), or a shape without the needed surface / SDF: counted in
  // the scene's error word, never dereferenced
  const int ns = a.S.n_shapes;
  if ((unsigned)shA >= (unsigned)ns || (unsigned)shB >= (unsigned)ns) {
    atomicAdd(a.S.err, 1u);
    return;
  }
  const ShapeRec sa = a.S.shapes[shA];
  const ShapeRec sb = a.S.shapes[shB];
  if ((int64_t)(unsigned)env >= a.n_env || (unsigned)slA >= (unsigned)a.n_slot || (unsigned)slB >= (unsigned)a.n_slot ||
      !(sb.has_sdf && sa.F > 0)) {
    atomicAdd(a.S.err, 1u);
    U.bad = 1;
  }
  const int ok = !U.bad;
  U.SA = sa;
  {
    int64_t o = __ldg(a.offsets + pi);
    if (side) {
      const ShapeRec s0 = a.S.shapes[__ldg(pr + 3)];
      o += full ? (int64_t)s0.V + s0.E : (int64_t)s0.F;
    }
    U.off = o;
    U.side = side;
  }
  if (ok) {
    const float4* A = reinterpret_cast<const float4*>(a.poses + 8 * ((int64_t)env * a.n_slot + slA));
    const float4* B = reinterpret_cast<const float4*>(a.poses + 8 * ((int64_t)env * a.n_slot + slB));
    const float4 a0 = __ldg(A), a1 = __ldg(A + 1), b0 = __ldg(B), b1 = __ldg(B + 1);
    const float pa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float pb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    pair_frame(pa, pb, U.F);
    U.SB = sb;
    U.valid = 1;
    U.cls = sb.uses_xpsq;
    if (a.mode & CM_BROAD_PHASE) {
      // certified culling (reading #46): every candidate lies in
      // A's vertex sphere and phi_B >= |x - c_B| - rho_B
      const float4 ma = __ldg(a.S.bounds + 2 * shA), mb = __ldg(a.S.bounds + 2 * shB + 1);
      if (mb.w < INFINITY && ma.w >= 0.f) {
        const float ca[3] = {ma.x, ma.y, ma.z}, cb[3] = {mb.x, mb.y, mb.z};
        float wa[3], wb[3];
        rot_vec(U.F.RA, ca, wa);
        rot_vec(U.F.RB, cb, wb);
        const float dx = wa[0] + U.F.tA[0] - wb[0] - U.F.tB[0], dy = wa[1] + U.F.tA[1] - wb[1] - U.F.tB[1],
                    dz = wa[2] + U.F.tA[2] - wb[2] - U.F.tB[2];
        const float lb = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))) - ma.w - mb.w;
        if (lb > 40.f * a.S.sp.tau_cmp) {
          U.valid = 0;
          U.culled = 1;
          U.lb = lb;
        }
      }
    }
  }
}

// per-chunk prologue: one thread per unit resolves its set-up once for the
// chunk's kernels (they copy it with 128-bit loads instead of each
// re-deriving it through dependent loads on one thread)
__global__ void __launch_bounds__(128) k_mf_units(const MfArgs a, int64_t nb) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = u < nb;
  UnitCtx U;
  U.valid = 0;
  U.cls = -1;
  U.bad = 0;
  U.culled = 0;
  if (in) unit_resolve(a, a.unit0 + u, U);
  if (in && U.bad) {   // an invalid record's rows: NaN in every float field, dom -1
    const bool fm = (a.mode & CM_FULL_MODE) != 0;
    const int nr = fm ? U.SA.V + U.SA.E : U.SA.F;
    const float qn = __int_as_float(0x7fc00000);
    const cm_manifold_out& o = a.out;
    const int64_t C = a.C;
    for (int r = 0; r < nr; ++r) {
      const int64_t c = U.off + r;
      for (int k = 0; k < 3; ++k) { o.point[k * C + c] = qn; o.normal[k * C + c] = qn; }
      o.depth[c] = qn;
      o.dom[c] = (int8_t)-1;
      if (o.W) o.W[c] = qn;
      if (o.q) for (int k = 0; k < 3; ++k) o.q[k * C + c] = qn;
      if (o.ddepth) for (int k = 0; k < 12; ++k) o.ddepth[k * C + c] = qn;
      if (o.dnormal) for (int k = 0; k < 36; ++k) o.dnormal[k * C + c] = qn;
      if (o.d2depth) for (int k = 0; k < 78; ++k) o.d2depth[k * C + c] = qn;
    }
  }
  // class lists in unit order within the block (ballot ranks + one atomic per
  // block and class), so neighbouring CTAs of a phase kernel take
  // neighbouring units
  __shared__ int s_cnt[CM_N_LISTS][4], s_base[CM_N_LISTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int rank = 0;
  // list of the unit: its SDF class, or the culled list
  const int mylist = !in ? -1 : (U.valid ? U.cls : (U.culled ? CM_N_CLASSES : -1));
#pragma unroll
  for (int c = 0; c < CM_N_LISTS; ++c) {
    const unsigned m = __ballot_sync(0xffffffffu, mylist == c);
    if (lane == 0) s_cnt[c][warp] = __popc(m);
    if (mylist == c) rank = __popc(m & lt);
  }
  __syncthreads();
  if (threadIdx.x < CM_N_LISTS) {
    const int c = threadIdx.x;
    const int tot = s_cnt[c][0] + s_cnt[c][1] + s_cnt[c][2] + s_cnt[c][3];
    s_base[c] = tot ? atomicAdd(a.cls_count + c, tot) : 0;
  }
  __syncthreads();
  if (!in) return;
  if (mylist >= 0) {
    const int c = mylist;
    int pre = 0;
    for (int w = 0; w < warp; ++w) pre += s_cnt[c][w];
    a.cls_list[(int64_t)c * a.chunk + s_base[c] + pre + rank] = (int)u;
  }
  float4* dst = reinterpret_cast<float4*>(a.ctx + u);
  const float4* src = reinterpret_cast<const float4*>(&U);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(UnitCtx) / 16); ++i) dst[i] = src[i];
}

// CLS: SDF class (cm_internal.h ShapeRec); XPM: XPSQ mode of leaf_eval
template <int CLS> struct ClsTraits {
  static constexpr int XPM = CLS == 3 ? 0 : (CLS == 4 ? 1 : CLS);
  static constexpr bool FLAT = CLS == 0;
  static constexpr bool CULL = CLS == 4;     // XPSQ operands of boolean trees
  static constexpr bool SINGLE = CLS == 1;   // a lone constant-schedule XPSQ
};
#define CM_EVAL(O, XP) eval_shape<O, ClsTraits<XP>::XPM, ClsTraits<XP>::FLAT, true, ClsTraits<XP>::CULL, ClsTraits<XP>::SINGLE>

// output columns of the (t_A, theta_A, t_B, theta_B) blocks in the pair's own
// (A, B) order: the transposed side writes its blocks swapped
#define CM_COLS(side) \
  const int cTA = (side) ? 6 : 0, cRA = (side) ? 9 : 3, cTB = (side) ? 0 : 6, cRB = (side) ? 3 : 9

// static edge geometry of the sampled surface (scene creation, FP64 from the
// FP32 vertices): x_I (local), L, unit direction e_t (local) in two float4
__device__ __forceinline__ void edge_geom(const float* eg, int e, float* xI, float& L, float* el) {
  const float4 g0 = __ldg(reinterpret_cast<const float4*>(eg) + 2 * e);
  const float4 g1 = __ldg(reinterpret_cast<const float4*>(eg) + 2 * e + 1);
  xI[0] = g0.x; xI[1] = g0.y; xI[2] = g0.z; L = g0.w;
  el[0] = g1.x; el[1] = g1.y; el[2] = g1.z;
}

// x_B = Rrel x + trel (B frame) and p = RA x + tA (world) of a local point
__device__ __forceinline__ void to_frames(const PairFrame& F, const float* x, float* xb, float* pw) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    xb[i] = F.Rrel[i * 3] * x[0] + F.Rrel[i * 3 + 1] * x[1] + F.Rrel[i * 3 + 2] * x[2] + F.trel[i];
    pw[i] = F.RA[i * 3] * x[0] + F.RA[i * 3 + 1] * x[1] + F.RA[i * 3 + 2] * x[2] + F.tA[i];
  }
}
__device__ __forceinline__ float4 ldv(const float* lv, int v) {   // padded vertex
  return __ldg(reinterpret_cast<const float4*>(lv) + v);
}
__device__ __forceinline__ void vertex_frames(const PairFrame& F, const float* lv, int v, float* xb, float* pw) {
  const float4 x4 = ldv(lv, v);
  const float x[3] = {x4.x, x4.y, x4.z};
  to_frames(F, x, xb, pw);
}

// ---- phase 1: vertices: phi, n (and H) of B ----------------
template <int TIER, int XP>
__device__ __forceinline__ void mf_vertices_unit(const MfArgs& a, const UnitCtx& U, int u) {
  constexpr int OV = TIER >= 2 ? 2 : 1;
  const PairFrame& F = U.F;
  const int V = U.SA.V;
  float* sv = a.scratch + (int64_t)u * a.slot;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const bool full = (a.mode & CM_FULL_MODE) != 0;
  const float itcmp = a.S.sp.i_cmp;
  if (CM_MF_TABLE_L1PF) {   // the mesh's vertex table into L1
    for (int o = threadIdx.x * 32; o < 4 * V; o += blockDim.x * 32)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(lv + o));
  }
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    float xb[3], pw[3];
    vertex_frames(F, lv, v, xb, pw);
    Res<OV> r;
    CM_EVAL(OV, XP)(a.S, U.SB, xb, r);
    float n[3];
    rot_vec(F.RB, r.g, n);
    float* rec = sv + v * vrec(TIER);
    st4(rec, r.v, n[0], n[1], n[2]);
    float h[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if constexpr (TIER >= 2) {
      rot_sym(F.RB, r.h, h);
      st4(rec + 4, h[0], h[1], h[2], h[3]);
      st4(rec + 8, h[4], h[5], 0.f, 0.f);
    }
    float d2[TIER >= 3 ? N45 : 1];
    if constexpr (TIER >= 3) {
      d2_point(n, h, pw, F.tA, F.tB, d2);
#pragma unroll
      for (int k = 0; k < N45; ++k) rec[VD2 + k] = d2[k];
    }
    if (full) {
      CM_COLS(U.side);
      store_candidate<TIER>(a.out, a.C, U.off + v, pw, n, r.v, h, nullptr, nullptr, F, 0, itcmp, cTA, cRA, cTB, cRB,
                            d2, U.side);
    }
  }
}

// ---- phase 2: sphere traces (Fig. 2), 2 per edge ----------------
template <int TIER, int XP>
__device__ __forceinline__ void mf_traces_unit(const MfArgs& a, const UnitCtx& U, int u) {
  constexpr int OT = TIER >= 3 ? 2 : (TIER >= 2 ? 1 : 0);   // order inside the trace
  const SmoothDev sp = a.S.sp;
  const float itcmp = sp.i_cmp;
  const float tca = sp.tau_clip_alpha, itca = sp.i_clip_alpha;
  const PairFrame& F = U.F;
  const int V = U.SA.V, E = U.SA.E;
  const float* sv = a.scratch + (int64_t)u * a.slot;
  float* se = a.scratch + (int64_t)u * a.slot + (int64_t)vrec(TIER) * V;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const int32_t* ed = a.S.edges + 2 * (int64_t)U.SA.e_off;
  for (int j = threadIdx.x; j < 2 * E; j += blockDim.x) {
    const int e = j < E ? j : j - E;
    const int dir = j < E ? 0 : 1;     // 0: from v_I along +e_t; 1: from v_II along -e_t
    const int v0 = __ldg(ed + 2 * e + dir);
    const float4 corner = ld4(sv + v0 * vrec(TIER));   // d, n of the start vertex (issued early)
    // edge geometry from the vertex buffer here (the static edge table of
    // the other kernels measured 3% slower in this one)
    float xl[3], el[3], L;
    {
      const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
      const float4 xa = ldv(lv, vI), xb4 = ldv(lv, vII);
      const float dl[3] = {xb4.x - xa.x, xb4.y - xa.y, xb4.z - xa.z};
      L = sqrtf(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
      const float iL = 1.f / L;
      el[0] = dl[0] * iL; el[1] = dl[1] * iL; el[2] = dl[2] * iL;
      xl[0] = xa.x; xl[1] = xa.y; xl[2] = xa.z;
    }
    float eb[3], ew[3];
    rot_vec(F.Rrel, el, eb);
    rot_vec(F.RA, el, ew);
    float xI[3], pI[3];
    to_frames(F, xl, xI, pI);
    float al = dir ? L : 0.f;
    const float sgn = dir ? -1.f : 1.f;
    float da[NDQ];
#pragma unroll
    for (int k = 0; k < NDQ; ++k) da[k] = 0.f;
    constexpr int N2 = TIER >= 3 ? N45 : 1;
    float d2a[N2];
#pragma unroll
    for (int k = 0; k < N2; ++k) d2a[k] = 0.f;
    for (int it = 0; it < sp.iters; ++it) {
      float phi, g[3];
      float h[6], fzz[N2];   // tier 3: world Hessian and d^2 phi / dz^2 at the iterate
      if (it == 0) {   // the corner itself: reuse the vertex evaluation (reading #22)
        phi = corner.x;
        g[0] = corner.y; g[1] = corner.z; g[2] = corner.w;
        if constexpr (TIER >= 3) {
          const float* cr = sv + v0 * vrec(TIER);
#pragma unroll
          for (int k = 0; k < 6; ++k) h[k] = cr[VH + k];
          ld45(cr + VD2, fzz);
        }
      } else {
        const float xb[3] = {fmaf(al, eb[0], xI[0]), fmaf(al, eb[1], xI[1]), fmaf(al, eb[2], xI[2])};
        Res<OT> r;
        CM_EVAL(OT, XP)(a.S, U.SB, xb, r);
        phi = r.v;
        if constexpr (TIER >= 2) rot_vec(F.RB, r.g, g);
        if constexpr (TIER >= 3) {
          rot_sym(F.RB, r.h, h);
          const float p[3] = {fmaf(al, ew[0], pI[0]), fmaf(al, ew[1], pI[1]), fmaf(al, ew[2], pI[2])};
          d2_point(g, h, p, F.tA, F.tB, fzz);
        }
      }
      // gated step G(phi) = sigma(phi / tau) phi  (reading #20)
      const float s = sigm(phi * itcmp);
      if constexpr (TIER >= 3) {
        // d2 alpha_{k+1} = d2 alpha_k + sgn [G'' Dphi Dphi^T + G' D2phi] with
        // Dphi = phi_z + phi_a d alpha_k and D2phi the total second derivative
        const float p[3] = {fmaf(al, ew[0], pI[0]), fmaf(al, ew[1], pI[1]), fmaf(al, ew[2], pI[2])};
        float gj[NDQ], fza[NDQ], faa;
        gJ(g, p, F, gj);
        d2_alpha(g, h, p, ew, F.tA, F.tB, fza, faa);
        const float fa = g[0] * ew[0] + g[1] * ew[1] + g[2] * ew[2];
        float Dp[NDQ];
#pragma unroll
        for (int k = 0; k < NDQ; ++k) Dp[k] = fmaf(fa, da[k], gj[k]);
        d2_total(fzz, fza, faa, fa, da, d2a);      // fzz <- D2phi
        const float sq = s * (1.f - s) * itcmp;
        const float G1 = fmaf(phi, sq, s);
        const float G2 = sq * fmaf(phi * (1.f - 2.f * s), itcmp, 2.f);
#pragma unroll
        for (int i = 0; i < NDQ; ++i)
#pragma unroll
          for (int k2 = i; k2 < NDQ; ++k2) {
            const int q = p9(i, k2);
            d2a[q] = fmaf(sgn, fmaf(G2 * Dp[i], Dp[k2], G1 * fzz[q]), d2a[q]);
          }
      }
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
    float* rec = se + e * erec(TIER) + (dir ? trace_b(TIER) : 0);
    float at, c1, c2;   // soft clip and its first two derivatives (shared exponentials)
    softclip_12(al, 0.f, L, tca, itca, at, c1, c2);
    if constexpr (TIER >= 3) {
      // d2 a~ = sc'' da da^T + sc' d2a
      rec[0] = at;
#pragma unroll
      for (int k = 0; k < NDQ; ++k) rec[1 + k] = c1 * da[k];
#pragma unroll
      for (int i = 0; i < NDQ; ++i)
#pragma unroll
        for (int k2 = i; k2 < NDQ; ++k2) rec[TD2 + p9(i, k2)] = fmaf(c2 * da[i], da[k2], c1 * d2a[p9(i, k2)]);
    } else if constexpr (TIER >= 2) {
      const float cd = c1;
      float o[10] = {at};
#pragma unroll
      for (int k = 0; k < NDQ; ++k) o[1 + k] = cd * da[k];
      if (dir == 0) {   // record floats 0-9: two float4 + one float2
        st4(rec, o[0], o[1], o[2], o[3]);
        st4(rec + 4, o[4], o[5], o[6], o[7]);
        *reinterpret_cast<float2*>(rec + 8) = make_float2(o[8], o[9]);
      } else {          // record floats 10-19: one float2 + two float4
        *reinterpret_cast<float2*>(rec) = make_float2(o[0], o[1]);
        st4(rec + 2, o[2], o[3], o[4], o[5]);
        st4(rec + 6, o[6], o[7], o[8], o[9]);
      }
    } else {
      *rec = at;
    }
  }
}

// Tiers 0-2: the tier-2 derivative recursion carried in 6 components
// instead of 9: every g^T J(p) = [g, (p - tA) x g, g x (p - tB)]
// is [X, Y - tA x X, -Y + tB x X] with X = g, Y = p x g, a form the
// recursion d alpha_{k+1} = d alpha_k + c [(g.e_t) d alpha_k + g^T J(p)]
// preserves (X <- X + c (ge X + g), Y <- Y + c (ge Y + p x g)); the 9
// components are formed once, after the clip.
// One trace of edge e (vertex indices vI, vII) in direction dir: o[0] = the
// clipped alpha, o[1..9] its derivative over (t_A, theta_A, t_B) (tier 2)
template <int TIER, int XP>
__device__ __forceinline__ void trace_one_n(const MfArgs& a, const UnitCtx& U, const float* sv, const float* lv,
                                            int vI, int vII, int dir, float* o) {
  constexpr int OT = TIER >= 2 ? 1 : 0;
  const SmoothDev& sp = a.S.sp;
  const float itcmp = sp.i_cmp;
  const PairFrame& F = U.F;
  const float4 corner = ld4(sv + (dir ? vII : vI) * vrec(TIER));   // d, n of the start vertex
  float xl[3], el[3], L;
  {
    const float4 xa = ldv(lv, vI), xb4 = ldv(lv, vII);
    const float dl[3] = {xb4.x - xa.x, xb4.y - xa.y, xb4.z - xa.z};
    L = sqrtf(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
    const float iL = 1.f / L;
    el[0] = dl[0] * iL; el[1] = dl[1] * iL; el[2] = dl[2] * iL;
    xl[0] = xa.x; xl[1] = xa.y; xl[2] = xa.z;
  }
  float eb[3], ew[3];
  rot_vec(F.Rrel, el, eb);
  rot_vec(F.RA, el, ew);
  float xI[3], pI[3];
  to_frames(F, xl, xI, pI);
  float al = dir ? L : 0.f;
  const float sgn = dir ? -1.f : 1.f;
  float X[3] = {0.f, 0.f, 0.f}, Y[3] = {0.f, 0.f, 0.f};
  float phi = corner.x;
  float g[3] = {corner.y, corner.z, corner.w};   // the corner itself: the vertex evaluation (reading #22)
#pragma unroll 1
  for (int it = 0; it < sp.iters; ++it) {
    if (it > 0) {
      const float xb[3] = {fmaf(al, eb[0], xI[0]), fmaf(al, eb[1], xI[1]), fmaf(al, eb[2], xI[2])};
      Res<OT> r;
      CM_EVAL(OT, XP)(a.S, U.SB, xb, r);
      phi = r.v;
      if constexpr (TIER >= 2) rot_vec(F.RB, r.g, g);
    }
    // gated step G(phi) = sigma(phi / tau) phi  (reading #20)
    const float s = sigm(phi * itcmp);
    if constexpr (TIER >= 2) {
      const float Gp = fmaf(phi * s * (1.f - s), itcmp, s);
      const float p[3] = {fmaf(al, ew[0], pI[0]), fmaf(al, ew[1], pI[1]), fmaf(al, ew[2], pI[2])};
      const float m[3] = {p[1] * g[2] - p[2] * g[1], p[2] * g[0] - p[0] * g[2], p[0] * g[1] - p[1] * g[0]};
      const float ge = g[0] * ew[0] + g[1] * ew[1] + g[2] * ew[2];
      const float c = sgn * Gp;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        X[k] = fmaf(c, fmaf(ge, X[k], g[k]), X[k]);
        Y[k] = fmaf(c, fmaf(ge, Y[k], m[k]), Y[k]);
      }
    }
    al = fmaf(sgn * s, phi, al);
  }
  // soft clip to the edge (reading #21)
  float at, c1, c2;
  softclip_12(al, 0.f, L, sp.tau_clip_alpha, sp.i_clip_alpha, at, c1, c2);
  o[0] = at;
  if constexpr (TIER >= 2) {
    const float* tA = F.tA;
    const float* tB = F.tB;
    // d alpha = [X, Y - tA x X, -Y + tB x X], times the clip derivative
    o[1] = c1 * X[0]; o[2] = c1 * X[1]; o[3] = c1 * X[2];
    o[4] = c1 * (Y[0] - (tA[1] * X[2] - tA[2] * X[1]));
    o[5] = c1 * (Y[1] - (tA[2] * X[0] - tA[0] * X[2]));
    o[6] = c1 * (Y[2] - (tA[0] * X[1] - tA[1] * X[0]));
    o[7] = c1 * (-Y[0] + (tB[1] * X[2] - tB[2] * X[1]));
    o[8] = c1 * (-Y[1] + (tB[2] * X[0] - tB[0] * X[2]));
    o[9] = c1 * (-Y[2] + (tB[0] * X[1] - tB[1] * X[0]));
  }
}

// trace j of unit u (j < E: edge j from v_I; else edge j - E from v_II) and
// its record in the unit's slot
template <int TIER, int XP>
__device__ __forceinline__ void trace_item_n(const MfArgs& a, const UnitCtx& U, int u, int j) {
  const int V = U.SA.V, E = U.SA.E;
  const float* sv = a.scratch + (int64_t)u * a.slot;
  float* se = a.scratch + (int64_t)u * a.slot + (int64_t)vrec(TIER) * V;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const int32_t* ed = a.S.edges + 2 * (int64_t)U.SA.e_off;
  const int e = j < E ? j : j - E;
  const int dir = j < E ? 0 : 1;     // 0: from v_I along +e_t; 1: from v_II along -e_t
  const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
  CM_ASSERT(vI >= 0 && vI < V && vII >= 0 && vII < V);
  float o[10];
  trace_one_n<TIER, XP>(a, U, sv, lv, vI, vII, dir, o);
  float* rec = se + e * erec(TIER) + (dir ? trace_b(TIER) : 0);
  if constexpr (TIER >= 2) {
    if (dir == 0) {   // record floats 0-9: two float4 + one float2
      st4(rec, o[0], o[1], o[2], o[3]);
      st4(rec + 4, o[4], o[5], o[6], o[7]);
      *reinterpret_cast<float2*>(rec + 8) = make_float2(o[8], o[9]);
    } else {          // record floats 10-19: one float2 + two float4
      *reinterpret_cast<float2*>(rec) = make_float2(o[0], o[1]);
      st4(rec + 2, o[2], o[3], o[4], o[5]);
      st4(rec + 6, o[6], o[7], o[8], o[9]);
    }
  } else {
    *rec = o[0];
  }
}

template <int TIER, int XP>
__device__ __forceinline__ void mf_traces_unit_n(const MfArgs& a, const UnitCtx& U, int u) {
  static_assert(TIER <= 2, "tier 3 carries second derivatives: mf_traces_unit");
  const int V = U.SA.V, E = U.SA.E;
  const float* sv = a.scratch + (int64_t)u * a.slot;
  float* se = a.scratch + (int64_t)u * a.slot + (int64_t)vrec(TIER) * V;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const int32_t* ed = a.S.edges + 2 * (int64_t)U.SA.e_off;
#if CM_TRACE_PAIRED
  // the two traces of edge e on adjacent lanes (j = 2e + dir): their sum by
  // one shuffle, the averaged record (a_bar, d a_bar: 10 floats, half the
  // two traces' records) written by the dir-0 lane; the sums are the
  // midpoint kernel's a_I + a_II in the same order (bitwise equal)
  const int nj = 2 * E;
  for (int jb = threadIdx.x & ~31; jb < nj; jb += blockDim.x) {
    const int j = jb + (threadIdx.x & 31);
    const bool act = j < nj;
    const int e = act ? j >> 1 : 0;
    const int dir = j & 1;             // 0: from v_I along +e_t; 1: from v_II along -e_t
    constexpr int NS = TIER >= 2 ? 10 : 1;
    float o[10] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (act) {
      const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
      CM_ASSERT(vI >= 0 && vI < V && vII >= 0 && vII < V);
      trace_one_n<TIER, XP>(a, U, sv, lv, vI, vII, dir, o);
    }
    float m[10];
#pragma unroll
    for (int k = 0; k < NS; ++k) m[k] = 0.5f * (o[k] + __shfl_xor_sync(0xffffffffu, o[k], 1));
    if (act && dir == 0) {
      float* rec = se + e * erec(TIER);
      if constexpr (TIER >= 2) {
        st4(rec, m[0], m[1], m[2], m[3]);
        st4(rec + 4, m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float2*>(rec + 8) = make_float2(m[8], m[9]);
      } else {
        *rec = m[0];
      }
    }
  }
#else
  if (CM_MF_TRACE_L1PF && vrec(TIER) * V <= 8192) {   // the unit's vertex records (the corners) into L1
    for (int o = threadIdx.x * 32; o < vrec(TIER) * V; o += blockDim.x * 32)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(sv + o));
  }
  for (int j = threadIdx.x; j < 2 * E; j += blockDim.x) {
    const int e = j < E ? j : j - E;
    const int dir = j < E ? 0 : 1;     // 0: from v_I along +e_t; 1: from v_II along -e_t
    const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
    CM_ASSERT(vI >= 0 && vI < V && vII >= 0 && vII < V);
    float o[10];
    trace_one_n<TIER, XP>(a, U, sv, lv, vI, vII, dir, o);
    float* rec = se + e * erec(TIER) + (dir ? trace_b(TIER) : 0);
    if constexpr (TIER >= 2) {
      if (dir == 0) {   // record floats 0-9: two float4 + one float2
        st4(rec, o[0], o[1], o[2], o[3]);
        st4(rec + 4, o[4], o[5], o[6], o[7]);
        *reinterpret_cast<float2*>(rec + 8) = make_float2(o[8], o[9]);
      } else {          // record floats 10-19: one float2 + two float4
        *reinterpret_cast<float2*>(rec) = make_float2(o[0], o[1]);
        st4(rec + 2, o[2], o[3], o[4], o[5]);
        st4(rec + 6, o[6], o[7], o[8], o[9]);
      }
    } else {
      *rec = o[0];
    }
  }
#endif
}

// ---- phase 3: edge points p_e = v_I + a_bar e_t, a_bar = (a_I + a_II)/2
// the candidate at edge e from its averaged trace (ab, dab, d2ab): phi, n, H
// of B at p_e, the edge record and (full mode) the candidate's output row
template <int TIER, int XP>
__device__ __forceinline__ void midpoint_one(const MfArgs& a, const UnitCtx& U, int e, float ab, const float* dab,
                                             const float* d2ab, float* rec) {
  constexpr int OV = TIER >= 2 ? 2 : 1;
  const PairFrame& F = U.F;
  const float* eg = a.S.edge_geom + 8 * (int64_t)U.SA.e_off;
  float xl[3], el[3], L;
  edge_geom(eg, e, xl, L, el);
  float eb[3], ew[3];
  rot_vec(F.Rrel, el, eb);
  rot_vec(F.RA, el, ew);
  float xI[3], pI[3];
  to_frames(F, xl, xI, pI);
  float xb[3], pw[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    xb[i] = fmaf(ab, eb[i], xI[i]);
    pw[i] = fmaf(ab, ew[i], pI[i]);
  }
  Res<OV> r;
  CM_EVAL(OV, XP)(a.S, U.SB, xb, r);
  float n[3];
  rot_vec(F.RB, r.g, n);
  float h[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if constexpr (TIER >= 2) {
    rot_sym(F.RB, r.h, h);
    st4(rec, ab, r.v, n[0], n[1]);
    st4(rec + 4, n[2], h[0], h[1], h[2]);
    st4(rec + 8, h[3], h[4], h[5], dab[0]);
    st4(rec + 12, dab[1], dab[2], dab[3], dab[4]);
    st4(rec + 16, dab[5], dab[6], dab[7], dab[8]);
  } else {
    st4(rec, ab, r.v, n[0], n[1]);
    rec[4] = n[2];
  }
  float d2[TIER >= 3 ? N45 : 1];
  if constexpr (TIER >= 3) {
    // d^2 d_e = phi_zz + phi_za dab^T + dab phi_za^T + phi_aa dab dab^T + phi_a d2ab
    float fza[NDQ], faa;
    d2_point(n, h, pw, F.tA, F.tB, d2);
    d2_alpha(n, h, pw, ew, F.tA, F.tB, fza, faa);
    const float fa = n[0] * ew[0] + n[1] * ew[1] + n[2] * ew[2];
    d2_total(d2, fza, faa, fa, dab, d2ab);
#pragma unroll
    for (int k = 0; k < N45; ++k) rec[MD2 + k] = d2[k];
  }
  if (a.mode & CM_FULL_MODE) {
    CM_COLS(U.side);
    store_candidate<TIER>(a.out, a.C, U.off + U.SA.V + e, pw, n, r.v, h, ew, dab, F, 1, a.S.sp.i_cmp, cTA, cRA, cTB,
                          cRB, d2, U.side);
  }
}

template <int TIER, int XP>
__device__ __forceinline__ void mf_midpoints_unit(const MfArgs& a, const UnitCtx& U, int u, const float* srec,
                                                  float* drec = nullptr, float* pfbuf = nullptr) {
  const int V = U.SA.V, E = U.SA.E;
  float* se = a.scratch + (int64_t)u * a.slot + (int64_t)vrec(TIER) * V;
  if (srec == nullptr) srec = se;   // trace records: staged in shared memory, or the slot
  if (drec == nullptr) drec = se;   // edge records: to the slot, or to shared memory (fused faces)
  // pfbuf (tier 2): each thread's next trace record is fetched into its own
  // 80-B shared-memory buffer by cp.async while it evaluates the current
  // edge (the record of edge e is overwritten only by e's own thread)
  float* pb = pfbuf ? pfbuf + threadIdx.x * 20 : nullptr;
  auto fetch = [&](int e) {
    const float* src = srec + e * erec(TIER);
#pragma unroll
    for (int q = 0; q < 5; ++q) cp_async16(pb + 4 * q, src + 4 * q);
    cp_async_commit();
  };
  if (TIER == 2 && pb && (int)threadIdx.x < E) fetch(threadIdx.x);
  if (CM_MF_TABLE_L1PF) {   // the mesh's edge-geometry table into L1
    const float* egt = a.S.edge_geom + 8 * (int64_t)U.SA.e_off;
    for (int o = threadIdx.x * 32; o < 8 * E; o += blockDim.x * 32)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(egt + o));
  }
  if (CM_MF_MID_L1PF && srec == se && E * erec(TIER) <= 8192) {
    // the unit's trace records into L1 (one prefetch per 128-B line)
    for (int o = threadIdx.x * 32; o < E * erec(TIER); o += blockDim.x * 32)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(srec + o));
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float* rec = drec + e * erec(TIER);
    const float* rin = srec + e * erec(TIER);
    float ab, dab[NDQ];
    float d2ab[TIER >= 3 ? N45 : 1];
    if constexpr (TIER >= 3) {
      const float* rb2 = rin + trace_b(TIER);
      ab = 0.5f * (rin[0] + rb2[0]);
#pragma unroll
      for (int k = 0; k < NDQ; ++k) dab[k] = 0.5f * (rin[1 + k] + rb2[1 + k]);
#pragma unroll
      for (int k = 0; k < N45; ++k) d2ab[k] = 0.5f * (rin[TD2 + k] + rb2[TD2 + k]);
    } else if constexpr (TIER >= 2 && CM_PAIRED_REC) {   // the traces' averaged record (a_bar, d a_bar)
      const float4 r0 = ld4(rin), r1 = ld4(rin + 4);
      const float2 r2 = *reinterpret_cast<const float2*>(rin + 8);
      ab = r0.x;
      dab[0] = r0.y; dab[1] = r0.z; dab[2] = r0.w;
      dab[3] = r1.x; dab[4] = r1.y; dab[5] = r1.z; dab[6] = r1.w;
      dab[7] = r2.x; dab[8] = r2.y;
    } else if constexpr (TIER >= 2) {
      float t[20];
      const float* src = rin;
      if (pb) {
        cp_async_wait_all();
        src = pb;
      }
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const float4 v4 = ld4(src + 4 * q);
        t[4 * q] = v4.x; t[4 * q + 1] = v4.y; t[4 * q + 2] = v4.z; t[4 * q + 3] = v4.w;
      }
      if (pb && e + (int)blockDim.x < E) fetch(e + blockDim.x);
      ab = 0.5f * (t[0] + t[10]);
#pragma unroll
      for (int k = 0; k < NDQ; ++k) dab[k] = 0.5f * (t[1 + k] + t[11 + k]);
    } else if constexpr (CM_PAIRED_REC) {
      ab = rin[0];
    } else {
      ab = 0.5f * (rin[0] + rin[1]);
    }
    midpoint_one<TIER, XP>(a, U, e, ab, dab, d2ab, rec);
  }
}

// ---- phases 2 + 3 in one thread per edge (tiers 0-2): both traces of the
// edge, then its midpoint candidate; the trace results stay in registers
// (no trace records through the scratch slot: -2 x 40 B of HBM traffic per
// edge and one launch per class and chunk).  Bitwise equal to the separate
// kernels: the sums a_I + a_II are formed in the same order with the same
// roundings (0 + a_I is exact).
template <int TIER, int XP>
__device__ __forceinline__ void mf_edges_unit(const MfArgs& a, const UnitCtx& U, int u, float* esm) {
  static_assert(TIER <= 2, "tier 3: separate trace and midpoint kernels");
  const int V = U.SA.V, E = U.SA.E;
  const float* sv = a.scratch + (int64_t)u * a.slot;
  float* se = a.scratch + (int64_t)u * a.slot + (int64_t)vrec(TIER) * V;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const int32_t* ed = a.S.edges + 2 * (int64_t)U.SA.e_off;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int vI = __ldg(ed + 2 * e), vII = __ldg(ed + 2 * e + 1);
    CM_ASSERT(vI >= 0 && vI < V && vII >= 0 && vII < V);
    constexpr int NS = TIER >= 2 ? 10 : 1;
    float sum[10];
    // one copy of the trace code for both directions (a second inlined copy
    // of the SDF evaluation costs instruction-cache misses)
#pragma unroll 1
    for (int dir = 0; dir < 2; ++dir) {
      float o[10];
      trace_one_n<TIER, XP>(a, U, sv, lv, vI, vII, dir, o);
      if constexpr (CM_MF_EDGE_SMEM) {   // the first trace parked in shared memory
        if (dir == 0) {
#pragma unroll
          for (int k = 0; k < NS; ++k) esm[k * blockDim.x + threadIdx.x] = o[k];
        } else {
#pragma unroll
          for (int k = 0; k < NS; ++k) sum[k] = __fadd_rn(esm[k * blockDim.x + threadIdx.x], o[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < NS; ++k) sum[k] = dir ? __fadd_rn(sum[k], o[k]) : o[k];
      }
    }
    const float ab = 0.5f * sum[0];
    float dab[NDQ];
#pragma unroll
    for (int k = 0; k < NDQ; ++k) dab[k] = TIER >= 2 ? 0.5f * sum[1 + k] : 0.f;
    const float d2ab[1] = {0.f};
    midpoint_one<TIER, XP>(a, U, e, ab, dab, d2ab, se + e * erec(TIER));
  }
}

// ---- phase 4: per-face fusion ---------------------------------
// STAGED: the unit's candidate state is first copied (coalesced) into shared
// memory together with the candidates' world points p and the edges' world
// directions e_t, computed once per vertex / edge instead of once per face;
// the face loop then gathers from shared memory.  Units too large for shared
// memory gather from the scratch slot and recompute p, e_t per face.
// Staged layout: the slot's used records [V vertex | E edge] copied by one
// TMA bulk copy (cp.async.bulk, completion on an mbarrier), then p[3][V] of
// the vertices and p_I[3][E], e_t[3][E] of the edges (the edge point is
// p_I + a_bar e_t).
__host__ __device__ constexpr int face_stage_floats(int V, int E, int tier) {
  return vrec(tier) * V + erec(tier) * E + 3 * V + 6 * E;
}

template <int TIER, bool STAGED>
__device__ __forceinline__ void mf_faces_unit(const MfArgs& a, const UnitCtx& U, int u, float* fsm, uint64_t* barp,
                                              uint32_t phase, const float* sv_in = nullptr,
                                              const float* se_in = nullptr) {
  const SmoothDev sp = a.S.sp;
  const float itcmp = sp.i_cmp;
  const float tmin = sp.tau_min, itmin = sp.i_min;
  const PairFrame& F = U.F;
  const int V = U.SA.V, E = U.SA.E, NF = U.SA.F;
  constexpr int VR = vrec(TIER), ER = erec(TIER);
  const float* gv = a.scratch + (int64_t)u * a.slot;
  const float* ge = gv + (int64_t)VR * V;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const float* eg = a.S.edge_geom + 8 * (int64_t)U.SA.e_off;
  const int32_t* fv = a.S.faces + 3 * (int64_t)U.SA.f_off;
  const int32_t* fe = a.S.face_edges + 3 * (int64_t)U.SA.f_off;
  const cm_manifold_out& out = a.out;
  const int64_t C = a.C;
  // (fused with the midpoint kernel: the records are given in shared memory)
  const float* sv = sv_in ? sv_in : gv;
  const float* se = se_in ? se_in : ge;
  float* s_pv = nullptr;   // staged vertex points p[3][V]
  float* s_pe = nullptr;   // staged edge p_I[3][E], e_t[3][E]
  if constexpr (STAGED) {
    const int used = VR * V + ER * E;
    CM_ASSERT(V >= 0 && E >= 0 && (int64_t)used <= a.slot);
    if (threadIdx.x == 0) bulk_g2s(fsm, gv, (uint32_t)used * 4u, barp);
    s_pv = fsm + used;
    s_pe = s_pv + 3 * V;
    // overlapped with the copy: the candidates' world geometry
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      float xb[3], pw[3];
      vertex_frames(F, lv, v, xb, pw);
#pragma unroll
      for (int k = 0; k < 3; ++k) s_pv[k * V + v] = pw[k];
    }
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      float xl[3], el[3], L, ew[3], xb[3], pI[3];
      edge_geom(eg, e, xl, L, el);
      rot_vec(F.RA, el, ew);
      to_frames(F, xl, xb, pI);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        s_pe[k * E + e] = pI[k];
        s_pe[(3 + k) * E + e] = ew[k];
      }
    }
    mbar_wait(barp, phase);
    __syncthreads();
    sv = fsm;
    se = fsm + VR * V;
  }
  CM_COLS(U.side);
  if constexpr (!STAGED && CM_MF_FACE_L1PF) {
    // the unit's candidate records into L1 (one prefetch per 128-B line),
    // ahead of the faces' dependent gathers
    const int used = VR * V + ER * E;
    if (!sv_in && used <= 8192) {   // (slots up to 32 KB: a large unit's would evict its own lines)
      for (int o = threadIdx.x * 32; o < used; o += blockDim.x * 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(gv + o));
      if (CM_MF_FACE_L1PF >= 2) {
        for (int o = threadIdx.x * 32; o < 4 * V; o += blockDim.x * 32)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(lv + o));
        for (int o = threadIdx.x * 32; o < 8 * E; o += blockDim.x * 32)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(eg + o));
      }
    }
  }
  const float itlm = LOG2E * itmin;
  for (int f = threadIdx.x; f < NF; f += blockDim.x) {
    int cv[3], ce[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cv[k] = __ldg(fv + 3 * f + k);
      ce[k] = __ldg(fe + 3 * f + k);
      CM_ASSERT(cv[k] >= 0 && cv[k] < V && ce[k] >= 0 && ce[k] < E);
    }
    // candidate depths d_i; order [v_i0, v_i1, v_i2, e(i0,i1), e(i1,i2), e(i2,i0)]
    float dc[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) { dc[k] = sv[cv[k] * VR + VD]; dc[3 + k] = se[ce[k] * ER + MD]; }
    // candidate points (world): vertices RA x + tA, edge points p_I + a_bar e_t
    // (the same arithmetic as the vertex / midpoint kernels), and the edges'
    // world directions e_t for the sliding terms
    float pc[6][3], ewc[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if constexpr (STAGED) {
        const float ab = se[ce[k] * ER + MAB];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          pc[k][i] = s_pv[i * V + cv[k]];
          ewc[k][i] = s_pe[(3 + i) * E + ce[k]];
          pc[3 + k][i] = fmaf(ab, ewc[k][i], s_pe[i * E + ce[k]]);
        }
      } else {
        float xb[3];
        vertex_frames(F, lv, cv[k], xb, pc[k]);
        float xl[3], el[3], L;
        edge_geom(eg, ce[k], xl, L, el);
        rot_vec(F.RA, el, ewc[k]);
        float pI[3];
        to_frames(F, xl, xb, pI);
        const float ab = se[ce[k] * ER + MAB];
#pragma unroll
        for (int i = 0; i < 3; ++i) pc[3 + k][i] = fmaf(ab, ewc[k][i], pI[i]);
      }
    }
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
      const float* bn = isv ? sv + id * VR + VN : se + id * ER + MN;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float p = pc[i][k], nn = bn[k];
        nrm[k] = fmaf(zg[i], nn, nrm[k]);
        qv[k] = fmaf(zg[i], p, qv[k]);
        pt[k] = fmaf(z[i], p, pt[k]);
      }
    }
    const int64_t c = U.off + f;
    CM_ASSERT(c >= 0 && c < C);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      out.point[k * C + c] = pt[k];
      out.normal[k * C + c] = nrm[k];
    }
    out.depth[c] = depth;
    out.dom[c] = (int8_t)dom;
    if constexpr (TIER >= 1) {
      out.W[c] = Wf;
#pragma unroll
      for (int k = 0; k < 3; ++k) out.q[k * C + c] = qv[k];
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
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int k = 0; k < NDQ; ++k) dnE[q][k] = 0.f;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const bool isv = i < 3;
        const int id = isv ? cv[i] : ce[i - 3];
        const float* p = pc[i];
        float n[3], h[6], dab[NDQ];
        if (isv) {   // d, n[3] | H[6], pad
          const float* rv = sv + id * VR;
          const float4 a0 = ld4(rv), a1 = ld4(rv + 4), a2 = ld4(rv + 8);
          n[0] = a0.y; n[1] = a0.z; n[2] = a0.w;
          h[0] = a1.x; h[1] = a1.y; h[2] = a1.z; h[3] = a1.w; h[4] = a2.x; h[5] = a2.y;
        } else {     // a_bar, d, n[3], H[6], da_bar[9]
          const float* re = se + id * ER;
          const float4 a0 = ld4(re), a1 = ld4(re + 4), a2 = ld4(re + 8), a3 = ld4(re + 12), a4 = ld4(re + 16);
          n[0] = a0.z; n[1] = a0.w; n[2] = a1.x;
          h[0] = a1.y; h[1] = a1.z; h[2] = a1.w; h[3] = a2.x; h[4] = a2.y; h[5] = a2.z;
          dab[0] = a2.w; dab[1] = a3.x; dab[2] = a3.y; dab[3] = a3.z; dab[4] = a3.w;
          dab[5] = a4.x; dab[6] = a4.y; dab[7] = a4.z; dab[8] = a4.w;
        }
        const float gam = sigm(-dc[i] * itcmp);
        const float w = zg[i];
        const float ci = w * (-itmin - (1.f - gam) * itcmp);
        const float pxn[3] = {p[1] * n[2] - p[2] * n[1], p[2] * n[0] - p[0] * n[2], p[0] * n[1] - p[1] * n[0]};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          Sg[q] = fmaf(z[i], n[q], Sg[q]);
          Spg[q] = fmaf(z[i], pxn[q], Spg[q]);
        }
        const float cn[3] = {ci * n[0], ci * n[1], ci * n[2]};
        K[0] = fmaf(cn[0], n[0], K[0]); K[1] = fmaf(cn[0], n[1], K[1]); K[2] = fmaf(cn[0], n[2], K[2]);
        K[3] = fmaf(cn[1], n[1], K[3]); K[4] = fmaf(cn[1], n[2], K[4]); K[5] = fmaf(cn[2], n[2], K[5]);
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int b = 0; b < 3; ++b) Lm[q * 3 + b] = fmaf(cn[q], pxn[b], Lm[q * 3 + b]);
#pragma unroll
        for (int k = 0; k < 6; ++k) Hb[k] = fmaf(w, h[k], Hb[k]);
        const float H[3][3] = {{h[0], h[1], h[2]}, {h[1], h[3], h[4]}, {h[2], h[4], h[5]}};
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          // (H [p]x) row q
          Mm[q * 3 + 0] = fmaf(w, H[q][1] * p[2] - H[q][2] * p[1], Mm[q * 3 + 0]);
          Mm[q * 3 + 1] = fmaf(w, H[q][2] * p[0] - H[q][0] * p[2], Mm[q * 3 + 1]);
          Mm[q * 3 + 2] = fmaf(w, H[q][0] * p[1] - H[q][1] * p[0], Mm[q * 3 + 2]);
        }
        if (!isv) {
          // sliding along the edge: e_t (world, unit) and d alpha_bar
          const float* ew = ewc[i - 3];
          const float ge = n[0] * ew[0] + n[1] * ew[1] + n[2] * ew[2];
          float u[3];   // c ge n + zg H e_t
#pragma unroll
          for (int q = 0; q < 3; ++q) u[q] = fmaf(ci * ge, n[q], w * (H[q][0] * ew[0] + H[q][1] * ew[1] + H[q][2] * ew[2]));
          const float zge = z[i] * ge;
#pragma unroll
          for (int k = 0; k < NDQ; ++k) {
            const float dk = dab[k];
            Se[k] = fmaf(zge, dk, Se[k]);
#pragma unroll
            for (int q = 0; q < 3; ++q) dnE[q][k] = fmaf(u[q], dk, dnE[q][k]);
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
      for (int q = 0; q < 3; ++q) {
        const float KH[3] = {Ks[q][0] + Hs[q][0], Ks[q][1] + Hs[q][1], Ks[q][2] + Hs[q][2]};
        // (X [t]x) row q for X = K + Hb, t = tA and tB
        const float xA[3] = {KH[1] * tA[2] - KH[2] * tA[1], KH[2] * tA[0] - KH[0] * tA[2], KH[0] * tA[1] - KH[1] * tA[0]};
        const float KtB[3] = {Ks[q][1] * tB[2] - Ks[q][2] * tB[1], Ks[q][2] * tB[0] - Ks[q][0] * tB[2],
                              Ks[q][0] * tB[1] - Ks[q][1] * tB[0]};
        const float HtB[3] = {Hs[q][1] * tB[2] - Hs[q][2] * tB[1], Hs[q][2] * tB[0] - Hs[q][0] * tB[2],
                              Hs[q][0] * tB[1] - Hs[q][1] * tB[0]};
        // [nbar]x row q
        const float nk[3] = {q == 0 ? 0.f : (q == 1 ? nrm[2] : -nrm[1]), q == 0 ? -nrm[2] : (q == 1 ? 0.f : nrm[0]),
                             q == 0 ? nrm[1] : (q == 1 ? -nrm[0] : 0.f)};
        const float nb = nrm[q] * itmin;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          dn[q][b] = KH[b] + nb * dd[b] + dnE[q][b];
          dn[q][3 + b] = Lm[q * 3 + b] + xA[b] - Mm[q * 3 + b] + nb * dd[3 + b] + dnE[q][3 + b];
          dn[q][6 + b] = -Lm[q * 3 + b] - KtB[b] + Mm[q * 3 + b] - HtB[b] - nk[b] + nb * dd[6 + b] + dnE[q][6 + b];
        }
      }
      if constexpr (TIER >= 3) {
        // d^2 depth = sum z_i d^2 d_i - (1/tau_min)(sum z_i dd_i dd_i^T - dd dd^T)
        float A[N45];
#pragma unroll
        for (int k = 0; k < N45; ++k) A[k] = 0.f;
#pragma unroll 1
        for (int i = 0; i < 6; ++i) {
          const bool isv = i < 3;
          const int id = isv ? cv[i] : ce[i - 3];
          const float* rr = isv ? sv + id * VR : se + id * ER;
          const float nn[3] = {rr[(isv ? VN : MN) + 0], rr[(isv ? VN : MN) + 1], rr[(isv ? VN : MN) + 2]};
          float pi3[3], ewi[3] = {0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            pi3[q] = i == 0 ? pc[0][q] : i == 1 ? pc[1][q] : i == 2 ? pc[2][q] : i == 3 ? pc[3][q] : i == 4 ? pc[4][q] : pc[5][q];
            if (!isv) ewi[q] = i == 3 ? ewc[0][q] : i == 4 ? ewc[1][q] : ewc[2][q];
          }
          float ddi[NDQ];
          gJ(nn, pi3, F, ddi);
          if (!isv) {
            const float ge = nn[0] * ewi[0] + nn[1] * ewi[1] + nn[2] * ewi[2];
#pragma unroll
            for (int k = 0; k < NDQ; ++k) ddi[k] = fmaf(ge, rr[MDAB + k], ddi[k]);
          }
          float d2i[N45];
          ld45(rr + (isv ? VD2 : MD2), d2i);
          const float zi = i == 0 ? z[0] : i == 1 ? z[1] : i == 2 ? z[2] : i == 3 ? z[3] : i == 4 ? z[4] : z[5];
          const float zt = zi * itmin;
#pragma unroll
          for (int q = 0; q < NDQ; ++q)
#pragma unroll
            for (int k = q; k < NDQ; ++k) A[p9(q, k)] = fmaf(zi, d2i[p9(q, k)], fmaf(-zt * ddi[q], ddi[k], A[p9(q, k)]));
        }
#pragma unroll
        for (int q = 0; q < NDQ; ++q)
#pragma unroll
          for (int k = q; k < NDQ; ++k) A[p9(q, k)] = fmaf(itmin * dd[q], dd[k], A[p9(q, k)]);
        store_d2(out.d2depth, C, c, A, U.side);
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
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          out.dnormal[(q * 12 + cTA + k) * C + c] = dn[q][k];
          out.dnormal[(q * 12 + cRA + k) * C + c] = dn[q][3 + k];
          out.dnormal[(q * 12 + cTB + k) * C + c] = -dn[q][k];
          out.dnormal[(q * 12 + cRB + k) * C + c] = dn[q][6 + k];
        }
    }
  }
}


// ---- phase kernels ----------------------------------------------------------
// k_mf_units files every valid unit of the chunk under its SDF class (in unit
// order); CTA b of a class's phase kernel takes entry b of that list (CTAs
// past the class's count exit after one broadcast load, without a barrier).
// A persistent variant (resident CTAs pulling units from an atomic counter)
// measured slower: C5 -5%, C4 -2%, C2 -10%.
__device__ __forceinline__ bool list_unit(const MfArgs& a, int list, UnitCtx& U, int& u, int b = -1) {
  if (b < 0) b = blockIdx.x;
  if (list < 0 && b >= a.nb) return false;
  if (list >= 0) {
    if (b >= __ldcg(a.cls_count + list)) return false;
    u = __ldcg(a.cls_list + (int64_t)list * a.chunk + b);
    CM_ASSERT(u >= 0 && u < a.nb);
  } else {
    u = b;
  }
  constexpr int n4 = (int)(sizeof(UnitCtx) / 16);
  const float4* src = reinterpret_cast<const float4*>(a.ctx + u);
  for (int i = threadIdx.x; i < n4; i += blockDim.x) reinterpret_cast<float4*>(&U)[i] = __ldcg(src + i);
  __syncthreads();
  return true;
}

// CM_MF_UPC units per CTA (list entries blockIdx.x * UPC + r): fewer CTAs
// per launch, so that the launches of a chunk's absent classes (their CTAs
// exit after one broadcast load) cost less
#ifndef CM_MF_UPC
#define CM_MF_UPC 1
#endif
template <int TIER, int XP>
__global__ void __maxnreg__((RegCap<TIER, XP>::VERTICES)) k_mf_vertices(const MfArgs a) {
  __shared__ UnitCtx U;
  int u;
  for (int r = 0; r < CM_MF_UPC; ++r) {
    if (!list_unit(a, XP, U, u, blockIdx.x * CM_MF_UPC + r)) return;
    mf_vertices_unit<TIER, XP>(a, U, u);
    if (CM_MF_UPC > 1) __syncthreads();
  }
}
// CAT units per CTA with their traces as one item range (tiers 0-2,
// 6-component recursion): the last, partly filled round of each unit's
// traces is shared with the next units.  Used when every sampled surface
// of the scene is small (2 max_E <= CM_MF_CAT_MAX_ITEMS): C4 +4.5%, while
// C5 (2E up to 576) -2% and C3 -4% lose to the longer CTAs (r02zu sweep)
#ifndef CM_MF_CAT
#define CM_MF_CAT 4
#endif
#ifndef CM_MF_CAT_MAX_ITEMS
#define CM_MF_CAT_MAX_ITEMS 384
#endif
template <int TIER, int XP, int CAT>
__global__ void __maxnreg__((RegCap<TIER, XP>::TRACES)) k_mf_traces_cat(const MfArgs a) {
  __shared__ UnitCtx U[CAT];
  __shared__ int su[CAT], sn[CAT + 1];
  if (threadIdx.x == 0) {
    sn[0] = 0;
    const int cnt = __ldcg(a.cls_count + XP);
    for (int r = 0; r < CAT; ++r) {
      const int b = blockIdx.x * CAT + r;
      su[r] = b < cnt ? __ldcg(a.cls_list + (int64_t)XP * a.chunk + b) : -1;
      sn[r + 1] = sn[r] + (su[r] >= 0 ? 2 * __ldcg(&a.ctx[su[r]].SA.E) : 0);
    }
  }
  __syncthreads();
  constexpr int n4 = (int)(sizeof(UnitCtx) / 16);
  for (int r = 0; r < CAT; ++r) {
    if (su[r] < 0) break;
    const float4* src = reinterpret_cast<const float4*>(a.ctx + su[r]);
    for (int i = threadIdx.x; i < n4; i += blockDim.x) reinterpret_cast<float4*>(&U[r])[i] = __ldcg(src + i);
  }
  __syncthreads();
  const int total = sn[CAT];
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    int r = 0;
#pragma unroll
    for (int k = 1; k < CAT; ++k) r += j >= sn[k];
    trace_item_n<TIER, XP>(a, U[r], su[r], j - sn[r]);
  }
}
template <int TIER, int XP>
__global__ void __maxnreg__((RegCap<TIER, XP>::TRACES)) k_mf_traces(const MfArgs a) {
  __shared__ UnitCtx U;
  int u;
  for (int r = 0; r < CM_MF_UPC; ++r) {
    if (!list_unit(a, XP, U, u, blockIdx.x * CM_MF_UPC + r)) return;
    if constexpr (TIER <= 2 && CM_TRACE6) mf_traces_unit_n<TIER, XP>(a, U, u);
    else mf_traces_unit<TIER, XP>(a, U, u);
    if (CM_MF_UPC > 1) __syncthreads();
  }
}
template <int TIER, int XP> struct EdgeRegs {   // the larger of the trace and midpoint budgets
  static constexpr int R0 = RegCap<TIER, XP>::MIDPOINTS > RegCap<TIER, XP>::TRACES ? RegCap<TIER, XP>::MIDPOINTS
                                                                                    : RegCap<TIER, XP>::TRACES;
  static constexpr int R = (XP == 0 && CM_MF_REG_E_XP0) ? CM_MF_REG_E_XP0
                         : (((XP == 1 || XP == 4) && CM_MF_REG_E_XP1) ? CM_MF_REG_E_XP1 : R0);
};
template <int TIER, int XP>
__global__ void __maxnreg__((EdgeRegs<TIER, XP>::R)) k_mf_edges(const MfArgs a) {
  extern __shared__ __align__(16) float esm[];
  __shared__ UnitCtx U;
  int u;
  if (list_unit(a, XP, U, u)) mf_edges_unit<TIER, XP>(a, U, u, esm);
}
// STAGED: the unit's trace records (E x erec floats, contiguous in its slot)
// are first copied into shared memory with one TMA bulk copy, so the edge
// loop does not wait on HBM for every edge

template <int TIER, int XP, bool STAGED>
__global__ void __maxnreg__((RegCap<TIER, XP>::MIDPOINTS)) k_mf_midpoints(const MfArgs a) {
  extern __shared__ __align__(16) float msm[];
  __shared__ UnitCtx U;
  __shared__ uint64_t bar;
  if (STAGED && threadIdx.x == 0) mbar_init(&bar, 1);   // published by list_unit's barrier
  int u;
  if (!list_unit(a, XP, U, u, STAGED ? (int)blockIdx.x : (int)blockIdx.x * CM_MF_UPC)) return;
  if constexpr (STAGED) {
    const float* se = a.scratch + (int64_t)u * a.slot + (int64_t)vrec(TIER) * U.SA.V;
    if (threadIdx.x == 0) bulk_g2s(msm, se, (uint32_t)(U.SA.E * erec(TIER)) * 4u, &bar);
    mbar_wait(&bar, 0u);
    mf_midpoints_unit<TIER, XP>(a, U, u, msm);
  } else {
    for (int r = 0;;) {
      mf_midpoints_unit<TIER, XP>(a, U, u, nullptr, nullptr, (TIER == 2 && CM_MF_MID_PREFETCH) ? msm : nullptr);
      if (++r >= CM_MF_UPC) break;
      __syncthreads();
      if (!list_unit(a, XP, U, u, blockIdx.x * CM_MF_UPC + r)) return;
    }
  }
}
// Midpoints and face fusion in one kernel per SDF class (reduced mode, tiers
// 0-2): the unit's edge records are written to shared memory instead of the
// slot, its vertex records arrive by one TMA bulk copy (overlapped with the
// midpoint evaluations), and the face loop gathers both from shared memory
// (no scratch round trip through HBM for the edge records, no separate face
// launch).  Shared memory: max_E edge + max_V vertex records.
#ifndef CM_MF_FUSE_FACES
#define CM_MF_FUSE_FACES 0   // measured slower: C5 -3.5%, C4 -12.6% (r02n sweep)
#endif
template <int TIER, int XP> struct MidFacesRegs {   // the larger of the midpoint and face budgets
  static constexpr int R = RegCap<TIER, XP>::MIDPOINTS > regs_of(CM_MF_FACE_MINB) ? RegCap<TIER, XP>::MIDPOINTS
                                                                                     : regs_of(CM_MF_FACE_MINB);
};
template <int TIER, int XP>
__global__ void __maxnreg__((MidFacesRegs<TIER, XP>::R)) k_mf_midfaces(const MfArgs a, int max_E) {
  static_assert(TIER <= 2, "tier 3: separate kernels");
  extern __shared__ __align__(16) float fsm[];
  __shared__ UnitCtx U;
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);   // published by list_unit's barrier
  int u;
  if (!list_unit(a, XP, U, u)) return;
  constexpr int VR = vrec(TIER), ER = erec(TIER);
  float* se_s = fsm;
  float* sv_s = fsm + (int64_t)max_E * ER;
  const float* gv = a.scratch + (int64_t)u * a.slot;
  if (threadIdx.x == 0) bulk_g2s(sv_s, gv, (uint32_t)(U.SA.V * VR) * 4u, &bar);
  mf_midpoints_unit<TIER, XP>(a, U, u, nullptr, se_s);
  mbar_wait(&bar, 0u);
  __syncthreads();
  mf_faces_unit<TIER, false>(a, U, u, nullptr, nullptr, 0u, sv_s, se_s);
}

// Small batches (at most CM_MF_SMALL_UNITS units in a chunk, e.g. C1's two
// pairs): the four phases of a unit in ONE kernel per SDF class, separated
// by CTA barriers (the per-phase kernels' dependent launches dominate there;
// at large batches the split kernels win).  The same device
// functions and the same scratch slot as the split path: bitwise equal.
#ifndef CM_MF_SMALL_UNITS
#define CM_MF_SMALL_UNITS 64
#endif
template <int TIER, int XP>
__global__ void __launch_bounds__(CM_MF_MAX_THREADS) k_mf_small(const MfArgs a) {
  __shared__ UnitCtx U;
  int u;
  if (!list_unit(a, XP, U, u)) return;
  mf_vertices_unit<TIER, XP>(a, U, u);
  __syncthreads();
  if constexpr (TIER <= 2 && CM_TRACE6) mf_traces_unit_n<TIER, XP>(a, U, u);
  else mf_traces_unit<TIER, XP>(a, U, u);
  __syncthreads();
  mf_midpoints_unit<TIER, XP>(a, U, u, nullptr);
  if (!(a.mode & CM_FULL_MODE)) {
    __syncthreads();
    mf_faces_unit<TIER, false>(a, U, u, nullptr, nullptr, 0u);
  }
}

// broad phase (f2): rows of the culled units (list CM_N_CLASSES), one CTA per
// unit, threads over its rows (coalesced field-major stores)
template <int TIER>
__global__ void __launch_bounds__(CM_MF_MAX_THREADS) k_mf_culled(const MfArgs a) {
  __shared__ UnitCtx U;
  int u;
  if (!list_unit(a, CM_N_CLASSES, U, u)) return;
  const bool full = (a.mode & CM_FULL_MODE) != 0;
  const PairFrame& F = U.F;
  const int V = U.SA.V, E = U.SA.E;
  const int nr = full ? V + E : U.SA.F;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const int32_t* fv = a.S.faces + 3 * (int64_t)U.SA.f_off;
  const int32_t* ed = a.S.edges + 2 * (int64_t)U.SA.e_off;
  const cm_manifold_out& o = a.out;
  const int64_t C = a.C;
  const float depth = full ? U.lb : fmaf(-a.S.sp.tau_min, 1.791759469228055f, U.lb);   // lb - tau ln 6
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    float x[3];
    if (!full) {   // the face centroid
      const float4 p0 = ldv(lv, __ldg(fv + 3 * r)), p1 = ldv(lv, __ldg(fv + 3 * r + 1)), p2 = ldv(lv, __ldg(fv + 3 * r + 2));
      x[0] = (p0.x + p1.x + p2.x) * (1.f / 3.f);
      x[1] = (p0.y + p1.y + p2.y) * (1.f / 3.f);
      x[2] = (p0.z + p1.z + p2.z) * (1.f / 3.f);
    } else if (r < V) {
      const float4 p0 = ldv(lv, r);
      x[0] = p0.x; x[1] = p0.y; x[2] = p0.z;
    } else {        // edge midpoint (edges in sorted (lo, hi) order)
      const float4 p0 = ldv(lv, __ldg(ed + 2 * (r - V))), p1 = ldv(lv, __ldg(ed + 2 * (r - V) + 1));
      x[0] = 0.5f * (p0.x + p1.x); x[1] = 0.5f * (p0.y + p1.y); x[2] = 0.5f * (p0.z + p1.z);
    }
    float xb[3], pw[3];
    to_frames(F, x, xb, pw);
    const int64_t c = U.off + r;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      o.point[k * C + c] = pw[k];
      o.normal[k * C + c] = 0.f;
    }
    o.depth[c] = depth;
    o.dom[c] = (int8_t)-2;
    if constexpr (TIER >= 1) {
      o.W[c] = 0.f;
#pragma unroll
      for (int k = 0; k < 3; ++k) o.q[k * C + c] = 0.f;
    }
    if constexpr (TIER >= 2) {
#pragma unroll
      for (int k = 0; k < 12; ++k) o.ddepth[k * C + c] = 0.f;
#pragma unroll
      for (int k = 0; k < 36; ++k) o.dnormal[k * C + c] = 0.f;
    }
    if constexpr (TIER >= 3) {
#pragma unroll 6
      for (int k = 0; k < 78; ++k) o.d2depth[k * C + c] = 0.f;
    }
  }
}

#ifndef CM_MF_FACE_L2PF
#define CM_MF_FACE_L2PF 0   // face kernel: L2 bulk prefetch of the records of the unit this many CTAs ahead
                           // (768 / 1536 / 3072: C5 -0.4 / -2.0 / -2.2%, C4 -0.2 / +0.5 / +0.4%; r02ze)
#endif
#ifndef CM_MF_FACE_REGS
#define CM_MF_FACE_REGS 0   // explicit register cap of the tier-0-2 face kernel (0: CM_MF_FACE_MINB)
#endif
template <int TIER> struct FaceRegs {
  static constexpr int R = TIER >= 3 ? (CM_MF_REG_T3 ? CM_MF_REG_T3 : 255) : (CM_MF_FACE_REGS ? CM_MF_FACE_REGS : regs_of(CM_MF_FACE_MINB));
};
template <int TIER, bool STAGED>
__global__ void __launch_bounds__(CM_MF_MAX_THREADS) __maxnreg__((FaceRegs<TIER>::R)) k_mf_faces(const MfArgs a) {
  extern __shared__ __align__(16) float fsm[];
  __shared__ UnitCtx U;
  __shared__ uint64_t bar;
  if (STAGED && threadIdx.x == 0) mbar_init(&bar, 1);   // published by list_unit's barrier
  int u;
  if (CM_MF_FACE_L2PF && !STAGED && threadIdx.x == 0) {
    // the candidate records of the unit CM_MF_FACE_L2PF CTAs ahead (about
    // one wave of resident CTAs) into L2, so that its face loads hit L2
    // instead of waiting on HBM; the first wave prefetches its own
    const int64_t b = blockIdx.x;
    for (int64_t v = (b < CM_MF_FACE_L2PF ? b : b + CM_MF_FACE_L2PF); v <= b + CM_MF_FACE_L2PF; v += CM_MF_FACE_L2PF) {
      if (v >= a.nb) break;
      const UnitCtx& c = a.ctx[v];
      const int V = c.SA.V, E = c.SA.E;
      const uint32_t bytes = (uint32_t)(vrec(TIER) * V + erec(TIER) * E) * 4u;
      if (bytes > 0 && c.valid) bulk_prefetch_l2(a.scratch + v * a.slot, bytes);
    }
  }
  if constexpr (STAGED) {
    if (list_unit(a, -1, U, u) && U.valid) mf_faces_unit<TIER, STAGED>(a, U, u, fsm, &bar, 0u);
  } else {
    for (int r = 0; r < CM_MF_UPC; ++r) {
      if (!list_unit(a, -1, U, u, blockIdx.x * CM_MF_UPC + r)) return;
      if (U.valid) mf_faces_unit<TIER, STAGED>(a, U, u, fsm, &bar, 0u);
      if (CM_MF_UPC > 1) __syncthreads();
    }
  }
}

// ---- shape-parameter VJP of the manifold depths (f4, reading #48) ----------
// vjp[poff[B] + k] += sum_rows w_r d depth_r / d theta_k for the parameters
// theta of the pair's SDF shape B (one-sided units; the sampled surface is
// data).  One CTA per unit, the manifold re-derived in B's frame:
//   forward  vertices phi_B(x_v); both traces of every edge (alpha_{k+1} =
//            alpha_k + sgn G(phi(x_k)), G(phi) = sigma(phi/tau) phi, the corner
//            iterate at the vertex), soft clips, the midpoint candidate
//            phi_B(x_e) and d phi / d alpha_bar = grad phi . e_B;
//   rows     reduced: depth = -tau LSE(-d_i / tau) over the face's six
//            candidates, so the candidate adjoints are dbar_i = sum_faces
//            w_f z_i (shared-memory atomics); full: dbar = w of its row;
//   reverse  dbar_v J(x_v) + dbar_e J(x_e), then the edge's alpha adjoint
//            dbar_e (grad phi . e_B) / 2 times each clip derivative, carried
//            back through the trace: theta_bar += lambda sgn G'(phi_k) J(x_k),
//            lambda <- lambda (1 + sgn G'(phi_k) grad phi_k . e_B),
// J(x) = d phi_B / d theta at x (cm_param.cuh shape_param_grad), summed per
// CTA in shared memory, one global atomic per parameter and unit.
#define CM_PV_THREADS 128
#define CM_PV_MAX_ITERS 16
__global__ void __launch_bounds__(CM_PV_THREADS) k_mf_param_vjp(const MfArgs a, const float* __restrict__ w,
                                                                float* __restrict__ vjp,
                                                                const int64_t* __restrict__ poff, int max_V,
                                                                int max_E) {
  extern __shared__ __align__(16) float psm[];
  __shared__ UnitCtx U;
  __shared__ int shB;
  if (threadIdx.x == 0) {
    unit_resolve(a, blockIdx.x, U);
    // the unit's SDF shape: B, or A for the transposed half of a two-sided pair
    const bool two = (a.mode & CM_TWO_SIDED) != 0;
    const int64_t pi = two ? (int64_t)blockIdx.x >> 1 : (int64_t)blockIdx.x;
    const int side = two ? (int)(blockIdx.x & 1) : 0;
    shB = __ldg(a.pairs + 5 * pi + 4 - side);
  }
  __syncthreads();
  if (!U.valid) return;
  const int V = U.SA.V, E = U.SA.E, NF = U.SA.F;
  const int64_t pb = __ldg(poff + shB);
  const int np = (int)(__ldg(poff + shB + 1) - pb);
  float* dV = psm;                  // [max_V] vertex candidate values
  float* adjV = dV + max_V;         // [max_V] their adjoints
  float* dE = adjV + max_V;         // [max_E] edge candidate values
  float* gE = dE + max_E;           // [max_E] grad phi . e_B at the edge point
  float* aE = gE + max_E;           // [max_E] alpha_bar
  float* adjE = aE + max_E;         // [max_E] adjoints
  float* thb = adjE + max_E;        // [np] parameter adjoint of this unit
  const PairFrame& F = U.F;
  const SmoothDev& sp = a.S.sp;
  const float* lv = a.S.verts + 4 * (int64_t)U.SA.v_off;
  const int32_t* ed = a.S.edges + 2 * (int64_t)U.SA.e_off;
  const int32_t* fv = a.S.faces + 3 * (int64_t)U.SA.f_off;
  const int32_t* fe = a.S.face_edges + 3 * (int64_t)U.SA.f_off;
  const bool full = (a.mode & CM_FULL_MODE) != 0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) thb[k] = 0.f;
  auto xB_of = [&](int v, float* xb) {
    const float4 x4 = ldv(lv, v);
    const float x[3] = {x4.x, x4.y, x4.z};
    float pw[3];
    to_frames(F, x, xb, pw);
  };
  // the edge in B's frame: start point, unit direction, length
  auto edge_B = [&](int e, float* xI, float* eb, float& L, int& vI, int& vII) {
    vI = __ldg(ed + 2 * e);
    vII = __ldg(ed + 2 * e + 1);
    const float4 xa = ldv(lv, vI), xc = ldv(lv, vII);
    const float dl[3] = {xc.x - xa.x, xc.y - xa.y, xc.z - xa.z};
    L = sqrtf(dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]);
    const float iL = 1.f / L;
    const float el[3] = {dl[0] * iL, dl[1] * iL, dl[2] * iL};
    rot_vec(F.Rrel, el, eb);
    xB_of(vI, xI);
  };
  auto phi1 = [&](const float* x, Res<1>& r) { eval_shape<1, 2, false, false, false, false>(a.S, U.SB, x, r); };
  // one trace: the final alpha; its iterates' alphas in al[] (al[0] the corner's)
  auto trace = [&](const float* xI, const float* eb, float L, const float* xc, int dir, float* al) {
    float alpha = dir ? L : 0.f;
    const float sgn = dir ? -1.f : 1.f;
    for (int it = 0; it < sp.iters; ++it) {
      al[it] = alpha;
      float x[3];
      if (it == 0) { x[0] = xc[0]; x[1] = xc[1]; x[2] = xc[2]; }
      else { for (int i = 0; i < 3; ++i) x[i] = fmaf(alpha, eb[i], xI[i]); }
      Res<0> r;
      eval_shape<0, 2, false, false, false, false>(a.S, U.SB, x, r);
      alpha = fmaf(sgn * sigm(r.v * sp.i_cmp), r.v, alpha);
    }
    return alpha;
  };
  // forward: vertex candidates
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    float xb[3];
    xB_of(v, xb);
    Res<0> r;
    eval_shape<0, 2, false, false, false, false>(a.S, U.SB, xb, r);
    dV[v] = r.v;
    adjV[v] = full ? __ldg(w + U.off + v) : 0.f;
  }
  // forward: edge candidates
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    float xI[3], eb[3], L;
    int vI, vII;
    edge_B(e, xI, eb, L, vI, vII);
    float xc[3], al[CM_PV_MAX_ITERS];
    float ab = 0.f;
    for (int dir = 0; dir < 2; ++dir) {
      xB_of(dir ? vII : vI, xc);
      const float afin = trace(xI, eb, L, xc, dir, al);
      float at, c1, c2;
      softclip_12(afin, 0.f, L, sp.tau_clip_alpha, sp.i_clip_alpha, at, c1, c2);
      ab += at;
    }
    ab *= 0.5f;
    const float x[3] = {fmaf(ab, eb[0], xI[0]), fmaf(ab, eb[1], xI[1]), fmaf(ab, eb[2], xI[2])};
    Res<1> r;
    phi1(x, r);
    dE[e] = r.v;
    gE[e] = r.g[0] * eb[0] + r.g[1] * eb[1] + r.g[2] * eb[2];
    aE[e] = ab;
    adjE[e] = full ? __ldg(w + U.off + V + e) : 0.f;
  }
  __syncthreads();
  // rows: the candidates' depth adjoints (reduced mode: face softmax)
  if (!full) {
    const float itl = LOG2E * sp.i_min;
    for (int f = threadIdx.x; f < NF; f += blockDim.x) {
      const float wf = __ldg(w + U.off + f);
      if (wf == 0.f) continue;
      int cv[3], ce[3];
      float dc[6];
      for (int k = 0; k < 3; ++k) {
        cv[k] = __ldg(fv + 3 * f + k);
        ce[k] = __ldg(fe + 3 * f + k);
        dc[k] = dV[cv[k]];
        dc[3 + k] = dE[ce[k]];
      }
      float dm = dc[0];
      for (int i = 1; i < 6; ++i) dm = fminf(dm, dc[i]);
      float z[6], Z = 0.f;
      for (int i = 0; i < 6; ++i) { z[i] = ex2((dm - dc[i]) * itl); Z += z[i]; }
      const float iZ = wf / Z;
      for (int k = 0; k < 3; ++k) {
        atomicAdd(adjV + cv[k], z[k] * iZ);
        atomicAdd(adjE + ce[k], z[3 + k] * iZ);
      }
    }
    __syncthreads();
  }
  auto accum = [&](const float* x, float scale) {
    shape_param_grad(a.S, U.SB, x, [&](int k, float v) { if (k < np) atomicAdd(thb + k, scale * v); });
  };
  // reverse: vertex candidates
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    if (adjV[v] == 0.f) continue;
    float xb[3];
    xB_of(v, xb);
    accum(xb, adjV[v]);
  }
  // reverse: edge candidates, their points and traces
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const float de = adjE[e];
    if (de == 0.f) continue;
    float xI[3], eb[3], L;
    int vI, vII;
    edge_B(e, xI, eb, L, vI, vII);
    const float ab = aE[e];
    const float x[3] = {fmaf(ab, eb[0], xI[0]), fmaf(ab, eb[1], xI[1]), fmaf(ab, eb[2], xI[2])};
    accum(x, de);
    const float abar_adj = de * gE[e];   // d depth / d alpha_bar
    float xc[3], al[CM_PV_MAX_ITERS];
    for (int dir = 0; dir < 2; ++dir) {
      xB_of(dir ? vII : vI, xc);
      const float afin = trace(xI, eb, L, xc, dir, al);
      float at, c1, c2;
      softclip_12(afin, 0.f, L, sp.tau_clip_alpha, sp.i_clip_alpha, at, c1, c2);
      const float sgn = dir ? -1.f : 1.f;
      float lam = 0.5f * abar_adj * c1;
      for (int it = sp.iters - 1; it >= 0; --it) {
        float xk[3];
        if (it == 0) { xk[0] = xc[0]; xk[1] = xc[1]; xk[2] = xc[2]; }
        else { for (int i = 0; i < 3; ++i) xk[i] = fmaf(al[it], eb[i], xI[i]); }
        Res<1> r;
        phi1(xk, r);
        const float s = sigm(r.v * sp.i_cmp);
        const float Gp = fmaf(r.v * s * (1.f - s), sp.i_cmp, s);
        accum(xk, lam * sgn * Gp);
        lam *= fmaf(sgn * Gp, r.g[0] * eb[0] + r.g[1] * eb[1] + r.g[2] * eb[2], 1.f);
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < np; k += blockDim.x)
    if (thb[k] != 0.f) atomicAdd(vjp + pb + k, thb[k]);
}

namespace cml {

// floats of one unit's scratch slot
int64_t manifold_slot_floats(int V, int E, int tier) {
  // records are multiples of 4 floats: every slot and record is 16-B aligned
  return (int64_t)vrec(tier) * V + (int64_t)erec(tier) * E;
}

// the fused midpoint + face kernel's shared memory (0: not used)
static int midfaces_bytes(int tier, uint32_t mode, int max_V, int max_E) {
  if (!CM_MF_FUSE_FACES || tier > 2 || (mode & CM_FULL_MODE)) return 0;
  const int b = (max_E * erec(tier) + max_V * vrec(tier)) * 4;
  return b <= 160 * 1024 ? b : 0;
}

template <int TIER, int XP>
static int launch_sdf_phases(MfArgs& a, int64_t nb, int T, int max_V, int max_E, cudaStream_t st) {
  if (nb <= CM_MF_SMALL_UNITS) {   // small batch: one kernel per class (faces included)
    k_mf_small<TIER, XP><<<(unsigned)nb, T, 0, st>>>(a);
    return check_launch("k_mf_small");
  }
  const unsigned gu = (unsigned)((nb + CM_MF_UPC - 1) / CM_MF_UPC);   // CTAs of CM_MF_UPC units
  k_mf_vertices<TIER, XP><<<gu, T, 0, st>>>(a);
  int rc = check_launch("k_mf_vertices");
  if (rc) return rc;
  if constexpr (TIER <= 2 && CM_MF_FUSE_EDGES && CM_TRACE6) {
    if (midfaces_bytes(TIER, a.mode, max_V, max_E) == 0) {
      k_mf_edges<TIER, XP><<<(unsigned)nb, T, CM_MF_EDGE_SMEM ? T * 10 * 4 : 0, st>>>(a);
      return check_launch("k_mf_edges");
    }
  }
  bool cat = false;
  if constexpr (TIER <= 2 && CM_TRACE6 && !CM_TRACE_PAIRED && CM_MF_CAT > 1) {
    if (2 * max_E <= CM_MF_CAT_MAX_ITEMS) {
      k_mf_traces_cat<TIER, XP, CM_MF_CAT><<<(unsigned)((nb + CM_MF_CAT - 1) / CM_MF_CAT), T, 0, st>>>(a);
      cat = true;
    }
  }
  if (!cat) k_mf_traces<TIER, XP><<<gu, T, 0, st>>>(a);
  if ((rc = check_launch("k_mf_traces"))) return rc;
  if constexpr (TIER <= 2) {
    const int fb = midfaces_bytes(TIER, a.mode, max_V, max_E);
    if (fb > 0) {
      if (fb > 48 * 1024)
        cudaFuncSetAttribute(k_mf_midfaces<TIER, XP>, cudaFuncAttributeMaxDynamicSharedMemorySize, fb);
      k_mf_midfaces<TIER, XP><<<(unsigned)nb, T, fb, st>>>(a, max_E);
      return check_launch("k_mf_midfaces");
    }
  }
  const int mid_bytes = max_E * erec(TIER) * 4;
  if (CM_MF_STAGE_MID && mid_bytes <= 96 * 1024) {
    if (mid_bytes > 48 * 1024)
      cudaFuncSetAttribute(k_mf_midpoints<TIER, XP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mid_bytes);
    k_mf_midpoints<TIER, XP, true><<<(unsigned)nb, T, mid_bytes, st>>>(a);
  } else {
    k_mf_midpoints<TIER, XP, false><<<gu, T, (TIER == 2 && CM_MF_MID_PREFETCH) ? T * 80 : 0, st>>>(a);
  }
  return check_launch("k_mf_midpoints");
}

constexpr int kStageSmallBytes = 24 * 1024;

template <int TIER>
static int launch_tier(MfArgs a, int class_mask, int max_V, int max_E, int64_t n_units, int64_t chunk,
                       cudaStream_t const* streams, int n_streams) {
  const bool full = (a.mode & CM_FULL_MODE) != 0;
  float* scratch0 = a.scratch;
  UnitCtx* ctx0 = a.ctx;
  int* lists0 = a.cls_list;
  int* ctrl0 = a.cls_count;   // per stream: [32] counts + counters
  // face-kernel staging in shared memory when the largest unit fits; used
  // for small staged footprints and for chunks too small to fill the SMs
  // anyway (measured: C4 / C2 gain 3-25%, C5 / C3 lose 8-10% to the lower
  // occupancy)
  int stage_bytes = (int)(face_stage_floats(max_V, max_E, TIER) * 4);
  {
    // (the attribute is per device and per kernel: set on every call for the
    // current device, no process-wide cache; a failure disables the staging)
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (stage_bytes + (int)sizeof(UnitCtx) + 1024 > optin) {
      stage_bytes = 0;
    } else if (stage_bytes > 48 * 1024 &&
               cudaFuncSetAttribute(k_mf_faces<TIER, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    stage_bytes) != cudaSuccess) {
      cudaGetLastError();
      stage_bytes = 0;
    }
  }
  // chunk k runs on stream k % n_streams in that stream's scratch region, so
  // one chunk's kernel tails overlap the next chunk's kernels
  for (int64_t u0 = 0, k = 0; u0 < n_units; u0 += chunk, ++k) {
    const int64_t nb = n_units - u0 < chunk ? n_units - u0 : chunk;
    cudaStream_t st = streams[k % n_streams];
    a.unit0 = u0;
    a.scratch = scratch0 + (k % n_streams) * chunk * a.slot;
    a.ctx = ctx0 + (k % n_streams) * chunk;
    a.cls_count = ctrl0 + 32 * (k % n_streams);
    a.cls_list = lists0 + (k % n_streams) * chunk * CM_N_LISTS;
    a.chunk = chunk;
    a.nb = nb;
    if (cudaMemsetAsync(a.cls_count, 0, 32 * sizeof(int), st) != cudaSuccess) {
      set_error("manifold: counter reset failed");
      return CM_ERR_CUDA;
    }
    k_mf_units<<<(unsigned)((nb + 127) / 128), 128, 0, st>>>(a, nb);
    if (int rcu = check_launch("k_mf_units")) return rcu;
    // >= 32 resident warps per SM over the chunk's units (small batches)
    int T = CM_MF_THREADS;
    while (T < CM_MF_MAX_THREADS && nb * (T / 32) < (int64_t)num_sms() * 32) T *= 2;
    int rc = CM_OK;
    // SDF phases: one instantiation per SDF class present in the scene
    // (cm_internal.h ShapeRec::uses_xpsq); each takes its class's units from
    // the list k_mf_units built
    if (class_mask & 1) rc = launch_sdf_phases<TIER, 0>(a, nb, T, max_V, max_E, st);
    if (!rc && (class_mask & 2)) rc = launch_sdf_phases<TIER, 1>(a, nb, T, max_V, max_E, st);
    if (!rc && (class_mask & 4)) rc = launch_sdf_phases<TIER, 2>(a, nb, T, max_V, max_E, st);
    if (!rc && (class_mask & 8)) rc = launch_sdf_phases<TIER, 3>(a, nb, T, max_V, max_E, st);
    if (!rc && (class_mask & 16)) rc = launch_sdf_phases<TIER, 4>(a, nb, T, max_V, max_E, st);
    if (rc) return rc;
    if (a.mode & CM_BROAD_PHASE) {   // the culled units' rows (f2)
      k_mf_culled<TIER><<<(unsigned)nb, T, 0, st>>>(a);
      if ((rc = check_launch("k_mf_culled"))) return rc;
    }
    if (!full && midfaces_bytes(TIER, a.mode, max_V, max_E) == 0 && nb > CM_MF_SMALL_UNITS) {   // the fusion does not depend on the SDF class: one launch
      if (stage_bytes > 0 && (stage_bytes <= kStageSmallBytes || nb < 8 * (int64_t)num_sms()))
        k_mf_faces<TIER, true><<<(unsigned)nb, T, stage_bytes, st>>>(a);
      else
        k_mf_faces<TIER, false><<<(unsigned)((nb + CM_MF_UPC - 1) / CM_MF_UPC), T, 0, st>>>(a);
      if ((rc = check_launch("k_mf_faces"))) return rc;
    }
  }
  return CM_OK;
}

int launch_manifold(const SceneDev& s, int class_mask, int max_V, int max_E, const int32_t* pairs,
                    int64_t n_pairs, const int64_t* offsets, const float* poses, int64_t n_env, int32_t n_slot,
                    uint32_t flags,
                    const cm_manifold_out* out, int64_t C, float* scratch, int64_t scratch_floats,
                    void* const* streams, int n_streams) {
  const int tier = (int)(flags & CM_TIER_MASK);
  const uint32_t mode = flags & (CM_FULL_MODE | CM_TWO_SIDED | CM_BROAD_PHASE);
  const int64_t n_units = (mode & CM_TWO_SIDED) ? 2 * n_pairs : n_pairs;
  const int64_t slot = manifold_slot_floats(max_V, max_E, tier);
  if (n_streams < 1) n_streams = 1;
  // each unit of a chunk: its candidate slot and its set-up record (after
  // all slots; slots are multiples of 4 floats so the records stay aligned)
  const int64_t ctxf = (int64_t)(sizeof(UnitCtx) / 4) + CM_N_LISTS;   // + the class-list entries
  int64_t chunk = slot > 0 ? (scratch_floats - 32 * n_streams) / n_streams / (slot + ctxf) : 0;
  if (scratch == nullptr || chunk < 1) {
    set_error("manifold: scene scratch missing or too small");
    return CM_ERR_UNSUPPORTED;
  }
  if (chunk > 0x7fffffff) chunk = 0x7fffffff;
  MfArgs a;
  a.S = s;
  a.pairs = pairs;
  a.n_pairs = n_pairs;
  a.unit0 = 0;
  a.offsets = offsets;
  a.poses = poses;
  a.n_env = n_env;
  a.n_slot = n_slot;
  a.out = *out;
  a.C = C;
  a.scratch = scratch;
  a.slot = slot;
  a.mode = mode;
  // scratch layout: [slots | unit records | class lists | counters], per stream
  a.ctx = reinterpret_cast<UnitCtx*>(scratch + (int64_t)n_streams * chunk * slot);
  a.cls_list = reinterpret_cast<int*>(a.ctx + (int64_t)n_streams * chunk);
  a.cls_count = a.cls_list + (int64_t)n_streams * chunk * CM_N_LISTS;
  a.chunk = chunk;
  a.nb = 0;
  cudaStream_t const* sts = (cudaStream_t const*)streams;
  if (tier >= 3) return launch_tier<3>(a, class_mask, max_V, max_E, n_units, chunk, sts, n_streams);
  if (tier == 2) return launch_tier<2>(a, class_mask, max_V, max_E, n_units, chunk, sts, n_streams);
  if (tier == 1) return launch_tier<1>(a, class_mask, max_V, max_E, n_units, chunk, sts, n_streams);
  return launch_tier<0>(a, class_mask, max_V, max_E, n_units, chunk, sts, n_streams);
}

int launch_manifold_param_vjp(const SceneDev& s, int max_V, int max_E, int pmax, const int32_t* pairs,
                              int64_t n_pairs, const int64_t* offsets, const float* poses, int64_t n_env,
                              int32_t n_slot, uint32_t mode, const float* w, float* vjp, const int64_t* poff,
                              void* stream) {
  if (s.sp.iters > CM_PV_MAX_ITERS) {
    set_error("manifold_param_vjp: more than 16 trace iterations");
    return CM_ERR_UNSUPPORTED;
  }
  if (n_pairs <= 0) return CM_OK;
  MfArgs a;
  memset(&a, 0, sizeof(a));
  a.S = s;
  a.pairs = pairs;
  a.n_pairs = n_pairs;
  a.offsets = offsets;
  a.poses = poses;
  a.n_env = n_env;
  a.n_slot = n_slot;
  a.mode = mode;
  const int bytes = (2 * max_V + 4 * max_E + pmax) * 4;
  if (bytes > 48 * 1024 &&
      cudaFuncSetAttribute(k_mf_param_vjp, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    set_error("manifold_param_vjp: shared memory");
    return CM_ERR_UNSUPPORTED;
  }
  const int upp = (mode & CM_TWO_SIDED) ? 2 : 1;   // units per pair
  for (int64_t p0 = 0; p0 < n_pairs; p0 += 0x3fffffff) {   // (grids of at most 2^31 - 1 CTAs)
    const int64_t nb = n_pairs - p0 < 0x3fffffff ? n_pairs - p0 : 0x3fffffff;
    MfArgs ac = a;
    ac.pairs = pairs + 5 * p0;
    ac.offsets = offsets + p0;
    ac.n_pairs = nb;
    k_mf_param_vjp<<<(unsigned)(nb * upp), CM_PV_THREADS, bytes, (cudaStream_t)stream>>>(ac, w, vjp, poff, max_V,
                                                                                           max_E);
    if (int rc = check_launch("k_mf_param_vjp")) return rc;
  }
  return CM_OK;
}

}  // namespace cml
