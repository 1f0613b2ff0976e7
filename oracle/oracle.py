"""ctypes wrapper of the FP64 oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never
imports this module.  It packs the shared scene descriptions
(paper_2604_17538_b200.synth) into the oracle's own record layout; it shares
no code with the product binding.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.cpp")

MAXP, MAXC = 8, 32
NI, NF = 3 + MAXC, 93
TYPES = {"halfspace": 0, "sq": 1, "psq": 2, "xpsq": 3, "union": 10, "intersection": 11, "subtraction": 12}


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-o", LIB, SRC])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        d, i, l, p = C.c_double, C.c_int, C.c_long, C.c_void_p
        L.ora_scene_create.restype = p
        L.ora_scene_create.argtypes = [i, p, p, p, p, p, p, p, p, i]
        L.ora_scene_destroy.argtypes = [p]
        for n, a in (("ora_sigmoid", [d]), ("ora_softplus", [d, d]), ("ora_softclip", [d, d, d, d]),
                     ("ora_lse", [p, i, d]), ("ora_sq_f", [p, d, d, p]), ("ora_sq_phi", [p, d, d, p])):
            getattr(L, n).restype = d
            getattr(L, n).argtypes = a
        L.ora_softargmax.argtypes = [p, i, d, p]
        L.ora_xpsq_roots.argtypes = [p, i, i, p, p, p, p]
        L.ora_xpsq_frame.argtypes = [p, i, i, d, p]
        L.ora_xpsq_class.argtypes = [p, i, i]
        L.ora_mesh_counts.argtypes = [p, i, p, p, p]
        L.ora_mesh_topology.argtypes = [p, i, p, p]
        L.ora_sdf_eval.argtypes = [p, p, p, p, l, l, i, p, p, p, p, p, p]
        L.ora_contact_manifold.argtypes = [p, p, l, p, l, i] + [p] * 12 + [i, i]
        L.ora_manifold_d2depth.argtypes = [p, p, l, p, l, i, p, i, i]
        L.ora_shape_param_count.argtypes = [p, i]
        L.ora_shape_param_count.restype = i
        L.ora_sdf_param_grad.argtypes = [p, p, p, p, l, l, i, p]
        L.ora_sdf_node_pose_grad.argtypes = [p, p, p, p, l, l, i, p]
        L.ora_manifold_param_jac.argtypes = [p, p, l, p, l, i, i, i, p]
        L.ora_shape_node_count.argtypes = [p, i]
        L.ora_shape_node_count.restype = i
        L.ora_max_threads.restype = i
        L.ora_shape_bound.argtypes = [p, i, p]
        L.ora_mesh_sphere.argtypes = [p, i, p]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ---- unit functions ---------------------------------------------------------
def sigmoid(x):
    return lib().ora_sigmoid(float(x))


def softplus(x, tau):
    return lib().ora_softplus(float(x), float(tau))


def softclip(x, lo, hi, tau):
    return lib().ora_softclip(float(x), float(lo), float(hi), float(tau))


def lse(xs, tau):
    a = np.ascontiguousarray(xs, dtype=np.float64)
    return lib().ora_lse(_ptr(a), len(a), float(tau))


def softargmax(xs, tau):
    a = np.ascontiguousarray(xs, dtype=np.float64)
    out = np.zeros_like(a)
    lib().ora_softargmax(_ptr(a), len(a), float(tau), _ptr(out))
    return out


def sq_f(y, eps, a):
    y = np.ascontiguousarray(y, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().ora_sq_f(_ptr(y), float(eps[0]), float(eps[1]), _ptr(a))


def sq_phi(y, eps, a):
    y = np.ascontiguousarray(y, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().ora_sq_phi(_ptr(y), float(eps[0]), float(eps[1]), _ptr(a))


# ---- scenes -----------------------------------------------------------------
def _pack_nodes(nodes):
    ints = np.zeros((len(nodes), NI), dtype=np.int32)
    flts = np.zeros((len(nodes), NF), dtype=np.float32)
    for k, n in enumerate(nodes):
        ints[k, 0] = TYPES[n["type"]]
        ints[k, 1] = len(n["children"])
        np_ = len(n["planes"])
        assert np_ <= MAXP and len(n["children"]) <= MAXC
        ints[k, 2] = np_
        ints[k, 3:3 + len(n["children"])] = n["children"]
        row = list(n["pose"]) + list(n["eps"][0]) + list(n["eps"][1]) + list(n["a"][0]) + list(n["a"][1])
        pl = np.zeros((2, MAXP, 4), dtype=np.float64)
        for j, r in enumerate(n["planes"]):
            pl[0, j] = r
        p1 = n["planes1"] if n["planes1"] else n["planes"]
        for j, r in enumerate(p1):
            pl[1, j] = r
        row += list(pl.ravel()) + list(n["ctrl"]) + list(n["up"])
        assert len(row) == NF
        flts[k] = row
    return ints, flts


class OracleScene:
    def __init__(self, scene):
        self.scene = scene
        shapes = scene.shapes
        counts, ints, flts, vc, vs, fc, fs = [], [], [], [], [], [], []
        for s in shapes:
            nodes = s.sdf or []
            counts.append(len(nodes))
            if nodes:
                i_, f_ = _pack_nodes(nodes)
                ints.append(i_)
                flts.append(f_)
            v = s.vertices if s.vertices is not None else np.zeros((0, 3), np.float32)
            f = s.faces if s.faces is not None else np.zeros((0, 3), np.int32)
            vc.append(len(v))
            fc.append(len(f))
            vs.append(v)
            fs.append(f)
        self._keep = [np.ascontiguousarray(np.array(counts, dtype=np.int32)),
                      np.ascontiguousarray(np.concatenate(ints) if ints else np.zeros((1, NI), np.int32)),
                      np.ascontiguousarray(np.concatenate(flts) if flts else np.zeros((1, NF), np.float32)),
                      np.ascontiguousarray(np.array(vc, dtype=np.int32)),
                      np.ascontiguousarray(np.concatenate(vs).astype(np.float32)),
                      np.ascontiguousarray(np.array(fc, dtype=np.int32)),
                      np.ascontiguousarray(np.concatenate(fs).astype(np.int32))]
        sp = scene.smooth
        self._sm = np.array([sp["tau_cmp"], sp["tau_min"], sp["tau_clip_alpha"], sp["tau_clip_t"], sp["tau_delta"]],
                            dtype=np.float64)
        k = self._keep
        self.h = lib().ora_scene_create(len(shapes), _ptr(k[0]), _ptr(k[1]), _ptr(k[2]), _ptr(k[3]), _ptr(k[4]),
                                        _ptr(k[5]), _ptr(k[6]), _ptr(self._sm), int(sp["trace_iters"]))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_scene_destroy(self.h)
            self.h = None

    def mesh_counts(self, shape):
        V, E, F = C.c_int(), C.c_int(), C.c_int()
        lib().ora_mesh_counts(self.h, shape, C.byref(V), C.byref(E), C.byref(F))
        return V.value, E.value, F.value

    def mesh_topology(self, shape):
        V, E, F = self.mesh_counts(shape)
        e = np.zeros((E, 2), np.int32)
        fe = np.zeros((F, 3), np.int32)
        lib().ora_mesh_topology(self.h, shape, _ptr(e), _ptr(fe))
        return e, fe

    def xpsq_roots(self, shape, node, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        t = np.zeros(3)
        dl, wn = C.c_double(), C.c_double()
        lib().ora_xpsq_roots(self.h, shape, node, _ptr(y), _ptr(t), C.byref(dl), C.byref(wn))
        return t, dl.value, wn.value

    def xpsq_frame(self, shape, node, t):
        R = np.zeros(9)
        lib().ora_xpsq_frame(self.h, shape, node, float(t), _ptr(R))
        return R.reshape(3, 3)

    def xpsq_class(self, shape, node):
        return lib().ora_xpsq_class(self.h, shape, node)

    def sdf_eval(self, shape_ids, poses, points, P, want_pose=True):
        shape_ids = np.ascontiguousarray(shape_ids, dtype=np.int32)
        # float32 inputs are promoted exactly; float64 inputs (finite-difference
        # tests) are used as given
        poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 8)
        points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        B = len(shape_ids)
        N = B * P
        assert points.shape[0] == N
        out = dict(d=np.zeros(N), grad=np.zeros((N, 3)), hess=np.zeros((N, 6)), dpose=np.zeros((N, 6)),
                   d2pose=np.zeros((N, 21)), dxdpose=np.zeros((N, 18)))
        lib().ora_sdf_eval(self.h, _ptr(shape_ids), _ptr(poses), _ptr(points), B, P, int(want_pose),
                           *[_ptr(out[k]) for k in ("d", "grad", "hess", "dpose", "d2pose", "dxdpose")])
        return out

    def contact_manifold(self, pairs=None, poses=None, n_threads=0, mode=0):
        """mode bits: 4 full mode (V + E contacts), 8 two-sided, 16 broad phase (f2)."""
        sc = self.scene
        pairs = np.ascontiguousarray(sc.pairs if pairs is None else pairs, dtype=np.int32)
        poses = np.ascontiguousarray(sc.poses if poses is None else poses, dtype=np.float64)
        n_env, n_slot = poses.shape[0], poses.shape[1]
        def cnt(s):
            V, E, F_ = self.mesh_counts(int(s))
            return V + E if mode & 4 else F_
        F = [cnt(a) + (cnt(b) if mode & 8 else 0) for a, b in zip(pairs[:, 3], pairs[:, 4])]
        Ct = int(sum(F))
        out = dict(point=np.zeros((Ct, 3)), normal=np.zeros((Ct, 3)), depth=np.zeros(Ct), W=np.zeros(Ct),
                   q=np.zeros((Ct, 3)), ddepth=np.zeros((Ct, 12)), dnormal=np.zeros((Ct, 3, 12)),
                   dom=np.zeros(Ct, np.int32), J=np.zeros((Ct, 3, 12)), z=np.zeros((Ct, 6)),
                   dcand=np.zeros((Ct, 6)), gamma=np.zeros((Ct, 6)))
        lib().ora_contact_manifold(self.h, _ptr(pairs), len(pairs), _ptr(poses), n_env, n_slot,
                                   *[_ptr(out[k]) for k in ("point", "normal", "depth", "W", "q", "ddepth",
                                                            "dnormal", "dom", "J", "z", "dcand", "gamma")],
                                   int(mode), int(n_threads))
        out["offsets"] = np.concatenate([[0], np.cumsum(F)]).astype(np.int64)
        return out

    def shape_bound(self, shape):
        """Broad phase (f2): (c, rho) with phi(x) >= |x - c| - rho in the body
        frame (rho = inf: no bound, e.g. a half-space)."""
        o = np.zeros(4)
        lib().ora_shape_bound(self.h, int(shape), _ptr(o))
        return o[:3], o[3]

    def mesh_sphere(self, shape):
        o = np.zeros(4)
        lib().ora_mesh_sphere(self.h, int(shape), _ptr(o))
        return o[:3], o[3]

    @staticmethod
    def pair_reduce(out, tau_min, w_depth=None, w_normal=None):
        """Pair-level reductions of a manifold computed by contact_manifold
        (plain numpy over its rows, pair i at rows offsets[i]:offsets[i+1]):
        pair_depth = -tau_min log sum exp(-depth / tau_min) (the fusion's
        smooth minimum, P:161 / reading #25), pair_W = sum W, and the
        vector-Jacobian product g_pose[i] = sum_rows w_depth ddepth + sum_k
        w_normal[:, k] dnormal[:, k, :] (12 per pair)."""
        off = out["offsets"]
        n = len(off) - 1
        pd, pw, gp = np.zeros(n), np.zeros(n), np.zeros((n, 12))
        for i in range(n):
            r = slice(off[i], off[i + 1])
            d = out["depth"][r]
            m = np.max(-d)
            pd[i] = -(m + tau_min * np.log(np.sum(np.exp((-d - m) / tau_min))))
            pw[i] = np.sum(out["W"][r])
            if w_depth is not None:
                gp[i] += w_depth[r] @ out["ddepth"][r]
            if w_normal is not None:
                gp[i] += np.einsum("rk,rkj->j", w_normal[r], out["dnormal"][r])
        return pd, pw, gp

    def param_count(self, shape):
        """Number of shape parameters (-1: an XPSQ node, not parametrised)."""
        return lib().ora_shape_param_count(self.h, int(shape))

    def sdf_param_grad(self, shape_ids, poses, points, P, pmax=None):
        """J [B*P, pmax]: d phi / d (shape parameters), zero-padded."""
        shape_ids = np.ascontiguousarray(shape_ids, dtype=np.int32)
        poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 8)
        points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        if pmax is None:
            pmax = max(self.param_count(s) for s in np.unique(shape_ids))
        J = np.zeros((len(points), pmax))
        lib().ora_sdf_param_grad(self.h, _ptr(shape_ids), _ptr(poses), _ptr(points), len(shape_ids), P, int(pmax),
                                 _ptr(J))
        return J

    def node_count(self, shape):
        """Number of SDF nodes of a shape (boolean nodes and leaves)."""
        return lib().ora_shape_node_count(self.h, int(shape))

    def sdf_node_pose_grad(self, shape_ids, poses, points, P, nmax=None):
        """J [B*P, nmax]: d phi / d (node twists), 6 per node in node order
        (dt, dtheta in the node's parent frame: R <- exp([dtheta]x) R,
        t <- t + dt), zero-padded (f4 node poses, DESIGN reading #47)."""
        shape_ids = np.ascontiguousarray(shape_ids, dtype=np.int32)
        poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 8)
        points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        if nmax is None:
            nmax = 6 * max(self.node_count(s) for s in np.unique(shape_ids))
        J = np.zeros((len(points), nmax))
        lib().ora_sdf_node_pose_grad(self.h, _ptr(shape_ids), _ptr(poses), _ptr(points), len(shape_ids), P,
                                     int(nmax), _ptr(J))
        return J

    def manifold_param_jac(self, pairs=None, poses=None, mode=0, pmax=None):
        """Jd [rows, pmax]: d depth(row) / d shape parameter of the row's SDF
        shape (B for the pair's first half, A for the second half of a
        two-sided manifold; the layout of sdf_param_grad), from the literal
        manifold with the parameter seeded (f4, reading #48).  Broad-phase
        culled rows have zero rows (their depth is a certified bound, not a
        differentiated output)."""
        sc = self.scene
        pairs = np.ascontiguousarray(sc.pairs if pairs is None else pairs, dtype=np.int32)
        poses = np.ascontiguousarray(sc.poses if poses is None else poses, dtype=np.float64)
        n_env, n_slot = poses.shape[0], poses.shape[1]
        two = bool(mode & 8)
        if pmax is None:
            sdf = np.unique(np.concatenate([pairs[:, 4], pairs[:, 3]] if two else [pairs[:, 4]]))
            pmax = max(self.param_count(int(b)) for b in sdf)
        full = bool(mode & 4)
        rows = 0
        for pr in pairs:
            for a in ((pr[3], pr[4]) if two else (pr[3],)):
                V, E, F = self.mesh_counts(int(a))
                rows += V + E if full else F
        Jd = np.zeros((rows, pmax))
        rc = lib().ora_manifold_param_jac(self.h, _ptr(pairs), len(pairs), _ptr(poses), n_env, n_slot, int(mode),
                                          int(pmax), _ptr(Jd))
        assert rc == 0
        return Jd

    def manifold_d2depth(self, pairs=None, poses=None, n_threads=0, mode=0):
        """d^2 depth / dq^2 per contact (packed upper triangle, 78 per row, q in
        the pair's (t_A, theta_A, t_B, theta_B) order) for the same rows as
        contact_manifold(pairs, poses, mode=mode)."""
        sc = self.scene
        pairs = np.ascontiguousarray(sc.pairs if pairs is None else pairs, dtype=np.int32)
        poses = np.ascontiguousarray(sc.poses if poses is None else poses, dtype=np.float64)
        n_env, n_slot = poses.shape[0], poses.shape[1]
        def cnt(s):
            V, E, F_ = self.mesh_counts(int(s))
            return V + E if mode & 4 else F_
        Ct = int(sum(cnt(a) + (cnt(b) if mode & 8 else 0) for a, b in zip(pairs[:, 3], pairs[:, 4])))
        out = np.zeros((Ct, 78))
        lib().ora_manifold_d2depth(self.h, _ptr(pairs), len(pairs), _ptr(poses), n_env, n_slot, _ptr(out),
                                   int(mode), int(n_threads))
        return out


def max_threads():
    return lib().ora_max_threads()
