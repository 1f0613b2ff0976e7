"""Thin Python binding of the C ABI (include/xpsq_cm.h) over torch tensors.

Argument marshalling only: every step of the hot path runs in the sm_100a
kernels of libxpsqcm.so.  PyTorch provides device memory and streams.  There
is no CPU fallback: if the library is missing or CUDA is unavailable the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XPSQCM_LIB") or os.path.join(HERE, "libxpsqcm.so")   # override: build experiments

CM_MAX_PLANES = 8
CM_MAX_CHILDREN = 32
NODE_TYPES = {"halfspace": 0, "sq": 1, "psq": 2, "xpsq": 3, "union": 10, "intersection": 11, "subtraction": 12}

SDF_VALUE, SDF_GRAD, SDF_HESS, SDF_POSE_GRAD, SDF_POSE_HESS = 1, 2, 4, 8, 16
FULL_MODE, TWO_SIDED, BROAD_PHASE = 4, 8, 16   # manifold mode bits (include/xpsq_cm.h)

EXPORTS = ["cm_version", "cm_last_error", "cm_scene_create", "cm_scene_destroy", "cm_shape_counts",
           "cm_param_layout", "cm_sdf_param_grad",
           "cm_shape_topology", "cm_sdf_eval", "cm_manifold_size", "cm_manifold_offsets_workspace",
           "cm_manifold_offsets", "cm_contact_manifold", "cm_expand_jacobian", "cm_launch_count",
           "cm_scene_error_count", "cm_manifold_pair_reduce", "cm_node_pose_layout", "cm_sdf_node_pose_grad",
           "cm_manifold_param_vjp", "cm_tessellate"]


class cm_node(C.Structure):
    _fields_ = [("type", C.c_int32), ("n_children", C.c_int32), ("children", C.c_int32 * CM_MAX_CHILDREN),
                ("n_planes", C.c_int32), ("pose", C.c_float * 7), ("eps", (C.c_float * 2) * 2),
                ("a", (C.c_float * 3) * 2), ("planes", ((C.c_float * 4) * CM_MAX_PLANES) * 2),
                ("ctrl", C.c_float * 9), ("up", C.c_float * 3)]


class cm_shape_desc(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nodes", C.POINTER(cm_node)), ("n_vertices", C.c_int32),
                ("vertices", C.POINTER(C.c_float)), ("n_faces", C.c_int32), ("faces", C.POINTER(C.c_int32)),
                ("sample_res", C.c_int32)]


class cm_smooth_params(C.Structure):
    _fields_ = [("tau_cmp", C.c_float), ("tau_min", C.c_float), ("tau_clip_alpha", C.c_float),
                ("tau_clip_t", C.c_float), ("tau_delta", C.c_float), ("trace_iters", C.c_int32)]


class cm_manifold_out(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("point", "normal", "depth", "W", "q", "ddepth", "dnormal", "dom", "d2depth")]


class CMError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libxpsqcm.so (in-tree).  Raises if it is missing: the product has
    no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CMError("libxpsqcm.so not built: run `python -m paper_2604_17538_b200.build` "
                          "(or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        p, i32, i64, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32
        L.cm_version.restype = C.c_int
        L.cm_last_error.restype = C.c_char_p
        L.cm_scene_create.argtypes = [p, i32, p, C.c_int, C.POINTER(p)]
        L.cm_scene_destroy.argtypes = [p]
        L.cm_shape_counts.argtypes = [p, i32, p, p, p]
        L.cm_shape_topology.argtypes = [p, i32, p, p]
        L.cm_sdf_eval.argtypes = [p, p, p, p, i64, i64, u32, p, p, p, p, p, p, p]
        L.cm_manifold_size.argtypes = [p, p, i64, u32, p]
        L.cm_param_layout.argtypes = [p, p, p]
        L.cm_sdf_param_grad.argtypes = [p, p, p, p, i64, i64, i32, p, p, p, p]
        L.cm_manifold_offsets_workspace.argtypes = [i64]
        L.cm_manifold_offsets_workspace.restype = i64
        L.cm_manifold_offsets.argtypes = [p, p, i64, u32, p, p, i64, p]
        L.cm_contact_manifold.argtypes = [p, p, i64, p, p, i64, i32, u32, p, i64, p]
        L.cm_expand_jacobian.argtypes = [p, p, i64, p, p, i64, i32, u32, p, p, i64, p, p]
        L.cm_launch_count.restype = i64
        if hasattr(L, "cm_scene_error_count"):   # (older builds in A/B sweeps lack these)
            L.cm_scene_error_count.argtypes = [p, p, C.c_int]
        if hasattr(L, "cm_manifold_pair_reduce"):
            L.cm_manifold_pair_reduce.argtypes = [p, p, i64, p, u32, p, i64, p, p, p, p, p, p]
        if hasattr(L, "cm_sdf_node_pose_grad"):
            L.cm_node_pose_layout.argtypes = [p, p, p]
            L.cm_sdf_node_pose_grad.argtypes = [p, p, p, p, i64, i64, i32, p, p, p, p]
        if hasattr(L, "cm_tessellate"):
            L.cm_tessellate.argtypes = [p, i32, p, p, p, p]
        if hasattr(L, "cm_manifold_param_vjp"):
            L.cm_manifold_param_vjp.argtypes = [p, p, i64, p, p, i64, i32, u32, p, p, p]
        _lib = L
    return _lib


def tessellate(node: dict, res: int):
    """Library-side sampled surface of one SQ / PSQ / XPSQ node (host call,
    no GPU needed): (vertices [V,3] float32, faces [F,3] int32)."""
    L = lib()
    cn = _pack_node(node)
    nv, nf = C.c_int32(), C.c_int32()
    _check(L.cm_tessellate(C.byref(cn), int(res), None, None, C.byref(nv), C.byref(nf)), "cm_tessellate")
    v = np.zeros((nv.value, 3), np.float32)
    f = np.zeros((nf.value, 3), np.int32)
    _check(L.cm_tessellate(C.byref(cn), int(res), v.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p),
                           C.byref(nv), C.byref(nf)), "cm_tessellate")
    return v, f


def _check(rc, what):
    if rc != 0:
        raise CMError("%s failed (%d): %s" % (what, rc, lib().cm_last_error().decode()))


def launch_count() -> int:
    return int(lib().cm_launch_count())


def _pack_node(n: dict) -> cm_node:
    c = cm_node()
    c.type = NODE_TYPES[n["type"]]
    ch = list(n["children"])
    c.n_children = len(ch)
    for k, v in enumerate(ch):
        c.children[k] = v
    planes = n["planes"]
    c.n_planes = len(planes)
    for k, v in enumerate(n["pose"]):
        c.pose[k] = v
    for e in range(2):
        for k in range(2):
            c.eps[e][k] = n["eps"][e][k]
        for k in range(3):
            c.a[e][k] = n["a"][e][k]
    p1 = n["planes1"] if n["planes1"] else planes
    for j, r in enumerate(planes):
        for k in range(4):
            c.planes[0][j][k] = r[k]
    for j, r in enumerate(p1):
        for k in range(4):
            c.planes[1][j][k] = r[k]
    for k in range(9):
        c.ctrl[k] = n["ctrl"][k]
    for k in range(3):
        c.up[k] = n["up"][k]
    return c


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


class Scene:
    """Immutable shape library on one device (cm_scene)."""

    def __init__(self, shapes, smooth: dict, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise CMError("CUDA device required: the XPSQ contact library has no CPU path")
        L = lib()
        self.shapes = shapes
        self.device = device
        descs = (cm_shape_desc * len(shapes))()
        self._keep = []
        for s, sh in enumerate(shapes):
            d = descs[s]
            if sh.sdf:
                arr = (cm_node * len(sh.sdf))(*[_pack_node(n) for n in sh.sdf])
                self._keep.append(arr)
                d.n_nodes = len(sh.sdf)
                d.nodes = C.cast(arr, C.POINTER(cm_node))
            if sh.faces is not None and len(sh.faces):
                v = np.ascontiguousarray(sh.vertices, dtype=np.float32)
                f = np.ascontiguousarray(sh.faces, dtype=np.int32)
                self._keep += [v, f]
                d.n_vertices, d.n_faces = len(v), len(f)
                d.vertices = v.ctypes.data_as(C.POINTER(C.c_float))
                d.faces = f.ctypes.data_as(C.POINTER(C.c_int32))
            elif getattr(sh, "sample_res", 0):
                d.sample_res = int(sh.sample_res)   # library-side tessellation (cm_tessellate)
        sp = cm_smooth_params(smooth["tau_cmp"], smooth["tau_min"], smooth["tau_clip_alpha"], smooth["tau_clip_t"],
                              smooth["tau_delta"], int(smooth["trace_iters"]))
        h = C.c_void_p()
        torch.cuda.set_device(device)
        _check(L.cm_scene_create(descs, len(shapes), C.byref(sp), device, C.byref(h)), "cm_scene_create")
        self.h = h
        self._keep = None

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().cm_scene_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def error_count(self, reset: bool = False) -> int:
        """Invalid batch records seen on the device (cm_scene_error_count;
        synchronises)."""
        n = C.c_int64()
        _check(lib().cm_scene_error_count(self.h, C.byref(n), int(reset)), "cm_scene_error_count")
        return n.value

    def counts(self, shape: int):
        V, E, F = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().cm_shape_counts(self.h, shape, C.byref(V), C.byref(E), C.byref(F)), "cm_shape_counts")
        return V.value, E.value, F.value

    def topology(self, shape: int):
        V, E, F = self.counts(shape)
        e = np.zeros((E, 2), np.int32)
        fe = np.zeros((F, 3), np.int32)
        _check(lib().cm_shape_topology(self.h, shape, e.ctypes.data_as(C.c_void_p), fe.ctypes.data_as(C.c_void_p)),
               "cm_shape_topology")
        return e, fe

    # ---- sdf_eval -----------------------------------------------------------
    def sdf_eval(self, shape_ids, poses, points, P: int, flags: int = SDF_VALUE | SDF_GRAD | SDF_HESS, out=None):
        """shape_ids int32 [B], poses float32 [B,8], points float32 [B*P,3]
        (CUDA tensors).  Returns a dict of SoA outputs (field-major)."""
        import torch
        B = shape_ids.shape[0]
        N = B * P
        dev = points.device
        for t in (shape_ids, poses, points):
            if not t.is_cuda or not t.is_contiguous():
                raise CMError("sdf_eval: inputs must be contiguous CUDA tensors")
        assert shape_ids.dtype == torch.int32 and poses.dtype == torch.float32 and points.dtype == torch.float32
        if out is None:
            e = lambda *s: torch.empty(*s, device=dev, dtype=torch.float32)
            out = dict(d=e(N))
            if flags & SDF_GRAD:
                out["grad"] = e(3, N)
            if flags & SDF_HESS:
                out["hess"] = e(6, N)
            if flags & SDF_POSE_GRAD:
                out["dpose"] = e(6, N)
            if flags & SDF_POSE_HESS:
                out["d2pose"] = e(21, N)
                out["dxdpose"] = e(18, N)
        g = lambda k: _ptr(out.get(k))
        _check(lib().cm_sdf_eval(self.h, _ptr(shape_ids), _ptr(poses), _ptr(points), B, P, flags, g("d"), g("grad"),
                                 g("hess"), g("dpose"), g("d2pose"), g("dxdpose"), _stream()), "cm_sdf_eval")
        return out

    # ---- shape-parameter derivatives (f4) -----------------------------------
    def param_layout(self):
        """(counts [n_shapes] int32, offsets [n_shapes + 1] int64) of the
        shape-parameter vectors (-1: not parametrised)."""
        n = len(self.shapes)
        counts = np.zeros(n, np.int32)
        offs = np.zeros(n + 1, np.int64)
        _check(lib().cm_param_layout(self.h, counts.ctypes.data_as(C.c_void_p), offs.ctypes.data_as(C.c_void_p)),
               "cm_param_layout")
        return counts, offs

    def sdf_param_grad(self, shape_ids, poses, points, P: int, pmax: int = 0, w=None, want_J: bool = True):
        """J [pmax, B*P] (d phi / d shape parameter) and, given w [B*P], the
        vector-Jacobian product vjp [n_params_total] (CUDA tensors)."""
        import torch
        counts, offs = self.param_layout()
        pmax = pmax or int(max(counts.max(), 1))
        N = shape_ids.shape[0] * P
        dev = points.device
        J = torch.empty(pmax, N, device=dev, dtype=torch.float32) if want_J else None
        vjp = torch.zeros(int(offs[-1]), device=dev, dtype=torch.float32) if w is not None else None
        _check(lib().cm_sdf_param_grad(self.h, _ptr(shape_ids), _ptr(poses), _ptr(points), shape_ids.shape[0], P,
                                       pmax, _ptr(J), _ptr(w), _ptr(vjp), _stream()), "cm_sdf_param_grad")
        return J, vjp

    # ---- node-pose derivatives (f4, reading #47) ----------------------------
    def node_pose_layout(self):
        """(counts [n_shapes] int32 = 6 x SDF nodes, offsets [n_shapes + 1]
        int64) of the node-pose parameter vectors (-1: not parametrised)."""
        n = len(self.shapes)
        counts = np.zeros(n, np.int32)
        offs = np.zeros(n + 1, np.int64)
        _check(lib().cm_node_pose_layout(self.h, counts.ctypes.data_as(C.c_void_p),
                                         offs.ctypes.data_as(C.c_void_p)), "cm_node_pose_layout")
        return counts, offs

    def sdf_node_pose_grad(self, shape_ids, poses, points, P: int, nmax: int = 0, w=None, want_J: bool = True):
        """J [nmax, B*P] (d phi / d node twist, 6 per node) and, given w
        [B*P], the vector-Jacobian product vjp [total] (CUDA tensors)."""
        import torch
        counts, offs = self.node_pose_layout()
        nmax = nmax or int(max(counts.max(), 1))
        N = shape_ids.shape[0] * P
        dev = points.device
        J = torch.empty(nmax, N, device=dev, dtype=torch.float32) if want_J else None
        vjp = torch.zeros(int(offs[-1]), device=dev, dtype=torch.float32) if w is not None else None
        _check(lib().cm_sdf_node_pose_grad(self.h, _ptr(shape_ids), _ptr(poses), _ptr(points), shape_ids.shape[0],
                                           P, nmax, _ptr(J), _ptr(w), _ptr(vjp), _stream()), "cm_sdf_node_pose_grad")
        return J, vjp

    def manifold_param_vjp(self, pairs, offsets, poses, w_depth, mode: int = 0):
        """vjp [n_params_total] (cm_param_layout order) = sum_rows w_depth
        d depth / d theta of each pair's SDF shape (one-sided modes; CUDA
        tensors in, a new zeroed-then-accumulated CUDA tensor out)."""
        import torch
        _, offs = self.param_layout()
        vjp = torch.zeros(int(offs[-1]), device=poses.device, dtype=torch.float32)
        n_env, n_slot = poses.shape[0], poses.shape[1]
        _check(lib().cm_manifold_param_vjp(self.h, _ptr(pairs), pairs.shape[0], _ptr(offsets), _ptr(poses), n_env,
                                           n_slot, mode, _ptr(w_depth), _ptr(vjp), _stream()),
               "cm_manifold_param_vjp")
        return vjp

    # ---- contact manifold ---------------------------------------------------
    def manifold_size(self, pairs_host: np.ndarray, mode: int = 0) -> int:
        """Contact count of a host pair list for the mode bits (FULL_MODE,
        TWO_SIDED)."""
        pairs_host = np.ascontiguousarray(pairs_host, dtype=np.int32)
        n = C.c_int64()
        _check(lib().cm_manifold_size(self.h, pairs_host.ctypes.data_as(C.c_void_p), len(pairs_host), mode,
                                      C.byref(n)), "cm_manifold_size")
        return n.value

    def manifold_offsets(self, pairs, mode: int = 0):
        """Device exclusive scan of the per-pair contact counts -> int64
        offsets [n_pairs]."""
        import torch
        n = pairs.shape[0]
        offs = torch.empty(n, dtype=torch.int64, device=pairs.device)
        ws_bytes = int(lib().cm_manifold_offsets_workspace(n))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=pairs.device)
        _check(lib().cm_manifold_offsets(self.h, _ptr(pairs), n, mode, _ptr(offs), _ptr(ws), ws_bytes, _stream()),
               "cm_manifold_offsets")
        return offs

    @staticmethod
    def alloc_manifold(C_, tier: int, device):
        import torch
        e = lambda *s: torch.empty(*s, device=device, dtype=torch.float32)
        out = dict(point=e(3, C_), normal=e(3, C_), depth=e(C_), dom=torch.empty(C_, dtype=torch.int8, device=device))
        if tier >= 1:
            out["W"] = e(C_)
            out["q"] = e(3, C_)
        if tier >= 2:
            out["ddepth"] = e(12, C_)
            out["dnormal"] = e(36, C_)
        if tier >= 3:
            out["d2depth"] = e(78, C_)
        return out

    def contact_manifold(self, pairs, offsets, n_contacts: int, poses, tier: int = 2, out=None, mode: int = 0):
        """pairs int32 [NP,5] (env, slotA, slotB, shapeA, shapeB), offsets
        int64 [NP] (manifold_offsets with the same mode), poses float32
        [n_env, n_slot, 8] (CUDA tensors); mode = FULL_MODE | TWO_SIDED bits."""
        for t in (pairs, offsets, poses):
            if not t.is_cuda or not t.is_contiguous():
                raise CMError("contact_manifold: inputs must be contiguous CUDA tensors")
        if out is None:
            out = self.alloc_manifold(n_contacts, tier, poses.device)
        o = cm_manifold_out(*[out[k].data_ptr() if k in out else None
                              for k in ("point", "normal", "depth", "W", "q", "ddepth", "dnormal", "dom", "d2depth")])
        _check(lib().cm_contact_manifold(self.h, _ptr(pairs), pairs.shape[0], _ptr(offsets), _ptr(poses),
                                         poses.shape[0], poses.shape[1], tier | mode, C.byref(o), n_contacts,
                                         _stream()), "cm_contact_manifold")
        return out

    def pair_reduce(self, pairs, offsets, out, n_contacts: int, mode: int = 0, w_depth=None, w_normal=None,
                    want_depth: bool = True, want_W: bool = True):
        """Pair-level reductions (cm_manifold_pair_reduce): pair_depth [NP],
        pair_W [NP] and, given w_depth [C] / w_normal [3, C], the pose VJP
        g_pose [NP, 12]."""
        import torch
        n = pairs.shape[0]
        dev = pairs.device
        pd = torch.empty(n, device=dev, dtype=torch.float32) if want_depth else None
        pw = torch.empty(n, device=dev, dtype=torch.float32) if want_W and "W" in out else None
        gp = torch.empty(n, 12, device=dev, dtype=torch.float32) if (w_depth is not None or w_normal is not None) \
            else None
        o = cm_manifold_out(*[out[k].data_ptr() if k in out else None
                              for k in ("point", "normal", "depth", "W", "q", "ddepth", "dnormal", "dom", "d2depth")])
        _check(lib().cm_manifold_pair_reduce(self.h, _ptr(pairs), n, _ptr(offsets), mode, C.byref(o), n_contacts,
                                             _ptr(w_depth), _ptr(w_normal), _ptr(pd), _ptr(pw), _ptr(gp), _stream()),
               "cm_manifold_pair_reduce")
        return pd, pw, gp

    def expand_jacobian(self, pairs, offsets, poses, W, q, n_contacts: int, mode: int = 0):
        import torch
        J = torch.empty(36, n_contacts, device=poses.device, dtype=torch.float32)
        _check(lib().cm_expand_jacobian(self.h, _ptr(pairs), pairs.shape[0], _ptr(offsets), _ptr(poses),
                                        poses.shape[0], poses.shape[1], mode, _ptr(W), _ptr(q), n_contacts, _ptr(J),
                                        _stream()), "cm_expand_jacobian")
        return J


def sdf_eval(scene: Scene, shape_ids, poses, points, P: int, flags: int = SDF_VALUE | SDF_GRAD | SDF_HESS):
    return scene.sdf_eval(shape_ids, poses, points, P, flags)


def contact_manifold(scene: Scene, pairs, offsets, n_contacts, poses, tier: int = 2, out=None, mode: int = 0):
    return scene.contact_manifold(pairs, offsets, n_contacts, poses, tier, out, mode)
