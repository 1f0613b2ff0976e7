"""The C-ABI library loads on a CPU-only host and exports every function
include/xpsq_cm.h declares; argument validation runs before any CUDA call
(no compute without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            src = open(os.path.join(ROOT, "include", f)).read()
            names |= set(re.findall(r"^(?:int|int64_t|const char\*)\s+(cm_\w+)\(", src, re.M))
    return names


@pytest.fixture(scope="module")
def L():
    from paper_2604_17538_b200 import build, binding
    build.build()
    return binding.lib()


def test_exports_every_declared_symbol(L):
    from paper_2604_17538_b200 import binding
    decl = _declared()
    assert len(decl) >= 12
    assert decl == set(binding.EXPORTS)
    for n in decl:
        assert getattr(L, n) is not None


def test_version_and_launch_counter(L):
    assert L.cm_version() == 6   # 3: error count; 4: node-pose derivatives; 5: manifold parameter VJP; 6: sample_res
    # no launch happens at load (a process that already ran GPU tests counts those)
    n = L.cm_launch_count()
    assert n >= 0


def test_struct_layout(L):
    from paper_2604_17538_b200 import binding
    # 4 + 4 + 32*4 + 4 + 7*4 + 4*4 + 6*4 + 64*4 + 9*4 + 3*4
    assert C.sizeof(binding.cm_node) == 4 + 4 + 128 + 4 + 28 + 16 + 24 + 256 + 36 + 12
    assert C.sizeof(binding.cm_smooth_params) == 24
    assert C.sizeof(binding.cm_manifold_out) == 9 * 8


def _desc(nodes):
    from paper_2604_17538_b200 import binding
    arr = (binding.cm_node * len(nodes))(*[binding._pack_node(n) for n in nodes])
    d = binding.cm_shape_desc()
    d.n_nodes = len(nodes)
    d.nodes = C.cast(arr, C.POINTER(binding.cm_node))
    return d, arr


def _create(L, nodes, **sp):
    from paper_2604_17538_b200 import binding, synth
    d, keep = _desc(nodes)
    p = dict(synth.DEFAULT_SMOOTH)
    p.update(sp)
    s = binding.cm_smooth_params(p["tau_cmp"], p["tau_min"], p["tau_clip_alpha"], p["tau_clip_t"], p["tau_delta"],
                                 p["trace_iters"])
    h = C.c_void_p()
    rc = L.cm_scene_create(C.byref(d), 1, C.byref(s), 0, C.byref(h))
    return rc, L.cm_last_error().decode()


def test_validation_errors(L):
    from paper_2604_17538_b200 import synth
    sq = synth.flatten(synth.sq((0.1, 0.1, 0.1), (0.5, 0.5)))
    rc, msg = _create(L, sq, tau_min=0.0)
    assert rc == -1 and "tau" in msg                                   # S:28 / S:603
    bad = synth.flatten(synth.sq((0.1, 0.1, 0.1), (0.05, 0.5)))
    rc, msg = _create(L, bad)
    assert rc == -1 and "eps" in msg
    nf = synth.flatten(synth.sq((0.1, float("nan"), 0.1), (0.5, 0.5)))
    rc, msg = _create(L, nf)
    assert rc == -2
    sub = synth.flatten(synth.op("subtraction", [synth.sq((0.1,) * 3, (1, 1))] * 3))
    rc, msg = _create(L, sub)
    assert rc == -4                                                    # S:184 arity
    deep = synth.sq((0.1,) * 3, (1, 1))
    for _ in range(4):
        deep = synth.op("union", [deep, synth.sq((0.1,) * 3, (1, 1))])
    rc, msg = _create(L, synth.flatten(deep))
    assert rc == -3 and "DEPTH" in msg
    hs = synth.flatten(synth.halfspace((0, 0, 1), 0.0))
    hs[0]["planes"][0][2] = 2.0
    rc, msg = _create(L, hs)
    assert rc == -1 and "unit" in msg


def test_binding_refuses_without_cuda():
    import torch
    from paper_2604_17538_b200 import binding, synth
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(binding.CMError):
        binding.Scene([synth.make_shape("s", synth.sq((0.1,) * 3, (1, 1)))], synth.smooth_params())
