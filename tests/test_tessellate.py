"""Library-side sampled surfaces (SURVEY §8(b) `sample_res`; P:131 samples
the surface of one shape): cm_tessellate against the Python synthetic
generators (same topology, vertices within FP32 rounding), closed 2-manifold
topology (every edge on exactly two faces, Euler V - E + F = 2), and the
vertices on the analytic surfaces: SQ vertices are zeros of the FP64
oracle's radial SQ distance (Eq. (1)); PSQ vertices lie on the SQ or on a
plane and inside every plane.  Host-only calls (no GPU)."""
import numpy as np
import pytest

from paper_2604_17538_b200 import synth

binding = pytest.importorskip("paper_2604_17538_b200.binding")


@pytest.fixture(scope="module")
def lib():
    try:
        return binding.lib()
    except binding.CMError as e:
        pytest.skip(str(e))


def _closed(v, f):
    e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    return (cnt == 2).all() and len(v) - len(cnt) + len(f) == 2


@pytest.mark.parametrize("a,eps,k", [((0.2, 0.15, 0.1), (0.3, 0.7), 3), ((0.05, 0.05, 0.05), (1.0, 1.0), 4),
                                     ((0.3, 0.1, 0.2), (1.8, 0.2), 2)])
def test_sq_surface(lib, oracle_mod, a, eps, k):
    v, f = binding.tessellate(synth.flatten(synth.sq(a, eps))[0], k)
    v2, f2 = synth.sq_mesh(a, eps, k)
    assert v.shape == (6 * k * k + 2, 3) and f.shape == (12 * k * k, 3)
    assert np.array_equal(f, f2) and np.allclose(v, v2, atol=1e-7)
    assert _closed(v, f)
    phi = np.array([oracle_mod.sq_phi(x.astype(np.float64), eps, a) for x in v])
    assert np.abs(phi).max() < 1e-6 * max(a)


def test_psq_surface(lib, oracle_mod):
    a, eps = (0.2, 0.15, 0.1), (0.5, 0.8)
    planes = [[0.3, 0.2, 0.93, -0.05], [-0.6, 0.1, -0.79, -0.08]]
    v, f = binding.tessellate(synth.flatten(synth.psq(a, eps, planes))[0], 3)
    v2, f2 = synth.psq_mesh(a, eps, planes, 3)
    assert np.array_equal(f, f2) and np.allclose(v, v2, atol=1e-7) and _closed(v, f)
    pl = np.asarray(planes, dtype=np.float64)
    pl[:, :3] /= np.linalg.norm(pl[:, :3], axis=1, keepdims=True)
    s = v.astype(np.float64) @ pl[:, :3].T + pl[:, 3]
    assert (s <= 1e-6).all()                                      # inside every plane
    phi = np.array([oracle_mod.sq_phi(x.astype(np.float64), eps, a) for x in v])
    on_sq, on_plane = np.abs(phi) < 1e-6, (np.abs(s) < 1e-6).any(axis=1)
    assert (on_sq | on_plane).all() and on_plane.any() and on_sq.any()


def test_xpsq_tube(lib):
    ctrl = [-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02]
    v, f = binding.tessellate(synth.flatten(synth.xpsq(ctrl, (0.12, 0.15, 0.1), (0.6, 0.8)))[0], 3)
    v2, f2 = synth.xpsq_mesh(ctrl, (0.12, 0.15, 0.1), 0.8, 7, 12)
    assert np.array_equal(f, f2) and np.allclose(v, v2, atol=1e-7) and _closed(v, f)
    # a straight spline takes its frame from the up hint
    line = synth.xpsq([-0.2, 0, 0, 0.0, 0, 0, 0.2, 0, 0], (0.05, 0.05, 0.03), (0.6, 0.8), up=(0, 0, 1))
    vl, fl = binding.tessellate(synth.flatten(line)[0], 2)
    assert _closed(vl, fl)
    ring = vl[:8]                                                 # the t = 0 ring: in the x = -0.2 plane
    assert np.allclose(ring[:, 0], -0.2, atol=1e-7) and np.allclose(np.abs(ring[:, 2]).max(), 0.03, atol=1e-7)


def test_tessellate_errors(lib):
    with pytest.raises(binding.CMError):
        binding.tessellate(synth.flatten(synth.halfspace((0, 0, 1), 0.0))[0], 3)
    with pytest.raises(binding.CMError):
        binding.tessellate(synth.flatten(synth.sq((0.1, 0.1, 0.1), (1, 1)))[0], 0)
    with pytest.raises(binding.CMError):   # a point spline has no tube
        binding.tessellate(synth.flatten(synth.xpsq([0.01, 0, 0] * 3, (0.1, 0.1, 0.1), (1, 1)))[0], 2)
