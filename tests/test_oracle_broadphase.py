"""Pins of the oracle's broad phase (DESIGN.md
reading #46): the SDF lower bounds hold at sampled points of every C5 SDF
prototype and C3's 18-SQ union (phi(x) >= |x - c| - rho), every sampled
vertex lies in its mesh sphere, and against the all-edges manifold: kept
pairs are identical, culled pairs have every gate below e^-40 and every
candidate depth above the certified bound."""
import math

import numpy as np

from helpers import scene_of, pose8
from paper_2604_17538_b200 import synth


def test_sdf_lower_bounds_hold(oracle_mod):
    O = oracle_mod
    sampled, sdf = synth.c5_library()
    shapes = sdf + [synth.make_shape("blob18", synth.blob18(3, 18)), synth.make_shape("cup", synth.cup())]
    osc = O.OracleScene(scene_of(shapes, ell=0.1))
    rng = np.random.default_rng(31)
    n_bounded = 0
    for s in range(len(shapes)):
        c, rho = osc.shape_bound(s)
        if not np.isfinite(rho):
            continue
        n_bounded += 1
        # points on shells around the bound sphere, from inside it to far outside
        u = rng.normal(size=(400, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        r = rng.uniform(0.0, 3.0, 400) * rho
        pts = c + u * r[:, None]
        d = osc.sdf_eval(np.array([s]), pose8().reshape(1, 8), pts, len(pts), want_pose=False)["d"]
        lb = np.linalg.norm(pts - c, axis=1) - rho
        assert (d >= lb - 1e-12).all(), (shapes[s].name, float((lb - d).max()))
    assert n_bounded == len(shapes)


def test_mesh_spheres_contain_vertices(oracle_mod):
    O = oracle_mod
    sampled, _ = synth.c5_library()
    osc = O.OracleScene(scene_of(sampled, ell=0.1))
    for s, sh in enumerate(sampled):
        c, r = osc.mesh_sphere(s)
        v = sh.vertices.astype(np.float64)
        assert (np.linalg.norm(v - c, axis=1) <= r + 1e-12).all()


def test_broad_phase_against_all_edges(oracle_mod):
    """C5-like pairs spread from touching to far apart (clearance scaled up):
    broad (mode 16) equals all-edges (mode 0) on kept pairs; on culled pairs
    the all-edges gates are all < e^-40, the candidate depths >= lb and the
    fused depth >= the reported bound lb - tau_min ln 6."""
    O = oracle_mod
    sc = synth.c5_scene(300)
    # push every other env apart along its offset direction
    poses = sc.poses.astype(np.float64).copy()
    far = np.arange(len(poses)) % 2 == 1
    poses[far, 0, :3] *= 3.0
    osc = O.OracleScene(sc)
    pairs = sc.pairs
    a = osc.contact_manifold(pairs=pairs, poses=poses, mode=0)
    b = osc.contact_manifold(pairs=pairs, poses=poses, mode=16)
    tau_cmp, tau_min = sc.smooth["tau_cmp"], sc.smooth["tau_min"]
    off = a["offsets"]
    n_cull = 0
    for i in range(len(pairs)):
        r = slice(off[i], off[i + 1])
        if (b["dom"][r] == -2).all():
            n_cull += 1
            lb = b["dcand"][r][0, 0]
            assert lb > 40 * tau_cmp
            assert (a["gamma"][r] < math.exp(-40)).all()
            assert (a["dcand"][r] >= lb - 1e-12).all()
            assert (a["depth"][r] >= b["depth"][r] - 1e-12).all()
            assert (b["W"][r] == 0).all() and (b["ddepth"][r] == 0).all()
        else:
            assert not (b["dom"][r] == -2).any()
            for k in ("point", "normal", "depth", "W", "q", "ddepth", "dnormal", "dom"):
                assert np.array_equal(a[k][r], b[k][r]), (i, k)
    assert 40 < n_cull < len(pairs) - 40, n_cull
