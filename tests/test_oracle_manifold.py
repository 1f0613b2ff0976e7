"""Pins of the oracle's contact manifold (§II-C):
topology counts, sphere-trace special cases, box-on-plane closed
forms, sphere-sphere candidate depths, the compact contact
Jacobian, finite differences of every derivative output over the pose chart,
rigid-motion invariance, weight partition, smooth-min bounds and sliding
continuity."""
import math

import numpy as np
import pytest

from helpers import scene_of, pose8, perturb, rand_pose, skew
from paper_2604_17538_b200 import synth

TAU_CMP, TAU_MIN, TAU_CLIP = 1e-3, 1e-2, 1e-3


def _sig(x):
    return 1.0 / (1.0 + math.exp(-x)) if x >= 0 else math.exp(x) / (1.0 + math.exp(x))


def _sp(x, t):
    return x + t * math.log1p(math.exp(-x / t)) if x > 0 else t * math.log1p(math.exp(x / t))


def _manifold(O, shapes, poses, pairs, ell=1.0):
    sc = scene_of(shapes, ell=ell, pairs=pairs, poses=poses)
    osc = O.OracleScene(sc)
    return osc.contact_manifold(), osc


def test_topology_counts(oracle_mod):
    O = oracle_mod
    cube = synth.make_shape("c", None, synth.box_mesh((0.5, 0.5, 0.5), 1))
    tri = synth.make_shape("t", None, (np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32),
                                       np.array([[0, 1, 2]], np.int32)))
    k3 = synth.make_shape("s", None, synth.sq_mesh((1, 1, 1), (1, 1), 3))
    patch = synth.make_shape("p", None, synth.plane_patch(16, 32, 0.4, 0.8))
    box6 = synth.make_shape("b", None, synth.box_mesh((0.1, 0.1, 0.1), 6))
    osc = O.OracleScene(scene_of([cube, tri, k3, patch, box6]))
    assert osc.mesh_counts(0) == (8, 18, 12)
    assert osc.mesh_counts(1) == (3, 3, 1)
    assert osc.mesh_counts(2) == (56, 162, 108)         # SURVEY §8a (C4 link)
    assert osc.mesh_counts(3) == (512, 1441, 930)       # SURVEY §8a (C3 patch)
    assert osc.mesh_counts(4) == (218, 648, 432)        # SURVEY §8a (C2 box)
    for s in range(5):
        V, E, F = osc.mesh_counts(s)
        e, fe = osc.mesh_topology(s)
        faces = [osc.scene.shapes[s].faces][0]
        assert np.all(e[:, 0] < e[:, 1])
        assert len({tuple(x) for x in e}) == E            # unique
        for f in range(F):                                # incidence closure
            vs = faces[f]
            for k in range(3):
                a, b = sorted((vs[k], vs[(k + 1) % 3]))
                assert tuple(e[fe[f, k]]) == (a, b)
        if s in (0, 2, 4):
            assert 2 * E == 3 * F and V - E + F == 2         # closed


def _segment_scene(vI, vII, sphere_r=1.0):
    """A thin triangle whose first edge is (vI, vII), against a sphere SDF at
    the origin."""
    v = np.array([vI, vII, [0.0, 0.0, 10.0]], np.float32)
    tri = synth.make_shape("t", None, (v, np.array([[0, 1, 2]], np.int32)))
    sph = synth.make_shape("s", synth.sq((sphere_r,) * 3, (1, 1)), None)
    poses = np.zeros((1, 2, 8), np.float32)
    poses[0, :, 3] = 1
    return [tri, sph], poses, np.array([[0, 0, 1, 0, 1]], np.int32)


def test_trace_examples(oracle_mod):
    """S:509-511 (offset by y = 0.3 from the sphere centre, where the radial
    SQ distance is degenerate, reading #2): unit sphere, edge
    (-2,.3,0)->(2,.3,0): the two traces are mirror images, so p_e = (0,.3,0)
    and phi = -0.7.  v_I inside at (0,.3,0), v_II = (2,.3,0): v_I does not
    move (gate ~ 0), soft clip moves it inward by tau ln 2, v_II follows the
    3-step sphere-trace recursion computed here with the exact sphere SDF."""
    O = oracle_mod
    shapes, poses, pairs = _segment_scene([-2, 0.3, 0], [2, 0.3, 0])
    out, _ = _manifold(O, shapes, poses, pairs)
    assert out["dcand"][0, 3] == pytest.approx(float(np.float32(0.3)) - 1.0, abs=1e-9)
    shapes, poses, pairs = _segment_scene([0, 0.3, 0], [2, 0.3, 0])
    out, _ = _manifold(O, shapes, poses, pairs)
    y = float(np.float32(0.3))
    phi = lambda x: math.hypot(x, y) - 1.0
    be = 2.0
    for _ in range(3):
        p = phi(be)
        be = be - _sig(p / TAU_CMP) * p
    clip = lambda x: _sp(x, TAU_CLIP) - _sp(x - 2.0, TAU_CLIP)
    al = 0.0 + _sig(phi(0.0) / TAU_CMP) * phi(0.0)
    assert abs(al) < 1e-300
    ab = 0.5 * (clip(0.0) + clip(be))
    assert clip(0.0) == pytest.approx(TAU_CLIP * math.log(2.0), rel=1e-12)
    assert out["dcand"][0, 3] == pytest.approx(phi(ab), abs=1e-9)
    # edge entirely outside: phi(p_e) > 0
    shapes, poses, pairs = _segment_scene([-2, 0, 3], [2, 0, 3])
    out, _ = _manifold(O, shapes, poses, pairs)
    assert out["dcand"][0, 3] > 0


def _trace_halfspace(phi0, c, L, iters=3):
    """Exact scalar recursion on a half-space: phi(alpha) = phi0 - c alpha."""
    G = lambda p: _sig(p / TAU_CMP) * p
    al = 0.0
    for _ in range(iters):
        al = al + G(phi0 - c * al)
    return al


def _box_on_plane(O, delta, tilt=0.0, yaw=0.3, s=2):
    box = synth.make_shape("b", None, synth.box_mesh((0.1, 0.1, 0.1), s))
    ground = synth.make_shape("g", synth.halfspace((0, 0, 1), 0.0), None)
    q = synth.quat_mul(synth.quat_from_axis_angle((1, 0, 0), tilt), synth.quat_from_axis_angle((0, 0, 1), yaw))
    poses = np.zeros((1, 2, 8))
    poses[0, 0] = synth.pose_row((0.01, -0.02, 0.1 - delta), q)
    poses[0, 1] = synth.pose_row((0, 0, 0), (1, 0, 0, 0))
    return _manifold(O, [box, ground], poses, np.array([[0, 0, 1, 0, 1]], np.int32))


@pytest.mark.parametrize("delta", [2e-3, 0.05])
def test_box_on_plane_closed_form(oracle_mod, delta):
    """Polyhedral box flat on z <= 0 with penetration delta:
    every bottom-face candidate has d = -delta, so z = 1/6, W = gamma =
    sigma(delta/tau_cmp), n = W (0,0,1), depth = -delta - tau_min ln 6.
    Vertical-edge midpoints follow the 3-step scalar recursion."""
    O = oracle_mod
    out, osc = _box_on_plane(O, delta)
    # penetration with FP32-rounded inputs (pose z and box half-size)
    d32 = float(np.float32(0.1)) - float(np.float32(0.1 - delta))
    bottom = np.all(np.abs(out["dcand"] + d32) < 1e-12, axis=1)
    assert bottom.sum() == 2 * 2 * 2                   # s = 2: 8 bottom triangles
    gam = _sig(d32 / TAU_CMP)
    assert np.allclose(out["z"][bottom], 1.0 / 6.0, atol=1e-12)
    assert np.allclose(out["W"][bottom], gam, atol=1e-12)
    assert np.allclose(out["normal"][bottom], [0, 0, gam], atol=1e-12)
    assert np.allclose(out["depth"][bottom], -d32 - TAU_MIN * math.log(6.0), atol=1e-7)
    # vertical edges (length 0.1 with s=2): candidate depth from the recursion
    L = 0.1
    # trace from the lower vertex (inside, phi0 = -delta) upwards (c = -1) and
    # from the upper vertex (phi0 = L - delta) downwards along -e_t
    a3 = _trace_halfspace(-d32, -1.0, L)
    b3 = L - _trace_halfspace(L - d32, 1.0, L)
    clip = lambda x: _sp(x, TAU_CLIP) - _sp(x - L, TAU_CLIP)
    abar = 0.5 * (clip(a3) + clip(b3))
    d_mid = -d32 + abar
    found = np.isclose(out["dcand"], d_mid, atol=1e-7) | np.isclose(out["dcand"], L - d32 - abar, atol=1e-7)
    assert found.sum() >= 8
    if delta == 0.05:   # SURVEY App. B asymptote: -delta/2 + tau ln2 / 2
        assert d_mid == pytest.approx(-0.024653, abs=2e-6)


def test_sphere_sphere_candidates(oracle_mod):
    """SQ-sphere tessellation sampled vs an SQ-sphere SDF: every vertex
    candidate depth is |p - c_B| - r_B exactly."""
    O = oracle_mod
    ra, rb = 0.1, 0.15
    A = synth.make_shape("a", None, synth.sq_mesh((ra,) * 3, (1, 1), 3))
    B = synth.make_shape("b", synth.sq((rb,) * 3, (1, 1)), None)
    poses = np.zeros((1, 2, 8))
    poses[0, 0] = synth.pose_row((0.2, 0.05, 0.03), synth.random_quats(np.random.default_rng(1), 1)[0])
    poses[0, 1] = synth.pose_row((0.0, 0.0, 0.0), (1, 0, 0, 0))
    poses = poses.astype(np.float32).astype(np.float64)
    out, osc = _manifold(O, [A, B], poses, np.array([[0, 0, 1, 0, 1]], np.int32))
    Rm = synth.quat_to_mat(poses[0, 0, 3:7])
    vw = A.vertices.astype(np.float64) @ Rm.T + poses[0, 0, :3]
    rb32 = float(np.float32(rb))
    for f, tri in enumerate(A.faces):
        for k in range(3):
            assert out["dcand"][f, k] == pytest.approx(np.linalg.norm(vw[tri[k]]) - rb32, abs=1e-9)


def _random_pair_scene(O, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "sq":
        A = synth.make_shape("a", None, synth.sq_mesh((0.08, 0.06, 0.05), (0.7, 0.9), 2))
        B = synth.make_shape("b", synth.sq((0.1, 0.08, 0.07), (0.5, 0.8)), None)
        ell = 1.0
        dist = 0.14
    elif kind == "blob":
        A = synth.make_shape("a", None, synth.sq_mesh((0.08, 0.06, 0.05), (0.7, 0.9), 2))
        B = synth.make_shape("b", synth.blob18(3, 4), None)
        ell = 1.0
        dist = 0.18
    else:
        A = synth.make_shape("a", None, synth.sq_mesh((0.01, 0.01, 0.025), (0.8, 1.0), 2))
        B = synth.make_shape("b", synth.cup(), None)
        ell = 0.04
        dist = 0.055
    poses = np.zeros((1, 2, 8))
    u = rng.normal(size=3)
    u /= np.linalg.norm(u)
    poses[0, 0] = synth.pose_row(dist * u, synth.random_quats(rng, 1)[0])
    poses[0, 1] = synth.pose_row(rng.uniform(-0.01, 0.01, 3), synth.random_quats(rng, 1)[0])
    return [A, B], poses, ell


@pytest.mark.parametrize("kind,seed", [("sq", 1), ("sq", 2), ("blob", 3), ("cup", 4)])
def test_manifold_derivatives_fd(oracle_mod, kind, seed):
    """ddepth/dq and dnormal/dq (q = world left twists of A then B, reading
    #28) vs central finite differences of the oracle's own values over the
    exp-map chart; plus translation/rotation invariance of depth
    (d/dq_B = -d/dq_A), weight partition, smooth-min bounds and the exact
    compact Jacobian J = [W I, -[q - W tA]x, -W I, [q - W tB]x]."""
    O = oracle_mod
    shapes, poses, ell = _random_pair_scene(O, seed, kind)
    poses = poses.astype(np.float32).astype(np.float64)   # the scene's FP32 inputs
    pairs = np.array([[0, 0, 1, 0, 1]], np.int32)
    base, osc = _manifold(O, shapes, poses, pairs, ell)
    sp = osc.scene.smooth
    # active faces only matter physically, but every face must pass
    h = 1e-6 * ell
    for j in range(12):
        e = np.zeros(6)
        e[j % 6] = h
        pp, pm = poses.copy(), poses.copy()
        slot = j // 6
        pp[0, slot] = perturb(poses[0, slot], e)
        pm[0, slot] = perturb(poses[0, slot], -e)
        op_ = osc.contact_manifold(poses=pp)
        om_ = osc.contact_manifold(poses=pm)
        fd = (op_["depth"] - om_["depth"]) / (2 * h)
        sc_d = np.maximum(1.0, np.abs(base["ddepth"]).max(1))
        assert np.all(np.abs(fd - base["ddepth"][:, j]) <= 1e-5 * sc_d), (j, np.abs(fd - base["ddepth"][:, j]).max())
        fdn = (op_["normal"] - om_["normal"]) / (2 * h)
        sc_n = np.maximum(1.0 / ell, np.abs(base["dnormal"]).max((1, 2)))
        err = np.abs(fdn - base["dnormal"][:, :, j]).max(1)
        assert np.all(err <= 1e-4 * sc_n), (j, err.max())
    # invariance under a common rigid motion of both bodies: a common
    # translation gives d/dt_B = -d/dt_A; a common rotation about the world
    # origin (dtheta_A = dtheta_B = w, dt_X = w x t_X) gives
    # d/dth_A + d/dth_B + t_A x d/dt_A + t_B x d/dt_B = 0
    g = base["ddepth"]
    tol = 1e-9 * np.abs(g).max()
    assert np.allclose(g[:, 6:9], -g[:, 0:3], atol=tol)
    tA, tB = poses[0, 0, :3], poses[0, 1, :3]
    assert np.allclose(g[:, 3:6] + g[:, 9:12] + np.cross(tA, g[:, 0:3]) + np.cross(tB, g[:, 6:9]), 0, atol=tol)
    # weight partition, depth bounds (brute force on the 6 candidates)
    assert np.allclose(base["z"].sum(1), 1.0, atol=1e-12)
    dmin = base["dcand"].min(1)
    assert np.all(base["depth"] <= dmin + 1e-15)
    assert np.all(base["depth"] >= dmin - sp["tau_min"] * math.log(6.0) - 1e-15)
    # dominant candidate = deepest (argmax z*gamma), lowest index on exact ties
    assert np.all(base["dom"] == np.argmin(base["dcand"], axis=1))
    # compact Jacobian equals the literal fused J (App. A.7)
    for c in range(len(base["W"])):
        W, q = base["W"][c], base["q"][c]
        Jc = np.concatenate([W * np.eye(3), -skew(q - W * tA), -W * np.eye(3), skew(q - W * tB)], axis=1)
        assert np.allclose(Jc, base["J"][c], atol=1e-12)


def test_rigid_motion_invariance(oracle_mod):
    """A common rigid motion T of both bodies leaves depth, W, dom unchanged
    and rotates points, normals and q (S:547 equivariance)."""
    O = oracle_mod
    shapes, poses, ell = _random_pair_scene(O, 5, "blob")
    poses = poses.astype(np.float32).astype(np.float64)
    pairs = np.array([[0, 0, 1, 0, 1]], np.int32)
    base, osc = _manifold(O, shapes, poses, pairs)
    rng = np.random.default_rng(6)
    qT = synth.random_quats(rng, 1)[0]
    tT = rng.uniform(-0.5, 0.5, 3)
    RT = synth.quat_to_mat(qT)
    p2 = poses.copy()
    for s in range(2):
        p2[0, s, :3] = RT @ poses[0, s, :3] + tT
        p2[0, s, 3:7] = synth.quat_mul(qT, poses[0, s, 3:7])
    o2 = osc.contact_manifold(poses=p2)
    assert np.allclose(o2["depth"], base["depth"], atol=1e-12)
    assert np.allclose(o2["W"], base["W"], atol=1e-12)
    assert np.array_equal(o2["dom"], base["dom"])
    assert np.allclose(o2["normal"], base["normal"] @ RT.T, atol=1e-10)
    assert np.allclose(o2["point"], base["point"] @ RT.T + tT, atol=1e-12)


def test_sliding_box_stack_continuity(oracle_mod):
    """S:553 / Fig. 4 analog: slide an SQ-box-sampled top over a MESH box...
    here a MESH box over an SQ box: every fused contact point moves <= 50
    delta per step of delta = 1e-3."""
    O = oracle_mod
    top = synth.make_shape("top", None, synth.box_mesh((0.1, 0.1, 0.1), 3))
    base = synth.make_shape("base", synth.sq((0.1, 0.1, 0.1), (0.1, 0.1)), None)
    osc = None
    prev = None
    for k in range(40):
        poses = np.zeros((1, 2, 8))
        poses[0, 0] = synth.pose_row((0.02 + 1e-3 * k, 0.0, 0.2 - 0.004), (1, 0, 0, 0))
        poses[0, 1] = synth.pose_row((0, 0, 0), (1, 0, 0, 0))
        if osc is None:
            sc = scene_of([top, base], pairs=np.array([[0, 0, 1, 0, 1]], np.int32), poses=poses)
            osc = O.OracleScene(sc)
        out = osc.contact_manifold(poses=poses)
        if prev is not None:
            active = out["W"] > 1e-3
            assert np.abs(out["point"] - prev)[active].max() <= 50 * 1e-3
        prev = out["point"]


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_oracle_outputs_finite_on_workloads(oracle_mod, cfg):
    """Every oracle output is finite on seeded samples of the benchmark
    workloads (guards readings #34 and #37: negligible soft-Cardano branches
    and the cancellation-free Cardano evaluation)."""
    O = oracle_mod
    sc = synth.c4_scene(48) if cfg == "C4" else synth.c5_scene(3000)
    osc = O.OracleScene(sc)
    r = osc.contact_manifold(pairs=sc.pairs[:900])
    for k in ("point", "normal", "depth", "W", "q", "ddepth", "dnormal"):
        assert np.isfinite(r[k]).all(), k


def test_full_mode_box_on_plane_and_consistency(oracle_mod):
    """Full mode: V + E rows, vertices first; every row is the
    candidate itself.  Box flat on a plane: bottom vertices have depth
    exactly -delta, W = sigma(delta/tau); each row equals the reduced mode's
    candidate of the same vertex / edge."""
    O = oracle_mod
    delta = 2e-3
    box = synth.make_shape("b", None, synth.box_mesh((0.1, 0.1, 0.1), 2))
    ground = synth.make_shape("g", synth.halfspace((0, 0, 1), 0.0), None)
    poses = np.zeros((1, 2, 8))
    poses[0, 0] = synth.pose_row((0.01, -0.02, 0.1 - delta), synth.quat_from_axis_angle((0, 0, 1), 0.3))
    poses[0, 1] = synth.pose_row((0, 0, 0), (1, 0, 0, 0))
    sc = scene_of([box, ground], pairs=np.array([[0, 0, 1, 0, 1]], np.int32), poses=poses)
    osc = O.OracleScene(sc)
    full = osc.contact_manifold(mode=4)
    red = osc.contact_manifold()
    V, E, F = osc.mesh_counts(0)
    assert len(full["depth"]) == V + E
    assert np.all(full["dom"][:V] == 0) and np.all(full["dom"][V:] == 1)
    d32 = float(np.float32(0.1)) - float(np.float32(0.1 - delta))
    zb = box.vertices[:, 2] < 0
    assert np.allclose(full["depth"][:V][zb], -d32, atol=1e-12)
    assert np.allclose(full["W"][:V][zb], 1.0 / (1.0 + math.exp(-d32 / TAU_CMP)), atol=1e-12)
    assert np.allclose(full["q"], full["W"][:, None] * full["point"], atol=1e-15)
    # consistency with the reduced mode's candidates
    e, fe = osc.mesh_topology(0)
    order = np.lexsort((e[:, 1], e[:, 0]))          # sorted (lo, hi) edge order
    rank = np.empty(E, int)
    rank[order] = np.arange(E)
    for f in range(F):
        for k in range(3):
            assert red["dcand"][f, k] == full["depth"][box.faces[f, k]]
            assert red["dcand"][f, 3 + k] == full["depth"][V + rank[fe[f, k]]]


def test_full_mode_derivatives_fd(oracle_mod):
    """Full-mode d depth/dq and d normal/dq vs central finite differences."""
    O = oracle_mod
    shapes, poses, ell = _random_pair_scene(O, 2, "sq")
    poses = poses.astype(np.float32).astype(np.float64)
    base, osc = _manifold(O, shapes, poses, np.array([[0, 0, 1, 0, 1]], np.int32), ell)
    base = osc.contact_manifold(mode=4)
    h = 1e-6
    for j in range(12):
        e = np.zeros(6)
        e[j % 6] = h
        pp, pm = poses.copy(), poses.copy()
        pp[0, j // 6] = perturb(poses[0, j // 6], e)
        pm[0, j // 6] = perturb(poses[0, j // 6], -e)
        op_, om_ = osc.contact_manifold(poses=pp, mode=4), osc.contact_manifold(poses=pm, mode=4)
        assert np.allclose((op_["depth"] - om_["depth"]) / (2 * h), base["ddepth"][:, j], atol=1e-5)
        assert np.allclose((op_["normal"] - om_["normal"]) / (2 * h), base["dnormal"][:, :, j], atol=1e-4)


def test_two_sided_equals_transposed_pair(oracle_mod):
    """Two-sided: the second half is the one-sided manifold of the
    transposed pair, with its derivative and Jacobian column blocks
    expressed in the pair's (A, B) order (its J rows are v_B - v_A, i.e. the
    negated side-0 formula [I, -[p - tA]x, -I, [p - tB]x])."""
    O = oracle_mod
    sc = synth.c1_scene()
    osc = O.OracleScene(sc)
    pair = sc.pairs[:1]                                  # box (sampled) on ground (SDF)
    two = osc.contact_manifold(pairs=pair, mode=8)
    one = osc.contact_manifold(pairs=pair)
    swp = osc.contact_manifold(pairs=pair[:, [0, 2, 1, 4, 3]])
    n0 = len(one["depth"])
    assert len(two["depth"]) == n0 + len(swp["depth"])
    for k in ("depth", "point", "normal", "W", "q", "dom"):
        assert np.array_equal(two[k][:n0], one[k])
        assert np.allclose(two[k][n0:], swp[k], atol=1e-15)
    perm = np.r_[6:12, 0:6]
    assert np.allclose(two["ddepth"][n0:], swp["ddepth"][:, perm], atol=1e-13)
    assert np.allclose(two["dnormal"][n0:], swp["dnormal"][:, :, perm], atol=1e-11)
    assert np.allclose(two["J"][n0:], swp["J"][:, :, perm], atol=1e-13)
    W, q = two["W"][n0:], two["q"][n0:]
    tA, tB = sc.poses[0, 0, :3].astype(np.float64), sc.poses[0, 1, :3].astype(np.float64)
    for c in range(len(W)):
        Jc = np.concatenate([W[c] * np.eye(3), -skew(q[c] - W[c] * tA), -W[c] * np.eye(3), skew(q[c] - W[c] * tB)], 1)
        assert np.allclose(two["J"][n0 + c], -Jc, atol=1e-12)


def test_two_sided_mirror_symmetry(oracle_mod):
    """Two identical spheres placed symmetrically: the two halves have equal
    depth multisets and opposite normals (SURVEY §8c.3 role swap)."""
    O = oracle_mod
    r = 0.1
    sph = synth.make_shape("s", synth.sq((r, r, r), (1, 1)), synth.sq_mesh((r, r, r), (1, 1), 3))
    poses = np.zeros((1, 2, 8))
    poses[0, 0] = synth.pose_row((-0.095, 0, 0), (1, 0, 0, 0))
    poses[0, 1] = synth.pose_row((0.095, 0, 0), (0, 0, 0, 1))   # rotated 180 deg about z: mirror image
    sc = scene_of([sph], pairs=np.array([[0, 0, 1, 0, 0]], np.int32), poses=poses)
    out = O.OracleScene(sc).contact_manifold(mode=8)
    n = len(out["depth"]) // 2
    assert np.allclose(np.sort(out["depth"][:n]), np.sort(out["depth"][n:]), atol=1e-12)
    assert np.allclose(out["normal"][:n].sum(0), -out["normal"][n:].sum(0), atol=1e-12)


# ---- second-order manifold derivatives -------------------
def _unpack78(h):
    iu = np.triu_indices(12)
    H = np.zeros(h.shape[:-1] + (12, 12))
    H[..., iu[0], iu[1]] = h
    H[..., iu[1], iu[0]] = h
    return H


def _d2_value_fd(osc, poses, mode, h):
    """Second central differences of the oracle's depth VALUES in the
    exp-map chart of each body (one exponential per body, so the chart's
    Hessian is symmetric): independent of the jets."""
    def f(dq):
        pp = poses.copy()
        pp[0, 0] = perturb(poses[0, 0], dq[:6])
        pp[0, 1] = perturb(poses[0, 1], dq[6:])
        return osc.contact_manifold(poses=pp, mode=mode)["depth"]
    iu = np.triu_indices(12)
    cols = []
    for i, j in zip(*iu):
        ei = np.zeros(12); ei[i] = h
        ej = np.zeros(12); ej[j] = h
        cols.append((f(ei + ej) - f(ei - ej) - f(-ei + ej) + f(-ei - ej)) / (4 * h * h))
    return np.stack(cols, 1)


@pytest.mark.parametrize("kind,seed,mode", [("sq", 1, 0), ("cup", 4, 0), ("blob", 3, 0), ("sq", 2, 4)])
def test_manifold_d2depth_fd(oracle_mod, kind, seed, mode):
    """d^2 depth / dq^2 (second-order q-jets through the whole manifold) vs
    second differences of the oracle's depth values (reduced and full mode)."""
    O = oracle_mod
    shapes, poses, ell = _random_pair_scene(O, seed, kind)
    poses = poses.astype(np.float32).astype(np.float64)
    pairs = np.array([[0, 0, 1, 0, 1]], np.int32)
    _, osc = _manifold(O, shapes, poses, pairs, ell)
    H = osc.manifold_d2depth(poses=poses, mode=mode)
    Hfd = _d2_value_fd(osc, poses, mode, 3e-5 * ell)
    scale = np.maximum(1.0 / ell, np.abs(H).max(1))
    err = np.abs(H - Hfd).max(1) / scale
    assert err.max() < 5e-3 and np.median(err) < 1e-4, (err.max(), np.median(err))


def test_manifold_d2depth_gradient_consistency_and_invariance(oracle_mod):
    """C1: the Hessian equals the symmetrised central difference of the
    first-order ddepth (the antisymmetric part of that difference is the
    Baker-Campbell-Hausdorff term of composing two left twists; pair 0, whose
    columns are slots 0 then 1), and on both pairs it inherits translation
    invariance: rows / columns of t_B are minus those of t_A."""
    O = oracle_mod
    sc = synth.c1_scene()
    osc = O.OracleScene(sc)
    poses = sc.poses.astype(np.float64)
    assert tuple(sc.pairs[0, 1:3]) == (0, 1)
    H = _unpack78(osc.manifold_d2depth(poses=poses))
    F0 = osc.mesh_counts(int(sc.pairs[0, 3]))[2]
    rows = np.arange(0, F0, 7)
    h = 1e-5
    cols = []
    for j in range(12):
        e = np.zeros(6); e[j % 6] = h
        pp, pm = poses.copy(), poses.copy()
        pp[0, j // 6] = perturb(poses[0, j // 6], e)
        pm[0, j // 6] = perturb(poses[0, j // 6], -e)
        cols.append((osc.contact_manifold(poses=pp)["ddepth"][rows] - osc.contact_manifold(poses=pm)["ddepth"][rows]) / (2 * h))
    Hfd = np.stack(cols, 2)                       # [row, i, j]
    Hs = 0.5 * (Hfd + np.swapaxes(Hfd, 1, 2))
    scale = np.maximum(1.0, np.abs(H[rows]).max((1, 2)))
    assert np.all(np.abs(H[rows] - Hs).max((1, 2)) <= 1e-3 * scale)
    tol = 1e-9 * np.abs(H).max()
    tA, tB = slice(0, 3), slice(6, 9)
    assert np.allclose(H[:, tB, 3:6], -H[:, tA, 3:6], atol=tol)
    assert np.allclose(H[:, tB, 9:12], -H[:, tA, 9:12], atol=tol)
    assert np.allclose(H[:, tB, tB], H[:, tA, tA], atol=tol)
    assert np.allclose(H[:, tA, tB], -H[:, tA, tA], atol=tol)


def test_manifold_d2depth_two_sided(oracle_mod):
    """Two-sided rows: the first half equals the one-sided Hessian; the second
    half equals the transposed pair's Hessian with the body blocks swapped."""
    O = oracle_mod
    sc = synth.c1_scene()
    osc = O.OracleScene(sc)
    pr = sc.pairs[:1]
    one = osc.manifold_d2depth(pairs=pr)
    two = osc.manifold_d2depth(pairs=pr, mode=8)
    n = len(one)
    assert np.allclose(two[:n], one, rtol=0, atol=1e-12 * np.abs(one).max())
    trp = pr[:, [0, 2, 1, 4, 3]]
    Ht = _unpack78(osc.manifold_d2depth(pairs=trp))
    perm = np.r_[6:12, 0:6]
    Hs = Ht[:, perm][:, :, perm]
    H2 = _unpack78(two[n:])
    assert np.allclose(H2, Hs, rtol=0, atol=1e-12 * np.abs(Hs).max())


def test_pair_reduce_pins(oracle_mod):
    """Pair-level reductions: pair_depth lies in the LSE
    sandwich [min d - tau ln n, min d]; pair_W = sum W; the pose VJP equals
    the central finite difference of sum(w_depth depth + w_normal . normal)
    over the world-frame twist chart of both bodies."""
    import numpy as np
    from helpers import perturb
    from paper_2604_17538_b200 import synth
    O = oracle_mod
    sc = synth.c4_scene(2)
    osc = O.OracleScene(sc)
    pairs = sc.pairs[:6]
    out = osc.contact_manifold(pairs=pairs)
    tau = sc.smooth["tau_min"]
    rng = np.random.default_rng(5)
    wd = rng.normal(size=out["depth"].shape)
    wn = rng.normal(size=out["normal"].shape)
    pd, pw, gp = O.OracleScene.pair_reduce(out, tau, wd, wn)
    off = out["offsets"]
    for i in range(len(pairs)):
        d = out["depth"][off[i]:off[i + 1]]
        assert d.min() - tau * np.log(len(d)) - 1e-12 <= pd[i] <= d.min() + 1e-12
        assert pw[i] == np.sum(out["W"][off[i]:off[i + 1]])
    h = 1e-6
    for i in (0, 3):
        env, sa, sb = pairs[i, 0], pairs[i, 1], pairs[i, 2]
        r = slice(off[i], off[i + 1])
        for j in range(12):
            dq = np.zeros(6)
            dq[j % 6] = h
            vals = []
            for sgn in (1, -1):
                poses = sc.poses.astype(np.float64).copy()
                slot = sa if j < 6 else sb
                poses[env, slot] = perturb(poses[env, slot], sgn * dq)
                o2 = osc.contact_manifold(pairs=pairs[i:i + 1], poses=poses)
                vals.append(np.sum(wd[r] * o2["depth"]) + np.sum(wn[r] * o2["normal"]))
            fd = (vals[0] - vals[1]) / (2 * h)
            assert abs(fd - gp[i, j]) <= 1e-4 * max(1.0, abs(gp[i, j])), (i, j, fd, gp[i, j])
