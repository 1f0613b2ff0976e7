"""GPU parity of the CUDA path (called through the C ABI) against the FP64
oracle on the same seeded inputs.  Needs a B200."""
import json
import math
import os

import numpy as np
import pytest

from helpers import scene_of, pose8
from paper_2604_17538_b200 import synth
import parity as PT

pytestmark = pytest.mark.gpu

ALL = 1 | 2 | 4 | 8 | 16


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_17538_b200 import binding
    binding.lib()
    return torch


def _report(name, rep):
    os.makedirs(os.path.join(os.path.dirname(__file__), "..", "gpurun_out"), exist_ok=True)
    with open(os.path.join(os.path.dirname(__file__), "..", "gpurun_out", "parity_%s.json" % name), "w") as f:
        json.dump(rep, f, indent=1)


def _sdf_shapes():
    rng = np.random.default_rng(5)
    return [
        ("sq", synth.sq((0.3, 0.2, 0.25), (0.6, 0.9))),
        ("sq_box01", synth.sq((0.1, 0.1, 0.1), (0.1, 0.1))),
        ("sq_eps2", synth.sq((0.2, 0.15, 0.1), (1.9, 2.0), pose=[0.05, -0.02, 0.01, *synth.random_quats(rng, 1)[0]])),
        ("psq", synth.psq((0.3, 0.3, 0.2), (0.8, 0.5), [[0, 0, 1, -0.05], [1, 1, 0, -0.1]])),
        ("halfspace", synth.halfspace((0.2, 0.3, 1.0), 0.05)),
        ("blob6", synth.blob18(3, 6)),
        ("blob18", synth.blob18(3, 18)),
        ("cup", synth.cup()),
        ("xpsq_vary", synth.xpsq(ctrl=[-0.1, 0, 0, 0.05, 0.12, 0.02, 0.15, -0.03, 0.05], a0=(0.05, 0.04, 0.03),
                                 eps0=(0.5, 0.8), a1=(0.03, 0.05, 0.04), eps1=(0.9, 0.4),
                                 planes0=[[0, 0, 1, -0.01]], planes1=[[0, 1, 1, -0.005]])),
        ("xpsq_line", synth.xpsq(ctrl=[-0.2, 0, 0, 0.0, 0.05, 0, 0.2, 0.1, 0], a0=(0.05, 0.05, 0.05), eps0=(1, 1))),
        ("xpsq_point", synth.xpsq(ctrl=[0.02, 0.01, 0.0] * 3, a0=(0.08, 0.05, 0.06), eps0=(0.6, 0.7),
                                  planes0=[[0, 0, 1, -0.02]])),
        # nearly straight curved splines (|A|/|B| = 1e-3, 5e-3): the literal
        # cubic (reading #14), Newton-polished in t on the GPU
        ("xpsq_near3", synth.xpsq(ctrl=_near_straight(1e-3), a0=(0.05, 0.04, 0.06), eps0=(0.4, 0.7),
                                  planes0=[[0, 0, 1, -0.02]])),
        ("xpsq_near2", synth.xpsq(ctrl=_near_straight(5e-3), a0=(0.06, 0.06, 0.06), eps0=(1.0, 1.0))),
    ]


def _near_straight(ratio):
    p1 = np.array([-0.2, 0.03, -0.01])
    B = np.array([0.4, 0.1, 0.05])
    A = np.cross(B, [0.2, -0.4, 1.0])
    A *= ratio * np.linalg.norm(B) / np.linalg.norm(A)
    p2 = p1 + B / 2
    return list(np.concatenate([p1, p2, A + 2 * p2 - p1]))


@pytest.mark.parametrize("k", range(13))
def test_sdf_eval_parity(cuda, oracle_mod, k):
    """Every primitive family, all outputs (value, gradient, Hessian, pose
    gradient, pose Hessian, mixed), random poses, points spanning inside,
    surface band and outside; B = 7 items x P = 333 points (ragged)."""
    from paper_2604_17538_b200 import binding
    name, root = _sdf_shapes()[k]
    ell = 0.04 if name == "cup" else 1.0
    sc = scene_of([synth.make_shape(name, root)], ell=ell)
    osc = oracle_mod.OracleScene(sc)
    S = binding.Scene(sc.shapes, sc.smooth)
    rng = np.random.default_rng(100 + k)
    B, P = 7, 333
    poses = np.stack([pose8(rng.uniform(-0.1, 0.1, 3), synth.random_quats(rng, 1)[0]) for _ in range(B)]).astype(np.float32)
    scale = 0.1 if name == "cup" else 0.45
    loc = rng.uniform(-scale, scale, (B, P, 3))
    pts = np.concatenate([loc[b] @ synth.quat_to_mat(poses[b, 3:7]).T + poses[b, :3] for b in range(B)]).astype(np.float32)
    ids = np.zeros(B, np.int32)
    gpu = PT.gpu_sdf(S, ids, poses, pts, P, ALL)
    nf, rep = PT.sdf_parity(osc, gpu, ids, poses, pts, P, rng, ell)
    _report("sdf_" + name, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01, rep
    # value-only and gradient-only instantiations agree with the full one
    # (nearly straight splines: the instantiations' Newton-polished roots may
    # differ by an ulp of t, which moves y by |p'| ulp(t); near the tube's
    # axis the sphere-section gradient y/|y| turns by that over |y|, so the
    # gradient check there uses the parity tolerance 1e-4)
    g0 = PT.gpu_sdf(S, ids, poses, pts, P, 1)
    g1 = PT.gpu_sdf(S, ids, poses, pts, P, 1 | 2)
    gtol = 1e-4 if name.startswith("xpsq_near") else 1e-5
    assert np.allclose(g0["d"], gpu["d"], atol=1e-6 * ell) and np.allclose(g1["grad"], gpu["grad"], atol=gtol)


def test_sdf_eval_mixed_batch(cuda, oracle_mod):
    """A batch mixing every shape (lean and XPSQ instantiations in one call)."""
    from paper_2604_17538_b200 import binding
    shapes = [synth.make_shape(n, r) for n, r in _sdf_shapes() if n != "cup"]
    sc = scene_of(shapes)
    osc = oracle_mod.OracleScene(sc)
    S = binding.Scene(sc.shapes, sc.smooth)
    rng = np.random.default_rng(7)
    B, P = 40, 37
    ids = rng.integers(0, len(shapes), B).astype(np.int32)
    poses = np.stack([pose8(rng.uniform(-0.1, 0.1, 3), synth.random_quats(rng, 1)[0]) for _ in range(B)]).astype(np.float32)
    pts = rng.uniform(-0.5, 0.5, (B * P, 3)).astype(np.float32)
    gpu = PT.gpu_sdf(S, ids, poses, pts, P, ALL)
    nf, rep = PT.sdf_parity(osc, gpu, ids, poses, pts, P, rng, 1.0)
    _report("sdf_mixed", rep)
    assert nf == 0, json.dumps(rep, indent=1)


def test_sdf_eval_side_stream_join(cuda):
    """A multi-class scene forks its class kernels onto the scene's streams
    and joins them back into the caller's stream: work queued on a side
    stream after the call sees every output (NaN-prefilled buffers, a large
    batch so the class kernels overlap), bit-identical to a default-stream
    call."""
    import torch
    from paper_2604_17538_b200 import binding
    shapes = [synth.make_shape(n, r) for n, r in _sdf_shapes() if n != "cup"]
    sc = scene_of(shapes)
    S = binding.Scene(sc.shapes, sc.smooth)
    rng = np.random.default_rng(17)
    B, P = 4096, 64
    ids = torch.from_numpy(rng.integers(0, len(shapes), B).astype(np.int32)).cuda()
    poses = torch.from_numpy(np.stack([pose8(rng.uniform(-0.1, 0.1, 3), synth.random_quats(rng, 1)[0])
                                       for _ in range(B)]).astype(np.float32)).cuda()
    pts = torch.from_numpy(rng.uniform(-0.5, 0.5, (B * P, 3)).astype(np.float32)).cuda()
    flags = binding.SDF_VALUE | binding.SDF_GRAD | binding.SDF_HESS
    ref = S.sdf_eval(ids, poses, pts, P, flags)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        out = {k: torch.full_like(v, float("nan")) for k, v in ref.items()}
        S.sdf_eval(ids, poses, pts, P, flags, out=out)
        seen = {k: v.clone() for k, v in out.items()}   # queued behind the join on `side`
    side.synchronize()
    for k in ref:
        assert torch.equal(seen[k], ref[k]), k


def test_sdf_eval_c1(cuda, oracle_mod):
    from paper_2604_17538_b200 import binding
    sc = synth.c1_scene()
    osc = oracle_mod.OracleScene(sc)
    S = binding.Scene(sc.shapes, sc.smooth)
    gpu = PT.gpu_sdf(S, sc.point_shapes, sc.point_poses, sc.points, sc.P, ALL)
    nf, rep = PT.sdf_parity(osc, gpu, sc.point_shapes, sc.point_poses, sc.points, sc.P, np.random.default_rng(0), 1.0)
    _report("sdf_c1", rep)
    assert nf == 0, json.dumps(rep, indent=1)


@pytest.mark.parametrize("tier", [0, 1, 2])
def test_manifold_c1(cuda, oracle_mod, tier):
    sc = synth.c1_scene()
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, tier)
    nf, rep = PT.manifold_parity(sc, osc, gpu, tier, np.arange(len(sc.pairs)), np.random.default_rng(1), sc.ell)
    _report("manifold_c1_t%d" % tier, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_c2(cuda, oracle_mod):
    """C2 at full size (1k envs, box on box, the pathological parallel-face
    case): every pair compared."""
    sc = synth.c2_scene(1000)
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, 2)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, np.arange(len(sc.pairs)), np.random.default_rng(2), sc.ell)
    _report("manifold_c2", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_c3_sampled(cuda, oracle_mod):
    """C3 at its BASELINE.json size (16k envs, 16x32 patch vs 18-SQ union),
    in bench.py's launch configuration; oracle on a seeded sample of 256
    pairs."""
    sc = synth.c3_scene(16384)
    osc = oracle_mod.OracleScene(sc)
    idx = np.sort(np.random.default_rng(3).choice(len(sc.pairs), 256, replace=False))
    gpu = PT.gpu_manifold_sampled(sc, idx, 2)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, idx, np.random.default_rng(4), sc.ell)
    _report("manifold_c3", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_c4_sampled(cuda, oracle_mod):
    """C4 (20 SQ links vs the cup with its XPSQ handle, ell = 0.04): GPU on
    512 envs x 20 pairs, oracle on a seeded sample of 256 pairs."""
    sc = synth.c4_scene(512)
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, 2)
    idx = np.random.default_rng(5).choice(len(sc.pairs), 256, replace=False)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, np.sort(idx), np.random.default_rng(6), sc.ell)
    _report("manifold_c4", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_edge_cases(cuda, oracle_mod):
    """Empty pair list, a single-triangle mesh, far-apart bodies (all gates
    closed) and tier-dependent NULL outputs."""
    import torch
    from paper_2604_17538_b200 import binding
    # (no vertex at the sphere centre: the radial SQ distance is not
    # differentiable there, reading #2)
    tri = synth.make_shape("tri", None, (np.array([[0.01, 0.02, 0.005], [0.1, 0, 0], [0, 0.1, 0]], np.float32),
                                         np.array([[0, 1, 2]], np.int32)))
    sph = synth.make_shape("sph", synth.sq((0.05,) * 3, (1, 1)), None)
    poses = np.zeros((2, 2, 8), np.float32)
    poses[:, :, 3] = 1
    poses[1, 1, :3] = (5.0, 5.0, 5.0)
    pairs = np.array([[0, 0, 1, 0, 1], [1, 0, 1, 0, 1]], np.int32)
    sc = scene_of([tri, sph], pairs=pairs, poses=poses)
    osc = oracle_mod.OracleScene(sc)
    gpu, S = PT.gpu_manifold(sc, 2)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, np.arange(2), np.random.default_rng(7), 1.0)
    assert nf == 0, rep
    assert gpu["W"][1] < 1e-6
    # empty batch: no launch, no error
    out = S.contact_manifold(torch.zeros((0, 5), dtype=torch.int32, device="cuda"),
                             torch.zeros(0, dtype=torch.int64, device="cuda"), 0,
                             torch.from_numpy(poses).cuda(), 2)
    torch.cuda.synchronize()
    assert out["depth"].numel() == 0


def test_topology_matches_oracle(cuda, oracle_mod):
    """Library-built topology equals the oracle's (as sets: edge ids may be
    numbered differently; face_edges must name the same vertex pairs)."""
    from paper_2604_17538_b200 import binding
    for sc in (synth.c1_scene(), synth.c2_scene(4)):
        osc = oracle_mod.OracleScene(sc)
        S = binding.Scene(sc.shapes, sc.smooth)
        for s, sh in enumerate(sc.shapes):
            if sh.faces is None:
                continue
            assert S.counts(s) == osc.mesh_counts(s)
            e1, fe1 = S.topology(s)
            e2, fe2 = osc.mesh_topology(s)
            assert {tuple(x) for x in e1} == {tuple(x) for x in e2}
            assert np.array_equal(e1[fe1], e2[fe2])


def test_expand_jacobian(cuda, oracle_mod):
    """cm_expand_jacobian reproduces the oracle's literal sum z_i gamma_i J_i."""
    import torch
    sc = synth.c1_scene()
    osc = oracle_mod.OracleScene(sc)
    gpu, S = PT.gpu_manifold(sc, 1)
    pairs_t = torch.from_numpy(sc.pairs).cuda()
    poses_t = torch.from_numpy(sc.poses).cuda()
    offs = torch.from_numpy(gpu["offsets"]).cuda()
    J = S.expand_jacobian(pairs_t, offs, poses_t, torch.from_numpy(gpu["W"]).cuda(),
                          torch.from_numpy(gpu["q"]).cuda(), gpu["C"]).cpu().numpy()
    ref = osc.contact_manifold()
    Jr = ref["J"].reshape(-1, 36).T
    assert np.allclose(J, Jr, atol=1e-5 * max(1.0, np.abs(Jr).max()))


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_manifold_full_size_sampled(cuda, oracle_mod, cfg):
    """BASELINE.json full sizes in bench.py's launch configuration: C4 (64k
    envs x 20 links) and C5 (1M envs, all SDF classes in one call); 256
    pairs sampled with a seeded generator and compared with the oracle."""
    sc = synth.c4_scene(65536) if cfg == "C4" else synth.c5_scene(1 << 20)
    idx = np.sort(np.random.default_rng(8).choice(len(sc.pairs), 256, replace=False))
    gpu = PT.gpu_manifold_sampled(sc, idx, 2)
    osc = oracle_mod.OracleScene(sc)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, idx, np.random.default_rng(9), sc.ell)
    _report("manifold_full_%s" % cfg, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


@pytest.mark.parametrize("mode,tier", [(4, 2), (8, 2), (12, 2), (4, 1), (8, 0)])
def test_manifold_modes_c1(cuda, oracle_mod, mode, tier):
    """Full mode (V + E contacts), two-sided (roles transposed)
    and both, on C1 (the box and the ground both carry an SDF and a mesh)."""
    sc = synth.c1_scene()
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, tier, mode=mode)
    nf, rep = PT.manifold_parity(sc, osc, gpu, tier, np.arange(len(sc.pairs)), np.random.default_rng(11), sc.ell,
                                 mode=mode)
    _report("manifold_c1_mode%d_t%d" % (mode, tier), rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_full_mode_c4(cuda, oracle_mod):
    sc = synth.c4_scene(64)
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, 2, mode=4)
    idx = np.sort(np.random.default_rng(12).choice(len(sc.pairs), 24, replace=False))
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, idx, np.random.default_rng(13), sc.ell, mode=4)
    _report("manifold_c4_full", rep)
    assert nf == 0, json.dumps(rep, indent=1)


def test_expand_jacobian_two_sided(cuda, oracle_mod):
    import torch
    sc = synth.c1_scene()
    osc = oracle_mod.OracleScene(sc)
    for mode in (8, 12):
        gpu, S = PT.gpu_manifold(sc, 1, mode=mode)
        J = S.expand_jacobian(torch.from_numpy(sc.pairs).cuda(), torch.from_numpy(gpu["offsets"]).cuda(),
                              torch.from_numpy(sc.poses).cuda(), torch.from_numpy(gpu["W"]).cuda(),
                              torch.from_numpy(gpu["q"]).cuda(), gpu["C"], mode=mode).cpu().numpy()
        Jr = osc.contact_manifold(mode=mode)["J"].reshape(-1, 36).T
        assert np.allclose(J, Jr, atol=1e-5 * max(1.0, np.abs(Jr).max()))


def test_sdf_workload_full_size_sampled(cuda, oracle_mod):
    """bench.py's SDF workload at its default size (262144 bodies x 64 points
    of the 32 C5 SDF prototypes, value + gradient + Hessian + pose gradient) in
    one launch; 256 bodies sampled with a seeded generator against the oracle."""
    import torch
    from paper_2604_17538_b200 import binding
    sc = synth.sdf_scene(1 << 18, 64)
    P = sc.P
    S = binding.Scene(sc.shapes, sc.smooth)
    flags = binding.SDF_VALUE | binding.SDF_GRAD | binding.SDF_HESS | binding.SDF_POSE_GRAD
    out = S.sdf_eval(torch.from_numpy(sc.point_shapes).cuda(), torch.from_numpy(sc.point_poses).cuda(),
                     torch.from_numpy(sc.points).cuda(), P, flags)
    torch.cuda.synchronize()
    bi = np.sort(np.random.default_rng(21).choice(len(sc.point_shapes), 256, replace=False))
    rows = torch.from_numpy((bi[:, None] * P + np.arange(P)[None, :]).reshape(-1)).cuda()
    gpu = {k: (v[..., rows] if v.dim() > 1 else v[rows]).cpu().numpy() for k, v in out.items()}
    osc = oracle_mod.OracleScene(sc)
    pts = sc.points.reshape(-1, P, 3)[bi].reshape(-1, 3)
    nf, rep = PT.sdf_parity(osc, gpu, sc.point_shapes[bi], sc.point_poses[bi], pts, P,
                            np.random.default_rng(22), sc.ell)
    _report("sdf_workload_full", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_large_patch_unstaged(cuda, oracle_mod):
    """A 40x40 plane patch (V = 1600, E = 4641, F = 3042): the unit's staged
    face state (~566 KB) exceeds shared memory, so the face kernel gathers from
    the scratch slot and recomputes the candidate points per face; sampled
    against a sphere and a PSQ at three poses."""
    patch = synth.make_shape("patch40", None, synth.plane_patch(40, 40, 0.6, 0.6))
    sph = synth.make_shape("sph", synth.sq((0.08,) * 3, (1, 1)), None)
    psq = synth.make_shape("psq", synth.psq((0.1, 0.07, 0.06), (0.6, 0.9), [[0.3, 0.2, 0.9, -0.02]]), None)
    n_env = 3
    poses = np.zeros((n_env, 3, 8), np.float32)
    poses[:, :, 3] = 1
    rng = np.random.default_rng(31)
    for e in range(n_env):
        poses[e, 1, :3] = (rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1), 0.07 - 0.01 * e)
        poses[e, 2, :3] = (rng.uniform(-0.1, 0.1), rng.uniform(-0.1, 0.1), 0.05 - 0.01 * e)
        poses[e, 1, 3:7] = synth.random_quats(rng, 1)[0]
        poses[e, 2, 3:7] = synth.random_quats(rng, 1)[0]
    pairs = np.array([[e, 0, 1 + k, 0, 1 + k] for e in range(n_env) for k in range(2)], np.int32)
    sc = scene_of([patch, sph, psq], ell=1.0, pairs=pairs, poses=poses)
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, 2)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 2, np.arange(len(pairs)), np.random.default_rng(32), sc.ell)
    _report("manifold_patch40", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


@pytest.mark.parametrize("mode", [0, 4, 8])
def test_manifold_tier3_c1(cuda, oracle_mod, mode):
    """Tier 3 (second derivatives d^2 depth / dq^2) on C1:
    reduced, full and two-sided modes against the oracle's second-order jets."""
    sc = synth.c1_scene()
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, 3, mode=mode)
    nf, rep = PT.manifold_parity(sc, osc, gpu, 3, np.arange(len(sc.pairs)), np.random.default_rng(41), sc.ell,
                                 mode=mode)
    _report("manifold_c1_t3_mode%d" % mode, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_manifold_tier3_sampled(cuda, oracle_mod, cfg):
    """Tier 3 on C4 (cup with its XPSQ handle) and C5 (every SDF class):
    GPU on a batch, oracle second-order jets on a seeded sample of pairs."""
    sc = synth.c4_scene(64) if cfg == "C4" else synth.c5_scene(512)
    osc = oracle_mod.OracleScene(sc)
    gpu, _ = PT.gpu_manifold(sc, 3)
    idx = np.sort(np.random.default_rng(42).choice(len(sc.pairs), 12, replace=False))
    nf, rep = PT.manifold_parity(sc, osc, gpu, 3, idx, np.random.default_rng(43), sc.ell)
    _report("manifold_%s_t3" % cfg, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def _param_scene():
    rng = np.random.default_rng(51)
    a = lambda: rng.uniform(0.03, 0.07, 3)
    e = lambda: rng.uniform(0.3, 1.5, 2)
    pose = lambda: [*rng.uniform(-0.03, 0.03, 3), *synth.random_quats(rng, 1)[0]]
    shapes = [
        synth.make_shape("sq", synth.sq(a(), e()), None),
        synth.make_shape("psq", synth.psq(a(), e(), [[*rng.normal(size=3), -0.01], [*rng.normal(size=3), -0.02]]), None),
        synth.make_shape("hs", synth.halfspace(rng.normal(size=3), 0.01), None),
        synth.make_shape("uni", synth.op("union", [synth.sq(a(), e(), pose=pose()) for _ in range(4)]), None),
        synth.make_shape("int", synth.op("intersection", [synth.sq(a(), e()), synth.halfspace(rng.normal(size=3), 0.01)]), None),
        synth.make_shape("sub", synth.op("subtraction", [synth.psq(a(), e(), [[*rng.normal(size=3), -0.01]]),
                                                         synth.sq(a() * 0.5, e(), pose=pose())]), None),
        synth.make_shape("xpsq", synth.xpsq([-0.05, 0, 0, 0.0, 0.06, 0.01, 0.05, 0, 0.004], (0.012, 0.015, 0.01),
                                            (0.6, 0.8), planes0=[[0.2, 0.3, 0.93, -0.005]]), None),
        synth.make_shape("uxp", synth.op("union", [synth.sq(a(), e()),
                                                   synth.xpsq([-0.05, 0, 0, 0.0, 0.05, 0.0, 0.05, 0, 0.0],
                                                              (0.01, 0.012, 0.01), (0.5, 0.9), pose=pose())]), None),
        # nested booleans: the cup (XPSQ handle, depth 2) and an SQ-family
        # tree three levels deep with every operator
        synth.make_shape("cup", synth.cup(), None),
        synth.make_shape("nest", synth.op("union", [
            synth.op("intersection", [synth.sq(a(), e(), pose=pose()),
                                      synth.op("union", [synth.sq(a(), e(), pose=pose()),
                                                         synth.sq(a(), e(), pose=pose())], pose=pose())]),
            synth.op("subtraction", [synth.psq(a(), e(), [[*rng.normal(size=3), -0.01]]),
                                     synth.sq(a() * 0.5, e(), pose=pose())], pose=pose()),
            synth.halfspace(rng.normal(size=3), -0.04)]), None),
        # varying schedules (a, eps and the plane all move along t): both
        # endpoints' slots, alone and under a subtraction
        synth.make_shape("xvary", synth.xpsq([-0.05, 0, 0, 0.0, 0.06, 0.01, 0.05, 0, 0.004], (0.012, 0.015, 0.01),
                                             (0.6, 0.8), a1=(0.008, 0.01, 0.016), eps1=(0.9, 0.5),
                                             planes0=[[0.2, 0.3, 0.93, -0.005]],
                                             planes1=[[-0.1, 0.4, 0.9, -0.008]]), None),
        # straight (p2 the midpoint: the chord p1 -> p3) and point splines:
        # control-point derivatives within their static class
        synth.make_shape("xline", synth.xpsq([-0.04, 0.01, 0.0, 0.0, 0.02, 0.01, 0.04, 0.03, 0.02], (0.01, 0.012, 0.01),
                                             (0.5, 0.9), up=(0.2, 0.1, 1.0)), None),
        synth.make_shape("xpoint", synth.xpsq([0.01, 0.0, 0.0] * 3, (0.01, 0.012, 0.015), (0.5, 0.9),
                                              planes0=[[0.1, 0.2, 0.97, -0.004]]), None),
        synth.make_shape("svary", synth.op("subtraction", [
            synth.sq(a(), e()),
            synth.xpsq([-0.05, 0, 0, 0.0, 0.05, 0.0, 0.05, 0, 0.0], (0.01, 0.012, 0.01), (0.5, 0.9),
                       a1=(0.006, 0.008, 0.012), eps1=(0.8, 0.4), pose=pose())]), None),
    ]
    return shapes, rng


def test_sdf_param_grad_parity(cuda, oracle_mod):
    """Shape-parameter derivatives: per-point J of every
    parametrised leaf kind (half-space, SQ, PSQ, constant-schedule XPSQ),
    flat booleans, nested boolean trees (the cup; a three-level SQ-family
    tree) and varying-schedule XPSQs (both endpoints' slots) against the
    oracle's parameter seeds, and the vector-Jacobian
    product sum_n w_n J_n against J^T w."""
    import torch
    from paper_2604_17538_b200 import binding
    shapes, rng = _param_scene()
    sc = scene_of(shapes, ell=0.1)
    S = binding.Scene(sc.shapes, sc.smooth)
    counts, offs = S.param_layout()
    osc = oracle_mod.OracleScene(sc)
    assert [osc.param_count(s) for s in range(len(shapes))] == list(counts)
    B, P = 4 * len(shapes), 96
    ids = np.repeat(np.arange(len(shapes)), B // len(shapes)).astype(np.int32)
    poses = np.stack([synth.pose_row(rng.uniform(-0.1, 0.1, 3), synth.random_quats(rng, 1)[0]) for _ in range(B)])
    poses = poses.astype(np.float32)
    pts = (poses[:, None, :3] + rng.normal(size=(B, P, 3)) * 0.05).reshape(-1, 3).astype(np.float32)
    w = rng.normal(size=B * P).astype(np.float32)
    pmax = int(counts.max())
    J, vjp = S.sdf_param_grad(torch.from_numpy(ids).cuda(), torch.from_numpy(poses).cuda(),
                              torch.from_numpy(pts).cuda(), P, pmax, w=torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    Jg = J.cpu().numpy().T
    Jr = osc.sdf_param_grad(ids, poses, pts, P, pmax)
    Jp = osc.sdf_param_grad(ids, PT.perturb_inputs(np.random.default_rng(52), poses), pts, P, pmax)
    rep = []
    nf = PT.compare("J", Jg, Jr, Jp, PT.tol_vec(Jr, 1), rep)
    ref_vjp = np.zeros(int(offs[-1]))
    for n in range(B * P):
        s = ids[n // P]
        ref_vjp[offs[s]:offs[s] + counts[s]] += w[n] * Jr[n, :counts[s]]
    # vjp tolerance: 1e-4 of sum |w J| (FP32 products and atomics), plus an
    # absolute floor of 1e-3 of the per-element J tolerance carried through
    # |w| (an entry summing tiny J values, e.g. a subtracted XPSQ far from
    # the points, cannot be resolved below the J scale's FP32 rounding)
    tolJ = PT.tol_vec(Jr, 1)[:, 0]
    bound = np.zeros_like(ref_vjp)
    floor = np.zeros_like(ref_vjp)
    for n in range(B * P):
        s = ids[n // P]
        bound[offs[s]:offs[s] + counts[s]] += np.abs(w[n] * Jr[n, :counts[s]])
        floor[offs[s]:offs[s] + counts[s]] += 1e-3 * abs(w[n]) * tolJ[n]
    nf += PT.compare("vjp", vjp.cpu().numpy(), ref_vjp, ref_vjp, 1e-4 * bound + floor, rep)
    _report("sdf_param_grad", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_sdf_param_grad_unsupported(cuda):
    """Scenes holding a shape with more boolean nodes than the parameter
    kernel tracks (17 > 16) report count -1 and the call is refused."""
    import torch
    from paper_2604_17538_b200 import binding
    big = synth.op("union", [synth.op("union", [synth.sq((0.01, 0.01, 0.01), (1, 1), pose=[0.02 * i, 0, 0, 1, 0, 0, 0]),
                                                synth.sq((0.01, 0.01, 0.01), (1, 1), pose=[0.02 * i, 0.02, 0, 1, 0, 0, 0])])
                             for i in range(16)])
    sc = scene_of([synth.make_shape("big", big, None)], ell=0.04)
    S = binding.Scene(sc.shapes, sc.smooth)
    counts, _ = S.param_layout()
    assert counts[0] == -1
    z = torch.zeros(1, 8, device="cuda")
    z[0, 3] = 1
    with pytest.raises(binding.CMError):
        S.sdf_param_grad(torch.zeros(1, dtype=torch.int32, device="cuda"), z,
                         torch.zeros(4, 3, device="cuda"), 4, 4)


def test_sdf_node_pose_grad_parity(cuda, oracle_mod):
    """Node poses as shape parameters (DESIGN reading #47):
    per-point d phi / d twist of every node (boolean nodes, leaves, the root)
    of the parameter scene against the oracle's node-pose seeds, and the
    vector-Jacobian product against J^T w."""
    import torch
    from paper_2604_17538_b200 import binding
    shapes, rng = _param_scene()
    sc = scene_of(shapes, ell=0.1)
    S = binding.Scene(sc.shapes, sc.smooth)
    counts, offs = S.node_pose_layout()
    osc = oracle_mod.OracleScene(sc)
    assert [6 * osc.node_count(s) for s in range(len(shapes))] == list(counts)
    B, P = 4 * len(shapes), 96
    ids = np.repeat(np.arange(len(shapes)), B // len(shapes)).astype(np.int32)
    poses = np.stack([synth.pose_row(rng.uniform(-0.1, 0.1, 3), synth.random_quats(rng, 1)[0]) for _ in range(B)])
    poses = poses.astype(np.float32)
    pts = (poses[:, None, :3] + rng.normal(size=(B, P, 3)) * 0.05).reshape(-1, 3).astype(np.float32)
    w = rng.normal(size=B * P).astype(np.float32)
    nmax = int(counts.max())
    J, vjp = S.sdf_node_pose_grad(torch.from_numpy(ids).cuda(), torch.from_numpy(poses).cuda(),
                                  torch.from_numpy(pts).cuda(), P, nmax, w=torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    Jg = J.cpu().numpy().T
    Jr = osc.sdf_node_pose_grad(ids, poses, pts, P, nmax)
    Jp = osc.sdf_node_pose_grad(ids, PT.perturb_inputs(np.random.default_rng(53), poses), pts, P, nmax)
    rep = []
    nf = PT.compare("J", Jg, Jr, Jp, PT.tol_vec(Jr, 1), rep)
    ref_vjp = np.zeros(int(offs[-1]))
    bound = np.zeros_like(ref_vjp)
    floor = np.zeros_like(ref_vjp)
    tolJ = PT.tol_vec(Jr, 1)[:, 0]
    for n in range(B * P):
        s = ids[n // P]
        ref_vjp[offs[s]:offs[s] + counts[s]] += w[n] * Jr[n, :counts[s]]
        bound[offs[s]:offs[s] + counts[s]] += np.abs(w[n] * Jr[n, :counts[s]])
        floor[offs[s]:offs[s] + counts[s]] += 1e-3 * abs(w[n]) * tolJ[n]
    nf += PT.compare("vjp", vjp.cpu().numpy(), ref_vjp, ref_vjp, 1e-4 * bound + floor, rep)
    _report("sdf_node_pose_grad", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01
    # the root's translation slots are the negated body gradient: a check of
    # the kernel against its own sdf_eval (rows of boolean-rooted shapes too)
    o = S.sdf_eval(torch.from_numpy(ids).cuda(), torch.from_numpy(poses).cuda(), torch.from_numpy(pts).cuda(), P,
                   binding.SDF_VALUE | binding.SDF_GRAD)
    torch.cuda.synchronize()
    g = o["grad"].cpu().numpy().T                       # world gradient
    R = synth.quats_to_mats(poses[:, 3:7].astype(np.float64))
    gb = np.einsum("bji,bpj->bpi", R, g.reshape(B, P, 3)).reshape(-1, 3)   # body frame
    assert np.allclose(Jg[:, 0:3], -gb, atol=2e-4 * max(1.0, np.abs(gb).max()))


def test_sdf_node_pose_grad_unsupported(cuda):
    """More boolean nodes than the kernel tracks (17 > 16): count -1, refused."""
    import torch
    from paper_2604_17538_b200 import binding
    big = synth.op("union", [synth.op("union", [synth.sq((0.01, 0.01, 0.01), (1, 1), pose=[0.02 * i, 0, 0, 1, 0, 0, 0]),
                                                synth.sq((0.01, 0.01, 0.01), (1, 1), pose=[0.02 * i, 0.02, 0, 1, 0, 0, 0])])
                             for i in range(16)])
    sc = scene_of([synth.make_shape("big", big, None)], ell=0.04)
    S = binding.Scene(sc.shapes, sc.smooth)
    counts, _ = S.node_pose_layout()
    assert counts[0] == -1
    z = torch.zeros(1, 8, device="cuda")
    z[0, 3] = 1
    with pytest.raises(binding.CMError):
        S.sdf_node_pose_grad(torch.zeros(1, dtype=torch.int32, device="cuda"), z,
                             torch.zeros(4, 3, device="cuda"), 4, 6)


def _vjp_scene():
    """A ball mesh against an SQ union, a curved XPSQ and the cup, plus the C1
    pairs (box on the ground half-space both ways): several envs each."""
    rng = np.random.default_rng(71)
    c1 = synth.c1_scene()
    ball = synth.make_shape("ball", None, synth.sq_mesh((0.12, 0.12, 0.12), (1.0, 1.0), 3))
    uni = synth.make_shape("uni", synth.op("union", [
        synth.sq((0.2, 0.15, 0.1), (0.5, 0.8)),
        synth.sq((0.1, 0.1, 0.25), (0.9, 0.4), pose=[0.1, 0.05, 0.0, 0.96, 0.2, 0.1, 0.17])]), None)
    xp = synth.make_shape("xp", synth.xpsq([-0.3, 0, 0, 0.0, 0.35, 0.05, 0.3, 0, 0.02], (0.12, 0.15, 0.1), (0.6, 0.8),
                                           planes0=[[0.2, 0.3, 0.93, -0.05]]), None)
    shapes = list(c1.shapes) + [ball, uni, xp]
    n_env = 6
    poses = np.zeros((n_env, 3, 8))
    pairs = []
    for e in range(n_env):
        poses[e, 0] = c1.poses[0, 0]
        poses[e, 1] = c1.poses[0, 1]
        poses[e, 1, :3] += rng.uniform(-0.002, 0.002, 3)
        t = [(0.05, 0.02, 0.3), (0.02, 0.22, 0.2), (0.04, 0.18, 0.18)][e % 3]
        poses[e, 2] = synth.pose_row(np.asarray(t) + rng.uniform(-0.02, 0.02, 3), synth.random_quats(rng, 1)[0])
        pairs += [[e, 0, 1, 0, 1], [e, 1, 0, 1, 0]]
        pairs += [[e, 2, 1, 2, 3 + e % 2]]   # ball (slot 2) against the union / the XPSQ at the ground's slot
    # the SDF bodies of the ball pairs sit at slot 1 (the ground pose, near the identity)
    pairs = np.asarray(pairs, dtype=np.int32)
    return scene_of(shapes, pairs=pairs, poses=poses.astype(np.float32)), rng


@pytest.mark.parametrize("mode", [0, 4, 8, 16])
def test_manifold_param_vjp_parity(cuda, oracle_mod, mode):
    """Shape-parameter VJP of the manifold depths (DESIGN
    reading #48) against the oracle's seeded manifold: random weights over
    all rows (each vjp entry within the sum of |w_r| x the per-row derivative
    tolerance 1e-4 max(|d depth_r / d theta|_inf, 1)), and one-hot weights on
    sampled rows (the rows' parameter Jacobians element by element)."""
    import torch
    from paper_2604_17538_b200 import binding
    sc, rng = _vjp_scene()
    if mode & binding.TWO_SIDED:   # both shapes need a surface and an SDF: the C1 pairs
        sc.pairs = np.ascontiguousarray(sc.pairs[sc.pairs[:, 3] <= 1])
    S = binding.Scene(sc.shapes, sc.smooth)
    osc = oracle_mod.OracleScene(sc)
    counts, offs = S.param_layout()
    pairs_t = torch.from_numpy(sc.pairs).cuda()
    poses_t = torch.from_numpy(sc.poses).cuda()
    offs_t = S.manifold_offsets(pairs_t, mode)
    C = S.manifold_size(sc.pairs, mode)
    pmax = int(counts.max())
    Jd = osc.manifold_param_jac(sc.pairs, sc.poses, mode=mode, pmax=pmax)
    Jp = osc.manifold_param_jac(sc.pairs, PT.perturb_inputs(np.random.default_rng(72), sc.poses), mode=mode, pmax=pmax)
    assert Jd.shape[0] == C
    # each row's SDF shape: B, or A for the transposed half of a two-sided pair
    offs_h = offs_t.cpu().numpy()
    row_pair = np.searchsorted(offs_h, np.arange(C), side="right") - 1
    shape_of_row = sc.pairs[row_pair, 4].copy()
    if mode & binding.TWO_SIDED:
        nA = np.array([S.counts(int(a))[2 if not mode & binding.FULL_MODE else 0] for a in sc.pairs[:, 3]])
        second = np.arange(C) - offs_h[row_pair] >= nA[row_pair]
        shape_of_row[second] = sc.pairs[row_pair[second], 3]
    tol_row = 1e-4 * np.maximum(np.abs(Jd).max(axis=1), 1.0)

    def ref_vjp(w, J):
        out = np.zeros(int(offs[-1]))
        for r in np.nonzero(w)[0]:
            s = shape_of_row[r]
            out[offs[s]:offs[s] + counts[s]] += w[r] * J[r, :counts[s]]
        return out

    def tol_vjp(w):
        out = np.full(int(offs[-1]), 1e-30)   # (entries no row touches must come back exactly 0)
        for r in np.nonzero(w)[0]:
            s = shape_of_row[r]
            out[offs[s]:offs[s] + counts[s]] += abs(w[r]) * tol_row[r]
        return out

    rep = []
    nf = 0
    for trial in range(3):
        w = rng.normal(size=C).astype(np.float32)
        got = S.manifold_param_vjp(pairs_t, offs_t, poses_t, torch.from_numpy(w).cuda(), mode).cpu().numpy()
        nf += PT.compare("vjp%d" % trial, got, ref_vjp(w, Jd), ref_vjp(w, Jp), tol_vjp(w), rep)
    for r in rng.choice(C, size=24, replace=False):
        w = np.zeros(C, np.float32)
        w[r] = 1.0
        got = S.manifold_param_vjp(pairs_t, offs_t, poses_t, torch.from_numpy(w).cuda(), mode).cpu().numpy()
        nf += PT.compare("row%d" % r, got, ref_vjp(w, Jd), ref_vjp(w, Jp), tol_vjp(w), rep)
    _report("manifold_param_vjp_m%d" % mode, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01
    assert np.abs(Jd).max() > 0.1


def test_manifold_param_vjp_cup(cuda, oracle_mod):
    """The manifold shape-parameter VJP on C4 (2 envs x 20 links against the
    cup: a nested boolean tree with an XPSQ handle, 24 parameters incl. the
    handle's control points): random weights and one-hot rows."""
    import torch
    from paper_2604_17538_b200 import binding
    sc = synth.c4_scene(2)
    S = binding.Scene(sc.shapes, sc.smooth)
    osc = oracle_mod.OracleScene(sc)
    counts, offs = S.param_layout()
    pairs_t = torch.from_numpy(sc.pairs).cuda()
    poses_t = torch.from_numpy(sc.poses).cuda()
    offs_t = S.manifold_offsets(pairs_t)
    C = S.manifold_size(sc.pairs)
    pmax = int(counts.max())
    Jd = osc.manifold_param_jac(sc.pairs, sc.poses, pmax=pmax)
    Jp = osc.manifold_param_jac(sc.pairs, PT.perturb_inputs(np.random.default_rng(74), sc.poses), pmax=pmax)
    nc = counts[0]                      # every row's SDF shape is the cup (shape 0)
    tol_row = 1e-4 * np.maximum(np.abs(Jd).max(axis=1), 1.0)
    rng = np.random.default_rng(75)
    rep = []
    nf = 0
    for trial in range(3):
        w = rng.normal(size=C).astype(np.float32)
        got = S.manifold_param_vjp(pairs_t, offs_t, poses_t, torch.from_numpy(w).cuda()).cpu().numpy()
        nf += PT.compare("vjp%d" % trial, got[offs[0]:offs[0] + nc], w @ Jd[:, :nc], w @ Jp[:, :nc],
                         np.abs(w) @ tol_row + 1e-30, rep)
    for r in rng.choice(C, size=16, replace=False):
        w = np.zeros(C, np.float32)
        w[r] = 1.0
        got = S.manifold_param_vjp(pairs_t, offs_t, poses_t, torch.from_numpy(w).cuda()).cpu().numpy()
        nf += PT.compare("row%d" % r, got[offs[0]:offs[0] + nc], Jd[r, :nc], Jp[r, :nc], tol_row[r], rep)
    _report("manifold_param_vjp_cup", rep)
    assert nf == 0, json.dumps(rep, indent=1)
    assert PT.excluded_fraction(rep) < 0.01


def test_manifold_param_vjp_unsupported(cuda):
    """A scene holding a shape the parameter layout cannot describe (more
    than 16 boolean nodes: count -1) refuses the manifold VJP."""
    import torch
    from paper_2604_17538_b200 import binding
    big = synth.op("union", [synth.op("union", [synth.sq((0.01, 0.01, 0.01), (1, 1), pose=[0.02 * i, 0, 0, 1, 0, 0, 0]),
                                                synth.sq((0.01, 0.01, 0.01), (1, 1), pose=[0.02 * i, 0.02, 0, 1, 0, 0, 0])])
                             for i in range(16)])
    c1 = synth.c1_scene()
    shapes = list(c1.shapes) + [synth.make_shape("big", big, None)]
    sc = scene_of(shapes, pairs=c1.pairs, poses=c1.poses)
    S = binding.Scene(sc.shapes, sc.smooth)
    pairs_t = torch.from_numpy(sc.pairs).cuda()
    poses_t = torch.from_numpy(sc.poses).cuda()
    offs_t = S.manifold_offsets(pairs_t)
    C = S.manifold_size(sc.pairs)
    with pytest.raises(binding.CMError):
        S.manifold_param_vjp(pairs_t, offs_t, poses_t, torch.zeros(C, device="cuda"))


def test_sdf_eval_xpsq_soft_cardano_band(cuda, oracle_mod):
    """Points inside the soft-Cardano band 10 tau_Delta < |Delta| < 46
    tau_Delta of a curved XPSQ (both branches blended): every
    output finite and within tolerance.  Near the band's edge the weaker
    branch's trigonometric roots nearly coincide (its projected discriminant
    s+(Delta) is tiny); their derivatives are taken from the cube roots, not
    through the implicit 1 / F'(s) (0 / 0 there: found as NaN normals on C5
    pairs in round 2)."""
    from paper_2604_17538_b200 import binding
    sampled, sdf = synth.c5_library()
    shape = next(s for s in sdf if s.name == "xpsq3")
    sc = scene_of([shape], ell=0.1)
    osc = oracle_mod.OracleScene(sc)
    S = binding.Scene(sc.shapes, sc.smooth)
    rng = np.random.default_rng(77)
    cand = rng.uniform(-0.12, 0.12, (40000, 3))
    keep = []
    for p in cand:
        _, delta, _ = osc.xpsq_roots(0, 0, p)
        if 10 < abs(delta) / sc.smooth["tau_delta"] < 46:
            keep.append(p)
        if len(keep) >= 400:
            break
    assert len(keep) >= 100, len(keep)
    pts = np.asarray(keep, np.float32)
    ids = np.zeros(1, np.int32)
    poses = pose8().reshape(1, 8).astype(np.float32)
    gpu = PT.gpu_sdf(S, ids, poses, pts, len(pts), ALL)
    for k, v in gpu.items():
        assert np.isfinite(v).all(), k
    nf, rep = PT.sdf_parity(osc, gpu, ids, poses, pts, len(pts), rng, 0.1)
    _report("sdf_xpsq_band", rep)
    assert nf == 0, json.dumps(rep, indent=1)


def test_sdf_eval_xpsq_cusp_finite(cuda, oracle_mod):
    """Points on and near the negative branch's cube-root cusp (Q ~ 0 with
    0 < Delta < 46 tau_Delta, reading #15: excluded from parity)
    give finite values, gradients and Hessians (found as NaN Hessians on C5
    pairs in round 2: P^3 + s+(Delta)/4 cancelled in FP32)."""
    from paper_2604_17538_b200 import binding
    sampled, sdf = synth.c5_library()
    shape = next(s for s in sdf if s.name == "xpsq3")
    n = shape.sdf[0]
    c = np.asarray(n["ctrl"], np.float64).reshape(3, 3)
    A, B = c[0] - 2 * c[1] + c[2], 2 * (c[1] - c[0])
    c3, c2 = -2 * A @ A, -3 * A @ B
    b = c2 / c3
    # depressed Q(w) = 2b^3/27 - b c1/(3 c3) + c0/c3, c1 = 2A.w - B.B, c0 = B.w: affine in w
    gQ = (B - (2 * b / 3) * A) / c3
    Q0 = 2 * b ** 3 / 27 + (b / 3) * (B @ B) / c3
    sc = scene_of([shape], ell=0.1)
    osc = oracle_mod.OracleScene(sc)
    S = binding.Scene(sc.shapes, sc.smooth)
    rng = np.random.default_rng(78)
    pts = []
    for q in (0.0, 1e-7, -1e-7, 1e-6, -1e-6, 1e-5):
        w = rng.uniform(-0.12, 0.12, (3000, 3))
        w -= np.outer((w @ gQ + Q0 - q) / (gQ @ gQ), gQ)      # onto the plane Q(w) = q
        y = w + c[0]
        for p in y:
            _, delta, _ = osc.xpsq_roots(0, 0, p)
            if 0 < delta / sc.smooth["tau_delta"] < 46:
                pts.append(p)
    assert len(pts) > 100, len(pts)
    pts = np.asarray(pts, np.float32)
    gpu = PT.gpu_sdf(S, np.zeros(1, np.int32), pose8().reshape(1, 8).astype(np.float32), pts, len(pts), ALL)
    for k, v in gpu.items():
        assert np.isfinite(v).all(), (k, int((~np.isfinite(v)).sum()))


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_pair_reduce(cuda, oracle_mod, cfg):
    """cm_manifold_pair_reduce (pair-level smooth-min depth, sum W, pose VJP
    of depths and normals, one warp per pair) against the oracle's reduction
    of its own contacts, on 64 sampled pairs of a 512-env scene.  Tolerances
    carried from the per-contact ones."""
    import torch
    sc = synth.c4_scene(512) if cfg == "C4" else synth.c5_scene(512)
    osc = oracle_mod.OracleScene(sc)
    gpu, S = PT.gpu_manifold(sc, 2)
    rng = np.random.default_rng(21)
    C = gpu["C"]
    wd = rng.normal(size=C).astype(np.float32)
    wn = rng.normal(size=(3, C)).astype(np.float32)
    dev = "cuda"
    out = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in gpu.items() if k not in ("offsets", "C")}
    pairs_t = torch.from_numpy(sc.pairs).to(dev)
    offs_t = torch.from_numpy(gpu["offsets"]).to(dev)
    pd, pw, gp = S.pair_reduce(pairs_t, offs_t, out, C, w_depth=torch.from_numpy(wd).to(dev),
                               w_normal=torch.from_numpy(wn).to(dev))
    pd, pw, gp = pd.cpu().numpy(), pw.cpu().numpy(), gp.cpu().numpy()
    idx = np.sort(rng.choice(len(sc.pairs), 64, replace=False))
    ref = osc.contact_manifold(pairs=sc.pairs[idx])
    refp = osc.contact_manifold(pairs=sc.pairs[idx], poses=PT.perturb_inputs(rng, sc.poses))
    rows = np.concatenate([np.arange(gpu["offsets"][i], gpu["offsets"][i] + (ref["offsets"][k + 1] - ref["offsets"][k]))
                           for k, i in enumerate(idx)])
    wd_s, wn_s = wd[rows].astype(np.float64), wn[:, rows].T.astype(np.float64)
    tau = sc.smooth["tau_min"]
    r_pd, r_pw, r_gp = oracle_mod.OracleScene.pair_reduce(ref, tau, wd_s, wn_s)
    p_pd, p_pw, p_gp = oracle_mod.OracleScene.pair_reduce(refp, tau, wd_s, wn_s)
    rep = []
    nf = PT.compare("pair_depth", pd[idx], r_pd, p_pd, PT.tol_value(r_pd, sc.ell), rep)
    off = ref["offsets"]
    cnt = np.diff(off)
    nf += PT.compare("pair_W", pw[idx], r_pw, p_pw, 1e-4 * np.maximum(np.abs(r_pw), cnt), rep)
    # g tolerance: the per-contact tolerances of ddepth and dnormal through |w|
    tg = np.zeros((len(idx), 1))
    for k in range(len(idx)):
        r = slice(off[k], off[k + 1])
        t_dd = 1e-4 * np.maximum(np.abs(ref["ddepth"][r]).max(1), 1.0)
        t_dn = 1e-3 * np.maximum(np.abs(ref["dnormal"][r]).max((1, 2)), 1.0 / sc.ell)
        tg[k] = np.sum(np.abs(wd_s[r]) * t_dd) + np.sum(np.abs(wn_s[r]).sum(1) * t_dn)
    nf += PT.compare("g_pose", gp[idx], r_gp, p_gp, tg, rep)
    _report("pair_reduce_%s" % cfg, rep)
    assert nf == 0, json.dumps(rep, indent=1)


@pytest.mark.parametrize("mode", [4, 8])
def test_broad_phase_modes(cuda, oracle_mod, mode):
    """CM_BROAD_PHASE with full mode (candidate rows) and two-sided manifolds
    (each side culled on its own bound): every row of a 128-pair C6 sample
    against the oracle's same mode, culled and kept alike."""
    from paper_2604_17538_b200 import binding
    sc = synth.c6_scene(8)
    osc = oracle_mod.OracleScene(sc)
    gb, S = PT.gpu_manifold(sc, 2, mode=binding.BROAD_PHASE | mode)
    assert 0.3 < float((gb["dom"] == -2).mean()) < 0.99
    rng = np.random.default_rng(29 + mode)
    idx = np.sort(rng.choice(len(sc.pairs), 128, replace=False))
    nf, rep = PT.manifold_parity(sc, osc, gb, 2, idx, rng, sc.ell, mode=16 | mode)
    _report("broad_phase_mode%d" % mode, rep)
    assert nf == 0, json.dumps(rep, indent=1)
    # (culled rows carry six equal candidate depths: the dom comparison skips
    # them as near ties, which is not a conditioning exclusion)
    assert PT.excluded_fraction([r for r in rep if r["field"] != "dom"]) < 0.01


def test_broad_phase_c6(cuda, oracle_mod):
    """CM_BROAD_PHASE (f2) on C6 (two 18-part SQ objects, 324 part pairs per
    env): the GPU's culled set equals the oracle's (outside a 1e-5 ell band
    around the 40 tau_cmp threshold), culled rows match the oracle's culled
    rows, kept pairs match the oracle's all-edges manifold (tolerances of
    DESIGN.md §6) and are bit-identical to the GPU call without the flag."""
    import torch
    from paper_2604_17538_b200 import binding
    sc = synth.c6_scene(32)
    osc = oracle_mod.OracleScene(sc)
    gb, S = PT.gpu_manifold(sc, 2, mode=binding.BROAD_PHASE)
    g0, _ = PT.gpu_manifold(sc, 2, S=S)
    C = gb["C"]
    off = gb["offsets"]
    F = np.array([S.counts(int(a))[2] for a in sc.pairs[:, 3]])
    culled = np.array([gb["dom"][off[i]] == -2 for i in range(len(sc.pairs))])
    assert 0.5 < culled.mean() < 0.99, culled.mean()
    # kept pairs: bit-identical to the unflagged call
    for i in np.nonzero(~culled)[0][:400]:
        r = slice(off[i], off[i] + F[i])
        for k in ("point", "normal", "depth", "W", "q", "ddepth", "dnormal", "dom"):
            assert np.array_equal(gb[k][..., r], g0[k][..., r]), (i, k)
    # oracle parity on a sample of pairs with both decisions compared
    rng = np.random.default_rng(23)
    idx = np.sort(rng.choice(len(sc.pairs), 256, replace=False))
    ref = osc.contact_manifold(pairs=sc.pairs[idx], mode=16)
    tau_cmp = sc.smooth["tau_cmp"]
    n_band = 0
    for k, i in enumerate(idx):
        lb = ref["dcand"][ref["offsets"][k], 0]
        ref_cull = ref["dom"][ref["offsets"][k]] == -2
        if abs(lb - 40 * tau_cmp) < 1e-5 * sc.ell and ref_cull:
            n_band += 1
            continue
        assert ref_cull == culled[i], (i, lb)
    kept = idx[~culled[idx]]
    nf, rep = PT.manifold_parity(sc, osc, gb, 2, kept, rng, sc.ell, mode=16)
    cul = idx[culled[idx]]
    nf2, rep2 = PT.manifold_parity(sc, osc, gb, 2, cul, rng, sc.ell, mode=16)
    _report("broad_phase_c6", rep + rep2)
    assert nf == 0 and nf2 == 0, json.dumps(rep + rep2, indent=1)
    assert (gb["dom"][np.concatenate([np.arange(off[i], off[i] + F[i]) for i in cul])] == -2).all()
