"""GPU tests of the call scheduling (scratch shared by manifold calls on one
scene) and of the env-range sharding of SURVEY §8(e): the library's outputs
do not depend on which stream a call came from, on chunk boundaries, or on
which shard of the global env sequence a rank owns.  Needs a B200."""
import numpy as np
import pytest

from paper_2604_17538_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_17538_b200 import binding
    binding.lib()
    return torch


def _same(a, b):
    """bitwise-equal values (NaN at the same places counts as equal)"""
    import torch
    if a.dtype.is_floating_point:
        return bool(((a == b) | (torch.isnan(a) & torch.isnan(b))).all())
    return bool(torch.equal(a, b))


def _inputs(S, sc, torch):
    pairs = torch.from_numpy(sc.pairs).cuda()
    poses = torch.from_numpy(sc.poses).cuda()
    offs = S.manifold_offsets(pairs)
    return pairs, poses, offs, S.manifold_size(sc.pairs)


def test_manifold_calls_on_two_streams(cuda):
    """A tier-2 call on stream s1 and a tier-0 call on stream s2, issued back
    to back on one scene without host synchronisation (their
    scratch splits between the internal streams differ by tier), give the
    same bits as the two calls run one after the other on one stream."""
    torch = cuda
    from paper_2604_17538_b200 import binding
    sc = synth.c5_scene(1 << 17)
    S = binding.Scene(sc.shapes, sc.smooth)
    pairs, poses, offs, C = _inputs(S, sc, torch)
    ref2 = S.contact_manifold(pairs, offs, C, poses, 2)
    ref0 = S.contact_manifold(pairs, offs, C, poses, 0)
    torch.cuda.synchronize()
    for rep in range(3):
        o2 = S.alloc_manifold(C, 2, poses.device)
        o0 = S.alloc_manifold(C, 0, poses.device)
        for v in list(o2.values()) + list(o0.values()):
            if v.dtype == torch.float32:
                v.fill_(float("nan"))
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            S.contact_manifold(pairs, offs, C, poses, 2, out=o2)
        with torch.cuda.stream(s2):
            S.contact_manifold(pairs, offs, C, poses, 0, out=o0)
        torch.cuda.synchronize()
        for k in ref2:
            assert _same(o2[k], ref2[k]), (rep, "tier 2", k)
        for k in ref0:
            assert _same(o0[k], ref0[k]), (rep, "tier 0", k)


@pytest.mark.parametrize("lo,n", [(300001, 262144), (1 << 19, 65536)])
def test_shard_rows_equal_full_run(cuda, lo, n):
    """SURVEY §8(e) check: the C5 envs [lo, lo + n) run as their own shard
    (what rank r of a G-GPU job computes) give outputs bitwise equal to the
    same rows of the full 1M-env single-GPU run (different chunk boundaries,
    different unit order inside the chunks)."""
    torch = cuda
    from paper_2604_17538_b200 import binding
    full = synth.c5_scene(1 << 20)
    shard = synth.c5_scene(n, env_lo=lo)
    assert np.array_equal(shard.pairs[:, 3:], full.pairs[lo:lo + n, 3:])
    assert np.array_equal(shard.poses, full.poses[lo:lo + n])
    S = binding.Scene(full.shapes, full.smooth)
    pairs, poses, offs, C = _inputs(S, full, torch)
    out_full = S.contact_manifold(pairs, offs, C, poses, 2)
    torch.cuda.synchronize()
    r0 = int(offs[lo].item())
    del pairs, poses
    ps, po, os_, Cs = _inputs(S, shard, torch)
    out_sh = S.contact_manifold(ps, os_, Cs, po, 2)
    torch.cuda.synchronize()
    for k, v in out_sh.items():
        assert _same(v, out_full[k][..., r0:r0 + Cs]), k


def test_invalid_records_counted_not_dereferenced(cuda):
    """Device-side validation: pair records with
    out-of-range env / slot indices get NaN rows, out-of-range shape ids get
    no rows, sdf_eval bodies with a bad shape id get NaN outputs; each is
    counted in cm_scene_error_count and the valid records' outputs are
    unchanged (no device fault)."""
    torch = cuda
    from paper_2604_17538_b200 import binding
    sc = synth.c5_scene(64)
    S = binding.Scene(sc.shapes, sc.smooth)
    assert S.error_count(reset=True) == 0
    good = sc.pairs.copy()
    bad = good.copy()
    bad[3, 0] = 10 ** 6                  # env out of range: NaN rows
    bad[7, 2] = 5                        # slot out of range: NaN rows
    bad[11, 4] = len(sc.shapes) + 3      # SDF shape id out of range: no rows
    ref = {}
    for name, pr in (("good", good), ("bad", bad)):
        pt = torch.from_numpy(pr).cuda()
        po = torch.from_numpy(sc.poses).cuda()
        offs = S.manifold_offsets(pt)
        # the host size call rejects the bad shape id; size the outputs from
        # the device offsets (what a caller with device-only pairs would do)
        last = int(offs[-1].item()) + S.counts(int(pr[-1, 3]))[2]
        out = S.contact_manifold(pt, offs, last, po, 2)
        torch.cuda.synchronize()
        ref[name] = (offs.cpu().numpy(), {k: v.cpu().numpy() for k, v in out.items()}, last)
    assert S.error_count() == 4   # offsets kernel: the bad shape id; manifold: the 3 bad records
    og, g, _ = ref["good"]
    ob, b, _ = ref["bad"]
    F = lambda i: S.counts(int(good[i, 3]))[2]
    for i in range(len(good)):
        if i == 11:
            assert ob[i + 1] == ob[i] if i + 1 < len(good) else True
            continue
        rg = slice(og[i], og[i] + F(i))
        rb = slice(ob[i], ob[i] + F(i))
        if i in (3, 7):
            assert np.isnan(b["depth"][rb]).all() and (b["dom"][rb] == -1).all()
        else:
            for k in g:
                assert np.array_equal(g[k][..., rg], b[k][..., rb], equal_nan=True), (i, k)
    # sdf_eval: body 1 names a shape id out of range
    ids = torch.tensor([16, 10 ** 5, 17], dtype=torch.int32, device="cuda")
    poses = torch.zeros(3, 8, device="cuda")
    poses[:, 3] = 1
    pts = torch.rand(3 * 5, 3, device="cuda") * 0.1
    S.error_count(reset=True)
    o = S.sdf_eval(ids, poses, pts, 5, binding.SDF_VALUE | binding.SDF_GRAD)
    torch.cuda.synchronize()
    d = o["d"].cpu().numpy()
    assert np.isnan(d[5:10]).all() and np.isfinite(d[:5]).all() and np.isfinite(d[10:]).all()
    assert S.error_count() == 5


@pytest.mark.parametrize("wl", ["C1", "C5"])
def test_manifold_cuda_graph_capture(cuda, wl):
    """cm_contact_manifold inside a CUDA graph (stream capture: the fork onto
    the scene's internal streams and the join back are events recorded on
    the capturing stream): replays with new poses copied into the captured
    input buffer give the same bits as eager calls."""
    torch = cuda
    from paper_2604_17538_b200 import binding
    sc = synth.c1_scene() if wl == "C1" else synth.c5_scene(4096)
    S = binding.Scene(sc.shapes, sc.smooth)
    pairs, poses, offs, C = _inputs(S, sc, torch)
    out = S.alloc_manifold(C, 2, poses.device)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):   # warm-up outside the capture
        S.contact_manifold(pairs, offs, C, poses, 2, out=out)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        S.contact_manifold(pairs, offs, C, poses, 2, out=out)
    rng = np.random.default_rng(9)
    for rep in range(3):
        p2 = sc.poses.copy()
        p2[..., :3] += rng.normal(size=p2[..., :3].shape).astype(np.float32) * 1e-3
        poses.copy_(torch.from_numpy(p2))
        for v in out.values():
            if v.dtype == torch.float32:
                v.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        ref = S.contact_manifold(pairs, offs, C, torch.from_numpy(p2).cuda(), 2)
        torch.cuda.synchronize()
        for k in ref:
            assert _same(out[k], ref[k]), (rep, k)


@pytest.mark.parametrize("rotated", [False, True])
def test_scene_sample_res_equals_explicit_mesh(cuda, rotated):
    """cm_shape_desc.sample_res: a shape whose sampled surface
    the library tessellates itself (placed by its root node's pose) gives the
    manifold of the same shape given the explicit mesh of cm_tessellate
    placed by that pose: bit for bit at the identity pose, within FP32
    rounding of the vertex placement otherwise."""
    torch = cuda
    import copy
    from paper_2604_17538_b200 import binding
    sc = synth.c1_scene()
    box, ground = sc.shapes
    pose = [0.01, -0.02, 0.005, 0.96, 0.1, 0.2, 0.17] if rotated else [0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0]
    root = synth.sq((0.2, 0.15, 0.1), (0.3, 0.3), pose=pose)
    node = synth.flatten(root)[0]
    v, f = binding.tessellate(node, 3)
    pz = np.asarray(node["pose"], dtype=np.float32).astype(np.float64)   # (the FP32 node pose)
    R = synth.quats_to_mats((pz[3:] / np.linalg.norm(pz[3:]))[None, :])[0]
    vt = (v.astype(np.float64) @ R.T + pz[:3]).astype(np.float32)
    explicit = synth.make_shape("box_mesh", root, (vt, f))
    implicit = copy.deepcopy(explicit)
    implicit.vertices, implicit.faces = None, None
    implicit.sample_res = 3
    outs = []
    for shp in (explicit, implicit):
        S = binding.Scene([shp, ground], sc.smooth)
        assert S.counts(0) == (len(v), 3 * (len(v) - 2), len(f))
        pairs, poses, offs, C = _inputs(S, sc, torch)
        outs.append({k: o.cpu() for k, o in S.contact_manifold(pairs, offs, C, poses, 2).items()})
    for k in outs[0]:
        if rotated and outs[0][k].dtype == torch.float32:
            a, b = outs[0][k].double(), outs[1][k].double()
            assert torch.allclose(a, b, rtol=1e-3, atol=1e-5 * max(1.0, float(a.abs().max()))), k
        elif not rotated:
            assert _same(outs[0][k], outs[1][k]), k
