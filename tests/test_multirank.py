"""The N > 1 path of bench.py on CPU (gloo, world_size 2): every rank owns
the env range [rank*n, (rank+1)*n) with inputs keyed by global env index, the
data path has no collective, and the reported time is the max over ranks.
Shard outputs (oracle) concatenated must equal a single-process run over the
whole range, bitwise (SURVEY §8e check)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_env, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as O
    scene = bench.make_scene("C5", n_env, rank * n_env)
    # the same global env ids a single process would generate
    assert scene.meta["env_lo"] == rank * n_env
    osc = O.OracleScene(scene)
    sub = scene.pairs[:6]
    out = osc.contact_manifold(pairs=sub, n_threads=1)
    # max-over-ranks timing, as bench.py does it
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # gather shard inputs and outputs on rank 0 for the comparison
    # the reference: the same global envs cut from a single-process
    # generation of the whole range, evaluated in this same process
    full = bench.make_scene("C5", world * n_env, 0)
    lo = rank * n_env
    ref = O.OracleScene(full).contact_manifold(pairs=full.pairs[lo:lo + 6].copy(), n_threads=1)
    same = all(np.array_equal(ref[k], out[k], equal_nan=True) for k in ("depth", "ddepth", "dnormal", "point", "W"))
    payload = dict(poses=scene.poses[:6].copy(), pairs=sub.copy(), t=float(t.item()), same=bool(same))
    objs = [None] * world
    dist.all_gather_object(objs, payload)
    if rank == 0:
        q.put(objs)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_match_single_process():
    world, n_env = 2, 70000     # shard 1 starts inside the first 65536-env block
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_env, q)) for r in range(world)]
    for p in procs:
        p.start()
    objs = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(o["t"] == float(world) for o in objs)
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    full = bench.make_scene("C5", world * n_env, 0)
    for r, o in enumerate(objs):
        lo = r * n_env
        assert np.array_equal(full.poses[lo:lo + 6], o["poses"])
        ref_pairs = full.pairs[lo:lo + 6].copy()
        assert np.array_equal(ref_pairs[:, 1:], o["pairs"][:, 1:])
        assert np.array_equal(ref_pairs[:, 0] - lo, o["pairs"][:, 0])
        assert o["same"]


def test_slice_envs_renumbers():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2604_17538_b200 import synth
    sc = synth.c4_scene(8)
    sh = sc.slice_envs(3, 6)
    assert sh.n_env == 3 and sh.pairs[:, 0].min() == 0 and sh.pairs[:, 0].max() == 2
    assert np.array_equal(sh.poses, sc.poses[3:6])


def test_sdf_workload_shards_match_single_generation():
    # sdf_eval workload: a rank's body range equals the same bodies cut from
    # one generation of the whole range (per-65536-block keys), points stay
    # near the bodies' surfaces, and the oracle values agree shard vs whole
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    full = bench.make_scene("SDF", 70000, 0)
    sh = bench.make_scene("SDF", 100, 65500)
    P = sh.P
    assert np.array_equal(sh.point_shapes, full.point_shapes[65500:65600])
    assert np.array_equal(sh.point_poses, full.point_poses[65500:65600])
    assert np.array_equal(sh.points, full.points[65500 * P:65600 * P])
    o1 = O.OracleScene(sh).sdf_eval(sh.point_shapes[:4], sh.point_poses[:4], sh.points[:4 * P], P)
    o2 = O.OracleScene(full).sdf_eval(full.point_shapes[65500:65504], full.point_poses[65500:65504],
                                      full.points[65500 * P:65504 * P], P)
    assert np.array_equal(o1["d"], o2["d"]) and np.array_equal(o1["hess"], o2["hess"])
    # the query points straddle the surfaces: both signs, most within 0.05
    d = O.OracleScene(sh).sdf_eval(sh.point_shapes, sh.point_poses, sh.points, P, want_pose=False)["d"]
    assert (d < 0).mean() > 0.2 and (d > 0).mean() > 0.2 and (np.abs(d) < 0.05).mean() > 0.9
