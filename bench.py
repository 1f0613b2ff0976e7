#!/usr/bin/env python
"""Benchmark of the hot path: smooth one-shot contact manifolds with full
derivatives (tier 2) for every (environment, pair) of a large batch
(arXiv 2604.17538 §II-C; BASELINE.json metric "contact-manifold evals/sec
with derivatives").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5]
  python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
  python bench.py --impl reference ...   (the FP64 oracle on host cores)

One step = one cm_contact_manifold call (tier 2) over the rank's whole env
shard.  Weak scaling: every rank owns n_env environments (global env ids
[rank*n_env, (rank+1)*n_env), inputs keyed by global env index), no
collective on the data path; timing is max over ranks.  Inputs (poses,
pairs, offsets) are resident in HBM for `value`; `e2e` re-times the same
step through the public API with the step's poses copied host->device from
pinned memory and the fused depths copied back every step (double buffered:
the copies of neighbouring steps overlap the compute on separate upload /
download streams).  L2 is flushed (256 MiB write) between timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic work per pair: FP32 FLOPs from the frozen cost
# table paper_2604_17538_b200/costmodel.json (per SDF shape and derivative
# order, measured once with ncu by tools/costmodel.py) composed with the
# pair's structure:
#   flop = M(mesh_A) + (V + E) [c(B,2) - c(hs,2)] + 2 E (iters - 1) [c(B,1) - c(hs,1)]
# with M(mesh_A) the tier-2 manifold FLOPs of the mesh against a half-space.
# Bytes per pair are algorithmic too (inputs: two poses + the pair record;
# outputs: F contacts x 237 B at tier 2).
OUT_BYTES_PER_CONTACT = {0: 33, 1: 45, 2: 237, 3: 237 + 78 * 4}
IN_BYTES_PER_PAIR = 2 * 32 + 20
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 at the 1965 MHz max SM clock


def _cost_key(workload, shape, kind):
    if workload == "C5":
        return shape.name
    if kind == "sdf":
        return {"C1": "C1:", "C2": "C2:", "C3": "C3:", "C4": "C4:"}[workload] + (
            {"blob18": "blob18"}.get(shape.name, shape.name))
    return {"C2": "C2:", "C3": "C3:", "C4": "C4:", "C1": "C1:"}[workload] + shape.name


def flop_per_launch(workload, scene, S):
    """Algorithmic FP32 FLOPs of one tier-2 call over scene.pairs."""
    with open(os.path.join(ROOT, "paper_2604_17538_b200", "costmodel.json")) as f:
        cm = json.load(f)
    hs1, hs2 = cm["halfspace_eval"]["order1"], cm["halfspace_eval"]["order2"]
    it = scene.smooth["trace_iters"]
    per_shape_pair = {}
    total = 0.0
    a_ids, b_ids = scene.pairs[:, 3], scene.pairs[:, 4]
    keys, counts = np.unique(np.stack([a_ids, b_ids], 1), axis=0, return_counts=True)
    for (a, b), n in zip(keys, counts):
        sa, sb = scene.shapes[a], scene.shapes[b]
        ka, kb = _cost_key(workload, sa, "mesh"), _cost_key(workload, sb, "sdf")
        if ka not in cm["manifold_with_halfspace"] or kb not in cm["sdf"]:
            return None
        V, E, F = S.counts(int(a))
        c = cm["manifold_with_halfspace"][ka]["flop_per_pair_total_with_halfspace"]
        c += (V + E) * (cm["sdf"][kb]["order2"]["flop"] - hs2) + 2 * E * (it - 1) * (cm["sdf"][kb]["order1"]["flop"] - hs1)
        total += n * c
    return total


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def make_scene(workload, n_env, env_lo, K=18):
    from paper_2604_17538_b200 import synth
    if workload == "C1":
        return synth.c1_scene()
    if workload == "C5":
        return synth.c5_scene(n_env, env_lo=env_lo)
    if workload == "C4":
        return synth.c4_scene(n_env, seed=4 + 1000 * (env_lo // max(n_env, 1)))
    if workload == "C3":
        return synth.c3_scene(n_env, seed=3 + 1000 * (env_lo // max(n_env, 1)), K=K)
    if workload == "C2":
        return synth.c2_scene(n_env, seed=2 + 1000 * (env_lo // max(n_env, 1)))
    if workload == "SDF":
        return synth.sdf_scene(n_env, SDF_P, env_lo=env_lo)
    raise SystemExit("unknown workload " + workload)


DEFAULT_NENV = {"C5": 1 << 20, "C4": 1 << 16, "C3": 1 << 14, "C2": 1000, "SDF": 1 << 18, "C1": 1}
SDF_P = 64            # query points per body (SDF workload)
SDF_METRIC = "sdf_eval point-evaluations/sec (value + gradient + Hessian + pose gradient)"
SDF_BYTES_PER_POINT = 12 + 4 + 12 + 24 + 24   # point in; d, grad, hess (6), dpose (6) out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_rate(scene, budget_s=15.0, threads=0, max_pairs=None):
    """The FP64 oracle (as it stands) on a bounded prefix of the workload's
    pairs on the host cores: returns (pairs/s, pairs timed, cores)."""
    from oracle import oracle as O
    osc = O.OracleScene(scene)
    cores = O.max_threads() if threads == 0 else threads
    # pilot large enough to keep every core busy, then scale to the budget
    n = min(len(scene.pairs), 16 * max(cores, 8))
    t0 = time.perf_counter()
    osc.contact_manifold(pairs=scene.pairs[:n], n_threads=threads)
    dt = time.perf_counter() - t0
    per = dt / n
    m = int(max(n, min(len(scene.pairs), budget_s / max(per, 1e-9))))
    if max_pairs:
        m = min(m, max_pairs)
    t0 = time.perf_counter()
    osc.contact_manifold(pairs=scene.pairs[:m], n_threads=threads)
    dt = time.perf_counter() - t0
    return m / dt, m, cores, dt


def run_reference_sdf(args):
    n_body = args.n_env or DEFAULT_NENV["SDF"]
    sc = make_scene("SDF", min(n_body, 65536), 0)
    from oracle import oracle as O
    osc = O.OracleScene(sc)
    P = sc.P

    def run(m):
        osc.sdf_eval(sc.point_shapes[:m], sc.point_poses[:m], sc.points[:m * P], P, want_pose=True)

    n = 64
    t0 = time.perf_counter()
    run(n)
    per = (time.perf_counter() - t0) / n
    m = int(max(n, min(len(sc.point_shapes), 150.0 / max(args.steps + args.warmup, 1) / max(per, 1e-9))))
    for _ in range(args.warmup):
        run(m)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(m)
    dt = (time.perf_counter() - t0) / args.steps
    val = m * P / dt
    line = {"impl": "reference", "metric": SDF_METRIC, "value": val, "unit": "points/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "SDF", "bodies_per_gpu": n_body, "points_per_body": P},
            "cpu_baseline": {"value": val, "unit": "points/s", "cores": O.max_threads(), "kind": "oracle",
                             "sample": "first %d bodies x %d points per step (FP64 jet oracle, OpenMP)" % (m, P)},
            "e2e": {"value": val, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload == "SDF":
        return run_reference_sdf(args)
    n_env = args.n_env or DEFAULT_NENV[args.workload]
    scene = make_scene(args.workload, min(n_env, 65536), 0)
    from oracle import oracle as O
    osc = O.OracleScene(scene)
    cores = O.max_threads()
    # each step: a bounded sample of the workload's pairs (same sample size
    # every step) sized so that W + K steps take a few minutes at most
    n = min(len(scene.pairs), max(cores, 8))
    t0 = time.perf_counter()
    osc.contact_manifold(pairs=scene.pairs[:n])
    per = (time.perf_counter() - t0) / n
    m = int(max(n, min(len(scene.pairs), 150.0 / max(args.steps + args.warmup, 1) / max(per, 1e-9))))
    sample = scene.pairs[:m]
    for _ in range(args.warmup):
        osc.contact_manifold(pairs=sample)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        osc.contact_manifold(pairs=sample)
    dt = (time.perf_counter() - t0) / args.steps
    val = m / dt
    line = {"impl": "reference", "metric": "contact-manifold evals/sec with derivatives (tier 2)", "value": val,
            "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "n_env_per_gpu": n_env, "tier": 2},
            "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                             "sample": "first %d pairs of %s per step (FP64 jet oracle, OpenMP over pairs)"
                                       % (m, args.workload)},
            "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _timed(step, args, stream, flush, world, local):
    """W warm-up steps, then K steps timed with CUDA events on the launching
    stream (L2 flushed before each), barrier + synchronize on both sides,
    clocks sampled during the timed region; returns (max-over-ranks ms per
    step, own kernel launches, clocks)."""
    import torch
    import torch.distributed as dist
    from paper_2604_17538_b200 import binding
    dev = torch.device("cuda", local)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = binding.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(float(i))
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    launches = binding.launch_count() - l0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = float(np.sum([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / args.steps, launches, clk


def _e2e_pipelined(run_step, h2d, d2h, steps, world, dev):
    """End-to-end loop through the public API with host buffers, double
    buffered: step i's host->device copy of its inputs (pinned) runs on an
    upload stream and step i-1's device->host read-back on a download stream,
    both overlapping step i's compute on the caller's stream (PCIe is full
    duplex).  h2d[s] = (device dst, pinned src), d2h[s] = (pinned dst, device
    src) for slot s in {0, 1}; run_step(s) enqueues the compute reading and
    writing slot s.  Every step copies its inputs and reads its result back;
    the time is from the first upload to the last read-back (CUDA events),
    max over ranks.  Returns ms per step."""
    import torch
    import torch.distributed as dist
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()
    ev_in, ev_comp, ev_out = [ev(), ev()], [ev(), ev()], [ev(), ev()]

    def go(n):
        for i in range(n):
            s = i % 2
            with torch.cuda.stream(up):
                if i >= 2:
                    up.wait_event(ev_comp[s])        # slot s inputs no longer read
                h2d[s][0].copy_(h2d[s][1], non_blocking=True)
                ev_in[s].record(up)
            comp.wait_event(ev_in[s])
            if i >= 2:
                comp.wait_event(ev_out[s])           # slot s result already read back
            run_step(s)
            ev_comp[s].record(comp)
            with torch.cuda.stream(down):
                down.wait_event(ev_comp[s])
                d2h[s][0].copy_(d2h[s][1], non_blocking=True)
                ev_out[s].record(down)
        for s in range(min(n, 2)):
            comp.wait_event(ev_out[s])

    go(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    up.wait_event(e0)
    go(steps)
    e1.record(comp)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    return float(te.item())


def run_sdf(args, sc, n_body, gen_s, world, rank, local):
    """Secondary metric: cm_sdf_eval of the 32 C5 SDF prototypes
    with value, gradient, Hessian and pose gradient at P points per body."""
    import torch
    import torch.distributed as dist
    from paper_2604_17538_b200 import binding
    dev = torch.device("cuda", local)
    S = binding.Scene(sc.shapes, sc.smooth, device=local)
    P = sc.P
    flags = binding.SDF_VALUE | binding.SDF_GRAD | binding.SDF_HESS | binding.SDF_POSE_GRAD
    ids = torch.from_numpy(sc.point_shapes).to(dev)
    poses = torch.from_numpy(sc.point_poses).to(dev)
    pts = torch.from_numpy(sc.points).to(dev)
    out = S.sdf_eval(ids, poses, pts, P, flags)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    ms, launches, clk = _timed(lambda: S.sdf_eval(ids, poses, pts, P, flags, out=out), args, stream, flush, world,
                               local)
    n_pts = len(sc.point_shapes) * P
    value = n_pts * world / (ms / 1e3)
    e2e = None
    if not args.no_e2e:
        pts_h = torch.from_numpy(sc.points).pin_memory()
        d_h = [torch.empty(n_pts, dtype=torch.float32).pin_memory() for _ in range(2)]
        pts_d = [torch.empty_like(pts) for _ in range(2)]
        outs = [out, {k: torch.empty_like(v) for k, v in out.items()}]
        ms_e = _e2e_pipelined(lambda s_: S.sdf_eval(ids, poses, pts_d[s_], P, flags, out=outs[s_]),
                              [(pts_d[k], pts_h) for k in range(2)], [(d_h[k], outs[k]["d"]) for k in range(2)],
                              args.steps, world, dev)
        e2e = {"value": n_pts * world / (ms_e / 1e3), "unit": "points/s",
               "h2d_bytes_per_step": int(pts_h.numel() * 4), "d2h_bytes_per_step": int(n_pts * 4),
               "pipeline": "double-buffered: upload / download streams overlap the compute"}
    with open(os.path.join(ROOT, "paper_2604_17538_b200", "costmodel.json")) as f:
        cm = json.load(f)
    names = [sc.shapes[i].name for i in range(len(sc.shapes))]
    cnt = np.bincount(sc.point_shapes, minlength=len(names))
    flop = float(sum(cnt[i] * P * cm["sdf"][names[i]]["order2"]["flop"] for i in range(len(names))))
    kern_s = ms / 1e3
    bytes_alg = n_pts * SDF_BYTES_PER_POINT + len(sc.point_shapes) * 36
    peaks, peak_src = load_peaks()
    achieved = flop / kern_s / 1e12
    hbm = bytes_alg / kern_s / 1e9
    roof = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP32_PEAK_TFLOPS, "traffic": None,
            "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md unit counts)",
            "flop_per_point": flop / n_pts, "flop_source": "costmodel.json order-2 evaluation FLOPs per shape",
            "hbm": {"achieved_gbs": hbm, "peak_gbs": peaks["hbm_gbs"], "frac": hbm / peaks["hbm_gbs"],
                    "bytes_alg": bytes_alg, "peak_source": peak_src}}
    if hbm / peaks["hbm_gbs"] > achieved / FP32_PEAK_TFLOPS:
        roof.update({"bound": "hbm", "achieved": hbm, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": hbm / peaks["hbm_gbs"]})
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        osc = O.OracleScene(sc)
        m = 256
        t0 = time.perf_counter()
        osc.sdf_eval(sc.point_shapes[:m], sc.point_poses[:m], sc.points[:m * P], P, want_pose=True)
        per = (time.perf_counter() - t0) / m
        m = int(max(m, min(len(sc.point_shapes), 15.0 / max(per, 1e-9))))
        t0 = time.perf_counter()
        osc.sdf_eval(sc.point_shapes[:m], sc.point_poses[:m], sc.points[:m * P], P, want_pose=True)
        dt = time.perf_counter() - t0
        cpu = {"value": m * P / dt, "unit": "points/s", "cores": O.max_threads(), "kind": "oracle",
               "sample": "first %d bodies x %d points of the SDF shard, FP64 jet oracle (with pose Hessians), "
                         "OpenMP, %.1f s" % (m, P, dt)}
    if rank == 0:
        line = {"metric": SDF_METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "SDF", "bodies_per_gpu": n_body, "points_per_body": P,
                           "l2": "flushed (256 MiB write) between steps",
                           "parallelism": "body-sharded dp%d, no data-path collective" % world,
                           "input_gen_s": round(gen_s, 1)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C5", "C4", "C3", "C2", "SDF", "C1"])
    ap.add_argument("--k", type=int, default=18, help="C3: number of SQs in the smooth union (P:200 sweep)")
    ap.add_argument("--n-env", type=int, default=0)
    ap.add_argument("--tier", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_17538_b200 import binding

    n_env = args.n_env or DEFAULT_NENV[args.workload]
    t0 = time.time()
    scene = make_scene(args.workload, n_env, rank * n_env, K=args.k)
    gen_s = time.time() - t0
    if args.workload == "SDF":
        return run_sdf(args, scene, n_env, gen_s, world, rank, local)
    S = binding.Scene(scene.shapes, scene.smooth, device=local)
    dev = torch.device("cuda", local)
    pairs = torch.from_numpy(scene.pairs).to(dev)
    poses = torch.from_numpy(scene.poses).to(dev)
    offs = S.manifold_offsets(pairs)
    C = S.manifold_size(scene.pairs)
    out = S.alloc_manifold(C, args.tier, dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)   # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream()

    def step():
        S.contact_manifold(pairs, offs, C, poses, args.tier, out)

    ms_per_step, launches, clk = _timed(step, args, stream, flush, world, local)
    n_pairs_all = len(scene.pairs) * world
    value = n_pairs_all / (ms_per_step / 1e3)

    # ---- end to end through the public API with host buffers --------------
    e2e = None
    if not args.no_e2e:
        poses_h = torch.from_numpy(scene.poses).pin_memory()
        depth_h = [torch.empty(C, dtype=torch.float32).pin_memory() for _ in range(2)]
        poses_d = [torch.empty_like(poses) for _ in range(2)]
        # slot 1 shares every output but the read-back field with slot 0
        outs = [out, dict(out, depth=torch.empty_like(out["depth"]))]
        ms_e = _e2e_pipelined(lambda s_: S.contact_manifold(pairs, offs, C, poses_d[s_], args.tier, outs[s_]),
                              [(poses_d[k], poses_h) for k in range(2)],
                              [(depth_h[k], outs[k]["depth"]) for k in range(2)], args.steps, world, dev)
        e2e = {"value": n_pairs_all / (ms_e / 1e3), "unit": "pairs/s",
               "h2d_bytes_per_step": int(poses_h.numel() * 4), "d2h_bytes_per_step": int(C * 4),
               "pipeline": "double-buffered: upload / download streams overlap the compute"}

    # ---- roofline of the manifold kernels ---------------------------------
    peaks, peak_src = load_peaks()
    n_pairs = len(scene.pairs)
    bytes_alg = n_pairs * IN_BYTES_PER_PAIR + C * OUT_BYTES_PER_CONTACT[args.tier]
    # the step is exactly the k_mf_* launches of one cm_contact_manifold call
    # (per chunk of units: vertices, traces, midpoints per SDF class, then
    # faces), timed together with CUDA events on the caller's stream; the
    # algorithmic FLOPs are those of the whole method, so the roofline covers
    # the kernels of the step together (per-kernel shares: profiles/traffic_*.json)
    kern_s = ms_per_step / 1e3
    hbm_gbs = bytes_alg / kern_s / 1e9
    flop_launch = flop_per_launch(args.workload, scene, S) if args.tier == 2 else None
    fpp = flop_launch / n_pairs if flop_launch else None
    if fpp:
        achieved = flop_launch / kern_s / 1e12
        traffic = None
        dominant = None
        tpath = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.workload.lower())
        if os.path.exists(tpath) and args.tier == 2:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj["bytes_per_pair"] * n_pairs   # measured DRAM bytes per step
            top = max(tj["kernels"], key=lambda k: k["share_of_chunk_time"])
            dominant = {"kernel": top["kernel"], "share_of_step": round(top["share_of_chunk_time"], 3),
                        "source": "ncu launch durations of one chunk (%s)" % os.path.basename(tpath)}
        roof = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic,
                "scope": "all k_mf_* kernels of the step (the step is exactly these launches)",
                "dominant_kernel": dominant,
                "traffic_unit": "bytes per step (ncu dram read + write of one chunk's kernels, cold-cache replays, "
                                "scaled per pair)",
                "bytes_alg": bytes_alg,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1965 MHz (B200_PROFILING.md unit counts)",
                "flop_per_pair": fpp, "flop_source": "costmodel.json (ncu-measured per-shape/order table, DESIGN.md §7)",
                "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"],
                                              "frac": hbm_gbs / peaks["hbm_gbs"], "peak_source": peak_src}}
    else:
        roof = {"bound": "hbm", "achieved": hbm_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_gbs / peaks["hbm_gbs"], "traffic": None, "peak_source": peak_src,
                "note": "FLOP/pair not yet frozen; HBM fraction of algorithmic bytes only"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, m, cores, dt = oracle_rate(scene, budget_s=20.0)
        cpu = {"value": rate, "unit": "pairs/s", "cores": cores, "kind": "oracle",
               "sample": "first %d pairs of the %s shard, FP64 jet oracle, OpenMP over pairs, %.1f s" % (m, args.workload, dt)}

    if rank == 0:
        line = {"metric": "contact-manifold evals/sec with derivatives (tier %d)" % args.tier, "value": value,
                "unit": "pairs/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": {"workload": args.workload, "n_env_per_gpu": n_env, "pairs_per_gpu": n_pairs,
                           "contacts_per_gpu": C, "tier": args.tier, "l2": "flushed (256 MiB write) between steps",
                           "parallelism": "env-sharded dp%d, no data-path collective" % world,
                           "input_gen_s": round(gen_s, 1)},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk}
        if args.workload == "C3" and args.k != 18:
            line["config"]["sqs_in_union"] = args.k
        if args.workload == "C1":   # latency-bound: report the per-call latency
            line["config"]["latency_us_per_call"] = ms_per_step * 1e3
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
