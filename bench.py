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
collective on the data path; timing is max over ranks.  `--gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N
ranks (127.0.0.1).  Inputs (poses, pairs, offsets) are resident in HBM for
`value`; `e2e` re-times the step through the public API with the poses
copied host->device from pinned memory and EVERY output field of the tier
copied back device->host (the whole manifold, in 8 sub-batches so the
copies of one sub-batch overlap the compute of the next on separate upload /
download streams); `e2e_depth_only` is the same loop reading back only the
fused depths.  L2 is flushed (256 MiB write) between timed steps.  With
N > 1 the optional NCCL all-gather of the tier-0 fields is timed separately
(`allgather`), never inside `value`.
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
FP32_PEAK_DERIVED_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4 at the 1965 MHz max SM clock
XU_PEAK_DERIVED_TOPS = 148 * 16 * 1.965e9 / 1e12           # 4.65 (16 MUFU lanes per SM per clock)


def load_alu_peaks():
    """FP32 and MUFU/XU peaks measured on a B200 of this pool by the K5
    microbenchmarks (tools/k5_peaks.cu -> profiles/peaks_fp32_xu.json);
    the spec arithmetic when that file is missing (say which)."""
    p = os.path.join(ROOT, "profiles", "peaks_fp32_xu.json")
    if os.path.exists(p):
        with open(p) as f:
            k = json.load(f)
        return (k["fp32_tflops"], k["xu_tops"],
                "measured: tools/k5_peaks.cu FFMA / MUFU chains on a B200 (profiles/peaks_fp32_xu.json, %s)" % k["when"])
    return FP32_PEAK_DERIVED_TFLOPS, XU_PEAK_DERIVED_TOPS, "derived: 148 SM x 128 FP32 / 16 MUFU lanes x 1965 MHz"


def _cost_key(workload, shape, kind):
    if workload == "C5":
        return shape.name
    if workload not in ("C1", "C2", "C3", "C4"):
        return None   # (no frozen cost entries: HBM roof only)
    if kind == "sdf":
        return {"C1": "C1:", "C2": "C2:", "C3": "C3:", "C4": "C4:"}[workload] + (
            {"blob18": "blob18"}.get(shape.name, shape.name))
    return {"C2": "C2:", "C3": "C3:", "C4": "C4:", "C1": "C1:"}[workload] + shape.name


def flop_per_launch(workload, scene, S):
    """Algorithmic work of one tier-2 call over scene.pairs from the frozen
    cost table: (FP32 FLOPs, MUFU ops of the SDF evaluations).  The MUFU
    count covers the (V + E) second-order and 2 E (iters - 1) first-order
    evaluations of the SDF side only (the table has no MUFU count of the
    manifold's own gates and softmax)."""
    with open(os.path.join(ROOT, "paper_2604_17538_b200", "costmodel.json")) as f:
        cm = json.load(f)
    hs1, hs2 = cm["halfspace_eval"]["order1"], cm["halfspace_eval"]["order2"]
    it = scene.smooth["trace_iters"]
    total = mufu = 0.0
    a_ids, b_ids = scene.pairs[:, 3], scene.pairs[:, 4]
    keys, counts = np.unique(np.stack([a_ids, b_ids], 1), axis=0, return_counts=True)
    for (a, b), n in zip(keys, counts):
        sa, sb = scene.shapes[a], scene.shapes[b]
        ka, kb = _cost_key(workload, sa, "mesh"), _cost_key(workload, sb, "sdf")
        if ka is None or kb is None or ka not in cm["manifold_with_halfspace"] or kb not in cm["sdf"]:
            return None, None
        V, E, F = S.counts(int(a))
        c = cm["manifold_with_halfspace"][ka]["flop_per_pair_total_with_halfspace"]
        c += (V + E) * (cm["sdf"][kb]["order2"]["flop"] - hs2) + 2 * E * (it - 1) * (cm["sdf"][kb]["order1"]["flop"] - hs1)
        total += n * c
        mufu += n * ((V + E) * cm["sdf"][kb]["order2"]["mufu"] + 2 * E * (it - 1) * cm["sdf"][kb]["order1"]["mufu"])
    return total, mufu


def roofline(flop, mufu, bytes_alg, kern_s, peaks, peak_src, extra=None):
    """The three roofs of SURVEY §8(d) (FP32 pipe, MUFU/XU pipe, HBM), each
    achieved = algorithmic work / time and frac = achieved / measured peak;
    `bound` is the roof with the largest fraction (the binding one)."""
    fp32_peak, xu_peak, alu_src = load_alu_peaks()
    roofs = {}
    if flop:
        a = flop / kern_s / 1e12
        roofs["fp32"] = {"achieved": a, "peak": fp32_peak, "unit": "TFLOP/s", "frac": a / fp32_peak,
                         "peak_source": alu_src}
    if mufu:
        a = mufu / kern_s / 1e12
        roofs["xu"] = {"achieved": a, "peak": xu_peak, "unit": "Tops/s", "frac": a / xu_peak, "peak_source": alu_src,
                       "scope": "MUFU ops of the SDF evaluations (cost table); the manifold's gates not counted"}
    a = bytes_alg / kern_s / 1e9
    roofs["hbm"] = {"achieved": a, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": a / peaks["hbm_gbs"],
                    "peak_source": "%s (MEASURED_PEAKS.json hbm_gbs)" % peak_src, "bytes_alg": bytes_alg}
    name = max(roofs, key=lambda k: roofs[k]["frac"])
    b = roofs[name]
    out = {"bound": {"fp32": "alu", "xu": "alu", "hbm": "hbm"}[name], "binding_roof": name,
           "achieved": b["achieved"], "peak": b["peak"], "unit": b["unit"], "frac": b["frac"],
           "peak_source": b["peak_source"], "traffic": None, "roofs": roofs}
    if extra:
        out.update(extra)
    return out


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


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
    if workload == "C6":
        return synth.c6_scene(n_env, env_lo=env_lo)
    raise SystemExit("unknown workload " + workload)


DEFAULT_NENV = {"C5": 1 << 20, "C4": 1 << 16, "C3": 1 << 14, "C2": 1000, "SDF": 1 << 18, "C1": 1, "C6": 4096}
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
    mode = 16 if args.broad else 0
    n = min(len(scene.pairs), max(cores, 8))
    t0 = time.perf_counter()
    osc.contact_manifold(pairs=scene.pairs[:n], mode=mode)
    per = (time.perf_counter() - t0) / n
    m = int(max(n, min(len(scene.pairs), 150.0 / max(args.steps + args.warmup, 1) / max(per, 1e-9))))
    sample = scene.pairs[:m]
    for _ in range(args.warmup):
        osc.contact_manifold(pairs=sample, mode=mode)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        osc.contact_manifold(pairs=sample, mode=mode)
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


def c1_graph_latency(step, args, dev):
    """Per-call latency of the same call captured once into a CUDA graph and
    replayed (C1 is launch-bound: ~11 kernels for 2 pairs); CUDA events
    around each replay on the current stream, median over K."""
    import torch
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(max(args.warmup, 3)):
        g.replay()
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(max(args.steps, 20)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


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
                for dst, src in (d2h[s] if isinstance(d2h[s], list) else [d2h[s]]):
                    dst.copy_(src, non_blocking=True)
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
        pts_d = [torch.empty_like(pts) for _ in range(2)]
        outs = [out, {k: torch.empty_like(v) for k, v in out.items()}]
        host = [{k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in out.items()} for _ in range(2)]
        ms_e = _e2e_pipelined(lambda s_: S.sdf_eval(ids, poses, pts_d[s_], P, flags, out=outs[s_]),
                              [(pts_d[k], pts_h) for k in range(2)],
                              [[(host[k][f], outs[k][f]) for f in out] for k in range(2)], args.steps, world, dev)
        e2e = {"value": n_pts * world / (ms_e / 1e3), "unit": "points/s",
               "h2d_bytes_per_step": int(pts_h.numel() * 4),
               "d2h_bytes_per_step": int(sum(v.numel() * v.element_size() for v in out.values())),
               "readback": "every output field (d, grad, hess, dpose)",
               "pipeline": "double-buffered: upload / download streams overlap the compute"}
    with open(os.path.join(ROOT, "paper_2604_17538_b200", "costmodel.json")) as f:
        cm = json.load(f)
    names = [sc.shapes[i].name for i in range(len(sc.shapes))]
    cnt = np.bincount(sc.point_shapes, minlength=len(names))
    flop = float(sum(cnt[i] * P * cm["sdf"][names[i]]["order2"]["flop"] for i in range(len(names))))
    mufu = float(sum(cnt[i] * P * cm["sdf"][names[i]]["order2"]["mufu"] for i in range(len(names))))
    kern_s = ms / 1e3
    bytes_alg = n_pts * SDF_BYTES_PER_POINT + len(sc.point_shapes) * 36
    peaks, peak_src = load_peaks()
    roof = roofline(flop, mufu, bytes_alg, kern_s, peaks, peak_src,
                    {"flop_per_point": flop / n_pts, "flop_source": "costmodel.json order-2 evaluation FLOPs per shape",
                     "scope": "every k_sdf_eval launch of the step (one per SDF class present)"})
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


def maybe_spawn(args):
    """`python bench.py --gpus N` outside torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (rendezvous on
    127.0.0.1).  Returns True when this process only spawned the ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    s = __import__("socket").socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd)
    if r.returncode:
        raise SystemExit(r.returncode)
    return True


def dry_run(args):
    """Process-group plumbing only (no GPU work): every rank reports its
    RANK / LOCAL_RANK / WORLD_SIZE; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    me = {"rank": rank, "local_rank": int(os.environ.get("LOCAL_RANK", "0")), "world": world,
          "env_range": [rank * (args.n_env or DEFAULT_NENV[args.workload]),
                        (rank + 1) * (args.n_env or DEFAULT_NENV[args.workload])]}
    ranks = [me]
    if world > 1:
        dist.init_process_group("gloo")
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        me["max_over_ranks"] = float(t.item())
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_full(S, scene, args, world, dev, n_sub=8):
    """End to end through the public API with host buffers: each step uploads
    the poses from pinned memory and reads EVERY output field of the tier back
    into pinned memory, in n_sub env sub-batches pipelined over an upload, a
    compute and a download stream (sub-batch i's read-back overlaps sub-batch
    i+1's compute).  Returns (ms per step, h2d bytes, d2h bytes)."""
    import torch
    import torch.distributed as dist
    from paper_2604_17538_b200 import binding
    n_env = scene.poses.shape[0]
    bounds = np.linspace(0, n_env, n_sub + 1).astype(np.int64)
    subs = []
    for i in range(n_sub):
        e0, e1 = int(bounds[i]), int(bounds[i + 1])
        m = (scene.pairs[:, 0] >= e0) & (scene.pairs[:, 0] < e1)
        pr = scene.pairs[m].copy()
        pr[:, 0] -= e0
        pairs_d = torch.from_numpy(pr).to(dev)
        C = S.manifold_size(pr)
        subs.append(dict(e0=e0, e1=e1, pairs=pairs_d, offs=S.manifold_offsets(pairs_d), C=C))
    subs = [x for x in subs if x["C"] > 0]   # (tiny workloads: empty sub-batches)
    Cmax = max(x["C"] for x in subs)
    nmax = max(x["e1"] - x["e0"] for x in subs)
    poses_h = torch.from_numpy(scene.poses).pin_memory()
    # flat per-field buffers; sub-batch b uses the contiguous [rows, C_b]
    # prefix view (the library's field stride is the call's n_contacts)
    proto = S.alloc_manifold(1, args.tier, dev)
    rows = {k: (v.shape[0] if v.dim() == 2 else 1) for k, v in proto.items()}
    dev_flat = [{k: torch.empty(rows[k] * Cmax, dtype=v.dtype, device=dev) for k, v in proto.items()}
                for _ in range(2)]
    host_flat = [{k: torch.empty(rows[k] * Cmax, dtype=v.dtype).pin_memory() for k, v in proto.items()}
                 for _ in range(2)]
    view = lambda buf, k, C: buf[k][:rows[k] * C].view(rows[k], C) if proto[k].dim() == 2 else buf[k][:C]
    dev_poses = [torch.empty((nmax,) + tuple(scene.poses.shape[1:]), dtype=torch.float32, device=dev)
                 for _ in range(2)]
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in, ev_comp, ev_out = ([torch.cuda.Event() for _ in range(2)] for _ in range(3))

    def go(steps):
        j = 0
        for _ in range(steps):
            for sb in subs:
                s_ = j % 2
                n, C = sb["e1"] - sb["e0"], sb["C"]
                with torch.cuda.stream(up):
                    if j >= 2:
                        up.wait_event(ev_comp[s_])           # slot s_ poses no longer read
                    dev_poses[s_][:n].copy_(poses_h[sb["e0"]:sb["e1"]], non_blocking=True)
                    ev_in[s_].record(up)
                comp.wait_event(ev_in[s_])
                if j >= 2:
                    comp.wait_event(ev_out[s_])              # slot s_ outputs already read back
                out = {k: view(dev_flat[s_], k, C) for k in proto}
                S.contact_manifold(sb["pairs"], sb["offs"], C, dev_poses[s_][:n], args.tier, out,
                                   binding.BROAD_PHASE if args.broad else 0)
                ev_comp[s_].record(comp)
                with torch.cuda.stream(down):
                    down.wait_event(ev_comp[s_])
                    for k in proto:
                        host_flat[s_][k][:rows[k] * C].copy_(dev_flat[s_][k][:rows[k] * C], non_blocking=True)
                    ev_out[s_].record(down)
                j += 1
        for s_ in range(2):
            comp.wait_event(ev_out[s_])

    go(1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    up.wait_event(e0)
    steps = max(1, min(args.steps, args.e2e_steps))
    go(steps)
    e1.record(comp)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    h2d = int(scene.poses.nbytes)
    per_contact = sum(v.element_size() * rows[k] for k, v in proto.items())
    d2h = int(sum(x["C"] for x in subs) * per_contact)
    return float(te.item()), h2d, d2h, steps


def allgather_tier0(out, C, world, dev):
    """Optional NCCL all-gather of the tier-0 fields (point, normal, depth) of
    every rank over NVLink, timed separately from the step."""
    import torch
    import torch.distributed as dist
    C_all = torch.tensor([C], dtype=torch.int64, device=dev)
    dist.all_reduce(C_all, op=dist.ReduceOp.MAX)
    Cm = int(C_all.item())
    send = torch.zeros(7, Cm, dtype=torch.float32, device=dev)
    send[0:3, :C] = out["point"]
    send[3:6, :C] = out["normal"]
    send[6, :C] = out["depth"]
    recv = torch.empty(world * 7 * Cm, dtype=torch.float32, device=dev)
    dist.all_gather_into_tensor(recv, send.reshape(-1))
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        dist.all_gather_into_tensor(recv, send.reshape(-1))
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 3], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    nbytes = world * 7 * Cm * 4
    return {"fields": "point, normal, depth (tier 0, 28 B per contact)", "bytes_gathered_per_rank": nbytes,
            "ms": ms, "recv_gbs_per_rank": (world - 1) / world * nbytes / (ms / 1e3) / 1e9,
            "note": "timed separately (max over ranks); not part of value"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C5", "C4", "C3", "C2", "SDF", "C1", "C6"])
    ap.add_argument("--broad", action="store_true", help="CM_BROAD_PHASE (f2): certified pair culling")
    ap.add_argument("--k", type=int, default=18, help="C3: number of SQs in the smooth union (P:200 sweep)")
    ap.add_argument("--n-env", type=int, default=0)
    ap.add_argument("--tier", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5, help="steps of the full-readback e2e loop (PCIe-bound)")
    ap.add_argument("--no-allgather", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="process-group plumbing only (CPU tests)")
    args = ap.parse_args()
    if maybe_spawn(args):
        return
    if args.dry_run:
        return dry_run(args)
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
    mode = binding.BROAD_PHASE if args.broad else 0

    def step():
        S.contact_manifold(pairs, offs, C, poses, args.tier, out, mode)

    ms_per_step, launches, clk = _timed(step, args, stream, flush, world, local)
    n_pairs_all = len(scene.pairs) * world
    graph_us = c1_graph_latency(step, args, dev) if args.workload == "C1" else None
    value = n_pairs_all / (ms_per_step / 1e3)

    gather = None
    if world > 1 and not args.no_allgather:
        gather = allgather_tier0(out, C, world, dev)

    # ---- end to end through the public API with host buffers --------------
    e2e = e2e_depth = None
    if not args.no_e2e:
        del flush
        ms_e, h2d, d2h, e_steps = e2e_full(S, scene, args, world, dev)
        e2e = {"value": n_pairs_all / (ms_e / 1e3), "unit": "pairs/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e_steps,
               "readback": "every tier-%d output field (the whole manifold)" % args.tier,
               "pipeline": "8 env sub-batches per step; upload / compute / download streams overlap"}
        poses_h = torch.from_numpy(scene.poses).pin_memory()
        depth_h = [torch.empty(C, dtype=torch.float32).pin_memory() for _ in range(2)]
        poses_d = [torch.empty_like(poses) for _ in range(2)]
        # slot 1 shares every output but the read-back field with slot 0
        outs = [out, dict(out, depth=torch.empty_like(out["depth"]))]
        ms_d = _e2e_pipelined(lambda s_: S.contact_manifold(pairs, offs, C, poses_d[s_], args.tier, outs[s_], mode),
                              [(poses_d[k], poses_h) for k in range(2)],
                              [(depth_h[k], outs[k]["depth"]) for k in range(2)], args.steps, world, dev)
        e2e_depth = {"value": n_pairs_all / (ms_d / 1e3), "unit": "pairs/s",
                     "h2d_bytes_per_step": int(poses_h.numel() * 4), "d2h_bytes_per_step": int(C * 4),
                     "readback": "fused depths only (4 of %d B per contact)" % OUT_BYTES_PER_CONTACT[args.tier]}

    # ---- roofline of the step's kernels ------------------------------------
    peaks, peak_src = load_peaks()
    n_pairs = len(scene.pairs)
    bytes_alg = n_pairs * IN_BYTES_PER_PAIR + C * OUT_BYTES_PER_CONTACT[args.tier]
    kern_s = ms_per_step / 1e3
    flop_launch, mufu_launch = flop_per_launch(args.workload, scene, S) if args.tier == 2 else (None, None)
    extra = {"scope": "every k_mf_* kernel of the step together (the step is exactly these launches)"}
    if flop_launch:
        extra.update({"flop_per_pair": flop_launch / n_pairs, "mufu_per_pair_sdf": mufu_launch / n_pairs,
                      "flop_source": "costmodel.json: frozen per-(shape, order) FP32 op table (DESIGN.md §7)"})
    roof = roofline(flop_launch, mufu_launch, bytes_alg, kern_s, peaks, peak_src, extra)
    tpath = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.workload.lower())
    if os.path.exists(tpath) and args.tier == 2:
        with open(tpath) as f:
            tj = json.load(f)
        roof["traffic"] = tj["bytes_per_pair"] * n_pairs   # measured DRAM bytes per step
        roof["traffic_unit"] = ("bytes per step (ncu dram read + write of one chunk's kernels, cold-cache replays, "
                                "scaled per pair; %s)" % os.path.basename(tpath))
        top = max(tj["kernels"], key=lambda k: k["share_of_chunk_time"])
        roof["dominant_kernel"] = {"kernel": top["kernel"], "share_of_step": round(top["share_of_chunk_time"], 3),
                                   "source": "ncu launch durations of one chunk (%s)" % os.path.basename(tpath)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, m, cores, dt = oracle_rate(scene, budget_s=20.0)
        rate1, m1, _, dt1 = oracle_rate(scene, budget_s=4.0, threads=1, max_pairs=256)
        cpu = {"value": rate, "unit": "pairs/s", "cores": cores, "kind": "oracle",
               "sample": "first %d pairs of the %s shard, FP64 jet oracle, OpenMP over pairs, %.1f s"
                         % (m, args.workload, dt),
               "single_thread": {"value": rate1, "sample": "first %d pairs, 1 thread, %.1f s" % (m1, dt1)}}
        cpu.update(cpu_info())

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
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_depth_only": e2e_depth,
                "gpu_launches": int(launches), "clocks": clk}
        if gather:
            line["allgather"] = gather
        if args.broad:
            line["config"]["broad_phase"] = "CM_BROAD_PHASE (certified pair culling, DESIGN.md reading #46)"
            line["config"]["culled_fraction"] = float((out["dom"] == -2).float().mean().item())
        if args.workload == "C3" and args.k != 18:
            line["config"]["sqs_in_union"] = args.k
        if args.workload == "C1":   # latency-bound: report the per-call latency
            line["config"]["latency_us_per_call"] = ms_per_step * 1e3
            if graph_us is not None:
                line["config"]["latency_us_per_call_cuda_graph"] = graph_us
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
