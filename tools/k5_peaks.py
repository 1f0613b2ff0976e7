#!/usr/bin/env python
"""K5 peak microbenchmarks: runs tools/k5_peaks (built
from tools/k5_peaks.cu, `python tools/k5_peaks.py --build` here) on the GPU
box with nvidia-smi clocks sampled during the run, and writes
profiles/peaks_fp32_xu.json:
  fp32_tflops  best FFMA-chain rate (2 FLOP per FFMA) -- the FP32 roof
  xu_tops      best MUFU-chain rate (ex2 / lg2 / rcp / rsqrt; 1 op each) -- the XU roof
plus every variant, the clocks seen and the derived per-clock rates.
bench.py reads this file for its FP32 / XU roofline denominators."""
from __future__ import annotations

import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "k5_peaks.cu")
BIN = os.path.join(HERE, "k5_peaks")


def build():
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-o", BIN, SRC])


def main():
    if "--build" in sys.argv:
        build()
        return
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "profiles",
                                                                                            "peaks_fp32_xu.json")
    lines = []
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                            "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    th = threading.Thread(target=lambda: [lines.append(l.strip()) for l in smi.stdout], daemon=True)
    th.start()
    time.sleep(0.3)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    time.sleep(0.3)
    smi.terminate()
    if r.returncode != 0:
        raise SystemExit("k5_peaks failed: " + r.stderr)
    res = json.loads(r.stdout)
    sm = []
    for l in lines:
        p = [x.strip() for x in l.split(",")]
        try:
            sm.append(float(p[0]))
        except (ValueError, IndexError):
            pass
    sm_load = sorted(sm)[len(sm) // 2] if sm else None
    k = res["kernels"]
    fp32 = max(k[n]["rate"] for n in ("ffma_reg", "ffma_imm", "ffma_mix"))
    xu = max(k[n]["rate"] for n in ("ex2", "lg2", "rcp", "rsqrt", "ex2_lg2"))
    doc = {"fp32_tflops": fp32 / 1e12, "xu_tops": xu / 1e12,
           "how": "tools/k5_peaks.cu: 148 x 8 CTAs x 256 threads, 8 independent chains per thread, "
                  "CUDA events over 10 launches, best of 2 rounds; FFMA = 2 FLOP, MUFU op = 1",
           "sm_mhz_median_during": sm_load, "sm_mhz_samples": len(sm), "variants": k, "sms": res["sms"],
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    if sm_load:
        for n, v in k.items():
            v["per_clk_per_sm_at_measured_clock"] = v["rate"] / (res["sms"] * sm_load * 1e6)
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
