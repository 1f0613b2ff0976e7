#!/usr/bin/env python
"""Registers / stack / spills per kernel from `nvcc -Xptxas -v` (one .cu of
the library), compact:  python tools/ptxas_table.py [file.cu] [-DFOO ...]
[--src-dir DIR] (DIR: a csrc tree to compile instead of the in-tree one)."""
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(ROOT, "paper_2604_17538_b200", "csrc")
args = sys.argv[1:]
if "--src-dir" in args:
    CSRC = args[args.index("--src-dir") + 1]
src = next((a for a in args if a.endswith(".cu")), "cm_kernels_manifold.cu")
defs = [a for a in args if a.startswith("-D")]
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
       "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, *defs, "-c", os.path.join(CSRC, src),
       "-o", "/tmp/ptxas_table_%d.o" % os.getpid()]
r = subprocess.run(cmd, capture_output=True, text=True)
name = None
rows = []
stack = spill = None
for line in r.stderr.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        name = name.replace("(MfArgs)", "").replace("void ", "")
        stack = spill = None
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        stack, spill = int(m.group(1)), int(m.group(2)) + int(m.group(3))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        rows.append((name, int(m.group(1)), stack, spill))
        name = None
for n, reg, st, sp in sorted(rows):
    print("%-60s regs %3d stack %5s spill %5s" % (n[:60], reg, st, sp))
if r.returncode:
    print(r.stderr[-3000:])
