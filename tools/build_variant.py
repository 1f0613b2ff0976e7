"""Build a variant of the library for A/B sweeps (tools/variant_sweep.sh):
  python tools/build_variant.py <name> [--src <csrc dir>] [-DFOO=1 ...]
-> exp/lib_<name>.so (exp/ is git-ignored; it travels to the GPU box)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name = sys.argv[1]
args = sys.argv[2:]
src = os.path.join(ROOT, "paper_2604_17538_b200", "csrc")
if "--src" in args:
    src = args[args.index("--src") + 1]
defs = [a for a in args if a.startswith("-D")]
bdir = os.path.join(ROOT, "exp", "b_" + name)
os.makedirs(bdir, exist_ok=True)
NVCC = "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + src, "-I" + os.path.join(ROOT, "include")]
srcs = ["cm_kernels_sdf.cu", "cm_kernels_manifold.cu", "cm_kernels_misc.cu", "cm_host.cpp", "cm_tessellate.cpp"]


def run(f):
    o = os.path.join(bdir, f + ".o")
    subprocess.check_call([NVCC, *ARCH, *COMMON, *defs, "-c", os.path.join(src, f), "-o", o])
    return o


with ThreadPoolExecutor(4) as ex:
    objs = list(ex.map(run, srcs))
lib = os.path.join(ROOT, "exp", "lib_%s.so" % name)
subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs])
print(lib)
