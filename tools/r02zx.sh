#!/bin/bash
set -u
O=gpurun_out/r02zx; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
WLS="C5 C4 C6" bash tools/variant_sweep.sh r02zx 2 def
