#!/bin/bash
set -u
O=gpurun_out/r02z5; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
WLS="C5 C4 C3 SDF" bash tools/variant_sweep.sh r02z5 2 def
