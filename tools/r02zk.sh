#!/bin/bash
set -u
O=gpurun_out/r02zk3; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams_shards.py -q -x -k "sdf" > $O/pytest_sdf.txt 2>&1; echo "rc=$?" >> $O/pytest_sdf.txt
WLS="SDF" bash tools/variant_sweep.sh r02zk3 3 def dy0 t64 dy0t64 old0
