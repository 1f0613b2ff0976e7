#!/bin/bash
set -u
T=$1
O=gpurun_out/$T
mkdir -p $O
CMD="python bench.py --workload SDF --n-env 65536 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain_sdf.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sdf_eval -c 3 \
  -o $O/sdf -f $CMD > $O/ncu_sdf.log 2>&1
echo prof-done
