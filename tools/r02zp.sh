#!/bin/bash
set -u
O=gpurun_out/r02zp; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_c5t3.csv python bench.py --tier 3 --n-env 262144 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
