#!/bin/bash
set -u
O=gpurun_out/r02zm; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_c4.csv python bench.py --workload C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
