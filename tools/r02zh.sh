#!/bin/bash
set -u
O=gpurun_out/r02zh; mkdir -p $O
bash tools/prof_sdf.sh r02zh
python tools/ncu_summary.py $O/sdf.ncu-rep > $O/sdf_ncu.txt 2>&1
python tools/ncu_lines.py $O/sdf.ncu-rep k_sdf_eval 40 > $O/sdf_lines.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sdf_launches.csv python bench.py --workload SDF --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
rm -f $O/sdf.ncu-rep
