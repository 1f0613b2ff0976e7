#!/bin/bash
set -u
O=gpurun_out/r02z6; mkdir -p $O
CMD="python bench.py --workload C5 --n-env 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_mf_ -c 11 -o $O/c5 -f $CMD > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/c5.ncu-rep > $O/summary.txt 2>&1
for k in "k_mf_traces<2, 0>" "k_mf_faces" "k_mf_midpoints<2, 0" "k_mf_traces<2, 1>" "k_mf_traces<2, 4>"; do
  python tools/ncu_lines.py $O/c5.ncu-rep "$k" 45 >> $O/lines.txt 2>&1
done
python tools/ncu_traffic.py $O/c5.ncu-rep $O/traffic.json C5 11 > /dev/null 2>&1
ls -la $O
