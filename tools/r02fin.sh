#!/bin/bash
# final tree: GPU suite, smoke, every bench line, launch list, ncu capture + traffic
set -u
O=gpurun_out/r02fin
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
bash tools/final_bench.sh r02fin
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
CMD="python bench.py --workload C5 --n-env 65536 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_mf_ -c 11 -o $O/manifold_C5 -f $CMD > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/manifold_C5.ncu-rep > $O/manifold_ncu.txt 2>&1
python tools/ncu_traffic.py $O/manifold_C5.ncu-rep $O/traffic_c5.json C5 11 > /dev/null 2>&1
python tools/ncu_lines.py $O/manifold_C5.ncu-rep "k_mf_faces" 40 > $O/faces_lines.txt 2>&1
rm -f $O/manifold_C5.ncu-rep
echo done
