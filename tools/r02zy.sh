#!/bin/bash
set -u
O=gpurun_out/r02zy; mkdir -p $O
for r in 1 2; do
  for v in def t3r168 t3r128; do
    L=exp/lib_$v.so; [ $v = def ] && L=paper_2604_17538_b200/libxpsqcm.so
    for w in C5 C4; do
      line=$(XPSQCM_LIB=$L timeout 600 python bench.py --workload $w --tier 3 --n-env $([ $w = C5 ] && echo 262144 || echo 16384) --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>>$O/err.log | tail -1)
      echo "{\"variant\": \"$v\", \"round\": $r, \"workload\": \"$w\", \"line\": $line}" >> $O/sweep.jsonl
    done
  done
done
