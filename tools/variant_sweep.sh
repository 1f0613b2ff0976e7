#!/bin/bash
# Build-knob A/B sweep on the GPU box: each variant library (built here with
# -D defines into exp/lib_<name>.so; "def" = the in-tree library) benches the
# C5 and C4 workloads (a "ch<N>" variant sets CM_CHUNK_UNITS=N), interleaved over R rounds so clock drift hits every
# variant alike.  Usage: tools/variant_sweep.sh <tag> <R> def cs0 fm1 ...
set -u
T=$1; R=$2; shift 2
O=gpurun_out/$T
mkdir -p $O
for r in $(seq 1 $R); do
  for v in "$@"; do
    # "def": the in-tree library; "ch<N>": it with CM_CHUNK_UNITS=N; else exp/lib_<v>.so
    E=""
    case $v in
      def) L=paper_2604_17538_b200/libxpsqcm.so ;;
      ch*) L=paper_2604_17538_b200/libxpsqcm.so; E="CM_CHUNK_UNITS=${v#ch}" ;;
      *) L=exp/lib_$v.so ;;
    esac
    for w in ${WLS:-C5 C4}; do
      line=$(env $E XPSQCM_LIB=$L timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>>$O/err.log | tail -1)
      echo "{\"variant\": \"$v\", \"round\": $r, \"workload\": \"$w\", \"line\": $line}" >> $O/sweep.jsonl
    done
  done
done
echo done
