#!/bin/bash
set -u
O=gpurun_out/r02z3; mkdir -p $O
for v in e1 nf0; do
  XPSQCM_LIB=exp/lib_$v.so timeout 600 python tools/out_hash.py > $O/hash_$v.json 2>$O/hash_$v.err
done
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02z3/hash_e1.json")); b=json.load(open("gpurun_out/r02z3/hash_nf0.json"))
d=[k for k in a if a[k]!=b.get(k)]
print("fields", len(a), len(b), "differ", len(d)); print("\n".join(d[:80]))
PY
for v in e1 nf0; do
  for w in C5 C4; do
    N=65536; [ $w = C4 ] && N=4096
    CMD="python bench.py --workload $w --n-env $N --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
    XPSQCM_LIB=exp/lib_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_${v}_$w.csv $CMD > /dev/null 2>&1
  done
done
XPSQCM_LIB=exp/lib_e1.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mf_edges -c 3 -o $O/edges_C5 -f python bench.py --workload C5 --n-env 16384 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
XPSQCM_LIB=exp/lib_e1.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mf_edges -c 1 -o $O/edges_C4 -f python bench.py --workload C4 --n-env 4096 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_full4.log 2>&1
for r in edges_C5 edges_C4; do
  python tools/ncu_summary.py $O/$r.ncu-rep > $O/${r}_summary.txt 2>&1
  python tools/ncu_lines.py $O/$r.ncu-rep k_mf_edges 40 > $O/${r}_lines.txt 2>&1
done
rm -f $O/*.ncu-rep
echo done
