#!/bin/bash
set -u
O=gpurun_out/r02zw; mkdir -p $O
for v in def cat1; do
  L=exp/lib_$v.so; [ $v = def ] && L=paper_2604_17538_b200/libxpsqcm.so
  XPSQCM_LIB=$L timeout 600 python tools/out_hash.py > $O/hash_$v.json 2>$O/hash_$v.err
done
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02zw/hash_def.json")); b=json.load(open("gpurun_out/r02zw/hash_cat1.json"))
d=[k for k in a if a[k]!=b.get(k)]
print("fields", len(a), len(b), "differ", len(d), d[:5])
PY
WLS="C4 C6 C5" bash tools/variant_sweep.sh r02zw 2 def cat1
