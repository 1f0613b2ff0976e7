#!/bin/bash
set -u
O=gpurun_out/r02zu; mkdir -p $O
for v in def cat2 cat4; do
  L=exp/lib_$v.so; [ $v = def ] && L=paper_2604_17538_b200/libxpsqcm.so
  XPSQCM_LIB=$L timeout 600 python tools/out_hash.py > $O/hash_$v.json 2>$O/hash_$v.err
done
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02zu/hash_def.json"))
for v in ("cat2","cat4"):
    b=json.load(open("gpurun_out/r02zu/hash_%s.json"%v))
    d=[k for k in a if a[k]!=b.get(k)]
    print(v, "fields", len(a), len(b), "differ", len(d), d[:5])
PY
WLS="C5 C4 C3" bash tools/variant_sweep.sh r02zu 2 def cat2 cat4
