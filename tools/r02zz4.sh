#!/bin/bash
set -u
O=gpurun_out/r02zz4; mkdir -p $O
XPSQCM_LIB=paper_2604_17538_b200/libxpsqcm.so timeout 600 python tools/out_hash.py > $O/hash_def.json 2>$O/hash_def.err
XPSQCM_LIB=exp/lib_l1p0.so timeout 600 python tools/out_hash.py > $O/hash_l1p0.json 2>$O/hash_l1p0.err
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02zz4/hash_def.json")); b=json.load(open("gpurun_out/r02zz4/hash_l1p0.json"))
d=[k for k in a if a[k]!=b.get(k)]
print("fields", len(a), len(b), "differ", len(d), d[:5])
PY
WLS="C5 C3 C2" bash tools/variant_sweep.sh r02zz4 2 def l1p0 l1p2
