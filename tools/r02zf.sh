#!/bin/bash
set -u
O=gpurun_out/r02zf; mkdir -p $O
XPSQCM_LIB=paper_2604_17538_b200/libxpsqcm.so timeout 600 python tools/out_hash.py > $O/hash_def.json 2>$O/hash_def.err
XPSQCM_LIB=exp/lib_tp0.so timeout 600 python tools/out_hash.py > $O/hash_tp0.json 2>$O/hash_tp0.err
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02zf/hash_def.json")); b=json.load(open("gpurun_out/r02zf/hash_tp0.json"))
d=[k for k in a if a[k]!=b.get(k)]
print("fields", len(a), len(b), "differ", len(d)); print("\n".join(d[:50]))
PY
WLS="C5 C4 C3" bash tools/variant_sweep.sh r02zf 2 def tp0
