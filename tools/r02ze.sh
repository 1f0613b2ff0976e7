#!/bin/bash
set -u
O=gpurun_out/r02ze; mkdir -p $O
XPSQCM_LIB=paper_2604_17538_b200/libxpsqcm.so timeout 600 python tools/out_hash.py > $O/hash_def.json 2>$O/hash_def.err
XPSQCM_LIB=exp/lib_l2p0.so timeout 600 python tools/out_hash.py > $O/hash_l2p0.json 2>$O/hash_l2p0.err
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02ze/hash_def.json")); b=json.load(open("gpurun_out/r02ze/hash_l2p0.json"))
d=[k for k in a if a[k]!=b.get(k)]
print("fields", len(a), len(b), "differ", len(d)); print("\n".join(d[:50]))
PY
WLS="C5 C4" bash tools/variant_sweep.sh r02ze 2 def l2p0 l2p768 l2p3072
