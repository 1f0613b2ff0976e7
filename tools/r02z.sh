#!/bin/bash
# edge-kernel fusion: bitwise A/B against the unfused build, then the sweep
set -u
O=gpurun_out/r02z; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/box.txt
for v in e1 nf0; do
  L=exp/lib_$v.so
  XPSQCM_LIB=$L timeout 600 python tools/out_hash.py > $O/hash_$v.json 2>$O/hash_$v.err
done
python - <<'PY' > $O/hash_cmp.txt
import json
a=json.load(open("gpurun_out/r02z/hash_e1.json")); b=json.load(open("gpurun_out/r02z/hash_nf0.json"))
d=[k for k in a if a[k]!=b.get(k)]
print("fields", len(a), "differ", len(d)); print("\n".join(d[:50]))
PY
WLS="C5 C4" bash tools/variant_sweep.sh r02z2 2 nf0 e1 e1r96 e1s
