set -u
O=gpurun_out/r02m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sdf_eval or C5 or c4" > $O/t.txt 2>&1
WLS="C5 C4 SDF" bash tools/variant_sweep.sh r02m 2 def e0 sxp2
echo done
