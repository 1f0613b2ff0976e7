set -u
O=gpurun_out/r02l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
bash tools/variant_sweep.sh r02l 2 def h0 e0 t32 t128
echo done
