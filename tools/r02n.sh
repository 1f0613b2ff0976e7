set -u
O=gpurun_out/r02n
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
bash tools/variant_sweep.sh r02n 2 def nf
echo done
