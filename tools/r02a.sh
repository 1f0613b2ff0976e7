set -u
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi -q | grep -E "Product Name|Driver Version|Max Clocks" -A0 > $O/box.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; nproc >> $O/lscpu.txt
python tools/k5_peaks.py --out $O/peaks_fp32_xu.json > $O/k5.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1
timeout 600 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
echo done
