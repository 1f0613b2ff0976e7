set -u
O=gpurun_out/r02c
mkdir -p $O
free -g > $O/free.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 2 > $O/bench_c5.json 2> $O/bench_c5.err
echo done
