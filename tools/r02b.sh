set -u
O=gpurun_out/r02b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --workload C4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
echo done
