set -u
O=gpurun_out/r02g
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 600 python tools/diag_det.py 1048576 > $O/diag_1M.json 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 2 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --workload C4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
echo done
