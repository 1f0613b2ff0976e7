set -u
O=gpurun_out/r02t
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sdf" > $O/t.txt 2>&1
timeout 600 python bench.py --workload SDF --no-cpu-baseline > $O/bench_sdf.json 2> $O/bench_sdf.err
echo done
