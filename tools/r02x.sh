set -u
O=gpurun_out/r02x
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "broad or pair_reduce" > $O/t.txt 2>&1
timeout 600 python bench.py --workload C6 --no-cpu-baseline --no-e2e > $O/bench_c6.json 2> $O/bench_c6.err
timeout 600 python bench.py --workload C6 --broad --no-cpu-baseline --no-e2e > $O/bench_c6_broad.json 2> $O/bench_c6_broad.err
timeout 600 python bench.py --workload C6 --impl reference --steps 2 --warmup 1 > $O/ref_c6.json 2> $O/ref_c6.err
timeout 600 python bench.py --workload C6 --broad --impl reference --steps 2 --warmup 1 > $O/ref_c6_broad.json 2> $O/ref_c6_broad.err
echo done
