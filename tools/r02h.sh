set -u
O=gpurun_out/r02h
mkdir -p $O
timeout 600 python tools/diag_nan.py 1048576 227550,300596,604409 > $O/nan.json 2> $O/nan.err
timeout 900 python -m pytest tests/test_gpu_streams_shards.py tests/test_gpu_parity.py -q -x -k "streams or shard or C5 or c4 or band" > $O/t.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --workload C4 --no-cpu-baseline --no-e2e > $O/bench_c4.json 2> $O/bench_c4.err
echo done
