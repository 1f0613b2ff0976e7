#!/bin/bash
set -u
O=gpurun_out/r02za; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_streams_shards.py -q -x -k graph > $O/pytest_graph.txt 2>&1; echo "rc=$?" >> $O/pytest_graph.txt
timeout 300 python bench.py --workload C1 --steps 20 --warmup 5 > $O/bench_C1.json 2>$O/bench_C1.err
