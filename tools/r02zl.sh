#!/bin/bash
set -u
O=gpurun_out/r02zl; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python bench.py --workload SDF > $O/bench_SDF.json 2> $O/bench_SDF.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
