#!/bin/bash
set -u
O=gpurun_out/r02zz; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python bench.py --workload C4 --e2e-steps 2 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
