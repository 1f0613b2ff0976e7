#!/bin/bash
# Round bench lines (GPU box): every workload's bench line, the C5 N_env
# sweep, the C3 K sweep, the reference (oracle) arm.
# Usage: bash tools/final_bench.sh <tag>
set -u
T=$1
O=gpurun_out/$T
mkdir -p $O
nvidia-smi -q | grep -E "Product Name|Driver Version" > $O/box.txt 2>&1
timeout 900 python bench.py > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python bench.py --tier 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5_t3.json 2> $O/bench_C5_t3.err
timeout 900 python bench.py --workload C4 --tier 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C4_t3.json 2> $O/bench_C4_t3.err
for w in C4 C3 C2 C1 SDF; do
  timeout 900 python bench.py --workload $w --e2e-steps 2 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 python bench.py --workload C6 --e2e-steps 2 > $O/bench_C6.json 2> $O/bench_C6.err
timeout 900 python bench.py --workload C6 --broad --e2e-steps 2 > $O/bench_C6_broad.json 2> $O/bench_C6_broad.err
for n in 1024 4096 16384 65536 262144 1048576; do
  timeout 600 python bench.py --n-env $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> $O/c5_nenv_sweep.jsonl 2>> $O/sweep.err
done
for k in 1 2 4 8 12 18; do
  timeout 600 python bench.py --workload C3 --k $k --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> $O/c3_k_sweep.jsonl 2>> $O/sweep.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
echo final-done
