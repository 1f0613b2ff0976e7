#!/bin/bash
# C3 runtime versus the number of SQs in the smooth union (the paper's
# geometry-complexity axis): one bench line per K on the GPU box.
for K in 1 2 4 8 12 18; do
  timeout 600 python bench.py --workload C3 --k $K --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | tail -1
done
