#!/bin/bash
# Profile capture on the GPU box: launch list of a short default bench and
# one `ncu --set full` capture (with source) of the first chunk's manifold
# kernels of a 65k-env C5 shard.  Usage: bash tools/prof.sh <tag> [C5|C4]
set -u
T=$1; W=${2:-C5}
O=gpurun_out/$T
mkdir -p $O
N=65536; [ "$W" = "C4" ] && N=4096
CMD="python bench.py --workload $W --n-env $N --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain_$W.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_mf_ -c 16 \
  -o $O/manifold_$W -f $CMD > $O/ncu_full_$W.log 2>&1
echo prof-done
