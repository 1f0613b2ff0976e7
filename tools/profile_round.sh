#!/bin/bash
# Round profile capture (run on the GPU box via gpurun):
#   bench lines (C5 default, C4, reference arm), the ncu launch list of the
#   default bench command, and one `ncu --set full` capture of the manifold
#   kernels on a 65k-env C5 shard.  Output: gpurun_out/<tag>/
#   ONLY_FULL=1: just the ncu --set full capture; SKIP_FULL=1: everything else.
set -u
T=${1:-rXX}
O=gpurun_out/$T
mkdir -p $O
python -m paper_2604_17538_b200.build > $O/build.log 2>&1 || exit 1
if [ -z "${ONLY_FULL:-}" ]; then
nvidia-smi -q | grep -E "Product Name|Driver Version|CUDA Version|Max Clocks" -A0 > $O/box.txt 2>&1
timeout 600 python bench.py > $O/bench_c5_1M.json 2> $O/bench_c5_1M.err
timeout 600 python bench.py --workload C4 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload SDF > $O/bench_sdf.json 2> $O/bench_sdf.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
fi
[ -n "${SKIP_FULL:-}" ] && { echo done; exit 0; }
# the 11 manifold kernels of the first chunk (unit set-up; vertices, traces,
# midpoints for the three SDF classes of C5; faces), then C4's 8 (two classes)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mf_ -c 11 \
  -o $O/manifold -f python bench.py --n-env 65536 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_mf_ -c 8 \
  -o $O/manifold_c4 -f python bench.py --workload C4 --n-env 4096 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_full_c4.log 2>&1
echo done
