set -u
O=gpurun_out/r02w
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
bash tools/prof.sh r02w C5
echo done
