set -u
O=gpurun_out/r02d
mkdir -p $O
timeout 600 python tools/diag_det.py 131072 > $O/diag.json 2> $O/diag.err
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
bash tools/prof.sh r02d C5
echo done
