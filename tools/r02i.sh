set -u
O=gpurun_out/r02i
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "band or cusp or near or xpsq" > $O/t.txt 2>&1
timeout 600 python tools/diag_det.py 1048576 > $O/diag_1M.json 2>&1
bash tools/variant_sweep.sh r02i 2 r1 def nostage
echo done
