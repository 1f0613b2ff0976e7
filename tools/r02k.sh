set -u
O=gpurun_out/r02k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_streams_shards.py tests/test_abi.py -q -x > $O/t.txt 2>&1
bash tools/variant_sweep.sh r02k 2 r1 def e0 f0 g0
echo done
