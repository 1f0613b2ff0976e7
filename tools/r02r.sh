set -u
O=gpurun_out/r02r
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_streams_shards.py -q -x -k "sdf or invalid or shard" > $O/t.txt 2>&1
WLS="SDF C5 C4" bash tools/variant_sweep.sh r02r 2 def sxi
echo done
