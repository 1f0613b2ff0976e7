#!/bin/bash
set -u
O=gpurun_out/r02zo; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_streams_shards.py tests/test_tessellate.py -q > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
