#!/bin/bash
set -u
O=gpurun_out/r02zq; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "broad_phase" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
