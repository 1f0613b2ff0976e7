#!/bin/bash
set -u
O=gpurun_out/r02zz2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "param_vjp_cup" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
cp gpurun_out/parity_manifold_param_vjp_cup.json $O/ 2>/dev/null
