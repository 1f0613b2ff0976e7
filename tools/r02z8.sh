#!/bin/bash
set -u
O=gpurun_out/r02z8; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "param_vjp or node_pose or param_grad" > $O/pytest_vjp.txt 2>&1; echo "rc=$?" >> $O/pytest_vjp.txt
cp gpurun_out/parity_manifold_param_vjp_m*.json $O/ 2>/dev/null
