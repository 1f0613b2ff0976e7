#!/bin/bash
set -u
O=gpurun_out/r02z7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "node_pose or param_grad" > $O/pytest_np.txt 2>&1; echo "rc=$?" >> $O/pytest_np.txt
cp gpurun_out/parity_sdf_node_pose_grad.json $O/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
