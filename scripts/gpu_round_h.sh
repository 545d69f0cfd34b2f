#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -rf -k "kernel_paths or remainder_paths or policy or config3 or slab or power" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/shape_probe.py > gpurun_out/shape_probe.log 2>&1
echo done
