#!/bin/bash
# Odd-bl TMA path: GPU suite, shape probe, c4 regression line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/shape_probe.py > gpurun_out/shape_probe.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo done
