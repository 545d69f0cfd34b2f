#!/bin/bash
# Re-entry check: GPU parity suite, smoke, and a default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo done
