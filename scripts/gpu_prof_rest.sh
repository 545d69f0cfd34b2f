#!/bin/bash
# One ncu --set full capture of rest_kernel and of the TMA kernel on config 3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline"
TAG=${1:-v7}
timeout 600 $CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rest_kernel|spmv_tma" -s 2 -c 2 -o gpurun_out/prof_c3_$TAG $CMD > gpurun_out/ncu_c3.log 2>&1
echo ncu=$? >> gpurun_out/ncu_c3.log
