#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 1 -c 1 -o gpurun_out/prof_c3_v6 $CMD > gpurun_out/ncu_c3.log 2>&1
