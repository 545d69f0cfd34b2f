#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in c4 c3; do
  CMD="python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 1 -c 1 -o gpurun_out/prof_${w}_v5 $CMD > gpurun_out/ncu_$w.log 2>&1
done
