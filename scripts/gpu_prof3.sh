#!/bin/bash
# Bench + one ncu --set full capture per workload of the TMA kernel (c4, c2, c3).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "kernel_paths or golden or acceptance or config3 or config2" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status.txt
for w in c4 c1 c2 c3; do timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>/dev/null; done
for w in c4 c2 c3; do
  CMD="python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline"
  timeout 600 $CMD > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 1 -c 1 -o gpurun_out/prof_${w}_v3 $CMD > gpurun_out/ncu_$w.log 2>&1
done
echo done >> gpurun_out/status.txt
