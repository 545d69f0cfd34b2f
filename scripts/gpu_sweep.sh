#!/bin/bash
# TMA kernel tuning sweep (stage KB x CTAs/SM) on c1 and c4, then ncu of c4 and c3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "kernel_paths or golden or acceptance or config3" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status.txt
for kb in 32 64 96; do for c in 2 3; do
  HDCG_TMA_STAGE_KB=$kb HDCG_TMA_CTAS=$c timeout 300 python bench.py --no-cpu-baseline --workload c1 --steps 20 --warmup 3 > gpurun_out/sweep_c1_${kb}_${c}.json 2>/dev/null
  HDCG_TMA_STAGE_KB=$kb HDCG_TMA_CTAS=$c timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/sweep_c4_${kb}_${c}.json 2>/dev/null
done; done
timeout 300 python bench.py --no-cpu-baseline --workload c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline --workload c2 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2>/dev/null
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 1 -c 1 -o gpurun_out/prof_c4_tma $CMD > gpurun_out/ncu_c4.log 2>&1
CMD3="python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 1 -c 1 -o gpurun_out/prof_c3_tma $CMD3 > gpurun_out/ncu_c3.log 2>&1
echo done >> gpurun_out/status.txt
