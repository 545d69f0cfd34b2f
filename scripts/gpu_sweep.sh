#!/bin/bash
# TMA kernel tuning sweep (ring KB x CTAs/SM) on c1, c4 and c3, after the parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status.txt
for cfg in "32 3" "48 3" "64 3" "48 4" "40 4"; do set -- $cfg; kb=$1; c=$2
  HDCG_TMA_STAGE_KB=$kb HDCG_TMA_CTAS=$c timeout 300 python bench.py --no-cpu-baseline --workload c1 --steps 20 --warmup 3 > gpurun_out/sweep_c1_${kb}_${c}.json 2>/dev/null
  HDCG_TMA_STAGE_KB=$kb HDCG_TMA_CTAS=$c timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/sweep_c4_${kb}_${c}.json 2>/dev/null
  HDCG_TMA_STAGE_KB=$kb HDCG_TMA_CTAS=$c timeout 300 python bench.py --no-cpu-baseline --workload c3 --steps 10 --warmup 3 > gpurun_out/sweep_c3_${kb}_${c}.json 2>/dev/null
done
timeout 300 python bench.py --no-cpu-baseline --workload c2 --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline --workload c1 --format hdc --steps 20 --warmup 3 > gpurun_out/bench_c1_hdc.json 2>/dev/null
echo done >> gpurun_out/status.txt
