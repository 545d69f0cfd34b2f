#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/diag.log
for cfg in "44 4" "44 3"; do set -- $cfg
  echo "== STAGE_KB=$1 CTAS=$2" >> gpurun_out/diag.log
  HDCG_TMA_STAGE_KB=$1 HDCG_TMA_CTAS=$2 timeout 300 python scripts/diag_c3.py 4194304 >> gpurun_out/diag.log 2>&1
done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status.txt
for w in c4 c1 c2 c3; do timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>/dev/null; done
