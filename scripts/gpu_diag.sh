#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "44 4" "44 3" "64 3"; do set -- $cfg
  echo "== STAGE_KB=$1 CTAS=$2" >> gpurun_out/diag.log
  HDCG_TMA_STAGE_KB=$1 HDCG_TMA_CTAS=$2 timeout 300 python scripts/diag_c3.py 4194304 >> gpurun_out/diag.log 2>&1
done
