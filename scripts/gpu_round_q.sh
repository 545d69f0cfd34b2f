#!/bin/bash
# spmv_blk_kernel occupancy / ring-size A/B (HDCG_TMA_CTAS, HDCG_TMA_STAGE_KB), same box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/q
O=gpurun_out/q
python scripts/bw_probe.py > $O/bw.json 2>&1
for cfg in "3 0" "4 0" "2 0" "2 100" "4 40" "3 60"; do
  set -- $cfg
  if [ $2 = 0 ]; then unset HDCG_TMA_STAGE_KB; else export HDCG_TMA_STAGE_KB=$2; fi
  echo "# ctas=$1 stage_kb=$2" >> $O/ab.log
  HDCG_TMA_CTAS=$1 timeout 300 python scripts/shape_probe.py lap256_bl50 lap256_bl100 >> $O/ab.log 2>>$O/ab.err
done
echo done
