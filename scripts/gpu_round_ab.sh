#!/bin/bash
# spmv_blk_kernel occupancy / ring-depth sweep (HDCG_TMA_CTAS x HDCG_TMA_STAGE_KB) on config 1's
# small-block cases, one box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
O=gpurun_out/ab
for c in 3 2 1; do
  for kb in 0 24 40 100; do
    echo "# CTAS=$c STAGE_KB=$kb" >> $O/ab.log
    if [ $kb = 0 ]; then unset HDCG_TMA_STAGE_KB; else export HDCG_TMA_STAGE_KB=$kb; fi
    HDCG_TMA_CTAS=$c timeout 200 python scripts/shape_probe.py lap256_bl100 lap256_bl50 >> $O/ab.log 2>>$O/ab.err
  done
done
echo done
