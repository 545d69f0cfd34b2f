#!/bin/bash
# spmv_blk_kernel v2 (tile-uniform range test, offsets/values by pointer): small-bl
# shape probe (blk on/off), ncu of the bl=100 launch, GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/p
O=gpurun_out/p
python scripts/bw_probe.py > $O/bw.json 2>&1
for blk in 1 0; do
  HDCG_BLK=$blk timeout 300 python scripts/shape_probe.py lap256_bl10 lap256_bl50 lap256_bl100 lap256_bl200 lap256_bl96 >> $O/ab.log 2>>$O/ab.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_blk -s 3 -c 1 -o $O/prof_blk100 python scripts/shape_probe.py lap256_bl100 > $O/ncu_blk.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
