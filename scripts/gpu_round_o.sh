#!/bin/bash
# spmv_blk_kernel with the remainder probe one tile ahead: GPU suite, small-bl
# A/B vs the general kernel, config-4 regression check, ncu of the bl=100 launch.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/o
O=gpurun_out/o
python scripts/bw_probe.py > $O/bw.json 2>&1
for blk in 0 1; do
  HDCG_BLK=$blk timeout 300 python scripts/shape_probe.py lap256_bl10 lap256_bl50 lap256_bl100 lap256_bl200 lap256_bl96 lap256_bl128 lap256_bl512 >> $O/ab.log 2>>$O/ab.err
done
timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_blk -s 3 -c 1 -o $O/prof_blk100 python scripts/shape_probe.py lap256_bl100 > $O/ncu_blk.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
