#!/bin/bash
# spmv_blk_kernel with the next tile's first x gathers issued before this tile's sums
# (second run: REST == 1 included -- the lap256 small-block cases carry a light remainder)
# (HDCG_BLK_XPIPE=1) against without (=0, the v21 behaviour) on one box, then parity.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/z2
O=gpurun_out/z2
python scripts/bw_probe.py > $O/bw.json 2>&1
for rep in 1 2; do
  for p in 0 1; do
    echo "# XPIPE=$p" >> $O/ab.log
    HDCG_BLK_XPIPE=$p timeout 300 python scripts/shape_probe.py lap256_bl100 lap256_bl200 lap256_bl50 lap256_bl10 lap256_bl128 >> $O/ab.log 2>>$O/ab.err
  done
done
timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl 100 --steps 20 --warmup 3 > $O/bench_c1_bl100.json 2> $O/bench_c1_bl100.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "kernel_paths or remainder or blk_tiles or golden or slab or block_range or cross_tile" > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
