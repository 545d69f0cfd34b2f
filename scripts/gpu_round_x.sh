#!/bin/bash
# spmv_blk_kernel with P tiles per stage (bl = 100/200: 5 tiles, 4 rows/thread): A/B
# against one tile per stage (HDCG_BLK_P=1, the v20 behaviour) on one box, then parity.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/x
O=gpurun_out/x
python scripts/bw_probe.py > $O/bw.json 2>&1
for rep in 1 2; do
  for p in 1 auto; do
    echo "# P=$p" >> $O/ab.log
    if [ $p = auto ]; then unset HDCG_BLK_P; else export HDCG_BLK_P=$p; fi
    timeout 300 python scripts/shape_probe.py lap256_bl100 lap256_bl200 lap256_bl96 lap256_bl150 >> $O/ab.log 2>>$O/ab.err
  done
done
unset HDCG_BLK_P
timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl 100 --steps 20 --warmup 3 > $O/bench_c1_bl100.json 2> $O/bench_c1_bl100.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "kernel_paths or remainder or blk_tiles or golden or slab or block_range" > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
