#!/bin/bash
# spmv_blk_kernel at 4 CTAs per SM (64 registers; the default now for instances that fit)
# against 3 (HDCG_TMA_CTAS=3, the v21 occupancy), then the small-block parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ac
O=gpurun_out/ac
for rep in 1 2; do
  for c in 3 0; do
    echo "# CTAS=$c (0 = default)" >> $O/ab.log
    if [ $c = 0 ]; then unset HDCG_TMA_CTAS; else export HDCG_TMA_CTAS=$c; fi
    timeout 300 python scripts/shape_probe.py lap256_bl100 lap256_bl200 lap256_bl50 lap256_bl10 lap256_bl96 >> $O/ab.log 2>>$O/ab.err
  done
done
unset HDCG_TMA_CTAS
timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl 100 --steps 20 --warmup 3 > $O/bench_c1_bl100.json 2> $O/bench_c1_bl100.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "kernel_paths or remainder or blk or golden or slab or block_range or several_tiles" > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
