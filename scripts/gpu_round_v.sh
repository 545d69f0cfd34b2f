#!/bin/bash
# Tile layout 4 (bl = 128 without remainder: one warp per block, rows lane + 32 r): A/B vs head (v19).
# layout 3, W = bl/128 warps per block) vs layout 3 for bl = 256 only (head).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v
O=gpurun_out/v
L=$PWD/paper_2105_04937_b200
python scripts/bw_probe.py > $O/bw.json 2>&1
for rep in 1 2; do
  for tag in head cur; do
    if [ $tag = cur ]; then lib=$L/libhdcgpu.so; else lib=$L/libhdcgpu_$tag.so; fi
    echo "# $tag" >> $O/ab.log
    HDCG_LIBRARY=$lib timeout 300 python scripts/shape_probe.py lap256_bl128 lap256_bl256 >> $O/ab.log 2>>$O/ab.err
  done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "kernel_paths or remainder or random_sweep or power or slab or block_range" > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
