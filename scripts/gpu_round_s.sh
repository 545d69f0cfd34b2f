#!/bin/bash
# Block-local interleaved rows for multi-block tiles (bl in {128, 256, 512}): same-box A/B
# against the previous build (libhdcgpu_head.so), then the GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s
O=gpurun_out/s
L=$PWD/paper_2105_04937_b200
python scripts/bw_probe.py > $O/bw.json 2>&1
for rep in 1 2; do
  for tag in head cur; do
    if [ $tag = cur ]; then lib=$L/libhdcgpu.so; else lib=$L/libhdcgpu_$tag.so; fi
    echo "# $tag" >> $O/ab.log
    HDCG_LIBRARY=$lib timeout 300 python scripts/shape_probe.py lap256_bl128 lap256_bl256 lap256_bl512 lap256_bl4096 >> $O/ab.log 2>>$O/ab.err
  done
done
timeout 1500 python -m pytest tests -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
