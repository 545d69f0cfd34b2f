#!/bin/bash
# Same-box A/B of two builds: libhdcgpu_base.so (A) vs libhdcgpu.so (B), alternating processes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/lib_ab.log
python scripts/bw_probe.py > $out 2>&1
for rep in 1 2 3; do
  HDCG_LIBRARY=$PWD/paper_2105_04937_b200/libhdcgpu_base.so timeout 300 python scripts/lib_ab.py base >> $out 2>&1
  timeout 300 python scripts/lib_ab.py new >> $out 2>&1
done
echo done
