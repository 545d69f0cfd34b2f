#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/round_i.log
python scripts/bw_probe.py > $out 2>&1
timeout 300 python scripts/c4_once.py > gpurun_out/c4_once_plain.log 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmv_tma -s 1 -c 1 --csv python scripts/c4_once.py 2>&1 | grep "Command line" | sed 's/.*metrics",//' >> $out
L=$PWD/paper_2105_04937_b200
for rep in 1 2; do
  HDCG_LIBRARY=$L/libhdcgpu_ebfb500.so timeout 300 python scripts/lib_ab.py ebfb500 >> $out 2>&1
  timeout 300 python scripts/lib_ab.py cur >> $out 2>&1
done
timeout 1500 python -m pytest tests -q -m gpu -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
echo done
