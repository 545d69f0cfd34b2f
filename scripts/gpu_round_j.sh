#!/bin/bash
# Interleaved row mapping: same-box A/B vs the previous build (libhdcgpu_head.so),
# ncu L1/DRAM metrics of one config-4 launch, GPU suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/round_j.log
python scripts/bw_probe.py > $out 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum
L=$PWD/paper_2105_04937_b200
timeout 300 python scripts/c4_once.py > gpurun_out/c4_once_plain.log 2>&1 && \
for tag in head cur; do
  if [ $tag = cur ]; then lib=$L/libhdcgpu.so; else lib=$L/libhdcgpu_$tag.so; fi
  echo "ncu $tag" >> $out
  HDCG_LIBRARY=$lib timeout 600 ncu --metrics $M --clock-control none -k regex:spmv_tma -s 1 -c 1 --csv python scripts/c4_once.py 2>&1 | grep "Command line" | sed 's/.*metrics",//' >> $out
done
for rep in 1 2 3; do
  HDCG_LIBRARY=$L/libhdcgpu_head.so timeout 300 python scripts/lib_ab.py head >> $out 2>&1
  timeout 300 python scripts/lib_ab.py cur >> $out 2>&1
done
timeout 1500 python -m pytest tests -q -m gpu -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/shape_probe.py > gpurun_out/shape_probe.log 2>&1
echo done
