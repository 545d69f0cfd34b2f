#!/bin/bash
# Same-box A/B of library builds (config 4 fused SpMV time + DRAM bytes of one launch).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/hist_ab.log
python scripts/bw_probe.py > $out 2>&1
L=$PWD/paper_2105_04937_b200
for rep in 1 2; do
  for tag in 753df94 ebfb500 base cur; do
    if [ $tag = cur ]; then lib=$L/libhdcgpu.so; else lib=$L/libhdcgpu_$tag.so; fi
    HDCG_LIBRARY=$lib timeout 300 python scripts/lib_ab.py $tag >> $out 2>&1
  done
done
for tag in 753df94 ebfb500 base cur; do
  if [ $tag = cur ]; then lib=$L/libhdcgpu.so; else lib=$L/libhdcgpu_$tag.so; fi
  echo "ncu $tag" >> $out
  HDCG_LIBRARY=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmv_tma -s 1 -c 1 --csv python scripts/c4_once.py 2>&1 | grep -v "^==" | tail -5 >> $out
done
echo done
