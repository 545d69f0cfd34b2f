#!/bin/bash
# gpu_ncu_knob.sh KNOB v1,v2,... : DRAM bytes / time of one config-4 SpMV launch per knob value (ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ncu_knob_$1.log
rm -f $out
timeout 300 python scripts/c4_once.py > gpurun_out/c4_once_plain.log 2>&1 || exit 1
for v in ${2//,/ }; do
  echo "$1=$v" >> $out
  env $1=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmv_tma -s 1 -c 1 --csv python scripts/c4_once.py 2>&1 | grep -v "^==" | grep "Command line" | sed 's/.*metrics",//' >> $out
done
echo done
