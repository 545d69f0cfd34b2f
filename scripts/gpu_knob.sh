#!/bin/bash
# gpu_knob.sh KNOB v1,v2 workloads... -> gpurun_out/knob_<KNOB>.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 1500 python scripts/knob_ab.py "$@" > gpurun_out/knob_$1.log 2>&1
echo done
