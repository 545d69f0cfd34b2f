#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 600 python scripts/c4_drift.py > gpurun_out/c4_drift.log 2>&1
python scripts/bw_probe.py >> gpurun_out/bw.json 2>&1
echo done
