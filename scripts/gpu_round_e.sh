#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 600 python scripts/shape_probe.py > gpurun_out/shape_probe.log 2>&1
timeout 900 python scripts/mm_bench.py 128 > gpurun_out/mm_bench.log 2>&1
echo done
