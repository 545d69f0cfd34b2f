#!/bin/bash
# Fused scale/norm cost (c1, c4) and the config-1 small-block bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 900 python scripts/fusion_ab.py > gpurun_out/fusion_ab.log 2>&1
for bl in 256 512; do
  timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl $bl --steps 20 --warmup 3 > gpurun_out/bench_c1_bl$bl.json 2> gpurun_out/bench_c1_bl$bl.err
done
echo done
