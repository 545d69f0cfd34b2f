#!/bin/bash
# Multi-block TMA tiles (bl in {128, 256, 512}): full GPU suite, then the config-1
# block-size sweep and the default config-4 line (regression check).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
for bl in 256 512 1024 4096 16384; do
  timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl $bl --steps 20 --warmup 3 > gpurun_out/bench_c1_bl$bl.json 2> gpurun_out/bench_c1_bl$bl.err
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1500 python -m pytest tests -q -m gpu -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
echo done
