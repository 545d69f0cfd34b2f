#!/bin/bash
# Remainder-mode tests, the config-3 overlap A/B, the config-1 block-size sweep and
# the CSR format lines (RP(M-HDC/CSR) on the device).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "remainder_paths or config3 or kernel_paths or policy" > gpurun_out/pytest_rest.log 2>&1; echo pytest=$? >> gpurun_out/pytest_rest.log
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 900 python scripts/c3_overlap_ab.py > gpurun_out/c3_overlap_ab.log 2>&1
for bl in 256 1024 16384; do
  timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl $bl --steps 20 --warmup 3 > gpurun_out/bench_c1_bl$bl.json 2> gpurun_out/bench_c1_bl$bl.err
done
for w in c1 c2 c3; do
  timeout 600 python bench.py --no-cpu-baseline --workload $w --format csr --steps 20 --warmup 3 > gpurun_out/bench_${w}_csr.json 2> gpurun_out/bench_${w}_csr.err
done
echo done
