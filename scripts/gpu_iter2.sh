#!/bin/bash
# parity diag (TMA path, repeated) + full GPU tests + bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/diag.log
timeout 300 python scripts/diag_c3.py 4194304 > gpurun_out/diag.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status.txt
for w in c4 c1 c2 c3; do timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>/dev/null; done
timeout 300 python bench.py --no-cpu-baseline --workload c1 --format hdc --steps 10 --warmup 3 > gpurun_out/bench_c1_hdc.json 2>/dev/null
