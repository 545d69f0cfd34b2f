#!/bin/bash
# One build->measure iteration: GPU parity tests, then bench lines for every workload.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -rf --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$? >> gpurun_out/status.txt
for w in c1 c2 c3; do timeout 600 python bench.py --no-cpu-baseline --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$? >> gpurun_out/status.txt; done
timeout 600 python bench.py --no-cpu-baseline --workload c1 --format hdc --steps 20 --warmup 3 > gpurun_out/bench_c1_hdc.json 2> gpurun_out/bench_c1_hdc.err
cat gpurun_out/status.txt
