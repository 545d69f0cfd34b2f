#!/bin/bash
# full GPU tests, bench lines, c3 launch list (rest_kernel vs TMA kernel split)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
timeout 1500 python -m pytest tests -q -m gpu -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/ab.log
for w in c1 c4 c2 c3; do
  timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'], d['e2e']['value'])" >> gpurun_out/ab.log
done
CMD="python bench.py --workload c3 --steps 3 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rest_kernel|spmv_tma" --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_c3.log 2>&1
