#!/bin/bash
# Config-4 evidence after the bench.py e2e fix: default bench line (with the
# reference CPU baseline), bench contract tests, launch list, ncu --set full.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
O=gpurun_out/ev
python scripts/bw_probe.py > $O/bw2.json 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python -m pytest tests/test_bench_gpu.py -q -x -rf > $O/pytest_bench.log 2>&1; echo pytest=$? >> $O/pytest_bench.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 3 -c 1 -o $O/prof_c4 $CMD > $O/ncu_full.log 2>&1
echo done
