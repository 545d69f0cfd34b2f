#!/bin/bash
# Evidence for profiles/: the default bench line (N=1, with CPU baseline), its ncu
# launch list, and one ncu --set full capture of the SpMV kernel of the same command.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/bw_probe.py > gpurun_out/bw.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for w in c1 c2 c3; do timeout 600 python bench.py --no-cpu-baseline --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
timeout 600 python bench.py --no-cpu-baseline --workload c1 --format hdc --steps 20 --warmup 3 > gpurun_out/bench_c1_hdc.json 2> gpurun_out/bench_c1_hdc.err
timeout 600 python bench.py --no-cpu-baseline --workload c3 --bl 1024 --steps 20 --warmup 3 > gpurun_out/bench_c3_bl1024.json 2> gpurun_out/bench_c3_bl1024.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 3 -c 1 -o gpurun_out/prof_c4_final $CMD > gpurun_out/ncu_full.log 2>&1
echo done
