#!/bin/bash
# Final round-1 evidence with the current library: GPU suite + smoke, every bench
# line (default with the CPU baseline, reference arm, config sweeps, CSR, small
# blocks), the config-4 launch list and one ncu --set full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fin
O=gpurun_out/fin
python scripts/bw_probe.py > $O/bw.json 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for bl in 100 256 512 1024 4096 16384; do
  timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl $bl --steps 20 --warmup 3 > $O/bench_c1_bl$bl.json 2> $O/bench_c1_bl$bl.err
done
timeout 600 python bench.py --no-cpu-baseline --workload c1 --format hdc --steps 20 --warmup 3 > $O/bench_c1_hdc.json 2> $O/bench_c1_hdc.err
timeout 600 python bench.py --no-cpu-baseline --workload c2 --steps 20 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --no-cpu-baseline --workload c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --no-cpu-baseline --workload c3 --bl 1024 --steps 20 --warmup 3 > $O/bench_c3_bl1024.json 2> $O/bench_c3_bl1024.err
HDCG_R4_MAXSEG=8 timeout 600 python bench.py --no-cpu-baseline --workload c3 --steps 20 --warmup 3 > $O/bench_c3_r4max8.json 2> $O/bench_c3_r4max8.err
HDCG_R4_MAXSEG=8 timeout 600 python bench.py --no-cpu-baseline --workload c3 --bl 1024 --steps 20 --warmup 3 > $O/bench_c3_bl1024_r4max8.json 2> $O/bench_c3_bl1024_r4max8.err
for w in c1 c2 c3; do
  timeout 600 python bench.py --no-cpu-baseline --workload $w --format csr --steps 20 --warmup 3 > $O/bench_${w}_csr.json 2> $O/bench_${w}_csr.err
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 3 -c 1 -o $O/prof_c4 $CMD > $O/ncu_full.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo done
