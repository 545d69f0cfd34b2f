#!/bin/bash
# A/B of TMA-kernel variants on ONE box (env knobs), with the box's copy bandwidth.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab.log gpurun_out/diag.log
python scripts/bw_probe.py >> gpurun_out/ab.log 2>&1
timeout 300 python scripts/diag_c3.py 4194304 > gpurun_out/diag.log 2>&1
run() {  # label, workload, env...
  local label=$1; shift; local w=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$w', d['value'], d['roofline']['frac'])" >> gpurun_out/ab.log
}
for w in c1 c2 c4 c3; do
  run cmax1 $w HDCG_TMA_CMAX=1
  run cmax4 $w HDCG_TMA_CMAX=4
  run general $w HDCG_KERNEL_POLICY=1
done
CMD="python bench.py --workload c4 --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_tma -s 1 -c 1 -o gpurun_out/prof_c4_v4 $CMD > gpurun_out/ncu_c4.log 2>&1
