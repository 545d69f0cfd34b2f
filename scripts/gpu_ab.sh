#!/bin/bash
# A/B of TMA-kernel variants on ONE box (env knobs), with the box's copy bandwidth.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
python scripts/bw_probe.py >> gpurun_out/ab.log 2>&1
run() {  # label, workload, env...
  local label=$1; shift; local w=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$w', d['value'], d['roofline']['frac'])" >> gpurun_out/ab.log
}
for w in c1 c4; do
  run default $w
  run susp100 $w HDCG_TMA_SUSPEND_NS=100
  run susp500 $w HDCG_TMA_SUSPEND_NS=500
  run susp2000 $w HDCG_TMA_SUSPEND_NS=2000
  run kb70_c3 $w HDCG_TMA_STAGE_KB=70 HDCG_TMA_CTAS=3
  run kb70_c3_s500 $w HDCG_TMA_STAGE_KB=70 HDCG_TMA_CTAS=3 HDCG_TMA_SUSPEND_NS=500
  run kb96_c2_s500 $w HDCG_TMA_STAGE_KB=100 HDCG_TMA_CTAS=2 HDCG_TMA_SUSPEND_NS=500
  run kb35_c4 $w HDCG_TMA_STAGE_KB=35
done
