#!/bin/bash
# A/B of TMA-kernel variants on ONE box (env knobs), with the box's copy bandwidth.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
python scripts/bw_probe.py >> gpurun_out/ab.log 2>&1
run() {  # label, env..., workload
  local label=$1; shift; local w=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$w', d['value'], d['roofline']['frac'])" >> gpurun_out/ab.log
}
for w in c1 c2 c4 c3; do
  run cmax1_ctas4 $w HDCG_TMA_CMAX=1
  run cmax4_ctas4 $w HDCG_TMA_CMAX=4
  run cmax1_ctas3 $w HDCG_TMA_CMAX=1 HDCG_TMA_CTAS=3
  run cmax4_ctas3 $w HDCG_TMA_CMAX=4 HDCG_TMA_CTAS=3
  run cmax4_xlast $w HDCG_TMA_CMAX=4 HDCG_TMA_X_POLICY=1
  run general $w HDCG_KERNEL_POLICY=1
done
python scripts/bw_probe.py >> gpurun_out/ab.log 2>&1
