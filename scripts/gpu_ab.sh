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
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$w', d['value'], d['roofline']['frac'], 'e2e', d['e2e']['value'])" >> gpurun_out/ab.log
}
for w in c1 c4 c2 c3; do
  run default $w
  run ctas2 $w HDCG_TMA_CTAS=2
done
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/ab.log
