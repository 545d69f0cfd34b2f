#!/bin/bash
# Remainder-path parity + config-3 A/B of the TMA kernel's remainder modes.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rest_ab.log
timeout 600 python -m pytest tests -q -m gpu -x -k "remainder or kernel_paths or config3 or golden or fixture or power or slab" > gpurun_out/pytest_rest.log 2>&1; echo pytest=$? >> gpurun_out/rest_ab.log
timeout 300 python scripts/diag_c3.py 4194304; HDCG_REST_KERNEL=2 timeout 300 python scripts/diag_c3.py 1048576; HDCG_REST_KERNEL=1 timeout 300 python scripts/diag_c3.py 1048576 > gpurun_out/diag.log 2>&1; echo diag=$? >> gpurun_out/rest_ab.log
run() {  # label, workload, extra args, env...
  local label=$1; shift; local w=$1; shift; local bl=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --workload $w --bl $bl --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$w', '$bl', d['value'], d['roofline']['frac'], 'e2e', d['e2e']['value'])" >> gpurun_out/rest_ab.log
}
for bl in 8192 1024; do
  for k in 0 1 2 3 4; do run rk$k c3 $bl HDCG_REST_KERNEL=$k; done; break
done


