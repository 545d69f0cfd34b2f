#!/bin/bash
# Same-box A/B of env knobs: gpu_ab_env.sh "w1 w2 ..." "label=ENV=val,ENV2=val" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/ab_env.log
rm -f $out
python scripts/bw_probe.py >> $out 2>&1
WL=$1; shift
for rep in 1 2; do
for w in $WL; do
  for spec in "$@"; do
    label=${spec%%=*}; envs=${spec#*=}
    env ${envs//,/ } timeout 300 python bench.py --no-cpu-baseline --workload $w --steps 10 --warmup 3 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', '$w', d['value'], d['roofline']['frac'])" >> $out
  done
done
done
