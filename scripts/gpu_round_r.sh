#!/bin/bash
# 4 rows/thread (1024-row tiles) for blocks with more than 8 segments: config 2 A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r
O=gpurun_out/r
python scripts/bw_probe.py > $O/bw.json 2>&1
for rep in 1 2; do
for ms in 8 32; do
  HDCG_R4_MAXSEG=$ms timeout 300 python bench.py --no-cpu-baseline --workload c2 --steps 20 --warmup 3 2>>$O/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'r4_maxseg': $ms, 'gflops': d['value'], 'frac': d['roofline']['frac'], 'kernel': d['roofline'].get('kernel')}))" >> $O/ab.log 2>>$O/ab.err
done
done
echo done
