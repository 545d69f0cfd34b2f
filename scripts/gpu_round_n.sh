#!/bin/bash
# spmv_blk_kernel (8 <= bl < 256): GPU suite, then same-box A/B against the
# general kernel (HDCG_BLK=0) on config 1 with the paper's small block widths.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/n
O=gpurun_out/n
timeout 1500 python -m pytest tests -q -m gpu -x -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
for bl in 10 50 100 200; do
  for blk in 0 1; do
    HDCG_BLK=$blk timeout 300 python bench.py --no-cpu-baseline --workload c1 --bl $bl --steps 20 --warmup 3 2>>$O/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'blk': $blk, 'bl': $bl, 'gflops': d['value'], 'frac': d['roofline']['frac'], 'kernel': d['roofline'].get('kernel'), 'ms': d['ms_per_step']}))" >> $O/ab.log 2>>$O/ab.err
  done
done
for w in c2 c3; do
  for blk in 0 1; do
    HDCG_BLK=$blk timeout 300 python bench.py --no-cpu-baseline --workload $w --bl 100 --steps 20 --warmup 3 2>>$O/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'blk': $blk, 'w': '$w', 'bl': 100, 'gflops': d['value'], 'frac': d['roofline']['frac'], 'kernel': d['roofline'].get('kernel'), 'ms': d['ms_per_step']}))" >> $O/ab.log 2>>$O/ab.err
  done
done
echo done
