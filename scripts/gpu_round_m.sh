#!/bin/bash
# rest_pipe_kernel: parity of every remainder variant, then a same-box A/B of the
# variants on the remainder-heavy workloads (config 3, CSR of configs 1-3).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/m
O=gpurun_out/m
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "remainder or random_sweep or golden or config3 or empty or csr" > $O/pytest_rest.log 2>&1; echo pytest=$? >> $O/pytest_rest.log
for v in 0 1 2 3 4; do
  for w in "--workload c3" "--workload c1 --format csr" "--workload c2 --format csr" "--workload c3 --format csr"; do
    HDCG_REST_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline $w --steps 20 --warmup 3 2>>$O/ab.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'v': $v, 'w': d['config']['workload'], 'gflops': d['value'], 'frac': d['roofline']['frac'], 'kernel_ms': d['roofline'].get('kernel_ms'), 'ms': d['ms_per_step']}))" >> $O/ab.log 2>>$O/ab.err
  done
done
echo done
