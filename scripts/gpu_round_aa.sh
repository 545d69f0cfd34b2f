#!/bin/bash
# Small blocks with a light remainder: remainder in the kernel (REST == 1, the default)
# against summed first by rest_pipe_kernel (HDCG_REST_MODE=2), on one box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/aa
O=gpurun_out/aa
for rep in 1 2; do
  for m in 0 2; do
    echo "# REST_MODE=$m" >> $O/ab.log
    HDCG_REST_MODE=$m timeout 300 python scripts/shape_probe.py lap256_bl100 lap256_bl200 lap256_bl50 lap256_bl10 lap256_bl512 >> $O/ab.log 2>>$O/ab.err
  done
done
echo done
