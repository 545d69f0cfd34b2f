#!/bin/bash
# Round-1 final evidence for the interleaved-mapping kernel (v15): GPU suite,
# then every bench line, launch list and ncu --set full capture (gpu_evidence.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
bash scripts/gpu_evidence.sh
