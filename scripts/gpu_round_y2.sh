#!/bin/bash
# Closing check of the session: the committed library (v21 kernels) passes the GPU suite
# GPU suite and smoke, and the default bench line and reference arm still hold.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/y2
O=gpurun_out/y2
python scripts/bw_probe.py > $O/bw.json 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done
