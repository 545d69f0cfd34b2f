#!/bin/bash
# Closing check with the v20 library (tile layout 4): GPU suite + smoke, the
# default bench line, the reference arm, config-1 bl = 128/256 and config 3 lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/w
O=gpurun_out/w
python scripts/bw_probe.py > $O/bw.json 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
for bl in 128 256; do
  timeout 600 python bench.py --no-cpu-baseline --workload c1 --bl $bl --steps 20 --warmup 3 > $O/bench_c1_bl$bl.json 2> $O/bench_c1_bl$bl.err
done
timeout 600 python bench.py --no-cpu-baseline --workload c3 --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 1500 python -m pytest tests -q -m gpu -rf > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo done
