#!/bin/bash
# compute-sanitizer memcheck over a parity subset that exercises both SpMV kernels,
# the converters (fast and general census paths), HDC, slabs and the host pipeline.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "golden or example or corner or dense_rows or kernel_paths or slab or block_range or power or edge or validation or empty or remainder or membench" \
  > gpurun_out/pytest_pre_sanitizer.log 2>&1 && \
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "golden or example or corner or dense_rows or kernel_paths or slab or block_range or power or edge or validation or empty or remainder or membench" \
  > gpurun_out/memcheck.log 2>&1; echo memcheck_rc=$? >> gpurun_out/memcheck.log
