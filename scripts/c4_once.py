"""Config-4 power-iteration SpMV launched 3 times (for ncu captures of one launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200.dist import SlabPlan  # noqa: E402

H.init(0)
nx, ny, nz = bench.GRID4
n = nx * ny * nz
plan = SlabPlan.make(n, 4096, nx * ny, 1, unit=nx * ny)
m, _, _ = bench.build_config4_slab(H, torch, plan, 0, 4096)
x = torch.empty(n, dtype=torch.float64, device="cuda")
H.gen_uniform_pm1(5, 0, 0, n, x.data_ptr())
y = torch.empty_like(x)
tiles = torch.empty(m.info.n_tiles, dtype=torch.float64, device="cuda")
sc = torch.tensor([0.5], dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, sc.data_ptr(), tiles.data_ptr(), st)
torch.cuda.synchronize()
print("ok")
