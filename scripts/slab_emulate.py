"""One rank's share of the N-GPU config-4 power iteration, timed alone on one B200.

Only one GPU is available to this build, so the N > 1 step cannot be timed over
NVLink here.  This script runs, in one process, exactly the kernel sequence rank
r of N launches per step (dist.SlabPowerIteration): the boundary blocks, the
interior blocks, the local tile tree and the top tree over the rank roots -- with the two things that need a second GPU replaced by local
stand-ins of the same size:
  * "p2p1": dist.py's default -- one launch over every block whose epilogue stores the
            halo rows, here into this rank's own halo regions (local HBM stores
            instead of NVLink stores); "p2p": boundary blocks first, then the interior;
  * "nccl": the send/recv of 2 x H rows is a device-to-device copy of the same rows
            into the halo regions, issued on a side stream like NCCL's;
  * the all-gather of the rank roots is a copy of the local root into roots[r].
So the numbers are each rank's compute-side step time; projected strong-scaling
efficiency = T(1 rank, whole matrix) / (N x max over the sampled ranks).  What is
left out: the NVLink latency of the halo (8 MB per neighbour, overlapped with the
interior blocks) and of an 8-double all-gather.

    python scripts/slab_emulate.py [--steps 20] [--warmup 3] [--worlds 1,2,4,8]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200.dist import CudaSlab, SlabPlan  # noqa: E402


def run_rank(plan, rank, bl, mode, steps, warmup):
    nx, ny, nz = bench.GRID4
    halo = nx * ny
    m, nnz, _ = bench.build_config4_slab(H, torch, plan, rank, bl)
    rows, row0, n = plan.rows[rank], plan.row0[rank], plan.n
    c = CudaSlab(m, halo)
    bufs = [torch.zeros(rows + 2 * halo, dtype=torch.float64, device="cuda") for _ in range(2)]
    g0, g1 = max(0, row0 - halo), min(n, row0 + rows + halo)
    H.gen_uniform_pm1(5, 0, g0, g1 - g0, bufs[0].data_ptr() + 8 * (g0 - (row0 - halo)))
    red = torch.tensor([0.0, 1.0], dtype=torch.float64, device="cuda")
    scale = red[1:2]  # the top tree writes the next step's scale in place (dist.SlabPowerIteration)
    tiles = torch.zeros(c.n_tiles, dtype=torch.float64, device="cuda")
    roots = torch.zeros(plan.world, dtype=torch.float64, device="cuda")
    parts, interior = plan.boundary_blocks(rank, c.blocks_per_tile)
    side = torch.cuda.Stream(priority=-1)
    has_lo, has_hi = rank > 0, rank < plan.world - 1

    def step():
        x, y = bufs
        if plan.world == 1:
            c.spmv(x, y, 0, c.n_blocks, scale, tiles)
            c.tree_into(tiles, red)
        else:
            if mode == "p2p1":  # dist.py's default: one launch, the halo rows stored from its epilogue
                lo = y.data_ptr() + 8 * (halo + rows) if has_lo else 0   # stands in for the neighbour's halo
                hi = y.data_ptr() if has_hi else 0
                c.spmv(x, y, 0, c.n_blocks, scale, tiles, lo, hi)
            elif mode == "p2p":
                lo = y.data_ptr() + 8 * (halo + rows) if has_lo else 0
                hi = y.data_ptr() if has_hi else 0
                for b0, b1 in parts:
                    c.spmv(x, y, b0, b1, scale, tiles, lo, hi)
            else:
                for b0, b1 in parts:
                    c.spmv(x, y, b0, b1, scale, tiles)
                ev = torch.cuda.Event()
                ev.record()
                with torch.cuda.stream(side):
                    side.wait_event(ev)
                    if has_lo:
                        y[0:halo].copy_(y[halo:2 * halo])
                    if has_hi:
                        y[halo + rows:].copy_(y[rows:rows + halo])
                    done = torch.cuda.Event()
                    done.record()
            if mode != "p2p1" and interior[1] > interior[0]:
                c.spmv(x, y, interior[0], interior[1], scale, tiles)
            if mode == "nccl":
                torch.cuda.current_stream().wait_event(done)
            local = c.tree(tiles)
            roots[rank:rank + 1].copy_(local[0:1])
            c.tree_into(roots, red)
        bufs.reverse()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    info = m.info
    by = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, rows,
                     halo_rows=(0 if plan.world == 1 else (has_lo + has_hi) * halo))
    del m, c, bufs
    torch.cuda.empty_cache()
    return {"world": plan.world, "rank": rank, "mode": mode if plan.world > 1 else "none", "rows": rows,
            "boundary_parts": parts if plan.world > 1 else [], "ms_per_step": round(ms, 4),
            "gbs": round(by / (ms * 1e-3) / 1e9, 1), "nnz": nnz}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--bl", type=int, default=4096)
    a = ap.parse_args()
    H.init(0)
    nx, ny, nz = bench.GRID4
    n, halo = nx * ny * nz, nx * ny
    peak, _ = bench.load_peaks()
    t1 = None
    for world in [int(w) for w in a.worlds.split(",")]:
        plan = SlabPlan.make(n, a.bl, halo, world, unit=nx * ny)
        ranks = sorted({0, world // 2, world - 1})
        for mode in (("none",) if world == 1 else ("p2p1", "p2p", "nccl")):
            res = [run_rank(plan, r, a.bl, mode, a.steps, a.warmup) for r in ranks]
            worst = max(r["ms_per_step"] for r in res)
            if world == 1:
                t1 = worst
            line = {"world": world, "mode": mode, "ranks": res, "max_ms_per_step": worst,
                    "projected_gflops": round(2.0 * bench.H_gen_laplacian7_nnz(nx, ny, nz) / (worst * 1e-3) / 1e9, 1)}
            if t1:
                line["projected_efficiency"] = round(t1 / (world * worst), 4)
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
