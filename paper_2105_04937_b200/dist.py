"""Row-slab sharding of the M-HDC SpMV across GPUs (one process per GPU).

The reference has no distributed path (OpenMP only); this is
the B200 scale-out for BASELINE config 4: contiguous z-slabs of rows, slab
sizes a multiple of bl (so every rank's blocks are exactly global blocks and
its conversion is bit-identical to the global one), and per SpMV one
exchange of the x halo of width H = max|offset| with the two neighbours.

Power iteration (config 4: x <- y/||y||) per step k, on rank r:
  1. boundary blocks (rows within H of either slab edge) of y_k = A (s_{k-1} y_{k-1})
  2. send y_k's first/last H rows to the neighbours' halo regions (NCCL P2P over
     NVLink, torch.distributed) -- overlapped with
  3. the interior blocks;
  4. per-tile sums of y_i^2 (fused into the SpMV) -> local pairwise tree ->
     all-gather of the rank roots -> top tree (the same tree kernel) -> s_k = 1/sqrt(sum).
The scale s is applied inside the next SpMV's x loads, so no separate
normalisation pass streams y again.  Every row is owned by one rank and keeps
its per-row operation order, so y is bitwise independent of the number of
ranks; the tree over tiles is split into per-rank subtrees (power-of-two tile
counts per rank) so the norm is bitwise independent of it too.

The compute backend is injected: CudaSlab (libhdcgpu.so, the product) or, in
the CPU tests only, an oracle-backed stand-in.  The halo transport is either
  * "nccl": torch.distributed send/recv of the boundary rows (NCCL over NVLink;
    gloo in the CPU tests), overlapped with the interior blocks, or
  * "p2p": PeerHalo -- the SpMV itself (one launch over every block) stores its halo
    rows into the neighbours' buffers through peer memory (CUDA IPC mappings,
    NVLink P2P stores from the kernel epilogue), so the exchange overlaps the
    computation tile by tile and no collective is launched for it.  The per-step norm
    all-gather orders those stores before the neighbours' next reads (and
    their reads before the next overwrite: x/y are double-buffered).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class SlabPlan:
    n: int            # global rows
    bl: int           # block width
    halo: int         # H = max |offset|
    world: int
    row0: list
    rows: list

    @staticmethod
    def make(n: int, bl: int, halo: int, world: int, unit: int | None = None) -> "SlabPlan":
        """Contiguous slabs; boundaries are multiples of `unit` (default bl; the
        z-plane size x bl lcm is passed for stencils so slabs are whole planes)."""
        unit = unit or bl
        if unit % bl:
            raise ValueError("slab unit must be a multiple of bl")
        n_units = (n + unit - 1) // unit
        row0, rows = [], []
        for r in range(world):
            u0, u1 = r * n_units // world, (r + 1) * n_units // world
            a, b = min(n, u0 * unit), min(n, u1 * unit)
            row0.append(a)
            rows.append(b - a)
        return SlabPlan(n, bl, halo, world, row0, rows)

    def boundary_blocks(self, rank: int, blocks_per_tile: int = 1):
        """[(b0, b1), ...] block ranges that read the halo, and the interior range."""
        rows = self.rows[rank]
        nb = (rows + self.bl - 1) // self.bl
        g = blocks_per_tile

        def down(b):
            return (b // g) * g

        def up(b):
            return min(nb, ((b + g - 1) // g) * g)

        left = up((min(rows, self.halo) + self.bl - 1) // self.bl) if rank > 0 else 0
        right = down(max(0, rows - self.halo) // self.bl) if rank < self.world - 1 else nb
        if left >= right:
            return [(0, nb)], (0, 0)
        parts = []
        if left > 0:
            parts.append((0, left))
        if right < nb:
            parts.append((right, nb))
        return parts, (left, right)


class HaloExchange:
    """x halo of a slab buffer laid out as [H left halo | rows owned | H right halo].

    NCCL sends the device slices directly (P2P over NVLink).  Under gloo (the CPU
    tests, and the one-GPU multi-process test of this code path) a CUDA buffer is
    staged through host tensors: the boundary rows are copied out, exchanged,
    and the received halos copied back in wait()."""

    def __init__(self, plan: SlabPlan, rank: int):
        self.plan, self.rank = plan, rank

    def start(self, buf: torch.Tensor):
        H, rows, r, p = self.plan.halo, self.plan.rows[self.rank], self.rank, self.plan.world
        stage = buf.is_cuda and dist.get_backend() == "gloo"
        pairs = []  # (send slice, recv slice, peer)
        if r > 0:
            pairs.append((buf[H:H + H], buf[0:H], r - 1))
        if r < p - 1:
            pairs.append((buf[rows:rows + H], buf[H + rows:H + rows + H], r + 1))
        ops, back = [], []
        for snd, rcv, peer in pairs:
            if stage:
                s_h, r_h = snd.cpu(), torch.empty(rcv.shape, dtype=rcv.dtype)
                back.append((rcv, r_h))
                snd, rcv = s_h, r_h
            ops.append(dist.P2POp(dist.isend, snd, peer))
            ops.append(dist.P2POp(dist.irecv, rcv, peer))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, back

    @staticmethod
    def wait(handle):
        reqs, back = handle
        for q in reqs:
            q.wait()
        for dst, src in back:  # staged receives (gloo + CUDA buffer)
            dst.copy_(src)


class PeerHalo:
    """Peer-memory halo delivery for a rank whose two slab buffers are
    hdcgpu.PeerBuffer objects (layout [H | rows | H]).  Maps the neighbours'
    buffers: lo[i] = the lower neighbour's buffer i at its upper halo (where
    this rank's first H rows go), hi[i] = the upper neighbour's buffer i at its
    lower halo (this rank's last H rows)."""

    def __init__(self, plan: SlabPlan, rank: int, peer_bufs):
        from . import hdcgpu as H
        self.H, self.plan, self.rank = H, plan, rank
        handles = [b.handle for b in peer_bufs]
        allh = [None] * plan.world
        dist.all_gather_object(allh, handles)  # every rank enters it, whatever happens next
        self.mapped, self.lo, self.hi = [], [0, 0], [0, 0]
        self.error = None
        try:
            if rank > 0:
                for i in range(2):
                    base = H.peer_open(allh[rank - 1][i])
                    self.mapped.append(base)
                    self.lo[i] = base + 8 * (plan.halo + plan.rows[rank - 1])
            if rank < plan.world - 1:
                for i in range(2):
                    base = H.peer_open(allh[rank + 1][i])
                    self.mapped.append(base)
                    self.hi[i] = base
        except Exception as e:  # noqa: BLE001 - reported to the caller, which falls back to NCCL
            self.error = repr(e)[:160]

    def close(self):
        for p in self.mapped:
            self.H.peer_close(p)
        self.mapped = []


def halo_checksums(plan: SlabPlan, rank: int, buf: torch.Tensor) -> torch.Tensor:
    """int64 sums of the bit patterns of [first H rows, last H rows, lower halo,
    upper halo] of a slab buffer (exact: integer arithmetic)."""
    Hh, rows = plan.halo, plan.rows[rank]
    v = buf.view(torch.int64)
    return torch.stack([v[Hh:2 * Hh].sum(), v[rows:rows + Hh].sum(), v[0:Hh].sum(),
                        v[Hh + rows:2 * Hh + rows].sum()])


def verify_halos(plan: SlabPlan, rank: int, buf: torch.Tensor) -> bool:
    """True when every rank's halos of `buf` hold exactly its neighbours' boundary rows."""
    cs = halo_checksums(plan, rank, buf)
    allc = [torch.zeros_like(cs) for _ in range(plan.world)]
    dist.all_gather(allc, cs)
    ok = True
    for r in range(plan.world):
        if r > 0 and int(allc[r][2]) != int(allc[r - 1][1]):
            ok = False
        if r < plan.world - 1 and int(allc[r][3]) != int(allc[r + 1][0]):
            ok = False
    return ok


def _all_gather_roots(out: torch.Tensor, local: torch.Tensor):
    if out.is_cuda and dist.get_backend() == "gloo":  # CPU tests on one GPU: stage through the host
        parts = [torch.zeros(1, dtype=out.dtype) for _ in range(out.numel())]
        dist.all_gather(parts, local.cpu())
        out.copy_(torch.cat(parts))
    else:
        dist.all_gather_into_tensor(out, local)


def pairwise_tree(vals: torch.Tensor) -> torch.Tensor:
    """Host-side twin of hdcg_tree_sum for tiny vectors (rank roots): pads to a
    power of two with +0.0 and adds adjacent pairs level by level."""
    v = vals.clone()
    p = 1
    while p < v.numel():
        p <<= 1
    if p != v.numel():
        v = torch.cat([v, torch.zeros(p - v.numel(), dtype=v.dtype, device=v.device)])
    while v.numel() > 1:
        v = v[0::2] + v[1::2]
    return v


class SlabPowerIteration:
    """Drives the config-4 power iteration over one rank's slab.

    compute must provide: n_tiles, blocks_per_tile, n_blocks,
      spmv(x_buf, y_buf, b0, b1, scale, tiles[, peer_lo, peer_hi])
                                                 -- y_buf[H:H+rows] <- A_slab (scale * x_buf)
      tree(tiles) -> tensor([sum, 1/sqrt(sum)])  -- deterministic pairwise tree
    peer: a PeerHalo (x0_buf and y_buf are then views of its two PeerBuffers,
    in that order) -- the boundary SpMVs deliver the halos; otherwise NCCL/gloo
    send/recv does.
    """

    def __init__(self, plan: SlabPlan, rank: int, compute, x0_buf: torch.Tensor, comm=True,
                 y_buf: torch.Tensor | None = None, peer: PeerHalo | None = None):
        self.plan, self.rank, self.c = plan, rank, compute
        self.bufs = [x0_buf, torch.empty_like(x0_buf) if y_buf is None else y_buf]
        self.bufs[1].zero_()
        self.peer = peer
        self.p2p_single_launch = True  # False: boundary blocks first, then the interior (A/B)
        self.yi = 1  # index (into the original pair) of the buffer y goes to this step
        dev = x0_buf.device
        # red = [sum of squares, 1/sqrt(sum)]; the scale the next SpMV applies is red[1],
        # written in place by the top tree (no copy kernel between the steps)
        self.red = torch.tensor([0.0, 1.0], dtype=torch.float64, device=dev)
        self.scale = self.red[1:2]
        self.tiles = torch.zeros(compute.n_tiles, dtype=torch.float64, device=dev)
        self.roots = torch.zeros(plan.world, dtype=torch.float64, device=dev)
        self.halo = HaloExchange(plan, rank)
        self.comm = comm and plan.world > 1
        self.parts, self.interior = plan.boundary_blocks(rank, compute.blocks_per_tile)
        if self.comm:
            # every rank's buffers are zeroed before any neighbour's first boundary
            # SpMV can store halo rows into them (peer mode), or send (NCCL mode)
            if dev.type == "cuda":
                torch.cuda.synchronize(dev)
            dist.barrier()

    def _top_tree(self, vals):
        """The pairwise tree over `vals` (tile partials, or the rank roots) into
        self.red; red[1] is the next step's scale."""
        into = getattr(self.c, "tree_into", None)
        if into is not None:
            into(vals, self.red)
        else:  # backends with tree() only (the CPU stand-in of the tests)
            self.red.copy_(self.c.tree(vals))

    def step(self):
        x, y = self.bufs
        if not self.comm:
            self.c.spmv(x, y, 0, self.c.n_blocks, self.scale, self.tiles)
            self._top_tree(self.tiles)
        elif self.peer is not None:
            # boundary blocks store their halo rows straight into the neighbours' y
            # buffers (same parity on every rank); the all-gather below orders them
            # One launch over every block: a neighbour reads this step's halo rows only
            # in its next step, after the all-gather, so it does not matter when inside
            # the step the boundary tiles run -- no separate boundary launches (their
            # ramp-up and tail cost ~25 us of an 8-GPU step of 0.75 ms).
            lo, hi = self.peer.lo[self.yi], self.peer.hi[self.yi]
            if self.p2p_single_launch:
                self.c.spmv(x, y, 0, self.c.n_blocks, self.scale, self.tiles, lo, hi)
            else:
                for b0, b1 in self.parts:
                    self.c.spmv(x, y, b0, b1, self.scale, self.tiles, lo, hi)
                if self.interior[1] > self.interior[0]:
                    self.c.spmv(x, y, self.interior[0], self.interior[1], self.scale, self.tiles)
            local = self.c.tree(self.tiles)
            _all_gather_roots(self.roots, local[0:1].contiguous())
            self._top_tree(self.roots)
        else:
            for b0, b1 in self.parts:
                self.c.spmv(x, y, b0, b1, self.scale, self.tiles)
            reqs = self.halo.start(y)
            if self.interior[1] > self.interior[0]:
                self.c.spmv(x, y, self.interior[0], self.interior[1], self.scale, self.tiles)
            HaloExchange.wait(reqs)
            local = self.c.tree(self.tiles)
            _all_gather_roots(self.roots, local[0:1].contiguous())
            # the top of the tree over the rank roots: the same padded pairwise tree,
            # one launch on the device (stream-ordered after the all-gather)
            self._top_tree(self.roots)
        self.bufs.reverse()
        self.yi ^= 1
        return self.red


def all_ranks_agree(flag: bool, device=None) -> bool:
    """True on every rank iff `flag` is true on every rank (one tiny all-reduce)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return bool(flag)
    t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


class SlabRunner:
    """Builds the power iteration of one rank with a halo transport, checks the
    halos, and falls back from peer memory to send/recv when the peer path cannot
    be set up or delivers a wrong halo -- every rank takes the same decision.

    transport: "p2p" (hdcgpu.PeerBuffer + PeerHalo; the boundary SpMVs store the
    halos), "nccl" (HaloExchange send/recv), "none" (one rank).  init_x(buf) fills
    the rank's [H | rows | H] x buffer (the halo included).  device / peer_buffer
    default to the current CUDA device and hdcgpu.PeerBuffer (the CPU tests
    inject their own to exercise the cross-rank decisions under gloo)."""

    def __init__(self, plan: SlabPlan, rank: int, compute, init_x, transport: str = "p2p", device=None,
                 peer_buffer=None):
        self.plan, self.rank, self.compute, self.init_x = plan, rank, compute, init_x
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.peer_buffer = peer_buffer
        self.world = plan.world
        self.pbufs, self.peer = [], None
        self.halo_ok = {}
        self.it, self.transport = None, None
        if self.world > 1 and transport == "p2p":
            self.it, self.transport = self._build(True)
        if self.it is None:
            note = self.transport
            self.it, self.transport = self._build(False)
            if note:
                self.transport = note

    def _dev(self):
        return self.device

    def _sync(self):
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)

    def release_peer(self):
        """Unmap the neighbours' buffers on every rank before any rank frees its own."""
        if self.peer is not None:
            self.peer.close()
        self.peer = None
        if self.world > 1:
            self._sync()
            dist.barrier()
        for b in self.pbufs:
            b.free()
        self.pbufs = []

    def _build(self, p2p: bool):
        from . import hdcgpu as H
        rows, halo = self.plan.rows[self.rank], self.plan.halo
        if p2p:
            err = ""
            make = self.peer_buffer or H.PeerBuffer
            try:  # local allocation first, agreed on before the collective handle exchange
                for _ in range(2):
                    self.pbufs.append(make(rows + 2 * halo))
            except Exception as e:  # noqa: BLE001 - IPC allocation refused on this box
                err = repr(e)[:120]
            if all_ranks_agree(not err, self._dev()):
                self.peer = PeerHalo(self.plan, self.rank, self.pbufs)
                err = self.peer.error or ""
                if all_ranks_agree(not err, self._dev()):
                    err = None
            if err is not None:
                self.release_peer()
                return None, f"nccl (peer-memory setup failed: {err or 'on another rank'})"
            xb, yb = (torch.as_tensor(b, device=self.device) for b in self.pbufs)
        else:
            xb, yb = torch.zeros(rows + 2 * halo, dtype=torch.float64, device=self.device), None
        xb.zero_()
        self.init_x(xb)
        it = SlabPowerIteration(self.plan, self.rank, self.compute, xb, comm=self.world > 1, y_buf=yb,
                                peer=self.peer)
        return it, ("p2p" if p2p else ("nccl" if self.world > 1 else "none"))

    def warm(self, steps: int, force_check_failure: bool = False):
        """`steps` untimed steps, then the halo check; a failed peer-memory check
        switches every rank to send/recv and warms that up instead.
        force_check_failure: treat the p2p check as failed (tests the fallback)."""
        for _ in range(steps):
            self.it.step()
        self._sync()
        if self.world == 1:
            return
        ok = verify_halos(self.plan, self.rank, self.it.bufs[0])
        self.halo_ok["after_warmup"] = ok
        if self.peer is not None and (not all_ranks_agree(ok, self._dev()) or force_check_failure):
            self.release_peer()
            self.it, _ = self._build(False)
            self.transport = "nccl (p2p halo check failed)"
            for _ in range(steps):
                self.it.step()
            self._sync()
            self.halo_ok["after_warmup_nccl"] = verify_halos(self.plan, self.rank, self.it.bufs[0])
        dist.barrier()

    def check_after(self, key: str = "after_timed"):
        if self.world > 1:
            self._sync()
            dist.barrier()
            self.halo_ok[key] = verify_halos(self.plan, self.rank, self.it.bufs[0])

    def halos_ok_everywhere(self) -> bool:
        return all_ranks_agree(all(self.halo_ok.values()), self._dev()) if self.world > 1 else True

    def y_checksum(self):
        """Sums of the low and high 32-bit halves of the final iterate's bit patterns
        over every rank's rows (exact in int64 for any partition): equal for every
        rank count when the sharded y is bitwise the one-GPU y."""
        halo, rows = self.plan.halo, self.plan.rows[self.rank]
        yv = self.it.bufs[0][halo:halo + rows].view(torch.int64)
        ck = torch.stack([(yv & 0xFFFFFFFF).sum(), (yv >> 32).sum()])
        if self.world > 1:
            dist.all_reduce(ck, op=dist.ReduceOp.SUM)
        return [int(v) for v in ck.tolist()]


class CudaSlab:
    """The product compute backend: libhdcgpu.so on the current CUDA stream."""

    def __init__(self, matrix, halo: int):
        from . import hdcgpu as H
        self.H, self.m, self.halo = H, matrix, halo
        self.n_tiles = matrix.info.n_tiles
        self.blocks_per_tile = matrix.info.blocks_per_tile
        self.n_blocks = matrix.n_blocks
        self.launches = 0
        self._per_spmv = len(H.spmv_kernels(matrix.info, scale=True, norm=True))
        self._out = None

    def spmv(self, x_buf, y_buf, b0, b1, scale, tiles, peer_lo=0, peer_hi=0):
        st = torch.cuda.current_stream().cuda_stream
        if peer_lo or peer_hi:
            self.H.spmv_slab_halo(self.m, x_buf.data_ptr() + 8 * self.halo, y_buf.data_ptr() + 8 * self.halo,
                                  b0, b1, scale.data_ptr(), tiles.data_ptr(), peer_lo, peer_hi, self.halo, st)
        else:
            self.H.spmv_slab(self.m, x_buf.data_ptr() + 8 * self.halo, y_buf.data_ptr() + 8 * self.halo,
                             b0, b1, scale.data_ptr(), tiles.data_ptr(), st)
        self.launches += self._per_spmv

    def tree(self, tiles):
        if self._out is None:
            self._out = torch.empty(2, dtype=torch.float64, device=tiles.device)
        return self.tree_into(tiles, self._out)

    def tree_into(self, tiles, out):
        """out[0] = the pairwise-tree sum of `tiles`, out[1] = 1/sqrt(out[0])."""
        st = torch.cuda.current_stream().cuda_stream
        self.H.tree_sum(tiles.data_ptr(), tiles.numel(), out.data_ptr(), st)
        self.launches += 1 if tiles.numel() <= 2048 else 2
        return out
