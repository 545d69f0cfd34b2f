"""Host<->device bandwidth of this box with pinned buffers: H2D alone, D2H alone, and
both at once on two streams (the e2e path's bound: x goes down while y comes back)."""
import json
import time

import torch

n = 1 << 29  # 4 GiB of fp64, the config-4 x / y size
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = n * 8


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


dup = timed(both)
print(json.dumps({"h2d_gbs": round(B / h2d / 1e9, 1), "d2h_gbs": round(B / d2h / 1e9, 1),
                  "duplex_gbs_each": round(B / dup / 1e9, 1), "bytes": B}))
