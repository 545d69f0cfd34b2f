"""HBM copy bandwidth of this box (same method as MEASURED_PEAKS.json: read+write
bytes of a 1 Gi-element bf16 copy, best of 10, CUDA events) -- used to normalise
A/B sweeps that run on different boxes."""
import json

import torch

a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
best = 1e9
for _ in range(12):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    b.copy_(a)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print(json.dumps({"copy_gbs": round(2 * a.numel() * 2 / (best * 1e-3) / 1e9, 1)}))
