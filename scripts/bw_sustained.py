"""The box's HBM copy bandwidth burst vs sustained, with SM clocks and power
sampled through NVML: separates the SpMV's SM-clock sensitivity under the
1000 W power cap from the memory system's.

A 4.3 GB read + 4.3 GB write copy (the config-4 SpMV moves 38.6 GB per step in
~6.4 ms; this copy ~1.3 ms) is repeated back to back for `seconds`; prints the
bandwidth of the first 10 copies and of the last 20% of the run, with the clock
and power medians of each window."""
import json
import os
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(seconds=2.0):
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(int((os.environ.get("CUDA_VISIBLE_DEVICES") or "0").split(",")[0]))
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((time.perf_counter(), N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                            N.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            N.nvmlDeviceGetCurrentClocksEventReasons(h)))
            stop.wait(0.01)

    a = torch.empty(1 << 29, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1.0)
    torch.cuda.synchronize()
    th = threading.Thread(target=sample, daemon=True)
    th.start()
    ev = []
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        b.copy_(a)
        e.record()
        ev.append((time.perf_counter(), s, e))
        if len(ev) % 50 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    nbytes = 2 * a.numel() * 8
    ms = [s.elapsed_time(e) for _, s, e in ev]
    k = max(1, len(ms) // 5)
    t_last = ev[-k][0]

    def window(lo, hi):
        w = [x for x in samples if lo <= x[0] <= hi]
        return {"sm_mhz_median": statistics.median(x[1] for x in w) if w else None,
                "power_w_median": round(statistics.median(x[2] for x in w), 1) if w else None,
                "power_cap_samples": sum(1 for x in w if x[3] & getattr(N, "nvmlClocksEventReasonSwPowerCap", 4))}

    out = {"copies": len(ms), "seconds": seconds,
           "burst_gbs": round(nbytes / (statistics.mean(ms[:10]) * 1e-3) / 1e9, 1),
           "sustained_gbs": round(nbytes / (statistics.mean(ms[-k:]) * 1e-3) / 1e9, 1),
           "burst_clocks": window(ev[0][0], ev[min(9, len(ev) - 1)][0]),
           "sustained_clocks": window(t_last, ev[-1][0])}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(float(sys.argv[1]) if len(sys.argv) > 1 else 2.0)
