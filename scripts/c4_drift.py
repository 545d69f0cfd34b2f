"""Does the config-4 SpMV slow down over a long run (HBM heat, power)?  300
back-to-back power-iteration SpMVs (x_scale + tile sums), each timed with CUDA
events, with NVML sampling SM/memory clocks, memory/GPU temperature, power and
clock-event reasons every 20 ms.  Prints per-30-launch means and the samples."""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as N  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_04937_b200 import hdcgpu as H  # noqa: E402
from paper_2105_04937_b200.dist import SlabPlan  # noqa: E402

H.init(0)
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
peak, _ = bench.load_peaks()
st = torch.cuda.current_stream().cuda_stream
nx, ny, nz = bench.GRID4
n = nx * ny * nz
plan = SlabPlan.make(n, 4096, nx * ny, 1, unit=nx * ny)
m, _, _ = bench.build_config4_slab(H, torch, plan, 0, 4096)
info = m.info
bts = bench.b_min(info.dia_slots, info.n_seg, info.n_blocks, info.nnz_rest, n)
x = torch.empty(n, dtype=torch.float64, device="cuda")
H.gen_uniform_pm1(5, 0, 0, n, x.data_ptr())
y = torch.empty_like(x)
tiles = torch.empty(info.n_tiles, dtype=torch.float64, device="cuda")
sc = torch.tensor([0.5], dtype=torch.float64, device="cuda")
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        try:
            samples.append({
                "t": round(time.time(), 3),
                "sm": N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                "mem": N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_MEM),
                "gpu_c": N.nvmlDeviceGetTemperature(h, N.NVML_TEMPERATURE_GPU),
                "w": round(N.nvmlDeviceGetPowerUsage(h) / 1000.0, 1),
                "reasons": N.nvmlDeviceGetCurrentClocksEventReasons(h)})
            try:
                samples[-1]["mem_c"] = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
            except Exception:  # noqa: BLE001
                pass
        except Exception as e:  # noqa: BLE001
            samples.append({"error": repr(e)[:100]})
        stop.wait(0.02)


th = threading.Thread(target=sampler, daemon=True)
th.start()
ev = []
for i in range(300):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    H.spmv_slab(m, x.data_ptr(), y.data_ptr(), 0, m.n_blocks, sc.data_ptr(), tiles.data_ptr(), st)
    e.record()
    ev.append((s, e))
torch.cuda.synchronize()
stop.set()
th.join()
ms = [s.elapsed_time(e) for s, e in ev]
for k in range(0, 300, 30):
    chunk = ms[k:k + 30]
    print(json.dumps({"launches": f"{k}-{k + 29}", "ms_mean": round(statistics.mean(chunk), 4),
                      "ms_min": round(min(chunk), 4), "frac_mean": round(bts / (statistics.mean(chunk) * 1e-3) / 1e9 / peak, 4)}))
print(json.dumps({"samples": samples[::5]}))
