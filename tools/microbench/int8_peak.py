"""Measured int8 tensor-core peak on this B200 (the roofline denominator of the Ozaki
emulation's int8 GEMM): cuBLAS int8 GEMM through torch._int_mm at 8192^3, best of 10
(burst, a kernel timed alone) and back to back for 4 s (sustained, under the power cap),
with nvidia-smi clocks sampled during the sustained loop.  Mirrors how the driver measured
MEASURED_PEAKS.json's bf16 figures.

    python tools/microbench/int8_peak.py > profiles/r02_int8_peak.json
"""
import json
import subprocess
import threading
import time

import torch

n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
ops = 2.0 * n ** 3
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
clk = []
stop = threading.Event()


def sample():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        if out:
            clk.append(out)
        stop.wait(0.2)


t = threading.Thread(target=sample, daemon=True)
t.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
count = 0
t0 = time.perf_counter()
e0.record()
while time.perf_counter() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    count += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
stop.set()
t.join()
sus = e0.elapsed_time(e1) / count
mhz = sorted(float(c.split(",")[0]) for c in clk if c.split(",")[0].strip().replace(".", "").isdigit())
print(json.dumps({"int8_tops_burst": round(ops / best / 1e9, 1), "int8_tops_sustained": round(ops / sus / 1e9, 1),
                  "shape": f"{n}^3 int8 -> int32 (torch._int_mm, cuBLAS)",
                  "sm_mhz_median_sustained": mhz[len(mhz) // 2] if mhz else None, "clock_samples": len(clk),
                  "power_cap_samples": sum("Active" in c and "Not" not in c for c in clk),
                  "fp64_dmma_tflops": 37.2, "fp64_source": "profiles/r01_fp64_peak.txt (DMMA.8x8x4 microbenchmark)"}))
