"""FP64 / HBM peak probe (tools/fp64_peak.cu) with the SM clock sampled by NVML during
the run (every ~2 ms): writes profiles/<tag>_peaks_fp64.json. Run on the GPU box:
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
    python tools/peaks.py r02"""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import pynvml

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], [False]


def poll():
    while not stop[0]:
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                        pynvml.nvmlDeviceGetUtilizationRates(h).gpu))
        time.sleep(0.002)


th = threading.Thread(target=poll, daemon=True)
th.start()
out = subprocess.run([os.path.join(root, "tools", "fp64_peak")], capture_output=True, text=True, check=True).stdout
stop[0] = True
th.join()
res = json.loads(out.strip().splitlines()[-1])
busy = [s for s in samples if s[4] > 50]
mhz = [s[1] for s in busy]
reasons = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}
res["clocks"] = {"sm_mhz_median_under_load": statistics.median(mhz) if mhz else None,
                 "sm_mhz_min_under_load": min(mhz) if mhz else None,
                 "sm_max_mhz": pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM),
                 "power_w_max": max(s[3] for s in samples) if samples else None,
                 "samples_under_load": len(busy),
                 "reasons_seen": sorted({n for s in busy for n, b in reasons.items() if s[2] & b})}
smx = res["clocks"]["sm_max_mhz"]
res["fp64_tflops_nominal_at_max_clock"] = 148 * 64 * 2 * smx * 1e6 / 1e12
if mhz:
    res["fp64_tflops_nominal_at_load_clock"] = 148 * 64 * 2 * statistics.median(mhz) * 1e6 / 1e12
res["note"] = ("DFMA: 8 independent FMA chains per thread, 2048 threads per SM; DMMA: m8n8k4 f64 chains; "
               "nominal = 148 SMs x 64 FP64 FMA/clk x 2 flop x clock")
path = os.path.join(root, "gpurun_out", f"{tag}_peaks_fp64.json")   # copy to profiles/ after the call
os.makedirs(os.path.dirname(path), exist_ok=True)
json.dump(res, open(path, "w"), indent=1)
print(json.dumps(res))
