"""Run tools/bin/fp64_peak (tools/fp64_peak.cu) with the SM clock sampled by nvidia-smi during the run and
write one JSON object: best and median of each peak over the repetitions, plus the clock record
(B200_PROFILING.md clocks line).

    python tools/fp64_peak.py [REPS] > profiles/fp64_peak_rNN.json
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
smi = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                       stdout=f, stderr=subprocess.DEVNULL)
out = subprocess.run([os.path.join(ROOT, "tools", "bin", "fp64_peak"), str(reps)], capture_output=True, text=True,
                     check=True).stdout
smi.terminate()
smi.wait()
f.seek(0)
sm, mx, pw, reasons = [], [], [], set()
for line in f.read().splitlines():
    c = [x.strip() for x in line.split(",")]
    try:
        sm.append(float(c[0])), mx.append(float(c[1])), pw.append(float(c[2]))
    except (ValueError, IndexError):
        continue
    for nm, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), c[3:7]):
        if v.lower() == "active":
            reasons.add(nm)
runs = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
res = {}
for key in ("dfma_tflops", "dmma_tflops", "sincos_rsqrt_geval_s"):
    v = [r[key] for r in runs]
    res[key] = max(v)
    res[key + "_median"] = float(np.median(v))
res["reps"] = len(runs)
res["clocks"] = {"sm_mhz_median": float(np.median(sm)) if sm else None, "sm_mhz_min": min(sm) if sm else None,
                 "sm_max_mhz": max(mx) if mx else None, "power_w_max": max(pw) if pw else None,
                 "samples": len(sm), "reasons": sorted(reasons)}
res["how"] = ("tools/fp64_peak.cu: DFMA = 8 independent fma chains per thread, 148x8 CTAs x 256 threads; DMMA = "
              "mma.sync.m8n8k4.f64 (512 flop per warp instruction); sincos+rsqrt evaluations/s; CUDA events; best "
              "and median over the repetitions; nvidia-smi sampled every 100 ms during the run")
print(json.dumps(res, indent=1))
