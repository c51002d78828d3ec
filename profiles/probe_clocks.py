#!/usr/bin/env python3
"""SM clock / power while the EM loop runs back to back (config 3), sampled
every 10 ms, and per-launch K3 time from CUDA events."""

import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import run_device, status_of  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
y, v, s, fl = (torch.from_numpy(x).cuda() for x in (Y, V, S, FL))
M, N, F, I = Y.shape
bufs = {"images": torch.empty((M, 2, N, F, I), dtype=torch.complex128, device="cuda"),
        "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device="cuda"),
        "v": torch.empty_like(v)}
r = run_device("fast", y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs)
status_of(r)
bufs["workspace"] = r.workspace
lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "10"], stdout=subprocess.PIPE,
                        text=True)
th = threading.Thread(target=lambda: [lines.append(ln.strip()) for ln in proc.stdout], daemon=True)
th.start()
time.sleep(0.3)
for rep in range(12):
    r = run_device("fast", y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                   timing=True, kernel_timing=True)
    status_of(r)
    if rep % 3 == 0:
        print("rep", rep, "K3 ms", [round(x, 3) for x in r.kernel_ms[:6]], "...",
              round(statistics.mean(r.kernel_ms), 3), flush=True)
time.sleep(0.2)
proc.terminate()
vals = [ln.split(",") for ln in lines if ln.count(",") >= 2]
clk = [float(a) for a, _, _ in vals]
pw = [float(b) for _, b, _ in vals]
print("samples", len(clk), "sm MHz min/med/max", min(clk), statistics.median(clk), max(clk))
print("power W min/med/max", min(pw), statistics.median(pw), max(pw))
print("reasons", sorted({c.strip() for _, _, c in vals}))
