#!/usr/bin/env python3
"""Host/device time breakdown of one EM step for a BASELINE config.

    python profiles/probe_step.py --config 0 --engine fast
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import run_device, status_of  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--engine", default="fast")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
    y, v, s, fl = (torch.from_numpy(x).cuda() for x in (Y, V, S, FL))
    M, N, F, I = Y.shape
    bufs = {"images": torch.empty((M, 2, N, F, I), dtype=torch.complex128, device="cuda"),
            "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device="cuda"),
            "v": torch.empty_like(v)}
    for _ in range(2):
        r = run_device(a.engine, y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs)
        status_of(r)
        bufs["workspace"] = r.workspace
    torch.cuda.synchronize()
    for _ in range(a.reps):
        t0 = time.perf_counter()
        r = run_device(a.engine, y, v, s, fl, cfg.L, likelihood=False, check=False, timing=True,
                       out=bufs)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        status_of(r)
        it = sum(r.iteration_ms)
        print(f"host enqueue {1e3 * (t1 - t0):8.3f} ms  wait {1e3 * (t2 - t1):8.3f} ms  "
              f"iterations {it:8.3f} ms", flush=True)


if __name__ == "__main__":
    main()
