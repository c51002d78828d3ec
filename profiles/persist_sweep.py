#!/usr/bin/env python3
"""KP (persistent EM kernel) against the plain schedule on small single-mixture
shapes: TF-bin*it/s of graph-replayed device runs, likelihood off.

    python profiles/persist_sweep.py [--steps 5]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06572_b200 import init_random  # noqa: E402
from paper_1805_06572_b200._engine import plan_chunks, run_device, status_of  # noqa: E402
from paper_1805_06572_b200.synth import make_mixture  # noqa: E402


def bench(y, init, L, persist, steps):
    Y = y[None]
    V, S, FL = init.v[None], init.S[None], init.v_floor[None]
    out = {"images": torch.empty((1, 2) + tuple(y.shape), dtype=torch.complex128, device="cuda"),
           "S": torch.empty_like(S), "v": torch.empty_like(V)}
    kw = dict(likelihood=False, timing=False, check=False, out=out, graph=True, persist=persist)
    r = run_device("fast", Y, V, S, FL, L, **kw)
    status_of(r)
    out["workspace"] = r.workspace
    for _ in range(3):
        run_device("fast", Y, V, S, FL, L, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run_device("fast", Y, V, S, FL, L, **kw)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    L = 20
    for I in (2, 3, 4):
        for F in (129, 257, 513, 1025):
            for N in (500, 1000, 2000, 4000):
                if F * N > (4 << 20):
                    continue
                y = torch.from_numpy(make_mixture(7, I, F, N, eps=1e-3, sigma=1.5)).cuda()
                init = init_random(y, 3)
                ms0 = bench(y, init, L, False, a.steps)
                ms1 = bench(y, init, L, True, a.steps)
                print(json.dumps({"I": I, "F": F, "N": N, "L": L,
                                  "plain_G": round(F * N * L / ms0 / 1e6, 2),
                                  "kp_G": round(F * N * L / ms1 / 1e6, 2),
                                  "kp_over_plain": round(ms0 / ms1, 3),
                                  "plain_us_per_it": round(ms0 * 1e3 / L, 2),
                                  "kp_us_per_it": round(ms1 * 1e3 / L, 2),
                                  "plain_plan": plan_chunks(F, N, I)}), flush=True)


if __name__ == "__main__":
    main()
