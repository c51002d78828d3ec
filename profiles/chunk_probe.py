#!/usr/bin/env python3
"""Plain-schedule FastFCA throughput of single small mixtures against the frame
chunking (graph-replayed device runs, likelihood off, KP off).

    python profiles/chunk_probe.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1805_06572_b200 import init_random  # noqa: E402
from paper_1805_06572_b200._engine import plan_chunks, run_device, status_of  # noqa: E402
from paper_1805_06572_b200.synth import make_mixture  # noqa: E402


def bench(y, init, L, cf, steps=5):
    Y, V, S, FL = y[None], init.v[None], init.S[None], init.v_floor[None]
    out = {"images": torch.empty((1, 2) + tuple(y.shape), dtype=torch.complex128, device="cuda"),
           "S": torch.empty_like(S), "v": torch.empty_like(V)}
    kw = dict(likelihood=False, timing=False, check=False, out=out, graph=True, persist=False,
              chunk_frames=cf)
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
    L = 20
    for I in (2, 3, 4):
        for F, N in ((257, 1000), (513, 1000), (513, 2000), (1025, 1000), (1025, 4000)):
            y = torch.from_numpy(make_mixture(7, I, F, N, eps=1e-3, sigma=1.5)).cuda()
            init = init_random(y, 3)
            plan = plan_chunks(F, N, I)
            row = {"I": I, "F": F, "N": N, "plan": plan}
            for nc in sorted({plan[1], 33, 26, 17, 13, 9, 6}):
                cf = -(-N // nc)
                ms = bench(y, init, L, cf)
                row[f"nc{-(-N // cf)}"] = round(F * N * L / ms / 1e6, 2)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
