#!/usr/bin/env python3
"""One FastFCA run of a BASELINE config (inputs resident), for ncu launch
lists of the per-bin pencil kernel (FFCA_K1=par|thread selects its variant).

    FFCA_K1=par ncu --metrics gpu__time_duration.sum -k regex:pencil \
        python profiles/k1_probe.py --config 3
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import run_device, status_of  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iterations", type=int, default=3)
    ap.add_argument("--engine", default="fast")
    ap.add_argument("--dtype", default="c128")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
    y, v, s, fl = (torch.from_numpy(x).cuda() for x in (Y, V, S, FL))
    if a.dtype == "c64":
        y, v = y.to(torch.complex64), v.to(torch.float32)
    r = run_device(a.engine, y, v, s, fl, a.iterations, likelihood=False, check=True,
                   dtype=a.dtype)
    status_of(r)
    torch.cuda.synchronize()
    print("ok", tuple(Y.shape), a.iterations)


if __name__ == "__main__":
    main()
