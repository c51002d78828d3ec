#!/usr/bin/env python3
"""Device init_from_masks on BASELINE shapes (inputs resident in HBM), with
the numpy oracle timed on a bounded sample for scale.

    python profiles/masks_bench.py [--config 3]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200.initializers import init_from_masks_batch  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    Y, _, _, _ = make_inputs(cfg, shard(cfg, 0, 1))
    yd = torch.from_numpy(Y).cuda()
    init_from_masks_batch(yd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        m = init_from_masks_batch(yd)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    M, N, F, I = Y.shape
    from oracle import masks_oracle as MO

    t0 = time.perf_counter()
    MO.init_from_masks(Y[0][:, : max(1, F // 8)])
    t_np = (time.perf_counter() - t0) * (F / max(1, F // 8)) * M
    print(json.dumps({"config": a.config, "shape": [M, N, F, I], "device_ms": round(ms, 3),
                      "bins_per_s": M * F / (ms / 1e3),
                      "numpy_oracle_s_estimate": round(t_np, 1),
                      "sample": f"1 mixture x {max(1, F // 8)} bins, scaled"}))


if __name__ == "__main__":
    main()
