#!/usr/bin/env python3
"""SDR (K8) throughput: a batch of (estimate, reference) signal pairs on the
device vs the numpy oracle (lstsq, the reference's algorithm) on a sample.

    python profiles/sdr_bench.py [--pairs 1024] [--length 160000]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1805_06572_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=1024)
    ap.add_argument("--length", type=int, default=160000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    ref = torch.randn((a.pairs, a.length), dtype=torch.float64, device="cuda", generator=g)
    est = 0.9 * ref + 0.3 * torch.randn(ref.shape, dtype=torch.float64, device="cuda", generator=g)
    P.sdr_pairs_device(est, ref)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        vals, _ = P.sdr_pairs_device(est, ref)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    # algorithmic bytes: est + ref read twice (two streaming passes)
    gbs = 2 * 2 * a.pairs * a.length * 8 / (ms / 1e3) / 1e9
    from oracle import metrics_oracle as MO

    n_cpu = 4
    t0 = time.perf_counter()
    cpu = [MO.channel_sdr(est[i].cpu().numpy(), ref[i].cpu().numpy()) for i in range(n_cpu)]
    cpu_s = (time.perf_counter() - t0) / n_cpu
    dev = max(abs(float(vals[i]) - cpu[i]) for i in range(n_cpu))
    print(json.dumps({"pairs": a.pairs, "length": a.length, "ms": round(ms, 3),
                      "pairs_per_s": a.pairs / (ms / 1e3), "GBps_2pass": round(gbs, 1),
                      "cpu_oracle_s_per_pair": round(cpu_s, 4),
                      "speedup_vs_oracle_1core": round(cpu_s * a.pairs / (ms / 1e3), 1),
                      "max_abs_dev_db": dev}), flush=True)


if __name__ == "__main__":
    main()
