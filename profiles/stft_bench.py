#!/usr/bin/env python3
"""Throughput of the device STFT kernels on the config-3 shape (256 mixtures
x 4 channels, frame_length 512 -> 1250 frames x 257 bins), inputs resident in
HBM, against the algorithmic bytes (read x once, write the spectrum; read the
spectrum, write x) and the measured HBM peak; plus numpy (the oracle's
rfft/irfft framing) on a bounded sample for scale.

    python profiles/stft_bench.py [--M 256] [--reps 5]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_06572_b200.stft import num_frames, stft_analyze_device, stft_synthesize_device  # noqa: E402


def timed(fn, reps, windows=3):
    """Best of `windows` CUDA-event windows of `reps` calls each (after warm-up)."""
    out = fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(windows):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=256)
    ap.add_argument("--C", type=int, default=4)
    ap.add_argument("--L", type=int, default=512)
    ap.add_argument("--frames", type=int, default=1250)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    S = a.L // 2
    length = (a.frames - 2) * S + 1
    assert num_frames(length, S) == a.frames
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((a.M, a.C, length), dtype=torch.float64, device="cuda", generator=g)
    ms_a, spec = timed(lambda: stft_analyze_device(x, a.L), a.reps)
    ms_s, back = timed(lambda: stft_synthesize_device(spec, a.L, length), a.reps)
    err = ((back - x).abs().max() / x.abs().max()).item()
    F = a.L // 2 + 1
    bytes_a = x.numel() * 8 + a.M * a.frames * F * a.C * 16
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    xs = x[:2].cpu().numpy()
    from oracle import stft_oracle as SO

    t0 = time.perf_counter()
    for m in range(xs.shape[0]):
        sp = SO.analyze(xs[m], a.L)
    t_np = (time.perf_counter() - t0) / xs.shape[0]
    for name, ms, nbytes in (("analyze", ms_a, bytes_a), ("synthesize", ms_s, bytes_a)):
        gbs = nbytes / (ms / 1e3) / 1e9
        print(json.dumps({"kernel": name, "ms": round(ms, 4), "GBps": round(gbs, 1),
                          "frac_hbm": round(gbs / peak, 4), "bytes": nbytes,
                          "shape": [a.M, a.C, length], "frame_length": a.L}))
    print(json.dumps({"roundtrip_rel_err": err, "numpy_analyze_s_per_mixture": round(t_np, 4),
                      "numpy_analyze_s_all": round(t_np * a.M, 2)}))


if __name__ == "__main__":
    main()
