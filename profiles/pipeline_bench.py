#!/usr/bin/env python3
"""Device-resident separation chain on the config-3 shape: 256 four-channel
mixtures of 20 s at 16 kHz (frame length 512 -> 1250 frames x 257 bins):
STFT analysis -> init (random or masks) -> 20 FastFCA iterations -> STFT
synthesis of both source images, inputs resident in HBM. Prints one JSON line
with the per-stage device times (CUDA events).

    python profiles/pipeline_bench.py [--init masks|random] [--M 256]
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1805_06572_b200._engine import run_device  # noqa: E402
from paper_1805_06572_b200.initializers import init_from_masks_batch, init_random_batch  # noqa: E402
from paper_1805_06572_b200.stft import stft_analyze_device, stft_synthesize_device  # noqa: E402


def mixtures(M, C, length, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    src = torch.randn((M, 2, length), dtype=torch.float64, device="cuda", generator=g)
    t = torch.arange(length, device="cuda", dtype=torch.float64)
    src[:, 1] *= torch.sin(t / 4000.0).abs()  # different activity
    taps = torch.randn((M, 2, C, 6), dtype=torch.float64, device="cuda", generator=g)
    taps *= torch.exp(-torch.arange(6, device="cuda", dtype=torch.float64))
    x = torch.zeros((M, C, length), dtype=torch.float64, device="cuda")
    for j in range(2):
        for k in range(6):
            x[:, :, k:] += taps[:, j, :, k, None] * src[:, j, None, : length - k]
    return x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=256)
    ap.add_argument("--C", type=int, default=4)
    ap.add_argument("--L", type=int, default=512)
    ap.add_argument("--frames", type=int, default=1250)
    ap.add_argument("--iterations", type=int, default=20)
    ap.add_argument("--init", default="masks")
    a = ap.parse_args()
    length = (a.frames - 2) * (a.L // 2) + 1
    x = mixtures(a.M, a.C, length)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def once():
        ev[0].record()
        spec = stft_analyze_device(x, a.L)
        ev[1].record()
        if a.init == "masks":
            m = init_from_masks_batch(spec)
        else:
            m = init_random_batch(spec, list(range(a.M)))
        ev[2].record()
        r = run_device("fast", spec, m.v, m.S, m.v_floor, a.iterations, likelihood=False,
                       timing=False, check=False)
        ev[3].record()
        out = stft_synthesize_device(r.images, a.L, length)
        ev[4].record()
        torch.cuda.synchronize()
        return out

    once()
    once()
    names = ["stft_analyze", "init_" + a.init, "em", "stft_synthesize"]
    ms = {n: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, n in enumerate(names)}
    total = ev[0].elapsed_time(ev[4])
    print(json.dumps({"workload": f"{a.M} mixtures x {a.C} ch x {length} samples, L={a.L}, "
                                  f"{a.iterations} FastFCA iterations",
                      "stage_ms": ms, "total_ms": round(total, 3),
                      "audio_seconds_per_s": round(a.M * length / 16000 / (total / 1e3), 1)}))


if __name__ == "__main__":
    main()
