#!/usr/bin/env python3
"""FastFCA pass time vs frame chunking (chunk_frames override) on one config.

    python profiles/chunk_sweep.py --config 4 --chunks 1539,770,514,385
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import plan_chunks, run_device  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--chunks", default="")
    ap.add_argument("--engine", default="fast")
    ap.add_argument("--iterations", type=int, default=10)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
    y, v, s, fl = (torch.from_numpy(x).cuda() for x in (Y, V, S, FL))
    M, N, F, I = Y.shape
    auto = plan_chunks(M * F, N, I, "c128", a.engine)[0]
    for cf in [auto] + [int(c) for c in a.chunks.split(",") if c]:
        for _ in range(2):
            r = run_device(a.engine, y, v, s, fl, a.iterations, likelihood=False, check=True,
                           chunk_frames=cf, kernel_timing=True, timing=True)
        hot = r.kernel_ms[:-1]
        print(json.dumps({"config": a.config, "engine": a.engine, "chunk_frames": cf,
                          "auto": cf == auto, "nchunk": -(-N // cf),
                          "pass_ms": sum(hot) / len(hot),
                          "iter_ms": sum(r.iteration_ms) / len(r.iteration_ms)}), flush=True)


if __name__ == "__main__":
    main()
