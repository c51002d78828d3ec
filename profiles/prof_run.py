#!/usr/bin/env python3
"""One device EM run of a BASELINE config for ncu / compute-sanitizer
captures (no graph, no timing): the kernels of every pass launch once per
iteration, so ``ncu -k <name> --launch-skip S -c 1`` picks a steady-state one.

    python profiles/prof_run.py --config 2 --engine fast [--dtype c128] [--iters 3] [--mixtures M]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import run_device, status_of, torch_types  # noqa: E402
from paper_1805_06572_b200.sharding import shard_chunk_frames  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--engine", default="fast")
    ap.add_argument("--dtype", default="c128")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--mixtures", type=int, default=0, help="batch subset (config 3)")
    ap.add_argument("--likelihood", action="store_true")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    sh = shard(cfg, 0, 1)
    if a.mixtures and cfg.M > 1:
        sh = ("mixtures", 0, a.mixtures)
    Y, V, S, FL = make_inputs(cfg, sh)
    ctype, rtype = torch_types(a.dtype)
    y = torch.from_numpy(Y).cuda().to(ctype)
    v = torch.from_numpy(V).cuda().to(rtype)
    s = torch.from_numpy(S).cuda()
    fl = torch.from_numpy(FL).cuda()
    cf = shard_chunk_frames(cfg.M, cfg.N, cfg.F, cfg.I, a.dtype, a.engine, max_world=cfg.max_world)
    r = run_device(a.engine, y, v, s, fl, a.iters, likelihood=a.likelihood, check=False,
                   chunk_frames=cf, dtype=a.dtype, timing=False)
    status_of(r)
    torch.cuda.synchronize()
    print(f"prof_run: config {cfg.index} {a.engine} {a.dtype} L={a.iters} M={Y.shape[0]} "
          f"chunk_frames={cf} ok", flush=True)


if __name__ == "__main__":
    main()
