#!/usr/bin/env python3
"""Throughput of both engines on all five BASELINE configs (1 GPU, inputs
resident in HBM, outputs preallocated), plus the CPU oracle port on a bounded
sample of each config. One JSON line per (config, engine, dtype).

    python profiles/all_configs.py [--cpu] [--steps 3]
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import plan_chunks, run_device, status_of, torch_types  # noqa: E402
from paper_1805_06572_b200.sharding import shard_chunk_frames  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def measure(cfg, engine, dtype, steps, Y, V, S, FL, graph=False, parts=0, chunk=0):
    ctype, rtype = torch_types(dtype)
    y = torch.from_numpy(Y).cuda().to(ctype)
    v = torch.from_numpy(V).cuda().to(rtype)
    s = torch.from_numpy(S).cuda()
    fl = torch.from_numpy(FL).cuda()
    M, N, F, I = Y.shape
    cf = chunk or shard_chunk_frames(cfg.M, cfg.N, cfg.F, cfg.I, dtype, engine,
                                     max_world=cfg.max_world)
    nc = (N + cf - 1) // cf
    bufs = {"images": torch.empty((M, 2, N, F, I), dtype=ctype, device="cuda"),
            "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device="cuda"),
            "v": torch.empty_like(v)}
    r = run_device(engine, y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                   chunk_frames=cf, dtype=dtype, timing=False, graph=graph, bin_parts=parts)
    status_of(r)
    bufs["workspace"] = r.workspace
    r = run_device(engine, y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                   chunk_frames=cf, dtype=dtype, timing=False, graph=graph, bin_parts=parts)  # graph built
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        r = run_device(engine, y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                       chunk_frames=cf, dtype=dtype, timing=False, graph=graph, bin_parts=parts)
    e1.record()
    torch.cuda.synchronize()
    status_of(r)
    ms = e0.elapsed_time(e1) / steps
    kr = run_device(engine, y, v, s, fl, cfg.L, likelihood=False, check=True, out=bufs,
                    chunk_frames=cf, kernel_timing=True, dtype=dtype, bin_parts=parts)
    hot = kr.kernel_ms[:-1] if len(kr.kernel_ms) > 1 else kr.kernel_ms
    k_ms = sum(hot) / len(hot) if hot else float("nan")
    r_bytes = 8 if dtype == "c128" else 4
    gbs = (2 * I + 4) * r_bytes * M * F * N / (k_ms / 1e3) / 1e9
    return {"config": cfg.index, "engine": engine, "dtype": dtype, "graph": graph,
            "tf_bin_it_per_s": M * F * N * cfg.L / (ms / 1e3), "ms_per_run": ms,
            "parts": parts, "pass_ms": k_ms, "pass_GBps": gbs, "chunk_frames": cf, "nchunk": nc}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--configs", default="0,1,2,3,4")
    ap.add_argument("--graph", type=int, default=1, help="replay runs as CUDA graphs")
    ap.add_argument("--engines", default="fast,fca")
    ap.add_argument("--parts", default="0", help="bin windows to sweep (0 = driver plan)")
    ap.add_argument("--chunks", default="0", help="chunk_frames to sweep (0 = shard plan)")
    ap.add_argument("--dtypes", default="", help="restrict dtypes (c128,c64)")
    a = ap.parse_args()
    for idx in [int(x) for x in a.configs.split(",")]:
        cfg = CONFIGS[idx]
        Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
        for engine in a.engines.split(","):
            dtypes = [d for d in cfg.dtypes if not a.dtypes or d in a.dtypes.split(",")]
            sweep = [(d, k, c) for d in dtypes for k in map(int, a.parts.split(","))
                     for c in map(int, a.chunks.split(","))]
            for dtype, parts, chunk in sweep:
                rec = measure(cfg, engine, dtype, a.steps, Y, V, S, FL, graph=bool(a.graph),
                              parts=parts, chunk=chunk)
                if a.cpu and dtype == "c128":
                    from oracle import cpu_port

                    t0 = time.time()
                    val, desc, kind, cores = cpu_port.measure(cfg, engine, 0,
                                                              len(os.sched_getaffinity(0)))
                    rec["cpu_port"] = {"tf_bin_it_per_s": val, "sample": desc, "cores": cores,
                                       "wall_s": round(time.time() - t0, 1)}
                print(json.dumps(rec), flush=True)
        del Y, V, S, FL
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
