#!/usr/bin/env python3
"""Device timeline of one EM run (torch.profiler / CUPTI kernel records):
per-kernel totals, device-busy union vs wall span, and idle gaps — where the
per-iteration overhead of a run goes.

    python profiles/timeline.py --config 3 [--streams 1|2] [--engine fast]
"""

import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import (plan_chunks, run_device, run_device_streams,  # noqa: E402
                                           status_of)
from paper_1805_06572_b200.sharding import shard_chunk_frames  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--engine", default="fast")
    ap.add_argument("--streams", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
    y, v, s, fl = (torch.from_numpy(x).cuda() for x in (Y, V, S, FL))
    M, N, F, I = Y.shape
    cf = shard_chunk_frames(cfg.M, cfg.N, cfg.F, cfg.I, "c128", a.engine, max_world=cfg.max_world)
    bufs = {"images": torch.empty((M, 2, N, F, I), dtype=torch.complex128, device="cuda"),
            "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device="cuda"),
            "v": torch.empty_like(v)}

    streams = [torch.cuda.Stream() for _ in range(a.streams)]
    wss = [None] * a.streams

    def step():
        if a.streams > 1:
            r = run_device_streams(a.engine, y, v, s, fl, cfg.L, nstreams=a.streams, out=bufs,
                                   workspaces=wss, streams=streams, likelihood=False, check=False,
                                   chunk_frames=cf)
            for i, p in enumerate(r.parts):
                wss[i] = p.workspace
            r.wait()
        else:
            r = run_device(a.engine, y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                           chunk_frames=cf)
            status_of(r)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    if not ks:
        print("no kernel records")
        return
    t0, t1 = ks[0][0], max(k[1] for k in ks)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for b, e, n in ks:
        tot[n[:70]] += (e - b) / 1e3
        cnt[n[:70]] += 1
    busy, cur_b, cur_e, prev = 0.0, None, None, None
    gaps, where = [], defaultdict(list)
    for b, e, n in ks:
        if cur_e is None or b > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_b
                gaps.append((b - cur_e) / 1e3)
                where[(prev[:28], n[:28])].append((b - cur_e) / 1e3)
            cur_b, cur_e = b, e
        else:
            cur_e = max(cur_e, e)
        prev = n
    busy += cur_e - cur_b
    rec = {"config": a.config, "engine": a.engine, "streams": a.streams,
           "span_ms": round((t1 - t0) / 1e3, 3), "busy_ms": round(busy / 1e3, 3),
           "idle_ms": round(sum(gaps), 3), "gaps": len(gaps),
           "gap_us_by_transition": {f"{k[0]} -> {k[1]}": [len(v), round(1e3 * sum(v) / len(v), 1)]
                                    for k, v in where.items()},
           "kernels": {k: {"n": cnt[k], "ms": round(v, 3)} for k, v in
                       sorted(tot.items(), key=lambda kv: -kv[1])}}
    print(json.dumps(rec))
    if a.out:
        prof.export_chrome_trace(a.out)


if __name__ == "__main__":
    main()
