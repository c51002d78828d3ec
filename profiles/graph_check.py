#!/usr/bin/env python3
"""Config-3 run time with and without the cached run graph (CUDA events
around K back-to-back runs on preallocated buffers)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200._engine import run_device, status_of  # noqa: E402
from paper_1805_06572_b200.sharding import shard_chunk_frames  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
y, v, s, fl = (torch.from_numpy(x).cuda() for x in (Y, V, S, FL))
M, N, F, I = Y.shape
cf = shard_chunk_frames(cfg.M, cfg.N, cfg.F, cfg.I, "c128", "fast", max_world=cfg.max_world)
bufs = {"images": torch.empty((M, 2, N, F, I), dtype=torch.complex128, device="cuda"),
        "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device="cuda"),
        "v": torch.empty_like(v)}
r = run_device("fast", y, v, s, fl, cfg.L, likelihood=False, check=True, out=bufs,
               chunk_frames=cf, timing=False)
bufs["workspace"] = r.workspace
for graph in (False, True, False, True):
    for _ in range(2):
        run_device("fast", y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                   chunk_frames=cf, timing=False, graph=graph)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        r = run_device("fast", y, v, s, fl, cfg.L, likelihood=False, check=False, out=bufs,
                       chunk_frames=cf, timing=False, graph=graph)
    e1.record()
    torch.cuda.synchronize()
    status_of(r)
    print(f"graph={graph}: {e0.elapsed_time(e1) / 5:.3f} ms per run", flush=True)
