"""Print the chunk plan (shard_chunk_frames) and modelled grids per config / engine / dtype."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1805_06572_b200.sharding import grid_model, plan_shard, shard_chunk_frames  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402

for c in CONFIGS.values():
    for eng in ("fast", "fca"):
        for dt in c.dtypes:
            cf = shard_chunk_frames(c.M, c.N, c.F, c.I, dt, eng, max_world=c.max_world)
            grids = {}
            for w in (1, 2, 4, 8):
                if w > c.max_world:
                    break
                sh = plan_shard(c.M, c.F, 0, w)
                G = sh.size * (c.F if sh.axis == "mixtures" else 1)
                grids[w] = grid_model(G, c.N, c.I, cf, dt, eng)
            print(c.index, eng, dt, "cf", cf, "nchunk", -(-c.N // cf), grids, flush=True)
