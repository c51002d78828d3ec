#!/usr/bin/env python3
"""One device init_from_masks on a BASELINE config (for ncu captures)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import make_inputs, shard  # noqa: E402
from paper_1805_06572_b200.initializers import init_from_masks_batch  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--mixtures", type=int, default=32)
a = ap.parse_args()
cfg = CONFIGS[a.config]
Y, _, _, _ = make_inputs(cfg, shard(cfg, 0, 1))
Y = Y[: a.mixtures]
m = init_from_masks_batch(torch.from_numpy(Y).cuda())
torch.cuda.synchronize()
print("ok", Y.shape)
