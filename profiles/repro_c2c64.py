import sys, os
sys.path.insert(0, '.')
import torch, numpy as np
from bench import make_inputs, shard
from profiles.all_configs import measure
from paper_1805_06572_b200.synth import CONFIGS
cfg = CONFIGS[2]
Y, V, S, FL = make_inputs(cfg, shard(cfg, 0, 1))
order = sys.argv[1].split(",")
for d in order:
    print("measure", d, flush=True)
    print(measure(cfg, "fast", d, 1, Y, V, S, FL), flush=True)
