import sys
sys.path.insert(0, ".")
import numpy as np, torch
from tests.instances import random_complex
import paper_1805_06572_b200 as P
from paper_1805_06572_b200._engine import run_device
gen = np.random.default_rng(23)
for shape in [(2, 70, 11, 3), (1, 70, 11, 3), (1, 200, 40, 2), (1, 300, 70, 4)]:
    Y = torch.from_numpy(random_complex(gen, shape)).cuda()
    M = shape[0]
    inits = [P.init_random(Y[m], 60 + m) for m in range(M)]
    V = torch.stack([i.v for i in inits]); S = torch.stack([i.S for i in inits]); FL = torch.stack([i.v_floor for i in inits])
    for ll in (False, True):
        for graph in (False, True):
            try:
                r = run_device("fast", Y, V, S, FL, 4, likelihood=ll, timing=False, graph=graph, persist=False)
                print(shape, "ll", ll, "graph", graph, "ok", float(r.v.sum()))
            except Exception as e:
                print(shape, "ll", ll, "graph", graph, "FAIL", type(e).__name__, str(e)[:60])
