#!/usr/bin/env python3
"""Locate bins of a config whose GPU FastFCA run raises, and dump them."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_1805_06572_b200 as P  # noqa: E402
from paper_1805_06572_b200.synth import CONFIGS, config_mixture, init_seed  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
y = config_mixture(cfg, 0)
model = P.init_random(y, init_seed(cfg, 0))


def fails(bins):
    yb = np.ascontiguousarray(y[:, bins])
    m = P.SpatialModel(v=np.ascontiguousarray(model.v[:, :, bins]),
                       S=np.ascontiguousarray(model.S[:, bins]),
                       v_floor=np.ascontiguousarray(model.v_floor[bins]))
    try:
        P.fastfca_run(yb, m, cfg.L, compute_likelihood=False)
        return None
    except Exception as exc:  # noqa: BLE001
        return repr(exc)


bad = []
for f in range(cfg.F):
    r = fails([f])
    if r:
        bad.append(f)
        print("bin", f, r, flush=True)
    if len(bad) >= 3:
        break
print("failing bins:", bad)
if bad:
    f = bad[0]
    np.savez("gpurun_out/c2_bad_bin.npz", y=y[:, [f]], v0=model.v[:, :, [f]], S0=model.S[:, [f]],
             floor=model.v_floor[[f]], L=cfg.L, f=f)
    for L in range(1, cfg.L + 1):
        m = P.SpatialModel(v=model.v[:, :, [f]], S=model.S[:, [f]], v_floor=model.v_floor[[f]])
        try:
            P.fastfca_run(np.ascontiguousarray(y[:, [f]]), m, L, compute_likelihood=False)
        except Exception as exc:  # noqa: BLE001
            print("first failing L =", L, repr(exc))
            break
