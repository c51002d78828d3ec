"""Full BASELINE.json sizes on the GPU: size-independent properties plus
oracle parity on sampled bins / mixtures.

Bins (and mixtures) are independent in both EM engines (the reference is
bitwise bin-shard invariant), so the oracle run on a handful of
bins of the full-size input is an exact reference for those bins of the GPU's
full-size run.
"""

import numpy as np
import pytest

from oracle import fastfca_oracle as O
from paper_1805_06572_b200.synth import CONFIGS, config_mixture, init_seed

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = 1e-9


def _ll_dev(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.abs(b)))


def _monotone(trace):
    return all(b >= a - 1e-8 * abs(a) for a, b in zip(trace, trace[1:]))


def _sampled_oracle(y, model, L, bins, engine):
    ys = np.ascontiguousarray(y[:, bins])
    v = np.ascontiguousarray(model.v[:, :, bins])
    S = np.ascontiguousarray(model.S[:, bins])
    fl = np.ascontiguousarray(model.v_floor[bins])
    run = O.fastfca_run if engine == "fast" else O.fca_run
    return run(ys, v, S, fl, L)


def _compare_bins(res, ref, bins):
    assert O.scale_dev(res.model.v[:, :, bins], ref.v) <= TOL
    assert O.scale_dev(res.model.S[:, bins], ref.S) <= TOL
    assert O.scale_dev(res.images[:, :, bins], ref.images) <= TOL


@pytest.mark.parametrize("idx", [0, 1, 2, 4])
def test_single_mixture_configs_fastfca_and_fca(idx):
    import paper_1805_06572_b200 as P

    cfg = CONFIGS[idx]
    y = config_mixture(cfg, 0)
    model = P.init_random(y, init_seed(cfg, 0))
    fast = P.fastfca_run(y, model, cfg.L)
    fca = P.fca_run(y, model, cfg.L)
    for res in (fast, fca):
        assert _monotone(res.loglik_trace)
        resid = res.images[0] + res.images[1] - y
        assert np.abs(resid).max() <= 1e-9 * np.abs(y).max()
    # the two engines are the same fixed-point map (reference criterion 1/2)
    assert O.scale_dev(fast.images, fca.images) <= 1e-8
    assert O.scale_dev(fast.model.v, fca.model.v) <= 1e-8
    assert _ll_dev(fast.loglik_trace, fca.loglik_trace) <= 1e-9
    bins = sorted({0, cfg.F // 3, cfg.F - 1})
    for engine, res in (("fast", fast), ("fca", fca)):
        ref = _sampled_oracle(y, model, cfg.L, bins, engine)
        _compare_bins(res, ref, bins)


@pytest.mark.parametrize("engine", ["fast", "fca"])
def test_config2_complex64_within_1e4(engine):
    """Full config 2 (I = 8) in complex64 against the complex128 oracle on
    sampled bins, both engines (BASELINE.json configs[2] names c64)."""
    import paper_1805_06572_b200 as P

    cfg = CONFIGS[2]
    y = config_mixture(cfg, 0)
    model = P.init_random(y, init_seed(cfg, 0))
    bins = [0, 256, 512]
    ref = _sampled_oracle(y, model, cfg.L, bins, engine)
    run = P.fastfca_run if engine == "fast" else P.fca_run
    res = run(y, model, cfg.L, dtype="c64")
    assert O.scale_dev(res.model.v[:, :, bins], ref.v) <= 1e-4
    assert O.scale_dev(res.model.S[:, bins], ref.S) <= 1e-4
    assert O.scale_dev(res.images[:, :, bins], ref.images) <= 1e-4


@pytest.fixture(scope="module")
def config3_batch():
    import paper_1805_06572_b200 as P

    cfg = CONFIGS[3]
    ys, models = [], []
    for m in range(cfg.M):
        y = config_mixture(cfg, m)
        ys.append(y)
        models.append(P.init_random(y, init_seed(cfg, m)))
    Y = np.stack(ys)
    batch = P.SpatialModel(v=np.stack([m.v for m in models]), S=np.stack([m.S for m in models]),
                           v_floor=np.stack([m.v_floor for m in models]))
    return cfg, ys, models, Y, batch


@pytest.mark.parametrize("engine", ["fast", "fca"])
@pytest.mark.parametrize("dtype,tol", [("c128", TOL), ("c64", 1e-4)])
def test_config3_batch_of_256(config3_batch, engine, dtype, tol):
    """The full 256-mixture config-3 batch through the public API (host
    buffers -> chunked, transfer-overlapped runs), both engines, both
    precisions; sampled mixtures and bins against the complex128 oracle."""
    import paper_1805_06572_b200 as P

    cfg, ys, models, Y, batch = config3_batch
    run = P.fastfca_run if engine == "fast" else P.fca_run
    res = run(Y, batch, cfg.L, dtype=dtype)
    for m in (0, 131, 255):
        assert _monotone(res.loglik_trace[m])
        bins = [3, 200]
        ref = _sampled_oracle(ys[m], models[m], cfg.L, bins, engine)
        assert O.scale_dev(res.model.v[m][:, :, bins], ref.v) <= tol
        assert O.scale_dev(res.model.S[m][:, bins], ref.S) <= tol
        assert O.scale_dev(res.images[m][:, :, bins], ref.images) <= tol
