"""GPU parity for the device-resident separation chain (pipeline.py): STFT
analysis -> init_random -> EM -> STFT synthesis, against the same chain
composed from the pinned oracles (stft_oracle + fastfca_oracle), for both
engines; and a batch of mixtures against per-mixture runs."""

import numpy as np
import pytest

from oracle import fastfca_oracle as O
from oracle import stft_oracle as SO

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _mixture(seed, C=3, length=12000):
    rng = np.random.default_rng(seed)
    src = rng.standard_normal((2, length))
    src[1] *= np.abs(np.sin(np.linspace(0, 20, length)))  # different activity
    taps = rng.standard_normal((2, C, 6)) * np.exp(-np.arange(6))[None, None]
    x = np.zeros((C, length))
    for j in range(2):
        for c in range(C):
            x[c] += np.convolve(src[j], taps[j, c])[:length]
    return x


def _oracle_chain(x, L, iters, seed, engine):
    spec = SO.analyze(x, L)
    v0, S0, fl = O.init_random(spec, seed)
    run = O.fastfca_run if engine == "fastfca" else O.fca_run
    r = run(spec, v0, S0, fl, iters, compute_likelihood=True)
    return r, np.stack([SO.synthesize(r.images[j], L, x.shape[1]) for j in range(2)])


@pytest.mark.parametrize("engine", ["fastfca", "fca"])
def test_separate_matches_oracle_chain(engine):
    from paper_1805_06572_b200 import AudioBuffer, separate

    x = _mixture(1)
    L, iters, seed = 512, 8, 3
    ref, ref_t = _oracle_chain(x, L, iters, seed, engine)
    res, outs = separate(AudioBuffer(16000, x), iters, L, engine, seed)
    got = np.stack([o.samples for o in outs])
    assert got.shape == ref_t.shape == (2, 3, x.shape[1])
    assert O.scale_dev(got, ref_t) <= TOL
    assert O.scale_dev(res.model.v, ref.v) <= TOL
    ll = np.asarray(res.loglik_trace)
    assert np.max(np.abs(ll - np.asarray(ref.loglik_trace)) / np.abs(ref.loglik_trace)) <= TOL
    # the two images partition the mixture (posterior means sum to y)
    assert np.abs(got.sum(axis=0) - x).max() <= 1e-9 * np.abs(x).max()


def test_batched_separation_matches_single():
    import torch

    from paper_1805_06572_b200 import separate_device

    X = np.stack([_mixture(s, C=2, length=8000) for s in (4, 5, 6)])
    L, iters = 256, 6
    _, outb = separate_device(torch.from_numpy(X).cuda(), iters, L, seeds=[7, 8, 9])
    assert tuple(outb.shape) == (3, 2, 2, 8000)
    for m, s in enumerate((7, 8, 9)):
        _, one = separate_device(X[m], iters, L, seed=s)
        d = (outb[m] - one).abs().max().item() / one.abs().max().item()
        assert d <= 1e-12
