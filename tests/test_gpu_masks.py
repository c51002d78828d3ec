"""GPU parity for the mask-clustering initialiser (csrc/ffca_masks.cu,
SURVEY.md §8(f) row 3): against the unmodified reference's outputs
(tests/golden/masks.npz) and the pinned oracle, plus the reference's own
properties (test_initializers.py:60-131): a valid model, channel
permutation equivariance, determinism, the N < 2 I fallback; batch == single.
Labels are discrete, so agreement is exact or fails loudly; continuous
outputs within 1e-10 relative."""

import numpy as np
import pytest

from oracle import masks_oracle as MO
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

TOL = 1e-10
G = load_golden("masks")
# shared_direction: every frame has the same direction, so all phase-aligned
# unit vectors coincide and the 2-means distances tie up to rounding; the
# reference's labels there are decided by its own rounding noise (its test
# only asserts a valid model, test_initializers.py:88-94) — checked below
# for validity instead of equality
DEGENERATE = {"shared_direction"}
CASES = [str(c) for c in G["cases"] if str(c) not in DEGENERATE]


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def _init(y):
    from paper_1805_06572_b200 import init_from_masks

    return init_from_masks(y)


@pytest.mark.parametrize("case", CASES)
def test_matches_reference(case):
    m = _init(G[f"{case}_y"])
    assert _rel(m.v, G[f"{case}_v"]) <= TOL
    assert _rel(m.S, G[f"{case}_S"]) <= TOL
    assert _rel(m.v_floor, G[f"{case}_floor"]) <= TOL


def test_degenerate_geometry_gives_valid_model():
    y = G["shared_direction_y"]
    m = _init(y)
    assert np.all(m.v >= m.v_floor[None, None, :]) and np.all(m.v_floor > 0)
    assert _rel(m.v_floor, G["shared_direction_floor"]) <= TOL
    assert np.abs(m.S - np.conj(np.swapaxes(m.S, -1, -2))).max() <= 1e-12
    assert np.linalg.eigvalsh(m.S).min() > 0
    tr = np.trace(m.S, axis1=-2, axis2=-1).real
    assert np.allclose(tr, 1.0 + 1e-2 * y.shape[-1])  # unit trace + ridge
    # each point's power goes to exactly one source (the other is floored)
    pp = (np.abs(y) ** 2).sum(-1) / y.shape[-1]
    got = np.where(m.v[0] > m.v_floor, m.v[0], 0) + np.where(m.v[1] > m.v_floor, m.v[1], 0)
    big = pp > m.v_floor
    assert np.allclose(got[big], pp[big], rtol=1e-12)


@pytest.mark.parametrize("shape", [(200, 33, 4), (150, 17, 2), (90, 11, 8), (1250, 5, 3)])
def test_matches_oracle(shape):
    rng = np.random.default_rng(sum(shape))
    N, F, I = shape
    # two directional sources with alternating activity plus noise
    d = rng.standard_normal((2, F, I)) + 1j * rng.standard_normal((2, F, I))
    act = (np.arange(N) // 7) % 2
    s = (rng.standard_normal((2, N, F)) + 1j * rng.standard_normal((2, N, F)))
    s[0] *= act[:, None]
    s[1] *= 1 - act[:, None]
    y = s[0][..., None] * d[0][None] + s[1][..., None] * d[1][None]
    y = y + 0.05 * (rng.standard_normal(y.shape) + 1j * rng.standard_normal(y.shape))
    v, S, fl = MO.init_from_masks(y)
    m = _init(y)
    assert _rel(m.v, v) <= TOL
    assert _rel(m.S, S) <= TOL
    assert _rel(m.v_floor, fl) <= TOL


def test_valid_model_permutation_and_determinism():
    rng = np.random.default_rng(3)
    y = rng.standard_normal((30, 5, 3)) + 1j * rng.standard_normal((30, 5, 3))
    m = _init(y)
    assert m.v.shape == (2, 30, 5) and m.S.shape == (2, 5, 3, 3)
    assert np.all(m.v >= m.v_floor[None, None, :]) and np.all(m.v_floor > 0)
    assert np.abs(m.S - np.conj(np.swapaxes(m.S, -1, -2))).max() <= 1e-12
    assert np.linalg.eigvalsh(m.S).min() > 0
    perm = np.array([2, 0, 1])
    mp = _init(y[:, :, perm])
    assert np.abs(mp.v - m.v).max() <= 1e-10 * m.v.max()
    assert np.abs(mp.S - m.S[:, :, perm][:, :, :, perm]).max() <= 1e-10 * np.abs(m.S).max()
    m2 = _init(y)
    assert np.array_equal(m.v, m2.v) and np.array_equal(m.S, m2.S)


def test_fallback_and_device_tensors():
    import torch

    from paper_1805_06572_b200 import init_random

    rng = np.random.default_rng(4)
    y = rng.standard_normal((3, 4, 2)) + 1j * rng.standard_normal((3, 4, 2))
    assert np.array_equal(_init(y).S, init_random(y, seed=0).S)
    y = rng.standard_normal((40, 6, 2)) + 1j * rng.standard_normal((40, 6, 2))
    md = _init(torch.from_numpy(y).cuda())
    assert md.v.is_cuda and md.S.is_cuda
    mh = _init(y)
    assert np.array_equal(md.v.cpu().numpy(), mh.v)


def test_batch_equals_single():
    from paper_1805_06572_b200 import init_from_masks_batch

    rng = np.random.default_rng(5)
    Y = rng.standard_normal((3, 50, 9, 2)) + 1j * rng.standard_normal((3, 50, 9, 2))
    mb = init_from_masks_batch(Y)
    for k in range(3):
        m = _init(Y[k])
        assert np.array_equal(mb.v[k], m.v)
        assert np.array_equal(mb.S[k], m.S)
        assert np.array_equal(mb.v_floor[k], m.v_floor)
