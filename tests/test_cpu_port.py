"""The C restatement used for the CPU baseline agrees with the pinned numpy
oracle (CPU only)."""

import numpy as np

from oracle import cpu_port
from oracle import fastfca_oracle as O
from tests.conftest import load_golden


def test_c_port_fastfca_matches_oracle():
    g = load_golden("runs_cfg3m0")
    y, v0, S0, fl, L = g["y"], g["v0"], g["S0"], g["floor"], int(g["L"])
    em, v, S_t, P, mu = cpu_port.fastfca_em(y[None], v0[None], S0[None], fl[None], L,
                                            want_images=True)
    assert em > 0
    assert O.scale_dev(v[0], g["fast_v"]) <= 1e-10


def test_c_port_fca_matches_oracle():
    g = load_golden("runs_acc2")
    y, v0, S0, fl, L = g["y"], g["v0"], g["S0"], g["floor"], int(g["L"])
    em, v, S, mu = cpu_port.fca_em(y[None], v0[None], S0[None], fl[None], L, want_images=True)
    assert O.scale_dev(v[0], g["fca_v"]) <= 1e-10
    assert O.scale_dev(S[0], g["fca_S"]) <= 1e-10
    assert O.scale_dev(mu[0], g["fca_images"]) <= 1e-10


def test_c_port_batch_equals_singles():
    gen = np.random.default_rng(3)
    Y = gen.standard_normal((3, 40, 5, 3)) + 1j * gen.standard_normal((3, 40, 5, 3))
    inits = [O.init_random(Y[m], 10 + m) for m in range(3)]
    V = np.stack([i[0] for i in inits])
    S = np.stack([i[1] for i in inits])
    FL = np.stack([i[2] for i in inits])
    _, vb, _, _, _ = cpu_port.fastfca_em(Y, V, S, FL, 4)
    for m in range(3):
        _, vs, _, _, _ = cpu_port.fastfca_em(Y[m:m + 1], V[m:m + 1], S[m:m + 1], FL[m:m + 1], 4)
        assert np.array_equal(vb[m], vs[0])
