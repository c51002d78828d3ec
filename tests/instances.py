"""Seeded random test instances (same recipe as the reference's
``tests/oracles.py:64-78`` ``random_instance`` and the backend cross-check
instance of ``tests/test_backend.py:16-22``)."""

import numpy as np


def random_instance(seed, n_frames=6, n_bins=3, n_chan=2):
    """y ~ CN(0, 2) i.i.d., v = 0.2 + U(0,1), S_j(f) = a a^H + 0.5 I."""
    gen = np.random.default_rng(seed)
    y = gen.standard_normal((n_frames, n_bins, n_chan)) + 1j * gen.standard_normal(
        (n_frames, n_bins, n_chan))
    v = 0.2 + gen.random((2, n_frames, n_bins))
    S = np.zeros((2, n_bins, n_chan, n_chan), dtype=complex)
    for j in range(2):
        for f in range(n_bins):
            a = gen.standard_normal((n_chan, n_chan)) + 1j * gen.standard_normal(
                (n_chan, n_chan))
            S[j, f] = a @ a.conj().T + 0.5 * np.eye(n_chan)
    return y, v, S


def kernel_instance():
    """(y, v, S, P, lam) with N=9, F=4, I=3 (test_backend.py:16-22 shapes)."""
    y, v, S = random_instance(50, n_frames=9, n_bins=4, n_chan=3)
    gen = np.random.default_rng(51)
    P = gen.standard_normal((4, 3, 3)) + 1j * gen.standard_normal((4, 3, 3))
    lam = 0.3 + gen.random((4, 3))
    return y, v, S, P, lam


def random_complex(gen, shape):
    return gen.standard_normal(shape) + 1j * gen.standard_normal(shape)
