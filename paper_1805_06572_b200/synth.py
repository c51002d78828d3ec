"""Seeded synthetic STFT-domain mixtures for the five BASELINE.json configs.

The reference ships no dataset for this path; BASELINE.json describes the
inputs generatively, so this module draws them (numpy, host side — it is the
input generator, not part of the EM path). SURVEY.md §8(d) fixes the recipe;
the draw order for one mixture seed ``s`` is, with
``gen = np.random.default_rng(s)``:

1. ``A_1``: real then imaginary part, each ``standard_normal((F, I, r))``;
2. ``A_2``: the same;
3. ``log v``: ``standard_normal((2, N, F))`` scaled by ``sigma``;
4. (config 4 only) the per-frame envelope: ``standard_normal((2, N))``
   innovations of a unit-variance AR(1) process with correlation time
   50 frames (``rho = exp(-1/50)``), added to ``log v`` for every bin;
5. the source excitations ``g_j``, in frame blocks of ``BLOCK`` frames: for
   each block, ``g_1`` real, ``g_1`` imaginary, ``g_2`` real, ``g_2``
   imaginary, each ``standard_normal((nb, F, I))``.

Then ``R_j(f) = A_j A_j^H + eps I``, ``x_j = sqrt(v_j) chol(R_j) g_j / sqrt 2``
and ``y = x_1 + x_2`` in the reference layout (N, F, I), complex128.
complex64 inputs are a cast of the same draw. Config 2 does not state
``sigma``; config 0's 1.5 is used. The config-4 envelope is not specified by
BASELINE.json; the AR(1) above is this repo's definition.

Initialisation for every config is the reference ``init_random`` recipe
(``initializers.py:20-39``) with seed ``s + 1_000_003``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BLOCK = 1000  # frames per excitation block (draw-order unit)
INIT_SEED_OFFSET = 1_000_003


@dataclass(frozen=True)
class Config:
    index: int
    M: int  # mixtures
    I: int  # channels
    F: int  # bins
    N: int  # frames
    L: int  # EM iterations
    rank: int  # rank of A (I unless rank-deficient)
    eps: float  # ridge on R_j
    sigma: float  # log-normal std of v
    envelope: bool
    dtypes: tuple
    description: str

    @property
    def tf_bins(self):
        return self.M * self.F * self.N

    @property
    def max_world(self):
        """GPUs the config is sharded over (BASELINE.json: config 3 by mixture
        and config 4 by bin across 1/2/4/8 GPUs; configs 0-2 are 1-GPU
        configs). The one chunk plan of every world size is the plan of the
        shard at this world size."""
        return 8 if self.index in (3, 4) else 1


CONFIGS = {
    0: Config(0, 1, 2, 257, 500, 10, 2, 1e-3, 1.5, False, ("c128",),
              "single mixture, I=2, F=257, N=500, L=10"),
    1: Config(1, 1, 3, 513, 1000, 50, 3, 1e-3, 2.0, False, ("c128",),
              "single mixture, I=3, F=513, N=1000, L=50"),
    2: Config(2, 1, 8, 513, 2000, 30, 2, 1e-2, 1.5, False, ("c128", "c64"),
              "single mixture, I=8 rank-2+1e-2, F=513, N=2000, L=30"),
    3: Config(3, 256, 4, 257, 1250, 20, 4, 1e-3, 1.5, False, ("c128", "c64"),
              "batch of 256 mixtures, I=4, F=257, N=1250, L=20"),
    4: Config(4, 1, 4, 1025, 20000, 50, 4, 1e-3, 2.0, True, ("c128",),
              "long mixture, I=4, F=1025, N=20000, L=50, AR(1) envelope"),
}


def _envelope(gen, N):
    rho = np.exp(-1.0 / 50.0)
    w = gen.standard_normal((2, N))
    e = np.empty((2, N))
    e[:, 0] = w[:, 0]
    s = np.sqrt(1.0 - rho * rho)
    for n in range(1, N):
        e[:, n] = rho * e[:, n - 1] + s * w[:, n]
    return e


def make_mixture(seed, I, F, N, rank=None, eps=1e-3, sigma=1.5, envelope=False,
                 return_truth=False):
    """Draw one 2-source mixture y (N, F, I) complex128 (see module docstring)."""
    r = I if rank is None else rank
    gen = np.random.default_rng(seed)
    A = []
    for _ in range(2):
        re = gen.standard_normal((F, I, r))
        im = gen.standard_normal((F, I, r))
        A.append(re + 1j * im)
    logv = sigma * gen.standard_normal((2, N, F))
    if envelope:
        logv += _envelope(gen, N)[:, :, None]
    v = np.exp(logv)
    eye = np.eye(I)
    R = np.stack([a @ np.conj(np.swapaxes(a, -1, -2)) + eps * eye for a in A])
    C = np.linalg.cholesky(R)  # (2, F, I, I)
    y = np.empty((N, F, I), dtype=np.complex128)
    sv = np.sqrt(v)
    inv_sqrt2 = 1.0 / np.sqrt(2.0)
    for n0 in range(0, N, BLOCK):
        n1 = min(N, n0 + BLOCK)
        nb = n1 - n0
        blk = np.zeros((nb, F, I), dtype=np.complex128)
        for j in range(2):
            gre = gen.standard_normal((nb, F, I))
            gim = gen.standard_normal((nb, F, I))
            g = (gre + 1j * gim) * inv_sqrt2
            x = np.matmul(C[j], g.transpose(1, 2, 0)).transpose(2, 0, 1)  # chol(R_j) g
            blk += sv[j, n0:n1, :, None] * x
        y[n0:n1] = blk
    if return_truth:
        return y, v, R
    return y


def config_mixture(cfg: Config, m=0, bins=None):
    """Mixture ``m`` of config ``cfg`` (seed = 1000*index + m), optional bin subset."""
    seed = 1000 * cfg.index + m
    y = make_mixture(seed, cfg.I, cfg.F, cfg.N, cfg.rank, cfg.eps, cfg.sigma, cfg.envelope)
    if bins is not None:
        y = np.ascontiguousarray(y[:, bins, :])
    return y


def init_seed(cfg: Config, m=0):
    return 1000 * cfg.index + m + INIT_SEED_OFFSET
