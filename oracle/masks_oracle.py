"""CPU oracle for the mask-clustering initialiser — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may use this module; the product path
(``paper_1805_06572_b200.initializers.init_from_masks``) runs on the GPU.

A numpy restatement of the reference ``init_from_masks``
(``initializers.py:42-143``): per bin, unit-normalise and phase-align the
observation vectors to the strongest channel (``:100-106``), split the
frames into two groups by deterministic 2-means (``_two_means``,
``:42-68``: seeds = highest-power frame and the frame farthest from it,
empty-cluster reseeding with the worst-fit frame, <= 50 iterations), build
unit-trace group covariances plus a 1e-2 ridge (``:108-115``); then align the
labels across bins by correlating centred binary mask profiles against a
global profile grown in decreasing bin-power order and refined by up to five
sweeps (``:117-137``); powers are the group-masked point powers, floored
(``:139-143``). Falls back to ``init_random(y, 0)`` when N < 2 I (``:84-85``).

The alignment correlations are evaluated here (and on the GPU) on the exact
integer form of the centred masks, N * mask - count, so a flip decision is
the sign of the exact rational correlation; the reference's float dot can
only disagree when that correlation is zero up to its rounding.

Pinned by ``tests/test_masks_oracle.py`` against golden outputs of the
unmodified reference (``tests/golden/make_golden_masks.py``).
"""

from __future__ import annotations

import numpy as np

from oracle import fastfca_oracle as O

MASK_COV_RIDGE = 1e-2
KMEANS_ITERS = 50


def two_means(z, weights):
    """initializers.py:42-68; True = cluster 0."""
    n = z.shape[0]
    c0 = z[int(np.argmax(weights))]
    d = np.sum(np.abs(z - c0) ** 2, axis=1)
    c1 = z[int(np.argmax(d))]
    labels = np.zeros(n, dtype=bool)
    for _ in range(KMEANS_ITERS):
        d0 = np.sum(np.abs(z - c0) ** 2, axis=1)
        d1 = np.sum(np.abs(z - c1) ** 2, axis=1)
        new = d0 <= d1
        if new.all() or not new.any():
            far = int(np.argmax(np.where(new, d0, d1)))
            new = new.copy()
            new[far] = ~new[far]
        if np.array_equal(new, labels):
            break
        labels = new
        c0 = z[labels].mean(axis=0)
        c1 = z[~labels].mean(axis=0)
    return labels


def bin_masks(y):
    """Per-bin labels (N, F) and group covariances S (2, F, I, I)."""
    N, F, I = y.shape
    power = (np.abs(y) ** 2).sum(axis=-1)
    masks = np.empty((N, F), dtype=bool)
    S = np.empty((2, F, I, I), dtype=np.complex128)
    eye = np.eye(I)
    for f in range(F):
        w = y[:, f, :]
        z = w / np.maximum(np.sqrt(power[:, f]), 1e-300)[:, None]
        ref = int(np.argmax((np.abs(w) ** 2).sum(axis=0)))
        rv = z[:, ref]
        mag = np.abs(rv)
        phase = np.where(mag > 0, rv / np.maximum(mag, 1e-300), 1.0)
        z = z * np.conj(phase)[:, None]
        lab = two_means(z, power[:, f])
        masks[:, f] = lab
        for j, sel in enumerate((lab, ~lab)):
            if sel.any():
                cov = w[sel].T @ w[sel].conj() / sel.sum()
            else:
                cov = eye.astype(np.complex128)
            tr = float(np.real(np.trace(cov)))
            cov = cov / tr if tr > 0 else eye / I
            S[j, f] = cov + MASK_COV_RIDGE * eye
    return masks, S, power


def align_flips(masks, bin_power):
    """initializers.py:117-137 on the exact integer centred masks."""
    N, F = masks.shape
    D = N * masks.astype(np.int64) - masks.sum(axis=0, keepdims=True).astype(np.int64)
    order = np.argsort(-bin_power, kind="stable")
    flip = np.zeros(F, dtype=bool)
    g = D[:, order[0]].copy()
    for f in order[1:]:
        if int(D[:, f] @ g) < 0:
            flip[f] = True
        g = g + (-D[:, f] if flip[f] else D[:, f])
    for _ in range(5):
        changed = False
        g = np.where(flip[None, :], -D, D).sum(axis=1)
        for f in order:
            d = -D[:, f] if flip[f] else D[:, f]
            if int(d @ (g - d)) < 0:
                flip[f] = ~flip[f]
                g = g - 2 * d
                changed = True
        if not changed:
            break
    return flip


def init_from_masks(y):
    """(v, S, floor) like the reference init_from_masks(y)."""
    y = np.asarray(y, dtype=np.complex128)
    N, F, I = y.shape
    if N < 2 * I:
        return O.init_random(y, 0)
    masks, S, power = bin_masks(y)
    flip = align_flips(masks, power.sum(axis=0))
    masks[:, flip] = ~masks[:, flip]
    S[:, flip] = S[::-1, flip]
    floor = O.power_floor(y)
    pp = power / I
    v = np.stack([masks * pp, (~masks) * pp])
    v = np.maximum(v, floor[None, None, :])
    return v, S, floor
