"""CPU tier for the mask-clustering initialiser row: the oracle
(oracle/masks_oracle.py) pinned to golden outputs of the unmodified reference
``init_from_masks`` (tests/golden/make_golden_masks.py)."""

import numpy as np
import pytest

from oracle import masks_oracle as MO
from tests.conftest import load_golden

G = load_golden("masks")
CASES = [str(c) for c in G["cases"]]


def _rel(a, b):
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference(case):
    v, S, fl = MO.init_from_masks(G[f"{case}_y"])
    assert v.shape == G[f"{case}_v"].shape and S.shape == G[f"{case}_S"].shape
    assert _rel(v, G[f"{case}_v"]) <= 1e-12
    assert _rel(S, G[f"{case}_S"]) <= 1e-12
    assert _rel(fl, G[f"{case}_floor"]) <= 1e-12


def test_two_means_reseeds_an_empty_cluster():
    z = np.ones((6, 2), dtype=complex)  # all identical: 2-means must still split
    lab = MO.two_means(z, np.ones(6))
    assert 0 < lab.sum() < 6
