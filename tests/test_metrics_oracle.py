"""The SDR oracle (oracle/metrics_oracle.py) pinned to golden values of the
unmodified reference fastfca.metrics (tests/golden/make_golden_sdr.py)."""

import numpy as np

from oracle import metrics_oracle as MO
from tests.conftest import load_golden


def test_sdr_oracle_matches_reference_golden():
    g = load_golden("sdr")
    for name in [str(n) for n in g["names"]]:
        val = MO.sdr(g[f"{name}_est"], g[f"{name}_ref"], int(g[f"{name}_max_shift"]))
        assert abs(val - float(g[f"{name}_sdr"])) <= 1e-9 * max(1.0, abs(float(g[f"{name}_sdr"]))), name


def test_sdr_pairing_oracle_matches_reference_golden():
    g = load_golden("sdr")
    vals, perm = MO.sdr_pairing((g["pair_e1"], g["pair_e2"]), (g["pair_r1"], g["pair_r2"]))
    assert tuple(perm) == tuple(int(x) for x in g["pair_perm"])
    assert np.allclose(vals, g["pair_values"], rtol=1e-12, atol=0)
