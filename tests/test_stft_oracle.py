"""CPU tier for the STFT row: the oracle pinned to golden vectors from the
unmodified reference (tests/golden/make_golden_stft.py) and to a direct DFT
matrix (reference test_stft.py:9-22); the device API's argument validation
(reference test_stft.py:107-115), which runs before any GPU work."""

import numpy as np
import pytest

from oracle import stft_oracle as SO
from tests.conftest import load_golden

TOL = 1e-12


def _dev(a, b):
    b = np.asarray(b)
    den = np.abs(b).max()
    return float(np.abs(np.asarray(a) - b).max() / (den if den > 0 else 1.0))


G = load_golden("stft")
CASES = [str(c) for c in G["cases"]]


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_reference_golden(case):
    x, L = G[f"{case}_x"], int(G[f"{case}_L"])
    trim = int(G[f"{case}_trim"])
    spec = SO.analyze(x, L)
    assert spec.shape == G[f"{case}_spec"].shape
    assert _dev(spec, G[f"{case}_spec"]) <= TOL
    back = SO.synthesize(G[f"{case}_spec"], L, x.shape[1] if trim < 0 else trim)
    assert back.shape == G[f"{case}_back"].shape
    assert _dev(back, G[f"{case}_back"]) <= TOL
    rback = SO.synthesize(G[f"{case}_rnd"], L)
    assert _dev(rback, G[f"{case}_rback"]) <= TOL


def test_oracle_matches_direct_dft():
    rng = np.random.default_rng(7)
    x = rng.standard_normal(3000)
    spec = SO.analyze(x[None], 256)
    for k in (0, 3, 10, spec.shape[0] - 1):
        ref = SO.direct_dft_frame(x, k, 256)
        assert np.abs(spec[k, :, 0] - ref).max() <= 1e-10 * np.abs(ref).max()


def test_frame_count_rule():
    assert SO.frames_for(1, 32) == 2
    assert SO.frames_for(64, 32) == 3
    assert SO.frames_for(65, 32) == 4


def test_bad_config_rejected_before_device_work():
    from paper_1805_06572_b200.errors import ConfigurationError
    from paper_1805_06572_b200.stft import stft_analyze, stft_synthesize
    from paper_1805_06572_b200.types import AudioBuffer, SpectrogramTensor

    audio = AudioBuffer(16000, np.zeros((1, 1000)))
    with pytest.raises(ConfigurationError):
        stft_analyze(audio, 1000, 500)  # not a power of two
    with pytest.raises(ConfigurationError):
        stft_analyze(audio, 1024, 256)  # shift mismatch
    spec = SpectrogramTensor(np.zeros((3, 513, 1), dtype=complex), 16000, 1024, 512, 1000)
    with pytest.raises(ConfigurationError):
        stft_synthesize(spec, 512, 256)  # bin count mismatch
