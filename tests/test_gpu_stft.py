"""GPU parity for the STFT front / back end: the CUDA
kernels (csrc/ffca_stft.cu) against the reference's golden vectors and the
pinned oracle, plus the reference's own STFT properties (test_stft.py):
zero in -> zero out, a sinusoid concentrates in its bin, linearity,
Parseval, exact overlap-add round trip. Tolerance: 1e-12 of the largest
magnitude (FP64 FFT vs numpy's pocketfft); round trips 1e-10."""

import numpy as np
import pytest

from oracle import stft_oracle as SO
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu

TOL = 1e-12
G = load_golden("stft")
CASES = [str(c) for c in G["cases"]]


def _dev(a, b):
    b = np.asarray(b)
    den = np.abs(b).max()
    return float(np.abs(np.asarray(a) - b).max() / (den if den > 0 else 1.0))


def _stft():
    from paper_1805_06572_b200 import stft

    return stft


def _audio(x, sr=16000):
    from paper_1805_06572_b200.types import AudioBuffer

    return AudioBuffer(sr, x)


@pytest.mark.parametrize("case", CASES)
def test_analyze_matches_reference(case):
    S = _stft()
    x, L = G[f"{case}_x"], int(G[f"{case}_L"])
    spec = S.stft_analyze(_audio(x), L, L // 2)
    assert spec.data.shape == G[f"{case}_spec"].shape
    assert spec.original_length == x.shape[1]
    assert _dev(spec.data, G[f"{case}_spec"]) <= TOL


@pytest.mark.parametrize("case", CASES)
def test_synthesize_matches_reference(case):
    S = _stft()
    from paper_1805_06572_b200.types import SpectrogramTensor

    x, L = G[f"{case}_x"], int(G[f"{case}_L"])
    trim = int(G[f"{case}_trim"])
    spec = SpectrogramTensor(G[f"{case}_spec"], 16000, L, L // 2, x.shape[1])
    back = S.stft_synthesize(spec, L, L // 2, length=None if trim < 0 else trim)
    assert back.samples.shape == G[f"{case}_back"].shape
    assert _dev(back.samples, G[f"{case}_back"]) <= TOL
    rnd = SpectrogramTensor(G[f"{case}_rnd"], 16000, L, L // 2, None)
    rb = S.stft_synthesize(rnd, L, L // 2)
    assert rb.samples.shape == G[f"{case}_rback"].shape
    assert _dev(rb.samples, G[f"{case}_rback"]) <= TOL


@pytest.mark.parametrize("L", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192])
@pytest.mark.parametrize("C", [1, 3, 8])
def test_every_length_against_oracle(L, C):
    S = _stft()
    rng = np.random.default_rng(L * 10 + C)
    x = rng.standard_normal((C, 3 * L + 5))
    spec = S.stft_analyze_device(x, L).cpu().numpy()
    ref = SO.analyze(x, L)
    assert _dev(spec, ref) <= TOL
    back = S.stft_synthesize_device(spec, L, x.shape[1]).cpu().numpy()
    assert _dev(back, SO.synthesize(ref, L, x.shape[1])) <= TOL
    assert np.abs(back - x).max() <= 1e-10 * np.abs(x).max()


def test_batched_equals_single():
    S = _stft()
    import torch

    rng = np.random.default_rng(11)
    X = rng.standard_normal((3, 2, 4, 2500))  # (batch..., C, length)
    spec = S.stft_analyze_device(torch.from_numpy(X).cuda(), 512)
    assert tuple(spec.shape) == (3, 2, SO.frames_for(2500, 256), 257, 4)
    back = S.stft_synthesize_device(spec, 512, 2500)
    for a in range(3):
        for b in range(2):
            one = S.stft_analyze_device(X[a, b], 512)
            assert torch.equal(spec[a, b], one)
            assert torch.equal(back[a, b], S.stft_synthesize_device(one, 512, 2500))


def test_zero_input_gives_zero_tensor_and_zero_round_trip():
    S = _stft()
    spec = S.stft_analyze(_audio(np.zeros((3, 5000))), 256, 128)
    assert np.all(spec.data == 0)
    back = S.stft_synthesize(S.stft_analyze(_audio(np.zeros((2, 10000))), 1024, 512), 1024, 512)
    assert np.all(back.samples == 0)


def test_sinusoid_concentrates_and_matches_direct_dft():
    S = _stft()
    sr, L, bin_index = 16000, 256, 16
    t = np.arange(sr) / sr
    x = np.cos(2 * np.pi * (bin_index * sr / L) * t)
    spec = S.stft_analyze(_audio(x[None, :], sr), L, L // 2)
    energy = np.abs(spec.data[10, :, 0]) ** 2
    assert energy.argmax() == bin_index
    assert energy[bin_index - 1:bin_index + 2].sum() > 0.95 * energy.sum()
    for frame in (3, 10, 25):
        ref = SO.direct_dft_frame(x, frame, L)
        assert np.abs(spec.data[frame, :, 0] - ref).max() <= 1e-10 * np.abs(ref).max()


def test_linearity():
    S = _stft()
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 4000))
    y = rng.standard_normal((2, 4000))
    a, b = 0.7, -1.3
    sx = S.stft_analyze(_audio(x, 8000), 512, 256).data
    sy = S.stft_analyze(_audio(y, 8000), 512, 256).data
    sxy = S.stft_analyze(_audio(a * x + b * y, 8000), 512, 256).data
    assert np.abs(sxy - (a * sx + b * sy)).max() <= 1e-12 * np.abs(sxy).max()


def test_parseval_per_frame():
    S = _stft()
    rng = np.random.default_rng(1)
    x = rng.standard_normal(3000)
    L = 512
    spec = S.stft_analyze(_audio(x[None, :], 8000), L, L // 2)
    k = 5
    full = np.concatenate([spec.data[k, :, 0], spec.data[k, -2:0:-1, 0].conj()])
    seg = np.concatenate([np.zeros(L // 2), x, np.zeros(L)])[k * L // 2:k * L // 2 + L]
    seg = seg * SO.window(L)
    assert (np.abs(full) ** 2).sum() == pytest.approx(L * (seg ** 2).sum(), rel=1e-9)


def test_round_trip_noise():
    S = _stft()
    rng = np.random.default_rng(2)
    x = rng.standard_normal((4, 3 * 16000))
    back = S.stft_synthesize(S.stft_analyze(_audio(x), 1024, 512), 1024, 512)
    assert back.samples.shape == x.shape
    assert np.abs(back.samples - x).max() <= 1e-10 * np.abs(x).max()


def test_length_beyond_extent_rejected():
    S = _stft()
    from paper_1805_06572_b200.errors import ConfigurationError

    spec = S.stft_analyze(_audio(np.ones((1, 1000))), 256, 128)
    with pytest.raises(ConfigurationError):
        S.stft_synthesize(spec, 256, 128, length=spec.frames * 128 + 1)
    full = S.stft_synthesize(spec, 256, 128, length=spec.frames * 128)
    assert full.samples.shape == (1, spec.frames * 128)
