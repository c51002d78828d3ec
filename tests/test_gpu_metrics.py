"""GPU SDR (K8, csrc/ffca_metrics.cu) against golden values of the unmodified
reference fastfca.metrics and the pinned oracle, plus the reference's own
metric tests (pkg/tests/test_metrics.py) run on the device path, and the
benchmark sweep's rows. Tolerance: 1e-9 dB relative (the device solves the
delay-basis normal equations; the reference lstsq's SVD)."""

import numpy as np
import pytest

from oracle import metrics_oracle as MO
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_1805_06572_b200 as P

    return P


def _close(a, b, tol=1e-9):
    return abs(a - b) <= tol * max(1.0, abs(b))


def test_sdr_matches_reference_golden():
    P = _pkg()
    g = load_golden("sdr")
    for name in [str(n) for n in g["names"]]:
        val = P.sdr(g[f"{name}_est"], g[f"{name}_ref"], int(g[f"{name}_max_shift"]))
        assert _close(val, float(g[f"{name}_sdr"])), (name, val, float(g[f"{name}_sdr"]))


def test_sdr_pairing_matches_reference_golden():
    P = _pkg()
    g = load_golden("sdr")
    vals, perm = P.sdr_pairing((g["pair_e1"], g["pair_e2"]), (g["pair_r1"], g["pair_r2"]))
    assert tuple(perm) == tuple(int(x) for x in g["pair_perm"])
    assert all(_close(a, float(b)) for a, b in zip(vals, g["pair_values"]))


def test_batched_pairs_match_the_oracle():
    """sdr_pairs_device over a batch (many pairs, several 4096-sample blocks)."""
    P = _pkg()
    rng = np.random.default_rng(9)
    ref = rng.standard_normal((6, 2, 9001))
    est = 0.8 * ref + rng.standard_normal(ref.shape) * rng.uniform(0.01, 2.0, (6, 2, 1))
    vals, flags = P.sdr_pairs_device(est, ref)
    vals = vals.cpu().numpy()
    assert not flags.cpu().numpy().any()
    for b in range(6):
        for c in range(2):
            assert _close(vals[b, c], MO.channel_sdr(est[b, c], ref[b, c]))


# ---- the reference's metric tests (pkg/tests/test_metrics.py) on the device ----
def _delayed_basis(ref, taps):
    length = ref.shape[0]
    basis = np.zeros((length, taps))
    for d in range(taps):
        basis[d:, d] = ref[: length - d]
    return basis


def test_perfect_estimate_caps_high():
    P = _pkg()
    x = np.random.default_rng(0).standard_normal((1, 8000))
    assert P.sdr(P.AudioBuffer(8000, x), P.AudioBuffer(8000, x)) >= 100.0


def test_equal_power_orthogonal_noise_gives_zero_db():
    P = _pkg()
    rng = np.random.default_rng(1)
    ref = rng.standard_normal(16000)
    noise = rng.standard_normal(16000)
    basis = _delayed_basis(ref, 32)
    h, *_ = np.linalg.lstsq(basis, noise, rcond=None)
    noise = noise - basis @ h
    noise *= np.linalg.norm(ref) / np.linalg.norm(noise)
    value = P.sdr(P.AudioBuffer(16000, (ref + noise)[None]), P.AudioBuffer(16000, ref[None]))
    assert value == pytest.approx(0.0, abs=0.1)


def test_scale_invariance():
    P = _pkg()
    rng = np.random.default_rng(2)
    ref = rng.standard_normal((2, 4000))
    est = ref + 0.3 * rng.standard_normal((2, 4000))
    a = P.sdr(P.AudioBuffer(8000, est), P.AudioBuffer(8000, ref))
    b = P.sdr(P.AudioBuffer(8000, 7.3 * est), P.AudioBuffer(8000, ref))
    assert b == pytest.approx(a, abs=1e-9)


def test_delay_within_shift_window_is_transparent():
    P = _pkg()
    ref = np.random.default_rng(3).standard_normal(8000)
    est = np.roll(ref, 5)
    est[:5] = 0.0
    assert P.sdr(P.AudioBuffer(8000, est[None]), P.AudioBuffer(8000, ref[None])) >= 100.0


def test_silent_reference_rejected():
    P = _pkg()
    with pytest.raises(P.MetricError):
        P.sdr(P.AudioBuffer(8000, np.ones((1, 100))), P.AudioBuffer(8000, np.zeros((1, 100))))


def test_shape_mismatch_rejected():
    P = _pkg()
    with pytest.raises(P.MetricError):
        P.sdr(P.AudioBuffer(8000, np.ones((1, 100))), P.AudioBuffer(8000, np.ones((1, 200))))


def test_pairing_picks_better_assignment():
    P = _pkg()
    rng = np.random.default_rng(4)
    r1 = rng.standard_normal((1, 4000))
    r2 = rng.standard_normal((1, 4000))
    refs = (P.AudioBuffer(8000, r1), P.AudioBuffer(8000, r2))
    ests = (P.AudioBuffer(8000, r2 + 0.1 * rng.standard_normal((1, 4000))),
            P.AudioBuffer(8000, r1 + 0.1 * rng.standard_normal((1, 4000))))
    values, perm = P.sdr_pairing(ests, refs)
    assert perm == (1, 0)
    assert min(values) > 10.0


def test_benchmark_sweep_rows():
    """benchmark_sweep on two synthetic conditions (sources + random mixing
    filters): row layout of the reference CSVs, SDRs equal to the metric on
    the separated outputs, both engines, RTF from em_seconds."""
    import torch

    from paper_1805_06572_b200.benchmark import (RESULTS_CSV_HEADER, TIMING_CSV_HEADER,
                                                 Condition, benchmark_sweep)

    P = _pkg()
    rng = np.random.default_rng(7)
    conds = []
    for label in (150.0, 300.0):
        T, C, n = 2, 2, 8000
        src = rng.standard_normal((T, 2, n)) * np.exp(rng.standard_normal((T, 2, 1)))
        imgs = np.empty((T, 2, C, n))
        for t in range(T):
            for j in range(2):
                for c in range(C):
                    h = rng.standard_normal(4) * np.exp(-np.arange(4))
                    imgs[t, j, c] = np.convolve(src[t, j], h)[:n]
        conds.append(Condition(label, imgs.sum(axis=1), imgs, 16000))
    rows, timing, summary = benchmark_sweep(conds, iterations=3, frame_length=256)
    assert len(rows) == 2 * (2 * 2 + 2) and all(len(r) == len(RESULTS_CSV_HEADER) for r in rows)
    assert len(timing) == 2 and all(len(r) == len(TIMING_CSV_HEADER) for r in timing)
    # each trial's SDRs are the metric of that trial's separated images
    _, out = P.separate_device(conds[0].mixtures, 3, 256, "fastfca", seed=0, seeds=[0, 1])
    for t in range(2):
        vals, _ = P.sdr_pairing([o for o in out[t].cpu().numpy()],
                                [r for r in conds[0].images[t]])
        row = [r for r in rows if r[0] == 1 and r[2] == t and r[3] == "FastFCA"
               and float(r[1]) == 150.0][0]
        assert np.allclose([float(row[4]), float(row[5])], vals, rtol=1e-8)
    assert summary[150.0]["fastfca"]["rtf"] > 0 and summary[300.0]["fca"]["em_seconds"] > 0
    del torch
