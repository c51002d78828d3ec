"""Separation quality (SDR) and runtime (RTF) — reference ``metrics.py``.

``sdr`` / ``sdr_pairing`` keep the reference's signatures, semantics and
errors (``metrics.py:27-80``): per channel the estimate is projected onto the
span of the reference delayed by 0..``max_shift`` samples (least squares),
SDR = 10 log10(|proj|^2 / max(|est - proj|^2, 1e-30 |proj|^2)) dB, -300 dB
for a zero projection, averaged over channels; a silent reference channel
raises :class:`MetricError`; pairing keeps the assignment with the larger SDR
sum. The projections run on the GPU (K8, ``csrc/ffca_metrics.cu``: normal
equations of the delay basis from one autocorrelation pass, FP64 Cholesky,
explicit residual pass). ``sdr_pairs_device`` / ``sdr_pairing_device``
evaluate whole batches of (estimate, reference) pairs in one launch — the
separation chain's outputs never leave HBM. ``measure_rtf`` is the
reference's host-side timing helper (``metrics.py:83-103``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from .errors import MetricError

DEFAULT_MAX_SHIFT = 31  # metrics.py:10
_MAX_PAIRS = 65535  # one launch (grid.y)


@dataclass
class EvalReport:
    """Per-run evaluation record (reference metrics.py:16-24)."""

    algorithm_label: str
    sdr_per_source: list = field(default_factory=list)
    sdr_mean: float = float("nan")
    rtf: float = float("nan")
    iteration_times: list = field(default_factory=list)


def _samples(x):
    return x.samples if hasattr(x, "samples") else x


def sdr_pairs_device(est, ref, max_shift=DEFAULT_MAX_SHIFT):
    """SDR (dB) of every signal pair ``est[..., :]`` vs ``ref[..., :]``
    (same shape (..., length), float64, CUDA tensors or host arrays), as a
    CUDA float64 tensor of shape ``est.shape[:-1]``, plus the per-pair flag
    tensor (bit 0: silent reference, bit 1: rank-deficient delay basis)."""
    lib = D.require()
    torch = D.torch
    e = D.to_device(est, torch.float64)
    r = D.to_device(ref, torch.float64)
    if tuple(e.shape) != tuple(r.shape):
        raise MetricError(f"shape mismatch: estimate {tuple(e.shape)} vs reference "
                          f"{tuple(r.shape)}")
    if e.dim() < 1 or e.shape[-1] < 1:
        raise MetricError("empty signals")
    if not (0 <= int(max_shift) <= 63):
        raise MetricError(f"max_shift {max_shift} unsupported (0..63)")
    lead = tuple(e.shape[:-1])
    L = int(e.shape[-1])
    if 1 < L < int(max_shift):
        # the reference's delay-basis fill fails for a delay in (L, 2L)
        # (metrics.py:31-32 raises numpy's broadcast ValueError)
        raise MetricError(f"signal length {L} shorter than the delay window {max_shift}")
    e2 = e.reshape(-1, L)
    r2 = r.reshape(-1, L)
    P = int(e2.shape[0])
    out = torch.empty(P, dtype=torch.float64, device=e.device)
    flags = torch.empty(P, dtype=torch.int32, device=e.device)
    for a in range(0, P, _MAX_PAIRS):
        b = min(P, a + _MAX_PAIRS)
        wsz = lib.ffca_sdr_workspace_size(b - a, L, int(max_shift))
        ws = D.workspace(wsz)
        D.check_rc(lib.ffca_sdr(D.ptr(e2[a:b]), D.ptr(r2[a:b]), b - a, L, int(max_shift),
                                D.ptr(out[a:b]), D.ptr(flags[a:b]), D.ptr(ws),
                                D.stream_handle()), "ffca_sdr")
    return out.reshape(lead), flags.reshape(lead)


def _raise_silent(flags, channel_axis_last=True):
    bad = np.argwhere((np.asarray(flags) & 1) != 0)
    if bad.size:
        ch = int(bad[0][-1]) if channel_axis_last else int(bad[0][0])
        raise MetricError(f"reference channel {ch} is silent; SDR undefined")


def sdr(estimate, reference, max_shift=DEFAULT_MAX_SHIFT):
    """Signal-to-distortion ratio in dB, averaged over channels (reference
    metrics.py:44-60). ``estimate`` / ``reference``: AudioBuffer or (C, length)
    / (length,) arrays of the same shape."""
    est = _samples(estimate)
    ref = _samples(reference)
    if not D.is_tensor(est):
        est = np.atleast_2d(np.asarray(est, dtype=np.float64))
    if not D.is_tensor(ref):
        ref = np.atleast_2d(np.asarray(ref, dtype=np.float64))
    if tuple(est.shape) != tuple(ref.shape):
        raise MetricError(f"shape mismatch: estimate {tuple(est.shape)} vs reference "
                          f"{tuple(ref.shape)}")
    vals, flags = sdr_pairs_device(est, ref, max_shift)
    _raise_silent(flags.cpu().numpy())
    return float(vals.cpu().numpy().mean())


def sdr_pairing(estimates, references, max_shift=DEFAULT_MAX_SHIFT):
    """Pairing-optimal SDR for two estimates against two references
    (reference metrics.py:63-80): ``(per_source, permutation)``. All four
    (estimate, reference) combinations run as one batch."""
    ests = [np.atleast_2d(np.asarray(_samples(e), dtype=np.float64)) for e in estimates]
    refs = [np.atleast_2d(np.asarray(_samples(r), dtype=np.float64)) for r in references]
    for a in ests:
        for b in refs:
            if a.shape != b.shape:
                raise MetricError(f"shape mismatch: estimate {a.shape} vs reference {b.shape}")
    E = np.stack([np.stack([a, a]) for a in ests])  # (e, r, C, L)
    R = np.stack([np.stack(refs) for _ in ests])
    vals, flags = sdr_pairs_device(E, R, max_shift)
    _raise_silent(flags.cpu().numpy())
    table = vals.cpu().numpy().mean(axis=-1)
    return _pick(table)


def _pick(table):
    if table[0, 0] + table[1, 1] >= table[1, 0] + table[0, 1]:
        return [float(table[0, 0]), float(table[1, 1])], (0, 1)
    return [float(table[1, 0]), float(table[0, 1])], (1, 0)


def sdr_pairing_device(estimates, references, max_shift=DEFAULT_MAX_SHIFT):
    """Batched pairing: ``estimates`` / ``references`` (..., 2, C, length)
    (CUDA tensors or arrays) -> (per_source (..., 2) numpy, permutations
    list): the four combinations of every batch entry in one launch."""
    torch = D.torch
    e = D.to_device(estimates, torch.float64)
    r = D.to_device(references, torch.float64)
    if tuple(e.shape) != tuple(r.shape) or e.dim() < 3 or e.shape[-3] != 2:
        raise MetricError(f"shape mismatch: estimates {tuple(e.shape)} vs references "
                          f"{tuple(r.shape)} (want (..., 2, C, length))")
    E = e.unsqueeze(-3).expand(*e.shape[:-3], 2, 2, *e.shape[-2:])  # (..., e, r, C, L)
    R = r.unsqueeze(-4).expand(*r.shape[:-3], 2, 2, *r.shape[-2:])
    vals, flags = sdr_pairs_device(E.contiguous(), R.contiguous(), max_shift)
    _raise_silent(flags.cpu().numpy())
    table = vals.cpu().numpy().mean(axis=-1)  # (..., 2, 2)
    flat = table.reshape(-1, 2, 2)
    picks = [_pick(t) for t in flat]
    per = np.asarray([p[0] for p in picks]).reshape(*table.shape[:-2], 2)
    return per, [p[1] for p in picks]


def measure_rtf(run, audio_duration, repeats=3):
    """Real-time factor of a separation closure (reference metrics.py:83-103):
    median of ``repeats`` EM times (``em_seconds`` of the returned object, a
    returned number, or the wall clock around the call) / audio duration."""
    if audio_duration <= 0:
        raise MetricError("audio_duration must be positive")
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        out = run()
        elapsed = time.perf_counter() - t0
        if hasattr(out, "em_seconds"):
            times.append(float(out.em_seconds))
        elif isinstance(out, (int, float)):
            times.append(float(out))
        else:
            times.append(elapsed)
    return float(np.median(times)) / audio_duration, times

