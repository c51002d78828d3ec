"""CPU oracle for the STFT front / back end — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (and ``smoke()`` / ``bench.py`` if they ever need it) may use
this module; the product path (``paper_1805_06572_b200.stft``) runs on the
GPU and never imports it.

A numpy restatement of the reference ``fastfca.stft`` (``stft.py:9-107``):
square-root periodic Hann window (``:16-19``), frame_shift = frame_length/2,
half a frame of leading zeros and enough trailing zeros that the frame grid
covers every sample (``:30-32,56-59``), ``rfft`` per windowed frame
(``:61-64``); synthesis zeroes the imaginary parts of DC and Nyquist
(``:91-92``), ``irfft`` times the window (``:93``), overlap-adds frames in
frame order (``:95-99``) and trims the half-frame padding and the tail
(``:101-106``). Written frame-by-frame over a (channels, frames) loop rather
than the reference's fancy-indexed gather; the arithmetic is the same.

Pinned by ``tests/test_stft_oracle.py`` against golden vectors from the
unmodified reference (``tests/golden/make_golden_stft.py``) and against a
direct DFT matrix (the reference test's own oracle idea, test_stft.py:9-22).
"""

from __future__ import annotations

import numpy as np


def window(frame_length):
    """stft.py:16-19."""
    t = np.arange(frame_length, dtype=np.float64)
    return np.sqrt(0.5 * (1.0 - np.cos(2.0 * np.pi * t / frame_length)))


def frames_for(length, shift):
    """stft.py:30-32."""
    return max((length - 1) // shift + 2, 2)


def analyze(x, frame_length):
    """x (C, length) -> (N, F, C) complex128 (stft.py:35-70)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    C, length = x.shape
    S = frame_length // 2
    N = frames_for(length, S)
    w = window(frame_length)
    F = frame_length // 2 + 1
    out = np.empty((N, F, C), dtype=np.complex128)
    for k in range(N):
        start = (k - 1) * S  # padded index k*S == signal index (k-1)*S
        lo, hi = max(start, 0), min(start + frame_length, length)
        seg = np.zeros((C, frame_length))
        if hi > lo:
            seg[:, lo - start:hi - start] = x[:, lo:hi]
        out[k] = np.fft.rfft(seg * w, axis=-1).T
    return out


def synthesize(spec, frame_length, length=None):
    """(N, F, C) -> (C, length) float64 (stft.py:73-107)."""
    spec = np.asarray(spec, dtype=np.complex128)
    N, F, C = spec.shape
    S = frame_length // 2
    w = window(frame_length)
    acc = np.zeros((C, (N + 1) * S))
    for k in range(N):
        half = spec[k].T.copy()  # (C, F)
        half[:, 0] = half[:, 0].real
        half[:, -1] = half[:, -1].real
        fr = np.fft.irfft(half, n=frame_length, axis=-1) * w
        acc[:, k * S:k * S + frame_length] += fr
    out = acc[:, S:]
    if length is not None:
        out = out[:, :length]
    return out


def direct_dft_frame(x, k, frame_length):
    """Frame k of channel signal x by an explicit DFT matrix (test_stft.py:9-22)."""
    S = frame_length // 2
    padded = np.concatenate([np.zeros(S), np.asarray(x, dtype=np.float64),
                             np.zeros(frame_length)])
    seg = padded[k * S:k * S + frame_length] * window(frame_length)
    kk = np.arange(frame_length // 2 + 1)
    n = np.arange(frame_length)
    return np.exp(-2j * np.pi * np.outer(kk, n) / frame_length) @ seg
