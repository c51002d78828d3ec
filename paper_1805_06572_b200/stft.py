"""STFT analysis / synthesis on the device (reference stft.py:9-107).

Same conventions as the reference: square-root periodic Hann window on both
sides, frame_shift = frame_length / 2, half a frame of leading zero padding,
tensors (frame n, bin f, channel i); exact overlap-add reconstruction. The
transforms run in ``ffca_stft_analyze`` / ``ffca_stft_synthesize``
(``csrc/ffca_stft.cu``): persistent FP64 shared-memory FFT kernels that write
the EM kernels' layout directly. There is no CPU fallback.

``stft_analyze`` / ``stft_synthesize`` keep the reference's host signatures
(numpy in, numpy out). ``stft_analyze_device`` / ``stft_synthesize_device``
take and return CUDA tensors with any number of leading batch axes, so a
separation pipeline (analysis -> EM -> synthesis of both images) stays in HBM.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from .errors import ConfigurationError
from .types import AudioBuffer, SpectrogramTensor

MAX_FRAME_LENGTH = 8192


def sqrt_hann(frame_length):
    """Square root of the periodic Hann window (stft.py:16-19)."""
    t = np.arange(frame_length)
    return np.sqrt(0.5 * (1.0 - np.cos(2.0 * np.pi * t / frame_length)))


def _validate_params(frame_length, frame_shift):
    """stft.py:22-28, plus the device limit on the frame length."""
    if frame_length < 2 or (frame_length & (frame_length - 1)) != 0:
        raise ConfigurationError(f"frame_length must be a power of two, got {frame_length}")
    if frame_shift * 2 != frame_length:
        raise ConfigurationError(
            f"frame_shift must be frame_length/2, got {frame_shift} for length {frame_length}")
    if frame_length > MAX_FRAME_LENGTH:
        raise ConfigurationError(
            f"frame_length {frame_length} exceeds the device limit {MAX_FRAME_LENGTH}")


def num_frames(length, frame_shift):
    """Frames needed so every sample gets full overlap-add weight (stft.py:30-32)."""
    return max((length - 1) // frame_shift + 2, 2)


def stft_analyze_device(x, frame_length=1024):
    """x (..., C, length) float64 (CUDA tensor or array) -> CUDA complex128
    tensor (..., N, frame_length/2 + 1, C)."""
    _validate_params(frame_length, frame_length // 2)
    lib = D.require()
    torch = D.torch
    xd = D.to_device(x, torch.float64)
    if xd.dim() < 2:
        xd = xd.reshape(1, -1)
    *lead, C, length = (int(s) for s in xd.shape)
    if length < 1 or C < 1:
        raise ConfigurationError("audio must have at least one channel and one sample")
    B = int(np.prod(lead)) if lead else 1
    N = num_frames(length, frame_length // 2)
    F = frame_length // 2 + 1
    spec = D.empty((*lead, N, F, C), torch.complex128)
    D.check_rc(lib.ffca_stft_analyze(D.ptr(xd), D.ptr(spec), B, C, length, frame_length,
                                     D.stream_handle()), "ffca_stft_analyze")
    return spec


def stft_synthesize_device(spec, frame_length=1024, length=None):
    """spec (..., N, frame_length/2 + 1, C) complex128 -> CUDA float64 tensor
    (..., C, length); ``length`` defaults to the full extent N * shift."""
    shift = frame_length // 2
    _validate_params(frame_length, shift)
    lib = D.require()
    torch = D.torch
    sd = D.to_device(spec, torch.complex128)
    if sd.dim() < 3:
        raise ConfigurationError("spectrogram data must be (..., frames, bins, channels)")
    *lead, N, F, C = (int(s) for s in sd.shape)
    if F != frame_length // 2 + 1:
        raise ConfigurationError(f"spectrogram has {F} bins, expected {frame_length // 2 + 1}")
    extent = N * shift
    if length is None:
        length = extent
    if length > extent:
        raise ConfigurationError(
            f"requested length {length} exceeds synthesized extent {extent}")
    B = int(np.prod(lead)) if lead else 1
    out = D.empty((*lead, C, length), torch.float64)
    if length > 0:
        D.check_rc(lib.ffca_stft_synthesize(D.ptr(sd), D.ptr(out), B, C, N, frame_length, length,
                                            D.stream_handle()), "ffca_stft_synthesize")
    return out


def stft_analyze(audio, frame_length=1024, frame_shift=512):
    """Reference ``stft_analyze`` (stft.py:35-70): AudioBuffer -> SpectrogramTensor."""
    _validate_params(frame_length, frame_shift)
    spec = stft_analyze_device(audio.samples, frame_length)
    return SpectrogramTensor(data=D.host(spec), sample_rate=audio.sample_rate,
                             frame_length=frame_length, frame_shift=frame_shift,
                             original_length=audio.length)


def stft_synthesize(spec, frame_length=1024, frame_shift=512, length=None):
    """Reference ``stft_synthesize`` (stft.py:73-107): SpectrogramTensor -> AudioBuffer."""
    _validate_params(frame_length, frame_shift)
    data = spec.data
    n_frames, n_bins, _ = data.shape
    if n_bins != frame_length // 2 + 1:
        raise ConfigurationError(
            f"spectrogram has {n_bins} bins, expected {frame_length // 2 + 1}")
    if length is None:
        length = spec.original_length
    if length is None:
        length = n_frames * frame_shift
    out = stft_synthesize_device(data, frame_length, length)
    return AudioBuffer(sample_rate=spec.sample_rate, samples=D.host(out))
