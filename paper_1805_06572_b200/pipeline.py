"""Device-resident separation chain: STFT analysis -> seeded init -> EM ->
STFT synthesis of both source images, the compute of the reference CLI's
``separate`` command (cli.py:93-98 ``_build_init`` with ``init="random"``,
cli.py:152-171 ``_separate_once``, cli.py:186-202 ``cmd_separate``) without
the file I/O, config and report plumbing. Everything between the input
samples and the output samples stays in HBM; a batch of mixtures
(..., C, length) runs as one batched EM.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from .conventional import fca_run
from .errors import ConfigurationError, PipelineError
from .fast import fastfca_run
from .initializers import init_from_masks, init_from_masks_batch, init_random, init_random_batch
from .stft import _validate_params, stft_analyze_device, stft_synthesize_device
from .types import AudioBuffer

ENGINES = {"fastfca": ("FastFCA", fastfca_run), "fca": ("FCA", fca_run)}


def _check_finite(t, stage):
    if not bool(D.torch.isfinite(t).all()):
        raise PipelineError(stage)


def separate_device(samples, iterations=20, frame_length=1024, algorithm="fastfca", seed=0,
                    seeds=None, compute_likelihood=False, dtype="c128", init="random"):
    """samples (C, length) or (M, C, length) float64 (CUDA tensor or array).
    ``init``: "random" (seeded ``init_random``) or "masks" (``init_from_masks``,
    the reference CLI's two choices, cli.py:93-98).

    Returns ``(result, images_time)``: the engine's :class:`SeparationResult`
    (device tensors) and the separated source images in the time domain,
    a CUDA float64 tensor (2, C, length) or (M, 2, C, length).
    """
    if algorithm not in ENGINES:
        raise ConfigurationError(f"unknown algorithm {algorithm!r}")
    _validate_params(frame_length, frame_length // 2)
    D.require()
    x = D.to_device(samples, D.torch.float64)
    batched = x.dim() == 3
    if x.dim() not in (2, 3):
        raise ConfigurationError("samples must be (C, length) or (M, C, length)")
    length = int(x.shape[-1])
    spec = stft_analyze_device(x, frame_length)  # (..., N, F, C)
    _check_finite(spec, "stft")
    if init not in ("random", "masks"):
        raise ConfigurationError(f"unknown init {init!r}; expected 'random' or 'masks'")
    if init == "masks":
        model = init_from_masks_batch(spec) if batched else init_from_masks(spec)
    elif batched:
        M = int(spec.shape[0])
        model = init_random_batch(spec, list(seeds) if seeds is not None
                                  else [seed + m for m in range(M)], dtype=dtype)
    else:
        model = init_random(spec, seed, dtype=dtype)
    _, run = ENGINES[algorithm]
    result = run(spec, model, iterations, compute_likelihood=compute_likelihood, dtype=dtype,
                 device_output=True)
    images = result.images  # (..., 2, N, F, C)
    _check_finite(images, f"separation ({ENGINES[algorithm][0]})")
    if images.dtype != D.torch.complex128:
        images = images.to(D.torch.complex128)
    out = stft_synthesize_device(images, frame_length, length)  # (..., 2, C, length)
    _check_finite(out, f"synthesis ({ENGINES[algorithm][0]})")
    return result, out


def _to_host(result):
    """Device tensors of a SeparationResult -> numpy, in place."""
    def h(x):
        return D.host(x) if D.is_tensor(x) else x

    result.images = h(result.images)
    m = result.model
    m.v, m.S, m.v_floor = h(m.v), h(m.S), h(m.v_floor)
    for rec in result.history:
        for k in list(rec):
            rec[k] = h(rec[k])
    return result


def separate(audio, iterations=20, frame_length=1024, algorithm="fastfca", seed=0,
             compute_likelihood=True):
    """Host-facing form: AudioBuffer in, ``(result, [AudioBuffer, AudioBuffer])``
    out (one per source image), like the reference ``_separate_once``."""
    result, out = separate_device(audio.samples, iterations, frame_length, algorithm, seed,
                                  compute_likelihood=compute_likelihood)
    host = D.host(out)
    _to_host(result)
    return result, [AudioBuffer(audio.sample_rate, np.ascontiguousarray(host[j]))
                    for j in range(2)]
