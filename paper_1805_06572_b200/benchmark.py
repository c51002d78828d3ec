"""Separation benchmark sweep — the compute of the reference CLI's
``benchmark`` command (cli.py:269-371) on the device.

For every condition (the reference sweeps reverberation times; here the
caller supplies each condition's time-domain mixtures and true source
images — the room simulator, WAV I/O and chart output are out of scope) the
trials of the condition are separated as ONE batch per engine (STFT analysis
-> initial model -> EM -> synthesis, ``pipeline.separate_device``), scored
with the pairing-optimal SDR of all trials in one launch
(``metrics.sdr_pairing_device``) and timed on the EM's own clock
(``em_seconds``). Rows follow the reference's CSV layouts
(``RESULTS_CSV_HEADER`` / ``TIMING_CSV_HEADER``, cli.py:29-50, values
formatted with ``%.10g`` as cli.py:70-71):

* results: per trial and engine ``[schema, condition, trial, algorithm,
  sdr_source1, sdr_source2, sdr_mean]`` plus one ``"mean"`` row per engine;
* timing: per condition ``[schema, condition, rtf_fca, rtf_fastfca,
  rtf_fca / rtf_fastfca, em_seconds_fca, em_seconds_fastfca]``.

A batched EM has one ``em_seconds`` for all T trials, so a trial's EM time is
that batch time / T and RTF = batch EM time / (T x duration) (the reference
takes the median over sequential per-trial runs, cli.py:261-266).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

from . import _device as D
from .errors import ConfigurationError
from .metrics import DEFAULT_MAX_SHIFT, sdr_pairing_device
from .pipeline import separate_device

SCHEMA_VERSION = 1  # cli.py:29
RESULTS_CSV_HEADER = ["schema_version", "rt60_ms", "trial", "algorithm", "sdr_source1_db",
                      "sdr_source2_db", "sdr_mean_db"]
TIMING_CSV_HEADER = ["schema_version", "rt60_ms", "rtf_fca", "rtf_fastfca", "speedup",
                     "em_seconds_fca", "em_seconds_fastfca"]
LABELS = {"fca": "FCA", "fastfca": "FastFCA"}


def _fmt(x):
    return f"{x:.10g}"


@dataclass
class Condition:
    """One sweep condition: ``mixtures`` (T, C, length) and the true source
    images ``images`` (T, 2, C, length), float64 (host arrays or CUDA
    tensors), at ``sample_rate``; ``label`` goes in the rt60_ms column."""

    label: float
    mixtures: object
    images: object
    sample_rate: int


def benchmark_sweep(conditions, iterations=20, frame_length=1024, init="random", seed=0,
                    engines=("fca", "fastfca"), max_shift=DEFAULT_MAX_SHIFT, dtype="c128"):
    """Run the sweep; returns ``(results_rows, timing_rows, summary)`` with
    ``summary[label] = {engine: {"sdr_mean", "rtf", "em_seconds"}}``."""
    for e in engines:
        if e not in LABELS:
            raise ConfigurationError(f"unknown engine {e!r}")
    results, timing, summary = [], [], {}
    for cond in conditions:
        mix = D.to_device(cond.mixtures, D.torch.float64)
        truth = D.to_device(cond.images, D.torch.float64)
        if mix.dim() != 3 or truth.dim() != 4 or tuple(truth.shape) != (
                mix.shape[0], 2, mix.shape[1], mix.shape[2]):
            raise ConfigurationError("condition wants mixtures (T, C, length) and images "
                                     "(T, 2, C, length)")
        T = int(mix.shape[0])
        duration = float(mix.shape[-1]) / float(cond.sample_rate)
        per = {}
        for e in engines:
            result, out = separate_device(mix, iterations, frame_length, e, seed=seed,
                                          seeds=[seed + t for t in range(T)], init=init,
                                          dtype=dtype)
            values, _ = sdr_pairing_device(out, truth, max_shift)  # (T, 2)
            em = float(result.em_seconds)
            per[e] = {"sdr": values, "em_seconds": em, "rtf": em / (T * duration)}
            for t in range(T):
                results.append([SCHEMA_VERSION, _fmt(cond.label), t, LABELS[e],
                                _fmt(values[t, 0]), _fmt(values[t, 1]),
                                _fmt(float(np.mean(values[t])))])
        for e in engines:
            v = per[e]["sdr"]
            results.append([SCHEMA_VERSION, _fmt(cond.label), "mean", LABELS[e],
                            _fmt(float(np.mean(v[:, 0]))), _fmt(float(np.mean(v[:, 1]))),
                            _fmt(float(np.mean(v)))])
        summary[cond.label] = {e: {"sdr_mean": float(np.mean(per[e]["sdr"])),
                                   "rtf": per[e]["rtf"], "em_seconds": per[e]["em_seconds"]}
                               for e in engines}
        if "fca" in per and "fastfca" in per:
            rf, rs = per["fca"]["rtf"], per["fastfca"]["rtf"]
            timing.append([SCHEMA_VERSION, _fmt(cond.label), _fmt(rf), _fmt(rs),
                           _fmt(rf / rs if rs > 0 else float("inf")),
                           _fmt(per["fca"]["em_seconds"]), _fmt(per["fastfca"]["em_seconds"])])
    return results, timing, summary


def write_csv(path, header, rows):
    """The reference's CSV writer convention (cli.py:353-362)."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)
