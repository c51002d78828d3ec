"""Golden vectors for the STFT front / back end from the UNMODIFIED reference
``fastfca.stft`` (``/root/reference/pkg/src``). Run once in the build
container:

    python tests/golden/make_golden_stft.py

Writes ``tests/golden/stft.npz``: for each case the input signal, the
reference ``stft_analyze`` output, the reference ``stft_synthesize`` of that
spectrum, and the synthesis of a seeded random (non-Hermitian-consistent)
spectrum with complex DC / Nyquist entries.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from fastfca.stft import stft_analyze, stft_synthesize  # noqa: E402
from fastfca.types import AudioBuffer, SpectrogramTensor  # noqa: E402

# (name, channels, length, frame_length, synth length or None, seed)
CASES = [
    ("l2", 1, 7, 2, None, 1),
    ("short", 2, 1, 64, None, 2),
    ("l256", 3, 3000, 256, None, 3),
    ("l512_trim", 2, 4001, 512, 3000, 4),
    ("l1024", 4, 5000, 1024, None, 5),
    ("l4096", 1, 9000, 4096, None, 6),
]


def main():
    out = {}
    for name, C, length, L, trim, seed in CASES:
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((C, length))
        spec = stft_analyze(AudioBuffer(16000, x), L, L // 2)
        back = stft_synthesize(spec, L, L // 2, length=trim)
        N, F, _ = spec.data.shape
        rnd = rng.standard_normal((N, F, C)) + 1j * rng.standard_normal((N, F, C))
        rback = stft_synthesize(SpectrogramTensor(rnd, 16000, L, L // 2, None), L, L // 2)
        out[f"{name}_x"] = x
        out[f"{name}_L"] = np.int64(L)
        out[f"{name}_trim"] = np.int64(-1 if trim is None else trim)
        out[f"{name}_spec"] = spec.data
        out[f"{name}_back"] = back.samples
        out[f"{name}_rnd"] = rnd
        out[f"{name}_rback"] = rback.samples
    out["cases"] = np.array([c[0] for c in CASES])
    np.savez_compressed(HERE / "stft.npz", **out)
    print("wrote", HERE / "stft.npz")


if __name__ == "__main__":
    main()
