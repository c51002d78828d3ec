"""Golden vectors for the mask-clustering initialiser from the UNMODIFIED
reference ``fastfca.initializers.init_from_masks``. Run once in the build
container:

    python tests/golden/make_golden_masks.py

Writes ``tests/golden/masks.npz``: inputs y and the reference (v, S, floor)
for random inputs, a degenerate shared-direction geometry, the N < 2 I
fallback, and an alternating-activity reverberant mixture built with the
reference's own simulator and STFT (its test_initializers.py scenario).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from fastfca.initializers import init_from_masks  # noqa: E402
from fastfca.simulate import RoomSpec, mix, speech_shaped_noise, synth_rir  # noqa: E402
from fastfca.stft import stft_analyze  # noqa: E402
from fastfca.types import AudioBuffer  # noqa: E402


def cases():
    rng = np.random.default_rng(2024)
    yield "rand_20x6x2", rng.standard_normal((20, 6, 2)) + 1j * rng.standard_normal((20, 6, 2))
    yield "rand_30x5x3", rng.standard_normal((30, 5, 3)) + 1j * rng.standard_normal((30, 5, 3))
    yield "rand_64x9x8", rng.standard_normal((64, 9, 8)) + 1j * rng.standard_normal((64, 9, 8))
    direction = rng.standard_normal(3) + 1j * rng.standard_normal(3)
    gains = rng.standard_normal((40, 6)) + 1j * rng.standard_normal((40, 6))
    yield "shared_direction", gains[:, :, None] * direction[None, None, :]
    yield "fallback", rng.standard_normal((3, 4, 2)) + 1j * rng.standard_normal((3, 4, 2))
    fs, dur = 16000, 2.0
    n = int(dur * fs)
    gate = (np.arange(n) // int(0.5 * fs)) % 2 == 0
    a = speech_shaped_noise(dur, fs, seed=70).samples[0] * gate
    b = speech_shaped_noise(dur, fs, seed=71).samples[0] * (~gate)
    truth = mix((AudioBuffer(fs, a[None]), AudioBuffer(fs, b[None])),
                synth_rir(RoomSpec(rt60=0.13, channels=2, seed=72)))
    yield "alternating", stft_analyze(truth.mixture, 512, 256).data


def main():
    out = {}
    names = []
    for name, y in cases():
        m = init_from_masks(y)
        out[f"{name}_y"] = y
        out[f"{name}_v"] = m.v
        out[f"{name}_S"] = m.S
        out[f"{name}_floor"] = m.v_floor
        names.append(name)
    out["cases"] = np.array(names)
    np.savez_compressed(HERE / "masks.npz", **out)
    print("wrote", HERE / "masks.npz", [(k, v.shape) for k, v in out.items() if k.endswith("_y")])


if __name__ == "__main__":
    main()
