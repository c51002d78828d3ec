"""Golden SDR values from the UNMODIFIED reference ``fastfca.metrics``
(``/root/reference/pkg/src``). Run once in the build container:

    python tests/golden/make_golden_sdr.py

Writes ``tests/golden/sdr.npz``: seeded (estimate, reference) signals — a
noisy filtered copy at several SNRs, a delayed copy, a scaled copy, a
multi-channel case, a short signal (40 samples, 32 taps), a different
max_shift, a long signal over several device blocks, and a two-source pairing case — with the
reference's ``sdr`` / ``sdr_pairing`` outputs.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from fastfca.metrics import sdr, sdr_pairing  # noqa: E402
from fastfca.types import AudioBuffer  # noqa: E402


def main():
    out = {}
    rng = np.random.default_rng(2024)
    cases = []
    for snr_db in (-10.0, 0.0, 10.0, 30.0):
        ref = rng.standard_normal((1, 6000))
        filt = np.convolve(ref[0], rng.standard_normal(8) * 0.5)[:6000]
        noise = rng.standard_normal(6000)
        noise *= np.linalg.norm(filt) / np.linalg.norm(noise) * 10 ** (-snr_db / 20)
        cases.append((f"snr{int(snr_db)}", (filt + noise)[None], ref, 31))
    ref = rng.standard_normal((1, 5000))
    est = np.roll(ref, 7)
    est[:, :7] = 0.0
    cases.append(("delay7", est + 0.01 * rng.standard_normal(est.shape), ref, 31))
    ref = rng.standard_normal((3, 9000))
    cases.append(("multich", 2.5 * ref + 0.4 * rng.standard_normal(ref.shape), ref, 31))
    ref = rng.standard_normal((2, 40))
    cases.append(("short", ref[:, ::-1] + 0.1 * rng.standard_normal(ref.shape), ref.copy(), 31))
    ref = rng.standard_normal((1, 12345))
    cases.append(("shift7", ref + 0.3 * rng.standard_normal(ref.shape), ref, 7))
    ref = rng.standard_normal((1, 20000))  # several device blocks (4096 samples)
    cases.append(("long", np.convolve(ref[0], [0.7, 0.2, -0.1])[:20000][None]
                  + 0.05 * rng.standard_normal((1, 20000)), ref, 31))
    names = []
    for name, est, ref, ms in cases:
        names.append(name)
        out[f"{name}_est"] = est
        out[f"{name}_ref"] = ref
        out[f"{name}_max_shift"] = ms
        out[f"{name}_sdr"] = sdr(AudioBuffer(16000, est), AudioBuffer(16000, ref), max_shift=ms)
    # pairing: estimates swapped relative to the references
    r1, r2 = rng.standard_normal((2, 8000)), rng.standard_normal((2, 8000))
    e1 = r2 + 0.2 * rng.standard_normal(r2.shape)
    e2 = r1 + 0.5 * rng.standard_normal(r1.shape)
    vals, perm = sdr_pairing((AudioBuffer(8000, e1), AudioBuffer(8000, e2)),
                             (AudioBuffer(8000, r1), AudioBuffer(8000, r2)))
    out.update(pair_e1=e1, pair_e2=e2, pair_r1=r1, pair_r2=r2, pair_values=np.asarray(vals),
               pair_perm=np.asarray(perm))
    out["names"] = np.asarray(names)
    np.savez_compressed(HERE / "sdr.npz", **out)
    print("wrote", HERE / "sdr.npz", names)


if __name__ == "__main__":
    main()
