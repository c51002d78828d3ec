"""CPU oracle for the SDR metric — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may use this module; the product path
(``paper_1805_06572_b200.metrics``) runs on the GPU and never imports it.

A numpy restatement of the reference ``fastfca.metrics`` SDR
(``metrics.py:27-80``): per channel the estimate is regressed on the
reference delayed by 0..max_shift samples (``np.linalg.lstsq`` on the
L x (max_shift+1) delay basis, ``:28-34``), target = |proj|^2, noise =
|est - proj|^2, SDR = 10 log10(target / max(noise, 1e-30 target)) and -300
for a zero target (``:35-39``); channels averaged; pairing keeps the larger
SDR sum (``:63-80``). Pinned by ``tests/test_metrics_oracle.py`` against
golden values from the unmodified reference (``tests/golden/make_golden_sdr.py``).
"""

from __future__ import annotations

import numpy as np

CAP = 1e-30


def channel_sdr(est, ref, max_shift=31):
    L = est.shape[0]
    taps = max_shift + 1
    B = np.zeros((L, taps))
    for d in range(taps):
        B[d:, d] = ref[: L - d]
    h = np.linalg.lstsq(B, est, rcond=None)[0]
    proj = B @ h
    target = float(np.sum(proj ** 2))
    noise = float(np.sum((est - proj) ** 2))
    if target <= 0.0:
        return -300.0
    return 10.0 * np.log10(target / max(noise, CAP * target))


def sdr(est, ref, max_shift=31):
    est = np.atleast_2d(est)
    ref = np.atleast_2d(ref)
    return float(np.mean([channel_sdr(est[c], ref[c], max_shift) for c in range(ref.shape[0])]))


def sdr_pairing(ests, refs, max_shift=31):
    t = np.array([[sdr(e, r, max_shift) for r in refs] for e in ests])
    if t[0, 0] + t[1, 1] >= t[1, 0] + t[0, 1]:
        return [float(t[0, 0]), float(t[1, 1])], (0, 1)
    return [float(t[1, 0]), float(t[0, 1])], (1, 0)
