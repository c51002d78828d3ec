"""CPU port of the reference EM loops for timing — TEST / BASELINE INFRASTRUCTURE.

Only bench.py (its ``cpu_baseline`` leg and ``--impl reference``) and tests
use this. It restates the reference drivers ``fastfca_run`` (fast.py:156-260)
and ``fca_run`` (conventional.py:104-164) with the per-(n, f) loops in C
(oracle/fca_oracle.c, restating _kernels_numba.py, OpenMP over independent
bins / mixtures on all host cores) and the per-bin small linear algebra in
numpy/LAPACK exactly as the reference does it (oracle/fastfca_oracle.py).
Timing mirrors the reference's ``em_seconds`` boundary: only the iterations
(no initial pencil, likelihood or image extraction) — which favours the CPU
relative to the GPU step, which includes all of them.
"""

from __future__ import annotations

import ctypes
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from . import fastfca_oracle as O

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle_fca.so"
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        _lib = ctypes.CDLL(str(LIB))
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        _lib.ffo_fast_iteration.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, ctypes.c_int, vp,
                                            vp, vp]
        _lib.ffo_fast_iteration.restype = None
        _lib.ffo_fca_iteration.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, ctypes.c_int, vp,
                                           vp, vp]
        _lib.ffo_fca_iteration.restype = ctypes.c_int64
        _lib.ffo_set_threads.argtypes = [ctypes.c_int]
        _lib.ffo_max_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def fast_iteration_c(Y, P, V, lam, floor, want_mu=False):
    """Batched C restatement of _fast_iteration. Y (M,N,F,I), P (M*F,I,I)."""
    M, N, F, I = Y.shape
    mu = np.empty((M, 2, N, F, I), dtype=np.complex128) if want_mu else None
    vn = np.empty((M, 2, N, F))
    Sr = np.empty((M, 2, F, I, I), dtype=np.complex128)
    lib().ffo_fast_iteration(_p(Y), _p(P), _p(V), _p(lam), _p(floor), M, N, F, I, _p(mu),
                             _p(vn), _p(Sr))
    return mu, vn, Sr


def fca_iteration_c(Y, V, S, Sinv, floor, want_mu=False):
    M, N, F, I = Y.shape
    mu = np.empty((M, 2, N, F, I), dtype=np.complex128) if want_mu else None
    vn = np.empty((M, 2, N, F))
    Sr = np.empty((M, 2, F, I, I), dtype=np.complex128)
    bad = lib().ffo_fca_iteration(_p(Y), _p(V), _p(S), _p(Sinv), _p(floor), M, N, F, I, _p(mu),
                                  _p(vn), _p(Sr))
    if bad >= 0:
        raise O.OracleSingularError("singular mixture covariance", bad)
    return mu, vn, Sr


def fastfca_em(Y, V0, S0, floor, L, want_images=False):
    """FastFCA EM over a batch; returns (em_seconds, v, S_t, P, mu_t)."""
    M, N, F, I = Y.shape
    Y = np.ascontiguousarray(Y)
    fl = np.ascontiguousarray(floor.reshape(M * F))
    lam, P = O.gevd_hpd(S0[:, 0].reshape(M * F, I, I), S0[:, 1].reshape(M * F, I, I))
    P = np.ascontiguousarray(P)
    lam = np.ascontiguousarray(lam)
    v = np.ascontiguousarray(V0, dtype=np.float64)
    em = 0.0
    mu = S_t = None
    for l in range(L):
        t0 = time.perf_counter()
        mu, v, S_raw = fast_iteration_c(Y, P, v, lam, fl, want_mu=want_images and l == L - 1)
        O._require_finite(v, S_raw)
        gram = np.conj(np.swapaxes(P, -1, -2)) @ P  # (M*F, I, I)
        S_t = O.regularize_transformed(S_raw.transpose(1, 0, 2, 3, 4).reshape(2, M * F, I, I),
                                       gram[None])
        lam, Q = O.gevd_hpd(S_t[0], S_t[1])
        P = np.ascontiguousarray(P @ Q)
        lam = np.ascontiguousarray(lam)
        em += time.perf_counter() - t0
    return em, v, S_t, P, mu


def fca_em(Y, V0, S0, floor, L, want_images=False):
    M, N, F, I = Y.shape
    Y = np.ascontiguousarray(Y)
    fl = np.ascontiguousarray(floor.reshape(M * F))
    v = np.ascontiguousarray(V0, dtype=np.float64)
    S = np.ascontiguousarray(S0)
    em = 0.0
    mu = None
    for l in range(L):
        t0 = time.perf_counter()
        Sinv = np.ascontiguousarray(O.cholesky_inverse(S))
        mu, v, S_raw = fca_iteration_c(Y, v, S, Sinv, fl, want_mu=want_images and l == L - 1)
        S = np.ascontiguousarray(O.regularize_covariances(S_raw))
        em += time.perf_counter() - t0
    return em, v, S, mu


def _sample_inputs(cfg, count):
    """Seeded inputs for a bounded sample: mixtures (batched configs) or a
    contiguous bin range (single-mixture configs; bins are independent)."""
    from paper_1805_06572_b200.synth import config_mixture, init_seed

    if cfg.M > 1:
        ms = list(range(min(count, cfg.M)))

        def one(m):
            y = config_mixture(cfg, m)
            v, S, fl = O.init_random(y, init_seed(cfg, m))
            return y, v, S, fl

        with ThreadPoolExecutor(8) as ex:
            parts = list(ex.map(one, ms))
        Y = np.stack([p[0] for p in parts])
        return (Y, np.stack([p[1] for p in parts]), np.stack([p[2] for p in parts]),
                np.stack([p[3] for p in parts]), f"{len(ms)} of {cfg.M} mixtures x {cfg.F} bins x "
                f"{cfg.N} frames x {cfg.L} iterations")
    y = config_mixture(cfg, 0)
    v, S, fl = O.init_random(y, init_seed(cfg, 0))
    nb = min(count, cfg.F)
    sl = slice(0, nb)
    return (np.ascontiguousarray(y[None, :, sl]), np.ascontiguousarray(v[None, :, :, sl]),
            np.ascontiguousarray(S[None, :, sl]), np.ascontiguousarray(fl[None, sl]),
            f"{nb} of {cfg.F} bins x {cfg.N} frames x {cfg.L} iterations")


_CACHE = {}


def measure(cfg, engine, sample, threads):
    """TF-bin*it/s of the CPU port on a bounded sample (reference em_seconds
    boundary). Returns (value, sample description, kind, cores)."""
    lib().ffo_set_threads(int(threads))
    if not sample:
        if cfg.M > 1:
            sample = max(2 * threads, 8) if engine == "fast" else max(threads // 2, 2)
        else:
            sample = cfg.F if engine == "fast" else max(4 * threads, 16)
    key = (cfg.index, int(sample))
    if key not in _CACHE:
        _CACHE[key] = _sample_inputs(cfg, int(sample))
    Y, V, S, FL, desc = _CACHE[key]
    M, N, F, I = Y.shape
    run = fastfca_em if engine == "fast" else fca_em
    em = run(Y, V, S, FL, cfg.L)[0]
    return M * F * N * cfg.L / em, desc, "port", int(threads)
