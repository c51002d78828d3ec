"""Model helpers (reference modelops.py:1-39), computed on the device."""

from __future__ import annotations

import numpy as np

from . import _device as D

V_FLOOR_FACTOR = 1e-10
COV_EPS_FACTOR = 1e-9


def power_floor(y):
    """``V_FLOOR_FACTOR`` x mean_n(||y(n,f)||^2)/I per bin (modelops.py:12-21)."""
    lib = D.require()
    yd = D.to_device(y, D.torch.complex128)
    N, F, I = (int(s) for s in yd.shape[-3:])
    M = int(np.prod(yd.shape[:-3])) if yd.dim() > 3 else 1
    v = D.empty((M, 2, N, F), D.torch.float64)
    floor = D.empty((M, F), D.torch.float64)
    D.check_rc(lib.ffca_init_powers(D.ptr(yd), D.ptr(v), D.ptr(floor), M, N, F, I, 0,
                                    D.stream_handle()), "ffca_init_powers")
    floor = floor.reshape(tuple(yd.shape[:-3]) + (F,))
    return floor if D.is_tensor(y) else D.host(floor)


def hermitize(S):
    """(S + S^H)/2 (modelops.py:24-26)."""
    if D.is_tensor(S):
        return 0.5 * (S + S.conj().transpose(-1, -2))
    Sd = D.to_device(S, D.torch.complex128)
    return D.host(0.5 * (Sd + Sd.conj().transpose(-1, -2)))


def regularize_covariances(S):
    """Hermitize plus ``COV_EPS_FACTOR`` tr/I ridge (modelops.py:29-39)."""
    lib = D.require()
    shape = tuple(S.shape)
    d = shape[-1]
    batch = int(np.prod(shape[:-2]))
    Sd = D.to_device(S, D.torch.complex128).reshape(batch, d, d)
    out = D.empty((batch, d, d), D.torch.complex128)
    D.check_rc(lib.ffca_regularize_covariances(D.ptr(Sd), D.ptr(out), batch, d,
                                               D.stream_handle()), "ffca_regularize_covariances")
    out = out.reshape(shape)
    return out if D.is_tensor(S) else D.host(out)
