"""CUDA kernel backend: the reference's 11-function kernel-module contract.

Drop-in for ``fastfca._kernels_numba`` / ``fastfca._kernels_numpy``
(reference _kernels_numpy.py:3-13,19-193; _kernels_numba.py:69-391): same
function names, argument order, layouts, return tuples and op counts. Arrays
come in and go out as host numpy (complex128 / float64) like the reference;
torch CUDA tensors are accepted too and then results stay on the device.
Each call is one or two kernel launches in libfastfca_b200.so; numerical
failures surface like the reference's (ZeroDivisionError-free: the engines
check finiteness; FCA singular points raise ``numpy.linalg.LinAlgError``
exactly where numba's ``np.linalg.inv`` would).
"""

from __future__ import annotations

import numpy as np

from . import _device as D


def _c(x):
    return D.to_device(x, D.torch.complex128)


def _r(x):
    return D.to_device(x, D.torch.float64)


def _out(t, like):
    return t if D.is_tensor(like) else D.host(t)


class SingularPointError(np.linalg.LinAlgError):
    """numba's ``np.linalg.inv`` LinAlgError, carrying the first singular (n, f)."""

    def __init__(self, frame, bin):
        super().__init__("Singular matrix")
        self.frame = frame
        self.bin = bin


def _raise_singular(st, F):
    s = st.read()
    if s.code:
        idx = int(s.index)
        raise SingularPointError(idx // F, idx % F)


def _dims(y):
    N, F, I = (int(s) for s in y.shape)
    return N, F, I


def fca_e_step(y, v, S):
    """-> (mu (2,N,F,I), Phi (2,N,F,I,I), inversions, products)."""
    lib = D.require()
    yd, vd, Sd = _c(y), _r(v), _c(S)
    N, F, I = _dims(yd)
    mu = D.empty((2, N, F, I), D.torch.complex128)
    Phi = D.empty((2, N, F, I, I), D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_fca_e_step(D.ptr(yd), D.ptr(vd), D.ptr(Sd), D.ptr(mu), D.ptr(Phi), N, F, I,
                                   st.handle, D.stream_handle()), "ffca_fca_e_step")
    _raise_singular(st, F)
    return _out(mu, y), _out(Phi, y), N * F, 3 * N * F


def fca_v_update(Phi, S_prev):
    """tr(S_prev^{-1} Phi)/I per (j, n, f), unfloored -> v (2,N,F)."""
    lib = D.require()
    Pd, Sd = _c(Phi), _c(S_prev)
    _, N, F, I, _ = (int(s) for s in Pd.shape)
    v = D.empty((2, N, F), D.torch.float64)
    st = D.StageStatus()
    D.check_rc(lib.ffca_fca_v_update(D.ptr(Pd), D.ptr(Sd), D.ptr(v), N, F, I, st.handle,
                                     D.stream_handle()), "ffca_fca_v_update")
    st.raise_if_error(N, F)
    return _out(v, Phi)


def fca_S_update(Phi, v):
    """(1/N) sum_n Phi_j / v_j -> S (2,F,I,I)."""
    lib = D.require()
    Pd, vd = _c(Phi), _r(v)
    _, N, F, I, _ = (int(s) for s in Pd.shape)
    S = D.empty((2, F, I, I), D.torch.complex128)
    D.check_rc(lib.ffca_S_update(D.ptr(Pd), D.ptr(vd), D.ptr(S), N, F, I, D.stream_handle()),
               "ffca_S_update")
    return _out(S, Phi)


def fca_log_likelihood(y, v, S):
    lib = D.require()
    yd, vd, Sd = _c(y), _r(v), _c(S)
    N, F, I = _dims(yd)
    out = D.empty((1,), D.torch.float64)
    st = D.StageStatus()
    D.check_rc(lib.ffca_fca_log_likelihood(D.ptr(yd), D.ptr(vd), D.ptr(Sd), D.ptr(out), N, F, I,
                                           st.handle, D.stream_handle()),
               "ffca_fca_log_likelihood")
    _raise_singular(st, F)
    return float(D.host(out)[0])


def fast_transform(y, P):
    """yt = P^H y per (n, f)."""
    lib = D.require()
    yd, Pd = _c(y), _c(P)
    N, F, I = _dims(yd)
    yt = D.empty((N, F, I), D.torch.complex128)
    D.check_rc(lib.ffca_fast_transform(D.ptr(yd), D.ptr(Pd), D.ptr(yt), N, F, I,
                                       D.stream_handle()), "ffca_fast_transform")
    return _out(yt, y)


def fast_e_step(yt, v, lam):
    """-> (mu (2,N,F,I), Phi (2,N,F,I,I), 0, 0) in the diagonal basis."""
    lib = D.require()
    yd, vd, ld = _c(yt), _r(v), _r(lam)
    N, F, I = _dims(yd)
    mu = D.empty((2, N, F, I), D.torch.complex128)
    Phi = D.empty((2, N, F, I, I), D.torch.complex128)
    D.check_rc(lib.ffca_fast_e_step(D.ptr(yd), D.ptr(vd), D.ptr(ld), D.ptr(mu), D.ptr(Phi), N, F,
                                    I, D.stream_handle()), "ffca_fast_e_step")
    return _out(mu, yt), _out(Phi, yt), 0, 0


def fast_v_update(Phi_t, lam):
    lib = D.require()
    Pd, ld = _c(Phi_t), _r(lam)
    _, N, F, I, _ = (int(s) for s in Pd.shape)
    v = D.empty((2, N, F), D.torch.float64)
    D.check_rc(lib.ffca_fast_v_update(D.ptr(Pd), D.ptr(ld), D.ptr(v), N, F, I, D.stream_handle()),
               "ffca_fast_v_update")
    return _out(v, Phi_t)


def fast_S_update(Phi_t, v):
    return fca_S_update(Phi_t, v)


def fast_log_likelihood(yt, v, lam, logdet2):
    lib = D.require()
    yd, vd, ld, dd = _c(yt), _r(v), _r(lam), _r(logdet2)
    N, F, I = _dims(yd)
    out = D.empty((1,), D.torch.float64)
    D.check_rc(lib.ffca_fast_log_likelihood(D.ptr(yd), D.ptr(vd), D.ptr(ld), D.ptr(dd), D.ptr(out),
                                            N, F, I, D.stream_handle()),
               "ffca_fast_log_likelihood")
    return float(D.host(out)[0])


def fca_iteration(y, v, S, Sinv, floor):
    """-> (mu, v_new, S_raw, inversions, products)."""
    lib = D.require()
    yd, vd, Sd, Sid, fd = _c(y), _r(v), _c(S), _c(Sinv), _r(floor)
    N, F, I = _dims(yd)
    mu = D.empty((2, N, F, I), D.torch.complex128)
    vn = D.empty((2, N, F), D.torch.float64)
    Sr = D.empty((2, F, I, I), D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_fca_iteration(D.ptr(yd), D.ptr(vd), D.ptr(Sd), D.ptr(Sid), D.ptr(fd),
                                      D.ptr(mu), D.ptr(vn), D.ptr(Sr), N, F, I, st.handle,
                                      D.stream_handle()), "ffca_fca_iteration")
    _raise_singular(st, F)
    return _out(mu, y), _out(vn, y), _out(Sr, y), N * F, 3 * N * F


def fast_iteration(y, P, v, lam, floor):
    """-> (mu_t, v_new, S_raw, 0, 0)."""
    lib = D.require()
    yd, Pd, vd, ld, fd = _c(y), _c(P), _r(v), _r(lam), _r(floor)
    N, F, I = _dims(yd)
    mu = D.empty((2, N, F, I), D.torch.complex128)
    vn = D.empty((2, N, F), D.torch.float64)
    Sr = D.empty((2, F, I, I), D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_fast_iteration(D.ptr(yd), D.ptr(Pd), D.ptr(vd), D.ptr(ld), D.ptr(fd),
                                       D.ptr(mu), D.ptr(vn), D.ptr(Sr), N, F, I, st.handle,
                                       D.stream_handle()), "ffca_fast_iteration")
    st.read()  # degenerate powers surface as non-finite values, as in the numpy backend
    return _out(mu, y), _out(vn, y), _out(Sr, y), 0, 0


def warmup():
    """Touch every kernel once (load the module, JIT-free: the library is AOT)."""
    gen = np.random.default_rng(0)
    y = gen.standard_normal((2, 2, 2)) + 1j * gen.standard_normal((2, 2, 2))
    v = np.abs(gen.standard_normal((2, 2, 2))) + 0.5
    S = np.stack([np.eye(2, dtype=np.complex128)] * 2)[:, None].repeat(2, axis=1)
    P = np.stack([np.eye(2, dtype=np.complex128)] * 2)
    lam = np.ones((2, 2))
    mu, Phi, _, _ = fca_e_step(y, v, S)
    fca_v_update(Phi, S)
    fca_S_update(Phi, v)
    fca_log_likelihood(y, v, S)
    yt = fast_transform(y, P)
    _, Phi_t, _, _ = fast_e_step(yt, v, lam)
    fast_v_update(Phi_t, lam)
    fast_S_update(Phi_t, v)
    fast_log_likelihood(yt, v, lam, np.zeros(2))
    floor = np.full(2, 1e-12)
    fca_iteration(y, v, S, S, floor)
    fast_iteration(y, P, v, lam, floor)
