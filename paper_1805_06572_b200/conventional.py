"""Conventional (frame-wise) FCA engine on the GPU (reference conventional.py).

The baseline the paper accelerates: every (n, f) point inverts its I x I
mixture covariance and forms I x I products. ``fca_run`` keeps the
reference signature and semantics (images from the final E-step, model
from the last M-step, likelihood trace incl. the initial model, history of
regularised (v, S)); the loop runs in ``ffca_fca_run`` on the device.
"""

from __future__ import annotations

import numpy as np

from . import _backend
from . import _device as D
from ._engine import as_batch, run_device, run_host_pipelined
from ._kernels_cuda import SingularPointError
from .errors import SingularMixtureError
from .fast import _finish, _finish_host, _pipelined_ok
from .modelops import regularize_covariances
from .types import OpCounts, PosteriorMoments, SpatialModel


def _data(y):
    return y if (D.is_tensor(y) or isinstance(y, np.ndarray)) else y.data


def log_likelihood(y, model):
    """Sum over (n, f) of -I log(pi) - log det R - y^H R^-1 y (conventional.py:41-56)."""
    try:
        value = _backend.kernels().fca_log_likelihood(_data(y), model.v, model.S)
    except SingularPointError as exc:
        raise SingularMixtureError(exc.frame, exc.bin) from None
    if not np.isfinite(value):
        raise SingularMixtureError(0, 0)
    return value


def e_step(y, model, counts=None):
    """Posterior means and second moments (conventional.py:59-80)."""
    try:
        mu, Phi, inv, prod = _backend.kernels().fca_e_step(_data(y), model.v, model.S)
    except SingularPointError as exc:
        raise SingularMixtureError(exc.frame, exc.bin) from None
    if counts is not None:
        counts.add(inversions=inv, products=prod)
    return PosteriorMoments(mu=mu, Phi=Phi)


def m_step(posterior, model_prev):
    """Power and covariance re-estimation, floored and regularised
    (conventional.py:83-95), on the device."""
    torch = D.torch
    kern = _backend.kernels()
    on_dev = D.is_tensor(posterior.Phi)
    Phi = D.to_device(posterior.Phi, torch.complex128)
    S_prev = D.to_device(model_prev.S, torch.complex128)
    fl = D.to_device(model_prev.v_floor, torch.float64)
    v = kern.fca_v_update(Phi, S_prev)
    v = torch.maximum(v, fl[None, None, :])
    S = regularize_covariances(kern.fca_S_update(Phi, v))
    if on_dev:
        return SpatialModel(v=v, S=S, v_floor=model_prev.v_floor)
    return SpatialModel(v=D.host(v), S=D.host(S), v_floor=model_prev.v_floor)


def _cholesky_inverse(S):
    """S^{-1} = L^{-H} L^{-1} per bin (conventional.py:98-101)."""
    lib = D.require()
    shape = tuple(S.shape)
    d = shape[-1]
    batch = int(np.prod(shape[:-2]))
    Sd = D.to_device(S, D.torch.complex128).reshape(batch, d, d)
    out = D.empty((batch, d, d), D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_cholesky_inverse(D.ptr(Sd), D.ptr(out), batch, d, st.handle,
                                         D.stream_handle()), "ffca_cholesky_inverse")
    st.raise_if_error()
    out = out.reshape(shape)
    return out if D.is_tensor(S) else D.host(out)


def fca_run(y, init, iterations, record_history=False, compute_likelihood=True, dtype="c128",
            device_output=None, chunk_frames=0):
    """Conventional EM for ``iterations`` passes + MMSE images (conventional.py:104-164)."""
    yb, vb, Sb, fb, batched = as_batch(_data(y), init)
    if device_output is None:
        device_output = D.is_tensor(yb)
    L = int(iterations)
    if _pipelined_ok(yb, batched, device_output, record_history):
        return _finish_host(run_host_pipelined("fca", yb, vb, Sb, fb, L,
                                               likelihood=compute_likelihood, dtype=dtype,
                                               chunk_frames=chunk_frames), "FCA", L)
    run = run_device("fca", yb, vb, Sb, fb, L, likelihood=compute_likelihood,
                     history=record_history, images=True, dtype=dtype,
                     chunk_frames=chunk_frames)
    run.floor = D.to_device(fb, D.torch.float64)
    M, N, F = int(run.v.shape[0]), int(run.v.shape[2]), int(run.v.shape[3])
    mult = M if batched else 1
    counts = OpCounts()
    counts.add(inversions=L * N * F * mult, products=3 * L * N * F * mult)
    if L == 0:  # images from e_step under the initial model (conventional.py:152-153)
        counts.add(inversions=N * F * mult, products=3 * N * F * mult)
    return _finish(run, "FCA", L, batched, device_output, counts, record_history)
