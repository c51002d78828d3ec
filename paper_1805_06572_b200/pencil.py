"""Hermitian-definite pencil decomposition on the GPU (reference pencil.py).

:func:`gevd_hpd` returns real generalized eigenvalues (descending) and a
basis ``P`` with ``P^H Psi P = I`` and ``P^H Phi P = diag(lam)``, columns
phase-pinned so that their largest-magnitude entry is real positive — the
reference's conventions (pencil.py:85-135). The solver is the batched
device kernel behind ``ffca_gevd_hpd`` (one thread per pencil: Jacobi
eigensolves of Psi and of the whitened Phi).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device as D
from .errors import NonHermitianError, SingularMatrixError

HERMITIAN_RTOL = 1e-10
DEFINITENESS_FLOOR = 1e-12


@dataclass
class PencilDecomposition:
    """Generalized eigenvalues (..., D) descending; eigenvectors (..., D, D) in columns."""

    eigenvalues: np.ndarray
    eigenvectors: np.ndarray


def _square(A, name):
    shape = tuple(A.shape)
    if len(shape) < 2 or shape[-1] != shape[-2]:
        raise NonHermitianError(f"{name} must be square, got shape {shape}")
    if shape[-1] > 8:
        raise NonHermitianError(f"{name}: order {shape[-1]} > 8 unsupported on the device path")
    return shape


def gevd_hpd(Phi, Psi):
    """Solve ``Phi p = lam Psi p`` per batch entry (reference pencil.py:85-135)."""
    lib = D.require()
    sp = _square(Phi, "Phi")
    sq = _square(Psi, "Psi")
    if sp != sq:
        raise NonHermitianError(f"Phi and Psi must share a shape, got {sp} and {sq}")
    d = sp[-1]
    batch = int(np.prod(sp[:-2])) if len(sp) > 2 else 1
    A = D.to_device(Phi, D.torch.complex128).reshape(batch, d, d)
    B = D.to_device(Psi, D.torch.complex128).reshape(batch, d, d)
    lam = D.empty((batch, d), D.torch.float64)
    P = D.empty((batch, d, d), D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_gevd_hpd(D.ptr(A), D.ptr(B), D.ptr(lam), D.ptr(P), batch, d, 1, st.handle,
                                 D.stream_handle()), "ffca_gevd_hpd")
    st.raise_if_error()
    lam = lam.reshape(sp[:-1])
    P = P.reshape(sp)
    if D.is_tensor(Phi):
        return PencilDecomposition(lam, P)
    return PencilDecomposition(D.host(lam), D.host(P))


def hermitian_eig(A):
    """Eigenvalues (descending) and unitary eigenvectors of Hermitian ``A``
    (reference pencil.py:54-73), via the pencil solver with ``Psi = I``."""
    shape = _square(A, "A")
    eye = np.broadcast_to(np.eye(shape[-1], dtype=np.complex128), shape)
    if D.is_tensor(A):
        eye = D.torch.as_tensor(np.ascontiguousarray(eye), device=A.device)
    dec = gevd_hpd(A, np.ascontiguousarray(eye) if not D.is_tensor(A) else eye)
    return dec.eigenvalues, dec.eigenvectors


def solve_hermitian_system(Psi, B, rtol=1e-10):
    """Solve ``Psi X = B`` per batch entry and verify the residual
    (reference pencil.py:138-157) — LU with partial pivoting in the
    ``ffca_solve`` kernel (the reference's np.linalg.solve / zgesv).

    ``Psi`` (..., D, D) nonsingular square; ``B`` (D,) with a single ``Psi``
    or (..., D, K). A singular system or a relative residual above ``rtol``
    (Frobenius norms over the whole batch, as the reference) raises
    :class:`SingularMatrixError`.
    """
    lib = D.require()
    torch = D.torch
    A = D.to_device(Psi, torch.complex128)
    b = D.to_device(B, torch.complex128)
    if A.dim() < 2 or A.shape[-1] != A.shape[-2]:
        raise SingularMatrixError(f"singular system: Psi must be square, got {tuple(A.shape)}")
    d = int(A.shape[-1])
    if d > 8:
        raise SingularMatrixError(f"singular system: order {d} > 8 unsupported on the device path")
    vec = b.dim() == 1
    rhs = b[:, None] if vec else b
    if vec and A.dim() != 2:
        raise SingularMatrixError("singular system: a vector right-hand side needs one Psi")
    if tuple(rhs.shape[:-1]) != tuple(A.shape[:-1]):
        raise SingularMatrixError(
            f"singular system: shapes {tuple(A.shape)} and {tuple(b.shape)} do not match")
    batch = int(np.prod(A.shape[:-2])) if A.dim() > 2 else 1
    K = int(rhs.shape[-1])
    Ad = A.reshape(batch, d, d).contiguous()
    Bd = rhs.reshape(batch, d, K).contiguous()
    X = D.empty((batch, d, K), torch.complex128)
    norms = D.empty((batch, 2), torch.float64)
    st = D.StageStatus()
    D.check_rc(lib.ffca_solve(D.ptr(Ad), D.ptr(Bd), D.ptr(X), D.ptr(norms), batch, d, K,
                              st.handle, D.stream_handle()), "ffca_solve")
    if st.read().code:
        raise SingularMatrixError("singular system: Singular matrix")
    tot = norms.sum(dim=0).cpu().numpy()
    norm_b = float(np.sqrt(tot[1]))
    resid = float(np.sqrt(tot[0]))
    if not bool(torch.isfinite(X).all()) or not np.isfinite(resid) or \
            resid > rtol * max(norm_b, 1e-300):
        raise SingularMatrixError(
            f"system too ill-conditioned: relative residual {resid / max(norm_b, 1e-300):.3e}")
    X = X.reshape(rhs.shape)
    X = X[..., 0] if vec else X
    return X if D.is_tensor(Psi) else D.host(X)


def logdet2(P):
    """2 log|det P| per bin (reference fast.py:151-153)."""
    lib = D.require()
    shape = tuple(P.shape)
    d = shape[-1]
    batch = int(np.prod(shape[:-2])) if len(shape) > 2 else 1
    Pd = D.to_device(P, D.torch.complex128).reshape(batch, d, d)
    out = D.empty((batch,), D.torch.float64)
    D.check_rc(lib.ffca_logdet2(D.ptr(Pd), D.ptr(out), batch, d, D.stream_handle()),
               "ffca_logdet2")
    out = out.reshape(shape[:-2])
    return out if D.is_tensor(P) else D.host(out)


_ = ctypes  # ctypes handles are created in _device
