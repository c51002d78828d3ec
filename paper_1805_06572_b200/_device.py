"""Device plumbing: torch supplies device memory and the stream; the math is
in libfastfca_b200.so. Every public entry point routes through here, and
there is no CPU fallback: a missing library or GPU raises immediately.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import (BackendUnavailableError, DefinitenessError, NonHermitianError,
                     SingularMatrixError, SingularMixtureError)

_DEGENERATE_MSG = "mixture covariance is singular (source powers collapsed to zero)"

try:  # torch is plumbing only (allocator, streams, events)
    import torch
except Exception as exc:  # pragma: no cover
    torch = None
    _TORCH_ERR = exc


def require():
    """Return the loaded library; raise if torch, CUDA or the library is missing."""
    if torch is None:
        raise BackendUnavailableError(f"torch unavailable: {_TORCH_ERR}")
    if not torch.cuda.is_available():
        raise BackendUnavailableError("no CUDA device: the fastfca_b200 path runs on the GPU only")
    return _lib.load()


def device():
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def is_tensor(x):
    return torch is not None and isinstance(x, torch.Tensor)


def to_device(x, dtype, non_blocking=True):
    """numpy / torch (any device) -> contiguous CUDA tensor of ``dtype``."""
    if is_tensor(x):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.to(device(), non_blocking=non_blocking and t.is_pinned())
    elif t.device != device():
        # the kernels run on the current device and stream: a tensor on another
        # GPU would be dereferenced there (illegal address) -> move it
        t = t.to(device())
    return t.contiguous()


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def empty(shape, dtype):
    return torch.empty(tuple(int(s) for s in shape), dtype=dtype, device=device())


def workspace(nbytes):
    # 256-B aligned (the caching allocator hands out 512-B aligned blocks)
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device())


def check_rc(rc, what):
    if rc == _lib.FFCA_OK:
        return
    if rc == _lib.FFCA_ERR_INVALID:
        raise ValueError(f"{what}: invalid arguments")
    raise RuntimeError(f"{what}: CUDA failure (code {rc})")


def raise_for_status(st, N=None, F=None):
    """Map a decoded device status onto the reference exception types."""
    code = st.code
    if code == _lib.FFCA_OK:
        return
    if code == _lib.FFCA_ERR_SINGULAR_MATRIX:
        raise SingularMatrixError(_DEGENERATE_MSG)
    if code == _lib.FFCA_ERR_SINGULAR_MIXTURE:
        idx = int(st.index)
        if N is not None and F is not None:
            f = idx % F
            n = (idx // F) % N
        else:
            n, f = idx, 0
        raise SingularMixtureError(int(n), int(f))
    if code == _lib.FFCA_ERR_DEFINITENESS:
        worst = float(st.value)
        raise DefinitenessError(f"Psi is not positive definite: min eigenvalue {worst:.6e}", worst)
    if code == _lib.FFCA_ERR_NON_HERMITIAN:
        raise NonHermitianError("Phi/Psi is not Hermitian beyond tolerance")
    if code == _lib.FFCA_ERR_SINGULAR_BASIS:
        raise SingularMatrixError("basis matrix is singular")
    if code == _lib.FFCA_ERR_NOT_PD:
        raise np.linalg.LinAlgError("Matrix is not positive definite")
    if code == _lib.FFCA_ERR_NO_CONVERGENCE:  # numpy eigh's message (LAPACK heevd info > 0)
        raise np.linalg.LinAlgError("Eigenvalues did not converge")
    raise RuntimeError(f"fastfca_b200: unknown status code {code}")


def decode_status(word):
    """Decode a 16-byte status word already in host memory (uint8 array / tensor)."""
    lib = _lib.load()
    raw = np.ascontiguousarray(np.asarray(word, dtype=np.uint8).reshape(16))
    st = _lib.Status()
    check_rc(lib.ffca_status_decode(raw.ctypes.data_as(ctypes.c_void_p), ctypes.byref(st)),
             "ffca_status_decode")
    return st


class StageStatus:
    """A device status word for stage-level calls."""

    def __init__(self):
        self.lib = require()
        self.buf = empty((16,), torch.uint8)
        check_rc(self.lib.ffca_status_reset(ptr(self.buf), stream_handle()), "status_reset")

    @property
    def handle(self):
        return ptr(self.buf)

    def read(self):
        st = _lib.Status()
        check_rc(self.lib.ffca_status_read(ptr(self.buf), stream_handle(), ctypes.byref(st)),
                 "status_read")
        return st

    def raise_if_error(self, N=None, F=None):
        raise_for_status(self.read(), N, F)


PINNED_MIN_BYTES = 1 << 20


def host(t, sync=True):
    """CUDA tensor -> numpy. Large results land in pinned (page-locked) host
    memory from torch's caching host allocator — a pageable destination would
    first-touch-fault every page and halve the PCIe rate."""
    t = t.detach()
    if not t.is_cuda:
        return t.numpy()
    nbytes = t.numel() * t.element_size()
    if nbytes < PINNED_MIN_BYTES:
        return t.cpu().numpy()
    dst = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    dst.copy_(t, non_blocking=True)
    if sync:
        torch.cuda.current_stream().synchronize()
    return dst.numpy()
