"""Device-resident EM runs through the C ABI (ffca_fastfca_run / ffca_fca_run).

``run_device`` is the throughput entry point: inputs are CUDA tensors with a
leading mixture axis, outputs stay on the device. The reference-shaped
``fastfca_run`` / ``fca_run`` wrappers (fast.py, conventional.py) sit on top.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .errors import ConfigurationError

DTYPES = {"c128": _lib.FFCA_C128, "c64": _lib.FFCA_C64}


def torch_types(dtype):
    torch = D.torch
    if dtype == "c128":
        return torch.complex128, torch.float64
    if dtype == "c64":
        return torch.complex64, torch.float32
    raise ConfigurationError(f"unknown dtype {dtype!r}; expected 'c128' or 'c64'")


@dataclass
class DeviceRun:
    """Outputs of one device run (all CUDA tensors, leading mixture axis)."""

    algorithm: str
    images: object  # (M,2,N,F,I) complex or None
    v: object  # (M,2,N,F) real
    S: object  # (M,2,F,I,I) complex128
    loglik: object  # (M,L+1) float64 or None
    S_hist: object = None  # (L,M,2,F,I,I)
    v_hist: object = None  # (L,M,2,N,F)
    iteration_ms: list = field(default_factory=list)
    workspace: object = None
    kernel_ms: list = field(default_factory=list)
    floor: object = None


def run_device(algorithm, y, v0, S0, v_floor, iterations, *, likelihood=True, history=False,
               images=True, dtype="c128", timing=True, check=True, out=None, chunk_frames=0,
               kernel_timing=False):
    """Run ``iterations`` EM passes of FastFCA (``algorithm='fast'``) or
    conventional FCA (``'fca'``) entirely on the current CUDA stream.

    y (M,N,F,I) complex, v0 (M,2,N,F) real, S0 (M,2,F,I,I) complex128,
    v_floor (M,F) float64 — CUDA tensors (moved if not). ``v0`` is not
    modified. With ``check`` the stream is synchronised and numerical
    failures are raised as the reference's exceptions.
    """
    lib = D.require()
    torch = D.torch
    ctype, rtype = torch_types(dtype)
    y = D.to_device(y, ctype)
    if y.dim() != 4:
        raise ConfigurationError("y must be (M, N, F, I)")
    M, N, F, I = (int(s) for s in y.shape)
    if not (1 <= I <= 8):
        raise ConfigurationError(f"channel count I={I} unsupported (1..8)")
    if N < 1 or F < 1:
        raise ConfigurationError("need at least one frame and one bin")
    L = int(iterations)
    if L < 0:
        raise ConfigurationError("iterations must be >= 0")
    v = D.to_device(v0, rtype)
    if D.is_tensor(v0) and v.data_ptr() == v0.data_ptr():
        v = v.clone()  # the run updates v in place; never clobber the caller's init
    S0 = D.to_device(S0, torch.complex128)
    fl = D.to_device(v_floor, torch.float64)
    if tuple(v.shape) != (M, 2, N, F) or tuple(S0.shape) != (M, 2, F, I, I) or \
            tuple(fl.shape) != (M, F):
        raise ConfigurationError(
            f"shape mismatch: y {tuple(y.shape)}, v {tuple(v.shape)}, S {tuple(S0.shape)}, "
            f"floor {tuple(fl.shape)}")
    flags = 0
    if likelihood:
        flags |= _lib.FLAG_LIKELIHOOD
    if history:
        flags |= _lib.FLAG_HISTORY
    if images:
        flags |= _lib.FLAG_IMAGES
    fast = algorithm == "fast"
    wsz = (lib.ffca_fastfca_workspace_size if fast else lib.ffca_fca_workspace_size)(
        M, N, F, I, L, flags, int(chunk_frames))
    ws = D.workspace(wsz)
    res = out or {}
    img = res.get("images") if images else None
    if images and img is None:
        img = D.empty((M, 2, N, F, I), ctype)
    S_out = res.get("S") if res.get("S") is not None else D.empty((M, 2, F, I, I), torch.complex128)
    ll = D.empty((M, L + 1), torch.float64) if likelihood else None
    S_hist = D.empty((L, M, 2, F, I, I), torch.complex128) if (history and L) else None
    v_hist = D.empty((L, M, 2, N, F), rtype) if (history and L) else None
    evs = None
    ev_arr = None
    if timing:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
        for e in evs:
            e.record()  # materialise the CUDA event handles
        ev_arr = (ctypes.c_void_p * (L + 1))(*[e.cuda_event for e in evs])
    kevs = None
    kev_arr = None
    if kernel_timing and L:
        kevs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * L)]
        for e in kevs:
            e.record()
        kev_arr = (ctypes.c_void_p * (2 * L))(*[e.cuda_event for e in kevs])
    args = _lib.RunArgs(
        M=M, N=N, F=F, I=I, dtype=DTYPES[dtype], iterations=L, flags=flags,
        y=D.ptr(y).value, v=D.ptr(v).value, S0=D.ptr(S0).value, v_floor=D.ptr(fl).value,
        images=D.ptr(img).value, S_out=D.ptr(S_out).value, loglik=D.ptr(ll).value,
        S_hist=D.ptr(S_hist).value, v_hist=D.ptr(v_hist).value,
        workspace=D.ptr(ws).value, workspace_bytes=wsz,
        iter_events=ctypes.cast(ev_arr, ctypes.c_void_p).value if ev_arr is not None else None,
        chunk_frames=int(chunk_frames),
        kernel_events=ctypes.cast(kev_arr, ctypes.c_void_p).value if kev_arr is not None
        else None)
    fn = lib.ffca_fastfca_run if fast else lib.ffca_fca_run
    D.check_rc(fn(ctypes.byref(args), D.stream_handle()), fn.__name__)
    run = DeviceRun("FastFCA" if fast else "FCA", img, v, S_out, ll, S_hist, v_hist, [], ws)
    if check:
        st = _lib.Status()
        D.check_rc(lib.ffca_run_status(D.ptr(ws), D.stream_handle(), ctypes.byref(st)),
                   "ffca_run_status")
        D.raise_for_status(st, N, F)
    run._events = evs
    run._kevents = kevs
    if check:
        _collect_timings(run)
    run._kevents = kevs
    return run


def _collect_timings(run):
    L = len(run._events) - 1 if run._events else 0
    if run._events and not run.iteration_ms:
        run.iteration_ms = [run._events[i].elapsed_time(run._events[i + 1]) for i in range(L)]
    if run._kevents:
        k = run._kevents
        run.kernel_ms = [k[2 * i].elapsed_time(k[2 * i + 1]) for i in range(len(k) // 2)]


def plan_chunks(G, N):
    """The frame chunking the drivers pick for G bins x N frames (per-bin
    reduction order: equal chunking => bitwise-equal per-bin results)."""
    lib = _lib.load()
    cf = ctypes.c_int64()
    nc = ctypes.c_int()
    D.check_rc(lib.ffca_plan_chunks(int(G), int(N), ctypes.byref(cf), ctypes.byref(nc)),
               "ffca_plan_chunks")
    return int(cf.value), int(nc.value)


def status_of(run, N=None, F=None):
    """Synchronise and raise for a run launched with ``check=False``."""
    lib = D.require()
    st = _lib.Status()
    D.check_rc(lib.ffca_run_status(D.ptr(run.workspace), D.stream_handle(), ctypes.byref(st)),
               "ffca_run_status")
    D.raise_for_status(st, N, F)
    _collect_timings(run)


def as_batch(y, init):
    """Normalise reference-shaped inputs to batched device tensors.

    Returns (y (M,N,F,I), v (M,2,N,F), S (M,2,F,I,I), floor (M,F), batched).
    """
    data = y.data if hasattr(y, "data") and not D.is_tensor(y) and not isinstance(y, np.ndarray) \
        else y
    nd = data.dim() if D.is_tensor(data) else np.ndim(data)
    if nd == 3:
        def add(x):
            return x[None] if D.is_tensor(x) else np.asarray(x)[None]
        return add(data), add(init.v), add(init.S), add(init.v_floor), False
    if nd == 4:
        return data, init.v, init.S, init.v_floor, True
    raise ConfigurationError("y must be (N, F, I) or (M, N, F, I)")
