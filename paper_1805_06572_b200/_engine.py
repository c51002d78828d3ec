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
               kernel_timing=False, graph=False, bin_parts=0, persist=None):
    """Run ``iterations`` EM passes of FastFCA (``algorithm='fast'``) or
    conventional FCA (``'fca'``) entirely on the current CUDA stream.

    y (M,N,F,I) complex, v0 (M,2,N,F) real, S0 (M,2,F,I,I) complex128,
    v_floor (M,F) float64 — CUDA tensors (moved if not). ``v0`` is not
    modified. With ``check`` the stream is synchronised and numerical
    failures are raised as the reference's exceptions. ``graph`` replays a
    cached CUDA graph of the whole run when the arguments (buffers, sizes,
    flags) repeat — for repeated runs on preallocated ``out`` buffers; it is
    ignored when ``timing`` / ``kernel_timing`` events are requested.
    ``bin_parts`` (FastFCA): bin windows of the split-phase schedule (0 =
    the driver's plan, 1 = none); results do not depend on it.
    ``persist`` (FastFCA): the persistent EM kernel — small complex128 runs
    without likelihood / history / timing events do their first L - 1
    iterations in one cooperative launch (the plain schedule's arithmetic;
    its own frame chunking unless ``chunk_frames`` is given). None: on the
    shapes where it measured faster; True: whenever the run fits; False: never.
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
    res = out or {}
    # preallocated outputs must match exactly: the kernels trust dtype/shape
    want = {"v": (rtype, (M, 2, N, F)), "images": (ctype, (M, 2, N, F, I)),
            "S": (torch.complex128, (M, 2, F, I, I)), "loglik": (torch.float64, (M, L + 1))}
    for key, (dt, shp) in want.items():
        t = res.get(key)
        if t is not None and (t.dtype != dt or tuple(t.shape) != shp or not t.is_cuda or
                              not t.is_contiguous()):
            raise ConfigurationError(
                f"out[{key!r}] must be a contiguous CUDA {dt} tensor of shape {shp}, got "
                f"{t.dtype} {tuple(t.shape)}")
    v = D.to_device(v0, rtype)
    v_in = None  # initial powers read by the first pass (the run writes `v`)
    if res.get("v") is not None:
        v_in, v = v, res["v"]  # preallocated output: no device copy of the init
    elif D.is_tensor(v0) and v.data_ptr() == v0.data_ptr():
        v_in, v = v, torch.empty_like(v)  # never clobber the caller's init
    S0 = D.to_device(S0, torch.complex128)
    fl = D.to_device(v_floor, torch.float64)
    if v_in is not None and (tuple(v_in.shape) != (M, 2, N, F) or not v_in.is_contiguous()):
        raise ConfigurationError(f"v must be (M, 2, N, F) = {(M, 2, N, F)}, got {tuple(v_in.shape)}")
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
    if graph:
        flags |= _lib.FLAG_GRAPH
    if persist is not None:
        flags |= _lib.FLAG_PERSIST if persist else _lib.FLAG_NO_PERSIST
    fast = algorithm == "fast"
    wsz = (lib.ffca_fastfca_workspace_size if fast else lib.ffca_fca_workspace_size)(
        M, N, F, I, L, flags, int(chunk_frames))
    ws = res.get("workspace")
    if ws is None or ws.numel() < wsz:
        ws = D.workspace(wsz)
    img = res.get("images") if images else None
    if images and img is None:
        img = D.empty((M, 2, N, F, I), ctype)
    S_out = res.get("S") if res.get("S") is not None else D.empty((M, 2, F, I, I), torch.complex128)
    ll = (res.get("loglik") if res.get("loglik") is not None else
          D.empty((M, L + 1), torch.float64)) if likelihood else None
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
        else None,
        v_in=D.ptr(v_in).value, bin_parts=int(bin_parts))
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


def plan_chunks(G, N, I=4, dtype="c128", algorithm="fast"):
    """The frame chunking the drivers pick for G bins x N frames (per-bin
    reduction order: equal chunking => bitwise-equal per-bin results)."""
    lib = D.require()
    cf = ctypes.c_int64()
    nc = ctypes.c_int()
    D.check_rc(lib.ffca_plan_chunks(int(G), int(N), int(I), DTYPES[dtype],
                                    0 if algorithm == "fast" else 1, ctypes.byref(cf),
                                    ctypes.byref(nc)), "ffca_plan_chunks")
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


def _host_tensor(x, dtype):
    """numpy / CPU tensor -> contiguous CPU tensor of ``dtype`` (no copy when possible)."""
    torch = D.torch
    t = x if D.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x))
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def run_host_pipelined(algorithm, y, v0, S0, v_floor, iterations, *, likelihood=True,
                       dtype="c128", chunk_frames=0, chunk_mixtures=None):
    """Batched run from HOST buffers with transfers overlapped with compute.

    The batch is split into mixture chunks; chunk k's EM run (compute stream)
    overlaps the H2D copy of chunk k+1 and the D2H copy of chunk k-1's images
    and model (two copy streams, double-buffered device slots). Results land
    in pinned host memory. Inputs: y (M,N,F,I), v0 (M,2,N,F), S0 (M,2,F,I,I),
    v_floor (M,F) as numpy or CPU tensors (pinned ones copy asynchronously).
    Returns dict of numpy arrays: images, v, S, loglik (or None), iteration_ms.
    """
    torch = D.torch
    D.require()
    ctype, rtype = torch_types(dtype)
    yh = _host_tensor(y, ctype)
    vh = _host_tensor(v0, rtype)
    Sh = _host_tensor(S0, torch.complex128)
    fh = _host_tensor(v_floor, torch.float64)
    M, N, F, I = (int(s) for s in yh.shape)
    L = int(iterations)
    if chunk_mixtures is None:
        # ~32 chunks: the D2H of the images is the bottleneck (PCIe), and the
        # pipeline fill before the first D2H (H2D + run of chunk 0) shrinks
        # with the chunk size
        chunk_mixtures = max(1, min(M, (M + 31) // 32))
    bounds = [(m0, min(M, m0 + chunk_mixtures)) for m0 in range(0, M, chunk_mixtures)]
    cm = chunk_mixtures
    dev = D.device()
    pin = dict(pin_memory=True)
    out_img = torch.empty((M, 2, N, F, I), dtype=ctype, **pin)
    out_v = torch.empty((M, 2, N, F), dtype=rtype, **pin)
    out_S = torch.empty((M, 2, F, I, I), dtype=torch.complex128, **pin)
    out_ll = torch.empty((M, L + 1), dtype=torch.float64, **pin) if likelihood else None
    pinned_in = yh.is_pinned() and vh.is_pinned()
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    slots = []
    for _ in range(2):
        slots.append(dict(
            y=torch.empty((cm, N, F, I), dtype=ctype, device=dev),
            v=torch.empty((cm, 2, N, F), dtype=rtype, device=dev),
            S0=torch.empty((cm, 2, F, I, I), dtype=torch.complex128, device=dev),
            fl=torch.empty((cm, F), dtype=torch.float64, device=dev),
            img=torch.empty((cm, 2, N, F, I), dtype=ctype, device=dev),
            S=torch.empty((cm, 2, F, I, I), dtype=torch.complex128, device=dev),
            free=torch.cuda.Event()))
    runs = []
    # every chunk's status word, copied out of its slot's workspace on the
    # compute stream right after the run (before the slot's next run resets it)
    status_h = torch.empty((len(bounds), 16), dtype=torch.uint8, pin_memory=True)
    caller = torch.cuda.current_stream()
    s_h2d.wait_stream(caller)
    s_cmp.wait_stream(caller)
    s_d2h.wait_stream(caller)
    for k, (m0, m1) in enumerate(bounds):
        sl = slots[k % 2]
        c = m1 - m0
        with torch.cuda.stream(s_h2d):
            if k >= 2:
                s_h2d.wait_event(sl["free"])
            sl["y"][:c].copy_(yh[m0:m1], non_blocking=pinned_in)
            sl["v"][:c].copy_(vh[m0:m1], non_blocking=pinned_in)
            sl["S0"][:c].copy_(Sh[m0:m1], non_blocking=True)
            sl["fl"][:c].copy_(fh[m0:m1], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_h2d)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_in)
            o = {"images": sl["img"][:c], "S": sl["S"][:c], "v": sl["v"][:c]}
            if sl.get("ws") is not None:
                o["workspace"] = sl["ws"]
            # the slot's v is the run's in-place work buffer (its init was just copied in);
            # repeated slot shapes replay a cached CUDA graph of the run
            run = run_device(algorithm, sl["y"][:c], sl["v"][:c], sl["S0"][:c], sl["fl"][:c], L,
                             likelihood=likelihood, history=False, images=True, dtype=dtype,
                             timing=(k == 0), check=False, chunk_frames=chunk_frames,
                             out=o, graph=(k > 0))
            sl["ws"] = run.workspace
            status_h[k].copy_(run.workspace[:16], non_blocking=True)
            ev_cmp = torch.cuda.Event()
            ev_cmp.record(s_cmp)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_cmp)
            out_img[m0:m1].copy_(sl["img"][:c], non_blocking=True)
            out_v[m0:m1].copy_(run.v, non_blocking=True)
            out_S[m0:m1].copy_(sl["S"][:c], non_blocking=True)
            if likelihood:
                out_ll[m0:m1].copy_(run.loglik, non_blocking=True)
            sl["free"].record(s_d2h)
        runs.append((run, c))
    for s in (s_h2d, s_cmp, s_d2h):
        s.synchronize()
    _raise_first(status_h.numpy(), N, F)
    _collect_timings(runs[0][0])
    return {"images": out_img.numpy(), "v": out_v.numpy(), "S": out_S.numpy(),
            "floor": fh.numpy(), "loglik": out_ll.numpy() if likelihood else None,
            "iteration_ms": runs[0][0].iteration_ms, "chunks": len(bounds)}


def _raise_first(words, N, F):
    """Raise for the earliest failure over a chunked batch, in the status key
    order of one run over the whole batch: iteration, then code, then the flat
    index, whose leading axis is the mixture (chunks cover increasing,
    disjoint mixture ranges, so chunk order breaks ties before the index)."""
    best = None
    for k, word in enumerate(words):
        st = D.decode_status(word)
        if st.code == _lib.FFCA_OK:
            continue
        key = (st.iteration, st.code, k, int(st.index))
        if best is None or key < best[0]:
            best = (key, st)
    if best is not None:
        D.raise_for_status(best[1], N, F)


class MultiStreamRun:
    """A batched device run split over several CUDA streams (see run_device_streams)."""

    def __init__(self, parts, streams, events):
        self.parts = parts
        self.streams = streams
        self.events = events

    def wait(self):
        cur = D.torch.cuda.current_stream()
        for e in self.events:
            cur.wait_event(e)


def run_device_streams(algorithm, y, v0, S0, v_floor, iterations, *, nstreams=2, out=None,
                       workspaces=None, **kw):
    """Independent mixtures of a batch run as ``nstreams`` concurrent device
    runs (one stream each): while one part is in its per-bin pencil update or
    its last partial wave, the other part's streaming pass fills the SMs.
    Outputs are written into ``out`` (images, S, v: full-batch tensors);
    per-part workspaces are reused when given. Same results as one run with
    the same ``chunk_frames``."""
    torch = D.torch
    M = int(y.shape[0])
    k = max(1, min(int(nstreams), M))
    bounds = [(M * i // k, M * (i + 1) // k) for i in range(k)]
    cur = torch.cuda.current_stream()
    streams = kw.pop("streams", None) or [torch.cuda.Stream() for _ in range(k)]
    parts, events = [], []
    for i, (a, b) in enumerate(bounds):
        s = streams[i]
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            o = None
            if out is not None:
                o = {key: (t[a:b] if key in ("images", "S", "v") and t is not None else t)
                     for key, t in out.items() if key != "workspace"}
                if workspaces is not None and workspaces[i] is not None:
                    o["workspace"] = workspaces[i]
            r = run_device(algorithm, y[a:b], v0[a:b], S0[a:b], v_floor[a:b], iterations,
                           out=o, **kw)
            ev = torch.cuda.Event()
            ev.record(s)
        parts.append(r)
        events.append(ev)
    for e in events:
        cur.wait_event(e)
    return MultiStreamRun(parts, streams, events)
