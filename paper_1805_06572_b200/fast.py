"""FastFCA engine on the GPU (reference fast.py:1-260).

``fastfca_run`` keeps the reference signature and semantics — initial
pencil, L x {fused transform/E/M pass, gram ridge, pencil refresh},
likelihood trace with ``loglik_trace[0]`` under the initial model, history
of (v, back-transformed S), images = posterior means of the last E-step
mapped back through the basis that produced them — but the whole loop is
one call into ``ffca_fastfca_run``: y is streamed from HBM once per
iteration by the fused kernel, the per-bin pencil work is a second kernel,
and nothing returns to the host until the run ends.

Inputs may be (N, F, I) for one mixture (reference shape) or (M, N, F, I)
for a batch; numpy inputs give numpy outputs, CUDA tensors stay on device.
"""

from __future__ import annotations

import numpy as np

from . import _backend
from . import _device as D
from ._engine import as_batch, run_device, run_host_pipelined, torch_types
from .errors import SingularMatrixError
from .modelops import COV_EPS_FACTOR  # noqa: F401  (re-exported like the reference)
from .pencil import gevd_hpd, logdet2
from .types import OpCounts, SeparationResult, SpatialModel


def _kern():
    return _backend.kernels()


def transform_observations(y, P):
    """``y_tilde = P^H y`` for all frames (fast.py:58-60)."""
    data = y if (D.is_tensor(y) or isinstance(y, np.ndarray)) else y.data
    return _kern().fast_transform(data, P)


def fast_e_step(y_tilde, v, Lambda):
    """Posterior moments in the diagonal basis (fast.py:63-71)."""
    mu, Phi, _, _ = _kern().fast_e_step(y_tilde, v, Lambda)
    return mu, Phi


def fast_m_step_v(Phi_tilde, Lambda):
    """v_1 = tr(diag(lam)^-1 Phi_1)/I, v_2 = tr(Phi_2)/I (fast.py:74-77)."""
    return _kern().fast_v_update(Phi_tilde, Lambda)


def regularize_transformed(S_raw, gram):
    """Hermitize + eps*gram ridge (fast.py:80-90) on the device."""
    lib = D.require()
    shape = tuple(S_raw.shape)
    d = shape[-1]
    batch = int(np.prod(shape[:-2]))
    Sd = D.to_device(S_raw, D.torch.complex128).reshape(batch, d, d)
    gd = None
    if gram is not None:
        g = D.to_device(gram, D.torch.complex128)
        gd = g.expand(shape[:-3] + tuple(g.shape[-3:])).reshape(batch, d, d).contiguous() \
            if len(shape) > 3 else g.reshape(batch, d, d)
    out = D.empty((batch, d, d), D.torch.complex128)
    D.check_rc(lib.ffca_regularize_transformed(D.ptr(Sd), D.ptr(gd), D.ptr(out), batch, d,
                                               D.stream_handle()), "ffca_regularize_transformed")
    out = out.reshape(shape)
    return out if D.is_tensor(S_raw) else D.host(out)


def fast_m_step_S(Phi_tilde, v, gram=None):
    """Transformed covariance update (1/N) sum_n Phi~/v, regularised (fast.py:93-104)."""
    return regularize_transformed(_kern().fast_S_update(Phi_tilde, v), gram)


def propagate_pencil(S_tilde_1, S_tilde_2, P_prev, counts=None):
    """Refresh the basis: ``P_next = P_prev @ Q`` with Q the pencil of the
    transformed covariances (fast.py:107-124)."""
    lib = D.require()
    shape = tuple(P_prev.shape)
    d = shape[-1]
    batch = int(np.prod(shape[:-2])) if len(shape) > 2 else 1
    a = D.to_device(S_tilde_1, D.torch.complex128).reshape(batch, d, d)
    b = D.to_device(S_tilde_2, D.torch.complex128).reshape(batch, d, d)
    p = D.to_device(P_prev, D.torch.complex128).reshape(batch, d, d)
    Pn = D.empty((batch, d, d), D.torch.complex128)
    lam = D.empty((batch, d), D.torch.float64)
    st = D.StageStatus()
    D.check_rc(lib.ffca_propagate_pencil(D.ptr(a), D.ptr(b), D.ptr(p), D.ptr(Pn), D.ptr(lam),
                                         batch, d, st.handle, D.stream_handle()),
               "ffca_propagate_pencil")
    st.raise_if_error()
    if counts is not None:
        counts.add(gevds=batch, bin_products=batch)
    Pn = Pn.reshape(shape)
    lam = lam.reshape(shape[:-1])
    if D.is_tensor(P_prev):
        return Pn, lam
    return D.host(Pn), D.host(lam)


def initial_pencil(model):
    """Pencil of the initial covariances (fast.py:127-130) -> (P, lam)."""
    dec = gevd_hpd(model.S[0], model.S[1])
    return dec.eigenvectors, dec.eigenvalues


def back_transform_images(mu_tilde, P):
    """Solve ``P^H mu = mu_tilde`` per bin (fast.py:133-141)."""
    lib = D.require()
    mu = D.to_device(mu_tilde, D.torch.complex128)
    Pd = D.to_device(P, D.torch.complex128)
    Src, N, F, I = (int(s) for s in mu.shape)
    out = D.empty((Src, N, F, I), D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_back_transform_images(D.ptr(mu), D.ptr(Pd), D.ptr(out), Src, N, F, I,
                                              st.handle, D.stream_handle()),
               "ffca_back_transform_images")
    if st.read().code:
        raise SingularMatrixError("basis matrix is singular")
    return out if D.is_tensor(mu_tilde) else D.host(out)


def back_transform_covariances(S_tilde, P):
    """``(P^H)^{-1} S_tilde P^{-1}`` per bin (fast.py:144-148)."""
    lib = D.require()
    S = D.to_device(S_tilde, D.torch.complex128)
    Pd = D.to_device(P, D.torch.complex128)
    shape = tuple(S.shape)
    F, I = int(Pd.shape[-3]), int(Pd.shape[-1])
    Src = int(np.prod(shape[:-3])) if len(shape) > 3 else 1
    out = D.empty(shape, D.torch.complex128)
    st = D.StageStatus()
    D.check_rc(lib.ffca_back_transform_covariances(D.ptr(S), D.ptr(Pd), D.ptr(out), Src, F, I,
                                                   st.handle, D.stream_handle()),
               "ffca_back_transform_covariances")
    if st.read().code:
        raise SingularMatrixError("basis matrix is singular")
    return out if D.is_tensor(S_tilde) else D.host(out)


def _finish(run, algorithm, L, batched, device_out, counts, record_history):
    """DeviceRun -> SeparationResult (reference shapes when not batched)."""
    def conv(t):
        if t is None:
            return None
        return t if device_out else D.host(t)

    sel = (lambda t: t) if batched else (lambda t: t[0])
    images = conv(sel(run.images)) if run.images is not None else None
    v = conv(sel(run.v))
    S = conv(sel(run.S))
    floor = conv(sel(run.floor))
    if run.loglik is not None:
        ll = D.host(run.loglik)
        trace = ll if batched else [float(x) for x in ll[0]]
    else:
        trace = []
    history = []
    if record_history and run.S_hist is not None:
        vh = conv(run.v_hist)
        Sh = conv(run.S_hist)
        for l in range(L):
            history.append({"v": vh[l] if batched else vh[l][0],
                            "S": Sh[l] if batched else Sh[l][0]})
    it_s = [ms / 1e3 for ms in run.iteration_ms]
    return SeparationResult(
        algorithm=algorithm, images=images, loglik_trace=trace, iteration_seconds=it_s,
        em_seconds=float(sum(it_s)), op_counts=counts,
        model=SpatialModel(v=v, S=S, v_floor=floor), history=history)


def fastfca_run(y, init, iterations, record_history=False, compute_likelihood=True,
                incremental_transform=False, dtype="c128", device_output=None, chunk_frames=0):
    """Joint-diagonalisation EM + MMSE images (reference fast.py:156-260).

    ``dtype='c64'`` streams y / v / images in complex64 with float64 per-bin
    state (B200 extension; the reference is complex128 only).
    """
    yb, vb, Sb, fb, batched = as_batch(y, init)
    if device_output is None:
        device_output = D.is_tensor(yb)
    L = int(iterations)
    if incremental_transform:
        return _incremental_run(yb, vb, Sb, fb, L, batched, device_output, record_history,
                                compute_likelihood)
    if _pipelined_ok(yb, batched, device_output, record_history):
        return _finish_host(run_host_pipelined("fast", yb, vb, Sb, fb, L,
                                               likelihood=compute_likelihood, dtype=dtype,
                                               chunk_frames=chunk_frames), "FastFCA", L)
    run = run_device("fast", yb, vb, Sb, fb, L, likelihood=compute_likelihood,
                     history=record_history, images=True, dtype=dtype,
                     chunk_frames=chunk_frames)
    run.floor = D.to_device(fb, D.torch.float64)
    M, F = int(run.v.shape[0]), int(run.v.shape[-1])
    counts = OpCounts()
    counts.add(gevds=L * F * (M if batched else 1), bin_products=2 * L * F * (M if batched else 1))
    return _finish(run, "FastFCA", L, batched, device_output, counts, record_history)


def _pipelined_ok(yb, batched, device_output, record_history):
    """Host-resident batches take the transfer/compute-overlapped path."""
    on_host = not (D.is_tensor(yb) and yb.is_cuda)
    return batched and on_host and not device_output and not record_history and \
        int(yb.shape[0]) > 1


def _finish_host(res, algorithm, L):
    M, _, N, F = res["v"].shape
    counts = OpCounts()
    if algorithm == "FastFCA":
        counts.add(gevds=L * F * M, bin_products=2 * L * F * M)
    else:
        counts.add(inversions=L * N * F * M, products=3 * L * N * F * M)
        if L == 0:
            counts.add(inversions=N * F * M, products=3 * N * F * M)
    it_s = [ms / 1e3 for ms in res["iteration_ms"]]
    return SeparationResult(
        algorithm=algorithm, images=res["images"],
        loglik_trace=res["loglik"] if res["loglik"] is not None else [],
        iteration_seconds=it_s, em_seconds=float(sum(it_s)), op_counts=counts,
        model=SpatialModel(v=res["v"], S=res["S"], v_floor=res["floor"]), history=[])


def _incremental_run(yb, vb, Sb, fb, L, batched, device_output, record_history,
                     compute_likelihood):
    """Benchmark-mode variant (fast.py:204-215): update y~ with the per-
    iteration pencil factor instead of re-transforming; stage kernels."""
    if batched:
        raise NotImplementedError("incremental_transform supports one mixture")
    torch = D.torch
    ctype, rtype = torch_types("c128")
    y = D.to_device(yb, ctype)[0]
    v = D.to_device(vb, rtype)[0].clone()
    S0 = D.to_device(Sb, torch.complex128)[0]
    fl = D.to_device(fb, torch.float64)[0]
    kern = _kern()
    dec = gevd_hpd(S0[0], S0[1])
    P, lam = dec.eigenvectors, dec.eigenvalues
    counts = OpCounts()
    trace, history = [], []
    if compute_likelihood:
        trace.append(kern.fast_log_likelihood(kern.fast_transform(y, P), v, lam, logdet2(P)))
    yt, Q, mu_t, P_e, S_t = None, None, None, P, None
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(L)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(L)]
    for l in range(L):
        starts[l].record()
        P_e = P
        yt = kern.fast_transform(y if yt is None else yt, P if yt is None else Q)
        mu_t, Phi_t, _, _ = kern.fast_e_step(yt, v, lam)
        v = torch.maximum(kern.fast_v_update(Phi_t, lam), fl[None, None, :])
        S_raw = kern.fast_S_update(Phi_t, v)
        if not (bool(torch.isfinite(v).all()) and bool(torch.isfinite(S_raw).all())):
            raise SingularMatrixError("mixture covariance is singular (source powers collapsed "
                                      "to zero)")
        gram = P.conj().transpose(-1, -2) @ P
        counts.add(bin_products=gram.shape[0])
        S_t = regularize_transformed(S_raw, gram)
        Q_new, lam = propagate_pencil(S_t[0], S_t[1], torch.eye(P.shape[-1], dtype=P.dtype,
                                                                 device=P.device).expand_as(P)
                                      .contiguous(), counts=counts)
        P = P @ Q_new
        Q = Q_new
        ends[l].record()
        if compute_likelihood:
            trace.append(kern.fast_log_likelihood(kern.fast_transform(y, P), v, lam, logdet2(P)))
        if record_history:
            history.append({"v": v.clone(), "S": back_transform_covariances(S_t, P_e)})
    if mu_t is None:
        mu_t, _, _, _ = kern.fast_e_step(kern.fast_transform(y, P), v, lam)
        P_e = P
    images = back_transform_images(mu_t, P_e)
    S_final = history[-1]["S"] if (L and history) else (
        back_transform_covariances(S_t, P_e) if L else S0.clone())
    torch.cuda.synchronize()
    it_s = [starts[i].elapsed_time(ends[i]) / 1e3 for i in range(L)]
    conv = (lambda t: t) if device_output else D.host
    return SeparationResult(
        algorithm="FastFCA", images=conv(images), loglik_trace=trace, iteration_seconds=it_s,
        em_seconds=float(sum(it_s)), op_counts=counts,
        model=SpatialModel(v=conv(v), S=conv(S_final), v_floor=conv(fl)),
        history=[{"v": conv(h["v"]), "S": conv(h["S"])} for h in history])
