"""Initial spatial models (reference initializers.py:20-143).

``init_random``: seeded random model (initializers.py:20-39).

``S_j = A A^H + I`` with one complex Gaussian I x I draw per source shared
across bins (drawn on the host with numpy's PCG64 so the stream is
bit-identical to the reference's), powers ``||y||^2/(2I)`` floored per bin,
computed on the device by ``ffca_init_powers``.

``init_from_masks``: direction-clustering model (initializers.py:42-143),
entirely on the device (``ffca_init_masks``, csrc/ffca_masks.cu): per-bin
2-means of the phase-aligned unit observation vectors, unit-trace group
covariances, cross-bin label alignment, masked floored powers.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from .types import SpatialModel


def draw_covariances(seed, n_bins, n_chan):
    gen = np.random.default_rng(seed)
    S = np.empty((2, n_bins, n_chan, n_chan), dtype=np.complex128)
    for j in range(2):
        re = gen.standard_normal((n_chan, n_chan))
        im = gen.standard_normal((n_chan, n_chan))
        A = re + 1j * im
        S[j] = (A @ A.conj().T + np.eye(n_chan))[None]
    return S


def init_random(y, seed, dtype="c128"):
    """Reference ``init_random(y, seed)``; device tensors in -> device tensors out."""
    lib = D.require()
    torch = D.torch
    data = y if (D.is_tensor(y) or isinstance(y, np.ndarray)) else y.data
    ctype, rtype = (torch.complex128, torch.float64) if dtype == "c128" else (torch.complex64,
                                                                             torch.float32)
    yd = D.to_device(data, ctype)
    N, F, I = (int(s) for s in yd.shape[-3:])
    v = D.empty((1, 2, N, F), rtype)
    floor = D.empty((1, F), torch.float64)
    D.check_rc(lib.ffca_init_powers(D.ptr(yd), D.ptr(v), D.ptr(floor), 1, N, F, I,
                                    0 if dtype == "c128" else 1, D.stream_handle()),
               "ffca_init_powers")
    S = draw_covariances(seed, F, I)
    if D.is_tensor(y):
        return SpatialModel(v=v[0], S=torch.as_tensor(S, device=yd.device), v_floor=floor[0])
    return SpatialModel(v=D.host(v[0]), S=S, v_floor=D.host(floor[0]))


def init_random_batch(Y, seeds, dtype="c128"):
    """``init_random`` for a batch Y (M, N, F, I): mixture m uses ``seeds[m]``.
    Powers and floors for the whole batch come from one ``ffca_init_powers``
    launch; CUDA input -> CUDA outputs, host input -> host outputs."""
    lib = D.require()
    torch = D.torch
    ctype, rtype = (torch.complex128, torch.float64) if dtype == "c128" else (torch.complex64,
                                                                             torch.float32)
    yd = D.to_device(Y, ctype)
    M, N, F, I = (int(s) for s in yd.shape)
    if len(seeds) != M:
        raise ValueError("one seed per mixture")
    v = D.empty((M, 2, N, F), rtype)
    floor = D.empty((M, F), torch.float64)
    D.check_rc(lib.ffca_init_powers(D.ptr(yd), D.ptr(v), D.ptr(floor), M, N, F, I,
                                    0 if dtype == "c128" else 1, D.stream_handle()),
               "ffca_init_powers")
    S = np.stack([draw_covariances(int(s), F, I) for s in seeds])
    if D.is_tensor(Y) and Y.is_cuda:
        return SpatialModel(v=v, S=torch.as_tensor(S, device=yd.device), v_floor=floor)
    return SpatialModel(v=D.host(v), S=S, v_floor=D.host(floor))


def _masks_device(yd, M, N, F, I):
    lib = D.require()
    torch = D.torch
    v = D.empty((M, 2, N, F), torch.float64)
    S = D.empty((M, 2, F, I, I), torch.complex128)
    floor = D.empty((M, F), torch.float64)
    wsz = lib.ffca_init_masks_workspace_size(M, N, F, I)
    ws = D.workspace(wsz)
    D.check_rc(lib.ffca_init_masks(D.ptr(yd), D.ptr(v), D.ptr(S), D.ptr(floor), M, N, F, I,
                                   D.ptr(ws), wsz, D.stream_handle()), "ffca_init_masks")
    return v, S, floor


def init_from_masks(y):
    """Reference ``init_from_masks(y)`` (initializers.py:71-143); CUDA tensor in
    -> CUDA tensors out, host in -> host out. Falls back to
    ``init_random(y, seed=0)`` when there are fewer than 2 I frames."""
    D.require()
    torch = D.torch
    data = y if (D.is_tensor(y) or isinstance(y, np.ndarray)) else y.data
    yd = D.to_device(data, torch.complex128)
    N, F, I = (int(s) for s in yd.shape[-3:])
    if N < 2 * I:
        return init_random(y, seed=0)
    v, S, floor = _masks_device(yd.reshape(1, N, F, I), 1, N, F, I)
    if D.is_tensor(y) and y.is_cuda:
        return SpatialModel(v=v[0], S=S[0], v_floor=floor[0])
    return SpatialModel(v=D.host(v[0]), S=D.host(S[0]), v_floor=D.host(floor[0]))


def init_from_masks_batch(Y):
    """``init_from_masks`` for every mixture of a batch Y (M, N, F, I) in one
    set of launches (bins and mixtures in parallel)."""
    D.require()
    torch = D.torch
    yd = D.to_device(Y, torch.complex128)
    M, N, F, I = (int(s) for s in yd.shape)
    if N < 2 * I:
        return init_random_batch(Y, [0] * M)
    v, S, floor = _masks_device(yd, M, N, F, I)
    if D.is_tensor(Y) and Y.is_cuda:
        return SpatialModel(v=v, S=S, v_floor=floor)
    return SpatialModel(v=D.host(v), S=D.host(S), v_floor=D.host(floor))
