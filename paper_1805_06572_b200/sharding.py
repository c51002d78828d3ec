"""Multi-GPU partitioning of the EM path: one process per GPU, no collective
inside the EM loop.

Every EM quantity is per frequency bin (and per mixture): nothing couples
bins inside the loop (the reference calls the work
"embarrassingly parallel over f", and its
per-bin loop is fast.py:200-223). Batches are therefore split by mixture
(config 3) and single long mixtures by contiguous bin ranges (config 4).

Every world size 1..MAX_WORLD uses ONE frame chunking — the plan that fills a
GPU with the shard of the largest world size (:func:`shard_chunk_frames`) —
so per-bin results are bitwise identical at every N, and the only cross-GPU
traffic is the final gather of the per-rank results to one rank (NCCL over
NVLink for CUDA tensors, gloo for host tensors) in fixed rank order.

Entry points: :func:`run_shard` (this rank's share of a global batch; what
each process runs), :func:`run_sharded` / :func:`fastfca_run_sharded` /
:func:`fca_run_sharded` (shard + run + gather under ``torch.distributed``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_range(total, rank, world):
    """Contiguous balanced [a, b) of ``total`` units for ``rank`` of ``world``."""
    per, extra = divmod(int(total), int(world))
    a = rank * per + min(rank, extra)
    return a, a + per + (1 if rank < extra else 0)


@dataclass(frozen=True)
class Shard:
    axis: str  # "mixtures" or "bins"
    start: int
    stop: int
    total: int = 0  # units of the whole problem along ``axis``

    @property
    def size(self):
        return self.stop - self.start


def plan_shard(M, F, rank, world):
    """Mixture shards for batches (M > 1), bin shards for one mixture."""
    if M > 1:
        return Shard("mixtures", *shard_range(M, rank, world), int(M))
    return Shard("bins", *shard_range(F, rank, world), int(F))


def take(shard, y, v, S, floor):
    """Slice reference-layout batched arrays (M,N,F,I), (M,2,N,F), (M,2,F,I,I),
    (M,F) to this rank's shard (contiguous copies)."""
    a, b = shard.start, shard.stop
    if shard.axis == "mixtures":
        sl = (slice(a, b),)
        return tuple(np.ascontiguousarray(x[sl]) for x in (y, v, S, floor))
    return (np.ascontiguousarray(y[:, :, a:b]), np.ascontiguousarray(v[:, :, :, a:b]),
            np.ascontiguousarray(S[:, :, a:b]), np.ascontiguousarray(floor[:, a:b]))


# axis of the shard dimension in each result array (batched layouts)
RESULT_AXES = {
    "mixtures": {"images": 0, "v": 0, "S": 0, "floor": 0, "loglik": 0},
    "bins": {"images": 3, "v": 3, "S": 2, "floor": 1, "loglik": None},
}


def gather_results(local, shard, group=None, dst=0):
    """Gather per-rank result arrays to ``dst`` and concatenate in rank order.

    ``local``: dict of torch tensors (CUDA with NCCL, CPU with gloo) in the
    batched layouts. Shards are padded to the largest shard and sent with one
    ``gather`` per array (only ``dst`` receives). For bin shards the per-rank
    log-likelihood partial sums are added in rank order (fixed order:
    deterministic). Returns the full dict on ``dst`` and None elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    axes = RESULT_AXES[shard.axis]
    out = {} if rank == dst else None
    # shard sizes are a pure function of (total, world): no size exchange
    sizes = [b - a for a, b in (shard_range(shard.total, r, world) for r in range(world))]
    # gloo gathers host tensors only: CUDA results are staged through the host
    stage = dist.get_backend(group) == "gloo"
    for key in sorted(local):
        t = local[key]
        if t is None:
            continue
        if stage and t.is_cuda:
            t = t.cpu()
        ax = axes.get(key)
        cplx = t.is_complex()
        # complex payloads travel as (..., 2) reals: gloo has no complex
        # reductions / gathers, and NCCL moves bytes either way
        t = torch.view_as_real(t.contiguous()) if cplx else t.contiguous()
        if ax is None:  # summed partials (bin-sharded log-likelihood)
            parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
            dist.gather(t, parts, dst=dst, group=group)
            if rank == dst:
                acc = parts[0].clone()
                for p in parts[1:]:
                    acc += p
                out[key] = acc
            continue
        mx = max(sizes)
        if t.shape[ax] != mx:
            pad_shape = list(t.shape)
            pad_shape[ax] = mx
            buf = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
            buf.narrow(ax, 0, t.shape[ax]).copy_(t)
        else:
            buf = t
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
        dist.gather(buf, parts, dst=dst, group=group)
        if rank == dst:
            full = torch.cat([p.narrow(ax, 0, n) for p, n in zip(parts, sizes)], dim=ax)
            out[key] = torch.view_as_complex(full) if cplx else full
    return out


# ---- sharded runs -------------------------------------------------------------
MAX_WORLD = 8  # one node of B200s


def _plan_cost(G, N, I, cf, dtype, algorithm):
    """The drivers' modelled makespan of one streaming pass (ffca_fast.cu
    plan_chunks): waves x (frames per chunk + per-CTA overhead)."""
    # bin windows of the split-phase schedule at I >= 5 (each window's pass has to
    # fill the GPU by itself; at I <= 4 the windows' passes are chained with
    # programmatic launch and fill one another's tails: whole-grid model)
    k = plan_parts(G, N, I, dtype, algorithm) if I >= 5 else 1
    gm = grid_model(-(-G // k), N, I, cf, dtype, algorithm)
    waves = -(-gm["ctas"] // max(gm["slots"], 1))
    return k * waves * (min(cf, N) + 24)


def plan_parts(G, N, I, dtype="c128", algorithm="fast"):
    """Bin windows the FastFCA driver pipelines for G bins (1 = plain schedule)."""
    from . import _device as D
    from ._engine import DTYPES

    lib = D.require()
    return max(1, int(lib.ffca_plan_parts(int(G), int(N), int(I), DTYPES[dtype],
                                          0 if algorithm == "fast" else 1)))


def shard_chunk_frames(M, N, F, I, dtype="c128", algorithm="fast", max_world=MAX_WORLD):
    """The frame chunking every world size 1..``max_world`` uses.

    Equal chunking at every N => bitwise-equal per-bin results (the per-bin
    reduction order depends on the chunking only). The plan is the one whose
    worst relative modelled cost over the world sizes 1, 2, 4, ..,
    ``max_world`` (rank 0's shard, the largest) is smallest (near-ties to
    the fewest chunks): a plan tuned
    for the 8-GPU shard alone can cost a 1-GPU run >10% (FCA at config 3:
    56 waves of short chunks instead of 7 of whole-mixture chunks)."""
    from ._engine import plan_chunks

    def shard_bins(w):
        sh = plan_shard(M, F, 0, w)
        return sh.size * F if sh.axis == "mixtures" else sh.size

    if max_world <= 1:
        return plan_chunks(M * F, N, I, dtype, algorithm)[0]
    worlds = sorted({w for w in (1, 2, 4, 8, 16, 32, 64) if w <= max_world} | {max_world})
    min_frames = 16 if I >= 5 else 32
    max_nc = max(1, min(4096, -(-N // min_frames)))
    if algorithm == "fast" and I <= 3:
        max_nc = min(max_nc, 17)  # (the per-bin refresh K1 reads every chunk: ffca_fast.cu)
    cands = sorted({-(-N // nc) for nc in range(1, max_nc + 1)}, reverse=True)
    costs = {w: [_plan_cost(shard_bins(w), N, I, cf, dtype, algorithm) for cf in cands]
             for w in worlds}
    best = {w: min(c) for w, c in costs.items()}
    score = [max(costs[w][i] / best[w] for w in worlds) for i in range(len(cands))]
    # near-ties (within the model's ~2% resolution) go to the fewest chunks:
    # every chunk costs a partial-sum write per bin and one more term in the
    # per-bin refresh, which the wave model ignores (config 3 FastFCA at 1 GPU:
    # 3 chunks 1.50 ms per pass vs 5 chunks 1.55 ms, modelled 6174 vs 6576
    # at 1 GPU but 882 vs 822 at 8 GPUs)
    top = min(score)
    return max(cf for cf, sc in zip(cands, score) if sc <= top * 1.02)


def grid_model(G, N, I, chunk_frames, dtype="c128", algorithm="fast"):
    """Modelled grid of one streaming pass: CTAs, resident slots, waves."""
    import ctypes

    from . import _device as D
    from ._engine import DTYPES

    lib = D.require()
    ctas, slots = ctypes.c_int64(), ctypes.c_int64()
    D.check_rc(lib.ffca_plan_grid(int(G), int(N), int(I), DTYPES[dtype],
                                  0 if algorithm == "fast" else 1, int(chunk_frames),
                                  ctypes.byref(ctas), ctypes.byref(slots)), "ffca_plan_grid")
    return {"ctas": int(ctas.value), "slots": int(slots.value),
            "waves": round(ctas.value / max(slots.value, 1), 3)}


def _host_array(x):
    if hasattr(x, "detach"):  # torch tensor
        x = x.detach()
        return x.cpu().numpy() if x.is_cuda else x.numpy()
    return np.asarray(x)


def _device_runner(algorithm, y, v, S, floor, L, *, chunk_frames, likelihood, images, dtype):
    from ._engine import run_device

    r = run_device(algorithm, y, v, S, floor, L, likelihood=likelihood, history=False,
                   images=images, dtype=dtype, timing=False, check=True,
                   chunk_frames=chunk_frames)
    return {"images": r.images, "v": r.v, "S": r.S, "loglik": r.loglik}


def _empty_local(shard, M, N, F, I, L, dtype, likelihood, images, device):
    """Results of an empty shard in the batched layouts (zero-size along the
    shard axis; a bin shard's likelihood partial is an exact zero)."""
    import torch

    from ._engine import torch_types

    ctype, rtype = torch_types(dtype)
    if shard.axis == "mixtures":
        m, f = 0, F
    else:
        m, f = M, 0
    kw = dict(device=device)
    out = {"v": torch.empty((m, 2, N, f), dtype=rtype, **kw),
           "S": torch.empty((m, 2, f, I, I), dtype=torch.complex128, **kw),
           "floor": torch.empty((m, f), dtype=torch.float64, **kw)}
    if images:
        out["images"] = torch.empty((m, 2, N, f, I), dtype=ctype, **kw)
    if likelihood:
        out["loglik"] = torch.zeros((m, L + 1), dtype=torch.float64, **kw)
    return out


def run_shard(algorithm, y, init, iterations, rank, world, *, chunk_frames=None, runner=None,
              likelihood=True, images=True, dtype="c128", global_size=None):
    """Run this rank's shard of a problem on the current device.

    ``y`` (M,N,F,I) or (N,F,I) and ``init`` (a SpatialModel of matching
    shape) are the GLOBAL inputs (host arrays or tensors; each rank slices its
    own contiguous mixture or bin range) — or, with ``global_size=(M, F)``
    (the whole problem's mixture and bin counts), this rank's shard already
    (what a caller that never holds the global batch passes; pinned host
    tensors then copy asynchronously). Returns ``(shard, local)`` with
    ``local`` the shard's results in the batched layouts (images, v, S,
    floor, loglik — for bin shards the partial log-likelihood over the
    shard's bins, which the gather sums). ``runner`` replaces the CUDA run
    (tests use the CPU oracle); ``chunk_frames`` defaults to
    :func:`shard_chunk_frames` of the whole problem.
    """
    import torch

    from ._engine import as_batch

    yb, vb, Sb, fb, _ = as_batch(y, init)
    M, N, F, I = (int(s) for s in yb.shape)
    if global_size is None:
        Mg, Fg = M, F
    else:
        Mg, Fg = (int(s) for s in global_size)
    shard = plan_shard(Mg, Fg, rank, world)
    if global_size is not None:
        got = M if shard.axis == "mixtures" else F
        if got != shard.size or (shard.axis == "mixtures" and F != Fg) or \
                (shard.axis == "bins" and M != Mg):
            raise ValueError(f"rank {rank}/{world}: local inputs (M={M}, F={F}) are not the "
                             f"{shard.axis} shard [{shard.start}, {shard.stop}) of "
                             f"(M={Mg}, F={Fg})")
    if chunk_frames is None:  # (a custom runner plans its own chunking)
        chunk_frames = shard_chunk_frames(Mg, N, Fg, I, dtype, algorithm) if runner is None else 0
    dev = "cpu" if runner is not None else "cuda"
    if shard.size == 0:  # more ranks than units: this rank only joins the gather
        return shard, _empty_local(shard, Mg, N, Fg, I, int(iterations), dtype, likelihood,
                                   images, dev)
    if global_size is None:
        ys, vs, Ss, fs = take(shard, *(_host_array(x) for x in (yb, vb, Sb, fb)))
    else:
        ys, vs, Ss, fs = yb, vb, Sb, fb
    run = runner or _device_runner
    local = run(algorithm, ys, vs, Ss, fs, int(iterations), chunk_frames=chunk_frames,
                likelihood=likelihood, images=images, dtype=dtype)
    local = {k: t for k, t in local.items() if t is not None}
    ref = local["v"]
    local["floor"] = (fs if torch.is_tensor(fs) else torch.from_numpy(np.asarray(fs))).to(
        device=ref.device, dtype=torch.float64)
    return shard, local


def run_sharded(algorithm, y, init, iterations, *, group=None, dst=0, runner=None,
                likelihood=True, images=True, dtype="c128", chunk_frames=None,
                global_size=None):
    """Shard a run over the ranks of ``group`` (one GPU per rank), run each
    shard with no collective, and gather the results to ``dst`` (NCCL for
    CUDA results; the only cross-GPU traffic of the run).

    Returns ``(shard, full)``: ``full`` is the dict of whole-problem results
    (images, v, S, floor, loglik; tensors on ``dst``'s device) on ``dst`` and
    None elsewhere. ``global_size``: see :func:`run_shard`.
    """
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    shard, local = run_shard(algorithm, y, init, iterations, rank, world,
                             chunk_frames=chunk_frames, runner=runner, likelihood=likelihood,
                             images=images, dtype=dtype, global_size=global_size)
    return shard, gather_results(local, shard, group=group, dst=dst)


def _result(algorithm, full, y, init, L):
    from . import _device as D
    from ._engine import as_batch
    from .types import OpCounts, SeparationResult, SpatialModel

    batched = as_batch(y, init)[4]
    sel = (lambda t: t) if batched else (lambda t: t[0])
    host = not (D.is_tensor(y) and y.is_cuda)
    conv = D.host if host else (lambda t: t)
    M, _, N, F = (int(s) for s in full["v"].shape)
    L = int(L)
    counts = OpCounts()
    if algorithm == "fast":
        counts.add(gevds=L * F * M, bin_products=2 * L * F * M)
    else:
        counts.add(inversions=L * N * F * M, products=3 * L * N * F * M)
        if L == 0:
            counts.add(inversions=N * F * M, products=3 * N * F * M)
    ll = full.get("loglik")
    if ll is None:
        trace = []
    else:
        llh = ll.cpu().numpy()
        trace = llh if batched else [float(x) for x in llh[0]]
    return SeparationResult(
        algorithm="FastFCA" if algorithm == "fast" else "FCA",
        images=conv(sel(full["images"])) if full.get("images") is not None else None,
        loglik_trace=trace, iteration_seconds=[], em_seconds=0.0, op_counts=counts,
        model=SpatialModel(v=conv(sel(full["v"])), S=conv(sel(full["S"])),
                           v_floor=conv(sel(full["floor"])) if "floor" in full
                           else init.v_floor),
        history=[])


def fastfca_run_sharded(y, init, iterations, compute_likelihood=True, *, group=None, dst=0,
                        dtype="c128", runner=None, chunk_frames=None, global_size=None):
    """``fastfca_run`` (reference fast.py:156-260) over all ranks of ``group``:
    returns the SeparationResult on ``dst`` (None elsewhere). Batches shard by
    mixture, single mixtures by bin; NCCL carries only the final gather.
    ``global_size=(M, F)``: ``y`` / ``init`` are this rank's shard already."""
    _, full = run_sharded("fast", y, init, iterations, group=group, dst=dst, runner=runner,
                          likelihood=compute_likelihood, dtype=dtype,
                          chunk_frames=chunk_frames, global_size=global_size)
    return None if full is None else _result("fast", full, y, init, iterations)


def fca_run_sharded(y, init, iterations, compute_likelihood=True, *, group=None, dst=0,
                    dtype="c128", runner=None, chunk_frames=None, global_size=None):
    """``fca_run`` (reference conventional.py:104-164) over all ranks of
    ``group`` (see :func:`fastfca_run_sharded`)."""
    _, full = run_sharded("fca", y, init, iterations, group=group, dst=dst, runner=runner,
                          likelihood=compute_likelihood, dtype=dtype,
                          chunk_frames=chunk_frames, global_size=global_size)
    return None if full is None else _result("fca", full, y, init, iterations)
