"""Multi-GPU partitioning of the EM path: one process per GPU, no collective
inside the EM loop.

Every EM quantity is per frequency bin (and per mixture): nothing couples
bins inside the loop (the reference is bitwise bin-shard
invariant). Batches are therefore split by mixture (config 3) and single
long mixtures by contiguous bin ranges (config 4). Each rank runs its shard
with the chunking the unsharded problem would use, so per-bin results are
bitwise identical to a 1-GPU run, and the only cross-GPU traffic is the final
gather of the per-rank results (NCCL over NVLink for CUDA tensors, gloo for
host tensors) in fixed rank order.
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

    @property
    def size(self):
        return self.stop - self.start


def plan_shard(M, F, rank, world):
    """Mixture shards for batches (M > 1), bin shards for one mixture."""
    if M > 1:
        return Shard("mixtures", *shard_range(M, rank, world))
    return Shard("bins", *shard_range(F, rank, world))


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
    "mixtures": {"images": 0, "v": 0, "S": 0, "loglik": 0},
    "bins": {"images": 3, "v": 3, "S": 2, "loglik": None},
}


def gather_results(local, shard, group=None, dst=0):
    """Gather per-rank result arrays to ``dst`` and concatenate in rank order.

    ``local``: dict of torch tensors (CUDA with NCCL, CPU with gloo) in the
    batched layouts. For bin shards the per-rank log-likelihood partial sums
    are added in rank order (fixed order: deterministic). Returns the full
    dict on ``dst`` and None elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    axes = RESULT_AXES[shard.axis]
    out = {} if rank == dst else None
    for key, t in local.items():
        if t is None:
            continue
        ax = axes.get(key)
        t = t.contiguous()
        if ax is None:  # summed partials (bin-sharded log-likelihood)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t, group=group)
            if rank == dst:
                acc = parts[0].clone()
                for p in parts[1:]:
                    acc += p
                out[key] = acc
            continue
        # variable shard sizes: exchange sizes, pad to the max, all_gather
        n = torch.tensor([t.shape[ax]], device=t.device, dtype=torch.int64)
        sizes = [torch.empty_like(n) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        sizes = [int(s.item()) for s in sizes]
        mx = max(sizes)
        pad_shape = list(t.shape)
        pad_shape[ax] = mx
        buf = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
        buf.narrow(ax, 0, t.shape[ax]).copy_(t)
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        if rank == dst:
            out[key] = torch.cat([p.narrow(ax, 0, s) for p, s in zip(parts, sizes)], dim=ax)
    return out
