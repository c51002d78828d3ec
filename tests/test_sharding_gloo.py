"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic:
shard planning, per-rank slicing, and the fixed-order final gather. The
per-rank EM here is the CPU oracle (tests may use it as the checker); the
claim tested is that sharding + gather reproduce the unsharded run exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1805_06572_b200.sharding import plan_shard, shard_range, take


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_range_partitions():
    for total in (1, 7, 256, 1025):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_plan_shard_axes():
    assert plan_shard(256, 257, 1, 8).axis == "mixtures"
    assert plan_shard(1, 1025, 7, 8) .axis == "bins"
    assert plan_shard(1, 1025, 7, 8).stop == 1025


def _instance(M, N, F, I, seed):
    from oracle import fastfca_oracle as O

    gen = np.random.default_rng(seed)
    y = gen.standard_normal((M, N, F, I)) + 1j * gen.standard_normal((M, N, F, I))
    inits = [O.init_random(y[m], seed + m) for m in range(M)]
    return (y, np.stack([i[0] for i in inits]), np.stack([i[1] for i in inits]),
            np.stack([i[2] for i in inits]))


def _worker(rank, world, port, M, result_q):
    import torch
    import torch.distributed as dist

    from oracle import fastfca_oracle as O
    from paper_1805_06572_b200.sharding import gather_results

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    y, v, S, fl = _instance(M, 24, 9, 3, 5)
    sh = plan_shard(M, y.shape[2], rank, world)
    ys, vs, Ss, fs = take(sh, y, v, S, fl)
    imgs, vv, SS, lls = [], [], [], []
    for m in range(ys.shape[0]):
        r = O.fastfca_run(ys[m], vs[m], Ss[m], fs[m], 4)
        imgs.append(r.images)
        vv.append(r.v)
        SS.append(r.S)
        lls.append(r.loglik_trace)
    local = {"images": torch.from_numpy(np.stack(imgs)), "v": torch.from_numpy(np.stack(vv)),
             "S": torch.from_numpy(np.stack(SS))}
    if sh.axis == "mixtures":
        local["loglik"] = torch.from_numpy(np.asarray(lls))
    out = gather_results(local, sh)
    if rank == 0:
        result_q.put({k: v.numpy() for k, v in out.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M", [3, 1])
def test_two_rank_gather_reproduces_unsharded_run(M):
    from oracle import fastfca_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    y, v, S, fl = _instance(M, 24, 9, 3, 5)
    for m in range(M):
        ref = O.fastfca_run(y[m], v[m], S[m], fl[m], 4)
        assert np.array_equal(out["images"][m], ref.images)
        assert np.array_equal(out["v"][m], ref.v)
        assert np.array_equal(out["S"][m], ref.S)
        if M > 1:
            assert np.array_equal(out["loglik"][m], np.asarray(ref.loglik_trace))
