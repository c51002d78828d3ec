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


def _oracle_runner(algorithm, ys, vs, Ss, fs, L, *, chunk_frames, likelihood, images, dtype):
    """Per-rank compute for the CPU test: the oracle (the checker) in place of
    the CUDA run, same inputs and result layout as sharding._device_runner."""
    import torch

    from oracle import fastfca_oracle as O

    run = O.fastfca_run if algorithm == "fast" else O.fca_run
    imgs, vv, SS, lls = [], [], [], []
    for m in range(ys.shape[0]):
        r = run(ys[m], vs[m], Ss[m], fs[m], L, compute_likelihood=likelihood)
        imgs.append(r.images)
        vv.append(r.v)
        SS.append(r.S)
        lls.append(r.loglik_trace)
    return {"images": torch.from_numpy(np.stack(imgs)), "v": torch.from_numpy(np.stack(vv)),
            "S": torch.from_numpy(np.stack(SS)),
            "loglik": torch.from_numpy(np.asarray(lls, dtype=np.float64)) if likelihood
            else None}


def _worker(rank, world, port, M, algorithm, result_q):
    import torch.distributed as dist

    from paper_1805_06572_b200 import SpatialModel
    from paper_1805_06572_b200.sharding import fastfca_run_sharded, fca_run_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    y, v, S, fl = _instance(M, 24, 9, 3, 5)
    if M == 1:  # one mixture in the reference shape -> bin shards
        y, v, S, fl = y[0], v[0], S[0], fl[0]
    init = SpatialModel(v=v, S=S, v_floor=fl)
    run = fastfca_run_sharded if algorithm == "fast" else fca_run_sharded
    # the real entry point: shard planning, per-rank slicing, the gather
    res = run(y, init, 4, runner=_oracle_runner, dst=0)
    if rank == 0:
        result_q.put({"images": res.images, "v": res.model.v, "S": res.model.S,
                      "loglik": np.asarray(res.loglik_trace)})
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M,algorithm", [(3, "fast"), (1, "fast"), (3, "fca"), (1, "fca")])
def test_two_rank_sharded_run_reproduces_unsharded_run(M, algorithm):
    from oracle import fastfca_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, algorithm, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    y, v, S, fl = _instance(M, 24, 9, 3, 5)
    orun = O.fastfca_run if algorithm == "fast" else O.fca_run
    for m in range(M):
        ref = orun(y[m], v[m], S[m], fl[m], 4)
        got = {k: (out[k][m] if M > 1 else out[k]) for k in ("images", "v", "S", "loglik")}
        # per-bin quantities are exact (bins never couple)
        assert np.array_equal(got["images"], ref.images)
        assert np.array_equal(got["v"], ref.v)
        assert np.array_equal(got["S"], ref.S)
        if M > 1:
            assert np.array_equal(got["loglik"], np.asarray(ref.loglik_trace))
        else:  # bin shards: per-rank partial sums added in rank order
            assert np.allclose(got["loglik"], np.asarray(ref.loglik_trace), rtol=1e-12, atol=0)
