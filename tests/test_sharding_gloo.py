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


def _worker(rank, world, port, M, algorithm, result_q, local=False):
    import torch.distributed as dist

    from paper_1805_06572_b200 import SpatialModel
    from paper_1805_06572_b200.sharding import fastfca_run_sharded, fca_run_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    y, v, S, fl = _instance(M, 24, 9, 3, 5)
    if M == 1:  # one mixture in the reference shape -> bin shards
        y, v, S, fl = y[0], v[0], S[0], fl[0]
    run = fastfca_run_sharded if algorithm == "fast" else fca_run_sharded
    if local:  # each rank holds only its own shard (global_size names the whole problem)
        Mg, Fg = (M, y.shape[-2])
        sh = plan_shard(Mg, Fg, rank, world)
        yb, vb, Sb, fb = (x if M > 1 else x[None] for x in (y, v, S, fl))
        ys, vs, Ss, fs = take(sh, yb, vb, Sb, fb)
        if M == 1:
            ys, vs, Ss, fs = ys[0], vs[0], Ss[0], fs[0]
        res = run(ys, SpatialModel(v=vs, S=Ss, v_floor=fs), 4, runner=_oracle_runner, dst=0,
                  global_size=(Mg, Fg))
    else:
        init = SpatialModel(v=v, S=S, v_floor=fl)
        # the real entry point: shard planning, per-rank slicing, the gather
        res = run(y, init, 4, runner=_oracle_runner, dst=0)
    if rank == 0:
        result_q.put({"images": res.images, "v": res.model.v, "S": res.model.S,
                      "floor": res.model.v_floor, "loglik": np.asarray(res.loglik_trace)})
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M,algorithm,local", [(3, "fast", False), (1, "fast", False),
                                               (3, "fca", False), (1, "fca", False),
                                               (3, "fast", True), (1, "fca", True)])
def test_two_rank_sharded_run_reproduces_unsharded_run(M, algorithm, local):
    from oracle import fastfca_oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, algorithm, q, local)) for r in range(2)]
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
        assert np.array_equal(out["floor"][m] if M > 1 else out["floor"], fl[m])
        if M > 1:
            assert np.array_equal(got["loglik"], np.asarray(ref.loglik_trace))
        else:  # bin shards: per-rank partial sums added in rank order
            assert np.allclose(got["loglik"], np.asarray(ref.loglik_trace), rtol=1e-12, atol=0)


@pytest.mark.parametrize("M", [1, 3])
def test_more_ranks_than_units(M):
    """World sizes above the unit count leave some ranks an empty shard; their
    zero-size results (and zero likelihood partials) still concatenate to the
    unsharded run (per-rank compute: the oracle)."""
    import torch

    from paper_1805_06572_b200 import SpatialModel
    from paper_1805_06572_b200.sharding import run_shard

    F = 3 if M == 1 else 9
    y, v, S, fl = _instance(M, 16, F, 2, 9)
    if M == 1:
        y, v, S, fl = y[0], v[0], S[0], fl[0]
    init = SpatialModel(v=v, S=S, v_floor=fl)
    _, one = run_shard("fast", y, init, 3, 0, 1, runner=_oracle_runner)
    world = 5
    parts = [run_shard("fast", y, init, 3, r, world, runner=_oracle_runner)[1]
             for r in range(world)]
    assert sum(1 for p in parts if p["v"].numel() == 0) == world - (F if M == 1 else M)
    ax = {"images": 3, "v": 3, "S": 2} if M == 1 else {"images": 0, "v": 0, "S": 0, "loglik": 0}
    for key, a in ax.items():
        assert torch.equal(torch.cat([p[key] for p in parts], dim=a), one[key]), key
    if M == 1:
        tot = sum(p["loglik"] for p in parts)
        assert torch.allclose(tot, one["loglik"], rtol=1e-12, atol=0)
