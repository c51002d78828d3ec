#!/usr/bin/env python3
"""Benchmark: EM TF-bin·iterations/s of the B200 FCA / FastFCA path.

Workload (BASELINE.json configs[3], the largest single-GPU config the
headline is quoted on): a batch of 256 independent 2-source mixtures,
I=4, F=257, N=1250, L=20 EM iterations, complex128, FastFCA. One "step"
is one complete ``fastfca_run`` over the batch — initial pencil, L fused
iterations, separated images — with the likelihood off (the reference's
``em_seconds`` boundary excludes it). Mixtures are sharded across ranks
(``--gpus N`` under torchrun): no collective inside the EM loop.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--engine fast|fca] [--config 3] [--dtype c128|c64]

Prints ONE JSON line on rank 0. ``value`` is measured with inputs resident
in HBM; ``e2e`` goes through the public API with pinned host buffers (H2D of
y and the init, D2H of images, v and S inside the timed region);
``roofline`` is the fused FastFCA kernel's algorithmic bytes / its average
launch time (CUDA events around the kernel inside the run); ``cpu_baseline``
is the CPU oracle port timed on this host on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

from paper_1805_06572_b200.synth import CONFIGS, config_mixture, init_seed  # noqa: E402

PEAKS = REPO / "MEASURED_PEAKS.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--engine", choices=["fast", "fca"], default="fast")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--dtype", choices=["c128", "c64"], default="c128")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pageable", action="store_true", help="skip the numpy-input e2e leg")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra resident lines (config 3 complex64, config 4)")
    ap.add_argument("--no-other", action="store_true", help="skip the second engine")
    ap.add_argument("--streams", type=int, default=2,
                    help="concurrent streams over independent mixtures (batched configs)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="mixtures/bins in the CPU sample")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="strong (default): the config's batch is sharded over the ranks "
                         "(config 3 by mixture, single mixtures by bin) with one chunk plan "
                         "at every N; weak: every rank runs its own full config batch")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(cfg, rank, world, scaling="strong"):
    """strong: mixture shard for config-3 batches, bin shard for single
    mixtures (paper_1805_06572_b200.sharding); weak: rank r runs its own full
    config batch of independent mixtures r*M .. r*M + M-1 (no collective)."""
    from paper_1805_06572_b200.sharding import plan_shard

    if scaling == "weak":
        return ("mixtures", rank * cfg.M, (rank + 1) * cfg.M)
    sh = plan_shard(cfg.M, cfg.F, rank, world)
    return (sh.axis, sh.start, sh.stop)


def make_inputs(cfg, sh, threads=16):
    """This rank's shard: y (M,N,F,I) drawn on the host (seeded generator) and
    the reference init_random model computed by the package on the device.
    Returns host numpy arrays (y, v, S, floor)."""
    from paper_1805_06572_b200.initializers import init_random_batch
    from paper_1805_06572_b200.sharding import Shard, take

    kind, a, b = sh
    if kind == "mixtures":
        with ThreadPoolExecutor(threads) as ex:
            Y = np.stack(list(ex.map(lambda m: config_mixture(cfg, m), range(a, b))))
        model = init_random_batch(Y, [init_seed(cfg, m) for m in range(a, b)])
        return Y, model.v, model.S, model.v_floor
    y = config_mixture(cfg, 0)[None]
    model = init_random_batch(y, [init_seed(cfg, 0)])
    return take(Shard(kind, a, b), y, model.v, model.S, model.v_floor)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def config_dict(cfg, args, world):
    """The workload description both arms print (identical dicts)."""
    axis = "mixtures" if cfg.M > 1 else "bins"
    y_gb = cfg.M * cfg.N * cfg.F * cfg.I * (16 if args.dtype == "c128" else 8) / 1e9
    return {"workload": cfg.description, "engine": args.engine, "iterations": cfg.L,
            "M": cfg.M, "F": cfg.F, "N": cfg.N, "I": cfg.I, "dtype": args.dtype,
            "parallelism": (f"independent {cfg.M}-mixture batch per GPU x{world}"
                            if args.scaling == "weak" else f"{axis}-sharded x{world}"),
            "global_batch": cfg.M * (world if args.scaling == "weak" else 1),
            "l2": "inputs larger than L2 (y = %.2f GB)" % (y_gb * (world if args.scaling ==
                                                                   "weak" else 1))}


def peaks():
    try:
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_port_time(cfg, engine, sample, threads):
    """Time the CPU oracle port (C restatement with OpenMP when built, else the
    numpy restatement) on a bounded sample. Returns (tf_it_per_s, desc, kind, cores)."""
    from oracle import cpu_port

    return cpu_port.measure(cfg, engine, sample, threads)


def resident_line(ecfg, dtype, engine, steps, inputs=None):
    """One more resident-in-HBM measurement for the bench line's `extras`
    (1 GPU, one stream, graph replays of the whole run): value, ms per run
    and the update pass's roofline (CUDA events around each pass)."""
    import torch

    from paper_1805_06572_b200._engine import run_device, status_of, torch_types
    from paper_1805_06572_b200.sharding import shard_chunk_frames

    Y, V, S, FL = inputs if inputs is not None else make_inputs(ecfg, shard(ecfg, 0, 1))
    ctype, rtype = torch_types(dtype)
    y = torch.from_numpy(Y).cuda().to(ctype)
    v = torch.from_numpy(V).cuda().to(rtype)
    s0 = torch.from_numpy(S).cuda()
    fl = torch.from_numpy(FL).cuda()
    M, N, F, I = (int(x) for x in Y.shape)
    cf = shard_chunk_frames(ecfg.M, ecfg.N, ecfg.F, ecfg.I, dtype, engine,
                            max_world=ecfg.max_world)
    bufs = {"images": torch.empty((M, 2, N, F, I), dtype=ctype, device="cuda"),
            "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device="cuda"),
            "v": torch.empty_like(v)}

    def run(graph=True, kernel_timing=False):
        return run_device(engine, y, v, s0, fl, ecfg.L, likelihood=False, history=False,
                          images=True, dtype=dtype, timing=False, check=False, out=bufs,
                          chunk_frames=cf, graph=graph and not kernel_timing,
                          kernel_timing=kernel_timing,
                          # kernel events bracket ONE whole-grid pass launch per iteration
                          # (plain schedule), not the split-phase windows' stream waits
                          bin_parts=1 if kernel_timing else 0)

    r = run(graph=False)
    status_of(r, N, F)
    bufs["workspace"] = r.workspace
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        r = run()
    e1.record()
    torch.cuda.synchronize()
    status_of(r, N, F)
    ms = e0.elapsed_time(e1) / steps
    run(kernel_timing=True)  # (warm the stream-launched plain schedule once)
    kr = run(kernel_timing=True)
    status_of(kr, N, F)
    hot = kr.kernel_ms[:-1] if len(kr.kernel_ms) > 1 else kr.kernel_ms
    k_avg = statistics.mean(hot)
    rb = 8 if dtype == "c128" else 4
    alg = (2 * I + 4) * rb * M * F * N
    peak, peak_kind = peaks()
    ach = alg / (k_avg / 1e3) / 1e9
    out = {"workload": ecfg.description, "engine": engine, "dtype": dtype,
           "value": M * F * N * ecfg.L / (ms / 1e3), "unit": "TF-bin*it/s",
           "ms_per_step": round(ms, 4), "steps": steps, "chunk_frames": cf,
           "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                        "frac": round(ach / peak, 4), "algorithmic_bytes_per_launch": alg,
                        "kernel_ms_avg": round(k_avg, 4), "launches_averaged": len(hot),
                        "peak_source": peak_kind}}
    del y, v, s0, fl, bufs, r, kr
    torch.cuda.empty_cache()
    return out


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU implementation on this host's
    cores — the UNMODIFIED reference package (numba backend) from
    baseline/_ref, one warmed process per core (baseline/reference_numba.py);
    the C/OpenMP oracle port only when baseline/_ref is absent. Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    sys.path.insert(0, str(REPO / "baseline"))
    import reference_numba as RN

    vals = []
    extra = {}
    if RN.available():
        pool = RN.ReferencePool(cfg, args.engine, threads)
        try:
            iters = RN.sample_iterations(cfg, args.engine)
            for i in range(args.warmup + args.steps):
                v = pool.step(iters)
                if i >= args.warmup:
                    vals.append(v)
            extra["one_core"] = pool.one_core(iters)
            desc, kind, cores = RN.describe(cfg, args.engine, pool, iters), "reference", pool.cores
        finally:
            pool.close()
        if not args.no_cpu:  # the C/OpenMP restatement beside it (one sample)
            from oracle import cpu_port

            pv, pdesc, _, pcores = cpu_port.measure(cfg, args.engine, args.cpu_sample, threads)
            extra["port"] = {"value": pv, "cores": pcores, "sample": pdesc}
    else:
        from oracle import cpu_port

        for i in range(args.warmup + args.steps):
            v, desc, kind, cores = cpu_port.measure(cfg, args.engine, args.cpu_sample, threads)
            if i >= args.warmup:
                vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": f"EM TF-bin*iterations/s ({'FastFCA' if args.engine == 'fast' else 'FCA'}, config {cfg.index})",
        "value": value, "unit": "TF-bin*it/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": args.scaling,
        "dtype": args.dtype, "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": config_dict(cfg, args, world),
        "cpu_baseline": {"value": value, "unit": "TF-bin*it/s", "cores": cores, "kind": kind,
                         "sample": desc, **extra},
        "e2e": {"value": value, "unit": "TF-bin*it/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    # FFCA_DIST_BACKEND=gloo (functional checks of the N>1 code on fewer GPUs
    # than ranks; never a timing) maps ranks onto the visible devices
    backend = os.environ.get("FFCA_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_1805_06572_b200 import SpatialModel, fastfca_run, fca_run
    from paper_1805_06572_b200._engine import run_device, torch_types

    sh = shard(cfg, rank, world, args.scaling)
    Y, V, S, FL = make_inputs(cfg, sh)
    M, N, F, I = Y.shape
    L = cfg.L
    ctype, rtype = torch_types(args.dtype)
    dev = torch.device("cuda", local)
    y_d = torch.from_numpy(Y).to(dev).to(ctype)
    v_d = torch.from_numpy(V).to(dev).to(rtype)
    S_d = torch.from_numpy(S).to(dev)
    fl_d = torch.from_numpy(FL).to(dev)
    # ONE frame chunking at every world size (the plan that fills a GPU with
    # the 8-rank shard) -> bitwise-identical per-bin results at N = 1..8
    from paper_1805_06572_b200._engine import plan_chunks
    from paper_1805_06572_b200.sharding import grid_model, plan_shard, shard_chunk_frames

    if args.scaling == "strong":
        cf = shard_chunk_frames(cfg.M, cfg.N, cfg.F, cfg.I, args.dtype, args.engine, max_world=cfg.max_world)
    else:
        cf, _ = plan_chunks(cfg.M * cfg.F, cfg.N, cfg.I, args.dtype, args.engine)
    G_rank = M * F
    sh8 = plan_shard(cfg.M, cfg.F, 0, cfg.max_world)
    grid = {"chunk_frames": cf, "this_rank": grid_model(G_rank, N, I, cf, args.dtype, args.engine),
            f"rank0_at_{cfg.max_world}_gpus": grid_model(
                sh8.size * (cfg.F if sh8.axis == "mixtures" else 1), N, I, cf, args.dtype,
                args.engine)}
    tf_it_rank = M * F * N * L
    # whole-job units: all ranks' mixtures (weak) or the one sharded batch (strong)
    tf_it_total = cfg.M * cfg.F * cfg.N * L * (world if args.scaling == "weak" else 1)

    from paper_1805_06572_b200._engine import status_of

    # outputs and workspace are allocated once: a step is the EM run, not cudaMalloc
    bufs = {"images": torch.empty((M, 2, N, F, I), dtype=ctype, device=dev),
            "S": torch.empty((M, 2, F, I, I), dtype=torch.complex128, device=dev),
            "v": torch.empty_like(v_d)}

    def step(timing=False):  # untimed-event steps replay a cached CUDA graph of the run
        return run_device(args.engine, y_d, v_d, S_d, fl_d, L, likelihood=False, history=False,
                          images=True, dtype=args.dtype, timing=timing, check=False,
                          chunk_frames=cf, kernel_timing=timing, out=bufs, graph=not timing,
                          bin_parts=1 if timing else 0)  # (kernel events: whole-grid passes)

    bufs["workspace"] = step().workspace
    nstreams = args.streams if M > 1 else 1
    if nstreams > 1:  # independent mixtures on concurrent streams (hides K1 and wave tails)
        from paper_1805_06572_b200._engine import run_device_streams

        sstreams = [torch.cuda.Stream() for _ in range(nstreams)]
        first = run_device_streams(args.engine, y_d, v_d, S_d, fl_d, L, nstreams=nstreams,
                                   out=bufs, likelihood=False, history=False, images=True,
                                   dtype=args.dtype, timing=False, check=False,
                                   chunk_frames=cf, streams=sstreams)
        torch.cuda.synchronize()
        wss = [r.workspace for r in first.parts]
        for r in first.parts:
            status_of(r, N, F)
        plain_step = step

        def step(timing=False):  # noqa: F811
            if timing:
                return plain_step(timing=True)
            return run_device_streams(args.engine, y_d, v_d, S_d, fl_d, L, nstreams=nstreams,
                                      out=bufs, workspaces=wss, likelihood=False, history=False,
                                      images=True, dtype=args.dtype, timing=False, check=False,
                                      chunk_frames=cf, streams=sstreams, graph=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(args.steps):
            last = step()
        end.record()
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    from paper_1805_06572_b200._engine import status_of

    for r in (last.parts if hasattr(last, "parts") else [last]):
        status_of(r, N, F)
    del last
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = tf_it_total / (ms_per_step / 1e3)

    # dominant-kernel roofline: events around each fused pass inside one run
    kr = step(timing=True)
    from paper_1805_06572_b200._engine import status_of as _st

    _st(kr, N, F)
    # launches 0..L-2 are the update-only pass (the dominant kernel); the last
    # one also writes the 10.5 GB of images and is reported on its own
    k_ms = kr.kernel_ms
    hot = k_ms[:-1] if len(k_ms) > 1 else k_ms
    k_avg = statistics.mean(hot) if hot else float("nan")
    r = 8 if args.dtype == "c128" else 4  # bytes per real
    bytes_per_tf = (2 * I + 4) * r  # read y (I complex), read v (2), write v (2)
    alg_bytes = bytes_per_tf * M * F * N
    achieved = alg_bytes / (k_avg / 1e3) / 1e9
    peak, peak_kind = peaks()
    traffic, traffic_src = None, None
    try:  # dram read+write per launch from the committed ncu --set full capture
        tj = json.loads((REPO / "profiles" / "traffic.json").read_text())
        for k, rec in tj.items():
            if (args.engine == "fast" and args.dtype == "c128" and world == 1
                    and f"config {cfg.index} " in k and "c128" in k):
                traffic = rec["dram_bytes_per_launch"]
                traffic_src = rec["source"]
    except Exception:
        traffic, traffic_src = None, None
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_source": traffic_src, "algorithmic_bytes_per_launch": alg_bytes,
            "kernel": ("fast_em2_kernel (update pass)" if args.engine == "fast"
                       else "fca_em_kernel (update pass)"),
            "kernel_ms_avg": round(k_avg, 4), "launches_averaged": len(hot),
            "last_pass_with_images_ms": round(k_ms[-1], 4) if k_ms else None,
            "bytes_per_tf_bin": bytes_per_tf,
            "peak_source": peak_kind,
            "iteration_ms_avg": round(statistics.mean(kr.iteration_ms), 4) if kr.iteration_ms
            else None}
    del kr
    torch.cuda.empty_cache()

    # end-to-end through the public API with pinned host buffers
    e2e = None
    e2e_more = {}
    if not args.no_e2e:
        yh = torch.from_numpy(Y).to(ctype).pin_memory()
        vh = torch.from_numpy(V).to(rtype).pin_memory()
        Sh = torch.from_numpy(S).pin_memory()
        flh = torch.from_numpy(FL).pin_memory()
        model = SpatialModel(v=vh, S=Sh, v_floor=flh)
        run = fastfca_run if args.engine == "fast" else fca_run
        kw = dict(compute_likelihood=False, device_output=False, dtype=args.dtype,
                  chunk_frames=cf)

        def nbytes(*ts):
            return int(sum(t.numel() * t.element_size() for t in ts))

        def over_ranks(x, op):
            t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=op)
            return float(t.item())

        def timed(fn, reps):
            fn()  # warm (pinned pools, graphs, NCCL communicators)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                r = fn()
                ts.append(time.perf_counter() - t0)
                del r
            return over_ranks(statistics.median(ts), dist.ReduceOp.MAX if world > 1 else None)

        reps = max(1, min(args.steps, 3))
        res = run(yh, model, L, **kw)
        h2d = over_ranks(nbytes(yh, vh, Sh, flh), dist.ReduceOp.SUM if world > 1 else None)
        d2h = over_ranks(sum(np.asarray(a).nbytes for a in (res.images, res.model.v,
                                                             res.model.S)),
                         dist.ReduceOp.SUM if world > 1 else None)
        del res  # results go back to the pinned cache: steady state, not cudaHostAlloc
        # (1) every rank: public fastfca_run on its own shard, pinned host in -> pinned host out
        t_sh = timed(lambda: run(yh, model, L, **kw), reps)
        shards_line = {"value": tf_it_total / t_sh, "unit": "TF-bin*it/s",
                       "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                       "s_per_step": round(t_sh, 4)}
        if world > 1 and args.scaling == "strong":
            # (2) the sharded public entry point: per-rank H2D of its shard, the
            # run, the NCCL gather of images / v / S / floor to rank 0's GPU and
            # rank 0's D2H of the whole result
            from paper_1805_06572_b200.sharding import fastfca_run_sharded, fca_run_sharded

            srun = fastfca_run_sharded if args.engine == "fast" else fca_run_sharded
            t_g = timed(lambda: srun(yh, model, L, compute_likelihood=False, dtype=args.dtype,
                                     chunk_frames=cf, global_size=(cfg.M, cfg.F)), reps)
            e2e = {"value": tf_it_total / t_g, "unit": "TF-bin*it/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "s_per_step": round(t_g, 4),
                   "path": "fastfca_run_sharded: per-rank H2D + run, NCCL gather to rank 0, "
                           "rank-0 D2H"}
            e2e_more["e2e_host_shards"] = dict(shards_line, path="per-rank fastfca_run on its "
                                               "shard, pinned host in/out (no gather)")
        else:
            e2e = dict(shards_line, path="fastfca_run, pinned host buffers (pipelined "
                                         "H2D / run / D2H)")
        if world == 1 and not args.no_pageable:
            # (3) a numpy caller: pageable host arrays in, numpy out
            model_np = SpatialModel(v=V.astype(np.float64 if args.dtype == "c128" else
                                               np.float32), S=S, v_floor=FL)
            Yc = Y if args.dtype == "c128" else Y.astype(np.complex64)
            t_pg = timed(lambda: run(Yc, model_np, L, **kw), 1)
            e2e_more["e2e_pageable"] = {"value": tf_it_total / t_pg, "unit": "TF-bin*it/s",
                                        "s_per_step": round(t_pg, 4),
                                        "path": "fastfca_run, numpy (pageable) inputs"}
            del Yc, model_np
        del yh, vh, Sh, flh, model

    # the other engine on the same resident inputs (the metric names both)
    other = "fca" if args.engine == "fast" else "fast"
    other_line = None
    if not args.no_other:
        ocf = (shard_chunk_frames(cfg.M, cfg.N, cfg.F, cfg.I, args.dtype, other, max_world=cfg.max_world)
               if args.scaling == "strong" else
               plan_chunks(cfg.M * cfg.F, cfg.N, cfg.I, args.dtype, other)[0])
        obufs = {"images": bufs["images"], "S": bufs["S"], "v": bufs["v"]}

        def ostep():
            return run_device(other, y_d, v_d, S_d, fl_d, L, likelihood=False, history=False,
                              images=True, dtype=args.dtype, timing=False, check=False,
                              chunk_frames=ocf, out=obufs)

        r0 = ostep()
        status_of(r0, N, F)
        obufs["workspace"] = r0.workspace
        del r0
        osteps = max(2, args.steps // 2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        o0 = torch.cuda.Event(enable_timing=True)
        o1 = torch.cuda.Event(enable_timing=True)
        o0.record()
        for _ in range(osteps):
            last = ostep()
        o1.record()
        torch.cuda.synchronize()
        status_of(last, N, F)
        del last
        ot = torch.tensor([o0.elapsed_time(o1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ot, op=dist.ReduceOp.MAX)
        oms = float(ot.item()) / osteps
        other_line = {"engine": other, "value": tf_it_total / (oms / 1e3),
                      "unit": "TF-bin*it/s", "ms_per_step": oms, "steps": osteps}
        del obufs

    # the other headline lines on this GPU: config 3 complex64 (same draw, cast)
    # and config 4 complex128, each with its own roofline block
    extras = None
    if (world == 1 and not args.no_extras and cfg.index == 3 and args.dtype == "c128"
            and args.engine == "fast"):
        del y_d, v_d, S_d, fl_d, bufs
        torch.cuda.empty_cache()
        extras = {"config3_c64": resident_line(cfg, "c64", "fast", max(2, args.steps // 2),
                                               inputs=(Y, V, S, FL)),
                  "config4_c128": resident_line(CONFIGS[4], "c128", "fast",
                                                max(2, args.steps // 2))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the unmodified reference (numba, baseline/_ref) on all host cores and
        # on one core, and the C/OpenMP oracle port beside it
        threads = len(os.sched_getaffinity(0))
        v_cpu, desc, kind, cores = cpu_port_time(cfg, args.engine, args.cpu_sample, threads)
        port = {"value": v_cpu, "unit": "TF-bin*it/s", "cores": cores, "kind": kind,
                "sample": desc}
        cpu = port
        sys.path.insert(0, str(REPO / "baseline"))
        import reference_numba as RN

        if RN.available():
            r = RN.measure(cfg, args.engine, threads)
            cpu = {"value": r["all_cores"], "unit": "TF-bin*it/s", "cores": r["cores"],
                   "kind": "reference", "sample": r["sample"], "one_core": r["one_core"],
                   "cpu_model": r["cpu_model"], "port": port}

    # status init + initial pencil + L x (fused pass + pencil), per concurrent part
    launches_per_step = (2 + 2 * L) * nstreams
    if rank == 0:
        line = {
            "metric": f"EM TF-bin*iterations/s ({'FastFCA' if args.engine == 'fast' else 'FCA'}, config {cfg.index})",
            "value": value, "unit": "TF-bin*it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded, BASELINE.json recipe)",
            "config": config_dict(cfg, args, world),
            "layout": {"streams_per_gpu": nstreams, "shard": list(sh), "grid": grid},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, **e2e_more,
            ("fca" if other == "fca" else "fastfca"): other_line,
            "extras": extras,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
