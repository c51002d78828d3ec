"""CPU baseline leg: the UNMODIFIED reference package, numba backend.

The reference (``fastfca`` 0.1.0, ``/root/reference/pkg``) is installed into
``baseline/_ref`` (git-ignored, travels to the GPU box with the snapshot) by

    cp -r /root/reference/pkg /tmp/refsrc
    python -m pip install --no-index --no-build-isolation --no-deps \\
        --find-links /opt/wheelhouse --target baseline/_ref /tmp/refsrc

and timed here through its own public API — ``fastfca.fast.fastfca_run`` /
``fastfca.conventional.fca_run`` with ``FASTFCA_BACKEND=numba`` and
``compute_likelihood=False`` — on its own ``em_seconds`` boundary, warmed
first (the template is ``pkg/benchmarks/backend_bench.py:22-28``), BLAS
limited to one thread per process (``threadpoolctl``). Two legs, as SURVEY.md
§8(d) prescribes:

* 1 core: one work unit in this process;
* all cores: one process per core (``multiprocessing``), each running its own
  unit — a different mixture (batched configs) or a different contiguous
  bin block (single mixtures; bins never couple, so a bin block is an exact
  share of the run) — throughput = total TF-bin*it / the slowest process's
  ``em_seconds``.

Inputs are this repo's seeded synthetic mixtures (``synth.py``, numpy on the
host) and the REFERENCE's ``init_random``; nothing of this repo's EM path is
imported. Samples are bounded (a mixture, or a bin block, and for FCA a few
iterations: every iteration does the same work) so the leg ends in tens of
seconds. Test infrastructure / baseline only: the product never imports it.
"""

from __future__ import annotations

import os
import platform
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF = REPO / "baseline" / "_ref"


def available():
    return (REF / "fastfca" / "__init__.py").exists()


def _setup():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ffca_numba_cache")
    os.environ["FASTFCA_BACKEND"] = "numba"
    for p in (str(REF), str(REPO)):
        if p not in sys.path:
            sys.path.insert(0, p)


def _unit(cfg_index, u, bins_per_unit):
    """Work unit ``u``: mixture ``u`` (batched) or bin block ``u`` (one mixture)."""
    import numpy as np

    from paper_1805_06572_b200.synth import CONFIGS, config_mixture, init_seed

    cfg = CONFIGS[cfg_index]
    if cfg.M > 1:
        return config_mixture(cfg, u % cfg.M), init_seed(cfg, u % cfg.M)
    nblk = max(1, cfg.F // bins_per_unit)
    b0 = (u % nblk) * bins_per_unit
    y = config_mixture(cfg, 0, bins=np.arange(b0, b0 + bins_per_unit))
    return y, init_seed(cfg, 0)


def _load_unit(cfg_index, engine, u, bins_per_unit):
    """Import the reference (numba backend, 1 BLAS thread), build unit ``u``'s
    input and the reference init, warm the compiled kernels. Returns a
    callable running ``iters`` iterations -> (em_seconds, TF-bin*it)."""
    _setup()
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    import fastfca
    from fastfca import _backend
    from fastfca.conventional import fca_run
    from fastfca.fast import fastfca_run
    from fastfca.initializers import init_random

    assert Path(fastfca.__file__).resolve().is_relative_to(REF.resolve()), fastfca.__file__
    _backend.select_backend("numba")
    run = fastfca_run if engine == "fast" else fca_run
    y, seed = _unit(cfg_index, u, bins_per_unit)
    init = init_random(y, seed)
    run(y, init, 1, compute_likelihood=False)  # warm the compiled kernels
    N, F, _ = y.shape

    def go(iters):
        res = run(y, init, iters, compute_likelihood=False)
        return res.em_seconds, N * F * iters

    go.backend = _backend.backend_name()
    return go


def _worker(conn, cfg_index, engine, u, bins_per_unit):
    try:
        go = _load_unit(cfg_index, engine, u, bins_per_unit)
        conn.send(("ready", go.backend))
        while True:
            msg = conn.recv()
            if msg is None:
                break
            conn.send(go(int(msg)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        conn.send(("error", repr(e)))
    finally:
        conn.close()


class ReferencePool:
    """One warmed reference process per core, each owning one work unit;
    ``step(iters)`` runs all of them once and returns the all-core
    TF-bin*it/s (total work / slowest process's em_seconds)."""

    def __init__(self, cfg, engine, cores=None):
        import multiprocessing as mp

        _setup()
        self.cores = int(cores or len(os.sched_getaffinity(0)))
        self.bpu = _bins_per_unit(cfg, engine)
        # compile once here (fills the on-disk JIT cache the workers load)
        self.local = _load_unit(cfg.index, engine, 0, self.bpu)
        self.backend = self.local.backend
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for u in range(self.cores):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_worker, args=(b, cfg.index, engine, u, self.bpu),
                             daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        for c in self.conns:
            msg = c.recv()
            if msg[0] != "ready":
                raise RuntimeError(f"reference worker failed: {msg[1]}")

    def one_core(self, iters):
        em, tf = self.local(iters)
        return tf / em

    def step(self, iters):
        for c in self.conns:
            c.send(iters)
        res = [c.recv() for c in self.conns]
        return sum(r[1] for r in res) / max(r[0] for r in res)

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except OSError:
                pass
        for pr in self.procs:
            pr.join(10)


def _bins_per_unit(cfg, engine):
    # single-mixture configs: a bin block of ~2-4 s of one-core work
    if cfg.M > 1:
        return 0
    per_bin_it = cfg.N * (cfg.I ** 2) * (1.0 if engine == "fast" else 7.0)  # rough cost
    return int(max(1, min(cfg.F, round(3e7 / per_bin_it / max(cfg.L, 1)))))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def sample_iterations(cfg, engine):
    """Iterations per timed sample (every iteration does the same work)."""
    return cfg.L if engine == "fast" else min(cfg.L, 2)


def describe(cfg, engine, pool, iters):
    unit = (f"1 mixture ({cfg.F} bins x {cfg.N} frames)" if cfg.M > 1 else
            f"{pool.bpu} bins x {cfg.N} frames")
    return (f"unmodified reference fastfca 0.1.0 ({pool.backend} backend, "
            f"{'fastfca_run' if engine == 'fast' else 'fca_run'}, compute_likelihood=False, "
            f"em_seconds): {pool.cores} processes x {unit} x {iters} iterations, 1 BLAS "
            f"thread each; CPU {cpu_model()}")


def measure(cfg, engine, cores=None, reps=1):
    """Time the reference on ``cfg``. Returns a dict with the 1-core and
    all-core TF-bin*it/s, the sample description, core count and CPU model."""
    t0 = time.perf_counter()
    pool = ReferencePool(cfg, engine, cores)
    try:
        iters = sample_iterations(cfg, engine)
        one = pool.one_core(iters)
        allc = max(pool.step(iters) for _ in range(reps))
        return {"one_core": one, "all_cores": allc, "cores": pool.cores,
                "backend": pool.backend, "cpu_model": cpu_model(),
                "sample": describe(cfg, engine, pool, iters),
                "wall_s": round(time.perf_counter() - t0, 1)}
    finally:
        pool.close()


if __name__ == "__main__":
    import json

    _setup()
    from paper_1805_06572_b200.synth import CONFIGS

    c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    e = sys.argv[2] if len(sys.argv) > 2 else "fast"
    print(json.dumps(measure(CONFIGS[c], e)))
