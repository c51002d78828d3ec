"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference package ``fastfca`` (``/root/reference/pkg/src``).

Run once in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs (``*.npz``, committed):

* ``runs_<name>.npz`` — inputs (y, init v/S/floor, L) and the reference's
  outputs of ``fastfca_run`` and ``fca_run`` with ``record_history=True``:
  images, final v and S, the log-likelihood trace, per-iteration S history
  (and v history where small), op counts.
* ``kernels.npz`` — the 11 kernel-contract functions of the reference numba
  backend (``_kernels_numba.py``) on one random instance.
* ``pencils.npz`` — ``gevd_hpd`` on random pencils of order 2..8.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from fastfca import _backend  # noqa: E402
from fastfca.conventional import fca_run  # noqa: E402
from fastfca.fast import fastfca_run  # noqa: E402
from fastfca.initializers import init_random  # noqa: E402
from fastfca.pencil import gevd_hpd  # noqa: E402
from fastfca import _kernels_numba as KN  # noqa: E402

from paper_1805_06572_b200.synth import CONFIGS, config_mixture, init_seed  # noqa: E402

from tests.instances import kernel_instance  # noqa: E402


def run_case(name, y, init_seed_, L, keep_v_history=False, image_stride=1):
    init = init_random(y, seed=init_seed_)
    out = {
        "y": y,
        "v0": init.v,
        "S0": init.S,
        "floor": init.v_floor,
        "L": np.int64(L),
        "init_seed": np.int64(init_seed_),
        "image_stride": np.int64(image_stride),
    }
    for tag, run in (("fast", fastfca_run), ("fca", fca_run)):
        res = run(y, init, L, record_history=True, compute_likelihood=True)
        out[f"{tag}_images"] = res.images[:, ::image_stride]
        out[f"{tag}_v"] = res.model.v
        out[f"{tag}_S"] = res.model.S
        out[f"{tag}_ll"] = np.asarray(res.loglik_trace)
        out[f"{tag}_Shist"] = np.stack([h["S"] for h in res.history]) if L else np.zeros(0)
        if keep_v_history and L:
            out[f"{tag}_vhist"] = np.stack([h["v"] for h in res.history])
        oc = res.op_counts
        out[f"{tag}_counts"] = np.array(
            [oc.frame_matrix_inversions, oc.frame_matrix_products, oc.bin_gevd_count,
             oc.bin_matrix_products], dtype=np.int64)
    np.savez_compressed(HERE / f"runs_{name}.npz", **out)
    print(f"{name}: y{y.shape} L={L} ll_fast[-1]={out['fast_ll'][-1]:.6f}")


def main():
    _backend.select_backend("numba")
    # acceptance-style instances (reference tests/test_acceptance.py:38-52)
    for k, I in enumerate((2, 3, 4)):
        gen = np.random.default_rng(9000 + k)
        y = gen.standard_normal((64, 33, I)) + 1j * gen.standard_normal((64, 33, I))
        run_case(f"acc{k}", y, 100 + k, 10, keep_v_history=(k == 0))
    # L = 0 and L = 1 edge cases
    gen = np.random.default_rng(4242)
    y = gen.standard_normal((16, 5, 3)) + 1j * gen.standard_normal((16, 5, 3))
    run_case("l0", y, 7, 0)
    run_case("l1", y, 7, 1, keep_v_history=True)
    # ragged: a single frame, a single bin
    gen = np.random.default_rng(4343)
    y = gen.standard_normal((1, 7, 2)) + 1j * gen.standard_normal((1, 7, 2))
    run_case("oneframe", y, 8, 3, keep_v_history=True)
    y = gen.standard_normal((40, 1, 4)) + 1j * gen.standard_normal((40, 1, 4))
    run_case("onebin", y, 9, 5, keep_v_history=True)
    # BASELINE config subsets (bins are independent: bin-shard invariance)
    subsets = {
        0: dict(bins=[0, 1, 100, 256]),
        1: dict(bins=[0, 257, 512]),
        2: dict(bins=[0, 300], image_stride=2),
        4: dict(bins=[511], image_stride=10),
    }
    for idx, spec in subsets.items():
        cfg = CONFIGS[idx]
        y = config_mixture(cfg, 0, bins=spec["bins"])
        run_case(f"cfg{idx}", y, init_seed(cfg, 0), cfg.L,
                 image_stride=spec.get("image_stride", 1))
    cfg = CONFIGS[3]
    for m in (0, 1):
        y = config_mixture(cfg, m, bins=[5, 200])
        run_case(f"cfg3m{m}", y, init_seed(cfg, m), cfg.L)

    # kernel contract (reference tests/test_backend.py:16-22 instance shape)
    y, v, S, P, lam = kernel_instance()
    floor = np.full(y.shape[1], 1e-3)
    kout = {"y": y, "v": v, "S": S, "P": P, "lam": lam, "floor": floor}
    mu, Phi, ninv, nprod = KN.fca_e_step(y, v, S)
    kout.update(fca_e_mu=mu, fca_e_Phi=Phi, fca_e_counts=np.array([ninv, nprod]))
    kout["fca_v"] = KN.fca_v_update(Phi, S)
    kout["fca_S"] = KN.fca_S_update(Phi, kout["fca_v"])
    kout["fca_ll"] = np.float64(KN.fca_log_likelihood(y, v, S))
    yt = KN.fast_transform(y, P)
    kout["yt"] = yt
    mu_t, Phi_t, _, _ = KN.fast_e_step(yt, v, lam)
    kout.update(fast_e_mu=mu_t, fast_e_Phi=Phi_t)
    kout["fast_v"] = KN.fast_v_update(Phi_t, lam)
    kout["fast_S"] = KN.fast_S_update(Phi_t, kout["fast_v"])
    logdet2 = np.linspace(-0.5, 0.7, y.shape[1])
    kout["logdet2"] = logdet2
    kout["fast_ll"] = np.float64(KN.fast_log_likelihood(yt, v, lam, logdet2))
    L_ = np.linalg.cholesky(S)
    Li = np.linalg.inv(L_)
    Sinv = np.conj(np.swapaxes(Li, -1, -2)) @ Li
    kout["Sinv"] = Sinv
    mu, vn, Sr, ninv, nprod = KN.fca_iteration(y, v, S, Sinv, floor)
    kout.update(fca_it_mu=mu, fca_it_v=vn, fca_it_S=Sr, fca_it_counts=np.array([ninv, nprod]))
    mu, vn, Sr, _, _ = KN.fast_iteration(y, P, v, lam, floor)
    kout.update(fast_it_mu=mu, fast_it_v=vn, fast_it_S=Sr)
    np.savez_compressed(HERE / "kernels.npz", **kout)
    print("kernels: done")

    # pencils (reference tests/test_acceptance.py:97-154 recipe, orders 2..8)
    gen = np.random.default_rng(777)
    pout = {}
    for count in range(140):
        d = 2 + count % 7
        a = gen.standard_normal((d, d)) + 1j * gen.standard_normal((d, d))
        phi = 0.5 * (a + a.conj().T)
        b = gen.standard_normal((d, d)) + 1j * gen.standard_normal((d, d))
        psi = b @ b.conj().T + 0.5 * np.eye(d)
        dec = gevd_hpd(phi, psi)
        pout[f"phi{count}"] = phi
        pout[f"psi{count}"] = psi
        pout[f"lam{count}"] = dec.eigenvalues
        pout[f"P{count}"] = dec.eigenvectors
    np.savez_compressed(HERE / "pencils.npz", **pout)
    print("pencils: done")


if __name__ == "__main__":
    main()
