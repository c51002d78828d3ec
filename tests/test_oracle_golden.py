"""Pin the CPU oracle (oracle/fastfca_oracle.py) against golden vectors that
the unmodified reference produced (tests/golden/make_golden.py).

CPU only. These tests are what makes the oracle trustworthy as the checker
for the CUDA path.
"""

import numpy as np
import pytest

from oracle import fastfca_oracle as O
from tests.conftest import RUN_CASES, load_golden

TOL = 1e-10  # oracle vs reference: both complex128 on LAPACK


def _check_run(res, g, tag):
    stride = int(g["image_stride"])
    assert O.scale_dev(res.images[:, ::stride], g[f"{tag}_images"]) <= TOL
    if g["L"] > 0:
        assert O.scale_dev(res.v, g[f"{tag}_v"]) <= TOL
    assert O.scale_dev(res.S, g[f"{tag}_S"]) <= TOL
    ll = np.asarray(res.loglik_trace)
    ref = g[f"{tag}_ll"]
    assert ll.shape == ref.shape
    assert np.max(np.abs(ll - ref) / np.abs(ref)) <= TOL
    if g["L"] > 0:
        hist = np.stack([h["S"] for h in res.history])
        assert O.scale_dev(hist, g[f"{tag}_Shist"]) <= TOL
        if f"{tag}_vhist" in g:
            vh = np.stack([h["v"] for h in res.history])
            assert O.scale_dev(vh, g[f"{tag}_vhist"]) <= TOL
    counts = [res.counts[k] for k in ("frame_matrix_inversions", "frame_matrix_products",
                                      "bin_gevd_count", "bin_matrix_products")]
    assert counts == list(g[f"{tag}_counts"])


@pytest.mark.parametrize("case", RUN_CASES)
def test_oracle_fastfca_matches_reference(case):
    g = load_golden(f"runs_{case}")
    res = O.fastfca_run(g["y"], g["v0"], g["S0"], g["floor"], int(g["L"]), record_history=True)
    _check_run(res, g, "fast")


@pytest.mark.parametrize("case", RUN_CASES)
def test_oracle_fca_matches_reference(case):
    g = load_golden(f"runs_{case}")
    res = O.fca_run(g["y"], g["v0"], g["S0"], g["floor"], int(g["L"]), record_history=True)
    _check_run(res, g, "fca")


def test_oracle_init_random_matches_reference():
    g = load_golden("runs_acc1")
    v, S, floor = O.init_random(g["y"], int(g["init_seed"]))
    assert O.scale_dev(v, g["v0"]) <= 1e-14
    assert O.scale_dev(S, g["S0"]) <= 1e-14
    assert O.scale_dev(floor, g["floor"]) <= 1e-14


def test_oracle_kernels_match_reference():
    k = load_golden("kernels")
    y, v, S, P, lam, floor = k["y"], k["v"], k["S"], k["P"], k["lam"], k["floor"]
    mu, Phi, ninv, nprod = O.fca_e_step(y, v, S)
    assert O.scale_dev(mu, k["fca_e_mu"]) <= 1e-12
    assert O.scale_dev(Phi, k["fca_e_Phi"]) <= 1e-12
    assert [ninv, nprod] == list(k["fca_e_counts"])
    vv = O.fca_v_update(k["fca_e_Phi"], S)
    assert O.scale_dev(vv, k["fca_v"]) <= 1e-12
    assert O.scale_dev(O.S_update(k["fca_e_Phi"], k["fca_v"]), k["fca_S"]) <= 1e-12
    assert O.fca_log_likelihood(y, v, S) == pytest.approx(float(k["fca_ll"]), rel=1e-12)
    yt = O.fast_transform(y, P)
    assert O.scale_dev(yt, k["yt"]) <= 1e-13
    mu_t, Phi_t = O.fast_e_step(k["yt"], v, lam)
    assert O.scale_dev(mu_t, k["fast_e_mu"]) <= 1e-12
    assert O.scale_dev(Phi_t, k["fast_e_Phi"]) <= 1e-12
    assert O.scale_dev(O.fast_v_update(k["fast_e_Phi"], lam), k["fast_v"]) <= 1e-12
    assert O.scale_dev(O.S_update(k["fast_e_Phi"], k["fast_v"]), k["fast_S"]) <= 1e-12
    ll = O.fast_log_likelihood(k["yt"], v, lam, k["logdet2"])
    assert ll == pytest.approx(float(k["fast_ll"]), rel=1e-12)
    mu, vn, Sr, ninv, nprod = O.fca_iteration(y, v, S, k["Sinv"], floor)
    assert O.scale_dev(mu, k["fca_it_mu"]) <= 1e-12
    assert O.scale_dev(vn, k["fca_it_v"]) <= 1e-12
    assert O.scale_dev(Sr, k["fca_it_S"]) <= 1e-12
    assert [ninv, nprod] == list(k["fca_it_counts"])
    mu, vn, Sr = O.fast_iteration(y, P, v, lam, floor)
    assert O.scale_dev(mu, k["fast_it_mu"]) <= 1e-12
    assert O.scale_dev(vn, k["fast_it_v"]) <= 1e-12
    assert O.scale_dev(Sr, k["fast_it_S"]) <= 1e-12


def test_oracle_pencils_match_reference():
    p = load_golden("pencils")
    n = len([k for k in p if k.startswith("phi")])
    for i in range(n):
        lam, P = O.gevd_hpd(p[f"phi{i}"], p[f"psi{i}"])
        assert np.abs(lam - p[f"lam{i}"]).max() <= 1e-12 * max(np.abs(lam).max(), 1.0)
        assert np.abs(P - p[f"P{i}"]).max() <= 1e-10 * np.abs(P).max()


def test_oracle_definiteness_error():
    with pytest.raises(O.OracleDefinitenessError) as exc:
        O.gevd_hpd(np.eye(2, dtype=complex), np.diag([1.0, -0.5]).astype(complex))
    assert exc.value.min_eigenvalue == pytest.approx(-0.5, abs=1e-12)


def test_oracle_synthetic_generator_shapes_and_determinism():
    from paper_1805_06572_b200.synth import make_mixture

    a = make_mixture(5, 3, 6, 1500, eps=1e-3, sigma=2.0, envelope=True)
    b = make_mixture(5, 3, 6, 1500, eps=1e-3, sigma=2.0, envelope=True)
    assert a.shape == (1500, 6, 3) and a.dtype == np.complex128
    assert np.array_equal(a, b)
