"""GPU parity: the CUDA path against the reference's golden vectors and the
pinned CPU oracle on identical seeded inputs.

Tolerances (north_star): relative error <= 1e-9 for complex128, <= 1e-4 for
complex64 (against the complex128 reference), measured as the reference's
``max|a-b| / max|b|`` per quantity (tests/test_acceptance.py:34-35) and
per-entry relative error for the log-likelihood trace. Compared quantities
are phase invariant: v, S (original basis), the likelihood trace, images.
"""

import numpy as np
import pytest

from oracle import fastfca_oracle as O
from tests.conftest import RUN_CASES, load_golden
from tests.instances import kernel_instance, random_complex, random_instance

pytestmark = pytest.mark.gpu

TOL = 1e-9
TOL_C64 = 1e-4


def _pkg():
    import paper_1805_06572_b200 as P

    return P


def _model(g):
    return _pkg().SpatialModel(v=g["v0"], S=g["S0"], v_floor=g["floor"])


def _ll_dev(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    assert a.shape == b.shape
    return float(np.max(np.abs(a - b) / np.abs(b))) if b.size else 0.0


def _check(res, g, tag, tol):
    stride = int(g["image_stride"])
    assert O.scale_dev(res.images[:, ::stride], g[f"{tag}_images"]) <= tol
    assert O.scale_dev(res.model.v, g[f"{tag}_v"]) <= tol
    assert O.scale_dev(res.model.S, g[f"{tag}_S"]) <= tol
    assert _ll_dev(res.loglik_trace, g[f"{tag}_ll"]) <= tol
    L = int(g["L"])
    assert len(res.history) == L
    if L:
        hist = np.stack([h["S"] for h in res.history])
        assert O.scale_dev(hist, g[f"{tag}_Shist"]) <= tol
        if f"{tag}_vhist" in g:
            assert O.scale_dev(np.stack([h["v"] for h in res.history]), g[f"{tag}_vhist"]) <= tol
    oc = res.op_counts
    assert [oc.frame_matrix_inversions, oc.frame_matrix_products, oc.bin_gevd_count,
            oc.bin_matrix_products] == list(g[f"{tag}_counts"])


@pytest.mark.parametrize("case", RUN_CASES)
def test_fastfca_run_matches_reference(case):
    g = load_golden(f"runs_{case}")
    res = _pkg().fastfca_run(g["y"], _model(g), int(g["L"]), record_history=True)
    assert res.algorithm == "FastFCA"
    _check(res, g, "fast", TOL)


@pytest.mark.parametrize("case", RUN_CASES)
def test_fca_run_matches_reference(case):
    g = load_golden(f"runs_{case}")
    res = _pkg().fca_run(g["y"], _model(g), int(g["L"]), record_history=True)
    assert res.algorithm == "FCA"
    _check(res, g, "fca", TOL)


@pytest.mark.parametrize("case", ["cfg3m0", "cfg2", "acc2"])
def test_complex64_within_1e4_of_reference(case):
    g = load_golden(f"runs_{case}")
    res = _pkg().fastfca_run(g["y"], _model(g), int(g["L"]), dtype="c64")
    stride = int(g["image_stride"])
    assert O.scale_dev(res.images[:, ::stride], g["fast_images"]) <= TOL_C64
    assert O.scale_dev(res.model.v, g["fast_v"]) <= TOL_C64
    assert O.scale_dev(res.model.S, g["fast_S"]) <= TOL_C64
    assert _ll_dev(res.loglik_trace, g["fast_ll"]) <= TOL_C64


@pytest.mark.parametrize("case", ["cfg3m0", "cfg2", "acc2"])
def test_fca_complex64_within_1e4_of_reference(case):
    """fca_run(dtype='c64') against the complex128 reference (conventional.py:
    104-164; the reference has no c64 path, so the c128 golden run is the bar).
    The c64 FCA pass streams y / v in complex64 and computes in FP64."""
    g = load_golden(f"runs_{case}")
    res = _pkg().fca_run(g["y"], _model(g), int(g["L"]), dtype="c64")
    stride = int(g["image_stride"])
    assert res.images.dtype == np.complex64
    assert O.scale_dev(res.images[:, ::stride], g["fca_images"]) <= TOL_C64
    assert O.scale_dev(res.model.v, g["fca_v"]) <= TOL_C64
    assert O.scale_dev(res.model.S, g["fca_S"]) <= TOL_C64
    assert _ll_dev(res.loglik_trace, g["fca_ll"]) <= TOL_C64


@pytest.mark.parametrize("I", [1, 2, 3, 4, 5, 6, 7, 8])
def test_every_channel_count_matches_oracle(I):
    y, v, S = random_instance(300 + I, n_frames=37, n_bins=6, n_chan=I)
    floor = O.power_floor(y)
    v = np.maximum(v, floor[None, None, :])
    P = _pkg()
    init = P.SpatialModel(v=v, S=S, v_floor=floor)
    for run, orun in ((P.fastfca_run, O.fastfca_run), (P.fca_run, O.fca_run)):
        res = run(y, init, 4, record_history=True)
        ref = orun(y, v, S, floor, 4, record_history=True)
        assert O.scale_dev(res.images, ref.images) <= TOL
        assert O.scale_dev(res.model.v, ref.v) <= TOL
        assert O.scale_dev(res.model.S, ref.S) <= TOL
        assert _ll_dev(res.loglik_trace, ref.loglik_trace) <= TOL


def test_batched_run_equals_single_runs():
    P = _pkg()
    ys, models = [], []
    for m in range(3):
        gen = np.random.default_rng(70 + m)
        y = random_complex(gen, (50, 9, 3))
        ys.append(y)
        models.append(P.init_random(y, 5 + m))
    Y = np.stack(ys)
    batch = P.SpatialModel(v=np.stack([m.v for m in models]), S=np.stack([m.S for m in models]),
                           v_floor=np.stack([m.v_floor for m in models]))
    for run in (P.fastfca_run, P.fca_run):
        rb = run(Y, batch, 6)
        for m in range(3):
            rs = run(ys[m], models[m], 6)
            assert O.scale_dev(rb.images[m], rs.images) <= 1e-12
            assert O.scale_dev(rb.model.v[m], rs.model.v) <= 1e-12
            assert _ll_dev(rb.loglik_trace[m], rs.loglik_trace) <= 1e-12


def test_pipelined_host_path_equals_device_path():
    """Host batches run chunked with H2D / compute / D2H overlapped on three
    streams; results must equal the plain device run bit for bit (same chunking)."""
    import torch

    from paper_1805_06572_b200._engine import plan_chunks, run_device, run_host_pipelined

    P = _pkg()
    gen = np.random.default_rng(21)
    Y = random_complex(gen, (5, 120, 11, 4))
    inits = [P.init_random(Y[m], 40 + m) for m in range(5)]
    V = np.stack([i.v for i in inits])
    S = np.stack([i.S for i in inits])
    FL = np.stack([i.v_floor for i in inits])
    cf, _ = plan_chunks(5 * 11, 120, 4)
    ref = run_device("fast", Y, V, S, FL, 7, chunk_frames=cf)
    yp = torch.from_numpy(Y).pin_memory()
    vp = torch.from_numpy(V).pin_memory()
    res = run_host_pipelined("fast", yp, vp, S, FL, 7, chunk_frames=cf, chunk_mixtures=2)
    assert res["chunks"] == 3
    assert np.array_equal(res["images"], ref.images.cpu().numpy())
    assert np.array_equal(res["v"], ref.v.cpu().numpy())
    assert np.array_equal(res["S"], ref.S.cpu().numpy())
    assert np.array_equal(res["loglik"], ref.loglik.cpu().numpy())


def test_multistream_run_equals_single_stream_run():
    import torch

    from paper_1805_06572_b200._engine import plan_chunks, run_device, run_device_streams

    P = _pkg()
    gen = np.random.default_rng(22)
    Y = torch.from_numpy(random_complex(gen, (6, 90, 13, 3))).cuda()
    inits = [P.init_random(Y[m], 50 + m) for m in range(6)]
    V = torch.stack([i.v for i in inits])
    S = torch.stack([i.S for i in inits])
    FL = torch.stack([i.v_floor for i in inits])
    cf, _ = plan_chunks(6 * 13, 90, 3)
    ref = run_device("fast", Y, V, S, FL, 5, likelihood=False, chunk_frames=cf)
    out = {"images": torch.empty_like(ref.images), "S": torch.empty_like(ref.S),
           "v": torch.empty_like(ref.v)}
    ms = run_device_streams("fast", Y, V, S, FL, 5, nstreams=3, out=out, likelihood=False,
                            chunk_frames=cf, check=False)
    torch.cuda.synchronize()
    assert torch.equal(out["images"], ref.images)
    assert torch.equal(out["v"], ref.v)
    assert torch.equal(out["S"], ref.S)
    assert len(ms.parts) == 3


@pytest.mark.parametrize("algorithm", ["fast", "fca"])
def test_graph_replay_equals_stream_launches(algorithm):
    """FFCA_FLAG_GRAPH: the cached CUDA graph of a run replays bitwise the
    same results, also with the likelihood trace, and picks up new inputs
    written into the same buffers."""
    import torch

    from paper_1805_06572_b200._engine import run_device

    P = _pkg()
    gen = np.random.default_rng(23)
    Y = torch.from_numpy(random_complex(gen, (2, 70, 11, 3))).cuda()
    inits = [P.init_random(Y[m], 60 + m) for m in range(2)]
    V = torch.stack([i.v for i in inits])
    S = torch.stack([i.S for i in inits])
    FL = torch.stack([i.v_floor for i in inits])
    V0 = V.clone()
    ref = run_device(algorithm, Y, V, S, FL, 4, likelihood=True, timing=False)
    out = {"images": torch.empty_like(ref.images), "S": torch.empty_like(ref.S),
           "v": torch.empty_like(ref.v), "loglik": torch.empty_like(ref.loglik)}
    for _ in range(3):  # capture, then two replays
        r = run_device(algorithm, Y, V, S, FL, 4, likelihood=True, timing=False, out=out,
                       graph=True)
        out["workspace"] = r.workspace
        for k in ("images", "S", "v", "loglik"):
            assert torch.equal(getattr(r, k), getattr(ref, k)), k
    Y2 = Y.clone()
    Y2 *= 1.5  # new data in a new buffer: a different graph; same buffer: replay sees it
    ref2 = run_device(algorithm, Y2, V, S, FL, 4, likelihood=True, timing=False)
    Y.copy_(Y2)
    r = run_device(algorithm, Y, V, S, FL, 4, likelihood=True, timing=False, out=out, graph=True)
    assert torch.equal(r.images, ref2.images) and torch.equal(r.loglik, ref2.loglik)
    # the initial powers are read through v_in, never written
    assert torch.equal(V, V0)
    r0 = run_device(algorithm, Y, V, S, FL, 0, likelihood=True, timing=False,
                    out={"v": torch.empty_like(V)})
    assert torch.equal(r0.v, V0) and torch.equal(V, V0)


def test_mismatched_output_buffers_are_rejected():
    import torch

    from paper_1805_06572_b200._engine import run_device
    from paper_1805_06572_b200.errors import ConfigurationError

    P = _pkg()
    gen = np.random.default_rng(23)
    y = random_complex(gen, (20, 5, 2))
    init = P.init_random(y, 1)
    bad = {"v": torch.empty((1, 2, 20, 5), dtype=torch.float32, device="cuda")}
    with pytest.raises(ConfigurationError):
        run_device("fast", y[None], init.v[None], init.S[None], init.v_floor[None], 2, out=bad)


def test_bin_shards_are_bitwise_identical_to_the_full_run():
    """Frequency bins are independent; with equal frame chunking the per-bin
    reduction order is the same, so 1-GPU and k-GPU runs agree bit for bit."""
    from paper_1805_06572_b200._engine import run_device

    P = _pkg()
    gen = np.random.default_rng(9)
    y = random_complex(gen, (300, 40, 4))
    init = P.init_random(y, 3)
    cf = 64
    full = run_device("fast", y[None], init.v[None], init.S[None], init.v_floor[None], 5,
                      chunk_frames=cf)
    cuts = [0, 7, 23, 40]
    for a, b in zip(cuts, cuts[1:]):
        part = run_device("fast", np.ascontiguousarray(y[None, :, a:b]),
                          np.ascontiguousarray(init.v[None, :, :, a:b]), init.S[None][:, :, a:b],
                          init.v_floor[None][:, a:b], 5, chunk_frames=cf)
        assert (part.v.cpu() == full.v[..., a:b].cpu()).all()
        assert (part.images.cpu() == full.images[:, :, :, a:b].cpu()).all()
        assert (part.S.cpu() == full.S[:, :, a:b].cpu()).all()


def test_kernel_contract_matches_reference_backend():
    """Template: reference tests/test_backend.py — CUDA vs numba at 1e-12."""
    from paper_1805_06572_b200 import _kernels_cuda as K

    k = load_golden("kernels")
    y, v, S, Pm, lam, floor = k["y"], k["v"], k["S"], k["P"], k["lam"], k["floor"]
    mu, Phi, ninv, nprod = K.fca_e_step(y, v, S)
    assert O.scale_dev(mu, k["fca_e_mu"]) <= 1e-12
    assert O.scale_dev(Phi, k["fca_e_Phi"]) <= 1e-12
    assert [ninv, nprod] == list(k["fca_e_counts"])
    assert O.scale_dev(K.fca_v_update(k["fca_e_Phi"], S), k["fca_v"]) <= 1e-12
    assert O.scale_dev(K.fca_S_update(k["fca_e_Phi"], k["fca_v"]), k["fca_S"]) <= 1e-12
    assert K.fca_log_likelihood(y, v, S) == pytest.approx(float(k["fca_ll"]), rel=1e-12)
    assert O.scale_dev(K.fast_transform(y, Pm), k["yt"]) <= 1e-13
    mu_t, Phi_t, _, _ = K.fast_e_step(k["yt"], v, lam)
    assert O.scale_dev(mu_t, k["fast_e_mu"]) <= 1e-12
    assert O.scale_dev(Phi_t, k["fast_e_Phi"]) <= 1e-12
    assert O.scale_dev(K.fast_v_update(k["fast_e_Phi"], lam), k["fast_v"]) <= 1e-12
    assert O.scale_dev(K.fast_S_update(k["fast_e_Phi"], k["fast_v"]), k["fast_S"]) <= 1e-12
    ll = K.fast_log_likelihood(k["yt"], v, lam, k["logdet2"])
    assert ll == pytest.approx(float(k["fast_ll"]), rel=1e-12)
    mu, vn, Sr, ninv, nprod = K.fca_iteration(y, v, S, k["Sinv"], floor)
    assert O.scale_dev(mu, k["fca_it_mu"]) <= 1e-12
    assert O.scale_dev(vn, k["fca_it_v"]) <= 1e-12
    assert O.scale_dev(Sr, k["fca_it_S"]) <= 1e-12
    assert [ninv, nprod] == list(k["fca_it_counts"])
    mu, vn, Sr, _, _ = K.fast_iteration(y, Pm, v, lam, floor)
    assert O.scale_dev(mu, k["fast_it_mu"]) <= 1e-12
    assert O.scale_dev(vn, k["fast_it_v"]) <= 1e-12
    assert O.scale_dev(Sr, k["fast_it_S"]) <= 1e-12


def test_gevd_matches_reference_pencils():
    """Acceptance criterion 3 style (test_acceptance.py:97-154) on reference outputs."""
    P = _pkg()
    p = load_golden("pencils")
    n = len([k for k in p if k.startswith("phi")])
    for i in range(n):
        phi, psi = p[f"phi{i}"], p[f"psi{i}"]
        dec = P.gevd_hpd(phi, psi)
        lam, Pm = dec.eigenvalues, dec.eigenvectors
        d = lam.shape[0]
        scale = max(np.abs(lam).max(), 1.0)
        assert np.abs(lam - p[f"lam{i}"]).max() <= 1e-10 * scale
        denom = np.linalg.norm(phi) + np.abs(lam).max() * np.linalg.norm(psi)
        for k in range(d):
            res = np.linalg.norm(phi @ Pm[:, k] - lam[k] * psi @ Pm[:, k])
            assert res / denom <= 1e-10
        assert np.abs(Pm.conj().T @ psi @ Pm - np.eye(d)).max() <= 1e-10
        assert np.abs(Pm.conj().T @ phi @ Pm - np.diag(lam)).max() <= 1e-10 * scale
        # phase convention: largest entry of each column real positive
        for k in range(d):
            lead = Pm[np.argmax(np.abs(Pm[:, k])), k]
            assert lead.real > 0 and abs(lead.imag) <= 1e-12 * abs(lead)
        gap = np.min(np.abs(np.diff(lam))) / scale
        if gap > 1e-6:  # non-degenerate: eigenvectors unique up to the pinned phase
            assert np.abs(Pm - p[f"P{i}"]).max() <= 1e-8 * np.abs(Pm).max()


def test_gevd_errors_match_reference():
    P = _pkg()
    with pytest.raises(P.DefinitenessError) as exc:
        P.gevd_hpd(np.eye(2, dtype=complex), np.diag([1.0, -0.5]).astype(complex))
    assert exc.value.min_eigenvalue == pytest.approx(-0.5, abs=1e-12)
    with pytest.raises(P.DefinitenessError):
        P.gevd_hpd(np.eye(2, dtype=complex), np.diag([1.0, 1e-15]).astype(complex))
    with pytest.raises(P.NonHermitianError):
        P.gevd_hpd(np.array([[1.0, 1.0], [0.0, 1.0]], dtype=complex), np.eye(2, dtype=complex))


def test_singular_mixture_names_the_point():
    """reference test_conventional.py:111-120 and :51-60."""
    P = _pkg()
    y = np.ones((3, 2, 2), dtype=complex)
    v = np.full((2, 3, 2), 1.0)
    v[:, 1, 0] = 0.0
    S = np.zeros((2, 2, 2, 2), dtype=complex)
    S[:, :] = np.eye(2)
    model = P.SpatialModel(v=v, S=S, v_floor=np.full(2, 0.0))
    with pytest.raises(P.SingularMixtureError) as exc:
        P.e_step(y, model)
    assert (exc.value.frame, exc.value.bin) == (1, 0)
    with pytest.raises(P.SingularMixtureError) as exc:
        P.fca_run(y, model, 2)
    assert (exc.value.frame, exc.value.bin) == (1, 0)
    y = np.ones((2, 2, 2), dtype=complex)
    S = np.zeros((2, 2, 2, 2), dtype=complex)
    S[:, :] = np.eye(2)
    S[:, 1] = 0.0
    model = P.SpatialModel(v=np.full((2, 2, 2), 1.0), S=S, v_floor=np.full(2, 1e-12))
    with pytest.raises(P.SingularMixtureError) as exc:
        P.log_likelihood(y, model)
    assert exc.value.bin == 1


def test_silent_input_is_a_singular_matrix_error():
    """reference test_cli.py silent input -> SingularMatrixError (fast.py:39-55)."""
    P = _pkg()
    y = np.zeros((8, 3, 2), dtype=complex)
    init = P.init_random(y, 1)
    with pytest.raises(P.SingularMatrixError):
        P.fastfca_run(y, init, 2)


def test_stage_api_matches_oracle():
    """fast_e_step / fast_m_step_* / propagate_pencil / back transforms
    (reference test_fast.py:70-182)."""
    P = _pkg()
    from paper_1805_06572_b200.fast import (back_transform_covariances, back_transform_images,
                                            initial_pencil)

    y, v, S = random_instance(26, n_frames=10, n_bins=2, n_chan=3)
    floor = O.power_floor(y)
    v = np.maximum(v, floor[None, None, :])
    model = P.SpatialModel(v=v, S=S, v_floor=floor)
    Pm, lam = initial_pencil(model)
    lam_o, P_o = O.gevd_hpd(S[0], S[1])
    assert np.abs(lam - lam_o).max() <= 1e-10 * np.abs(lam_o).max()
    yt = P.transform_observations(y, Pm)
    mu_t, phi_t = P.fast_e_step(yt, v, lam)
    post = P.e_step(y, model)
    mu_o, phi_o, _, _ = O.fca_e_step(y, v, S)
    assert O.scale_dev(post.mu, mu_o) <= 1e-12
    assert O.scale_dev(back_transform_images(mu_t, Pm), mu_o) <= 1e-10
    # m_step (conventional.py:83-95) against the oracle's v / S updates
    new = P.m_step(post, model)
    v_o = np.maximum(O.fca_v_update(phi_o, S), floor[None, None, :])
    S_o = O.regularize_covariances(O.S_update(phi_o, v_o))
    assert O.scale_dev(new.v, v_o) <= 1e-12
    assert O.scale_dev(new.S, S_o) <= 1e-12
    # fast_m_step_v / fast_m_step_S (fast.py:74-104) against the oracle in the
    # transformed basis, and back-transformed against the conventional update
    # (the two engines' M-steps are the same map, test_fast.py:185-252)
    yt_o = O.fast_transform(y, P_o)
    mu_to, phi_to = O.fast_e_step(yt_o, v, lam_o)
    v_fast = np.maximum(P.fast_m_step_v(phi_t, lam), floor[None, None, :])
    v_fast_o = np.maximum(O.fast_v_update(phi_to, lam_o), floor[None, None, :])
    assert O.scale_dev(v_fast, v_fast_o) <= 1e-12
    assert O.scale_dev(v_fast, v_o) <= 1e-10
    gram = np.conj(np.swapaxes(Pm, -1, -2)) @ Pm
    s_t = P.fast_m_step_S(phi_t, v_fast, gram=gram)
    gram_o = np.conj(np.swapaxes(P_o, -1, -2)) @ P_o
    s_to = O.regularize_transformed(O.S_update(phi_to, v_fast_o), gram_o)
    s_back = back_transform_covariances(s_t, Pm)
    assert O.scale_dev(s_back, O.back_transform_covariances(s_to, P_o)) <= 1e-10
    assert O.scale_dev(s_back, S_o) <= 1e-10
    p_next, lam_next = P.propagate_pencil(s_t[0], s_t[1], Pm)
    for f in range(2):
        ph = p_next[f].conj().T
        d1 = ph @ s_back[0, f] @ p_next[f]
        d2 = ph @ s_back[1, f] @ p_next[f]
        assert np.abs(d1 - np.diag(lam_next[f])).max() <= 1e-9 * max(np.abs(lam_next[f]).max(), 1)
        assert np.abs(d2 - np.eye(3)).max() <= 1e-9


def test_incremental_transform_close_to_literal():
    """reference test_fast.py:239-245."""
    P = _pkg()
    y, v, S = random_instance(44, n_frames=8, n_bins=3, n_chan=2)
    floor = O.power_floor(y)
    model = P.SpatialModel(v=np.maximum(v, floor[None, None, :]), S=S, v_floor=floor)
    lit = P.fastfca_run(y, model, 6)
    inc = P.fastfca_run(y, model, 6, incremental_transform=True)
    assert np.abs(inc.images - lit.images).max() <= 1e-8 * np.abs(lit.images).max()
    assert _ll_dev(inc.loglik_trace, lit.loglik_trace) <= 1e-9


def test_init_random_matches_oracle():
    P = _pkg()
    g = load_golden("runs_acc1")
    m = P.init_random(g["y"], int(g["init_seed"]))
    assert O.scale_dev(m.v, g["v0"]) <= 1e-14
    assert O.scale_dev(m.S, g["S0"]) <= 1e-14
    assert O.scale_dev(m.v_floor, g["floor"]) <= 1e-14


def test_kernel_instance_shapes():
    y, v, S, Pm, lam = kernel_instance()
    assert y.shape == (9, 4, 3) and Pm.shape == (4, 3, 3)


# ---- exported per-bin helpers (reference pencil.py, conventional.py) ---------
def _random_hermitian(gen, d):
    a = gen.standard_normal((d, d)) + 1j * gen.standard_normal((d, d))
    return 0.5 * (a + a.conj().T)


def _random_hpd(gen, d):
    a = gen.standard_normal((d, d)) + 1j * gen.standard_normal((d, d))
    return a @ a.conj().T + d * np.eye(d)


def test_hermitian_eig_matches_reference_contract():
    """reference test_pencil.py:37-67 (TestHermitianEig) and eigh's values."""
    P = _pkg()
    w, u = P.hermitian_eig(np.eye(2, dtype=complex))
    assert np.allclose(w, [1.0, 1.0]) and np.allclose(u @ u.conj().T, np.eye(2), atol=1e-14)
    w, u = P.hermitian_eig(np.diag([2.0, 1.0]).astype(complex))
    assert np.allclose(w, [2.0, 1.0]) and np.allclose(np.abs(u), np.eye(2), atol=1e-14)
    gen = np.random.default_rng(7)
    for d in (2, 3, 4, 8):
        hs = np.stack([_random_hermitian(gen, d) for _ in range(20)])
        w, u = P.hermitian_eig(hs)  # batched
        for h, wk, uk in zip(hs, w, u):
            scale = max(np.abs(h).max(), 1.0)
            assert np.abs((uk * wk) @ uk.conj().T - h).max() <= 1e-12 * scale
            assert np.abs(uk.conj().T @ uk - np.eye(d)).max() <= 1e-12
            assert np.all(np.diff(wk) <= 1e-12 * scale)
            assert np.abs(wk - np.linalg.eigvalsh(h)[::-1]).max() <= 1e-12 * scale
    with pytest.raises(P.NonHermitianError):
        P.hermitian_eig(np.array([[1.0, 1.0], [0.0, 1.0]], dtype=complex))
    with pytest.raises(P.NonHermitianError):
        P.hermitian_eig(np.ones((2, 3), dtype=complex))


def test_solve_hermitian_system_matches_reference_contract():
    """reference test_pencil.py:146-166 (TestSolveHermitianSystem) and
    np.linalg.solve (the reference's zgesv) on HPD and general systems."""
    P = _pkg()
    b = np.arange(6, dtype=complex).reshape(3, 2)
    assert np.allclose(P.solve_hermitian_system(np.eye(3, dtype=complex), b), b)
    x = P.solve_hermitian_system(np.diag([2.0, 4.0]).astype(complex), np.array([2.0, 4.0]))
    assert x.shape == (2,) and np.allclose(x, [1.0, 1.0])
    gen = np.random.default_rng(3)
    for d in (2, 4, 8):
        for _ in range(10):
            a = _random_hpd(gen, d)
            rhs = gen.standard_normal((d, 3)) + 1j * gen.standard_normal((d, 3))
            x = P.solve_hermitian_system(a, rhs)
            assert np.linalg.norm(a @ x - rhs) <= 1e-10 * np.linalg.norm(rhs)
            assert O.scale_dev(x, np.linalg.solve(a, rhs)) <= 1e-12
    # a non-Hermitian nonsingular matrix needs the pivoting (zero leading entry)
    a = np.array([[0.0, 2.0, 1.0], [1.0, 1.0, 0.0], [3.0, 0.0, 1.0]], dtype=complex)
    rhs = np.array([1.0, 2.0, 3.0], dtype=complex)
    assert O.scale_dev(P.solve_hermitian_system(a, rhs), np.linalg.solve(a, rhs)) <= 1e-14
    # batched
    A = np.stack([_random_hpd(gen, 4) for _ in range(5)])
    Bm = gen.standard_normal((5, 4, 2)) + 0j
    assert O.scale_dev(P.solve_hermitian_system(A, Bm), np.linalg.solve(A, Bm)) <= 1e-12
    with pytest.raises(P.SingularMatrixError):
        P.solve_hermitian_system(np.zeros((2, 2), dtype=complex), np.ones(2))
    with pytest.raises(P.SingularMatrixError):  # numerically singular: residual test
        P.solve_hermitian_system(np.array([[1.0, 1.0], [1.0, 1.0 + 1e-17]], dtype=complex),
                                 np.array([1.0, 0.0], dtype=complex))


def test_cholesky_inverse_matches_oracle():
    """conventional._cholesky_inverse (reference conventional.py:98-101)."""
    from paper_1805_06572_b200.conventional import _cholesky_inverse

    gen = np.random.default_rng(11)
    for d in (1, 2, 3, 4, 8):
        S = np.stack([np.stack([_random_hpd(gen, d) for _ in range(6)]) for _ in range(2)])
        out = _cholesky_inverse(S)
        assert out.shape == S.shape
        assert O.scale_dev(out, O.cholesky_inverse(S)) <= 1e-12
        assert O.scale_dev(out @ S, np.broadcast_to(np.eye(d), S.shape)) <= 1e-12
    bad = np.stack([np.eye(2, dtype=complex), np.diag([1.0, -1.0]).astype(complex)])[None]
    with pytest.raises(np.linalg.LinAlgError):
        _cholesky_inverse(bad)


def test_degenerate_mixture_in_any_host_chunk_raises():
    """A failing mixture in the FIRST chunk of a chunked host batch (whose
    device slot is reused by later chunks) still raises like a single run."""
    P = _pkg()
    gen = np.random.default_rng(31)
    ys = [random_complex(gen, (40, 5, 2)) for _ in range(5)]
    ys[0][:] = 0.0  # silent mixture -> collapsed powers (fast.py:39-55)
    inits = [P.init_random(y, 90 + m) for m, y in enumerate(ys)]
    Y = np.stack(ys)
    batch = P.SpatialModel(v=np.stack([i.v for i in inits]), S=np.stack([i.S for i in inits]),
                           v_floor=np.stack([i.v_floor for i in inits]))
    from paper_1805_06572_b200._engine import run_host_pipelined

    with pytest.raises(P.SingularMatrixError):
        run_host_pipelined("fast", Y, batch.v, batch.S, batch.v_floor, 3, chunk_mixtures=1)
    with pytest.raises(P.SingularMatrixError):
        P.fastfca_run(Y, batch, 3)  # public API, ~one mixture per chunk
    ok = run_host_pipelined("fast", Y[1:], batch.v[1:], batch.S[1:], batch.v_floor[1:], 3,
                            chunk_mixtures=1)
    assert np.isfinite(ok["images"]).all()


def test_second_device_in_one_process():
    """Kernels opting into > 48 KB of shared memory must be configured per
    device: a run on cuda:1 after cuda:0 in the same process."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_1805_06572_b200._engine import run_device

    P = _pkg()
    gen = np.random.default_rng(5)
    y = random_complex(gen, (64, 40, 4))
    init = P.init_random(y, 2)
    outs = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            r = run_device("fast", y[None], init.v[None], init.S[None], init.v_floor[None], 3)
            outs.append(r.images.cpu())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("M", [1, 5])
def test_sharded_runs_bitwise_equal_at_every_world_size(M):
    """sharding.run_shard with the one chunk plan (the largest world size's):
    the shards of world sizes 1, 2, 3 and 8, run one after another on this
    GPU and concatenated, are bitwise the 1-rank run (bins and mixtures never
    couple; equal chunking => equal per-bin reduction order)."""
    import torch

    from paper_1805_06572_b200.sharding import run_shard

    P = _pkg()
    gen = np.random.default_rng(17)
    if M == 1:
        y = random_complex(gen, (700, 37, 4))
        init = P.init_random(y, 8)
        ax = {"images": 3, "v": 3, "S": 2}
    else:
        y = random_complex(gen, (M, 300, 9, 3))
        inits = [P.init_random(y[m], 20 + m) for m in range(M)]
        init = P.SpatialModel(v=np.stack([i.v for i in inits]), S=np.stack([i.S for i in inits]),
                              v_floor=np.stack([i.v_floor for i in inits]))
        ax = {"images": 0, "v": 0, "S": 0, "loglik": 0}
    for algorithm in ("fast", "fca"):
        _, one = run_shard(algorithm, y, init, 4, 0, 1)
        for world in (2, 3, 8):
            parts = [run_shard(algorithm, y, init, 4, r, world)[1] for r in range(world)]
            for key, a in ax.items():
                cat = torch.cat([p[key] for p in parts], dim=a)
                assert torch.equal(cat, one[key]), (algorithm, world, key)
            if M == 1:  # bin shards: likelihood partials add up to the full trace
                tot = sum(p["loglik"] for p in parts)
                assert torch.allclose(tot, one["loglik"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("I,dtype", [(2, "c128"), (3, "c128"), (4, "c128"), (4, "c64"), (8, "c128"),
                                     (8, "c64")])
def test_runs_are_bitwise_deterministic(I, dtype):
    """Repeated runs give bitwise identical images, v, S and likelihood
    (reference acceptance criterion, pkg/tests/test_acceptance.py:263-296).
    compute-sanitizer is closed on the GPU pool, so this also stands in for
    racecheck over the shared-memory frame rings, the cross-warp reductions
    and the staged image stores: a race would show up as run-to-run
    differences. Sizes give many CTAs, several frame chunks per bin, tiles
    across mixture boundaries and a partial last tile."""
    P = _pkg()
    gen = np.random.default_rng(100 + I)
    M, N, F = 3, 400, 45
    y = random_complex(gen, (M, N, F, I))
    inits = [P.init_random(y[m], 30 + m) for m in range(M)]
    init = P.SpatialModel(v=np.stack([i.v for i in inits]), S=np.stack([i.S for i in inits]),
                          v_floor=np.stack([i.v_floor for i in inits]))
    for run in (P.fastfca_run, P.fca_run):
        outs = [run(y, init, 3, dtype=dtype) for _ in range(3)]
        for o in outs[1:]:
            assert np.array_equal(o.images, outs[0].images), run.__name__
            assert np.array_equal(o.model.v, outs[0].model.v), run.__name__
            assert np.array_equal(o.model.S, outs[0].model.S), run.__name__
            assert np.array_equal(np.asarray(o.loglik_trace), np.asarray(outs[0].loglik_trace))


@pytest.mark.parametrize("I,dtype,M,F", [(2, "c128", 1, 200), (3, "c128", 2, 70), (4, "c128", 1, 300),
                                         (4, "c64", 1, 300), (8, "c128", 1, 140)])
@pytest.mark.parametrize("graph", [False, True])
def test_split_phase_windows_bitwise(I, dtype, M, F, graph):
    """The split-phase schedule (bin windows whose pencil refreshes run on a
    second stream while the next window streams, passes chained with
    programmatic serialisation) only restricts which bins each launch
    covers: images, v, S and the likelihood are bitwise those of the plain
    schedule for any window count (ragged last window, windows across a
    mixture boundary, more windows than tiles clamp), and match the oracle."""
    import torch

    from paper_1805_06572_b200._engine import run_device, status_of

    P = _pkg()
    gen = np.random.default_rng(7 + I)
    N, L = 260, 4
    y = random_complex(gen, (M, N, F, I))
    inits = [P.init_random(y[m], 11 + m) for m in range(M)]
    v0 = np.stack([i.v for i in inits])
    S0 = np.stack([i.S for i in inits])
    fl = np.stack([i.v_floor for i in inits])
    outs = {}
    for k in (1, 2, 3, 64):
        r = run_device("fast", y, v0, S0, fl, L, dtype=dtype, chunk_frames=40, graph=graph,
                       timing=False, bin_parts=k)
        status_of(r)
        torch.cuda.synchronize()
        outs[k] = [r.images.cpu().numpy(), r.v.cpu().numpy(), r.S.cpu().numpy(),
                   r.loglik.cpu().numpy()]
    for k in (2, 3, 64):
        for a, b in zip(outs[k], outs[1]):
            assert np.array_equal(a, b), (k, I, dtype)
    tol = TOL if dtype == "c128" else TOL_C64
    ref = O.fastfca_run(y[0], v0[0], S0[0], fl[0], L)
    assert O.scale_dev(outs[3][1][0], ref.v) <= tol
    assert O.scale_dev(outs[3][2][0], ref.S) <= tol
    assert O.scale_dev(outs[3][0][0], ref.images) <= tol


@pytest.mark.parametrize("shape,L", [((2, 90, 40, 2), 6), ((1, 150, 70, 3), 5), ((1, 120, 33, 4), 4),
                                     ((3, 64, 11, 1), 3)])
def test_persistent_em_kernel_equals_the_plain_schedule(shape, L):
    """KP (opt-in): small complex128 runs without likelihood / history / events
    do their first L - 1 iterations in ONE persistent cooperative launch
    (streaming and refresher CTAs synchronised per tile through global
    flags). With equal chunking the arithmetic is the plain schedule's:
    bitwise equal results; also as a replayed graph, with a separate
    initial-power buffer, and against the oracle."""
    import torch

    from paper_1805_06572_b200._engine import run_device

    P = _pkg()
    M, N, F, I = shape
    gen = np.random.default_rng(41 + I)
    Y = torch.from_numpy(random_complex(gen, shape)).cuda()
    inits = [P.init_random(Y[m], 80 + m) for m in range(M)]
    V = torch.stack([i.v for i in inits])
    S = torch.stack([i.S for i in inits])
    FL = torch.stack([i.v_floor for i in inits])
    V0 = V.clone()
    kw = dict(likelihood=False, timing=False, chunk_frames=32)  # (KP's own plan differs)
    plain = run_device("fast", Y, V, S, FL, L, persist=False, **kw)
    kw["persist"] = True
    kp = run_device("fast", Y, V, S, FL, L, **kw)
    for k in ("images", "v", "S"):
        if I == 4:  # the plain schedule refreshes few I = 4 bins with the lane-parallel K1p
            a, b = getattr(kp, k).cpu().numpy(), getattr(plain, k).cpu().numpy()
            assert O.scale_dev(a, b) <= 1e-12, k
        else:
            assert torch.equal(getattr(kp, k), getattr(plain, k)), k
    out = {"images": torch.empty_like(plain.images), "S": torch.empty_like(plain.S),
           "v": torch.empty_like(plain.v)}
    for _ in range(3):  # captured graph, then replays
        r = run_device("fast", Y, V, S, FL, L, out=out, graph=True, **kw)
        out["workspace"] = r.workspace
        for k in ("images", "v", "S"):
            assert torch.equal(getattr(r, k), getattr(kp, k)), k
    assert torch.equal(V, V0)
    # the oracle on the first mixture
    y0 = Y[0].cpu().numpy()
    ref = O.fastfca_run(y0, inits[0].v.cpu().numpy(), inits[0].S.cpu().numpy(),
                        inits[0].v_floor.cpu().numpy(), L)
    auto = run_device("fast", Y, V, S, FL, L, likelihood=False, timing=False, persist=True)
    for r in (kp, auto):  # (auto: KP's own chunk plan)
        assert O.scale_dev(r.images[0].cpu().numpy(), ref.images) <= TOL
        assert O.scale_dev(r.v[0].cpu().numpy(), ref.v) <= TOL
        assert O.scale_dev(r.S[0].cpu().numpy(), ref.S) <= TOL


def test_persistent_em_kernel_reports_collapsed_powers():
    """A silent mixture under KP raises like the plain schedule."""
    from paper_1805_06572_b200._engine import run_device

    P = _pkg()
    y = np.zeros((40, 20, 2), dtype=complex)
    init = P.init_random(y, 1)
    for persist in (False, True):
        with pytest.raises(P.SingularMatrixError):
            run_device("fast", y[None], init.v[None], init.S[None], init.v_floor[None], 4,
                       likelihood=False, timing=False, persist=persist)
