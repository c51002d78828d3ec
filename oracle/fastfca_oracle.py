"""CPU oracle for the FCA / FastFCA EM path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it. The shipped package
``paper_1805_06572_b200`` never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

What it is: a numpy restatement of the reference package ``fastfca`` 0.1.0
(``/root/reference/pkg/src/fastfca``) on the hot path named by
``BASELINE.json`` — both EM engines, their per-(n, f) kernels, the per-bin
Hermitian-definite pencil decomposition and the model helpers. It is written
bin-by-bin (numpy vectorised over frames inside one bin) rather than in the
reference's einsum-over-everything or scalar-loop styles; the arithmetic is
the same, term for term, and every function cites the reference lines it
restates.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by running the *unmodified reference* in the build container
(``tests/golden/make_golden.py``; the reference cannot travel to the GPU box,
its outputs can). The reference itself is complex128 only; so is this oracle.

Array layout (the reference's, ``_kernels_numpy.py:3-13``)::

    y    (N, F, I)      complex observations, frame-major
    v    (2, N, F)      source powers
    S    (2, F, I, I)   spatial covariances
    P    (F, I, I)      per-bin joint-diagonalising basis
    lam  (F, I)         generalised eigenvalues (descending)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# --- constants (reference modelops.py:6,9; pencil.py:22,25) -----------------
V_FLOOR_FACTOR = 1e-10
COV_EPS_FACTOR = 1e-9
HERMITIAN_RTOL = 1e-10
DEFINITENESS_FLOOR = 1e-12


class OracleError(ValueError):
    """Base for oracle-side numerical errors (mirrors reference errors.py)."""


class OracleDefinitenessError(OracleError):
    """reference errors.py:12-20 (DefinitenessError, carries min eigenvalue)."""

    def __init__(self, message, min_eigenvalue):
        super().__init__(message)
        self.min_eigenvalue = min_eigenvalue


class OracleNonHermitianError(OracleError):
    """reference errors.py:8 (NonHermitianError)."""


class OracleSingularError(OracleError):
    """reference errors.py:23,27-38 (SingularMatrixError / SingularMixtureError)."""

    def __init__(self, message, frame=None, bin=None):
        super().__init__(message)
        self.frame = frame
        self.bin = bin


def _ct(a):
    return np.conj(np.swapaxes(a, -1, -2))


# --- model helpers (reference modelops.py:12-39) -----------------------------
def power_floor(y):
    """V_FLOOR_FACTOR * mean_n(||y(n,f)||^2) / I per bin (modelops.py:12-21)."""
    y = np.asarray(y)
    per_point = (y.real**2 + y.imag**2).sum(axis=-1)
    return V_FLOOR_FACTOR * per_point.mean(axis=0) / y.shape[-1]


def hermitize(S):
    """(S + S^H) / 2 (modelops.py:24-26)."""
    return 0.5 * (S + _ct(S))


def regularize_covariances(S):
    """hermitize + COV_EPS_FACTOR * tr(S)/I * Id (modelops.py:29-39)."""
    H = hermitize(S)
    d = H.shape[-1]
    tr = np.trace(H, axis1=-2, axis2=-1).real
    return H + (COV_EPS_FACTOR * tr / d)[..., None, None] * np.eye(d)


def init_random(y, seed):
    """Seeded random model (initializers.py:20-39).

    One I x I complex Gaussian draw per source, shared across bins:
    S_j = A A^H + Id; v_j = ||y||^2 / (2I), floored per bin.
    """
    y = np.asarray(y)
    N, F, I = y.shape
    gen = np.random.default_rng(seed)
    S = np.empty((2, F, I, I), dtype=np.complex128)
    for j in range(2):
        re = gen.standard_normal((I, I))
        im = gen.standard_normal((I, I))
        A = re + 1j * im
        S[j] = (A @ A.conj().T + np.eye(I))[None]
    split = (y.real**2 + y.imag**2).sum(axis=-1) / (2 * I)
    floor = power_floor(y)
    v = np.maximum(np.stack([split, split]), floor[None, None, :])
    return v, S, floor


# --- pencil (reference pencil.py:40-135) -------------------------------------
def check_hermitian(A, name):
    """pencil.py:40-51: square, and asymmetry <= 1e-10 * max|A|."""
    A = np.asarray(A, dtype=np.complex128)
    if A.ndim < 2 or A.shape[-1] != A.shape[-2]:
        raise OracleNonHermitianError(f"{name} must be square, got {A.shape}")
    scale = np.abs(A).max(axis=(-2, -1))
    asym = np.abs(A - _ct(A)).max(axis=(-2, -1))
    if np.any(asym > HERMITIAN_RTOL * np.maximum(scale, 1e-300)):
        raise OracleNonHermitianError(f"{name} is not Hermitian")
    return A


def fix_column_phases(P):
    """pencil.py:76-82: rotate each column so its largest |entry| is real > 0."""
    P = np.array(P, copy=True)
    cols = P.shape[-1]
    for k in range(cols):
        col = P[..., :, k]
        idx = np.argmax(np.abs(col), axis=-1)
        lead = np.take_along_axis(col, idx[..., None], axis=-1)[..., 0]
        mag = np.abs(lead)
        ph = np.where(mag > 0, lead / np.where(mag > 0, mag, 1.0), 1.0)
        P[..., :, k] = col * np.conj(ph)[..., None]
    return P


def gevd_hpd(Phi, Psi):
    """Hermitian-definite pencil (Phi, Psi) -> (lam desc, P) (pencil.py:85-135).

    eigh(Psi) -> definiteness floor 1e-12 tr/D -> whiten -> eigh -> descending
    -> P = U Sigma^{-1/2} Q -> column phase fix.
    """
    Phi = check_hermitian(Phi, "Phi")
    Psi = check_hermitian(Psi, "Psi")
    if Phi.shape != Psi.shape:
        raise OracleNonHermitianError("Phi and Psi shapes differ")
    D = Psi.shape[-1]
    sig, U = np.linalg.eigh(Psi)
    thr = DEFINITENESS_FLOOR * np.trace(Psi, axis1=-2, axis2=-1).real / D
    if np.any(sig[..., 0] <= thr):
        worst = float(np.min(sig[..., 0]))
        raise OracleDefinitenessError(f"Psi not positive definite: {worst:.6e}", worst)
    isq = 1.0 / np.sqrt(sig)
    W = isq[..., :, None] * (_ct(U) @ Phi @ U) * isq[..., None, :]
    W = hermitize(W)
    lam, Q = np.linalg.eigh(W)
    lam = lam[..., ::-1].copy()
    Q = Q[..., ::-1]
    P = U @ (isq[..., :, None] * Q)
    return lam, fix_column_phases(P)


def logdet2(P):
    """2 log|det P| per bin (fast.py:151-153)."""
    return 2.0 * np.linalg.slogdet(P)[1]


# --- FastFCA per-point kernels (reference _kernels_numba.py:147-243,328-391)
def fast_transform(y, P):
    """z(n,f) = P(f)^H y(n,f) (_kernels_numba.py:147-162)."""
    N, F, I = y.shape
    z = np.empty_like(y, dtype=np.complex128)
    for f in range(F):
        z[:, f, :] = y[:, f, :] @ np.conj(P[f])
    return z


def _fast_gains(v1, v2, lam_f):
    # per (n, i): den, g1, g2, c  (_kernels_numba.py:352-360)
    la = lam_f[None, :]
    den = v1[:, None] * la + v2[:, None]
    g1 = v1[:, None] * la / den
    g2 = v2[:, None] / den
    c = v2[:, None] * g1
    return den, g1, g2, c


def fast_e_step(z, v, lam):
    """Posterior moments in the diagonal basis (_kernels_numba.py:165-193)."""
    N, F, I = z.shape
    mu = np.empty((2, N, F, I), dtype=np.complex128)
    Phi = np.empty((2, N, F, I, I), dtype=np.complex128)
    eye = np.eye(I)
    for f in range(F):
        _, g1, g2, c = _fast_gains(v[0, :, f], v[1, :, f], lam[f])
        m1 = g1 * z[:, f]
        m2 = g2 * z[:, f]
        mu[0, :, f], mu[1, :, f] = m1, m2
        Phi[0, :, f] = m1[:, :, None] * m1[:, None, :].conj() + c[:, :, None] * eye
        Phi[1, :, f] = m2[:, :, None] * m2[:, None, :].conj() + c[:, :, None] * eye
    return mu, Phi


def fast_v_update(Phi_t, lam):
    """v1 = sum_i Phi1_ii/lam_i / I, v2 = sum_i Phi2_ii / I (_kernels_numba.py:196-213)."""
    I = Phi_t.shape[-1]
    d = np.diagonal(Phi_t, axis1=-2, axis2=-1).real  # (2, N, F, I)
    return np.stack([(d[0] / lam[None]).sum(-1), d[1].sum(-1)]) / I


def S_update(Phi, v):
    """(1/N) sum_n Phi_j / v_j (_kernels_numba.py:98-113, shared by both engines)."""
    N = Phi.shape[1]
    out = np.empty((2,) + Phi.shape[2:], dtype=np.complex128)
    for j in range(2):
        out[j] = (Phi[j] / v[j][..., None, None]).sum(axis=0) / N
    return out


def fast_log_likelihood(z, v, lam, ld2):
    """Diagonal-basis log-likelihood (_kernels_numba.py:220-243)."""
    N, F, I = z.shape
    total = -N * F * I * np.log(np.pi) + N * float(np.sum(ld2))
    for f in range(F):
        den, _, _, _ = _fast_gains(v[0, :, f], v[1, :, f], lam[f])
        p = z[:, f].real ** 2 + z[:, f].imag ** 2
        total -= float(np.sum(np.log(den)) + np.sum(p / den))
    return total


def fast_iteration(y, P, v, lam, floor):
    """Fused transform + E + M pass (_kernels_numba.py:328-391).

    Returns (mu_t, v_new, S_raw) with S_raw the unregularised transformed
    covariance average.
    """
    N, F, I = y.shape
    mu = np.empty((2, N, F, I), dtype=np.complex128)
    v_new = np.empty((2, N, F))
    S_raw = np.empty((2, F, I, I), dtype=np.complex128)
    for f in range(F):
        z = y[:, f, :] @ np.conj(P[f])
        _, g1, g2, c = _fast_gains(v[0, :, f], v[1, :, f], lam[f])
        m1 = g1 * z
        m2 = g2 * z
        pz = z.real**2 + z.imag**2
        tr1 = ((g1 * g1 * pz + c) / lam[f][None, :]).sum(-1)
        tr2 = (g2 * g2 * pz + c).sum(-1)
        w1 = np.maximum(tr1 / I, floor[f])
        w2 = np.maximum(tr2 / I, floor[f])
        v_new[0, :, f], v_new[1, :, f] = w1, w2
        mu[0, :, f], mu[1, :, f] = m1, m2
        for j, (m, w) in enumerate(((m1, w1), (m2, w2))):
            iw = 1.0 / w
            acc = (m * iw[:, None]).T @ m.conj()  # sum_n m_a conj(m_b) / w
            acc[np.diag_indices(I)] += (c * iw[:, None]).sum(0)
            S_raw[j, f] = acc / N
    return mu, v_new, S_raw


# --- conventional FCA kernels (reference _kernels_numba.py:12-144,246-325) ---
def _mixture_cov(v, S, f):
    # R(n) = v1 S1 + v2 S2 for one bin, (N, I, I)
    return v[0, :, f, None, None] * S[0, f] + v[1, :, f, None, None] * S[1, f]


def fca_e_step(y, v, S):
    """Posterior moments with frame-wise inverses (_kernels_numba.py:12-72)."""
    N, F, I = y.shape
    mu = np.empty((2, N, F, I), dtype=np.complex128)
    Phi = np.empty((2, N, F, I, I), dtype=np.complex128)
    for f in range(F):
        Rinv = np.linalg.inv(_mixture_cov(v, S, f))
        A1 = S[0, f] @ Rinv
        A2 = S[1, f] @ Rinv
        m1 = v[0, :, f, None] * (A1 @ y[:, f, :, None])[..., 0]
        m2 = v[1, :, f, None] * (A2 @ y[:, f, :, None])[..., 0]
        cross = (v[0, :, f] * v[1, :, f])[:, None, None] * (A1 @ S[1, f])
        mu[0, :, f], mu[1, :, f] = m1, m2
        Phi[0, :, f] = m1[:, :, None] * m1[:, None, :].conj() + cross
        Phi[1, :, f] = m2[:, :, None] * m2[:, None, :].conj() + cross
    return mu, Phi, N * F, 3 * N * F


def cholesky_inverse(S):
    """S^{-1} = L^{-H} L^{-1} per bin (conventional.py:98-101)."""
    L = np.linalg.cholesky(S)
    Li = np.linalg.inv(L)
    return _ct(Li) @ Li


def fca_v_update(Phi, S_prev):
    """tr(S_prev^{-1} Phi)/I (_kernels_numba.py:75-95)."""
    I = Phi.shape[-1]
    Si = cholesky_inverse(S_prev)  # (2, F, I, I)
    return np.stack(
        [np.einsum("fab,nfba->nf", Si[j], Phi[j]).real / I for j in range(2)]
    )


def fca_log_likelihood(y, v, S):
    """sum -I log pi - log det R - y^H R^{-1} y (_kernels_numba.py:116-144)."""
    N, F, I = y.shape
    total = -N * F * I * np.log(np.pi)
    for f in range(F):
        R = _mixture_cov(v, S, f)
        sign, ld = np.linalg.slogdet(R)
        x = np.linalg.solve(R, y[:, f, :, None])[..., 0]
        quad = (np.conj(y[:, f, :]) * x).sum(-1).real
        total += float(np.sum(-ld - quad))
    return total


def fca_iteration(y, v, S, Sinv, floor):
    """Fused conventional E+M pass (_kernels_numba.py:246-325)."""
    N, F, I = y.shape
    mu = np.empty((2, N, F, I), dtype=np.complex128)
    v_new = np.empty((2, N, F))
    S_raw = np.empty((2, F, I, I), dtype=np.complex128)
    for f in range(F):
        Rinv = np.linalg.inv(_mixture_cov(v, S, f))
        A1 = S[0, f] @ Rinv
        A2 = S[1, f] @ Rinv
        m1 = v[0, :, f, None] * (A1 @ y[:, f, :, None])[..., 0]
        m2 = v[1, :, f, None] * (A2 @ y[:, f, :, None])[..., 0]
        cross = (v[0, :, f] * v[1, :, f])[:, None, None] * (A1 @ S[1, f])
        ws = []
        for j, m in enumerate((m1, m2)):
            Phi = m[:, :, None] * m[:, None, :].conj() + cross
            tr = np.einsum("ab,nba->n", Sinv[j, f], Phi).real
            w = np.maximum(tr / I, floor[f])
            ws.append(w)
            S_raw[j, f] = (Phi / w[:, None, None]).sum(0) / N
        v_new[0, :, f], v_new[1, :, f] = ws
        mu[0, :, f], mu[1, :, f] = m1, m2
    return mu, v_new, S_raw, N * F, 3 * N * F


# --- drivers (reference fast.py:80-260, conventional.py:104-164) -------------
@dataclass
class OracleResult:
    """Mirror of reference types.SeparationResult (types.py:132-150)."""

    algorithm: str
    images: np.ndarray
    loglik_trace: list
    v: np.ndarray
    S: np.ndarray
    v_floor: np.ndarray
    history: list = field(default_factory=list)
    counts: dict = field(default_factory=dict)


def regularize_transformed(S_raw, gram):
    """fast.py:80-90: hermitize + eps * gram, eps = 1e-9 tr(gram^{-1} S)/I."""
    S_t = hermitize(S_raw)
    d = S_t.shape[-1]
    tr = np.trace(np.linalg.solve(gram, S_t), axis1=-2, axis2=-1).real
    return S_t + (COV_EPS_FACTOR * tr / d)[..., None, None] * gram


def back_transform_images(mu_t, P):
    """Solve P^H mu = mu_t per bin (fast.py:133-141)."""
    out = np.empty_like(mu_t)
    F = P.shape[0]
    for f in range(F):
        Ph = np.conj(P[f]).T
        # (2, N, I) -> (I, 2N)
        rhs = mu_t[:, :, f, :].reshape(-1, P.shape[-1]).T
        out[:, :, f, :] = np.linalg.solve(Ph, rhs).T.reshape(mu_t.shape[0], mu_t.shape[1], -1)
    return out


def back_transform_covariances(S_t, P):
    """(P^H)^{-1} S_t P^{-1} per bin (fast.py:144-148)."""
    Ph = _ct(P)
    half = np.linalg.solve(Ph, S_t)
    return _ct(np.linalg.solve(Ph, _ct(half)))


def _require_finite(*arrs):
    # fast.py:51-55
    for a in arrs:
        if not np.all(np.isfinite(a)):
            raise OracleSingularError("mixture covariance is singular")


def fastfca_run(y, v0, S0, floor, iterations, record_history=False, compute_likelihood=True):
    """FastFCA EM (fast.py:156-260), non-incremental transform."""
    y = np.asarray(y, dtype=np.complex128)
    v = np.array(v0, dtype=np.float64, copy=True)
    lam, P = gevd_hpd(S0[0], S0[1])  # initial_pencil, fast.py:127-130
    trace, history = [], []
    counts = dict(frame_matrix_inversions=0, frame_matrix_products=0, bin_gevd_count=0,
                  bin_matrix_products=0)
    F = y.shape[1]
    if compute_likelihood:
        trace.append(fast_log_likelihood(fast_transform(y, P), v, lam, logdet2(P)))
    mu_t = None
    P_e = P
    S_t = None
    for _ in range(int(iterations)):
        P_e = P
        mu_t, v, S_raw = fast_iteration(y, P, v, lam, floor)
        _require_finite(v, S_raw)
        gram = _ct(P) @ P
        counts["bin_matrix_products"] += F
        S_t = regularize_transformed(S_raw, gram)
        lam, Q = gevd_hpd(S_t[0], S_t[1])
        P = P @ Q
        counts["bin_gevd_count"] += F
        counts["bin_matrix_products"] += F
        if compute_likelihood:
            trace.append(fast_log_likelihood(fast_transform(y, P), v, lam, logdet2(P)))
        if record_history:
            history.append({"v": v.copy(), "S": back_transform_covariances(S_t, P_e)})
    if mu_t is None:
        mu_t, _ = fast_e_step(fast_transform(y, P), v, lam)
        P_e = P
    images = back_transform_images(mu_t, P_e)
    if iterations and history:
        S_final = history[-1]["S"]
    elif iterations:
        S_final = back_transform_covariances(S_t, P_e)
    else:
        S_final = np.array(S0, dtype=np.complex128, copy=True)
    return OracleResult("FastFCA", images, trace, v, S_final, np.asarray(floor), history, counts)


def fca_run(y, v0, S0, floor, iterations, record_history=False, compute_likelihood=True):
    """Conventional FCA EM (conventional.py:104-164)."""
    y = np.asarray(y, dtype=np.complex128)
    v = np.array(v0, dtype=np.float64, copy=True)
    S = np.array(S0, dtype=np.complex128, copy=True)
    trace, history = [], []
    counts = dict(frame_matrix_inversions=0, frame_matrix_products=0, bin_gevd_count=0,
                  bin_matrix_products=0)
    if compute_likelihood:
        trace.append(fca_log_likelihood(y, v, S))
    mu = None
    for _ in range(int(iterations)):
        Sinv = cholesky_inverse(S)
        mu, v, S_raw, ninv, nprod = fca_iteration(y, v, S, Sinv, floor)
        S = regularize_covariances(S_raw)
        counts["frame_matrix_inversions"] += ninv
        counts["frame_matrix_products"] += nprod
        _require_finite(mu)
        if compute_likelihood:
            trace.append(fca_log_likelihood(y, v, S))
        if record_history:
            history.append({"v": v.copy(), "S": S.copy()})
    if mu is None:
        mu, _, ninv, nprod = fca_e_step(y, v, S)
        counts["frame_matrix_inversions"] += ninv
        counts["frame_matrix_products"] += nprod
    return OracleResult("FCA", mu, trace, v, S, np.asarray(floor), history, counts)


def scale_dev(a, b):
    """max|a-b| / max|b| (reference tests/test_acceptance.py:34-35)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
