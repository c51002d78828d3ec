/*
 * CPU oracle port of the reference's per-(n, f) EM kernels — TEST
 * INFRASTRUCTURE / CPU BASELINE ONLY (never linked into the product).
 *
 * Plain C restatement of the loops in the reference numba backend
 * (/root/reference/pkg/src/fastfca/_kernels_numba.py):
 *   ffo_fast_iteration  <- _fast_iteration  (:328-391)
 *   ffo_fca_iteration   <- _fca_iteration   (:246-325), with np.linalg.inv
 *                          restated as Gauss-Jordan with partial pivoting
 * extended with a leading mixture axis and an OpenMP loop over independent
 * (mixture, bin) pairs — the reference is bin-shard invariant, so this is the
 * same arithmetic per bin, run on all host cores. Layouts are the
 * reference's: y (M,N,F,I), v (M,2,N,F), P (M*F,I,I), lam (M*F,I),
 * floor (M*F), S / Sinv / S_raw (M,2,F,I,I), mu (M,2,N,F,I).
 * Used by oracle/cpu_port.py for bench.py's cpu_baseline and --impl
 * reference legs; parity of this port against the numpy oracle is checked in
 * tests/test_cpu_port.py.
 */
#include <complex.h>
#undef I /* the channel count is called I here, as in the reference */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef double complex cplx;

#define MAXI 8

#ifdef _OPENMP
#include <omp.h>
#endif

int ffo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ffo_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

void ffo_fast_iteration(const cplx* y, const cplx* P, const double* v, const double* lam,
                        const double* floor_, int64_t M, int64_t N, int64_t F, int I,
                        cplx* mu, double* v_new, cplx* S_raw) {
  const int64_t G = M * F;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t g = 0; g < G; ++g) {
    const int64_t m = g / F, f = g % F;
    const cplx* Pf = P + g * I * I;
    const double* lam_f = lam + g * I;
    const double floor_f = floor_[g];
    cplx S1f[MAXI * MAXI], S2f[MAXI * MAXI];
    cplx m1[MAXI], m2[MAXI];
    double cdiag[MAXI];
    for (int e = 0; e < I * I; ++e) S1f[e] = S2f[e] = 0.0;
    for (int64_t n = 0; n < N; ++n) {
      const cplx* yn = y + ((m * N + n) * F + f) * I;
      const double v1 = v[(m * 2 + 0) * N * F + n * F + f];
      const double v2 = v[(m * 2 + 1) * N * F + n * F + f];
      double tr1 = 0.0, tr2 = 0.0;
      for (int a = 0; a < I; ++a) {
        cplx acc = 0.0;
        for (int b = 0; b < I; ++b) acc += conj(Pf[b * I + a]) * yn[b];
        const double la = lam_f[a];
        const double den = v1 * la + v2;
        const double g1 = v1 * la / den;
        const double g2 = v2 / den;
        m1[a] = g1 * acc;
        m2[a] = g2 * acc;
        const double c = v2 * g1;
        cdiag[a] = c;
        const double p_yy = creal(acc) * creal(acc) + cimag(acc) * cimag(acc);
        tr1 += (g1 * g1 * p_yy + c) / la;
        tr2 += g2 * g2 * p_yy + c;
      }
      const double w1 = fmax(tr1 / I, floor_f);
      const double w2 = fmax(tr2 / I, floor_f);
      v_new[(m * 2 + 0) * N * F + n * F + f] = w1;
      v_new[(m * 2 + 1) * N * F + n * F + f] = w2;
      const double iw1 = 1.0 / w1, iw2 = 1.0 / w2;
      for (int a = 0; a < I; ++a) {
        if (mu) {
          mu[(((m * 2 + 0) * N + n) * F + f) * I + a] = m1[a];
          mu[(((m * 2 + 1) * N + n) * F + f) * I + a] = m2[a];
        }
        const cplx m1a = m1[a] * iw1, m2a = m2[a] * iw2;
        for (int b = 0; b < I; ++b) {
          S1f[a * I + b] += m1a * conj(m1[b]);
          S2f[a * I + b] += m2a * conj(m2[b]);
        }
        S1f[a * I + a] += cdiag[a] * iw1;
        S2f[a * I + a] += cdiag[a] * iw2;
      }
    }
    for (int e = 0; e < I * I; ++e) {
      S_raw[((m * 2 + 0) * F + f) * I * I + e] = S1f[e] / (double)N;
      S_raw[((m * 2 + 1) * F + f) * I * I + e] = S2f[e] / (double)N;
    }
  }
}

/* Gauss-Jordan inverse with partial pivoting; returns 0 if singular. */
static int inv_gj(const cplx* A, cplx* X, int I) {
  cplx W[MAXI * MAXI];
  memcpy(W, A, sizeof(cplx) * I * I);
  for (int i = 0; i < I; ++i)
    for (int j = 0; j < I; ++j) X[i * I + j] = (i == j) ? 1.0 : 0.0;
  for (int k = 0; k < I; ++k) {
    int r = k;
    double best = cabs(W[k * I + k]);
    for (int i = k + 1; i < I; ++i)
      if (cabs(W[i * I + k]) > best) {
        best = cabs(W[i * I + k]);
        r = i;
      }
    if (best == 0.0) return 0;
    if (r != k)
      for (int j = 0; j < I; ++j) {
        cplx t = W[k * I + j];
        W[k * I + j] = W[r * I + j];
        W[r * I + j] = t;
        t = X[k * I + j];
        X[k * I + j] = X[r * I + j];
        X[r * I + j] = t;
      }
    const cplx ip = 1.0 / W[k * I + k];
    for (int j = 0; j < I; ++j) {
      W[k * I + j] *= ip;
      X[k * I + j] *= ip;
    }
    for (int i = 0; i < I; ++i) {
      if (i == k) continue;
      const cplx fct = W[i * I + k];
      if (fct == 0.0) continue;
      for (int j = 0; j < I; ++j) {
        W[i * I + j] -= fct * W[k * I + j];
        X[i * I + j] -= fct * X[k * I + j];
      }
    }
  }
  return 1;
}

/* Returns -1 on success, else the flat (m, n, f) index of the first singular
 * point (numba's np.linalg.inv raises there). */
int64_t ffo_fca_iteration(const cplx* y, const double* v, const cplx* S, const cplx* Sinv,
                          const double* floor_, int64_t M, int64_t N, int64_t F, int I, cplx* mu,
                          double* v_new, cplx* S_raw) {
  const int64_t G = M * F;
  int64_t bad = -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t g = 0; g < G; ++g) {
    const int64_t m = g / F, f = g % F;
    const cplx* S1 = S + ((m * 2 + 0) * F + f) * I * I;
    const cplx* S2 = S + ((m * 2 + 1) * F + f) * I * I;
    const cplx* Si1 = Sinv + ((m * 2 + 0) * F + f) * I * I;
    const cplx* Si2 = Sinv + ((m * 2 + 1) * F + f) * I * I;
    cplx R[MAXI * MAXI], Rinv[MAXI * MAXI], A1[MAXI * MAXI], A2[MAXI * MAXI],
        cross[MAXI * MAXI];
    cplx S1n[MAXI * MAXI], S2n[MAXI * MAXI];
    cplx mu1[MAXI], mu2[MAXI];
    for (int e = 0; e < I * I; ++e) S1n[e] = S2n[e] = 0.0;
    for (int64_t n = 0; n < N; ++n) {
      const cplx* yn = y + ((m * N + n) * F + f) * I;
      const double v1 = v[(m * 2 + 0) * N * F + n * F + f];
      const double v2 = v[(m * 2 + 1) * N * F + n * F + f];
      for (int a = 0; a < I; ++a)
        for (int b = 0; b < I; ++b) R[a * I + b] = v1 * S1[a * I + b] + v2 * S2[a * I + b];
      if (!inv_gj(R, Rinv, I)) {
#pragma omp critical
        {
          const int64_t key = (m * N + n) * F + f;
          if (bad < 0 || key < bad) bad = key;
        }
        break;
      }
      for (int a = 0; a < I; ++a)
        for (int b = 0; b < I; ++b) {
          cplx acc1 = 0.0, acc2 = 0.0;
          for (int c = 0; c < I; ++c) {
            acc1 += S1[a * I + c] * Rinv[c * I + b];
            acc2 += S2[a * I + c] * Rinv[c * I + b];
          }
          A1[a * I + b] = acc1;
          A2[a * I + b] = acc2;
        }
      for (int a = 0; a < I; ++a) {
        cplx acc1 = 0.0, acc2 = 0.0;
        for (int b = 0; b < I; ++b) {
          acc1 += A1[a * I + b] * yn[b];
          acc2 += A2[a * I + b] * yn[b];
        }
        mu1[a] = v1 * acc1;
        mu2[a] = v2 * acc2;
      }
      for (int a = 0; a < I; ++a)
        for (int b = 0; b < I; ++b) {
          cplx acc = 0.0;
          for (int c = 0; c < I; ++c) acc += A1[a * I + c] * S2[c * I + b];
          cross[a * I + b] = v1 * v2 * acc;
        }
      double tr1 = 0.0, tr2 = 0.0;
      for (int a = 0; a < I; ++a)
        for (int b = 0; b < I; ++b) {
          const cplx phi1 = mu1[b] * conj(mu1[a]) + cross[b * I + a];
          const cplx phi2 = mu2[b] * conj(mu2[a]) + cross[b * I + a];
          tr1 += creal(Si1[a * I + b] * phi1);
          tr2 += creal(Si2[a * I + b] * phi2);
        }
      const double w1 = fmax(tr1 / I, floor_[g]);
      const double w2 = fmax(tr2 / I, floor_[g]);
      v_new[(m * 2 + 0) * N * F + n * F + f] = w1;
      v_new[(m * 2 + 1) * N * F + n * F + f] = w2;
      for (int a = 0; a < I; ++a) {
        if (mu) {
          mu[(((m * 2 + 0) * N + n) * F + f) * I + a] = mu1[a];
          mu[(((m * 2 + 1) * N + n) * F + f) * I + a] = mu2[a];
        }
        for (int b = 0; b < I; ++b) {
          const cplx phi1 = mu1[a] * conj(mu1[b]) + cross[a * I + b];
          const cplx phi2 = mu2[a] * conj(mu2[b]) + cross[a * I + b];
          S1n[a * I + b] += phi1 / w1;
          S2n[a * I + b] += phi2 / w2;
        }
      }
    }
    for (int e = 0; e < I * I; ++e) {
      S_raw[((m * 2 + 0) * F + f) * I * I + e] = S1n[e] / (double)N;
      S_raw[((m * 2 + 1) * F + f) * I * I + e] = S2n[e] / (double)N;
    }
  }
  return bad;
}
