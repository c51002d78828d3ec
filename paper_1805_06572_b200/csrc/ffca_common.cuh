// Common device helpers for the B200 FCA / FastFCA EM kernels.
//
// Complex numbers are double2 / float2 (x = re, y = im). Small per-bin
// matrices (order I <= 8) live in per-thread arrays indexed by compile-time
// constants (every loop over I is unrolled), so for I <= 4 they stay in
// registers.
#pragma once

// Jacobi rotation threshold (squared): rotate (p, q) while
// |a_pq|^2 > FFCA_JACOBI_TOL2 |a_pp a_qq| (Demmel-Veselic relative criterion)
#ifndef FFCA_JACOBI_TOL2
#define FFCA_JACOBI_TOL2 1e-32
#endif


#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fastfca_b200.h"

#define FFCA_DEV __device__ __forceinline__

namespace ffca {

constexpr int kMaxOrder = 8;
constexpr double kLogPi = 1.1447298858494002;  // log(pi)
constexpr double kCovEps = 1e-9;               // reference modelops.py:9
constexpr double kDefFloor = 1e-12;            // reference pencil.py:25
constexpr double kHermRtol = 1e-10;            // reference pencil.py:22

// ---- fast FP64 reciprocal / reciprocal square root --------------------------
// MUFU seed (rcp/rsqrt.approx.ftz.f64) + two Newton steps: ~1 ulp, no IEEE
// division / sqrt subroutine (special-case branches) on the per-point paths.
// Non-positive / non-finite inputs give non-finite or meaningless results;
// callers test the input (d > 0) themselves.
FFCA_DEV double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
FFCA_DEV double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double e = fma(-x * y, y, 1.0);  // 1 - x y^2
    y = fma(0.5 * y, e, y);
  }
  return y;
}

// ---- complex arithmetic --------------------------------------------------
FFCA_DEV double2 cmk(double re, double im) { return make_double2(re, im); }
// sum_{c < n} src[c * stride] in the fixed order ((s_0 + s_1) + s_2) + ...
// (bitwise equal to the plain loop), with the loads issued in batches of 8 so
// their latencies overlap instead of forming one load -> add chain
FFCA_DEV double ordered_sum(const double* __restrict__ src, int n, size_t stride) {
  double s = 0.0;
  for (int c = 0; c < n; c += 8) {
    double t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = (c + k < n) ? src[(size_t)(c + k) * stride] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (c + k < n) s += t[k];
  }
  return s;
}

FFCA_DEV double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
FFCA_DEV double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
FFCA_DEV double2 cconj(double2 a) { return cmk(a.x, -a.y); }
FFCA_DEV double2 cscale(double2 a, double s) { return cmk(a.x * s, a.y * s); }
FFCA_DEV double2 cmul(double2 a, double2 b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
FFCA_DEV double2 cmulc(double2 a, double2 b) {
  return cmk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// conj(a) * b
FFCA_DEV double2 cconjmul(double2 a, double2 b) {
  return cmk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
FFCA_DEV double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// Fused complex multiply-accumulates: 4 DFMA per complex MAC instead of the
// DMUL + DFMA + DADD per component that s + a*b compiles to (the compiler may
// not reassociate s + (p - q)); rounding differs from the unfused form at the
// last-bit level.
FFCA_DEV double2 cmac(double2 s, double2 a, double2 b) {  // s + a b
  return cmk(fma(a.x, b.x, fma(-a.y, b.y, s.x)), fma(a.x, b.y, fma(a.y, b.x, s.y)));
}
FFCA_DEV double2 cmsub(double2 s, double2 a, double2 b) {  // s - a b
  return cmk(fma(-a.x, b.x, fma(a.y, b.y, s.x)), fma(-a.x, b.y, fma(-a.y, b.x, s.y)));
}
FFCA_DEV double2 cmsubc(double2 s, double2 a, double2 b) {  // s - a conj(b)
  return cmk(fma(-a.x, b.x, fma(-a.y, b.y, s.x)), fma(-a.y, b.x, fma(a.x, b.y, s.y)));
}
FFCA_DEV double2 cmac_cj(double2 s, double2 a, double2 b) {  // s + conj(a) b
  return cmk(fma(a.x, b.x, fma(a.y, b.y, s.x)), fma(a.x, b.y, fma(-a.y, b.x, s.y)));
}
FFCA_DEV double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return cmk((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.x * r + b.y;
    return cmk((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}
FFCA_DEV double2 to_c128(double2 a) { return a; }
FFCA_DEV double2 to_c128(float2 a) { return cmk((double)a.x, (double)a.y); }

template <typename C>
struct CplxOf;
template <>
struct CplxOf<double> {
  using type = double2;
};
template <>
struct CplxOf<float> {
  using type = float2;
};

template <typename R>
FFCA_DEV typename CplxOf<R>::type from_c128(double2 a);
template <>
FFCA_DEV double2 from_c128<double>(double2 a) {
  return a;
}
template <>
FFCA_DEV float2 from_c128<float>(double2 a) {
  return make_float2((float)a.x, (float)a.y);
}

// ---- packed Hermitian storage ---------------------------------------------
// I real diagonal entries followed by the strictly-upper entries (row-major
// a < b) as (re, im) pairs: exactly I*I doubles.
template <int I>
struct Herm {
  static constexpr int NP = I * I;
  static constexpr int NOFF = I * (I - 1) / 2;
  FFCA_DEV static constexpr int off(int a, int b) {
    // index of pair (a, b), a < b, in row-major upper order
    return a * I - a * (a + 1) / 2 + (b - a - 1);
  }
  FFCA_DEV static constexpr int re(int a, int b) { return I + 2 * off(a, b); }
  FFCA_DEV static constexpr int im(int a, int b) { return I + 2 * off(a, b) + 1; }
};

template <int I>
FFCA_DEV void unpack_herm(const double (&p)[I * I], double2 (&A)[I][I]) {
#pragma unroll
  for (int a = 0; a < I; ++a) {
    A[a][a] = cmk(p[a], 0.0);
#pragma unroll
    for (int b = a + 1; b < I; ++b) {
      A[a][b] = cmk(p[Herm<I>::re(a, b)], p[Herm<I>::im(a, b)]);
      A[b][a] = cconj(A[a][b]);
    }
  }
}

// ---- error reporting -------------------------------------------------------
// First error wins by (iteration, code, index) order through a 64-bit
// atomicMin on  iter<<48 | code<<44 | index  (index < 2^44).
FFCA_DEV void report_error(ffca_status_dev* st, int iter, int code, unsigned long long index) {
  unsigned long long key = ((unsigned long long)(iter & 0xffff) << 48) |
                           ((unsigned long long)(code & 0xf) << 44) |
                           (index & ((1ull << 44) - 1));
  atomicMin(&st->first, key);
}
FFCA_DEV void report_min_value(ffca_status_dev* st, double val) {
  // running minimum of a double (definiteness: worst minimum eigenvalue)
  unsigned long long* addr = (unsigned long long*)&st->value;
  unsigned long long old = *addr, assumed;
  do {
    assumed = old;
    if (!(val < __longlong_as_double((long long)assumed))) break;
    old = atomicCAS(addr, assumed, (unsigned long long)__double_as_longlong(val));
  } while (assumed != old);
}

// ---- small dense routines (order I, compile-time) ---------------------------
template <int I>
FFCA_DEV void set_identity(double2 (&A)[I][I]) {
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) A[a][b] = cmk(a == b ? 1.0 : 0.0, 0.0);
}

// C = A * B
template <int I>
FFCA_DEV void matmul(const double2 (&A)[I][I], const double2 (&B)[I][I], double2 (&C)[I][I]) {
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) {
        acc = cmac(acc, A[a][k], B[k][b]);
      }
      C[a][b] = acc;
    }
}

// C = A^H * B
template <int I>
FFCA_DEV void matmul_hn(const double2 (&A)[I][I], const double2 (&B)[I][I], double2 (&C)[I][I]) {
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) {
        acc = cmac_cj(acc, A[k][a], B[k][b]);
      }
      C[a][b] = acc;
    }
}

// C = A * B^H
template <int I>
FFCA_DEV void matmul_nh(const double2 (&A)[I][I], const double2 (&B)[I][I], double2 (&C)[I][I]) {
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) {
        acc = cmac(acc, A[a][k], cconj(B[b][k]));
      }
      C[a][b] = acc;
    }
}

// Cyclic complex Jacobi on a Hermitian matrix (full storage). On exit A is
// diagonal (eigenvalues on the diagonal, real parts) and V holds the
// eigenvectors in its columns: A_in = V diag(A_out) V^H.
// Returns false when kJacobiSweeps sweeps did not converge (LAPACK's heevd
// reports that as "Eigenvalues did not converge"; a NaN input stops at once
// and is caught by the callers' finiteness / definiteness tests).
constexpr int kJacobiSweeps = 30;
template <int I>
FFCA_DEV bool jacobi_herm(double2 (&A)[I][I], double2 (&V)[I][I]) {
  set_identity<I>(V);
  if (I == 1) return true;
  // Rotate (p, q) only while |a_pq| exceeds eps * sqrt(|a_pp a_qq|) (the
  // Demmel-Veselic threshold: every eigenvalue then carries high relative
  // accuracy); stop after a sweep without rotations. A fixed "off(A) < tiny"
  // test would never trigger: rotations keep re-creating roundoff-level
  // off-diagonal entries.
  constexpr double kTol2 = FFCA_JACOBI_TOL2;
  for (int sweep = 0; sweep < kJacobiSweeps; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < I - 1; ++p) {
#pragma unroll
      for (int q = p + 1; q < I; ++q) {
        const double2 apq = A[p][q];
        const double mag2 = cabs2(apq);
        if (mag2 > kTol2 * fabs(A[p][p].x * A[q][q].x) && mag2 > 0.0) {
          rotated = true;
          // rotation parameters with MUFU seeds + Newton (rsqrt_fast /
          // rcp_fast, ~1 ulp): this chain is the latency of the per-bin
          // pencil refresh; c^2 + s^2 = 1 holds to rounding as before
          const double rmag = rsqrt_fast(mag2);
          const double mag = mag2 * rmag;
          // e^{-i phi} where apq = |apq| e^{i phi}
          const double2 emi = cmk(apq.x * rmag, -apq.y * rmag);
          const double app = A[p][p].x, aqq = A[q][q].x;
          const double theta = (aqq - app) * (0.5 * rmag);
          double t;
          if (fabs(theta) > 1e150) {
            t = 0.5 / theta;
          } else {
            const double h = fma(theta, theta, 1.0);
            t = rcp_fast(fabs(theta) + h * rsqrt_fast(h));
            if (theta < 0.0) t = -t;
          }
          const double c = rsqrt_fast(fma(t, t, 1.0));
          const double s = t * c;
          // columns p, q of A (rows k != p, q), mirrored into rows p, q
#pragma unroll
          for (int k = 0; k < I; ++k) {
            if (k == p || k == q) continue;
            const double2 akp = A[k][p];
            const double2 akq_r = cmul(A[k][q], emi);
            const double2 nkp = cmk(c * akp.x - s * akq_r.x, c * akp.y - s * akq_r.y);
            const double2 nkq = cmk(s * akp.x + c * akq_r.x, s * akp.y + c * akq_r.y);
            A[k][p] = nkp;
            A[k][q] = nkq;
            A[p][k] = cconj(nkp);
            A[q][k] = cconj(nkq);
          }
          A[p][p] = cmk(app - t * mag, 0.0);
          A[q][q] = cmk(aqq + t * mag, 0.0);
          A[p][q] = cmk(0.0, 0.0);
          A[q][p] = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) {
            const double2 vkp = V[k][p];
            const double2 vkq_r = cmul(V[k][q], emi);
            V[k][p] = cmk(c * vkp.x - s * vkq_r.x, c * vkp.y - s * vkq_r.y);
            V[k][q] = cmk(s * vkp.x + c * vkq_r.x, s * vkp.y + c * vkq_r.y);
          }
        }
      }
    }
    if (!rotated) return true;  // converged (NaN input also stops: comparisons fail)
  }
  return false;
}

// Sort eigenpairs descending (stable for equal keys is not needed).
template <int I>
FFCA_DEV void sort_desc(double (&w)[I], double2 (&V)[I][I]) {
#pragma unroll
  for (int i = 0; i < I; ++i) {
#pragma unroll
    for (int j = 0; j < I - 1 - i; ++j) {
      const bool sw = w[j] < w[j + 1];
      const double a = w[j], b = w[j + 1];
      w[j] = sw ? b : a;
      w[j + 1] = sw ? a : b;
#pragma unroll
      for (int k = 0; k < I; ++k) {
        const double2 x = V[k][j], y = V[k][j + 1];
        V[k][j] = sw ? y : x;
        V[k][j + 1] = sw ? x : y;
      }
    }
  }
}

// Rotate each column so its largest-magnitude entry (first on ties) is real
// positive (reference pencil.py:76-82).
template <int I>
FFCA_DEV void fix_column_phases(double2 (&P)[I][I]) {
#pragma unroll
  for (int k = 0; k < I; ++k) {
    double best = cabs2(P[0][k]);
    double2 lead = P[0][k];
#pragma unroll
    for (int i = 1; i < I; ++i) {
      const double m = cabs2(P[i][k]);
      if (m > best) {
        best = m;
        lead = P[i][k];
      }
    }
    const double mag = sqrt(best);
    if (mag > 0.0) {
      const double2 cph = cmk(lead.x / mag, -lead.y / mag);  // conj(phase)
#pragma unroll
      for (int i = 0; i < I; ++i) P[i][k] = cmul(P[i][k], cph);
    }
  }
}

// Hermitian-definite pencil decomposition, eigen-whitening variant (the
// reference's own construction, pencil.py:85-135): eig(Psi) -> definiteness
// floor -> whiten Phi -> eig -> descending -> P = U Sigma^{-1/2} Q -> column
// phases. Psi is read from its lower triangle (as LAPACK zheevd does for
// numpy.linalg.eigh); Phi is used in full. Returns 0, or 3 (definiteness)
// with *min_sigma set. Used when the Cholesky path below cannot certify
// definiteness cheaply.
template <int I>
FFCA_DEV int gevd_hpd_eig(const double2 (&Phi)[I][I], const double2 (&Psi)[I][I], double (&lam)[I],
                          double2 (&P)[I][I], double* min_sigma) {
  double2 A[I][I];
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < I; ++a) {
    tr += Psi[a][a].x;
#pragma unroll
    for (int b = 0; b < I; ++b) A[a][b] = (a > b) ? Psi[a][b] : (a == b ? cmk(Psi[a][a].x, 0.0) : cconj(Psi[b][a]));
  }
  double2 U[I][I];
  if (!jacobi_herm<I>(A, U)) return FFCA_ERR_NO_CONVERGENCE;
  double sig[I];
  double smin = 1e308;
#pragma unroll
  for (int a = 0; a < I; ++a) {
    sig[a] = A[a][a].x;
    smin = fmin(smin, sig[a]);
  }
  *min_sigma = smin;
  if (!(smin > kDefFloor * tr / I)) return FFCA_ERR_DEFINITENESS;
  double isq[I];
#pragma unroll
  for (int a = 0; a < I; ++a) isq[a] = 1.0 / sqrt(sig[a]);
  // W = diag(isq) U^H Phi U diag(isq), then re-symmetrise
  double2 T[I][I];
  matmul<I>(Phi, U, T);
  matmul_hn<I>(U, T, A);
  double2 W[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) W[a][b] = cscale(A[a][b], isq[a] * isq[b]);
#pragma unroll
  for (int a = 0; a < I; ++a) {
    W[a][a] = cmk(W[a][a].x, 0.0);
#pragma unroll
    for (int b = a + 1; b < I; ++b) {
      const double2 h = cmk(0.5 * (W[a][b].x + W[b][a].x), 0.5 * (W[a][b].y - W[b][a].y));
      W[a][b] = h;
      W[b][a] = cconj(h);
    }
  }
  double2 Q[I][I];
  if (!jacobi_herm<I>(W, Q)) return FFCA_ERR_NO_CONVERGENCE;
#pragma unroll
  for (int a = 0; a < I; ++a) lam[a] = W[a][a].x;
  sort_desc<I>(lam, Q);
  // P = U diag(isq) Q
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) T[a][b] = cscale(U[a][b], isq[b]);
  matmul<I>(T, Q, P);
  fix_column_phases<I>(P);
  return 0;
}

template <int I>
FFCA_DEV bool cholesky(const double2 (&A)[I][I], double2 (&L)[I][I]);
template <int I>
FFCA_DEV void tril_inverse(const double2 (&L)[I][I], double2 (&Li)[I][I]);
template <int I>
FFCA_DEV bool cholesky_fast(const double2 (&A)[I][I], double2 (&L)[I][I], double (&ild)[I]);
template <int I>
FFCA_DEV void tril_inverse_d(const double2 (&L)[I][I], const double (&ild)[I], double2 (&Li)[I][I]);

// Hermitian-definite pencil decomposition (reference pencil.py:85-135),
// Cholesky-whitened like LAPACK zhegv: Psi = L L^H, eig(L^-1 Phi L^-H) = Q
// diag(lam) Q^H, P = L^-H Q, descending order, column phases pinned. The
// generalized eigenpairs are the reference's (unique up to the pinned phase
// for distinct lam); one Jacobi eigensolve instead of two. Definiteness
// (reference: min eig(Psi) > 1e-12 tr(Psi)/D) is certified by the bound
// lambda_min(Psi) >= 1 / tr(Psi^-1) = 1 / ||L^-1||_F^2; when the bound cannot
// certify it, the exact eigenvalues decide (gevd_hpd_eig).
template <int I>
FFCA_DEV int gevd_hpd(const double2 (&Phi)[I][I], const double2 (&Psi)[I][I], double (&lam)[I],
                      double2 (&P)[I][I], double* min_sigma) {
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < I; ++a) tr += Psi[a][a].x;
  const double thr = kDefFloor * tr / I;
  double2 L[I][I], Li[I][I];
  double ild[I];
  bool certified = cholesky_fast<I>(Psi, L, ild);
  if (certified) {
    tril_inverse_d<I>(L, ild, Li);
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) s += cabs2(Li[a][b]);
    certified = (1.0 / s) > thr;
  }
  if (!certified) return gevd_hpd_eig<I>(Phi, Psi, lam, P, min_sigma);
  *min_sigma = 0.0;
  // Wh = Li Phi Li^H (Li lower triangular), re-symmetrised
  double2 T[I][I], Wh[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k <= a; ++k) acc = cmac(acc, Li[a][k], Phi[k][b]);
      T[a][b] = acc;
    }
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = a; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k <= b; ++k) acc = cmac(acc, T[a][k], cconj(Li[b][k]));
      Wh[a][b] = acc;
    }
#pragma unroll
  for (int a = 0; a < I; ++a) {
    Wh[a][a] = cmk(Wh[a][a].x, 0.0);
#pragma unroll
    for (int b = a + 1; b < I; ++b) Wh[b][a] = cconj(Wh[a][b]);
  }
  double2 Q[I][I];
  if (!jacobi_herm<I>(Wh, Q)) return FFCA_ERR_NO_CONVERGENCE;
#pragma unroll
  for (int a = 0; a < I; ++a) lam[a] = Wh[a][a].x;
  sort_desc<I>(lam, Q);
  // P = Li^H Q (Li^H upper triangular)
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = a; k < I; ++k) acc = cmac_cj(acc, Li[k][a], Q[k][b]);
      P[a][b] = acc;
    }
  fix_column_phases<I>(P);
  return 0;
}

// Gauss-Jordan inverse with partial pivoting; also log|det A|.
// Returns false when a pivot is exactly zero or non-finite.
template <int I>
FFCA_DEV bool lu_inverse(const double2 (&A)[I][I], double2 (&Inv)[I][I], double* logabsdet) {
  double2 M[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) M[a][b] = A[a][b];
  set_identity<I>(Inv);
  double lad = 0.0;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < I; ++k) {
    int r = k;
    double best = cabs2(M[k][k]);
#pragma unroll
    for (int i = k + 1; i < I; ++i) {
      const double m = cabs2(M[i][k]);
      if (m > best) {
        best = m;
        r = i;
      }
    }
#pragma unroll
    for (int i = k + 1; i < I; ++i) {
      if (i == r) {
#pragma unroll
        for (int j = 0; j < I; ++j) {
          double2 t = M[k][j];
          M[k][j] = M[i][j];
          M[i][j] = t;
          t = Inv[k][j];
          Inv[k][j] = Inv[i][j];
          Inv[i][j] = t;
        }
      }
    }
    if (!(best > 0.0) || !isfinite(best)) ok = false;
    lad += 0.5 * log(best);
    // 1 / m = conj(m) / |m|^2 (the pivot's |m|^2 is `best`; MUFU seed + Newton)
    const double ib = rcp_fast(best);
    const double2 ip = cmk(M[k][k].x * ib, -M[k][k].y * ib);
#pragma unroll
    for (int j = 0; j < I; ++j) {
      M[k][j] = cmul(M[k][j], ip);
      Inv[k][j] = cmul(Inv[k][j], ip);
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
      if (i == k) continue;
      const double2 fct = M[i][k];
#pragma unroll
      for (int j = 0; j < I; ++j) {
        M[i][j] = cmsub(M[i][j], fct, M[k][j]);
        Inv[i][j] = cmsub(Inv[i][j], fct, Inv[k][j]);
      }
    }
  }
  *logabsdet = lad;
  return ok;
}

// Cholesky A = L L^H of a Hermitian matrix given in full storage (lower
// triangle used). Returns false if a pivot is not strictly positive.
template <int I>
FFCA_DEV bool cholesky(const double2 (&A)[I][I], double2 (&L)[I][I]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < I; ++j) {
    double d = A[j][j].x;
#pragma unroll
    for (int k = 0; k < j; ++k) d -= cabs2(L[j][k]);
    if (!(d > 0.0)) ok = false;
    const double ljj = sqrt(fmax(d, 0.0));
    L[j][j] = cmk(ljj, 0.0);
    const double il = 1.0 / ljj;
#pragma unroll
    for (int i = j + 1; i < I; ++i) {
      double2 s = A[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = cmsubc(s, L[i][k], L[j][k]);
      L[i][j] = cscale(s, il);
    }
#pragma unroll
    for (int i = 0; i < j; ++i) L[i][j] = cmk(0.0, 0.0);
  }
  return ok;
}

// Cholesky for the per-point paths: as cholesky() but with rsqrt_fast and
// multiplications by the returned inverse diagonal (no IEEE sqrt / division).
template <int I>
FFCA_DEV bool cholesky_fast(const double2 (&A)[I][I], double2 (&L)[I][I], double (&ild)[I]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < I; ++j) {
    double d = A[j][j].x;
#pragma unroll
    for (int k = 0; k < j; ++k) d -= cabs2(L[j][k]);
    if (!(d > 0.0)) ok = false;
    const double il = rsqrt_fast(d);
    ild[j] = il;
    L[j][j] = cmk(d * il, 0.0);
#pragma unroll
    for (int i = j + 1; i < I; ++i) {
      double2 s = A[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = cmsubc(s, L[i][k], L[j][k]);
      L[i][j] = cscale(s, il);
    }
#pragma unroll
    for (int i = 0; i < j; ++i) L[i][j] = cmk(0.0, 0.0);
  }
  return ok;
}
// tril_inverse with the inverse diagonal given (from cholesky_fast)
template <int I>
FFCA_DEV void tril_inverse_d(const double2 (&L)[I][I], const double (&ild)[I], double2 (&Li)[I][I]) {
#pragma unroll
  for (int c = 0; c < I; ++c) {
#pragma unroll
    for (int r = 0; r < I; ++r) {
      if (r < c) {
        Li[r][c] = cmk(0.0, 0.0);
        continue;
      }
      double2 s = cmk(r == c ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int k = c; k < r; ++k) s = cmsub(s, L[r][k], Li[k][c]);
      Li[r][c] = cscale(s, ild[r]);
    }
  }
}

// In-place inverse of a Hermitian positive-definite matrix in packed storage
// (Herm<I>) by the symmetric sweep operator, no pivoting: sweeping pivot k
// maps a_kk -> -1/a_kk, a_ik -> a_ik/a_kk, a_ij -> a_ij - a_ik a_kj/a_kk, every
// intermediate stays Hermitian (only the packed half is touched) and after
// all I sweeps the array holds -A^-1 (negated on return). The pivots are the
// LDL^H pivots of A (the squared Cholesky diagonal): A is positive definite
// iff all are > 0, and det A is their product. 24 FP64 operations per pivot at
// I = 4 against Cholesky + triangular inverse + L^-H L^-1
// (about half the work, and no L / L^-1 register arrays).
template <int I>
FFCA_DEV bool herm_sweep_inverse(double (&A)[I * I], double& pivprod) {
  using H = Herm<I>;
  bool ok = true;
  pivprod = 1.0;
#pragma unroll
  for (int k = 0; k < I; ++k) {
    const double pk = A[k];
    if (!(pk > 0.0)) ok = false;
    pivprod *= pk;
    const double d = rcp_fast(pk);
    double2 c[I], s[I];  // column k (entries A[i][k], i != k) and d * column k
#pragma unroll
    for (int i = 0; i < I; ++i) {
      if (i == k) continue;
      c[i] = i < k ? cmk(A[H::re(i, k)], A[H::im(i, k)]) : cmk(A[H::re(k, i)], -A[H::im(k, i)]);
      s[i] = cscale(c[i], d);
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
      if (i == k) continue;
      A[i] = fma(-s[i].x, c[i].x, fma(-s[i].y, c[i].y, A[i]));
#pragma unroll
      for (int j = i + 1; j < I; ++j) {
        if (j == k) continue;
        // A[i][j] -= s_i conj(c_j)
        A[H::re(i, j)] = fma(-s[i].x, c[j].x, fma(-s[i].y, c[j].y, A[H::re(i, j)]));
        A[H::im(i, j)] = fma(-s[i].y, c[j].x, fma(s[i].x, c[j].y, A[H::im(i, j)]));
      }
    }
#pragma unroll
    for (int i = 0; i < I; ++i) {
      if (i == k) continue;
      if (i < k) {
        A[H::re(i, k)] = s[i].x;
        A[H::im(i, k)] = s[i].y;
      } else {
        A[H::re(k, i)] = s[i].x;
        A[H::im(k, i)] = -s[i].y;
      }
    }
    A[k] = -d;
  }
#pragma unroll
  for (int e = 0; e < I * I; ++e) A[e] = -A[e];
  return ok;
}

// Inverse of a lower-triangular matrix (forward substitution per column).
template <int I>
FFCA_DEV void tril_inverse(const double2 (&L)[I][I], double2 (&Li)[I][I]) {
#pragma unroll
  for (int c = 0; c < I; ++c) {
#pragma unroll
    for (int r = 0; r < I; ++r) {
      if (r < c) {
        Li[r][c] = cmk(0.0, 0.0);
        continue;
      }
      double2 s = cmk(r == c ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int k = c; k < r; ++k) s = cmsub(s, L[r][k], Li[k][c]);
      Li[r][c] = cscale(s, 1.0 / L[r][r].x);
    }
  }
}

}  // namespace ffca
