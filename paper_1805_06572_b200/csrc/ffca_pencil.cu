// K1 — per-bin pencil refresh for FastFCA, one thread per (mixture, bin):
//   sum the frame-chunk partials of S~ (fixed order) and divide by N,
//   ridge with eps * P^H P (fast.py:80-90: the image of FCA's eps*I ridge),
//   back-transform S = P^{-H} S~ P^{-1} for the model / history
//   (fast.py:144-148), Hermitian-definite GEVD of (S~1, S~2)
//   (pencil.py:85-135), P <- P Q (fast.py:107-113), P^{-H} and log|det P|^2
//   for the next pass (fast.py:151-153).
// Plus the stand-alone batched per-bin routines of the C ABI.
#include <cstdlib>

#include "ffca_internal.cuh"
#include "ffca_pencil_body.cuh"

namespace ffca {

#ifndef FFCA_K1_MINB
#define FFCA_K1_MINB 1  // CTAs per SM the one-thread-per-bin refresh is budgeted for
#endif
// Threads per CTA of the one-thread-per-bin refresh. Each thread runs ~5k
// straight-line instructions once, so on the few-bin configs (513 bins:
// 9 CTAs of 64) the pass is instruction-fetch bound (ncu stall_no_instruction
// 4.2 per issue): larger CTAs put more warps behind every i-cache fill.
#ifndef FFCA_K1_THREADS
#define FFCA_K1_THREADS 64
#endif
template <int I>
__global__ void __launch_bounds__(FFCA_K1_THREADS, FFCA_K1_MINB) pencil_update_kernel(const PencilParams p) {
  const int64_t g = p.g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= window_end(p.g1, p.G)) {
    // (griddepcontrol.launch_dependents counts per CTA: a bin-less thread must
    // not release the next pass before the pass this kernel depends on is done)
    if (p.pdl_wait) pdl_wait_primary();
    return;
  }
  pencil_update_body<I>(p, g, PdlGateSum{p.pdl_wait != 0});
}

// split path, step 1: S_t -> scratch [2][G][I][I]
template <int I>
__global__ void __launch_bounds__(64) pencil_prep_kernel(const PencilParams p) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.G) return;
  double2 S1[I][I], S2[I][I], Pe[I][I];
  pencil_prep<I>(p, g, S1, S2, Pe);
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      p.St[g * NP + a * I + b] = S1[a][b];
      p.St[(p.G + g) * NP + a * I + b] = S2[a][b];
    }
}

template <int I>
__global__ void __launch_bounds__(64)
    initial_pencil_kernel(const double2* __restrict__ S0, double2* P, double2* W, double* lam,
                          double* logdet2, int64_t G, int64_t F, ffca_status_dev* st) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int64_t m = (unsigned)g / (unsigned)F, f = g - m * F;  // (32-bit division)
  double2 A[I][I], B[I][I];
  const double2* s1 = S0 + ((m * 2 + 0) * F + f) * NP;
  const double2* s2 = S0 + ((m * 2 + 1) * F + f) * NP;
  double sc1 = 0.0, sc2 = 0.0, as1 = 0.0, as2 = 0.0;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      A[a][b] = s1[a * I + b];
      B[a][b] = s2[a * I + b];
    }
  // _check_hermitian (pencil.py:40-51)
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      sc1 = fmax(sc1, sqrt(cabs2(A[a][b])));
      sc2 = fmax(sc2, sqrt(cabs2(B[a][b])));
      as1 = fmax(as1, sqrt(cabs2(csub(A[a][b], cconj(A[b][a])))));
      as2 = fmax(as2, sqrt(cabs2(csub(B[a][b], cconj(B[b][a])))));
    }
  if ((as1 > kHermRtol * fmax(sc1, 1e-300)) || (as2 > kHermRtol * fmax(sc2, 1e-300))) {
    if (st) report_error(st, 0, FFCA_ERR_NON_HERMITIAN, (unsigned long long)g);
  }
  double l[I];
  double2 Pn[I][I];
  double msig = 0.0;
  const int rc = gevd_hpd<I>(A, B, l, Pn, &msig);
  if (rc != 0 && st) {
    report_error(st, 0, rc, (unsigned long long)g);
    report_min_value(st, msig);
  }
  double2 Inv[I][I];
  double lad = 0.0;
  lu_inverse<I>(Pn, Inv, &lad);
#pragma unroll
  for (int a = 0; a < I; ++a) {
    lam[g * I + a] = l[a];
#pragma unroll
    for (int b = 0; b < I; ++b) {
      P[g * NP + a * I + b] = Pn[a][b];
      W[g * NP + a * I + b] = cconj(Inv[b][a]);
    }
  }
  logdet2[g] = 2.0 * lad;
}

#define FFCA_DISPATCH_I(I, CALL)   \
  switch (I) {                     \
    case 1: {                      \
      constexpr int II = 1;        \
      CALL;                        \
    } break;                       \
    case 2: {                      \
      constexpr int II = 2;        \
      CALL;                        \
    } break;                       \
    case 3: {                      \
      constexpr int II = 3;        \
      CALL;                        \
    } break;                       \
    case 4: {                      \
      constexpr int II = 4;        \
      CALL;                        \
    } break;                       \
    case 5: {                      \
      constexpr int II = 5;        \
      CALL;                        \
    } break;                       \
    case 6: {                      \
      constexpr int II = 6;        \
      CALL;                        \
    } break;                       \
    case 7: {                      \
      constexpr int II = 7;        \
      CALL;                        \
    } break;                       \
    case 8: {                      \
      constexpr int II = 8;        \
      CALL;                        \
    } break;                       \
    default:                       \
      return cudaErrorInvalidValue; \
  }

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <int I>
__global__ void gevd_batch_kernel(const double2* Phi, const double2* Psi, double* lam,
                                  double2* P, const double2* Pprev, int64_t B, int check,
                                  ffca_status_dev* st, int iter);
template <int I>
__global__ void inverse_h_kernel(const double2* P, double2* W, double* logdet2, int64_t B,
                                 ffca_status_dev* st, int iter);

cudaError_t launch_pencil_par(const PencilParams& p, int I, cudaStream_t s);
cudaError_t launch_initial_par(const double2* S0, double2* P, double2* W, double* lam,
                               double* logdet2, int64_t G, int64_t F, int I, ffca_status_dev* st,
                               cudaStream_t s);

// Which per-bin kernel: the lane-parallel one (ffca_pencil_par.cu) for
// I >= 5 (no register spills) and for I = 4 with few bins (latency bound:
// config 4, 46 vs 65 us); the one-thread-per-bin kernel for I <= 3 at any
// size (configs 0/1: 0.28 vs 0.34 ms and 2.25 vs 2.66 ms per run) and for
// big I = 4 batches. FFCA_K1=par|thread overrides (experiments).
static bool use_par(int64_t G, int I);
bool pencil_window_capable(int64_t G, int I) { return use_par(G, I) || I <= 4; }
static bool use_par(int64_t G, int I) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("FFCA_K1");
    mode = (e && e[0] == 'p') ? 1 : ((e && e[0] == 't') ? 2 : 0);
  }
  if (mode == 1) return true;
  if (mode == 2) return I >= 5;
  return I >= 5 || (I == 4 && G < 16384);
}

// whether launch_pencil_update takes the one-thread-per-bin kernel (which honours
// PencilParams::pdl_wait)
bool pencil_thread_kernel(int64_t G, int I) { return !use_par(G, I) && I <= 4; }

cudaError_t launch_pencil_update(const PencilParams& p, int I, cudaStream_t s) {
  if (use_par(p.G, I)) return launch_pencil_par(p, I, s);
  if (I <= 4) {  // fused single kernel; only instantiated for I <= 4
    constexpr int T = FFCA_K1_THREADS;
    const unsigned nb = nblk(window_end(p.g1, p.G) - p.g0, T);
    switch (I) {
      case 1: return launch_ex(pencil_update_kernel<1>, dim3(nb), dim3(T), 0, s, p.pdl_wait != 0, p.prio, p);
      case 2: return launch_ex(pencil_update_kernel<2>, dim3(nb), dim3(T), 0, s, p.pdl_wait != 0, p.prio, p);
      case 3: return launch_ex(pencil_update_kernel<3>, dim3(nb), dim3(T), 0, s, p.pdl_wait != 0, p.prio, p);
      default: return launch_ex(pencil_update_kernel<4>, dim3(nb), dim3(T), 0, s, p.pdl_wait != 0, p.prio, p);
    }
    return cudaGetLastError();
  }
  // I >= 5: three leaner kernels (S_t, GEVD + P Q, P^{-H} + log|det P|^2)
  const unsigned nb = nblk(p.G, 64);
  const double2* St1 = p.St;
  const double2* St2 = p.St + p.G * (int64_t)I * I;
  FFCA_DISPATCH_I(I, (pencil_prep_kernel<II><<<nb, 64, 0, s>>>(p)));
  FFCA_DISPATCH_I(I, (gevd_batch_kernel<II><<<nb, 64, 0, s>>>(St1, St2, p.lam, p.P, p.P, p.G, 0,
                                                              p.st, p.iter)));
  FFCA_DISPATCH_I(I, (inverse_h_kernel<II><<<nb, 64, 0, s>>>(p.P, p.W, p.logdet2, p.G, p.st,
                                                             p.iter)));
  return cudaGetLastError();
}

cudaError_t launch_initial_pencil(const double2* S0, double2* P, double2* W, double* lam,
                                  double* logdet2, int64_t G, int64_t F, int I,
                                  ffca_status_dev* st, cudaStream_t s) {
  if (use_par(G, I)) return launch_initial_par(S0, P, W, lam, logdet2, G, F, I, st, s);
  FFCA_DISPATCH_I(I, (initial_pencil_kernel<II><<<nblk(G, 64), 64, 0, s>>>(S0, P, W, lam,
                                                                            logdet2, G, F, st)));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Stand-alone batched per-bin routines (C ABI stage level)
// ---------------------------------------------------------------------------
template <int I>
__global__ void gevd_batch_kernel(const double2* Phi, const double2* Psi, double* lam,
                                  double2* P, const double2* Pprev, int64_t B, int check,
                                  ffca_status_dev* st, int iter) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B) return;
  double2 A[I][I], Bm[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      A[a][b] = Phi[g * NP + a * I + b];
      Bm[a][b] = Psi[g * NP + a * I + b];
    }
  if (check) {
    double sc1 = 0.0, sc2 = 0.0, as1 = 0.0, as2 = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        sc1 = fmax(sc1, sqrt(cabs2(A[a][b])));
        sc2 = fmax(sc2, sqrt(cabs2(Bm[a][b])));
        as1 = fmax(as1, sqrt(cabs2(csub(A[a][b], cconj(A[b][a])))));
        as2 = fmax(as2, sqrt(cabs2(csub(Bm[a][b], cconj(Bm[b][a])))));
      }
    if ((as1 > kHermRtol * fmax(sc1, 1e-300)) || (as2 > kHermRtol * fmax(sc2, 1e-300))) {
      if (st) report_error(st, iter, FFCA_ERR_NON_HERMITIAN, (unsigned long long)g);
      return;
    }
  }
  double l[I];
  double2 Q[I][I];
  double msig = 0.0;
  const int rc = gevd_hpd<I>(A, Bm, l, Q, &msig);
  if (rc != 0 && st) {
    report_error(st, iter, rc, (unsigned long long)g);
    report_min_value(st, msig);
  }
  if (Pprev) {
    double2 Pp[I][I], Pn[I][I];
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) Pp[a][b] = Pprev[g * NP + a * I + b];
    matmul<I>(Pp, Q, Pn);
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) Q[a][b] = Pn[a][b];
  }
#pragma unroll
  for (int a = 0; a < I; ++a) {
    lam[g * I + a] = l[a];
#pragma unroll
    for (int b = 0; b < I; ++b) P[g * NP + a * I + b] = Q[a][b];
  }
}

template <int I>
__global__ void cholinv_kernel(const double2* S, double2* Sinv, int64_t B, ffca_status_dev* st) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B) return;
  double2 A[I][I], L[I][I], Li[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) A[a][b] = S[g * NP + a * I + b];
  if (!cholesky<I>(A, L) && st) report_error(st, 0, FFCA_ERR_NOT_PD, (unsigned long long)g);
  tril_inverse<I>(L, Li);
  // Sinv = Li^H Li
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) {
        if (k < a || k < b) continue;
        acc = cmac_cj(acc, Li[k][a], Li[k][b]);
      }
      Sinv[g * NP + a * I + b] = acc;
    }
}

// X = A^{-1} B per batch entry (reference pencil.py:138-157, which calls
// np.linalg.solve = LAPACK zgesv): LU with partial pivoting on |re| + |im|
// (zgetrf's izamax), one thread per system, then for each of the K right-hand
// sides the permuted forward / back substitution. Also writes ||A X - B||^2
// and ||B||^2 of the entry (norms[2g], norms[2g+1]) for the caller's residual
// test. An exactly zero pivot is zgetrf's "singular" -> FFCA_ERR_SINGULAR_MATRIX.
template <int I>
__global__ void solve_kernel(const double2* __restrict__ A, const double2* __restrict__ B,
                             double2* __restrict__ X, double* __restrict__ norms, int64_t batch,
                             int64_t K, ffca_status_dev* st) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= batch) return;
  double2 LU[I][I];
  int piv[I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) LU[a][b] = A[g * NP + a * I + b];
  bool singular = false;
#pragma unroll
  for (int k = 0; k < I; ++k) {
    int p = k;
    double best = fabs(LU[k][k].x) + fabs(LU[k][k].y);
#pragma unroll
    for (int r = k + 1; r < I; ++r) {
      const double c = fabs(LU[r][k].x) + fabs(LU[r][k].y);
      if (c > best) best = c, p = r;
    }
    piv[k] = p;
#pragma unroll
    for (int r = k + 1; r < I; ++r)  // swap rows k and p (compile-time indices)
      if (r == p) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          const double2 t = LU[k][c];
          LU[k][c] = LU[r][c];
          LU[r][c] = t;
        }
      }
    if (best == 0.0) {
      singular = true;
      continue;
    }
    const double2 inv = cdiv(cmk(1.0, 0.0), LU[k][k]);
#pragma unroll
    for (int r = k + 1; r < I; ++r) {
      const double2 l = cmul(LU[r][k], inv);
      LU[r][k] = l;
#pragma unroll
      for (int c = k + 1; c < I; ++c) LU[r][c] = cmsub(LU[r][c], l, LU[k][c]);
    }
  }
  if (singular) {
    if (st) report_error(st, 0, FFCA_ERR_SINGULAR_MATRIX, (unsigned long long)g);
    return;
  }
  double res2 = 0.0, nb2 = 0.0;
  for (int64_t j = 0; j < K; ++j) {
    double2 b0[I], x[I];
#pragma unroll
    for (int a = 0; a < I; ++a) b0[a] = x[a] = B[(g * I + a) * K + j];
#pragma unroll
    for (int k = 0; k < I; ++k)
#pragma unroll
      for (int r = k + 1; r < I; ++r)
        if (r == piv[k]) {
          const double2 t = x[k];
          x[k] = x[r];
          x[r] = t;
        }
#pragma unroll
    for (int r = 1; r < I; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) x[r] = cmsub(x[r], LU[r][c], x[c]);
#pragma unroll
    for (int r = I - 1; r >= 0; --r) {
#pragma unroll
      for (int c = r + 1; c < I; ++c) x[r] = cmsub(x[r], LU[r][c], x[c]);
      x[r] = cdiv(x[r], LU[r][r]);
    }
#pragma unroll
    for (int a = 0; a < I; ++a) {
      X[(g * I + a) * K + j] = x[a];
      double2 t = cmk(-b0[a].x, -b0[a].y);
#pragma unroll
      for (int c = 0; c < I; ++c) t = cmac(t, A[g * NP + a * I + c], x[c]);
      res2 += cabs2(t);
      nb2 += cabs2(b0[a]);
    }
  }
  norms[2 * g] = res2;
  norms[2 * g + 1] = nb2;
}

template <int I>
__global__ void regularize_kernel(const double2* S, double2* out, int64_t B) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B) return;
  double2 H[I][I];
  double tr = 0.0;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      const double2 x = S[g * NP + a * I + b], y = S[g * NP + b * I + a];
      H[a][b] = cmk(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
    }
#pragma unroll
  for (int a = 0; a < I; ++a) tr += H[a][a].x;
  const double eps = kCovEps * tr / I;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 v = H[a][b];
      if (a == b) v.x += eps;
      out[g * NP + a * I + b] = v;
    }
}

// S_t = herm(S_raw) + eps gram, eps = 1e-9 tr(gram^{-1} herm(S_raw))/I  (fast.py:80-90)
template <int I>
__global__ void reg_transformed_kernel(const double2* S, const double2* gram, double2* out,
                                       int64_t B) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B) return;
  double2 H[I][I], Gm[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      const double2 x = S[g * NP + a * I + b], y = S[g * NP + b * I + a];
      H[a][b] = cmk(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
      Gm[a][b] = gram ? gram[g * NP + a * I + b] : cmk(a == b ? 1.0 : 0.0, 0.0);
    }
  double tr = 0.0;
  if (gram) {
    double2 Gi[I][I];
    double lad;
    lu_inverse<I>(Gm, Gi, &lad);
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int k = 0; k < I; ++k) tr += Gi[a][k].x * H[k][a].x - Gi[a][k].y * H[k][a].y;
  } else {
#pragma unroll
    for (int a = 0; a < I; ++a) tr += H[a][a].x;
  }
  const double eps = kCovEps * tr / I;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) out[g * NP + a * I + b] = cadd(H[a][b], cscale(Gm[a][b], eps));
}

// W = (P^{-1})^H per bin; logdet2 optional
template <int I>
__global__ void inverse_h_kernel(const double2* P, double2* W, double* logdet2, int64_t B,
                                 ffca_status_dev* st, int iter) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B) return;
  double2 A[I][I], Inv[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) A[a][b] = P[g * NP + a * I + b];
  double lad = 0.0;
  const bool ok = lu_inverse<I>(A, Inv, &lad);
  if (!ok && st) report_error(st, iter, FFCA_ERR_SINGULAR_BASIS, (unsigned long long)g);
  if (W) {
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) W[g * NP + a * I + b] = cconj(Inv[b][a]);
  }
  if (logdet2) logdet2[g] = 2.0 * lad;
}

// out(s,n,f,:) = W(f) mu_t(s,n,f,:)
template <int I>
__global__ void apply_w_kernel(const double2* mu_t, const double2* W, double2* out, int64_t Src,
                               int64_t N, int64_t F) {
  constexpr int NP = I * I;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Src * N * F) return;
  const int64_t f = t % F;
  double2 x[I];
#pragma unroll
  for (int a = 0; a < I; ++a) x[a] = mu_t[t * I + a];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    double2 s = cmk(0.0, 0.0);
#pragma unroll
    for (int b = 0; b < I; ++b) s = cmac(s, W[f * NP + a * I + b], x[b]);
    out[t * I + a] = s;
  }
}

// out(s,f) = W(f) S(s,f) W(f)^H
template <int I>
__global__ void conj_w_kernel(const double2* S, const double2* W, double2* out, int64_t Src,
                              int64_t F) {
  constexpr int NP = I * I;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Src * F) return;
  const int64_t f = t % F;
  double2 A[I][I], Wm[I][I], T[I][I], R[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      A[a][b] = S[t * NP + a * I + b];
      Wm[a][b] = W[f * NP + a * I + b];
    }
  matmul_nh<I>(A, Wm, T);
  matmul<I>(Wm, T, R);
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) out[t * NP + a * I + b] = R[a][b];
}

cudaError_t launch_gevd_batch(const double2* Phi, const double2* Psi, double* lam, double2* P,
                              const double2* Pprev, int64_t B, int I, int check,
                              ffca_status_dev* st, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (gevd_batch_kernel<II><<<nblk(B, 64), 64, 0, s>>>(Phi, Psi, lam, P, Pprev,
                                                                        B, check, st, 0)));
  return cudaGetLastError();
}
cudaError_t launch_cholinv(const double2* S, double2* Sinv, int64_t B, int I, ffca_status_dev* st,
                           cudaStream_t s) {
  FFCA_DISPATCH_I(I, (cholinv_kernel<II><<<nblk(B, 64), 64, 0, s>>>(S, Sinv, B, st)));
  return cudaGetLastError();
}
cudaError_t launch_solve(const double2* A, const double2* B, double2* X, double* norms,
                         int64_t batch, int I, int64_t K, ffca_status_dev* st, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (solve_kernel<II><<<nblk(batch, 64), 64, 0, s>>>(A, B, X, norms, batch, K,
                                                                       st)));
  return cudaGetLastError();
}
cudaError_t launch_regularize(const double2* S, double2* out, int64_t B, int I, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (regularize_kernel<II><<<nblk(B, 128), 128, 0, s>>>(S, out, B)));
  return cudaGetLastError();
}
cudaError_t launch_reg_transformed(const double2* S, const double2* gram, double2* out,
                                   int64_t B, int I, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (reg_transformed_kernel<II><<<nblk(B, 64), 64, 0, s>>>(S, gram, out, B)));
  return cudaGetLastError();
}
cudaError_t launch_inverse_h(const double2* P, double2* W, double* logdet2, int64_t B, int I,
                             ffca_status_dev* st, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (inverse_h_kernel<II><<<nblk(B, 64), 64, 0, s>>>(P, W, logdet2, B, st, 0)));
  return cudaGetLastError();
}
cudaError_t launch_apply_w(const double2* mu_t, const double2* W, double2* out, int64_t Src,
                           int64_t N, int64_t F, int I, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (apply_w_kernel<II><<<nblk(Src * N * F, 128), 128, 0, s>>>(mu_t, W, out,
                                                                                Src, N, F)));
  return cudaGetLastError();
}
cudaError_t launch_conj_w(const double2* S, const double2* W, double2* out, int64_t Src,
                          int64_t F, int I, cudaStream_t s) {
  FFCA_DISPATCH_I(I, (conj_w_kernel<II><<<nblk(Src * F, 64), 64, 0, s>>>(S, W, out, Src, F)));
  return cudaGetLastError();
}

}  // namespace ffca
