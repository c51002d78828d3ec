// K4 — fused conventional FCA iteration (the frame-wise baseline the paper
// accelerates): per (n, f) the mixture covariance R = v1 S1 + v2 S2 is
// inverted (Cholesky; R is Hermitian positive definite), posterior means
// mu_j = v_j S_j R^{-1} y and the shared cross term v1 v2 S1 R^{-1} S2 are
// formed with I x I complex products, the powers are updated from
// tr(S_j^{-1} Phi_j)/I and the covariance sums accumulated.
// Reference: _kernels_numba.py:246-325 (_fca_iteration) fused with
// _kernels_numba.py:116-144 (_fca_log_likelihood); per-bin steps
// conventional.py:98-101 (_cholesky_inverse) and modelops.py:29-39
// (regularize_covariances).
//
// Mapping as K3: lane <-> bin, warps <-> frame slices. The CTA's 32 bins keep
// S1, S2 (packed Hermitian) in shared memory, bin-minor so each lane's reads
// are bank-conflict free. The power-update traces tr(S_j^-1 Phi_j) are taken
// through identities that need no S_j^-1 (see the trace block).
#include "ffca_internal.cuh"

namespace ffca {

template <int I, typename R, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) fca_em_kernel(const FcaIterParams p) {
  using C = typename CplxOf<R>::type;
  constexpr int NP = I * I;
  constexpr int NE = 2 * NP + 1;
  extern __shared__ double smem[];
  double* sS = smem;                    // [2][NP][32]: S1, S2 (the traces need no S^-1)
  double* red = smem + 2 * NP * 32;     // [(WARPS-1)][NE][32]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t G = p.G;
  int64_t g = (int64_t)blockIdx.x * 32 + lane;
  const bool active = g < G;
  if (!active) g = G - 1;
  const int64_t m = g / p.F;
  const int64_t f = g - m * p.F;
  for (int e = warp; e < 2 * NP; e += WARPS) sS[e * 32 + lane] = p.Sp[(size_t)e * G + g];
  __syncthreads();
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  const C* __restrict__ yb = (const C*)p.y + (m * p.N * p.F + f) * I;
  R* __restrict__ vb = (R*)p.v + m * 2 * NF + f;
  const double fl = p.floor[g];
  const double invI = 1.0 / I;

  auto Sget = [&](int which, int a, int b) -> double2 {
    // full entry (a, b) of packed Hermitian matrix `which`
    const double* base = sS + which * NP * 32 + lane;
    if (a == b) return cmk(base[a * 32], 0.0);
    if (a < b) return cmk(base[Herm<I>::re(a, b) * 32], base[Herm<I>::im(a, b) * 32]);
    return cmk(base[Herm<I>::re(b, a) * 32], -base[Herm<I>::im(b, a) * 32]);
  };

  double acc[2][NP];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[j][e] = 0.0;
  double llacc = 0.0;
  const bool do_ll = p.llbin != nullptr;
  int64_t bad_n = 0;

  for (int64_t n = n0 + warp; n < n1; n += WARPS) {
    const C* yp = yb + n * p.F * I;
    double2 yv[I];
#pragma unroll
    for (int a = 0; a < I; ++a) yv[a] = to_c128(yp[a]);
    const double v1 = (double)vb[n * p.F];
    const double v2 = (double)vb[NF + n * p.F];
    // R = v1 S1 + v2 S2 and its Cholesky factor
    double2 Lm[I][I];
    {
      double2 Rm[I][I];
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          const double2 s1 = Sget(0, a, b), s2 = Sget(1, a, b);
          Rm[a][b] = cmk(v1 * s1.x + v2 * s2.x, v1 * s1.y + v2 * s2.y);
        }
      if (!cholesky<I>(Rm, Lm) && bad_n == 0) bad_n = n + 1;
    }
    double2 Li[I][I];
    tril_inverse<I>(Lm, Li);
    if (do_ll) {
      // log det R + y^H R^{-1} y = 2 sum log L_ii + |L^{-1} y|^2
      double prod = 1.0, quad = 0.0;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        prod *= Lm[a][a].x;
        double2 u = cmk(0.0, 0.0);
#pragma unroll
        for (int b = 0; b <= a; ++b) u = cadd(u, cmul(Li[a][b], yv[b]));
        quad += cabs2(u);
      }
      llacc += 2.0 * log(prod) + quad;
    }
    // Rinv = Li^H Li (frame-wise inverse; Hermitian: upper triangle computed,
    // lower mirrored), x = Rinv y
    double2 Ri[I][I];
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = a; b < I; ++b) {
        double2 s = cmk(0.0, 0.0);
#pragma unroll
        for (int k = b; k < I; ++k) s = cadd(s, cconjmul(Li[k][a], Li[k][b]));
        if (a == b) s.y = 0.0;
        Ri[a][b] = s;
        Ri[b][a] = cconj(s);
      }
    double2 x[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      double2 s = cmk(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < I; ++b) s = cadd(s, cmul(Ri[a][b], yv[b]));
      x[a] = s;
    }
    // mu_j = v_j S_j x
    double2 mu1[I], mu2[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      double2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < I; ++b) {
        s1 = cadd(s1, cmul(Sget(0, a, b), x[b]));
        s2 = cadd(s2, cmul(Sget(1, a, b), x[b]));
      }
      mu1[a] = cscale(s1, v1);
      mu2[a] = cscale(s2, v2);
    }
    if (p.mu_out != nullptr && active) {
      C* mo = (C*)p.mu_out;
      C* d1 = mo + (((m * 2 + 0) * p.N + n) * p.F + f) * I;
      C* d2 = mo + (((m * 2 + 1) * p.N + n) * p.F + f) * I;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        d1[a] = from_c128<R>(mu1[a]);
        d2[a] = from_c128<R>(mu2[a]);
      }
    }
    if (!p.update) continue;
    // cross term Cm = v1 v2 S1 (Rinv S2)  (Hermitian; upper triangle)
    double2 Cm[I][I];
    double Tdiag[I];  // Re diag(Rinv S2), for the source-1 trace
    {
      double2 T[I][I];
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = 0; b < I; ++b) {
          double2 s = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) s = cadd(s, cmul(Ri[a][k], Sget(1, k, b)));
          T[a][b] = s;
        }
#pragma unroll
      for (int a = 0; a < I; ++a) Tdiag[a] = T[a][a].x;
      const double vv = v1 * v2;
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = a; b < I; ++b) {
          double2 s = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) s = cadd(s, cmul(Sget(0, a, k), T[k][b]));
          Cm[a][b] = cscale(s, vv);
          if (a == b) Cm[a][b].y = 0.0;
        }
    }
    // tr_j = Re tr(S_j^-1 Phi_j), Phi_j = mu_j mu_j^H + Cm, without S_j^-1:
    //   mu_j^H S_j^-1 mu_j = v_j Re(x^H mu_j)          (mu_j = v_j S_j x)
    //   tr(S_1^-1 Cm) = v1 v2 Re tr(Rinv S2) = v1 v2 Re tr(T)
    //   tr(S_2^-1 Cm) = v1 v2 Re tr(S1 Rinv)             (cyclic trace)
    // every term is non-negative (no cancellation)
    double tr[2];
    {
      double q1 = 0.0, q2 = 0.0, tT = 0.0, tSR = 0.0;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        q1 += x[a].x * mu1[a].x + x[a].y * mu1[a].y;
        q2 += x[a].x * mu2[a].x + x[a].y * mu2[a].y;
        tT += Tdiag[a];
#pragma unroll
        for (int b = 0; b < I; ++b) {  // Re(S1[a][b] Ri[b][a])
          const double2 s1 = Sget(0, a, b);
          tSR += s1.x * Ri[b][a].x - s1.y * Ri[b][a].y;
        }
      }
      const double vv = v1 * v2;
      tr[0] = v1 * q1 + vv * tT;
      tr[1] = v2 * q2 + vv * tSR;
    }
    const double q1 = tr[0] * invI, q2 = tr[1] * invI;
    const double w1 = (q1 < fl) ? fl : q1;
    const double w2 = (q2 < fl) ? fl : q2;
    if (active) {
      vb[n * p.F] = (R)w1;
      vb[NF + n * p.F] = (R)w2;
    }
    const double iw1 = 1.0 / w1, iw2 = 1.0 / w2;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      acc[0][a] += (cabs2(mu1[a]) + Cm[a][a].x) * iw1;
      acc[1][a] += (cabs2(mu2[a]) + Cm[a][a].x) * iw2;
#pragma unroll
      for (int b = a + 1; b < I; ++b) {
        const double2 p1 = cadd(cmulc(mu1[a], mu1[b]), Cm[a][b]);
        const double2 p2 = cadd(cmulc(mu2[a], mu2[b]), Cm[a][b]);
        acc[0][Herm<I>::re(a, b)] += p1.x * iw1;
        acc[0][Herm<I>::im(a, b)] += p1.y * iw1;
        acc[1][Herm<I>::re(a, b)] += p2.x * iw2;
        acc[1][Herm<I>::im(a, b)] += p2.y * iw2;
      }
    }
  }
  if (bad_n && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MIXTURE,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));

  if (!p.update && !do_ll) return;
  if (WARPS > 1) {
    if (warp > 0) {
      double* r = red + (size_t)(warp - 1) * NE * 32;
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        r[e * 32 + lane] = acc[0][e];
        r[(NP + e) * 32 + lane] = acc[1][e];
      }
      r[2 * NP * 32 + lane] = llacc;
    }
    __syncthreads();
    if (warp != 0) return;
#pragma unroll 1
    for (int w = 1; w < WARPS; ++w) {
      const double* r = red + (size_t)(w - 1) * NE * 32;
#pragma unroll
      for (int e = 0; e < NP; ++e) {
        acc[0][e] += r[e * 32 + lane];
        acc[1][e] += r[(NP + e) * 32 + lane];
      }
      llacc += r[2 * NP * 32 + lane];
    }
  }
  if (!active) return;
  const int64_t c = blockIdx.y;
  if (p.update) {
    double* sp = p.Spart + (size_t)c * 2 * NP * G + g;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      sp[(size_t)e * G] = acc[0][e];
      sp[(size_t)(NP + e) * G] = acc[1][e];
    }
  }
  if (do_ll) p.llbin[(size_t)c * G + g] = llacc;
}

template <int I, typename R>
static cudaError_t launch_fca_em_t(const FcaIterParams& p, cudaStream_t s) {
  constexpr int NP = I * I;
  constexpr int NE = 2 * NP + 1;
  const size_t smem = ((size_t)2 * NP * 32 + (size_t)(kWarps - 1) * NE * 32) * sizeof(double);
  auto kern = fca_em_kernel<I, R, kWarps>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((unsigned)((p.G + 31) / 32), (unsigned)p.nchunk);
  kern<<<grid, kWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

template <int I, typename R>
static int fca_bpsm_t() {
  constexpr int NP = I * I;
  constexpr int NE = 2 * NP + 1;
  const size_t smem = ((size_t)2 * NP * 32 + (size_t)(kWarps - 1) * NE * 32) * sizeof(double);
  auto kern = fca_em_kernel<I, R, kWarps>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, smem);
  return n > 0 ? n : 1;
}

cudaError_t launch_fca_par(const FcaIterParams& p, int I, int dtype, cudaStream_t s);
int fca_par_blocks_per_sm(int I, int dtype);
int fca_par_bins_per_cta(int I);

void plan_fca_chunks(int64_t G, int64_t N, int I, int dtype, int64_t* chunk_frames, int* nchunk) {
  if (I >= 5)
    plan_chunks(G, N, fca_par_blocks_per_sm(I, dtype), chunk_frames, nchunk,
                fca_par_bins_per_cta(I), 16);
  else
    plan_chunks(G, N, fca_blocks_per_sm(I, dtype), chunk_frames, nchunk);
}

int fca_blocks_per_sm(int I, int dtype) {
  static int cache[2][9] = {};
  const int d = dtype == FFCA_C64 ? 1 : 0;
  if (I < 1 || I > 8) return 1;
  if (cache[d][I]) return cache[d][I];
  int n = 1;
  switch (I) {
#define FFCA_OCC(II) \
  case II:           \
    n = d ? fca_bpsm_t<II, float>() : fca_bpsm_t<II, double>(); \
    break;
    FFCA_OCC(1)
    FFCA_OCC(2)
    FFCA_OCC(3)
    FFCA_OCC(4)
    FFCA_OCC(5)
    FFCA_OCC(6)
    FFCA_OCC(7)
    FFCA_OCC(8)
#undef FFCA_OCC
  }
  cache[d][I] = n;
  return n;
}

cudaError_t launch_fca_em(const FcaIterParams& p, int I, int dtype, cudaStream_t s) {
  if (I >= 5) return launch_fca_par(p, I, dtype, s);  // lane-parallel (ffca_fca_par.cu)
#define FFCA_CASE(II)                                                    \
  case II:                                                               \
    return dtype == FFCA_C64 ? launch_fca_em_t<II, float>(p, s)          \
                             : launch_fca_em_t<II, double>(p, s);
  switch (I) {
    FFCA_CASE(1)
    FFCA_CASE(2)
    FFCA_CASE(3)
    FFCA_CASE(4)
    default:
      return cudaErrorInvalidValue;
  }
#undef FFCA_CASE
}

// ---- per-bin prepare / finish -----------------------------------------------
template <int I>
FFCA_DEV void pack_and_invert(const double2 (&S1)[I][I], const double2 (&S2)[I][I], double* Sp,
                              int64_t g, int64_t G, ffca_status_dev* st, int iter) {
  constexpr int NP = I * I;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double2(&A)[I][I] = j == 0 ? S1 : S2;
    double* dst = Sp + (size_t)j * NP * G + g;
    double* dsti = Sp + (size_t)(2 + j) * NP * G + g;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      dst[(size_t)a * G] = A[a][a].x;
#pragma unroll
      for (int b = a + 1; b < I; ++b) {
        dst[(size_t)Herm<I>::re(a, b) * G] = A[a][b].x;
        dst[(size_t)Herm<I>::im(a, b) * G] = A[a][b].y;
      }
    }
    double2 L[I][I], Li[I][I];
    if (!cholesky<I>(A, L) && st) report_error(st, iter, FFCA_ERR_NOT_PD, (unsigned long long)g);
    tril_inverse<I>(L, Li);
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = a; b < I; ++b) {
        double2 s = cmk(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < I; ++k) {
          if (k < a || k < b) continue;
          s = cadd(s, cconjmul(Li[k][a], Li[k][b]));
        }
        if (a == b)
          dsti[(size_t)a * G] = s.x;
        else {
          dsti[(size_t)Herm<I>::re(a, b) * G] = s.x;
          dsti[(size_t)Herm<I>::im(a, b) * G] = s.y;
        }
      }
  }
}

template <int I>
__global__ void __launch_bounds__(64)
    fca_prepare_kernel(const double2* __restrict__ S, double* Sp, int64_t G, int64_t F,
                       ffca_status_dev* st, int iter) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int64_t m = g / F, f = g - m * F;
  double2 S1[I][I], S2[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      S1[a][b] = S[((m * 2 + 0) * F + f) * NP + a * I + b];
      S2[a][b] = S[((m * 2 + 1) * F + f) * NP + a * I + b];
    }
  pack_and_invert<I>(S1, S2, Sp, g, G, st, iter);
}

template <int I>
__global__ void __launch_bounds__(64)
    fca_finish_kernel(const double* __restrict__ Spart, int nchunk, int64_t N, int64_t G,
                      int64_t F, double* Sp, double2* S_model, double2* S_hist,
                      const double* llbin, double* llg, ffca_status_dev* st, int iter) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const int64_t m = g / F, f = g - m * F;
  if (llg) {
    llg[g] = -ordered_sum(llbin + g, nchunk, (size_t)G);
  }
  double2 S[2][I][I];
  const double invN = 1.0 / (double)N;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    double s[NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) s[e] = 0.0;
    // unrolled: the loads of several chunks are in flight together; the adds
    // keep the chunk order (bitwise identical sums)
#pragma unroll 4
    for (int c = 0; c < nchunk; ++c) {
      const double* sp = Spart + (size_t)c * 2 * NP * G + (size_t)j * NP * G + g;
#pragma unroll
      for (int e = 0; e < NP; ++e) s[e] += sp[(size_t)e * G];
    }
    double tr = 0.0;
#pragma unroll
    for (int e = 0; e < NP; ++e) s[e] *= invN;
#pragma unroll
    for (int a = 0; a < I; ++a) tr += s[a];
    // regularize_covariances: hermitize (exact for packed) + 1e-9 tr/I ridge
    const double eps = kCovEps * tr / I;
#pragma unroll
    for (int a = 0; a < I; ++a) s[a] += eps;
    unpack_herm<I>(s, S[j]);
    double2* dst = S_model + ((m * 2 + j) * F + f) * NP;
    double2* hst = S_hist ? S_hist + ((m * 2 + j) * F + f) * NP : nullptr;
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        dst[a * I + b] = S[j][a][b];
        if (hst) hst[a * I + b] = S[j][a][b];
      }
  }
  pack_and_invert<I>(S[0], S[1], Sp, g, G, st, iter + 1);
}

#define FFCA_DISPATCH_I2(I, CALL)   \
  switch (I) {                      \
    case 1: {                       \
      constexpr int II = 1;         \
      CALL;                         \
    } break;                        \
    case 2: {                       \
      constexpr int II = 2;         \
      CALL;                         \
    } break;                        \
    case 3: {                       \
      constexpr int II = 3;         \
      CALL;                         \
    } break;                        \
    case 4: {                       \
      constexpr int II = 4;         \
      CALL;                         \
    } break;                        \
    case 5: {                       \
      constexpr int II = 5;         \
      CALL;                         \
    } break;                        \
    case 6: {                       \
      constexpr int II = 6;         \
      CALL;                         \
    } break;                        \
    case 7: {                       \
      constexpr int II = 7;         \
      CALL;                         \
    } break;                        \
    case 8: {                       \
      constexpr int II = 8;         \
      CALL;                         \
    } break;                        \
    default:                        \
      return cudaErrorInvalidValue; \
  }

cudaError_t launch_fca_prepare(const double2* S, double* Sp, int64_t G, int64_t F, int I,
                               ffca_status_dev* st, int iter, cudaStream_t s) {
  const unsigned nb = (unsigned)((G + 63) / 64);
  FFCA_DISPATCH_I2(I, (fca_prepare_kernel<II><<<nb, 64, 0, s>>>(S, Sp, G, F, st, iter)));
  return cudaGetLastError();
}

cudaError_t launch_fca_finish(const double* Spart, int nchunk, int64_t N, int64_t G, int64_t F,
                              double* Sp, double2* S_model, double2* S_hist,
                              const double* llbin, double* llg, int I, ffca_status_dev* st,
                              int iter, cudaStream_t s) {
  const unsigned nb = (unsigned)((G + 63) / 64);
  FFCA_DISPATCH_I2(I, (fca_finish_kernel<II><<<nb, 64, 0, s>>>(Spart, nchunk, N, G, F, Sp,
                                                                S_model, S_hist, llbin, llg,
                                                                st, iter)));
  return cudaGetLastError();
}

}  // namespace ffca
