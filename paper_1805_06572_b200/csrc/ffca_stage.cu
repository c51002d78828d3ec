// Stage-level kernels: the 11-function kernel-module contract of the
// reference backend plugin (_kernels_numpy.py:19-193, _kernels_numba.py:12-391)
// with materialised posterior second moments, for callers that use the
// stage API (reference e_step / m_step / fast_* functions, tests) rather than
// the fused run loop. Single mixture (M = 1), layouts as the reference.
// Reductions are fixed-order (deterministic).
#include "ffca_internal.cuh"

namespace ffca {

namespace {
inline unsigned nb(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

// ---- init_random powers (initializers.py:29-31, modelops.py:12-21) ---------
// One CTA per tile of 32 bins: lane = bin (coalesced rows of y and v), the 32
// warps take interleaved frame slices; per-bin frame sums are combined over
// the warps in a fixed order (deterministic), floor = 1e-10 * mean_n ||y||^2 / I,
// then v = max(||y||^2 / (2I), floor) for both sources.
constexpr int kPowWarps = 32;
template <int I, typename R>
__global__ void __launch_bounds__(kPowWarps * 32)
    init_powers_kernel(const void* y_, void* v_, double* floor, int64_t M, int64_t N, int64_t F) {
  using C = typename CplxOf<R>::type;
  __shared__ double part[kPowWarps][32];
  __shared__ double sfl[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tiles = (F + 31) / 32;
  const int64_t m = blockIdx.x / tiles;
  const int64_t f = (blockIdx.x - m * tiles) * 32 + lane;
  const bool act = f < F;
  const C* y = (const C*)y_ + (m * N * F + (act ? f : 0)) * I;
  R* v = (R*)v_ + m * 2 * N * F + f;
  auto power = [&](int64_t n) {
    double p = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 x = to_c128(y[n * F * I + a]);
      p += x.x * x.x + x.y * x.y;
    }
    return p;
  };
  double s = 0.0;
  if (act)
    for (int64_t n = warp; n < N; n += kPowWarps) s += power(n);
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int w = 0; w < kPowWarps; ++w) t += part[w][lane];
    const double fl = 1e-10 * (t / (double)N) / I;
    sfl[lane] = fl;
    if (act) floor[m * F + f] = fl;
  }
  __syncthreads();
  if (!act) return;
  const double fl = sfl[lane];
  for (int64_t n = warp; n < N; n += kPowWarps) {
    const double q = power(n) / (2.0 * I);
    const double w = q < fl ? fl : q;
    v[n * F] = (R)w;
    v[N * F + n * F] = (R)w;
  }
}

cudaError_t launch_init_powers(const void* y, void* v, double* floor, int64_t M, int64_t N,
                               int64_t F, int I, int dtype, cudaStream_t s) {
  const unsigned grid = (unsigned)(M * ((F + 31) / 32));
#define FFCA_CASE(II)                                                                       \
  case II:                                                                                  \
    if (dtype == FFCA_C64)                                                                  \
      init_powers_kernel<II, float><<<grid, kPowWarps * 32, 0, s>>>(y, v, floor, M, N, F);  \
    else                                                                                    \
      init_powers_kernel<II, double><<<grid, kPowWarps * 32, 0, s>>>(y, v, floor, M, N, F); \
    break;
  switch (I) {
    FFCA_CASE(1)
    FFCA_CASE(2)
    FFCA_CASE(3)
    FFCA_CASE(4)
    FFCA_CASE(5)
    FFCA_CASE(6)
    FFCA_CASE(7)
    FFCA_CASE(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef FFCA_CASE
  return cudaGetLastError();
}

#define FFCA_DISPATCH(I, CALL)      \
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
      return FFCA_ERR_INVALID;      \
  }

// ---- fast_transform (_kernels_numba.py:147-162) ------------------------------
template <int I>
__global__ void transform_kernel(const double2* y, const double2* P, double2* yt, int64_t N,
                                 int64_t F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * F) return;
  const int64_t f = t % F;
  double2 x[I];
#pragma unroll
  for (int a = 0; a < I; ++a) x[a] = y[t * I + a];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    double2 s = cmk(0.0, 0.0);
#pragma unroll
    for (int b = 0; b < I; ++b) s = cadd(s, cconjmul(P[f * I * I + b * I + a], x[b]));
    yt[t * I + a] = s;
  }
}

// ---- fast_e_step (_kernels_numba.py:165-193) ---------------------------------
template <int I>
__global__ void fast_estep_kernel(const double2* yt, const double* v, const double* lam,
                                  double2* mu, double2* Phi, int64_t N, int64_t F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * F) return;
  const int64_t f = t % F;
  const int64_t NF = N * F;
  const double v1 = v[t], v2 = v[NF + t];
  double2 m1[I], m2[I];
  double cd[I];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    const double la = lam[f * I + a];
    const double den = v1 * la + v2;
    const double2 z = yt[t * I + a];
    m1[a] = cscale(z, v1 * la / den);
    m2[a] = cscale(z, v2 / den);
    cd[a] = v1 * v2 * la / den;
    mu[t * I + a] = m1[a];
    mu[(NF + t) * I + a] = m2[a];
  }
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 p1 = cmulc(m1[a], m1[b]), p2 = cmulc(m2[a], m2[b]);
      if (a == b) {
        p1.x += cd[a];
        p2.x += cd[a];
      }
      Phi[(t * I + a) * I + b] = p1;
      Phi[((NF + t) * I + a) * I + b] = p2;
    }
}

// ---- fast_v_update (_kernels_numba.py:196-213) -------------------------------
template <int I>
__global__ void fast_vupd_kernel(const double2* Phi, const double* lam, double* v, int64_t N,
                                 int64_t F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * F) return;
  const int64_t f = t % F;
  const int64_t NF = N * F;
  double a1 = 0.0, a2 = 0.0;
#pragma unroll
  for (int a = 0; a < I; ++a) {
    a1 += Phi[(t * I + a) * I + a].x / lam[f * I + a];
    a2 += Phi[((NF + t) * I + a) * I + a].x;
  }
  v[t] = a1 / I;
  v[NF + t] = a2 / I;
}

// ---- S update (_kernels_numba.py:98-113): one thread per (j, f, a, b) --------
__global__ void s_update_kernel(const double2* Phi, const double* v, double2* S, int64_t N,
                                int64_t F, int I) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t II = (int64_t)I * I;
  if (t >= 2 * F * II) return;
  const int64_t e = t % II;
  const int64_t f = (t / II) % F;
  const int64_t j = t / (II * F);
  double2 s = cmk(0.0, 0.0);
  for (int64_t n = 0; n < N; ++n) {
    const double w = 1.0 / v[(j * N + n) * F + f];
    const double2 ph = Phi[((j * N + n) * F + f) * II + e];
    s.x += w * ph.x;
    s.y += w * ph.y;
  }
  S[t] = cscale(s, 1.0 / (double)N);
}

// ---- likelihoods: one CTA per bin, fixed-order tree -------------------------
template <int I>
__global__ void fast_ll_kernel(const double2* yt, const double* v, const double* lam,
                               const double* logdet2, double* llf, int64_t N, int64_t F) {
  const int64_t f = blockIdx.x;
  __shared__ double sh[128];
  double s = 0.0;
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
    const int64_t t = n * F + f;
    const double v1 = v[t], v2 = v[N * F + t];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double den = v1 * lam[f * I + a] + v2;
      s += log(den) + cabs2(yt[t * I + a]) / den;
    }
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) llf[f] = (double)N * logdet2[f] - sh[0];
}

template <int I>
__global__ void fca_ll_kernel(const double2* y, const double* v, const double2* S, double* llf,
                              int64_t N, int64_t F, ffca_status_dev* st) {
  const int64_t f = blockIdx.x;
  constexpr int NP = I * I;
  __shared__ double sh[128];
  double s = 0.0;
  int64_t bad = -1;
  for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
    const int64_t t = n * F + f;
    const double v1 = v[t], v2 = v[N * F + t];
    double2 R[I][I], L[I][I];
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b)
        R[a][b] = cadd(cscale(S[f * NP + a * I + b], v1), cscale(S[(F + f) * NP + a * I + b], v2));
    if (!cholesky<I>(R, L) && bad < 0) bad = n;
    double2 u[I];
    double prod = 1.0, quad = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      double2 r = y[t * I + a];
#pragma unroll
      for (int b = 0; b < a; ++b) r = csub(r, cmul(L[a][b], u[b]));
      u[a] = cscale(r, 1.0 / L[a][a].x);
      quad += cabs2(u[a]);
      prod *= L[a][a].x;
    }
    s += 2.0 * log(prod) + quad;
  }
  if (bad >= 0 && st) report_error(st, 0, FFCA_ERR_SINGULAR_MIXTURE, (unsigned long long)(bad * F + f));
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) llf[f] = -sh[0];
}

__global__ void sum_ll_kernel(const double* llf, int64_t F, int64_t N, int I, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) s += llf[f];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0] - (double)N * (double)F * (double)I * kLogPi;
}

// ---- conventional e-step with materialised Phi (_kernels_numba.py:12-72) -----
template <int I>
__global__ void fca_estep_kernel(const double2* y, const double* v, const double2* S, double2* mu,
                                 double2* Phi, int64_t N, int64_t F, ffca_status_dev* st) {
  constexpr int NP = I * I;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= N * F) return;
  const int64_t f = t % F;
  const int64_t NF = N * F;
  const double v1 = v[t], v2 = v[NF + t];
  double2 S1[I][I], S2[I][I], R[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      S1[a][b] = S[f * NP + a * I + b];
      S2[a][b] = S[(F + f) * NP + a * I + b];
      R[a][b] = cadd(cscale(S1[a][b], v1), cscale(S2[a][b], v2));
    }
  double2 Ri[I][I];
  double lad;
  if (!lu_inverse<I>(R, Ri, &lad) && st)
    report_error(st, 0, FFCA_ERR_SINGULAR_MIXTURE, (unsigned long long)t);
  double2 A1[I][I], A2[I][I], Cx[I][I];
  matmul<I>(S1, Ri, A1);
  matmul<I>(S2, Ri, A2);
  matmul<I>(A1, S2, Cx);
  double2 m1[I], m2[I];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    double2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
#pragma unroll
    for (int b = 0; b < I; ++b) {
      const double2 yb = y[t * I + b];
      s1 = cadd(s1, cmul(A1[a][b], yb));
      s2 = cadd(s2, cmul(A2[a][b], yb));
    }
    m1[a] = cscale(s1, v1);
    m2[a] = cscale(s2, v2);
    mu[t * I + a] = m1[a];
    mu[(NF + t) * I + a] = m2[a];
  }
  const double vv = v1 * v2;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      const double2 cr = cscale(Cx[a][b], vv);
      Phi[(t * I + a) * I + b] = cadd(cmulc(m1[a], m1[b]), cr);
      Phi[((NF + t) * I + a) * I + b] = cadd(cmulc(m2[a], m2[b]), cr);
    }
}

// ---- conventional v update (_kernels_numba.py:75-95) -------------------------
template <int I>
__global__ void fca_vupd_kernel(const double2* Phi, const double2* Sinv, double* v, int64_t N,
                                int64_t F) {
  constexpr int NP = I * I;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 2 * N * F) return;
  const int64_t f = t % F;
  const int64_t j = t / (N * F);
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) {
      const double2 m = Sinv[(j * F + f) * NP + a * I + b];
      const double2 p = Phi[t * NP + b * I + a];
      acc += m.x * p.x - m.y * p.y;
    }
  v[t] = acc / I;
}

// pack S (2,F,I,I) into the SoA layout of K4 (the pass needs no S^-1: the
// reference's Sinv argument is accepted and validated, not read)
template <int I>
__global__ void pack_fca_kernel(const double2* S, double* Sp, int64_t F) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= F) return;
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const double2* src = S + (w * F + g) * NP;
    double* dst = Sp + (size_t)w * NP * F + g;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      dst[(size_t)a * F] = src[a * I + a].x;
#pragma unroll
      for (int b = a + 1; b < I; ++b) {
        dst[(size_t)Herm<I>::re(a, b) * F] = src[a * I + b].x;
        dst[(size_t)Herm<I>::im(a, b) * F] = src[a * I + b].y;
      }
    }
  }
}

// S_raw (2,F,I,I) = sum_c Spart / N, unpacked
template <int I>
__global__ void finalize_sraw_kernel(const double* Spart, int nchunk, int64_t N, int64_t F,
                                     double2* S_raw) {
  constexpr int NP = I * I;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= F) return;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    double s[NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) s[e] = 0.0;
    // unrolled: the loads of several chunks are in flight together; the adds
    // keep the chunk order (bitwise identical sums)
#pragma unroll 4
    for (int c = 0; c < nchunk; ++c)
#pragma unroll
      for (int e = 0; e < NP; ++e) s[e] += Spart[((size_t)c * 2 * NP + j * NP + e) * F + g];
#pragma unroll
    for (int e = 0; e < NP; ++e) s[e] /= (double)N;
    double2 A[I][I];
    unpack_herm<I>(s, A);
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) S_raw[((size_t)j * F + g) * NP + a * I + b] = A[a][b];
  }
}

}  // namespace ffca

using namespace ffca;

namespace {
inline int cu(cudaError_t e) { return e == cudaSuccess ? FFCA_OK : FFCA_ERR_CUDA; }
bool bad_dims(int64_t N, int64_t F, int I) { return N < 1 || F < 1 || I < 1 || I > kMaxOrder; }
}  // namespace

extern "C" {

int ffca_fast_transform(const double* y, const double* P, double* yt, int64_t N, int64_t F, int I,
                        void* stream) {
  if (!y || !P || !yt || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  FFCA_DISPATCH(I, (transform_kernel<II><<<nb(N * F, 128), 128, 0, s>>>(
                        (const double2*)y, (const double2*)P, (double2*)yt, N, F)));
  return cu(cudaGetLastError());
}

int ffca_fast_e_step(const double* yt, const double* v, const double* lam, double* mu, double* Phi,
                     int64_t N, int64_t F, int I, void* stream) {
  if (!yt || !v || !lam || !mu || !Phi || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  FFCA_DISPATCH(I, (fast_estep_kernel<II><<<nb(N * F, 128), 128, 0, s>>>(
                        (const double2*)yt, v, lam, (double2*)mu, (double2*)Phi, N, F)));
  return cu(cudaGetLastError());
}

int ffca_fast_v_update(const double* Phi, const double* lam, double* v, int64_t N, int64_t F,
                       int I, void* stream) {
  if (!Phi || !lam || !v || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  FFCA_DISPATCH(I, (fast_vupd_kernel<II><<<nb(N * F, 128), 128, 0, s>>>((const double2*)Phi, lam,
                                                                         v, N, F)));
  return cu(cudaGetLastError());
}

int ffca_S_update(const double* Phi, const double* v, double* S, int64_t N, int64_t F, int I,
                  void* stream) {
  if (!Phi || !v || !S || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  s_update_kernel<<<nb(2 * F * I * I, 128), 128, 0, s>>>((const double2*)Phi, v, (double2*)S, N,
                                                         F, I);
  return cu(cudaGetLastError());
}

int ffca_fast_log_likelihood(const double* yt, const double* v, const double* lam,
                             const double* logdet2, double* out, int64_t N, int64_t F, int I,
                             void* stream) {
  if (!yt || !v || !lam || !logdet2 || !out || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  double* llf = nullptr;
  if (cudaMallocAsync((void**)&llf, F * sizeof(double), s) != cudaSuccess) return FFCA_ERR_CUDA;
  int rc = FFCA_OK;
  switch (I) {
#define FFCA_CASE(II)                                                                         \
  case II:                                                                                    \
    fast_ll_kernel<II><<<(unsigned)F, 128, 0, s>>>((const double2*)yt, v, lam, logdet2, llf, \
                                                   N, F);                                     \
    break;
    FFCA_CASE(1)
    FFCA_CASE(2)
    FFCA_CASE(3)
    FFCA_CASE(4)
    FFCA_CASE(5)
    FFCA_CASE(6)
    FFCA_CASE(7)
    FFCA_CASE(8)
#undef FFCA_CASE
  }
  sum_ll_kernel<<<1, 256, 0, s>>>(llf, F, N, I, out);
  rc = cu(cudaGetLastError());
  cudaFreeAsync(llf, s);
  return rc;
}

int ffca_fca_log_likelihood(const double* y, const double* v, const double* S, double* out,
                            int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream) {
  if (!y || !v || !S || !out || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  double* llf = nullptr;
  if (cudaMallocAsync((void**)&llf, F * sizeof(double), s) != cudaSuccess) return FFCA_ERR_CUDA;
  switch (I) {
#define FFCA_CASE(II)                                                                        \
  case II:                                                                                   \
    fca_ll_kernel<II><<<(unsigned)F, 128, 0, s>>>((const double2*)y, v, (const double2*)S,  \
                                                  llf, N, F, st);                            \
    break;
    FFCA_CASE(1)
    FFCA_CASE(2)
    FFCA_CASE(3)
    FFCA_CASE(4)
    FFCA_CASE(5)
    FFCA_CASE(6)
    FFCA_CASE(7)
    FFCA_CASE(8)
#undef FFCA_CASE
  }
  sum_ll_kernel<<<1, 256, 0, s>>>(llf, F, N, I, out);
  const int rc = cu(cudaGetLastError());
  cudaFreeAsync(llf, s);
  return rc;
}

int ffca_fca_e_step(const double* y, const double* v, const double* S, double* mu, double* Phi,
                    int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream) {
  if (!y || !v || !S || !mu || !Phi || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  FFCA_DISPATCH(I, (fca_estep_kernel<II><<<nb(N * F, 64), 64, 0, s>>>(
                        (const double2*)y, v, (const double2*)S, (double2*)mu, (double2*)Phi, N,
                        F, st)));
  return cu(cudaGetLastError());
}

int ffca_fca_v_update(const double* Phi, const double* S_prev, double* v, int64_t N, int64_t F,
                      int I, ffca_status_dev* st, void* stream) {
  if (!Phi || !S_prev || !v || bad_dims(N, F, I)) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  double2* Sinv = nullptr;
  if (cudaMallocAsync((void**)&Sinv, 2 * F * I * I * sizeof(double2), s) != cudaSuccess)
    return FFCA_ERR_CUDA;
  int rc = ffca_cholesky_inverse(S_prev, (double*)Sinv, 2 * F, I, st, stream);
  if (rc == FFCA_OK) {
    switch (I) {
#define FFCA_CASE(II)                                                                         \
  case II:                                                                                    \
    fca_vupd_kernel<II><<<nb(2 * N * F, 128), 128, 0, s>>>((const double2*)Phi, Sinv, v, N,  \
                                                           F);                                \
    break;
      FFCA_CASE(1)
      FFCA_CASE(2)
      FFCA_CASE(3)
      FFCA_CASE(4)
      FFCA_CASE(5)
      FFCA_CASE(6)
      FFCA_CASE(7)
      FFCA_CASE(8)
#undef FFCA_CASE
    }
    rc = cu(cudaGetLastError());
  }
  cudaFreeAsync(Sinv, s);
  return rc;
}

int ffca_fast_iteration(const double* y, const double* P, const double* v, const double* lam,
                        const double* v_floor, double* mu, double* v_new, double* S_raw,
                        int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream) {
  if (!y || !P || !v || !lam || !v_floor || !v_new || !S_raw || bad_dims(N, F, I))
    return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(v_new, v, 2 * N * F * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return FFCA_ERR_CUDA;
  FastIterParams p{};
  plan_fast_chunks(F, N, I, FFCA_C128, &p.chunk_frames, &p.nchunk);
  double* Spart = nullptr;
  if (cudaMallocAsync((void**)&Spart, (size_t)p.nchunk * 2 * I * I * F * sizeof(double), s) !=
      cudaSuccess)
    return FFCA_ERR_CUDA;
  p.y = y;
  p.v = v_new;
  p.P = (const double2*)P;
  p.W = nullptr;
  p.lam = lam;
  p.floor = v_floor;
  p.Spart = Spart;
  p.llbin = nullptr;
  p.mu_out = mu;
  p.mu_back = 0;
  p.update = 1;
  p.M = 1;
  p.N = N;
  p.F = F;
  p.G = F;
  p.st = st;
  p.iter = 0;
  int rc = cu(launch_fast_em(p, I, FFCA_C128, s));
  if (rc == FFCA_OK) {
    switch (I) {
#define FFCA_CASE(II)                                                                          \
  case II:                                                                                     \
    finalize_sraw_kernel<II><<<nb(F, 64), 64, 0, s>>>(Spart, p.nchunk, N, F, (double2*)S_raw); \
    break;
      FFCA_CASE(1)
      FFCA_CASE(2)
      FFCA_CASE(3)
      FFCA_CASE(4)
      FFCA_CASE(5)
      FFCA_CASE(6)
      FFCA_CASE(7)
      FFCA_CASE(8)
#undef FFCA_CASE
    }
    rc = cu(cudaGetLastError());
  }
  cudaFreeAsync(Spart, s);
  return rc;
}

int ffca_fca_iteration(const double* y, const double* v, const double* S, const double* Sinv,
                       const double* v_floor, double* mu, double* v_new, double* S_raw,
                       int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream) {
  if (!y || !v || !S || !Sinv || !v_floor || !v_new || !S_raw || bad_dims(N, F, I))
    return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(v_new, v, 2 * N * F * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return FFCA_ERR_CUDA;
  FcaIterParams p{};
  plan_fca_chunks(F, N, I, FFCA_C128, &p.chunk_frames, &p.nchunk);
  double *Spart = nullptr, *Sp = nullptr;
  if (cudaMallocAsync((void**)&Spart, (size_t)p.nchunk * kFcaParts * I * I * F * sizeof(double), s) !=
          cudaSuccess ||
      cudaMallocAsync((void**)&Sp, (size_t)2 * I * I * F * sizeof(double), s) != cudaSuccess)
    return FFCA_ERR_CUDA;
  int rc = FFCA_OK;
  switch (I) {
#define FFCA_CASE(II)                                                                      \
  case II:                                                                                 \
    pack_fca_kernel<II><<<nb(F, 64), 64, 0, s>>>((const double2*)S, Sp, F);                \
    break;
    FFCA_CASE(1)
    FFCA_CASE(2)
    FFCA_CASE(3)
    FFCA_CASE(4)
    FFCA_CASE(5)
    FFCA_CASE(6)
    FFCA_CASE(7)
    FFCA_CASE(8)
#undef FFCA_CASE
  }
  p.y = y;
  p.v = v_new;
  p.Sp = Sp;
  p.floor = v_floor;
  p.Spart = Spart;
  p.llbin = nullptr;
  p.mu_out = mu;
  p.update = 1;
  p.M = 1;
  p.N = N;
  p.F = F;
  p.G = F;
  p.st = st;
  p.iter = 0;
  rc = cu(launch_fca_em(p, I, FFCA_C128, s));
  if (rc == FFCA_OK) rc = cu(launch_fca_sraw(Spart, p.nchunk, N, F, Sp, (double2*)S_raw, I, s));
  cudaFreeAsync(Spart, s);
  cudaFreeAsync(Sp, s);
  return rc;
}

}  // extern "C"
