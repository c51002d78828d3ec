// K3 — fused FastFCA iteration: z = P^H y, diagonal posterior, v update,
// per-bin transformed covariance accumulation, optional log-likelihood and
// optional posterior-mean / separated-image write, in ONE streaming pass.
//
// Reference: _kernels_numba.py:328-391 (_fast_iteration) fused with
// _kernels_numba.py:220-243 (_fast_log_likelihood) and fast.py:133-141
// (back_transform_images, via W = P^{-H}).
//
// Thread mapping: lane <-> global bin g = m*F + f (32 consecutive bins per
// warp, so every frame row of y and v is a coalesced load), warps <-> frame
// slices. Each thread keeps its bin's P, lambda and the packed Hermitian
// accumulators of both sources in registers and streams its frames; the
// per-bin sums are reduced across the CTA's warps in shared memory and
// written as one partial per (frame chunk, bin). Reduction order is fixed, so
// results are deterministic and independent of how bins are sharded.
#include "ffca_internal.cuh"

namespace ffca {

template <int I, typename R, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    fast_em_kernel(const FastIterParams p) {
  using C = typename CplxOf<R>::type;
  constexpr int NP = I * I;
  constexpr int NE = 2 * NP + 1;
  extern __shared__ double red[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t G = p.G;
  int64_t g = (int64_t)blockIdx.x * 32 + lane;
  const bool active = g < G;
  if (!active) g = G - 1;
  const int64_t m = g / p.F;
  const int64_t f = g - m * p.F;
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  const C* __restrict__ yb = (const C*)p.y + (m * p.N * p.F + f) * I;
  R* __restrict__ vb = (R*)p.v + m * 2 * NF + f;

  double2 Pm[I][I];
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) Pm[a][b] = p.P[g * NP + a * I + b];
  double lam[I], il[I];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    lam[a] = p.lam[g * I + a];
    il[a] = 1.0 / lam[a];
  }
  const double fl = p.floor[g];
  const double invI = 1.0 / I;

  double acc[2][NP];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[j][e] = 0.0;
  double llacc = 0.0;
  const bool do_ll = p.llbin != nullptr;
  bool bad = false;
  int64_t bad_n = 0;

  for (int64_t n = n0 + warp; n < n1; n += WARPS) {
    const C* yp = yb + n * p.F * I;
    double2 yv[I];
#pragma unroll
    for (int a = 0; a < I; ++a) yv[a] = to_c128(yp[a]);
    const double v1 = (double)vb[n * p.F];
    const double v2 = (double)vb[NF + n * p.F];
    // z = P^H y
    double2 z[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      double zr = 0.0, zi = 0.0;
#pragma unroll
      for (int b = 0; b < I; ++b) {
        zr += Pm[b][a].x * yv[b].x + Pm[b][a].y * yv[b].y;
        zi += Pm[b][a].x * yv[b].y - Pm[b][a].y * yv[b].x;
      }
      z[a] = cmk(zr, zi);
    }
    double g1[I], g2[I], t1[I], t2[I];
    double tr1 = 0.0, tr2 = 0.0, lprod = 1.0, quad = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double v1l = v1 * lam[a];
      const double den = v1l + v2;
      const double rden = 1.0 / den;
      g1[a] = v1l * rden;
      g2[a] = v2 * rden;
      const double c = v2 * g1[a];
      const double pz = z[a].x * z[a].x + z[a].y * z[a].y;
      t1[a] = g1[a] * g1[a] * pz + c;
      t2[a] = g2[a] * g2[a] * pz + c;
      tr1 += t1[a] * il[a];
      tr2 += t2[a];
      if (do_ll) {
        lprod *= den;
        quad += pz * rden;
      }
      if (den == 0.0) bad = true;
    }
    if (do_ll) llacc += log(lprod) + quad;
    if (p.update) {
      const double q1 = tr1 * invI, q2 = tr2 * invI;
      const double w1 = (q1 < fl) ? fl : q1;  // NaN propagates like np.maximum
      const double w2 = (q2 < fl) ? fl : q2;
      if (active) {
        vb[n * p.F] = (R)w1;
        vb[NF + n * p.F] = (R)w2;
      }
      if (!(isfinite(w1) && isfinite(w2) && w1 > 0.0 && w2 > 0.0)) bad = true;
      const double iw1 = 1.0 / w1, iw2 = 1.0 / w2;
      double2 m1[I], m2[I];
#pragma unroll
      for (int a = 0; a < I; ++a) {
        m1[a] = cscale(z[a], g1[a]);
        m2[a] = cscale(z[a], g2[a]);
        acc[0][a] += t1[a] * iw1;
        acc[1][a] += t2[a] * iw2;
      }
#pragma unroll
      for (int a = 0; a < I; ++a) {
        const double2 s1 = cscale(m1[a], iw1);
        const double2 s2 = cscale(m2[a], iw2);
#pragma unroll
        for (int b = a + 1; b < I; ++b) {
          acc[0][Herm<I>::re(a, b)] += s1.x * m1[b].x + s1.y * m1[b].y;
          acc[0][Herm<I>::im(a, b)] += s1.y * m1[b].x - s1.x * m1[b].y;
          acc[1][Herm<I>::re(a, b)] += s2.x * m2[b].x + s2.y * m2[b].y;
          acc[1][Herm<I>::im(a, b)] += s2.y * m2[b].x - s2.x * m2[b].y;
        }
      }
    }
    if (p.mu_out != nullptr && active) {
      C* mo = (C*)p.mu_out;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        double2 mm[I];
#pragma unroll
        for (int a = 0; a < I; ++a) mm[a] = cscale(z[a], j == 0 ? g1[a] : g2[a]);
        C* dst = mo + (((m * 2 + j) * p.N + n) * p.F + f) * I;
        if (p.mu_back) {
          const double2* Wg = p.W + g * NP;
#pragma unroll
          for (int a = 0; a < I; ++a) {
            double2 s = cmk(0.0, 0.0);
#pragma unroll
            for (int b = 0; b < I; ++b) {
              const double2 w = Wg[a * I + b];
              s.x += w.x * mm[b].x - w.y * mm[b].y;
              s.y += w.x * mm[b].y + w.y * mm[b].x;
            }
            dst[a] = from_c128<R>(s);
          }
        } else {
#pragma unroll
          for (int a = 0; a < I; ++a) dst[a] = from_c128<R>(mm[a]);
        }
      }
    }
    if (bad && bad_n == 0) bad_n = n + 1;
  }
  if (bad_n && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));

  if (!p.update && !do_ll) return;
  // --- cross-warp reduction (fixed order) ---
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
static cudaError_t launch_fast_em_t(const FastIterParams& p, cudaStream_t s) {
  constexpr int NE = 2 * I * I + 1;
  const size_t smem = (size_t)(kWarps - 1) * NE * 32 * sizeof(double);
  auto kern = fast_em_kernel<I, R, kWarps>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((unsigned)((p.G + 31) / 32), (unsigned)p.nchunk);
  kern<<<grid, kWarps * 32, smem, s>>>(p);
  return cudaGetLastError();
}

// v2 kernels for I <= 4 (ffca_fast2.cuh, instantiated in ffca_fast_i<I>.cu)
template <int I, typename R>
cudaError_t launch_fast2(const FastIterParams& p, cudaStream_t s);
template <int I, typename R>
int fast2_blocks_per_sm();

template <int I, typename R>
static int fast_v1_blocks_per_sm() {
  constexpr int NE = 2 * I * I + 1;
  const size_t smem = (size_t)(kWarps - 1) * NE * 32 * sizeof(double);
  auto kern = fast_em_kernel<I, R, kWarps>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, smem);
  return n > 0 ? n : 1;
}

int fast_blocks_per_sm(int I, int dtype) {
  static int cache[2][9] = {};
  const int d = dtype == FFCA_C64 ? 1 : 0;
  if (I < 1 || I > 8) return 1;
  if (cache[d][I]) return cache[d][I];
  int n = 1;
#define FFCA_OCC(II)                                                               \
  case II:                                                                         \
    if (II <= 4)                                                                   \
      n = d ? fast2_blocks_per_sm<(II <= 4 ? II : 4), float>()                     \
            : fast2_blocks_per_sm<(II <= 4 ? II : 4), double>();                   \
    else                                                                           \
      n = d ? fast_v1_blocks_per_sm<II, float>() : fast_v1_blocks_per_sm<II, double>(); \
    break;
  switch (I) {
    FFCA_OCC(1)
    FFCA_OCC(2)
    FFCA_OCC(3)
    FFCA_OCC(4)
    FFCA_OCC(5)
    FFCA_OCC(6)
    FFCA_OCC(7)
    FFCA_OCC(8)
  }
#undef FFCA_OCC
  cache[d][I] = n;
  return n;
}

cudaError_t launch_fast_em(const FastIterParams& p, int I, int dtype, cudaStream_t s) {
#define FFCA_CASE2(II)                                                      \
  case II:                                                                  \
    return dtype == FFCA_C64 ? launch_fast2<II, float>(p, s)                \
                             : launch_fast2<II, double>(p, s);
#define FFCA_CASE(II)                                                       \
  case II:                                                                  \
    return dtype == FFCA_C64 ? launch_fast_em_t<II, float>(p, s)            \
                             : launch_fast_em_t<II, double>(p, s);
  switch (I) {
    FFCA_CASE2(1)
    FFCA_CASE2(2)
    FFCA_CASE2(3)
    FFCA_CASE2(4)
    FFCA_CASE(5)
    FFCA_CASE(6)
    FFCA_CASE(7)
    FFCA_CASE(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef FFCA_CASE
#undef FFCA_CASE2
}

// ---- likelihood bookkeeping ------------------------------------------------
__global__ void ll_collect_kernel(const double* __restrict__ llbin, int nchunk,
                                  const double* __restrict__ logdet2, int64_t N, int64_t G,
                                  double* __restrict__ llg) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += llbin[(size_t)c * G + g];
  const double ld = logdet2 ? (double)N * logdet2[g] : 0.0;
  llg[g] = ld - s;
}

cudaError_t launch_ll_collect(const double* llbin, int nchunk, const double* logdet2, int64_t N,
                              int64_t G, double* llg, cudaStream_t s) {
  ll_collect_kernel<<<(unsigned)((G + 255) / 256), 256, 0, s>>>(llbin, nchunk, logdet2, N, G,
                                                                llg);
  return cudaGetLastError();
}

// one CTA per (m, level): fixed-order tree over bins
__global__ void ll_reduce_kernel(const double* __restrict__ llg, int64_t M, int64_t F, int64_t N,
                                 int I, int Lp1, double* __restrict__ loglik) {
  const int64_t m = blockIdx.x;
  const int l = blockIdx.y;
  const int64_t G = M * F;
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) s += llg[(size_t)l * G + m * F + f];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    loglik[m * Lp1 + l] = sh[0] - (double)N * (double)F * (double)I * kLogPi;
}

cudaError_t launch_ll_reduce(const double* llg, int64_t M, int64_t F, int64_t N, int I, int nlev,
                             int Lp1, double* loglik, cudaStream_t s) {
  dim3 grid((unsigned)M, (unsigned)nlev);
  ll_reduce_kernel<<<grid, 256, 0, s>>>(llg, M, F, N, I, Lp1, loglik);
  return cudaGetLastError();
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

void plan_chunks(int64_t G, int64_t N, int blocks_per_sm, int64_t* chunk_frames, int* nchunk,
                 int tile_bins, int64_t min_frames) {
  // Pick the frame chunking that minimises the modelled makespan
  //   waves(tiles * nchunk / resident CTAs) * (frames per chunk + per-CTA overhead)
  // so that the grid does not end on a mostly idle last wave (config 4:
  // 33 bin tiles; config 3: 2056). >= 16 frames per warp per chunk.
  const int64_t tiles = (G + tile_bins - 1) / tile_bins;
  const int64_t slots = (int64_t)sm_count() * (blocks_per_sm > 0 ? blocks_per_sm : 1);
  int64_t max_nc = (N + min_frames - 1) / min_frames;
  if (max_nc < 1) max_nc = 1;
  if (max_nc > 4096) max_nc = 4096;
  constexpr int64_t kOverhead = 24;  // frames-equivalent: P/W load, ring fill, reduction
  int64_t best_cf = N, best_cost = -1;
  for (int64_t nc = 1; nc <= max_nc; ++nc) {
    const int64_t cf = (N + nc - 1) / nc;
    const int64_t ncv = (N + cf - 1) / cf;
    if (ncv != nc) continue;  // same chunking as a smaller nc
    const int64_t waves = (tiles * ncv + slots - 1) / slots;
    const int64_t cost = waves * (cf + kOverhead);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_cf = cf;
    }
  }
  *chunk_frames = best_cf;
  *nchunk = (int)((N + best_cf - 1) / best_cf);
}

}  // namespace ffca
