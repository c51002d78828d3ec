// K8 — separation quality on the device: the reference's SDR (metrics.py:27-60).
//
// Per signal pair (estimate channel e, reference channel r, length L) the
// reference projects e onto the span of r delayed by 0..T-1 samples
// (T = max_shift + 1 taps; an L x T least-squares problem, lstsq) and reports
// 10 log10(|proj|^2 / max(|e - proj|^2, 1e-30 |proj|^2)), -300 dB for a zero
// projection. Here the same least-squares solution comes from the normal
// equations of the delay basis B:
//   G = B^T B, G[d1][d2] = sum_{n >= max(d1,d2)} r[n-d1] r[n-d2]
//                        = A(d2-d1) - sum_{j=L-d1}^{L-1} r[j] r[j-(d2-d1)]   (d2 >= d1)
//   c = B^T e, c[d] = sum_{n >= d} e[n] r[n-d]
// with A(k) = sum_{n >= k} r[n] r[n-k] the autocorrelation: one streaming
// pass computes the 2T lags per sample block (lane = lag), a per-pair warp
// sums the block partials in fixed order, applies the end corrections,
// factors G (Cholesky, FP64) and solves for the taps h; a second streaming
// pass forms proj = B h with a T-tap FIR and the two energies explicitly
// (as the reference does: the residual is never taken as |e|^2 - |proj|^2).
// All reductions are in fixed order: deterministic. A delay basis that is
// numerically rank deficient (pivot <= 1e-13 of the largest diagonal; e.g. a
// reference shorter than T or periodic with a period dividing a delay) has
// the dependent columns dropped — the reference's lstsq takes the minimum-
// norm solution there, whose projection is the same span's; flagged.
#include "ffca_internal.cuh"

namespace ffca {
namespace {

constexpr int kMaxTaps = 64;
constexpr int kTile = 4096;       // samples per block of a streaming pass
constexpr int kThreads = 256;     // 8 warps
constexpr double kCapRatio = 1e-30;  // metrics.py:13 (_SDR_CAP_RATIO)

struct SdrWs {
  double* stats;  // [nblk][P][2 T]: A(k), c(d) partials
  double* h;      // [P][T]
  double* en;     // [nblk][P][2]: target, noise partials
  size_t bytes;
};

SdrWs carve_sdr(void* base, int64_t P, int64_t L, int T) {
  const int64_t nblk = (L + kTile - 1) / kTile;
  SdrWs w{};
  size_t off = 0;
  auto take = [&](size_t n) {
    double* p = base ? (double*)((char*)base + off) : nullptr;
    off += ((n * sizeof(double) + 255) / 256) * 256;
    return p;
  };
  w.stats = take((size_t)nblk * P * 2 * T);
  w.h = take((size_t)P * T);
  w.en = take((size_t)nblk * P * 2);
  w.bytes = off;
  return w;
}

// stage r[n0 - (T-1) .. n0 + kTile) (zeros outside [0, L)) and e[n0 .. n0 + kTile)
__device__ void stage_tile(const double* __restrict__ r, const double* __restrict__ e, int64_t L,
                           int64_t n0, int T, double* sr, double* se) {
  for (int i = threadIdx.x; i < kTile + T - 1; i += blockDim.x) {
    const int64_t n = n0 - (T - 1) + i;
    sr[i] = (n >= 0 && n < L) ? r[n] : 0.0;
  }
  if (se)
    for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
      const int64_t n = n0 + i;
      se[i] = n < L ? e[n] : 0.0;
    }
  __syncthreads();
}

// pass 1: per block, A(k) and c(d) partials (lane = lag; warps split the block)
__global__ void __launch_bounds__(kThreads) sdr_stats_kernel(const double* __restrict__ est,
                                                             const double* __restrict__ ref,
                                                             int64_t P, int64_t L, int T,
                                                             double* __restrict__ stats) {
  extern __shared__ double sm[];
  double* sr = sm;                     // kTile + T - 1
  double* se = sr + kTile + kMaxTaps;  // kTile
  double* red = se + kTile;            // [8 warps][2 T]
  const int64_t p = blockIdx.y, blk = blockIdx.x;
  const int64_t n0 = blk * kTile;
  stage_tile(ref + p * L, est + p * L, L, n0, T, sr, se);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kPer = kTile / (kThreads / 32);
  double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;  // lags lane, lane + 32
  const int i0 = warp * kPer;
  const int l0 = lane < T ? lane : 0;  // lanes past the last lag read lag 0 (discarded)
#pragma unroll 4
  for (int i = i0; i < i0 + kPer; ++i) {
    const double rn = sr[i + T - 1], en = se[i];
    const double r0 = sr[i + T - 1 - l0];
    a0 = fma(rn, r0, a0);
    c0 = fma(en, r0, c0);
    if (T > 32) {
      const double r1 = lane + 32 < T ? sr[i + T - 1 - lane - 32] : 0.0;
      a1 = fma(rn, r1, a1);
      c1 = fma(en, r1, c1);
    }
  }
  double* rw = red + warp * 2 * kMaxTaps;
  rw[lane] = a0;
  rw[lane + 32] = a1;
  rw[kMaxTaps + lane] = c0;
  rw[kMaxTaps + lane + 32] = c1;
  __syncthreads();
  // fixed-order sum over the warps, lag-parallel
  for (int t = threadIdx.x; t < 2 * T; t += blockDim.x) {
    const int which = t / T, k = t - which * T;
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w * 2 * kMaxTaps + which * kMaxTaps + k];
    stats[(blk * P + p) * 2 * T + t] = s;
  }
}

// per pair: ordered block sums, end corrections, Cholesky of G, taps h
__global__ void __launch_bounds__(kMaxTaps) sdr_solve_kernel(const double* __restrict__ ref,
                                                             int64_t P, int64_t L, int T,
                                                             int64_t nblk,
                                                             const double* __restrict__ stats,
                                                             double* __restrict__ h_out,
                                                             int* __restrict__ flags) {
  __shared__ double G[kMaxTaps][kMaxTaps + 1];
  __shared__ double A[kMaxTaps], c[kMaxTaps], tail[2 * kMaxTaps], piv[2];
  __shared__ double z[kMaxTaps];
  __shared__ int drop[kMaxTaps];
  const int64_t p = blockIdx.x;
  const int t = threadIdx.x;
  if (t < T) {
    double sa = 0.0, sc = 0.0;
    for (int64_t b = 0; b < nblk; ++b) {
      sa += stats[(b * P + p) * 2 * T + t];
      sc += stats[(b * P + p) * 2 * T + T + t];
    }
    A[t] = sa;
    c[t] = sc;
  }
  // the last 2T samples of r (end corrections), zeros before the start
  for (int i = t; i < 2 * T; i += blockDim.x) {
    const int64_t n = L - 2 * T + i;
    tail[i] = n >= 0 ? ref[p * L + n] : 0.0;
  }
  __syncthreads();
  const double* rt = tail + 2 * T;  // rt[j - L] = r[j] for j in [L - 2T, L)
  if (t < T) {
    const int d1 = t;
    for (int d2 = d1; d2 < T; ++d2) {
      const int k = d2 - d1;
      double corr = 0.0;
      for (int j = -d1; j < 0; ++j)  // j - L in [-d1, 0): r[j] r[j - k]
        corr = fma(rt[j], (L + j - k >= 0) ? rt[j - k] : 0.0, corr);
      const double g = A[k] - corr;
      G[d1][d2] = g;
      G[d2][d1] = g;
    }
  }
  __syncthreads();
  int flag = (A[0] == 0.0) ? 1 : 0;  // silent reference (MetricError in the wrapper)
  double gmax = 0.0;
  for (int d = 0; d < T; ++d) gmax = fmax(gmax, G[d][d]);
  // Cholesky G = L L^T in place (lower), column-sequential, row-parallel;
  // numerically dependent columns (pivot <= 1e-13 gmax) are dropped
  for (int j = 0; j < T; ++j) {
    if (t == j) {
      double d = G[j][j];
      for (int k = 0; k < j; ++k) d -= G[j][k] * G[j][k];
      const bool ok = d > 1e-13 * gmax && d > 0.0;
      drop[j] = ok ? 0 : 1;
      piv[0] = ok ? sqrt(d) : 0.0;
      piv[1] = ok ? 1.0 / piv[0] : 0.0;
      G[j][j] = piv[0];
    }
    __syncthreads();
    if (t > j && t < T) {
      double s = G[t][j];
      for (int k = 0; k < j; ++k) s -= G[t][k] * G[j][k];
      G[t][j] = s * piv[1];
    }
    __syncthreads();
  }
  // forward (L z = c) and back (L^T h = z) substitution, dropped columns -> 0
  if (t == 0) {
    for (int i = 0; i < T; ++i) {
      if (drop[i]) {
        z[i] = 0.0;
        continue;
      }
      double s = c[i];
      for (int k = 0; k < i; ++k) s -= G[i][k] * z[k];
      z[i] = s / G[i][i];
    }
    for (int i = T - 1; i >= 0; --i) {
      if (drop[i]) {
        z[i] = 0.0;
        continue;
      }
      double s = z[i];
      for (int k = i + 1; k < T; ++k) s -= G[k][i] * z[k];
      z[i] = s / G[i][i];
    }
  }
  __syncthreads();
  if (t < T) h_out[p * T + t] = z[t];
  if (t == 0) {
    int nd = 0;
    for (int i = 0; i < T; ++i) nd += drop[i];
    if (nd) flag |= 2;
    flags[p] = flag;
  }
}

// pass 2: proj = B h (T-tap FIR), partial target / noise energies per block
__global__ void __launch_bounds__(kThreads) sdr_resid_kernel(const double* __restrict__ est,
                                                             const double* __restrict__ ref,
                                                             int64_t P, int64_t L, int T,
                                                             const double* __restrict__ h_in,
                                                             double* __restrict__ en) {
  extern __shared__ double sm[];
  double* sr = sm;                     // kTile + T - 1
  double* sh = sr + kTile + kMaxTaps;  // T
  __shared__ double red[2][kThreads / 32];
  const int64_t p = blockIdx.y, blk = blockIdx.x;
  const int64_t n0 = blk * kTile;
  for (int i = threadIdx.x; i < T; i += blockDim.x) sh[i] = h_in[p * T + i];
  stage_tile(ref + p * L, nullptr, L, n0, T, sr, nullptr);
  const double* e = est + p * L;
  double tg = 0.0, ns = 0.0;
  for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
    const int64_t n = n0 + i;
    if (n >= L) break;
    double pr = 0.0;
    for (int d = 0; d < T; ++d) pr = fma(sh[d], sr[i + T - 1 - d], pr);
    const double rs = e[n] - pr;
    tg = fma(pr, pr, tg);
    ns = fma(rs, rs, ns);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tg += __shfl_xor_sync(0xffffffffu, tg, o);
    ns += __shfl_xor_sync(0xffffffffu, ns, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = tg;
    red[1][warp] = ns;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    en[(blk * P + p) * 2 + 0] = a;
    en[(blk * P + p) * 2 + 1] = b;
  }
}

__global__ void sdr_final_kernel(int64_t P, int64_t nblk, const double* __restrict__ en,
                                 double* __restrict__ sdr_db) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double target = 0.0, noise = 0.0;
  for (int64_t b = 0; b < nblk; ++b) {
    target += en[(b * P + p) * 2 + 0];
    noise += en[(b * P + p) * 2 + 1];
  }
  sdr_db[p] = target <= 0.0 ? -300.0 : 10.0 * log10(target / fmax(noise, kCapRatio * target));
}

}  // namespace
}  // namespace ffca

extern "C" {

size_t ffca_sdr_workspace_size(int64_t pairs, int64_t length, int max_shift) {
  if (pairs < 1 || length < 1 || max_shift < 0 || max_shift + 1 > ffca::kMaxTaps) return 0;
  return ffca::carve_sdr(nullptr, pairs, length, max_shift + 1).bytes;
}

int ffca_sdr(const double* est, const double* ref, int64_t pairs, int64_t length, int max_shift,
             double* sdr_db, int* flags, void* workspace, void* stream) {
  using namespace ffca;
  if (!est || !ref || !sdr_db || !flags || !workspace || pairs < 1 || length < 1 ||
      max_shift < 0 || max_shift + 1 > kMaxTaps || pairs > 65535)
    return FFCA_ERR_INVALID;
  const int T = max_shift + 1;
  const int64_t P = pairs, L = length;
  const int64_t nblk = (L + kTile - 1) / kTile;
  if (nblk > 0x7fffffff) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  SdrWs w = carve_sdr(workspace, P, L, T);
  const size_t sm1 = (size_t)(kTile + kMaxTaps + kTile + (kThreads / 32) * 2 * kMaxTaps) * 8;
  const size_t sm3 = (size_t)(kTile + kMaxTaps + kMaxTaps) * 8;
  if (ensure_smem<sdr_stats_kernel>(sm1) != cudaSuccess) return FFCA_ERR_CUDA;
  sdr_stats_kernel<<<dim3((unsigned)nblk, (unsigned)P), kThreads, sm1, s>>>(est, ref, P, L, T,
                                                                          w.stats);
  sdr_solve_kernel<<<(unsigned)P, kMaxTaps, 0, s>>>(ref, P, L, T, nblk, w.stats, w.h, flags);
  if (ensure_smem<sdr_resid_kernel>(sm3) != cudaSuccess) return FFCA_ERR_CUDA;
  sdr_resid_kernel<<<dim3((unsigned)nblk, (unsigned)P), kThreads, sm3, s>>>(est, ref, P, L, T,
                                                                          w.h, w.en);
  sdr_final_kernel<<<(unsigned)((P + 127) / 128), 128, 0, s>>>(P, nblk, w.en, sdr_db);
  return cudaGetLastError() == cudaSuccess ? FFCA_OK : FFCA_ERR_CUDA;
}

}  // extern "C"
