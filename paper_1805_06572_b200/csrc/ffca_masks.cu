// Mask-clustering initial model on the device (reference initializers.py:42-143,
// SURVEY.md §8(f) row 3).
//
//  K7a masks_bin_kernel   one CTA per (mixture, bin): channel energies and
//                         frame powers, unit-normalised phase-aligned
//                         observations z (stored bin-major in the
//                         workspace), deterministic 2-means over the frames
//                         (_two_means, :42-68), unit-trace group
//                         covariances + 1e-2 ridge (:108-115);
//  K7b masks_pack / masks_gram / masks_align: cross-bin label alignment —
//                         greedy pass in decreasing bin-power order, then up
//                         to five refinement sweeps (:117-137) — on the exact
//                         integer centred masks N * mask - count (a flip is
//                         the sign of the exact rational correlation),
//                         evaluated through their Gram matrix (bit-packed
//                         popcounts) so each sequential step is O(F);
//  K7c masks_apply_kernel masked, floored powers (:139-143) and the S swap of
//                         flipped bins.
// Frames are spread over the CTA's threads with a fixed thread->frame map and
// fixed-order block reductions, so the result is deterministic.
#include <cstdio>
#include <cstdlib>

#include "ffca_internal.cuh"

namespace ffca {
namespace {

// threads per bin CTA (measured: 256 beats 32/64/128 even for 1250 frames)
constexpr int kMTLarge = 256;
// a bin whose phase-aligned observations fit keeps them (and its labels) in
// shared memory for all 2-means iterations instead of re-reading HBM
constexpr size_t kMaskSmemBytes = 100 * 1024;
inline size_t mask_smem(int64_t N, int I) {
  const size_t b = (size_t)N * I * 16 + (size_t)N;
  return b <= kMaskSmemBytes ? b : 0;
}
constexpr int kKmeansIters = 50;
constexpr double kMaskRidge = 1e-2;

constexpr int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
constexpr int ilog2(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}
struct NoFin {
  FFCA_DEV double operator()(int, double s) const { return s; }
};

// Sum of NV <= 32 values over the CTA, every thread receiving fin(k, total_k).
// Warp level: reduce-scatter (each butterfly step halves the values a lane
// holds: P2-1 shuffles instead of 5 NV), then plain butterflies; CTA level:
// thread k < NV adds the W warp partials in warp order and applies fin (e.g.
// the centroid division, done once instead of by every thread); the totals
// are broadcast through shared memory. Fixed order: deterministic.
// red: >= W * 32 + 32 doubles.
template <int NV, int W, typename Fin = NoFin>
FFCA_DEV void block_sum(double (&v)[NV], double* red, Fin fin = Fin()) {
  static_assert(NV >= 1 && NV <= 32, "block_sum handles up to 32 values per call");
  constexpr int P2 = pow2ceil(NV), LP = ilog2(P2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double h[P2];
#pragma unroll
  for (int k = 0; k < P2; ++k) h[k] = k < NV ? v[k] : 0.0;
#pragma unroll
  for (int st = 0; st < LP; ++st) {
    const int o = 16 >> st;
    const int half = P2 >> (st + 1);
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < P2 / 2; ++k) {
      if (k < half) {
        const double send = upper ? h[k] : h[k + half];
        const double keep = upper ? h[k + half] : h[k];
        h[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
  }
#pragma unroll
  for (int o = 16 >> LP; o > 0; o >>= 1) h[0] += __shfl_xor_sync(0xffffffffu, h[0], o);
  const int j = LP ? (lane >> (5 - LP)) & (P2 - 1) : 0;
  if ((lane & ((32 >> LP) - 1)) == 0 && j < NV) red[warp * P2 + j] = h[0];
  __syncthreads();
  if (threadIdx.x < NV) {
    double t = 0.0;
    for (int w = 0; w < W; ++w) t += red[w * P2 + threadIdx.x];
    red[W * P2 + threadIdx.x] = fin((int)threadIdx.x, t);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = red[W * P2 + k];
  __syncthreads();
}

// more than 32 values: chunks of 32
template <int NV, int W>
FFCA_DEV void block_sum_wide(double (&v)[NV], double* red) {
  if constexpr (NV <= 32) {
    block_sum<NV, W>(v, red);
  } else {
    double a[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) a[k] = v[k];
    block_sum<32, W>(a, red);
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = a[k];
    double b[NV - 32];
#pragma unroll
    for (int k = 0; k < NV - 32; ++k) b[k] = v[32 + k];
    block_sum_wide<NV - 32, W>(b, red);
#pragma unroll
    for (int k = 0; k < NV - 32; ++k) v[32 + k] = b[k];
  }
}

// (value, index, payload) with numpy argmax semantics: largest value, first
// index among equals
struct ArgMax {
  double v;
  int i;
  int pay;
};
FFCA_DEV bool better(const ArgMax& a, const ArgMax& b) {
  return a.v > b.v || (a.v == b.v && a.i < b.i);
}
template <int W>
FFCA_DEV ArgMax block_argmax(ArgMax a, double* rv, int* ri) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    b.pay = __shfl_xor_sync(0xffffffffu, a.pay, o);
    if (better(b, a)) a = b;
  }
  if (lane == 0) {
    rv[warp] = a.v;
    ri[2 * warp] = a.i;
    ri[2 * warp + 1] = a.pay;
  }
  __syncthreads();
  ArgMax r{rv[0], ri[0], ri[1]};
  for (int w = 1; w < W; ++w) {
    ArgMax b{rv[w], ri[2 * w], ri[2 * w + 1]};
    if (better(b, r)) r = b;
  }
  __syncthreads();
  return r;
}

template <int I, int kMT, bool SM>
__global__ void __launch_bounds__(kMT)
    masks_bin_kernel(const double2* __restrict__ y, int64_t N, int64_t F,
                     double2* __restrict__ zs, uint8_t* __restrict__ lab,
                     double* __restrict__ fpow, double* __restrict__ bpow, int* __restrict__ cnt,
                     double2* __restrict__ S) {
  constexpr int kMW = kMT / 32;
  constexpr int NE = I * (I + 1) / 2;  // upper-triangle entries of a covariance
  __shared__ double red[kMW * 32 + 32];
  __shared__ double rv[kMW];
  __shared__ int ri[2 * kMW];
  __shared__ int ired[2 * kMW];
  const int tid = threadIdx.x;
  const int64_t g = blockIdx.x;
  const int64_t m = (unsigned)g / (unsigned)F, f = g - m * F;  // (32-bit division)
  const double2* yb = y + (m * N * F + f) * I;
  const int64_t FI = F * I;
  extern __shared__ __align__(16) unsigned char zsm[];
  const int Ni = (int)N;  // N < 2^31 (checked by the caller)
  // SM: z and the labels live in shared memory (compile-time, so the loads
  // are LDS, not generic), channel-major ([a][n]: consecutive frames are
  // consecutive 16-B words, bank-conflict free); otherwise z is frame-major
  // in the workspace (one contiguous 16 I-byte row per frame)
  constexpr bool in_smem = SM;
  double2* zb = SM ? (double2*)zsm : zs + g * N * I;
  // element (a, n) of z; shared-memory indices fit 32 bits
  auto zat = [&](int a, int n) -> double2& {
    if constexpr (SM)
      return zb[a * Ni + n];
    else
      return zb[(size_t)n * I + a];
  };
  auto zdist = [&](int n, const double2(&c)[I]) {
    double d = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 za = zat(a, n);
      const double2 e = make_double2(za.x - c[a].x, za.y - c[a].y);
      d += e.x * e.x + e.y * e.y;
    }
    return d;
  };
  uint8_t* lb_out = lab + g * N;
  uint8_t* lb = in_smem ? zsm + (size_t)N * I * 16 : lb_out;
  double* pb = fpow + g * N;

  // 1. channel energies (reference channel) and frame powers
  double E[I];
#pragma unroll
  for (int a = 0; a < I; ++a) E[a] = 0.0;
  for (int n = tid; n < Ni; n += kMT) {
    double p = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 x = yb[n * FI + a];
      const double e = x.x * x.x + x.y * x.y;
      E[a] += e;
      p += e;
    }
    pb[n] = p;
  }
  block_sum<I, kMW>(E, red);
  int ref = 0;
  double tot = E[0];
#pragma unroll
  for (int a = 1; a < I; ++a) {
    if (E[a] > E[ref]) ref = a;
    tot += E[a];
  }
  if (tid == 0) bpow[g] = tot;

  // 2. z = w / max(|w|, 1e-300) * conj(phase of the reference channel)
  //    (initializers.py:100-106); highest-power frame seeds cluster 0
  ArgMax best{-1.0, 0x7fffffff, 0};
  for (int n = tid; n < Ni; n += kMT) {
    const double p = pb[n];
    const double nrm = fmax(sqrt(p), 1e-300);
    double2 z[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 x = yb[n * FI + a];
      z[a] = make_double2(x.x / nrm, x.y / nrm);
    }
    const double2 rvv = z[ref];
    const double mag = hypot(rvv.x, rvv.y);
    double2 ph = make_double2(1.0, 0.0);
    if (mag > 0.0) {
      const double d = fmax(mag, 1e-300);
      ph = make_double2(rvv.x / d, rvv.y / d);
    }
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 t = z[a];
      zat(a, n) = make_double2(t.x * ph.x + t.y * ph.y, t.y * ph.x - t.x * ph.y);
    }
    ArgMax c{p, (int)n, 0};
    if (better(c, best)) best = c;
  }
  best = block_argmax<kMW>(best, rv, ri);
  __syncthreads();  // z visible to the CTA
  double2 c0[I], c1[I];
#pragma unroll
  for (int a = 0; a < I; ++a) c0[a] = zat(a, best.i);
  // farthest frame from c0 seeds cluster 1
  ArgMax far{-1.0, 0x7fffffff, 0};
  for (int n = tid; n < Ni; n += kMT) {
    ArgMax c{zdist(n, c0), (int)n, 0};
    if (better(c, far)) far = c;
    lb[n] = 0;
  }
  far = block_argmax<kMW>(far, rv, ri);
#pragma unroll
  for (int a = 0; a < I; ++a) c1[a] = zat(a, far.i);

  // 3. 2-means (_two_means, initializers.py:42-68); label 1 = cluster 0
  long long count0 = 0;
#pragma unroll 1
  for (int it = 0; it < kKmeansIters; ++it) {
    // labels with the current centroids; counts by warp REDUX + one smem stage
    int cnt = 0, chg = 0;
#pragma unroll 4
    for (int n = tid; n < Ni; n += kMT) {
      const double d0 = zdist(n, c0);
      const double d1 = zdist(n, c1);
      const int nw = d0 <= d1 ? 1 : 0;
      const int old = lb[n] & 1;
      cnt += nw;
      chg += (nw != old);
      lb[n] = (uint8_t)(nw | (old << 1));  // bit 0: label, bit 1: previous label
    }
    cnt = (int)__reduce_add_sync(0xffffffffu, (unsigned)cnt);
    chg = (int)__reduce_add_sync(0xffffffffu, (unsigned)chg);
    if ((tid & 31) == 0) {
      ired[tid >> 5] = cnt;
      ired[kMW + (tid >> 5)] = chg;
    }
    __syncthreads();
    count0 = 0;
    long long changed = 0;
#pragma unroll
    for (int w = 0; w < kMW; ++w) {
      count0 += ired[w];
      changed += ired[kMW + w];
    }
    if (count0 == 0 || count0 == N) {  // re-seed the empty cluster with the worst fit
      ArgMax worst{-1.0, 0x7fffffff, 0};
      for (int n = tid; n < Ni; n += kMT) {  // rare: recompute the fits
        const double d0 = zdist(n, c0);
        const double d1 = zdist(n, c1);
        const int nw = lb[n] & 1;
        ArgMax c{nw ? d0 : d1, n, lb[n]};
        if (better(c, worst)) worst = c;
      }
      worst = block_argmax<kMW>(worst, rv, ri);
      const int nw = worst.pay & 1, old = (worst.pay >> 1) & 1;
      if (tid == 0) lb[worst.i] = (uint8_t)(1 - nw);
      count0 += nw ? -1 : 1;
      changed += (nw == old) ? 1 : -1;
    }
    __syncthreads();
    if (changed == 0) break;
    // centroids of the new groups
    double s[4 * I];
#pragma unroll
    for (int k = 0; k < 4 * I; ++k) s[k] = 0.0;
#pragma unroll 4
    for (int n = tid; n < Ni; n += kMT) {
      const int l = lb[n] & 1;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        const double2 z = zat(a, n);
        if (l) {
          s[2 * a] += z.x;
          s[2 * a + 1] += z.y;
        } else {
          s[2 * I + 2 * a] += z.x;
          s[2 * I + 2 * a + 1] += z.y;
        }
      }
    }
    const double n0 = (double)count0, n1 = (double)(N - count0);
    // centroids = group sums / group sizes (the division done once per value)
    block_sum<4 * I, kMW>(s, red, [=](int k, double t) { return t / (k < 2 * I ? n0 : n1); });
#pragma unroll
    for (int a = 0; a < I; ++a) {
      c0[a] = make_double2(s[2 * a], s[2 * a + 1]);
      c1[a] = make_double2(s[2 * I + 2 * a], s[2 * I + 2 * a + 1]);
    }
  }
  if (tid == 0) cnt[g] = (int)count0;
  if (in_smem)
    for (int n = tid; n < Ni; n += kMT) lb_out[n] = lb[n] & 1;

  // 4. group covariances sum w w^H / |group|, unit trace, + ridge (:108-115)
#pragma unroll 1
  for (int j = 0; j < 2; ++j) {
    const int want = j == 0 ? 1 : 0;
    const long long ng = j == 0 ? count0 : N - count0;
    double s[2 * NE];
#pragma unroll
    for (int k = 0; k < 2 * NE; ++k) s[k] = 0.0;
    for (int n = tid; n < Ni; n += kMT) {
      if ((lb[n] & 1) != want) continue;
      double2 w[I];
#pragma unroll
      for (int a = 0; a < I; ++a) w[a] = yb[n * FI + a];
      int e = 0;
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = a; b < I; ++b, ++e) {  // w_a conj(w_b)
          s[2 * e] += w[a].x * w[b].x + w[a].y * w[b].y;
          s[2 * e + 1] += w[a].y * w[b].x - w[a].x * w[b].y;
        }
    }
    block_sum_wide<2 * NE, kMW>(s, red);
    double2* Sd = S + ((m * 2 + j) * F + f) * I * I;
    if (tid == 0) {
      double tr = 0.0;
      double2 cov[I][I];
      int e = 0;
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = a; b < I; ++b, ++e) {
          double2 v = ng > 0 ? make_double2(s[2 * e] / (double)ng, s[2 * e + 1] / (double)ng)
                             : make_double2(a == b ? 1.0 : 0.0, 0.0);
          cov[a][b] = v;
          cov[b][a] = make_double2(v.x, -v.y);
        }
#pragma unroll
      for (int a = 0; a < I; ++a) tr += cov[a][a].x;
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = 0; b < I; ++b) {
          double2 v = tr > 0.0 ? make_double2(cov[a][b].x / tr, cov[a][b].y / tr)
                               : make_double2(a == b ? 1.0 / I : 0.0, 0.0);
          if (a == b) v.x += kMaskRidge;
          Sd[a * I + b] = v;
        }
    }
  }
}

// cross-bin alignment of one mixture; D_f[n] = N lab_f[n] - cnt_f (exact)
// ---- K7b: cross-bin alignment through the Gram matrix of the centred masks.
// With D_f = N b_f - k_f (b_f the bin's 0/1 labels, k_f their count), every
// correlation the reference evaluates is a signed sum of
//   Gram[f][h] = D_f . D_h = N^2 popc(b_f & b_h) - N k_f k_h   (exact, int64),
// so the running profile g = sum_h s_h D_h is tracked through
// hv[f] = D_f . g: a greedy step or a refinement flip of bin f updates hv
// with one Gram row (O(F) parallel work), and each decision is the sign of
// an exact integer — the same decisions as evaluating the dot products
// directly.

// labels (G, N) bytes -> bits (G, NW) words
__global__ void masks_pack_kernel(const uint8_t* __restrict__ lab, unsigned long long* __restrict__ bits,
                                  int64_t G, int64_t N, int64_t NW) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= G * NW) return;
  const int64_t g = t / NW, w = t - g * NW;
  const uint8_t* l = lab + g * N + w * 64;
  const int64_t nb = min((int64_t)64, N - w * 64);
  unsigned long long x = 0;
  for (int64_t i = 0; i < nb; ++i) x |= (unsigned long long)(l[i] & 1) << i;
  bits[t] = x;
}

// Gram[m][f][h] for one 32 x 32 tile of (f, h) per CTA (bit rows staged in
// shared memory in chunks of words)
constexpr int kGramWords = 32;
__global__ void __launch_bounds__(1024)
    masks_gram_kernel(const unsigned long long* __restrict__ bits, const int* __restrict__ cnt,
                      int64_t F, int64_t N, int64_t NW, long long* __restrict__ gram) {
  __shared__ unsigned long long ra[32][kGramWords + 1], rb[32][kGramWords + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t tiles = (F + 31) / 32;
  const int64_t m = blockIdx.z;
  const int64_t f = blockIdx.y * 32 + ty, h = blockIdx.x * 32 + tx;
  const unsigned long long* B = bits + m * F * NW;
  long long c = 0;
  for (int64_t w0 = 0; w0 < NW; w0 += kGramWords) {
    // stage rows f0..f0+31 and h0..h0+31, words w0..w0+31
    const int64_t fr = blockIdx.y * 32 + ty, hr = blockIdx.x * 32 + ty;
    const int64_t w = w0 + tx;
    ra[ty][tx] = (fr < F && w < NW) ? B[fr * NW + w] : 0ull;
    rb[ty][tx] = (hr < F && w < NW) ? B[hr * NW + w] : 0ull;
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < kGramWords; ++k) c += __popcll(ra[ty][k] & rb[tx][k]);
    __syncthreads();
  }
  (void)tiles;
  if (f < F && h < F) {
    const long long NN = (long long)N;
    const int* K = cnt + m * F;
    gram[(m * F + f) * F + h] = NN * NN * c - NN * (long long)K[f] * (long long)K[h];
  }
}

// one CTA per mixture: order, greedy pass, refinement sweeps (:117-137)
constexpr int kAlignT = 1024;
__global__ void __launch_bounds__(kAlignT)
    masks_align_kernel(const long long* __restrict__ gram, const double* __restrict__ bpow,
                       int64_t F, int* __restrict__ order, long long* __restrict__ hbuf,
                       uint8_t* __restrict__ flip) {
  __shared__ int sflip;
  const int tid = threadIdx.x;
  const int64_t m = blockIdx.x;
  const long long* Gm = gram + m * F * F;
  const double* P = bpow + m * F;
  int* ord = order + m * F;
  long long* hv = hbuf + m * F;
  uint8_t* fl = flip + m * F;
  // decreasing bin power, ties by index (stable)
  for (int64_t f = tid; f < F; f += kAlignT) {
    int64_t r = 0;
    const double pf = P[f];
    for (int64_t h = 0; h < F; ++h) r += (P[h] > pf) || (P[h] == pf && h < f);
    ord[r] = (int)f;
    fl[f] = 0;
  }
  __syncthreads();
  // greedy: g = D_{o0}; bin o_i flips when D . g < 0, then g += +-D
  {
    const int64_t f0 = ord[0];
    for (int64_t f = tid; f < F; f += kAlignT) hv[f] = Gm[f0 * F + f];  // Gram symmetric
  }
  __syncthreads();
#pragma unroll 1
  for (int64_t i = 1; i < F; ++i) {
    const int64_t f = ord[i];
    const bool neg = hv[f] < 0;
    __syncthreads();  // everyone read hv[f] before it changes
    const long long* row = Gm + f * F;
    if (neg) {
      if (tid == 0) fl[f] = 1;
      for (int64_t h = tid; h < F; h += kAlignT) hv[h] -= row[h];
    } else {
      for (int64_t h = tid; h < F; h += kAlignT) hv[h] += row[h];
    }
    __syncthreads();
  }
  // refinement: g = sum_h s_h D_h; flip f when s_f hv[f] - Gram[f][f] < 0
#pragma unroll 1
  for (int sweep = 0; sweep < 5; ++sweep) {
    for (int64_t f = tid; f < F; f += kAlignT) {
      long long acc = 0;
      const long long* row = Gm + f * F;
      for (int64_t h = 0; h < F; ++h) acc += fl[h] ? -row[h] : row[h];
      hv[f] = acc;
    }
    if (tid == 0) sflip = 0;
    __syncthreads();
#pragma unroll 1
    for (int64_t i = 0; i < F; ++i) {
      const int64_t f = ord[i];
      const long long sgn = fl[f] ? -1 : 1;
      const bool go = sgn * hv[f] - Gm[f * F + f] < 0;
      __syncthreads();
      if (go) {  // g -= 2 s D_f
        const long long* row = Gm + f * F;
        for (int64_t h = tid; h < F; h += kAlignT) hv[h] -= 2 * sgn * row[h];
        if (tid == 0) {
          fl[f] = fl[f] ? 0 : 1;
          sflip = 1;
        }
      }
      __syncthreads();
    }
    if (!sflip) break;
    __syncthreads();
  }
}

// v = max(mask * |y|^2 / I, floor) per source (:139-143); swap S of flipped bins
template <int I>
__global__ void masks_apply_kernel(const uint8_t* __restrict__ lab, const uint8_t* __restrict__ flip,
                                   const double* __restrict__ fpow, const double* __restrict__ floor,
                                   double* __restrict__ v, double2* __restrict__ S, int64_t M,
                                   int64_t N, int64_t F) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < M * F && flip[t]) {  // swap the two sources' covariances of this bin
    const int64_t m = t / F, f = t - m * F;
    double2* a = S + ((m * 2 + 0) * F + f) * I * I;
    double2* b = S + ((m * 2 + 1) * F + f) * I * I;
    for (int e = 0; e < I * I; ++e) {
      const double2 x = a[e];
      a[e] = b[e];
      b[e] = x;
    }
  }
  if (t >= M * N * F) return;
  const int64_t m = t / (N * F);
  const int64_t r = t - m * N * F;
  const int64_t n = r / F, f = r - n * F;
  const int64_t g = m * F + f;
  const int l = lab[g * N + n] ^ flip[g];
  const double pp = fpow[g * N + n] / I;
  const double fl = floor[g];
  const double a = l ? pp : 0.0, b = l ? 0.0 : pp;
  v[(m * 2 + 0) * N * F + n * F + f] = a < fl ? fl : a;
  v[(m * 2 + 1) * N * F + n * F + f] = b < fl ? fl : b;
}

struct MaskWs {
  double2* zs;
  double* fpow;
  double* bpow;
  long long* gram;
  long long* hbuf;
  unsigned long long* bits;
  int* cnt;
  int* order;
  uint8_t* lab;
  uint8_t* flip;
  size_t bytes;
};

MaskWs carve_masks(void* base, int64_t M, int64_t N, int64_t F, int I) {
  MaskWs w{};
  size_t off = 0;
  auto take = [&](size_t nbytes) {
    const size_t o = off;
    off += (nbytes + 255) / 256 * 256;
    return base ? (char*)base + o : nullptr;
  };
  const int64_t G = M * F;
  w.zs = (double2*)take((size_t)G * N * I * sizeof(double2));
  w.fpow = (double*)take((size_t)G * N * sizeof(double));
  w.bpow = (double*)take((size_t)G * sizeof(double));
  const int64_t NW = (N + 63) / 64;
  w.gram = (long long*)take((size_t)M * F * F * sizeof(long long));
  w.hbuf = (long long*)take((size_t)G * sizeof(long long));
  w.bits = (unsigned long long*)take((size_t)G * NW * sizeof(unsigned long long));
  w.cnt = (int*)take((size_t)G * sizeof(int));
  w.order = (int*)take((size_t)G * sizeof(int));
  w.lab = (uint8_t*)take((size_t)G * N);
  w.flip = (uint8_t*)take((size_t)G);
  w.bytes = off;
  return w;
}

// a failing step is named on stderr when FFCA_DEBUG_SYNC is set
int masks_fail(const char* step, cudaError_t e) {
  if (getenv("FFCA_DEBUG_SYNC"))
    fprintf(stderr, "ffca_init_masks: %s: %s\n", step, cudaGetErrorString(e));
  return FFCA_ERR_CUDA;
}

}  // namespace

cudaError_t launch_init_powers(const void* y, void* v, double* floor, int64_t M, int64_t N,
                               int64_t F, int I, int dtype, cudaStream_t s);

}  // namespace ffca

using namespace ffca;

extern "C" {

size_t ffca_init_masks_workspace_size(int64_t M, int64_t N, int64_t F, int I) {
  if (M < 1 || N < 1 || F < 1 || I < 1 || I > kMaxOrder) return 0;
  return carve_masks(nullptr, M, N, F, I).bytes;
}

int ffca_init_masks(const double* y, double* v, double* S, double* v_floor, int64_t M, int64_t N,
                    int64_t F, int I, void* workspace, size_t workspace_bytes, void* stream) {
  if (!y || !v || !S || !v_floor || !workspace || M < 1 || F < 1 || I < 1 || I > kMaxOrder ||
      N < 2 * I || N > 0x7fffffff)
    return FFCA_ERR_INVALID;
  const MaskWs w = carve_masks(workspace, M, N, F, I);
  if (w.bytes > workspace_bytes) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_init_powers(y, v, v_floor, M, N, F, I, FFCA_C128, s);  // floor
  if (e != cudaSuccess) return masks_fail("init_powers", e);
  const double2* y2 = (const double2*)y;
  double2* S2 = (double2*)S;
  const size_t zsmem = mask_smem(N, I);
  switch (I) {
#define FFCA_MASK_CASE(II)                                                                  \
  case II:                                                                                  \
    if (zsmem > 0) {                                                                        \
      if ((e = cudaFuncSetAttribute(masks_bin_kernel<II, kMTLarge, true>,                   \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                                    (int)zsmem)) != cudaSuccess)                            \
        return masks_fail("bin kernel smem attribute", e);                                  \
      masks_bin_kernel<II, kMTLarge, true><<<(unsigned)(M * F), kMTLarge, zsmem, s>>>(      \
          y2, N, F, w.zs, w.lab, w.fpow, w.bpow, w.cnt, S2);                                \
    } else {                                                                                \
      masks_bin_kernel<II, kMTLarge, false><<<(unsigned)(M * F), kMTLarge, 0, s>>>(         \
          y2, N, F, w.zs, w.lab, w.fpow, w.bpow, w.cnt, S2);                                \
    }                                                                                       \
    break;
    FFCA_MASK_CASE(1)
    FFCA_MASK_CASE(2)
    FFCA_MASK_CASE(3)
    FFCA_MASK_CASE(4)
    FFCA_MASK_CASE(5)
    FFCA_MASK_CASE(6)
    FFCA_MASK_CASE(7)
    FFCA_MASK_CASE(8)
#undef FFCA_MASK_CASE
    default:
      return FFCA_ERR_INVALID;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return masks_fail("bin kernel", e);
  {
    const int64_t NW = (N + 63) / 64;
    const int64_t G = M * F;
    masks_pack_kernel<<<(unsigned)((G * NW + 255) / 256), 256, 0, s>>>(w.lab, w.bits, G, N, NW);
    const unsigned t = (unsigned)((F + 31) / 32);
    masks_gram_kernel<<<dim3(t, t, (unsigned)M), 1024, 0, s>>>(w.bits, w.cnt, F, N, NW, w.gram);
    masks_align_kernel<<<(unsigned)M, kAlignT, 0, s>>>(w.gram, w.bpow, F, w.order, w.hbuf,
                                                       w.flip);
    if ((e = cudaGetLastError()) != cudaSuccess) return masks_fail("alignment", e);
  }
  const int64_t total = M * N * F;
  const unsigned nb = (unsigned)((total + 255) / 256);
  switch (I) {
#define FFCA_APPLY_CASE(II)                                                               \
  case II:                                                                                \
    masks_apply_kernel<II><<<nb, 256, 0, s>>>(w.lab, w.flip, w.fpow, v_floor, v, S2, M,  \
                                              N, F);                                      \
    break;
    FFCA_APPLY_CASE(1)
    FFCA_APPLY_CASE(2)
    FFCA_APPLY_CASE(3)
    FFCA_APPLY_CASE(4)
    FFCA_APPLY_CASE(5)
    FFCA_APPLY_CASE(6)
    FFCA_APPLY_CASE(7)
    FFCA_APPLY_CASE(8)
#undef FFCA_APPLY_CASE
    default:
      return FFCA_ERR_INVALID;
  }
  return cudaGetLastError() == cudaSuccess ? FFCA_OK : FFCA_ERR_CUDA;
}

}  // extern "C"
