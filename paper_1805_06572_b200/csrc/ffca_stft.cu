// STFT front and back end on the device (reference stft.py:9-107):
// square-root periodic Hann window, 50% overlap, half a frame of leading zero
// padding, rfft / irfft per frame and overlap-add.
//
// Frame lengths up to 4096 run the team-FFT kernels below (register radix-16
// Stockham passes); 8192 runs the simpler radix-2 shared-memory kernels.
// Both directions are persistent kernels (grid = resident CTAs, each CTA a
// contiguous run of frames / output hops) so the per-CTA tables (twiddles
// e^{-2 pi i k / L} and the window) are built once per CTA, not per frame.
// A length-L real transform is a length-H = L/2 complex FFT of the packed
// even/odd samples (radix-2 DIT in shared memory, input in bit-reversed
// order) plus an O(H) split step; everything is FP64.
//  * analysis: x (B, C, length) f64 -> spec (B, N, H+1, C) c128, the EM
//    kernels' (frame, bin, channel) layout, written bin-major/channel-minor so
//    a frame's (F, C) block leaves the CTA as one contiguous run;
//  * synthesis: spec (B, N, H+1, C) -> out (B, C, length): output hop q is the
//    second half of frame q plus the first half of frame q+1 (the reference's
//    overlap-add order), gathered by the CTA that owns hop q — deterministic,
//    no atomics; a CTA keeps the previous frame's second half in shared
//    memory, so each frame is inverse-transformed once (plus one per CTA run).
#include "ffca_internal.cuh"

namespace ffca {
namespace {

constexpr int kStftThreads = 256;
constexpr int kStftMaxLength = 8192;
#ifndef FFCA_TEAM_THREADS
#define FFCA_TEAM_THREADS 128
#endif
constexpr int kTeamThreads = FFCA_TEAM_THREADS;  // team kernels: small CTAs, several per SM
constexpr double kPi = 3.141592653589793;  // np.pi

struct StftSmem {
  int H;
  size_t tw, win, buf, prev, bytes;
};

// layout: tw[H] c128 | win[L] f64 | buf[nc][H] c128 | prev[nc][H] f64
__host__ __device__ StftSmem stft_smem(int L, int nc, bool synth) {
  StftSmem s{};
  s.H = L / 2;
  s.tw = 0;
  s.win = s.tw + (size_t)s.H * 16;
  s.buf = s.win + (size_t)L * 8;
  s.prev = s.buf + (size_t)nc * s.H * 16;
  s.bytes = s.prev + (synth ? (size_t)nc * s.H * 8 : 0);
  return s;
}

FFCA_DEV void stft_tables(double2* tw, double* win, int L) {
  const int H = L / 2;
  for (int k = threadIdx.x; k < H; k += blockDim.x) {
    double sn, cs;
    sincospi(-2.0 * (double)k / (double)L, &sn, &cs);  // exact argument (L = 2^p)
    tw[k] = make_double2(cs, sn);
  }
  // stft.py:16-19, same evaluation order: sqrt(0.5 * (1 - cos(2 pi t / L)))
  for (int t = threadIdx.x; t < L; t += blockDim.x)
    win[t] = sqrt(0.5 * (1.0 - cos(2.0 * kPi * (double)t / (double)L)));
}

// in-place radix-2 DIT over nc independent length-H rows (input bit-reversed)
FFCA_DEV void fft_rows(double2* buf, int nc, int logH, const double2* tw) {
  const int H = 1 << logH;
  const int half = H >> 1;
  const int nb = nc * half;
  for (int lm = 0; lm < logH; ++lm) {
    const int m = 1 << lm;
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const int c = t / half;
      const int b = t - c * half;
      const int j = b & (m - 1);
      const int i0 = ((b >> lm) << (lm + 1)) + j;
      double2* x = buf + (size_t)c * H;
      const double2 w = tw[j << (logH - lm)];  // e^{-2 pi i j / (2m)}
      const double2 a = x[i0];
      const double2 bw = cmul(x[i0 + m], w);
      x[i0] = cadd(a, bw);
      x[i0 + m] = csub(a, bw);
    }
    __syncthreads();
  }
}

FFCA_DEV int bitrev(int n, int logH) {
  return logH == 0 ? 0 : (int)(__brev((unsigned)n) >> (32 - logH));
}

__global__ void __launch_bounds__(kStftThreads)
    stft_analyze_kernel(const double* __restrict__ x, double2* __restrict__ out, int64_t B, int C,
                        int64_t len, int L, int logH, int64_t N, int cg) {
  extern __shared__ __align__(16) unsigned char sm[];
  const StftSmem lay = stft_smem(L, cg, false);
  const int H = lay.H;
  const int F = H + 1;
  double2* tw = (double2*)(sm + lay.tw);
  double* win = (double*)(sm + lay.win);
  double2* buf = (double2*)(sm + lay.buf);
  stft_tables(tw, win, L);
  __syncthreads();

  const int64_t total = B * N;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = (int64_t)blockIdx.x * per;
  const int64_t u1 = min(total, u0 + per);
  for (int64_t u = u0; u < u1; ++u) {
    const int64_t b = u / N, k = u - b * N;
    const int64_t base = (k - 1) * H;  // frame k starts at padded k*H = signal (k-1)*H
    for (int c0 = 0; c0 < C; c0 += cg) {
      const int nc = min(cg, C - c0);
      // windowed samples, packed z_n = x_2n + i x_2n+1, bit-reversed
      for (int t = threadIdx.x; t < nc * H; t += blockDim.x) {
        const int c = t / H, n = t - c * H;
        const double* xc = x + ((size_t)b * C + c0 + c) * len;
        const int64_t i0 = base + 2 * n, i1 = i0 + 1;
        const double a0 = (i0 >= 0 && i0 < len) ? xc[i0] : 0.0;
        const double a1 = (i1 >= 0 && i1 < len) ? xc[i1] : 0.0;
        buf[(size_t)c * H + bitrev(n, logH)] = make_double2(a0 * win[2 * n], a1 * win[2 * n + 1]);
      }
      __syncthreads();
      fft_rows(buf, nc, logH, tw);
      // split: X_f = E_f + e^{-2 pi i f / L} O_f, E/O = even/odd-sample spectra
      double2* o = out + ((size_t)b * N + k) * F * C + c0;
      for (int t = threadIdx.x; t < F * nc; t += blockDim.x) {
        const int f = t / nc, c = t - f * nc;
        const double2* z = buf + (size_t)c * H;
        const double2 zk = z[f & (H - 1)];
        const double2 zm = cconj(z[(H - f) & (H - 1)]);
        const double2 e = cscale(cadd(zk, zm), 0.5);
        const double2 d = cscale(csub(zk, zm), 0.5);
        const double2 od = make_double2(d.y, -d.x);  // d / i
        const double2 w = f < H ? tw[f] : make_double2(-1.0, 0.0);
        o[(size_t)f * C + c] = cadd(e, cmul(w, od));
      }
      __syncthreads();
    }
  }
}

// inverse-transform frame k of item b for channels [c0, c0 + nc) into buf as
// windowed time samples (buf viewed as double[nc][L])
FFCA_DEV void synth_frame(const double2* __restrict__ spec, int64_t b, int64_t k, int64_t N, int C,
                          int c0, int nc, int logH, const double2* tw, const double* win,
                          double2* buf) {
  const int H = 1 << logH;
  const int F = H + 1;
  const double2* s = spec + ((size_t)b * N + k) * F * C + c0;
  const int hh = H / 2;  // pairs (kk, H - kk) for kk = 0 .. H/2
  for (int t = threadIdx.x; t < (hh + 1) * nc; t += blockDim.x) {
    const int kk = t / nc, c = t - kk * nc;
    double2 xa = s[(size_t)kk * C + c];
    double2 xb = s[(size_t)(H - kk) * C + c];
    if (kk == 0) {  // DC and Nyquist are real-valued (stft.py:91-92)
      xa.y = 0.0;
      xb.y = 0.0;
    }
    double2* z = buf + (size_t)c * H;
    // Z_k = E_k + i O_k, E = (X_k + X*_{H-k}) / 2, O = (X_k - X*_{H-k}) e^{+2 pi i k / L} / 2
    {
      const double2 xm = cconj(xb);
      const double2 e = cscale(cadd(xa, xm), 0.5);
      const double2 d = cscale(csub(xa, xm), 0.5);
      const double2 od = cmul(d, cconj(tw[kk]));
      const double2 zk = make_double2(e.x - od.y, e.y + od.x);
      z[bitrev(kk, logH)] = cconj(zk);  // inverse FFT = conj(FFT(conj Z))
    }
    if (kk != 0 && kk != H - kk) {
      const int k2 = H - kk;
      const double2 xm = cconj(xa);
      const double2 e = cscale(cadd(xb, xm), 0.5);
      const double2 d = cscale(csub(xb, xm), 0.5);
      const double2 od = cmul(d, cconj(tw[k2]));
      const double2 zk = make_double2(e.x - od.y, e.y + od.x);
      z[bitrev(k2, logH)] = cconj(zk);
    }
  }
  __syncthreads();
  fft_rows(buf, nc, logH, tw);
  const double invH = 1.0 / (double)H;
  for (int t = threadIdx.x; t < nc * H; t += blockDim.x) {
    const int c = t / H, n = t - c * H;
    double2 r = buf[(size_t)c * H + n];
    r.x = r.x * invH * win[2 * n];
    r.y = -r.y * invH * win[2 * n + 1];
    buf[(size_t)c * H + n] = r;  // (x_2n, x_2n+1)
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kStftThreads)
    stft_synth_kernel(const double2* __restrict__ spec, double* __restrict__ out, int64_t B, int C,
                      int64_t N, int L, int logH, int64_t len, int cg) {
  extern __shared__ __align__(16) unsigned char sm[];
  const StftSmem lay = stft_smem(L, cg, true);
  const int H = lay.H;
  double2* tw = (double2*)(sm + lay.tw);
  double* win = (double*)(sm + lay.win);
  double2* buf = (double2*)(sm + lay.buf);
  double* prev = (double*)(sm + lay.prev);
  stft_tables(tw, win, L);
  __syncthreads();

  const int64_t Q = (len + H - 1) / H;  // output hops per item
  const int64_t total = B * Q;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = (int64_t)blockIdx.x * per;
  const int64_t u1 = min(total, u0 + per);
  for (int c0 = 0; c0 < C; c0 += cg) {
    const int nc = min(cg, C - c0);
    int64_t have_b = -1, have_q = -1;  // prev holds frame have_q's second half
    for (int64_t u = u0; u < u1; ++u) {
      const int64_t b = u / Q, q = u - b * Q;
      const double* fb = (const double*)buf;
      if (have_b != b || have_q != q) {  // start of a run: frame q itself
        synth_frame(spec, b, q, N, C, c0, nc, logH, tw, win, buf);
        for (int t = threadIdx.x; t < nc * H; t += blockDim.x) {
          const int c = t / H, s = t - c * H;
          prev[(size_t)c * H + s] = fb[(size_t)c * L + H + s];
        }
        __syncthreads();
      }
      const bool next = q + 1 < N;
      if (next) synth_frame(spec, b, q + 1, N, C, c0, nc, logH, tw, win, buf);
      // out[q H + s] = frame_q[H + s] + frame_{q+1}[s] (stft.py:97-99 order)
      const int64_t t0 = q * H;
      for (int t = threadIdx.x; t < nc * H; t += blockDim.x) {
        const int c = t / H, s = t - c * H;
        const double a = prev[(size_t)c * H + s];
        const double v = next ? a + fb[(size_t)c * L + s] : a;
        if (t0 + s < len) out[((size_t)b * C + c0 + c) * len + t0 + s] = v;
      }
      __syncthreads();
      if (next) {
        for (int t = threadIdx.x; t < nc * H; t += blockDim.x) {
          const int c = t / H, s = t - c * H;
          prev[(size_t)c * H + s] = fb[(size_t)c * L + H + s];
        }
        __syncthreads();
      }
      have_b = b;
      have_q = q + 1;
    }
  }
}

int log2_exact(int L) {
  if (L < 2 || L > kStftMaxLength || (L & (L - 1))) return -1;
  int p = 0;
  while ((1 << p) < L) ++p;
  return p;
}

// channels per pass so that a CTA's shared memory stays within budget
int stft_group(int L, int C, bool synth, size_t* bytes) {
  const size_t budget = 112 * 1024;
  int cg = C;
  while (cg > 1 && stft_smem(L, cg, synth).bytes > budget) --cg;
  *bytes = stft_smem(L, cg, synth).bytes;
  return cg;
}

template <typename K>
int stft_grid(K kern, size_t smem, int64_t work, int threads = kStftThreads) {
  static int dev_max = -1;
  if (dev_max < 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    dev_max = v;
  }
  if ((int)smem > dev_max) return -1;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  return (int)(work < cap ? work : cap);
}

// ---------------------------------------------------------------------------
// Team FFT kernels (frame lengths 2 .. 4096): a transform of H = L/2 complex
// points is owned by a team of T = H/E lanes, each holding E = min(H, 16)
// points in registers. Stockham autosort passes of radix 16 (the last one
// radix 2..16): a lane's radix-R butterflies run in registers, and one
// shared-memory exchange (padded 1-in-16 against bank conflicts) separates
// consecutive passes — 1-3 exchanges per transform instead of log2(H)
// synchronised radix-2 stages. A CTA runs 256/T transforms per round: groups
// of whole frames (all channels, when they fit), so the analysis writes a
// round's output as one contiguous run of the (frame, bin, channel) tensor.
// ---------------------------------------------------------------------------
template <int LOGH>
struct TeamFft {
  static constexpr int H = 1 << LOGH;
  static constexpr int L = 2 * H;
  static constexpr int LOGE = LOGH < 4 ? LOGH : 4;
  static constexpr int E = 1 << LOGE;
  static constexpr int T = H / E;  // lanes per transform
  static constexpr int THREADS = 2 * T > kTeamThreads ? 2 * T : kTeamThreads;
  static constexpr int TEAMS = THREADS / T;
  static constexpr int MINB = 512 / THREADS;
  static constexpr int NPASS = LOGH == 0 ? 1 : (LOGH + LOGE - 1) / LOGE;
  // team buffer stride: padded length rounded to an odd number of 16-B
  // units, so equal offsets in different teams fall in different banks
  static constexpr int PADH = (H + (H >> 4)) | 1;
  static constexpr int rlog(int p) { return p < NPASS - 1 ? LOGE : LOGH - (NPASS - 1) * LOGE; }
  static constexpr int ns(int p) {
    int v = 1;
    for (int i = 0; i < p; ++i) v <<= rlog(i);
    return v;
  }
  static constexpr int tw_off(int p) {  // pass p >= 1 twiddle table offset
    int o = 0;
    for (int i = 1; i < p; ++i) o += ns(i) << rlog(i);
    return o;
  }
  static constexpr int TW = tw_off(NPASS);
  // shared memory (bytes): win[L] f64 | tws[H] c128 | twp[TW] c128 |
  // data[TEAMS][PADH] c128 | analysis: stage[E][THREADS] c128 (next round's
  // samples, lane-private) | synthesis: carry[TEAMS][H] f64
  static constexpr size_t OFF_TWS = (size_t)L * 8;
  static constexpr size_t OFF_TWP = OFF_TWS + (size_t)H * 16;
  static constexpr size_t OFF_DATA = OFF_TWP + (size_t)TW * 16;
  static constexpr size_t OFF_CARRY = OFF_DATA + (size_t)TEAMS * PADH * 16;
  static constexpr size_t STAGE_B = (size_t)E * THREADS * 16;
  static constexpr bool STAGED = OFF_CARRY + STAGE_B <= 200 * 1024;  // else direct loads
  static constexpr size_t SMEM_A = OFF_CARRY + (STAGED ? STAGE_B : 0);
  static constexpr int NBP = (H + 1) | 1;  // staged spectrum row (odd # of 16-B units)
  static constexpr size_t OFF_SSTAGE = OFF_CARRY + (size_t)TEAMS * H * 8;
  static constexpr bool SSTAGED = OFF_SSTAGE + (size_t)TEAMS * NBP * 16 <= 200 * 1024;
  static constexpr size_t SMEM_S = OFF_SSTAGE + (SSTAGED ? (size_t)TEAMS * NBP * 16 : 0);
};

FFCA_DEV int pad16(int i) { return i + (i >> 4); }

// x * e^{-2 pi i k / 16} for a compile-time k in [0, 8)
FFCA_DEV double2 mul_w16(double2 x, int k) {
  constexpr double c1 = 0.92387953251128674, s1 = 0.38268343236508978, h = 0.70710678118654752;
  switch (k) {
    case 0: return x;
    case 1: return make_double2(c1 * x.x + s1 * x.y, c1 * x.y - s1 * x.x);
    case 2: return make_double2(h * (x.x + x.y), h * (x.y - x.x));
    case 3: return make_double2(s1 * x.x + c1 * x.y, s1 * x.y - c1 * x.x);
    case 4: return make_double2(x.y, -x.x);
    case 5: return make_double2(-s1 * x.x + c1 * x.y, -s1 * x.y - c1 * x.x);
    case 6: return make_double2(h * (x.y - x.x), -h * (x.x + x.y));
    default: return make_double2(-c1 * x.x + s1 * x.y, -c1 * x.y - s1 * x.x);
  }
}

constexpr int brev_c(int v, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
  return r;
}

// in-register DFT of R = 2^LR points v[OFF .. OFF+R), natural order in and out
template <int LR, int OFF, int N>
FFCA_DEV void dft_reg(double2 (&v)[N]) {
  constexpr int R = 1 << LR;
  if constexpr (R > 1) {
    double2 a[R];
#pragma unroll
    for (int i = 0; i < R; ++i) a[i] = v[OFF + brev_c(i, LR)];
#pragma unroll
    for (int m = 1; m < R; m <<= 1)
#pragma unroll
      for (int blk = 0; blk < R; blk += 2 * m)
#pragma unroll
        for (int j = 0; j < m; ++j) {
          const double2 b = mul_w16(a[blk + j + m], j * (8 / m));
          const double2 x = a[blk + j];
          a[blk + j] = cadd(x, b);
          a[blk + j + m] = csub(x, b);
        }
#pragma unroll
    for (int i = 0; i < R; ++i) v[OFF + i] = a[i];
  }
}

// Stockham pass P on a lane's registers: v[m*R + r] = in[j_m + r*H/R],
// j_m = t + m*T; outputs to the team buffer (natural order after the last pass)
template <int LOGH, int P, int M = 0>
FFCA_DEV void team_pass_m(double2 (&v)[TeamFft<LOGH>::E], int t, double2* buf,
                          const double2* twp) {
  using F = TeamFft<LOGH>;
  constexpr int LR = F::rlog(P), R = 1 << LR, NS = F::ns(P), MB = F::E / R;
  if constexpr (M < MB) {
    const int j = t + M * F::T;
    const int sidx = j & (NS - 1);
    if constexpr (P > 0) {
#pragma unroll
      for (int r = 1; r < R; ++r)
        v[M * R + r] = cmul(v[M * R + r], twp[F::tw_off(P) + r * NS + sidx]);
    }
    dft_reg<LR, M * R>(v);
    const int base = (j / NS) * NS * R + sidx;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[pad16(base + r * NS)] = v[M * R + r];
    team_pass_m<LOGH, P, M + 1>(v, t, buf, twp);
  }
}

template <int LOGH, int P>
FFCA_DEV void team_load_pass(double2 (&v)[TeamFft<LOGH>::E], int t, const double2* buf) {
  using F = TeamFft<LOGH>;
  constexpr int R = 1 << F::rlog(P), MB = F::E / R;
#pragma unroll
  for (int m = 0; m < MB; ++m)
#pragma unroll
    for (int r = 0; r < R; ++r) v[m * R + r] = buf[pad16(t + m * F::T + r * (F::H / R))];
}

// passes 1 .. NPASS-1 (pass 0 is issued by the caller from its own loads);
// every team of the CTA runs in lockstep, so CTA barriers separate passes
template <int LOGH, int P = 1>
FFCA_DEV void team_rest(double2 (&v)[TeamFft<LOGH>::E], int t, double2* buf, const double2* twp) {
  if constexpr (P < TeamFft<LOGH>::NPASS) {
    __syncthreads();
    team_load_pass<LOGH, P>(v, t, buf);
    __syncthreads();
    team_pass_m<LOGH, P>(v, t, buf, twp);
    team_rest<LOGH, P + 1>(v, t, buf, twp);
  }
}

template <int LOGH>
FFCA_DEV void team_tables(double* win, double2* tws, double2* twp) {
  using F = TeamFft<LOGH>;
  for (int k = threadIdx.x; k < F::H; k += blockDim.x) {
    double sn, cs;
    sincospi(-2.0 * (double)k / (double)F::L, &sn, &cs);
    tws[k] = make_double2(cs, sn);
  }
  for (int i = threadIdx.x; i < F::L; i += blockDim.x)
    win[i] = sqrt(0.5 * (1.0 - cos(2.0 * kPi * (double)i / (double)F::L)));  // stft.py:16-19
#pragma unroll 1
  for (int p = 1; p < F::NPASS; ++p) {
    const int ns = F::ns(p), R = 1 << F::rlog(p);
    for (int i = threadIdx.x; i < ns * R; i += blockDim.x) {
      const int r = i / ns, sidx = i - r * ns;
      double sn, cs;
      sincospi(-2.0 * (double)(sidx * r) / (double)(ns * R), &sn, &cs);
      twp[F::tw_off(p) + i] = make_double2(cs, sn);
    }
  }
}

// rounds: channel groups of ncl = min(C, TEAMS) channels (outer), groups of
// nfr = TEAMS / ncl consecutive frames (inner); team tm -> (frame, channel)
template <int LOGH>
__global__ void __launch_bounds__(TeamFft<LOGH>::THREADS, TeamFft<LOGH>::MINB)
    stft_team_analyze(const double* __restrict__ x, double2* __restrict__ out, int64_t B, int C,
                      int64_t len, int64_t N) {
  using F = TeamFft<LOGH>;
  extern __shared__ __align__(16) unsigned char sm[];
  double* win = (double*)sm;
  double2* tws = (double2*)(sm + F::OFF_TWS);
  double2* twp = (double2*)(sm + F::OFF_TWP);
  double2* data = (double2*)(sm + F::OFF_DATA);
  team_tables<LOGH>(win, tws, twp);
  __syncthreads();
  constexpr int H = F::H, NB = H + 1;
  const int ncl = C < F::TEAMS ? C : F::TEAMS;
  const int nfr = F::TEAMS / ncl;
  const int ngroups = (C + ncl - 1) / ncl;
  const int64_t BN = B * N;
  const int64_t rpg = (BN + nfr - 1) / nfr;  // rounds per channel group
  const int64_t total = rpg * ngroups;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(total, r0 + per);
  const int tm = threadIdx.x / F::T, t = threadIdx.x - tm * F::T;
  const int fr = tm / ncl, cl = tm - fr * ncl;
  double2* buf = data + (size_t)tm * F::PADH;
  double2* stage = (double2*)(sm + F::OFF_CARRY);  // [E][THREADS], lane-private slots
  const bool vec = (len & 1) == 0;  // rows 16-B aligned: pairs never straddle an edge

  // cp.async the samples of round rr for this lane (pairs n = t + r T), zero
  // fill outside [0, len) (the half-frame / tail padding, stft.py:56-59)
  auto issue = [&](int64_t rr) {
    if constexpr (!F::STAGED) return;
    const int g = (int)(rr / rpg);
    const int64_t f0 = (rr - (int64_t)g * rpg) * nfr;
    const int nf = (int)min((int64_t)nfr, BN - f0);
    const int c0 = g * ncl;
    const bool act = fr < nf && cl < min(ncl, C - c0);
    const int64_t fl = f0 + fr;
    const int64_t b = act ? fl / N : 0, k = act ? fl - b * N : 0;
    const double* xc = x + ((size_t)b * C + (act ? c0 + cl : 0)) * len;
    const int64_t base = (k - 1) * H;
#pragma unroll
    for (int r = 0; r < F::E; ++r) {
      const int64_t i0 = base + 2 * (t + r * F::T);
      double2* dst = stage + r * F::THREADS + threadIdx.x;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
      if (vec) {
        const bool ok = act && i0 >= 0 && i0 < len;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                     "l"(ok ? xc + i0 : x), "r"(ok ? 16 : 0));
      } else {
        const bool ok0 = act && i0 >= 0 && i0 < len;
        const bool ok1 = act && i0 + 1 >= 0 && i0 + 1 < len;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa),
                     "l"(ok0 ? xc + i0 : x), "r"(ok0 ? 8 : 0));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa + 8),
                     "l"(ok1 ? xc + i0 + 1 : x), "r"(ok1 ? 8 : 0));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  if (r0 < r1) issue(r0);
  for (int64_t rr = r0; rr < r1; ++rr) {
    const int g = (int)(rr / rpg);
    const int64_t f0 = (rr - (int64_t)g * rpg) * nfr;
    const int nf = (int)min((int64_t)nfr, BN - f0);
    const int c0 = g * ncl;
    const int nc = min(ncl, C - c0);
    double2 v[F::E];
    if constexpr (F::STAGED) {
      asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
      for (int r = 0; r < F::E; ++r) {
        const int n = t + r * F::T;
        const double2 a = stage[r * F::THREADS + threadIdx.x];
        v[r] = make_double2(a.x * win[2 * n], a.y * win[2 * n + 1]);
      }
    } else {
      const bool act = fr < nf && cl < nc;
      const int64_t fl = f0 + fr;
      const int64_t b = act ? fl / N : 0, k = act ? fl - b * N : 0;
      const double* xc = x + ((size_t)b * C + (act ? c0 + cl : 0)) * len;
      const int64_t base = (k - 1) * H;
      const bool inner = act && base >= 0 && base + F::L <= len;
#pragma unroll
      for (int r = 0; r < F::E; ++r) {
        const int n = t + r * F::T;
        const int64_t i0 = base + 2 * n;
        double a0 = 0.0, a1 = 0.0;
        if (inner) {
          a0 = xc[i0];
          a1 = xc[i0 + 1];
        } else if (act) {
          if (i0 >= 0 && i0 < len) a0 = xc[i0];
          if (i0 + 1 >= 0 && i0 + 1 < len) a1 = xc[i0 + 1];
        }
        v[r] = make_double2(a0 * win[2 * n], a1 * win[2 * n + 1]);
      }
    }
    if (rr + 1 < r1) issue(rr + 1);  // overlaps this round's passes and stores
    team_pass_m<LOGH, 0>(v, t, buf, twp);
    team_rest<LOGH>(v, t, buf, twp);
    __syncthreads();
    // split + store: X_f = E_f + e^{-2 pi i f / L} O_f, contiguous (frame, bin, channel)
    double2* o = out + (size_t)f0 * NB * C + c0;
    const int cnt = nf * NB * nc;
    // (q, f, c) walk of the round's output with carries instead of divisions
    int q = 0, f = 0, c = threadIdx.x;
    {
      const int per = NB * nc;
      q = c / per;
      c -= q * per;
      f = c / nc;
      c -= f * nc;
    }
    const int sq = F::THREADS / (NB * nc);
    int sr = F::THREADS - sq * NB * nc;
    const int sf = sr / nc, sc = sr - (sr / nc) * nc;
    for (int i = threadIdx.x; i < cnt; i += F::THREADS) {
      const double2* z = data + (size_t)(q * ncl + c) * F::PADH;
      const double2 zk = z[pad16(f & (H - 1))];
      const double2 zm = cconj(z[pad16((H - f) & (H - 1))]);
      const double2 e = cscale(cadd(zk, zm), 0.5);
      const double2 d = cscale(csub(zk, zm), 0.5);
      const double2 od = make_double2(d.y, -d.x);
      const double2 w = f < H ? tws[f] : make_double2(-1.0, 0.0);
      o[((size_t)q * NB + f) * C + c] = cadd(e, cmul(w, od));
      c += sc;
      f += sf;
      q += sq;
      if (c >= nc) {
        c -= nc;
        ++f;
      }
      if (f >= NB) {
        f -= NB;
        ++q;
      }
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_all;\n" ::);
}

// windowed time sample s of the frame held (as FFT(conj Z)) in team buffer z
FFCA_DEV double synth_sample(const double2* z, int s, double invH, const double* win) {
  const double2 y = z[pad16(s >> 1)];
  return ((s & 1) ? -y.y : y.x) * invH * win[s];
}

// rounds: channel group (outer), mixture b, hop group [q0, q0 + nh) with
// nh <= nfr; a round transforms frames q0+1 .. q0+nh and takes frame q0's
// second half from `carry` (the previous round of this CTA, or a one-frame
// prologue at the start of a run). The spectra of the next round's frames are
// cp.async-copied (coalesced, one 16-B bin per copy) into a transposed
// [team][bin] stage while the current round computes.
template <int LOGH>
__global__ void __launch_bounds__(TeamFft<LOGH>::THREADS, TeamFft<LOGH>::MINB)
    stft_team_synth(const double2* __restrict__ spec, double* __restrict__ out, int64_t B, int C,
                    int64_t N, int64_t len) {
  using F = TeamFft<LOGH>;
  extern __shared__ __align__(16) unsigned char sm[];
  double* win = (double*)sm;
  double2* tws = (double2*)(sm + F::OFF_TWS);
  double2* twp = (double2*)(sm + F::OFF_TWP);
  double2* data = (double2*)(sm + F::OFF_DATA);
  double* carry = (double*)(sm + F::OFF_CARRY);
  double2* stage = (double2*)(sm + F::OFF_SSTAGE);
  team_tables<LOGH>(win, tws, twp);
  __syncthreads();
  constexpr int H = F::H, NB = H + 1;
  const double invH = 1.0 / (double)H;
  const int ncl = C < F::TEAMS ? C : F::TEAMS;
  const int nfr = F::TEAMS / ncl;
  const int ngroups = (C + ncl - 1) / ncl;
  const int64_t Q = (len + H - 1) / H;
  const int64_t rq = (Q + nfr - 1) / nfr;  // rounds per (group, mixture)
  const int64_t total = rq * B * ngroups;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(total, r0 + per);
  const int tm = threadIdx.x / F::T, t = threadIdx.x - tm * F::T;
  const int fr = tm / ncl, cl = tm - fr * ncl;
  double2* buf = data + (size_t)tm * F::PADH;
  int64_t ckey = -1;  // carry holds frame (key % N) second half of (group, b) = key / N

  struct Round {
    int64_t b, q0;
    int g, c0, nc, nh, nnext;
  };
  auto round_of = [&](int64_t rr) {
    Round R;
    const int64_t gb = rr / rq;
    R.g = (int)(gb / B);
    R.b = gb - (int64_t)R.g * B;
    R.q0 = (rr - gb * rq) * nfr;
    R.nh = (int)min((int64_t)nfr, Q - R.q0);
    R.c0 = R.g * ncl;
    R.nc = min(ncl, C - R.c0);
    R.nnext = (int)min((int64_t)R.nh, N - 1 - R.q0);  // frames q0+1 .. q0+nnext exist
    return R;
  };
  // stage the spectra of frames q0+1 .. q0+nnext (channels c0 .. c0+nc)
  auto issue = [&](const Round& R) {
    if constexpr (F::SSTAGED) {
      const int per_f = NB * R.nc;
      const int cnt = R.nnext * per_f;
      const double2* src = spec + ((size_t)R.b * N + R.q0 + 1) * NB * C + R.c0;
      // (q, f, c) walk with carries: source reads stay contiguous per frame
      int q = threadIdx.x / per_f;
      int rem = threadIdx.x - q * per_f;
      int f = rem / R.nc, c = rem - f * R.nc;
      const int sq = F::THREADS / per_f;
      const int sr = F::THREADS - sq * per_f;
      const int sf = sr / R.nc, sc = sr - sf * R.nc;
      for (int i = threadIdx.x; i < cnt; i += F::THREADS) {
        const unsigned sa =
            (unsigned)__cvta_generic_to_shared(stage + (size_t)(q * ncl + c) * F::NBP + f);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa),
                     "l"(src + ((size_t)q * NB + f) * C + c));
        c += sc;
        f += sf;
        q += sq;
        if (c >= R.nc) {
          c -= R.nc;
          ++f;
        }
        if (f >= NB) {
          f -= NB;
          ++q;
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  // conj(Z_n) from X_n, X_{H-n} (DC / Nyquist real-valued, stft.py:91-92);
  // the inverse FFT is the forward FFT of conj(Z)
  auto zconj = [&](double2 xa, double2 xb, int n) {
    if (n == 0) {
      xa.y = 0.0;
      xb.y = 0.0;
    }
    const double2 xm = cconj(xb);
    const double2 e = cscale(cadd(xa, xm), 0.5);
    const double2 d = cscale(csub(xa, xm), 0.5);
    const double2 od = cmul(d, cconj(tws[n]));
    return make_double2(e.x - od.y, -(e.y + od.x));
  };

  // prologue transform of frame k straight from HBM (team fr == 0 only)
  auto transform_direct = [&](int64_t b, int64_t k, int c0, bool act) {
    double2 v[F::E];
    const double2* sp = spec + ((size_t)b * N + k) * NB * C + c0 + cl;
#pragma unroll
    for (int r = 0; r < F::E; ++r) {
      const int n = t + r * F::T;
      v[r] = act ? zconj(sp[(size_t)n * C], sp[(size_t)(H - n) * C], n) : make_double2(0.0, 0.0);
    }
    team_pass_m<LOGH, 0>(v, t, buf, twp);
    team_rest<LOGH>(v, t, buf, twp);
    __syncthreads();
  };

  if (r0 < r1) {
    const Round R = round_of(r0);
    issue(R);
  }
  for (int64_t rr = r0; rr < r1; ++rr) {
    const Round R = round_of(rr);
    const int64_t key = (rr / rq) * N + R.q0;
    if (ckey != key) {  // prologue: frame q0 -> carry
      transform_direct(R.b, R.q0, R.c0, fr == 0 && cl < R.nc);
      for (int i = threadIdx.x; i < R.nc * H; i += F::THREADS) {
        const int c = i / H, sx = i - c * H;
        carry[(size_t)c * H + sx] = synth_sample(data + (size_t)c * F::PADH, H + sx, invH, win);
      }
      __syncthreads();
    }
    // frames q0+1 .. q0+nnext
    {
      const bool act = fr < R.nnext && cl < R.nc;
      double2 v[F::E];
      if constexpr (F::SSTAGED) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();  // every lane's copies landed
        const double2* st = stage + (size_t)tm * F::NBP;
#pragma unroll
        for (int r = 0; r < F::E; ++r) {
          const int n = t + r * F::T;
          v[r] = act ? zconj(st[n], st[H - n], n) : make_double2(0.0, 0.0);
        }
      } else {
        const double2* sp = spec + ((size_t)R.b * N + R.q0 + 1 + fr) * NB * C + R.c0 + cl;
#pragma unroll
        for (int r = 0; r < F::E; ++r) {
          const int n = t + r * F::T;
          v[r] = act ? zconj(sp[(size_t)n * C], sp[(size_t)(H - n) * C], n)
                     : make_double2(0.0, 0.0);
        }
      }
      team_pass_m<LOGH, 0>(v, t, buf, twp);
      __syncthreads();  // stage fully consumed: prefetch the next round
      if (rr + 1 < r1) issue(round_of(rr + 1));
      team_rest<LOGH>(v, t, buf, twp);
      __syncthreads();
    }
    // hop q0 + h: frame (q0+h) second half + frame (q0+h+1) first half
    // (stft.py:95-99 order). Each thread emits a pair of samples (one 16-B
    // shared load per frame); walk (c, h, pair) with carries, no divisions.
    {
      constexpr int HP = H / 2 > 0 ? H / 2 : 1;  // sample pairs per hop (H = 1: one single)
      const int nhP = R.nh * HP;
      const int cnt = R.nc * nhP;
      int c = threadIdx.x / nhP;
      int rem = threadIdx.x - c * nhP;
      int h = rem / HP, px = rem - h * HP;
      const int sc = F::THREADS / nhP;
      const int srem = F::THREADS - sc * nhP;
      const int sh = srem / HP, sp = srem - sh * HP;
      const bool vec2 = (H >= 2) && ((len & 1) == 0);
      for (int i = threadIdx.x; i < cnt; i += F::THREADS) {
        const int sx = 2 * px;
        const int64_t tt = (R.q0 + h) * H + sx;
        double* dst = out + ((size_t)R.b * C + R.c0 + c) * len + tt;
        if (H == 1) {
          if (tt < len) {
            const double a = h == 0 ? carry[c]
                                    : synth_sample(data + (size_t)((h - 1) * ncl + c) * F::PADH,
                                                   1, invH, win);
            *dst = h < R.nnext
                       ? a + synth_sample(data + (size_t)(h * ncl + c) * F::PADH, 0, invH, win)
                       : a;
          }
        } else if (tt < len) {
          double a0, a1;
          if (h == 0) {
            a0 = carry[(size_t)c * H + sx];
            a1 = carry[(size_t)c * H + sx + 1];
          } else {  // second half of frame q0+h: pair index (H + sx) / 2
            const double2 y = data[(size_t)((h - 1) * ncl + c) * F::PADH + pad16((H + sx) >> 1)];
            a0 = y.x * invH * win[H + sx];
            a1 = -y.y * invH * win[H + sx + 1];
          }
          if (h < R.nnext) {
            const double2 y = data[(size_t)(h * ncl + c) * F::PADH + pad16(sx >> 1)];
            a0 = a0 + y.x * invH * win[sx];
            a1 = a1 + -y.y * invH * win[sx + 1];
          }
          if (vec2 && tt + 1 < len) {
            *(double2*)dst = make_double2(a0, a1);
          } else {
            dst[0] = a0;
            if (tt + 1 < len) dst[1] = a1;
          }
        }
        px += sp;
        h += sh;
        c += sc;
        if (px >= HP) {
          px -= HP;
          ++h;
        }
        if (h >= R.nh) {
          h -= R.nh;
          ++c;
        }
      }
    }
    __syncthreads();
    if (R.nnext == R.nh) {  // frame q0 + nh exists: its second half seeds the next round
      for (int i = threadIdx.x; i < R.nc * H; i += F::THREADS) {
        const int c = i >> LOGH, sx = i & (H - 1);
        carry[(size_t)c * H + sx] =
            synth_sample(data + (size_t)((R.nh - 1) * ncl + c) * F::PADH, H + sx, invH, win);
      }
      ckey = key + R.nh;
    } else {
      ckey = -1;
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_all;\n" ::);
}

template <int LOGH>
cudaError_t launch_team(const double* x, double2* spec, const double2* spec_in, double* out,
                        int64_t B, int C, int64_t len, int64_t N, bool synth, cudaStream_t s) {
  using F = TeamFft<LOGH>;
  const size_t smem = synth ? F::SMEM_S : F::SMEM_A;
  const int ncl = C < F::TEAMS ? C : F::TEAMS;
  const int nfr = F::TEAMS / ncl;
  const int ngroups = (C + ncl - 1) / ncl;
  if (synth) {
    const int64_t Q = (len + F::H - 1) / F::H;
    const int64_t work = ((Q + nfr - 1) / nfr) * B * ngroups;
    const int grid = stft_grid(stft_team_synth<LOGH>, smem, work, F::THREADS);
    if (grid < 1) return cudaErrorInvalidValue;
    stft_team_synth<LOGH><<<grid, F::THREADS, smem, s>>>(spec_in, out, B, C, N, len);
  } else {
    const int64_t work = ((B * N + nfr - 1) / nfr) * ngroups;
    const int grid = stft_grid(stft_team_analyze<LOGH>, smem, work, F::THREADS);
    if (grid < 1) return cudaErrorInvalidValue;
    stft_team_analyze<LOGH><<<grid, F::THREADS, smem, s>>>(x, spec, B, C, len, N);
  }
  return cudaGetLastError();
}

cudaError_t dispatch_team(int logH, const double* x, double2* spec, const double2* spec_in,
                          double* out, int64_t B, int C, int64_t len, int64_t N, bool synth,
                          cudaStream_t s) {
  switch (logH) {
#define FFCA_TEAM(K) \
  case K:            \
    return launch_team<K>(x, spec, spec_in, out, B, C, len, N, synth, s);
    FFCA_TEAM(0) FFCA_TEAM(1) FFCA_TEAM(2) FFCA_TEAM(3) FFCA_TEAM(4) FFCA_TEAM(5)
    FFCA_TEAM(6) FFCA_TEAM(7) FFCA_TEAM(8) FFCA_TEAM(9) FFCA_TEAM(10) FFCA_TEAM(11)
#undef FFCA_TEAM
    default: return cudaErrorInvalidValue;
  }
}
constexpr int kTeamMaxLogH = 11;

}  // namespace

int64_t stft_frames(int64_t length, int frame_shift) {
  const int64_t n = (length - 1) / frame_shift + 2;  // stft.py:30-32
  return n > 2 ? n : 2;
}

cudaError_t launch_stft_analyze(const double* x, double2* spec, int64_t B, int C, int64_t len,
                                int L, cudaStream_t s) {
  const int logL = log2_exact(L);
  if (logL < 0 || B < 1 || C < 1 || len < 1) return cudaErrorInvalidValue;
  const int64_t N = stft_frames(len, L / 2);
  if (logL - 1 <= kTeamMaxLogH)
    return dispatch_team(logL - 1, x, spec, nullptr, nullptr, B, C, len, N, false, s);
  size_t smem = 0;
  const int cg = stft_group(L, C, false, &smem);
  const int grid = stft_grid(stft_analyze_kernel, smem, B * N);
  if (grid < 1) return cudaErrorInvalidValue;
  stft_analyze_kernel<<<grid, kStftThreads, smem, s>>>(x, spec, B, C, len, L, logL - 1, N, cg);
  return cudaGetLastError();
}

cudaError_t launch_stft_synthesize(const double2* spec, double* out, int64_t B, int C, int64_t N,
                                   int L, int64_t len, cudaStream_t s) {
  const int logL = log2_exact(L);
  if (logL < 0 || B < 1 || C < 1 || N < 1 || len < 1 || len > N * (L / 2))
    return cudaErrorInvalidValue;
  if (logL - 1 <= kTeamMaxLogH)
    return dispatch_team(logL - 1, nullptr, nullptr, spec, out, B, C, len, N, true, s);
  size_t smem = 0;
  const int cg = stft_group(L, C, true, &smem);
  const int64_t Q = (len + L / 2 - 1) / (L / 2);
  const int grid = stft_grid(stft_synth_kernel, smem, B * Q);
  if (grid < 1) return cudaErrorInvalidValue;
  stft_synth_kernel<<<grid, kStftThreads, smem, s>>>(spec, out, B, C, N, L, logL - 1, len, cg);
  return cudaGetLastError();
}

}  // namespace ffca

using namespace ffca;

extern "C" {

int64_t ffca_stft_frames(int64_t length, int frame_shift) {
  if (length < 1 || frame_shift < 1) return -1;
  return stft_frames(length, frame_shift);
}

int ffca_stft_analyze(const double* x, double* spec, int64_t batch, int channels, int64_t length,
                      int frame_length, void* stream) {
  if (!x || !spec) return FFCA_ERR_INVALID;
  const cudaError_t e = launch_stft_analyze(x, (double2*)spec, batch, channels, length,
                                            frame_length, (cudaStream_t)stream);
  return e == cudaSuccess ? FFCA_OK : (e == cudaErrorInvalidValue ? FFCA_ERR_INVALID : FFCA_ERR_CUDA);
}

int ffca_stft_synthesize(const double* spec, double* out, int64_t batch, int channels,
                         int64_t frames, int frame_length, int64_t length, void* stream) {
  if (!spec || !out) return FFCA_ERR_INVALID;
  const cudaError_t e = launch_stft_synthesize((const double2*)spec, out, batch, channels, frames,
                                               frame_length, length, (cudaStream_t)stream);
  return e == cudaSuccess ? FFCA_OK : (e == cudaErrorInvalidValue ? FFCA_ERR_INVALID : FFCA_ERR_CUDA);
}

}  // extern "C"
