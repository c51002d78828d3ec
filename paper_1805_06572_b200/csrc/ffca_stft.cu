// STFT front and back end on the device (reference stft.py:9-107):
// square-root periodic Hann window, 50% overlap, half a frame of leading zero
// padding, rfft / irfft per frame and overlap-add.
//
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
int stft_grid(K kern, size_t smem, int64_t work) {
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
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStftThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  return (int)(work < cap ? work : cap);
}

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
