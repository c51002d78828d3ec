// K3t — the complex128 FastFCA update pass with a CTA-wide TMA frame ring.
//
// Same per-point arithmetic as the update-only fast_em2_kernel (reference
// _kernels_numba.py:328-391), different data movement:
//  * a CTA owns a 128-bin tile (warp w: bins 32w .. 32w+31, lane = bin) and
//    EVERY warp streams every frame of the CTA's frame chunk, so one frame of
//    the tile — its y row (128 x I x 16 contiguous bytes) and its v1 / v2
//    runs — is fetched by ONE elected thread (lane 0 of warp n mod 4) with
//    cp.async.bulk into a ring
//    stage (3 bulk copies per 128 bin-frames; 6 when the tile crosses into the
//    next mixture), completing on the stage's "full" mbarrier (expect-tx);
//  * consumers wait on "full", read their bin, and each warp arrives on the
//    stage's "empty" mbarrier; the producing thread waits on "empty" before
//    refilling the stage (S-stage full/empty pipeline, no per-lane copies, no
//    LDGSTS, no __syncthreads in the loop);
//  * no cross-warp reduction at the end: each warp owns distinct bins and
//    writes its per-(chunk, bin) partial sums directly.
// A v frame row is only 8-B aligned when F is odd, so v runs are copied as
// their 16-B aligned supersets; y rows land linearly (bin b at b * 16 I) and
// lanes read their I units in the rotated order (k + sw(lane)) mod I, with the
// P tile's rows stored in the same rotation (conflict-free reads, as the
// RingSlot swizzle on the write side of the cp.async ring).
// Per-bin summation order: frames of a chunk in sequence (the cp.async ring
// kernel interleaves 4 warps and adds them in fixed order) — deterministic
// and bitwise independent of sharding for a fixed chunking.
#pragma once

#include "ffca_fast2.cuh"

namespace ffca {

template <int I>
struct TmaLayout {
  static constexpr int TB = 128;  // bins per CTA tile
  static constexpr int WARPS = TB / 32;
  static constexpr int YB = I * 16, VB = 8, NP = I * I;
  static constexpr int VA = ((TB * VB + 64) + 15) / 16 * 16;  // a v run + alignment slack, 2 segments
  static constexpr int STAGE = TB * YB + 2 * VA;
  static constexpr size_t PT = (size_t)NP * TB * 16;  // P tile (rotated rows)
};

#ifndef FFCA_K3T_STAGES
#define FFCA_K3T_STAGES 4
#endif
template <int I>
constexpr size_t tma_smem_bytes() {
  using Lay = TmaLayout<I>;
  return (size_t)FFCA_K3T_STAGES * Lay::STAGE + Lay::PT + 2 * FFCA_K3T_STAGES * 8;
}

template <int I, int STAGES>
__global__ void __launch_bounds__(TmaLayout<I>::TB, 3) fast_tma_kernel(const FastIterParams p) {
  pdl_release_dependents();
  using Lay = TmaLayout<I>;
  using Slot = RingSlot<I, double>;
  constexpr int TB = Lay::TB, NP = Lay::NP, YB = Lay::YB, VB = Lay::VB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* ring = smem_raw;
  double2* sP = (double2*)(smem_raw + (size_t)STAGES * Lay::STAGE);
  const unsigned full0 = smem_u32(smem_raw + (size_t)STAGES * Lay::STAGE + Lay::PT);
  const unsigned empty0 = full0 + STAGES * 8;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = threadIdx.x;  // bin within the tile
  const int64_t G = p.G, F = p.F, N = p.N, NF = N * F;
  const int64_t tile0 = p.g0 + (int64_t)blockIdx.x * TB;
  int64_t g = tile0 + b;
  const bool active = g < G;
  if (!active) g = G - 1;
  const int64_t m = g / F, f = g - m * F;
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(N, n0 + p.chunk_frames);
  const int K = (int)(n1 - n0);
  double* vw = (double*)p.v + m * 2 * NF + f + n0 * F;  // v written in place (frame n0)

  // ---- P tile (coalesced copy; row r of bin b stored at its rotated slot) ----
  const int rot = Slot::sw(lane);
  for (int u = threadIdx.x; u < TB * NP; u += TB) {
    const int bb = u / NP, e = u - bb * NP;
    int64_t gb = tile0 + bb;
    if (gb >= G) gb = G - 1;
    const int row = e / I;
    const int es = ((row - Slot::sw(bb & 31) + Slot::Q) % Slot::Q) * I + (e - row * I);
    sP[es * TB + bb] = p.P[gb * NP + e];
  }
  double lam[I], il[I];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    lam[a] = p.lam[g * I + a];
    il[a] = 1.0 / ((double)I * lam[a]);
  }
  const double fl = p.floor[g];

  // ---- tile geometry: valid bins, split into (at most) two mixtures ----
  const int nval = (int)min((int64_t)TB, G - tile0);
  const int64_t m0 = tile0 / F, f0 = tile0 - m0 * F;
  const int s1 = (int)min((int64_t)nval, F - f0);  // bins in the first mixture
  const unsigned char* vbase = (const unsigned char*)(p.v_src ? p.v_src : p.v);
  // byte offsets (frame 0) of the segments: y, v1 (v2 = v1 + NF VB)
  const int64_t yo[2] = {((m0 * N) * F + f0) * YB, (((m0 + 1) * N) * F) * YB};
  const int64_t vo[2] = {(m0 * 2 * NF + f0) * VB, ((m0 + 1) * 2 * NF) * VB};
  const int cnt[2] = {s1, nval - s1};
  const int d2 = (16 + s1 * VB + 15) / 16 * 16;  // v-area offset of segment 2
  // this lane's v offset within a v area at frame n: seg base + (addr & 15) + position
  const int seg = b < s1 ? 0 : 1;
  const int pos = (seg == 0 ? b : b - s1) * VB + (seg == 0 ? 0 : d2);
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(full0 + st * 8, 1);
      mbar_init(empty0 + st * 8, Lay::WARPS);
    }
    mbar_init_fence();
  }
  __syncthreads();  // P tile + barriers

  auto issue = [&](int j) {  // producer thread: frame n0 + j into stage j % STAGES
    const int st = j % STAGES;
    if (j >= STAGES) mbar_wait(empty0 + st * 8, (unsigned)((j / STAGES - 1) & 1));
    const int64_t n = n0 + j;
    unsigned char* dst = ring + (size_t)st * Lay::STAGE;
    const unsigned bar = full0 + st * 8;
    const unsigned char* src[3][2];
    unsigned len[3][2], off[3][2];
    unsigned bytes = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      src[0][q] = (const unsigned char*)p.y + yo[q] + n * F * YB;
      len[0][q] = (unsigned)(cnt[q] * YB);
      off[0][q] = q == 0 ? 0u : (unsigned)(s1 * YB);
#pragma unroll
      for (int jv = 0; jv < 2; ++jv) {
        const uintptr_t a = (uintptr_t)(vbase + vo[q] + (int64_t)jv * NF * VB + n * F * VB);
        const uintptr_t lo = a & ~(uintptr_t)15;
        const uintptr_t hi = (a + (uintptr_t)cnt[q] * VB + 15) & ~(uintptr_t)15;
        src[1 + jv][q] = (const unsigned char*)lo;
        len[1 + jv][q] = cnt[q] > 0 ? (unsigned)(hi - lo) : 0u;
        off[1 + jv][q] = (unsigned)(TB * YB + jv * Lay::VA + (q == 0 ? 0 : d2));
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) bytes += len[c][0] + len[c][1];
    fence_proxy_async_smem();
    mbar_expect_tx(bar, bytes);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (len[c][q]) bulk_g2s(smem_u32(dst + off[c][q]), src[c][q], len[c][q], bar);
  };
  // producers: lane 0 of warp (j mod WARPS) issues frame j — round-robin, so
  // the issue work (and its waits on "empty") is spread over the warps
  // instead of slowing one warp that the others then wait for
  if (lane == 0)
    for (int j = warp; j < STAGES - 1 && j < K; j += Lay::WARPS) issue(j);

  double acc[2][NP];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[j][e] = 0.0;
  bool any_bad = false;
  constexpr double invI = 1.0 / I;

#pragma unroll 1
  for (int k = 0; k < K; ++k) {
    if (lane == 0 && k + STAGES - 1 < K && (k + STAGES - 1) % Lay::WARPS == warp)
      issue(k + STAGES - 1);
    const int st = k % STAGES;
    mbar_wait(full0 + st * 8, (unsigned)((k / STAGES) & 1));
    const unsigned char* slot = ring + (size_t)st * Lay::STAGE;
    const int64_t n = n0 + k;
    double2 yv[I];
    const unsigned char* row = slot + b * YB;
#pragma unroll
    for (int u = 0; u < I; ++u) yv[u] = *(const double2*)(row + 16 * ((u + rot) % Slot::Q));
    // v supersets: the run of this lane's segment starts (addr & 15) bytes in
    const uintptr_t a1 = (uintptr_t)(vbase + vo[seg] + n * F * VB);
    const int sub1 = (int)(a1 & 15);
    const int sub2 = (int)((a1 + (uintptr_t)NF * VB) & 15);
    const double v1 = *(const double*)(slot + TB * YB + pos + sub1);
    const double v2 = *(const double*)(slot + TB * YB + Lay::VA + pos + sub2);
    __syncwarp();
    if (lane == 0) {  // this warp is done with the stage
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(empty0 + st * 8) : "memory");
    }
    // z = P^H y (rows in the lane's rotated order)
    double2 z[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 p0 = sP[(0 * I + a) * TB + b];
      double zr = p0.x * yv[0].x + p0.y * yv[0].y;
      double zi = p0.x * yv[0].y - p0.y * yv[0].x;
#pragma unroll
      for (int c = 1; c < I; ++c) {
        const double2 pc = sP[(c * I + a) * TB + b];
        zr = fma(pc.x, yv[c].x, fma(pc.y, yv[c].y, zr));
        zi = fma(pc.x, yv[c].y, fma(-pc.y, yv[c].x, zi));
      }
      z[a] = cmk(zr, zi);
    }
    double g1[I], g2[I], t1[I], t2[I], v1l[I], den[I], rden[I];
    double tr1 = 0.0, tr2 = 0.0;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      v1l[a] = v1 * lam[a];
      den[a] = v1l[a] + v2;
    }
    rcp_batch<I>(den, rden);
#pragma unroll
    for (int a = 0; a < I; ++a) {
      g1[a] = v1l[a] * rden[a];
      g2[a] = v2 * rden[a];
      const double pz = fma(z[a].x, z[a].x, z[a].y * z[a].y);
      t1[a] = g1[a] * fma(g1[a], pz, v2);
      t2[a] = g2[a] * fma(g2[a], pz, v1l[a]);
      tr1 = fma(t1[a], il[a], tr1);
      tr2 = fma(t2[a], invI, tr2);
    }
    const double w1 = (tr1 < fl) ? fl : tr1;  // NaN propagates like np.maximum
    const double w2 = (tr2 < fl) ? fl : tr2;
    if (active) {
      vw[0] = w1;
      vw[NF] = w2;
    }
    vw += F;
    {
      const long long q1 = __double_as_longlong(w1), q2 = __double_as_longlong(w2);
      any_bad |= (((q1 >> 52) & 0x7ff) == 0x7ff) | (((q2 >> 52) & 0x7ff) == 0x7ff) | (q1 <= 0) |
                 (q2 <= 0);
    }
    double wv[2] = {w1, w2}, iw[2];
    rcp_batch<2>(wv, iw);
    double h1[I], h2[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      acc[0][a] = fma(t1[a], iw[0], acc[0][a]);
      acc[1][a] = fma(t2[a], iw[1], acc[1][a]);
      h1[a] = g1[a] * iw[0];
      h2[a] = g2[a] * iw[1];
    }
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int c = a + 1; c < I; ++c) {
        const double zr = fma(z[a].x, z[c].x, z[a].y * z[c].y);  // z_a conj(z_c)
        const double zi = fma(z[a].y, z[c].x, -z[a].x * z[c].y);
        const double k1 = h1[a] * g1[c], k2 = h2[a] * g2[c];
        acc[0][Herm<I>::re(a, c)] = fma(k1, zr, acc[0][Herm<I>::re(a, c)]);
        acc[0][Herm<I>::im(a, c)] = fma(k1, zi, acc[0][Herm<I>::im(a, c)]);
        acc[1][Herm<I>::re(a, c)] = fma(k2, zr, acc[1][Herm<I>::re(a, c)]);
        acc[1][Herm<I>::im(a, c)] = fma(k2, zi, acc[1][Herm<I>::im(a, c)]);
      }
  }
  if (any_bad && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX,
                 (unsigned long long)((m * N + n0) * F + f));
  if (!active) return;
  double* sp = p.Spart + (size_t)blockIdx.y * 2 * NP * G + g;
#pragma unroll
  for (int e = 0; e < NP; ++e) {
    sp[(size_t)e * G] = acc[0][e];
    sp[(size_t)(NP + e) * G] = acc[1][e];
  }
}

template <int I>
cudaError_t launch_fast_tma(const FastIterParams& p, cudaStream_t s) {
  constexpr size_t SM = tma_smem_bytes<I>();
  if (cudaError_t e = ensure_smem<fast_tma_kernel<I, FFCA_K3T_STAGES>>(SM)) return e;
  dim3 grid((unsigned)((window_end(p.g1, p.G) - p.g0 + TmaLayout<I>::TB - 1) / TmaLayout<I>::TB),
            (unsigned)p.nchunk);
  if (cudaError_t e = launch_ex(fast_tma_kernel<I, FFCA_K3T_STAGES>, grid, dim3(TmaLayout<I>::TB),
                                SM, s, p.pdl != 0, 0, p))
    return e;
  return cudaGetLastError();
}

template <int I>
int fast_tma_blocks_per_sm() {
  constexpr size_t SM = tma_smem_bytes<I>();
  auto kern = fast_tma_kernel<I, FFCA_K3T_STAGES>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, TmaLayout<I>::TB, SM);
  return n > 0 ? n : 1;
}

}  // namespace ffca
