// K3 v2 — fused FastFCA pass for small orders (I <= 4), register-resident
// per-bin state, cp.async frame ring.
//
// Same arithmetic as fast_em_kernel (ffca_fast.cu; reference
// _kernels_numba.py:328-391), reorganised for the B200 memory system:
//  * each thread streams its bin's frames through a private STAGES-deep
//    cp.async ring in shared memory, so ~STAGES-1 frames per thread are in
//    flight without holding registers (the v1 kernel kept <= 1 frame in flight
//    and was latency bound at 12% warps active);
//  * ring slots are an odd number of 16-B units wide, so the per-lane 16-B
//    shared loads are bank-conflict free;
//  * reciprocals use rcp.approx.f64 + two Newton steps (<= 1 ulp) instead of
//    IEEE division sequences, and the rank-1 covariance updates share one
//    z_a conj(z_b) product between both sources;
//  * likelihood / mean-writing variants are compile-time, so the hot
//    update-only pass carries no dead code.
#pragma once

#include "ffca_internal.cuh"

namespace ffca {

FFCA_DEV double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  return r;
}

FFCA_DEV void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
FFCA_DEV void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
FFCA_DEV void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
FFCA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
FFCA_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
FFCA_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

template <int I, typename R>
struct RingSlot {
  using C = typename CplxOf<R>::type;
  static constexpr int YB = I * (int)sizeof(C);
  static constexpr int VB = (int)sizeof(R);
  static constexpr int RAW = YB + 2 * VB;
  static constexpr int U16 = (RAW + 15) / 16;
  static constexpr int BYTES = 16 * ((U16 % 2) ? U16 : U16 + 1);  // odd # of 16-B units
};

template <int I, typename R, int WARPS, int STAGES, bool MU = false>
struct Fast2Smem {
  static constexpr int NE = 2 * I * I + 1;
  static constexpr size_t RING = (size_t)STAGES * WARPS * 32 * RingSlot<I, R>::BYTES;
  static constexpr size_t RED = (size_t)(WARPS - 1) * NE * 32 * sizeof(double);
  static constexpr size_t PB = (size_t)I * I * 32 * sizeof(double2);  // P tile, after RING
  static constexpr size_t WB = MU ? PB : 0;                           // W tile, after P
  static constexpr size_t BYTES = (RING + PB + WB) > RED ? (RING + PB + WB) : RED;
};

template <int I, typename R, int WARPS, int STAGES, bool UPDATE, bool LL, bool MU>
__global__ void __launch_bounds__(WARPS * 32, MU ? 2 : 3) fast_em2_kernel(const FastIterParams p) {
  using C = typename CplxOf<R>::type;
  using Slot = RingSlot<I, R>;
  constexpr int NP = I * I;
  constexpr int NE = 2 * NP + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
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
  const int64_t FI = p.F * I;
  const C* __restrict__ yb = (const C*)p.y + (m * p.N * p.F + f) * I;
  R* __restrict__ vb = (R*)p.v + m * 2 * NF + f;

  // P lives in shared memory (bin-minor SoA after the frame ring): the 4
  // warps of the CTA work on the same 32 bins, so one 16*I*I-byte column per
  // lane serves all of them and frees the registers for the accumulators.
  double2* sP = (double2*)(smem_raw + Fast2Smem<I, R, WARPS, STAGES, MU>::RING);
  for (int e = warp; e < NP; e += WARPS) sP[e * 32 + lane] = p.P[g * NP + e];
  // W = P^{-H} for the image write (last pass only), same bin-minor tile layout
  double2* sW = sP + NP * 32;
  if (MU && p.mu_back)
    for (int e = warp; e < NP; e += WARPS) sW[e * 32 + lane] = p.W[g * NP + e];
  __syncthreads();
  double lam[I], il[I];
#pragma unroll
  for (int a = 0; a < I; ++a) {
    lam[a] = p.lam[g * I + a];
    il[a] = 1.0 / lam[a];
  }
  const double fl = p.floor[g];
  constexpr double invI = 1.0 / I;

  double acc[2][NP];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[j][e] = 0.0;
  double llacc = 0.0;
  int64_t bad_n = 0;

  unsigned char* myslots = smem_raw + ((size_t)warp * 32 + lane) * Slot::BYTES;
  constexpr size_t kStageStride = (size_t)WARPS * 32 * Slot::BYTES;
  const int64_t nfirst = n0 + warp;
  const int K = nfirst < n1 ? (int)((n1 - nfirst + WARPS - 1) / WARPS) : 0;

  auto issue = [&](int k) {
    const int64_t n = nfirst + (int64_t)k * WARPS;
    unsigned char* slot = myslots + (size_t)(k % STAGES) * kStageStride;
    const unsigned char* ysrc = (const unsigned char*)(yb + n * FI);
    if constexpr (Slot::YB % 16 == 0) {
#pragma unroll
      for (int c = 0; c < Slot::YB / 16; ++c) cp_async16(slot + 16 * c, ysrc + 16 * c);
    } else {
#pragma unroll
      for (int c = 0; c < Slot::YB / 8; ++c) cp_async8(slot + 8 * c, ysrc + 8 * c);
    }
    if constexpr (sizeof(R) == 8) {
      cp_async8(slot + Slot::YB, vb + n * p.F);
      cp_async8(slot + Slot::YB + 8, vb + NF + n * p.F);
    } else {
      cp_async4(slot + Slot::YB, vb + n * p.F);
      cp_async4(slot + Slot::YB + 4, vb + NF + n * p.F);
    }
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < K) issue(s);
    cp_async_commit();
  }

#pragma unroll 1
  for (int k = 0; k < K; ++k) {
    if (k + STAGES - 1 < K) issue(k + STAGES - 1);
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    const int64_t n = nfirst + (int64_t)k * WARPS;
    const unsigned char* slot = myslots + (size_t)(k % STAGES) * kStageStride;
    double2 yv[I];
#pragma unroll
    for (int a = 0; a < I; ++a) yv[a] = to_c128(((const C*)slot)[a]);
    const double v1 = (double)*(const R*)(slot + Slot::YB);
    const double v2 = (double)*(const R*)(slot + Slot::YB + sizeof(R));

    double2 z[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double2 p0 = sP[(0 * I + a) * 32 + lane];
      double zr = p0.x * yv[0].x + p0.y * yv[0].y;
      double zi = p0.x * yv[0].y - p0.y * yv[0].x;
#pragma unroll
      for (int b = 1; b < I; ++b) {
        const double2 pb = sP[(b * I + a) * 32 + lane];
        zr = fma(pb.x, yv[b].x, fma(pb.y, yv[b].y, zr));
        zi = fma(pb.x, yv[b].y, fma(-pb.y, yv[b].x, zi));
      }
      z[a] = cmk(zr, zi);
    }
    double g1[I], g2[I], t1[I], t2[I];
    double tr1 = 0.0, tr2 = 0.0, lprod = 1.0, quad = 0.0;
    bool bad = false;
#pragma unroll
    for (int a = 0; a < I; ++a) {
      const double v1l = v1 * lam[a];
      const double den = v1l + v2;
      const double rden = rcp_nr(den);
      g1[a] = v1l * rden;
      g2[a] = v2 * rden;
      const double c = v2 * g1[a];
      const double pz = fma(z[a].x, z[a].x, z[a].y * z[a].y);
      t1[a] = fma(g1[a] * g1[a], pz, c);
      t2[a] = fma(g2[a] * g2[a], pz, c);
      tr1 = fma(t1[a], il[a], tr1);
      tr2 += t2[a];
      if (LL) {
        lprod *= den;
        quad = fma(pz, rden, quad);
      }
      // den == 0 needs no test: rcp_nr(0) is NaN and poisons w below
    }
    if (LL) llacc += log(lprod) + quad;
    if (UPDATE) {
      const double q1 = tr1 * invI, q2 = tr2 * invI;
      const double w1 = (q1 < fl) ? fl : q1;  // NaN propagates like np.maximum
      const double w2 = (q2 < fl) ? fl : q2;
      if (active) {
        vb[n * p.F] = (R)w1;
        vb[NF + n * p.F] = (R)w2;
      }
      {  // non-finite or non-positive w (integer tests keep the FP64 pipe free)
        const long long b1 = __double_as_longlong(w1), b2 = __double_as_longlong(w2);
        bad |= (((b1 >> 52) & 0x7ff) == 0x7ff) | (((b2 >> 52) & 0x7ff) == 0x7ff) | (b1 <= 0) |
               (b2 <= 0);
      }
      const double iw1 = rcp_nr(w1), iw2 = rcp_nr(w2);
      double h1[I], h2[I];
#pragma unroll
      for (int a = 0; a < I; ++a) {
        acc[0][a] = fma(t1[a], iw1, acc[0][a]);
        acc[1][a] = fma(t2[a], iw2, acc[1][a]);
        h1[a] = g1[a] * iw1;
        h2[a] = g2[a] * iw2;
      }
#pragma unroll
      for (int a = 0; a < I; ++a) {
#pragma unroll
        for (int b = a + 1; b < I; ++b) {
          // z_a conj(z_b), shared by both sources
          const double zr = fma(z[a].x, z[b].x, z[a].y * z[b].y);
          const double zi = fma(z[a].y, z[b].x, -z[a].x * z[b].y);
          const double k1 = h1[a] * g1[b];
          const double k2 = h2[a] * g2[b];
          acc[0][Herm<I>::re(a, b)] = fma(k1, zr, acc[0][Herm<I>::re(a, b)]);
          acc[0][Herm<I>::im(a, b)] = fma(k1, zi, acc[0][Herm<I>::im(a, b)]);
          acc[1][Herm<I>::re(a, b)] = fma(k2, zr, acc[1][Herm<I>::re(a, b)]);
          acc[1][Herm<I>::im(a, b)] = fma(k2, zi, acc[1][Herm<I>::im(a, b)]);
        }
      }
    }
    if (MU && active) {
      C* mo = (C*)p.mu_out;
      C* d1 = mo + (((m * 2 + 0) * p.N + n) * p.F + f) * I;
      C* d2 = mo + (((m * 2 + 1) * p.N + n) * p.F + f) * I;
      if (p.mu_back) {
        // images (fast.py:133-141): mu_1 = P^{-H} (g1 z); mu_2 = y - mu_1, the
        // posterior partition mu_1 + mu_2 = y (g1 + g2 = 1, P^{-H} P^H = I),
        // exact up to rounding (reference test_fast.py:247-252)
#pragma unroll
        for (int a = 0; a < I; ++a) {
          double sx = 0.0, sy = 0.0;
#pragma unroll
          for (int b = 0; b < I; ++b) {
            const double2 w = sW[(a * I + b) * 32 + lane];
            const double mx = g1[b] * z[b].x, my = g1[b] * z[b].y;
            sx = fma(w.x, mx, fma(-w.y, my, sx));
            sy = fma(w.x, my, fma(w.y, mx, sy));
          }
          d1[a] = from_c128<R>(cmk(sx, sy));
          d2[a] = from_c128<R>(cmk(yv[a].x - sx, yv[a].y - sy));
        }
      } else {
#pragma unroll
        for (int a = 0; a < I; ++a) {
          d1[a] = from_c128<R>(cscale(z[a], g1[a]));
          d2[a] = from_c128<R>(cscale(z[a], g2[a]));
        }
      }
    }
    if (bad && bad_n == 0) bad_n = n + 1;
  }
  cp_async_wait_all();
  if (bad_n && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));

  if (!UPDATE && !LL) return;
  // --- cross-warp reduction (fixed order), reusing the ring memory ---
  __syncthreads();
  double* red = (double*)smem_raw;
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
  if (UPDATE) {
    double* sp = p.Spart + (size_t)c * 2 * NP * G + g;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      sp[(size_t)e * G] = acc[0][e];
      sp[(size_t)(NP + e) * G] = acc[1][e];
    }
  }
  if (LL) p.llbin[(size_t)c * G + g] = llacc;
}

template <int I, typename R, bool UPDATE, bool LL, bool MU>
cudaError_t launch_fast2_variant(const FastIterParams& p, cudaStream_t s) {
  constexpr int WARPS = kWarps;
  constexpr int STAGES = 6;
  using Sm = Fast2Smem<I, R, WARPS, STAGES, MU>;
  auto kern = fast_em2_kernel<I, R, WARPS, STAGES, UPDATE, LL, MU>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Sm::BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid((unsigned)((p.G + 31) / 32), (unsigned)p.nchunk);
  kern<<<grid, WARPS * 32, Sm::BYTES, s>>>(p);
  return cudaGetLastError();
}

template <int I, typename R>
cudaError_t launch_fast2(const FastIterParams& p, cudaStream_t s) {
  const bool ll = p.llbin != nullptr;
  const bool mu = p.mu_out != nullptr;
  if (p.update) {
    if (!ll && !mu) return launch_fast2_variant<I, R, true, false, false>(p, s);
    if (ll && !mu) return launch_fast2_variant<I, R, true, true, false>(p, s);
    if (!ll && mu) return launch_fast2_variant<I, R, true, false, true>(p, s);
    return launch_fast2_variant<I, R, true, true, true>(p, s);
  }
  if (ll && !mu) return launch_fast2_variant<I, R, false, true, false>(p, s);
  if (!ll && mu) return launch_fast2_variant<I, R, false, false, true>(p, s);
  if (ll && mu) return launch_fast2_variant<I, R, false, true, true>(p, s);
  return cudaSuccess;
}

}  // namespace ffca
