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
#include "ffca_fast2.cuh"  // FrameRing (warp-cooperative frame staging)

namespace ffca {

// orders up to which the pass uses rsqrt/rcp seeds + Newton instead of the
// IEEE sqrt / division subroutines (with the fused complex MACs this is
// faster at every order: config 3 FCA 15.8 -> 18.4 G at I = 4)
#ifndef FFCA_FCA_FASTMATH_MAXI
#define FFCA_FCA_FASTMATH_MAXI 4
#endif
#ifndef FFCA_FCA_STAGES
#define FFCA_FCA_STAGES 4  // frame ring depth of the FCA pass
#endif
#ifndef FFCA_K4_RING_FIRST
#define FFCA_K4_RING_FIRST 0  // 1: issue the frame ring before loading S1, S2
#endif
#ifndef FFCA_K4_SWEEP
#define FFCA_K4_SWEEP 1  // frame-wise inverse by the Hermitian sweep (0: Cholesky chain)
#endif
#ifndef FFCA_K4_XX_RECOMPUTE
#define FFCA_K4_XX_RECOMPUTE 1  // form the x x^H entries twice instead of holding I^2 registers (config 3 FCA 22.2 -> 22.7 G)
#endif
#ifndef FFCA_K4_LAUNDER
#define FFCA_K4_LAUNDER 0  // 1: plain shared loads through per-phase laundered addresses
#endif
#ifndef FFCA_K4_STAGED_MU
#define FFCA_K4_STAGED_MU 0  // 1: image rows stored through the consumed ring stage
#endif
#ifndef FFCA_K4_TR
#define FFCA_K4_TR 2  // interleaved partial sums per power-update trace (1, 2 or 4; config 3 pass 3.49 / 3.42 / 3.46 ms)
#endif
#ifndef FFCA_FCA_MINB3_MAXI
#define FFCA_FCA_MINB3_MAXI 0  // orders up to which the pass is budgeted for 3 CTAs / SM (I <= 3 fits 168
                               // registers, but config 1 FCA measured 16.6 vs 18.6 G: off)
#endif
#ifndef FFCA_FCA_WARPS
#define FFCA_FCA_WARPS 4  // warps per CTA of the I <= 4 FCA pass
#endif
constexpr int kFcaWarps = FFCA_FCA_WARPS;
#ifndef FFCA_FCA_MINB
#define FFCA_FCA_MINB 1  // CTAs per SM the I <= 4 pass is register-budgeted for
#endif

// UPDATE / LL / MU (power + covariance update, likelihood, posterior-mean
// write) are compile-time variants, so the hot update-only pass carries
// neither the image nor the likelihood code (register pressure: the fused
// runtime-branch kernel spilled ~550 B per thread at I = 4).
// shared-memory load the compiler may not merge with an earlier load of the
// same address
__device__ __forceinline__ double lds_reload(unsigned addr) {
  double v;
#if FFCA_K4_LAUNDER
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));  // (address laundered per phase)
#else
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
#endif
  return v;
}
// an address the compiler must treat as new: loads through it are neither
// hoisted out of the frame loop nor merged with another phase's loads, but
// stay freely schedulable within their phase
__device__ __forceinline__ unsigned launder(unsigned a) {
#if FFCA_K4_LAUNDER
  asm volatile("" : "+r"(a));
#endif
  return a;
}

// CTAs per SM the pass is register-budgeted for (FFCA_FCA_MINB3_MAXI: orders
// budgeted for 3 CTAs / SM instead; at I = 4 the four packed accumulators need
// all 255 registers)
template <int I>
constexpr int fca_minb() {
  return I <= FFCA_FCA_MINB3_MAXI ? 3 : FFCA_FCA_MINB;
}

template <int I, typename R, int WARPS, bool UPDATE, bool LL, bool MU>
__global__ void __launch_bounds__(WARPS * 32, (fca_minb<I>())) fca_em_kernel(const FcaIterParams p) {
  using C = typename CplxOf<R>::type;
  constexpr int NP = I * I;
  constexpr int NE = kFcaParts * NP + 1;
  constexpr bool kFastMath = I <= FFCA_FCA_FASTMATH_MAXI;
  using Ring = FrameRing<I, R, WARPS, FFCA_FCA_STAGES>;
  extern __shared__ __align__(16) double smem[];
  // frame ring, then S1, S2 ([2][NP][32] packed; the traces need no S^-1); the
  // cross-warp reduction buffer [(WARPS-1)][NE][32] reuses it after the loop
  double* sS = (double*)((unsigned char*)smem + Ring::BYTES);
  double* red = smem;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t G = p.G;
  int64_t g = (int64_t)blockIdx.x * 32 + lane;
  const bool active = g < G;
  if (!active) g = G - 1;
  const int64_t m = (unsigned)g / (unsigned)p.F;  // (32-bit division)
  const int64_t f = g - m * p.F;
  auto load_tile = [&]() {  // S1, S2 of the tile (packed, bin-minor)
    for (int e = warp; e < 2 * NP; e += WARPS) sS[e * 32 + lane] = p.Sp[(size_t)e * G + g];
    __syncthreads();
  };
  const bool ring_first = FFCA_K4_RING_FIRST || p.pdl_wait;
  if (!ring_first) load_tile();
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  R* vb = (R*)p.v + m * 2 * NF + f;  // no __restrict__: may alias vr (in place)
  const R* vr = (p.v_src ? (const R*)p.v_src : (const R*)p.v) + m * 2 * NF + f;
  const double fl = p.floor[g];
  const double invI = 1.0 / I;
  const int64_t nfirst = n0 + warp;
  Ring ring;
  ring.init((unsigned char*)smem, warp, lane, (int64_t)blockIdx.x * 32, G, p.N, p.F, p.y, vr,
            nfirst);
  const int K = nfirst < n1 ? (int)((n1 - nfirst + WARPS - 1) / WARPS) : 0;
#pragma unroll
  for (int s = 0; s < FFCA_FCA_STAGES - 1; ++s) {
    if (s < K) ring.issue();
    cp_async_commit();
  }
  if (ring_first) {  // (S1, S2 after the ring prologue)
    if (p.pdl_wait) {  // chained schedule: the finish that wrote S1, S2 may still run
      pdl_wait_primary();
      pdl_release_dependents();
    }
    load_tile();
  }

  const unsigned sS_addr = (unsigned)__cvta_generic_to_shared(sS + lane);
  auto Sget = [&](int which, int a, int b) -> double2 {
    // full entry (a, b) of packed Hermitian matrix `which`
    const double* base = sS + which * NP * 32 + lane;
    if (a == b) return cmk(base[a * 32], 0.0);
    if (a < b) return cmk(base[Herm<I>::re(a, b) * 32], base[Herm<I>::im(a, b) * 32]);
    return cmk(base[Herm<I>::re(b, a) * 32], -base[Herm<I>::im(b, a) * 32]);
  };

#if FFCA_K4_STAGED_MU
  ImageRowStore<I, R> img;
  if constexpr (MU) img.init((int64_t)blockIdx.x * 32, G, p.N, p.F, lane);
#endif
  double acc[kFcaParts][NP];  // packed Hermitian B1, B2, X1, X2 (see the update block)
#pragma unroll
  for (int j = 0; j < kFcaParts; ++j)
#pragma unroll
    for (int e = 0; e < NP; ++e) acc[j][e] = 0.0;
  double llacc = 0.0;
  constexpr bool do_ll = LL;
  int64_t bad_n = 0;

  for (int k = 0; k < K; ++k) {
    const int64_t n = nfirst + (int64_t)k * WARPS;
    __syncwarp();  // every lane is done with the stage the next copy overwrites
    if (k + FFCA_FCA_STAGES - 1 < K) ring.issue();
    cp_async_commit();
    cp_async_wait<FFCA_FCA_STAGES - 1>();
    __syncwarp();  // the other lanes' copies of this stage are visible
    double2 yv[I];
    double v1, v2;
#if FFCA_K4_SWEEP
    ring.load_v(v1, v2);
#else
    ring.load(yv, v1, v2);
#endif
#if FFCA_K4_SWEEP
    // R = v1 S1 + v2 S2 (packed Hermitian) inverted in place by the
    // symmetric sweep (herm_sweep_inverse): Ri = R^-1, the pivots' product is
    // det R, and R is singular / indefinite iff a pivot is <= 0
    double Ri[NP];
    double detR;
    {
      // (volatile loads: S1, S2 are loop invariant, and plain loads get hoisted
      // out of the frame loop into 2 I^2 registers' worth of spills)
      const unsigned aR = launder(sS_addr);
#pragma unroll
      for (int e = 0; e < NP; ++e)
        Ri[e] = fma(v1, lds_reload(aR + (unsigned)(e * 32) * 8u),
                    v2 * lds_reload(aR + (unsigned)((NP + e) * 32) * 8u));
      const bool ok = herm_sweep_inverse<I>(Ri, detR);
      if (!ok && bad_n == 0) bad_n = n + 1;
    }
    asm volatile("" ::: "memory");  // y is loaded after the inversion (register budget)
    ring.load_y(yv);
#else
    // R = v1 S1 + v2 S2 and its Cholesky factor
    double2 Lm[I][I];
    [[maybe_unused]] double ild[I];
    {
      double2 Rm[I][I];
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) {
          const double2 s1 = Sget(0, a, b), s2 = Sget(1, a, b);
          Rm[a][b] = cmk(v1 * s1.x + v2 * s2.x, v1 * s1.y + v2 * s2.y);
        }
      const bool ok = kFastMath ? cholesky_fast<I>(Rm, Lm, ild) : cholesky<I>(Rm, Lm);
      if (!ok && bad_n == 0) bad_n = n + 1;
    }
    double2 Li[I][I];
    if constexpr (kFastMath)
      tril_inverse_d<I>(Lm, ild, Li);
    else
      tril_inverse<I>(Lm, Li);
    // Rinv = Li^H Li (frame-wise inverse), packed Hermitian: real diagonal +
    // strictly-upper entries; x = Rinv y
    double Ri[NP];
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = a; b < I; ++b) {
        double2 s = cmk(0.0, 0.0);
#pragma unroll
        for (int k = b; k < I; ++k) s = cmac_cj(s, Li[k][a], Li[k][b]);
        if (a == b) {
          Ri[a] = s.x;
        } else {
          Ri[Herm<I>::re(a, b)] = s.x;
          Ri[Herm<I>::im(a, b)] = s.y;
        }
      }
#endif
    double2 x[I];
#pragma unroll
    for (int a = 0; a < I; ++a) {
      double2 s = cmk(Ri[a] * yv[a].x, Ri[a] * yv[a].y);
#pragma unroll
      for (int b = 0; b < I; ++b) {
        if (b == a) continue;
        const double2 r = a < b ? cmk(Ri[Herm<I>::re(a, b)], Ri[Herm<I>::im(a, b)])
                                : cmk(Ri[Herm<I>::re(b, a)], -Ri[Herm<I>::im(b, a)]);
        s = cmac(s, r, yv[b]);
      }
      x[a] = s;
    }
    if constexpr (LL) {
      // log det R + y^H R^{-1} y = 2 sum log L_ii + Re(y^H x)
      double quad = 0.0;
#pragma unroll
      for (int a = 0; a < I; ++a) quad += yv[a].x * x[a].x + yv[a].y * x[a].y;
#if FFCA_K4_SWEEP
      llacc += log(detR) + quad;
#else
      double prod = 1.0;
#pragma unroll
      for (int a = 0; a < I; ++a) prod *= Lm[a][a].x;
      llacc += 2.0 * log(prod) + quad;
#endif
    }
    if constexpr (MU) {
      // mu_j = v_j S_j x (the posterior means; written by the image pass
      // only). Direct lane-strided stores: at 255 registers the staged
      // warp-cooperative store (ImageRowStore, as K3) spilled its addressing
      // and made this pass slower (config 3: 7.0 -> 9.2 ms).
#if FFCA_K4_STAGED_MU
      {  // warp-cooperative row stores through the consumed ring stage (as K3)
        double2 o[2][I];
#pragma unroll
        for (int a = 0; a < I; ++a) {
          double2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
#pragma unroll
          for (int b = 0; b < I; ++b) {
            s1 = cmac(s1, Sget(0, a, b), x[b]);
            s2 = cmac(s2, Sget(1, a, b), x[b]);
          }
          o[0][a] = cscale(s1, v1);
          o[1][a] = cscale(s2, v2);
        }
        img.store(p.mu_out, ring.cur, n, o);
      }
#else
      if (active) {
        C* mo = (C*)p.mu_out;
        C* d1 = mo + (((m * 2 + 0) * p.N + n) * p.F + f) * I;
        C* d2 = mo + (((m * 2 + 1) * p.N + n) * p.F + f) * I;
#pragma unroll
        for (int a = 0; a < I; ++a) {
          double2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
#pragma unroll
          for (int b = 0; b < I; ++b) {
            s1 = cmac(s1, Sget(0, a, b), x[b]);
            s2 = cmac(s2, Sget(1, a, b), x[b]);
          }
          d1[a] = from_c128<R>(cscale(s1, v1));
          d2[a] = from_c128<R>(cscale(s2, v2));
        }
      }
#endif
    }
    if constexpr (!UPDATE) continue;
    // Phi_j = mu_j mu_j^H + v1 v2 S1 Rinv S2 with mu_j = v_j S_j x, so
    //   sum_n Phi_j / w_j = S_j (sum v_j^2/w_j x x^H) S_j + S1 (sum v1 v2/w_j Rinv) S2:
    // the per-point I x I products of the reference (_kernels_numba.py:290-314)
    // move to the per-bin finish (fca_finish_kernel), the points accumulate
    // B_j += v_j^2/w_j x x^H and X_j += v1 v2/w_j Rinv. The power-update
    // traces tr(S_j^-1 Phi_j) need no S_j^-1 either (tr(AB) of Hermitian
    // A, B = sum_a A_aa B_aa + 2 sum_{a<b} Re(A_ab conj(B_ab))):
    //   mu_j^H S_j^-1 mu_j = v_j^2 x^H S_j x = v_j^2 tr(S_j x x^H)
    //   tr(S_1^-1 v1 v2 S1 Rinv S2) = v1 v2 tr(Rinv S2), tr(S_2^-1 ...) = v1 v2 tr(Rinv S1)
    // every term is non-negative (no cancellation).
    // x x^H, packed (|x_a|^2, x_a conj(x_b)); with FFCA_K4_XX_RECOMPUTE the
    // entries are formed from x where they are used (twice: traces and sums)
    // instead of held in I^2 registers across the power update
    auto xx_entry = [&](int e) -> double {
      if (e < I) return cabs2(x[e]);
      int a = 0, b = 1;
#pragma unroll
      for (int aa = 0; aa < I; ++aa)
#pragma unroll
        for (int bb = aa + 1; bb < I; ++bb)
          if (Herm<I>::re(aa, bb) == e || Herm<I>::im(aa, bb) == e) {
            a = aa;
            b = bb;
          }
      return e == Herm<I>::re(a, b) ? fma(x[a].x, x[b].x, x[a].y * x[b].y)
                                    : fma(x[a].y, x[b].x, -x[a].x * x[b].y);
    };
#if FFCA_K4_XX_RECOMPUTE
#define FFCA_XX(e) xx_entry(e)
#else
    double xx[NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) xx[e] = xx_entry(e);
#define FFCA_XX(e) xx[e]
#endif
    // S1, S2 re-read from shared memory (volatile, as for R)
    // (kTr interleaved partial sums per trace: shorter dependent FMA chains)
    const unsigned aT = launder(sS_addr);
    constexpr int kTr = FFCA_K4_TR;
    double qf1p[kTr], qf2p[kTr], tR1p[kTr], tR2p[kTr];
#pragma unroll
    for (int t = 0; t < kTr; ++t) qf1p[t] = qf2p[t] = tR1p[t] = tR2p[t] = 0.0;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      const double s1 = lds_reload(aT + (unsigned)(e * 32) * 8u);
      const double s2 = lds_reload(aT + (unsigned)((NP + e) * 32) * 8u);
      const double wgt = e < I ? 1.0 : 2.0;  // compile-time after unrolling
      const double xe = FFCA_XX(e);
      qf1p[e % kTr] = fma(wgt * s1, xe, qf1p[e % kTr]);
      qf2p[e % kTr] = fma(wgt * s2, xe, qf2p[e % kTr]);
      tR1p[e % kTr] = fma(wgt * s1, Ri[e], tR1p[e % kTr]);
      tR2p[e % kTr] = fma(wgt * s2, Ri[e], tR2p[e % kTr]);
    }
    auto fold = [](const double (&t)[kTr]) {
      if constexpr (kTr == 4) return (t[0] + t[1]) + (t[2] + t[3]);
      else if constexpr (kTr == 2) return t[0] + t[1];
      else return t[0];
    };
    const double qf1 = fold(qf1p), qf2 = fold(qf2p), tR1 = fold(tR1p), tR2 = fold(tR2p);
    const double vv = v1 * v2;
    const double q1 = (v1 * v1 * qf1 + vv * tR2) * invI;
    const double q2 = (v2 * v2 * qf2 + vv * tR1) * invI;
    const double w1 = (q1 < fl) ? fl : q1;
    const double w2 = (q2 < fl) ? fl : q2;
    if (active) {
      vb[n * p.F] = (R)w1;
      vb[NF + n * p.F] = (R)w2;
    }
#if FFCA_K4_XX_RECOMPUTE
#pragma unroll
    for (int a = 0; a < I; ++a)  // opaque: the x x^H entries below are formed again
      asm volatile("" : "+d"(x[a].x), "+d"(x[a].y));
#endif
    const double iw1 = kFastMath ? rcp_fast(w1) : 1.0 / w1;
    const double iw2 = kFastMath ? rcp_fast(w2) : 1.0 / w2;
    const double cb1 = v1 * v1 * iw1, cb2 = v2 * v2 * iw2;
    const double cx1 = vv * iw1, cx2 = vv * iw2;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      const double xe = FFCA_XX(e);
      acc[0][e] = fma(cb1, xe, acc[0][e]);
      acc[1][e] = fma(cb2, xe, acc[1][e]);
      acc[2][e] = fma(cx1, Ri[e], acc[2][e]);
      acc[3][e] = fma(cx2, Ri[e], acc[3][e]);
    }
  }
  if (bad_n && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MIXTURE,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));

  cp_async_wait_all();
  if constexpr (!UPDATE && !LL) return;
  if (WARPS > 1) {
    __syncthreads();  // ring and sS are dead: the reduction buffer reuses them
    if (warp > 0) {
      double* r = red + (size_t)(warp - 1) * NE * 32;
#pragma unroll
      for (int j = 0; j < kFcaParts; ++j)
#pragma unroll
        for (int e = 0; e < NP; ++e) r[(j * NP + e) * 32 + lane] = acc[j][e];
      r[kFcaParts * NP * 32 + lane] = llacc;
    }
    __syncthreads();
    if (warp != 0) return;
#pragma unroll 1
    for (int w = 1; w < WARPS; ++w) {
      const double* r = red + (size_t)(w - 1) * NE * 32;
#pragma unroll
      for (int j = 0; j < kFcaParts; ++j)
#pragma unroll
        for (int e = 0; e < NP; ++e) acc[j][e] += r[(j * NP + e) * 32 + lane];
      llacc += r[kFcaParts * NP * 32 + lane];
    }
  }
  if (!active) return;
  const int64_t c = blockIdx.y;
  if constexpr (UPDATE) {
    double* sp = p.Spart + (size_t)c * kFcaParts * NP * G + g;
#pragma unroll
    for (int j = 0; j < kFcaParts; ++j)
#pragma unroll
      for (int e = 0; e < NP; ++e) sp[(size_t)(j * NP + e) * G] = acc[j][e];
  }
  if constexpr (LL) p.llbin[(size_t)c * G + g] = llacc;
}

template <int I, typename R>
constexpr size_t fca_smem_bytes() {
  constexpr size_t NP = (size_t)I * I;
  constexpr size_t ss = FrameRing<I, R, kFcaWarps, FFCA_FCA_STAGES>::BYTES + 2 * NP * 32 * sizeof(double);
  constexpr size_t red = (size_t)(kFcaWarps - 1) * (kFcaParts * NP + 1) * 32 * sizeof(double);
  return ss > red ? ss : red;
}

template <int I, typename R, bool UPDATE, bool LL, bool MU>
static cudaError_t launch_fca_em_v(const FcaIterParams& p, cudaStream_t s) {
  const size_t smem = fca_smem_bytes<I, R>();
  auto kern = fca_em_kernel<I, R, kFcaWarps, UPDATE, LL, MU>;
  if (cudaError_t e = ensure_smem<fca_em_kernel<I, R, kFcaWarps, UPDATE, LL, MU>>(smem)) return e;
  dim3 grid((unsigned)((p.G + 31) / 32), (unsigned)p.nchunk);
  return launch_ex(kern, grid, dim3(kFcaWarps * 32), smem, s, p.pdl_wait != 0, 0, p);
}

template <int I, typename R>
static cudaError_t launch_fca_em_t(const FcaIterParams& p, cudaStream_t s) {
  const bool ll = p.llbin != nullptr, mu = p.mu_out != nullptr;
  if (p.update) {
    if (!ll && !mu) return launch_fca_em_v<I, R, true, false, false>(p, s);
    if (ll && !mu) return launch_fca_em_v<I, R, true, true, false>(p, s);
    if (!ll && mu) return launch_fca_em_v<I, R, true, false, true>(p, s);
    return launch_fca_em_v<I, R, true, true, true>(p, s);
  }
  if (ll && !mu) return launch_fca_em_v<I, R, false, true, false>(p, s);
  if (!ll && mu) return launch_fca_em_v<I, R, false, false, true>(p, s);
  if (ll && mu) return launch_fca_em_v<I, R, false, true, true>(p, s);
  return cudaSuccess;
}

template <int I, typename R>
static int fca_bpsm_t() {
  const size_t smem = fca_smem_bytes<I, R>();
  auto kern = fca_em_kernel<I, R, kFcaWarps, true, false, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kFcaWarps * 32, smem);
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

// ---- per-bin prepare / finish: lane-parallel (fca_bin_par_kernel, ffca_fca_par.cu)
cudaError_t launch_fca_prepare(const double2* S, double* Sp, int64_t G, int64_t F, int I,
                               ffca_status_dev* st, int iter, cudaStream_t s) {
  return launch_fca_bin_par(nullptr, 0, 1, G, F, Sp, nullptr, nullptr, nullptr, nullptr, nullptr,
                            S, I, st, iter, s);
}

cudaError_t launch_fca_finish(const double* Spart, int nchunk, int64_t N, int64_t G, int64_t F,
                              double* Sp, double2* S_model, double2* S_hist,
                              const double* llbin, double* llg, int I, ffca_status_dev* st,
                              int iter, cudaStream_t s, int pdl) {
  return launch_fca_bin_par(Spart, nchunk, N, G, F, Sp, S_model, S_hist, llbin, llg, nullptr,
                            nullptr, I, st, iter, s, pdl);
}

cudaError_t launch_fca_sraw(const double* Spart, int nchunk, int64_t N, int64_t G,
                            const double* Sp, double2* S_raw, int I, cudaStream_t s) {
  return launch_fca_bin_par(Spart, nchunk, N, G, G, const_cast<double*>(Sp), nullptr, nullptr,
                            nullptr, nullptr, S_raw, nullptr, I, nullptr, 0, s);
}

}  // namespace ffca
