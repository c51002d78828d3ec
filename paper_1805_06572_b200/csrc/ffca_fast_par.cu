// K3p — fused FastFCA pass for large orders (5 <= I <= 8), lane-parallel.
//
// At I = 8 one thread per bin would need P (64 complex) and 2 x 36 packed
// accumulators in registers, so the v1 kernel (ffca_fast.cu) spills. Here a
// group of 8 lanes owns one bin and streams its frames; lane r owns channel
// r: column r of P (z_r = sum_b conj(P[b][r]) y_b), the scalar posterior of
// channel r (den, g1, g2, t1, t2), the diagonal entry r and a circulant share
// of the off-diagonal entries of both transformed covariance accumulators
// ((r, r + s mod I), s = 1..I/2: <= 4 per lane at I = 8 instead of a
// triangular row of up to 7). The power update needs sums over channels (group shuffles);
// the rank-1 updates need every z_c, g1_c, g2_c (exchanged through a few
// bytes of shared memory per bin). Same arithmetic as fast_em2_kernel
// (reference _kernels_numba.py:328-391), same Spart / llbin / mu layouts.
#include "ffca_fast2.cuh"
#include "ffca_pencil_par.cuh"

#ifdef FFCA_DEBUG_BOUNDS
#include <cassert>
#define FFCA_CHECK(cond) assert(cond)
#else
#define FFCA_CHECK(cond) ((void)0)
#endif

namespace ffca {

namespace {
template <int I, bool PAIR = false>
struct FastParLayout {
  static constexpr int LB = 8;
  static constexpr int WARPS = 2;
  static constexpr int BPB = WARPS * 32 / LB;  // bins per CTA
  // per group: y (2I), z (2I), (g1, g2) (2I) doubles (x2 frames when PAIR);
  // odd # of 16-B units
  static constexpr int RAW = 6 * I * (PAIR ? 2 : 1);
  static constexpr int U16 = (RAW + 1) / 2;
  static constexpr int GROUP_DOUBLES = 2 * ((U16 % 2) ? U16 : U16 + 1);
  static constexpr size_t RINGB = (size_t)8 * WARPS * 32 * 48;  // 8 stages x 64 lanes x 48 B
  static constexpr size_t SMEM = (size_t)BPB * GROUP_DOUBLES * sizeof(double) + RINGB;
};
}  // namespace

#ifndef FAST_PAR_MINB
#define FAST_PAR_MINB 8  // CTAs per SM the lane-parallel pass is register-budgeted for
#endif
#ifndef FAST_PAR_PAIR_MINB
#define FAST_PAR_PAIR_MINB 6  // ... and its two-frames-per-trip update pass
#endif
#ifndef FFCA_K3P_PAIR
#define FFCA_K3P_PAIR 1  // update pass: two frames per loop trip (ILP across the frame chains)
#endif
template <int I, typename R, bool UPDATE, bool LL, bool MU, bool PAIR = false>
__global__ void __launch_bounds__(FastParLayout<I>::WARPS * 32, PAIR ? FAST_PAR_PAIR_MINB : FAST_PAR_MINB) fast_par_kernel(const FastIterParams p) {
  pdl_release_dependents();
  static_assert(!PAIR || (UPDATE && !LL && !MU), "the paired loop is the update-only pass");
  using Lay = FastParLayout<I, PAIR>;
  using C = typename CplxOf<R>::type;
  constexpr int NP = I * I;
  constexpr int LB = Lay::LB;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane % LB;
  const int grp = warp * (32 / LB) + lane / LB;
  const int64_t G = p.G;
  int64_t g = p.g0 + (int64_t)blockIdx.x * Lay::BPB + grp;
  const bool active = g < G;
  if (!active) g = G - 1;
  const bool own = r < I;
  const int rr = own ? r : 0;  // clamped channel for idle lanes
  const int64_t m = (unsigned)g / (unsigned)p.F, f = g - m * p.F;  // (32-bit division)
  double* base = sm + (size_t)grp * Lay::GROUP_DOUBLES;
  double2* sy = (double2*)base;      // y
  double2* sz = sy + I;              // z
  double2* sgg = sz + I;             // (g1, g2): one 16-B read per exchanged channel

  double2 pc[I];  // column rr of P
  double2 wr[I];  // row rr of W = P^-H (images only)
#pragma unroll
  for (int b = 0; b < I; ++b) {
    pc[b] = p.P[g * NP + b * I + rr];
    wr[b] = MU && p.mu_back ? p.W[g * NP + rr * I + b] : cmk(0.0, 0.0);
  }
  const double lam = p.lam[g * I + rr];
  const double il = 1.0 / lam;
  const double fl = p.floor[g];
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  const C* __restrict__ yb = (const C*)p.y + (m * p.N * p.F + f) * I;
  R* vb = (R*)p.v + m * 2 * NF + f;  // no __restrict__: may alias vr (in place)
  const R* vr = (p.v_src ? (const R*)p.v_src : (const R*)p.v) + m * 2 * NF + f;
  FFCA_CHECK(g >= 0 && g < G && m < p.M && n0 >= 0 && n1 <= p.N);
#ifdef FFCA_DEBUG_BOUNDS
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    printf("fast_par I=%d R=%d U%d L%d M%d: M=%ld N=%ld F=%ld G=%ld cf=%ld nc=%d y=%p v=%p P=%p W=%p lam=%p fl=%p Sp=%p ll=%p mu=%p st=%p\n",
           I, (int)sizeof(R), (int)UPDATE, (int)LL, (int)MU, (long)p.M, (long)p.N, (long)p.F,
           (long)p.G, (long)p.chunk_frames, p.nchunk, p.y, p.v, (const void*)p.P,
           (const void*)p.W, (const void*)p.lam, (const void*)p.floor, (void*)p.Spart,
           (void*)p.llbin, p.mu_out, (void*)p.st);
#endif

  // accumulators: the diagonal entry (rr, rr) (real) and the off-diagonal
  // entries (rr, rr + s mod I), s = 1..I/2, dealt circulantly so every lane
  // owns ceil or floor of (I-1)/2 of them (the s = I/2 entries of an even
  // order to the lower half of the lanes); arrays are only ever indexed by
  // the compile-time slot s (runtime indexing would demote them to local
  // memory)
  constexpr int NO = I / 2;  // off-diagonal slots per lane
  int ob[NO + 1];
  bool ov[NO + 1];
#pragma unroll
  for (int s = 1; s <= NO; ++s) {
    ob[s] = (rr + s) % I;
    ov[s] = own && (s < NO || (I % 2) == 1 || rr < NO);
  }
  double accd1 = 0.0, accd2 = 0.0;
  double acc1[NO + 1], acc2[NO + 1], acc1i[NO + 1], acc2i[NO + 1];
#pragma unroll
  for (int c = 0; c <= NO; ++c) acc1[c] = acc2[c] = acc1i[c] = acc2i[c] = 0.0;
  double llacc = 0.0;
  int64_t bad_n = 0;

  // per-lane cp.async ring (kStages frames in flight, no registers held):
  // slot = y_r | v1 | v2, padded to an odd number of 16-B units
  constexpr int kStages = 8;
  constexpr int YB = (int)sizeof(C), VB = (int)sizeof(R);
  constexpr int SLOT = 16 * ((((YB + 2 * VB + 15) / 16) % 2) ? (YB + 2 * VB + 15) / 16
                                                                : (YB + 2 * VB + 15) / 16 + 1);
  unsigned char* ring = (unsigned char*)(sm + (size_t)Lay::BPB * Lay::GROUP_DOUBLES) +
                        (size_t)threadIdx.x * SLOT;
  constexpr size_t kStageStride = (size_t)Lay::WARPS * 32 * SLOT;
  const int K = (int)(n1 - n0 > 0 ? n1 - n0 : 0);
  // frames are issued in order: running pointers, no per-frame n * F products
  const C* ynext = yb + n0 * p.F * I + rr;
  const R* vnext = vr + n0 * p.F;
  const int64_t ystep = p.F * I;
  auto issue = [&](int k) {
    unsigned char* slot = ring + (size_t)(k % kStages) * kStageStride;
    if constexpr (YB == 16)
      cp_async16(slot, ynext);
    else
      cp_async8(slot, ynext);
    if constexpr (VB == 8) {
      cp_async8(slot + YB, vnext);
      cp_async8(slot + YB + 8, vnext + NF);
    } else {
      cp_async4(slot + YB, vnext);
      cp_async4(slot + YB + 4, vnext + NF);
    }
    ynext += ystep;
    vnext += p.F;
  };
  if constexpr (PAIR) {
    // Two frames per trip: the per-frame chains (exchange -> z -> posterior
    // -> group sums -> exchange -> accumulate) of frames k and k+1 run
    // interleaved, with one set of warp barriers per pair. The per-lane ring
    // runs a full kStages frames ahead: the two slots just read are refilled
    // with frames k + kStages, k + kStages + 1 (no other lane reads them).
    double2* syB = sgg + I;  // frame k+1's exchange buffers
    double2* szB = syB + I;
    double2* sggB = szB + I;
#pragma unroll
    for (int k = 0; k < kStages; ++k) {
      if (k < K) issue(k);
      cp_async_commit();
    }
#pragma unroll 1
    for (int k = 0; k < K; k += 2) {
      const bool two = k + 1 < K;  // (warp-uniform)
      cp_async_wait<kStages - 2>();  // frames k and k+1 have landed
      const unsigned char* slA = ring + (size_t)(k % kStages) * kStageStride;
      const unsigned char* slB = ring + (size_t)((k + 1) % kStages) * kStageStride;
      const double2 yA = to_c128(*(const C*)slA), yB = to_c128(*(const C*)slB);
      const double v1A = (double)*(const R*)(slA + YB), v2A = (double)*(const R*)(slA + YB + VB);
      const double v1B = (double)*(const R*)(slB + YB), v2B = (double)*(const R*)(slB + YB + VB);
      if (k + kStages < K) issue(k + kStages);
      cp_async_commit();
      if (k + kStages + 1 < K) issue(k + kStages + 1);
      cp_async_commit();
      if (own) {
        sy[r] = yA;
        syB[r] = yB;
      }
      __syncwarp();
      double zrA = 0.0, ziA = 0.0, zrB = 0.0, ziB = 0.0;
#pragma unroll
      for (int b = 0; b < I; ++b) {
        const double2 a_ = sy[b], b_ = syB[b];
        zrA = fma(pc[b].x, a_.x, fma(pc[b].y, a_.y, zrA));
        ziA = fma(pc[b].x, a_.y, fma(-pc[b].y, a_.x, ziA));
        zrB = fma(pc[b].x, b_.x, fma(pc[b].y, b_.y, zrB));
        ziB = fma(pc[b].x, b_.y, fma(-pc[b].y, b_.x, ziB));
      }
      const double v1lA = v1A * lam, v1lB = v1B * lam;
      const double rdA = rcp_nr(v1lA + v2A), rdB = rcp_nr(v1lB + v2B);
      const double g1A = v1lA * rdA, g2A = v2A * rdA, g1B = v1lB * rdB, g2B = v2B * rdB;
      const double cA = v2A * g1A, cB = v2B * g1B;
      const double pzA = fma(zrA, zrA, ziA * ziA), pzB = fma(zrB, zrB, ziB * ziB);
      const double t1A = fma(g1A * g1A, pzA, cA), t2A = fma(g2A * g2A, pzA, cA);
      const double t1B = fma(g1B * g1B, pzB, cB), t2B = fma(g2B * g2B, pzB, cB);
      if (own) {
        sz[r] = cmk(zrA, ziA);
        sgg[r] = cmk(g1A, g2A);
        szB[r] = cmk(zrB, ziB);
        sggB[r] = cmk(g1B, g2B);
      }
      double q1A = own ? t1A * il : 0.0, q2A = own ? t2A : 0.0;
      double q1B = own ? t1B * il : 0.0, q2B = own ? t2B : 0.0;
#pragma unroll
      for (int o = LB / 2; o > 0; o >>= 1) {  // four group sums, interleaved
        q1A += __shfl_xor_sync(0xffffffffu, q1A, o);
        q2A += __shfl_xor_sync(0xffffffffu, q2A, o);
        q1B += __shfl_xor_sync(0xffffffffu, q1B, o);
        q2B += __shfl_xor_sync(0xffffffffu, q2B, o);
      }
      q1A /= I, q2A /= I, q1B /= I, q2B /= I;
      const double w1A = (q1A < fl) ? fl : q1A, w2A = (q2A < fl) ? fl : q2A;
      const double w1B = (q1B < fl) ? fl : q1B, w2B = (q2B < fl) ? fl : q2B;
      if (r == 0) {
        const int64_t nA = n0 + k;
        if (active) {
          vb[nA * p.F] = (R)w1A;
          vb[NF + nA * p.F] = (R)w2A;
          if (two) {
            vb[(nA + 1) * p.F] = (R)w1B;
            vb[NF + (nA + 1) * p.F] = (R)w2B;
          }
        }
        auto badw = [](double w1, double w2) {
          const long long b1 = __double_as_longlong(w1), b2 = __double_as_longlong(w2);
          return (((b1 >> 52) & 0x7ff) == 0x7ff) | (((b2 >> 52) & 0x7ff) == 0x7ff) | (b1 <= 0) |
                 (b2 <= 0);
        };
        if (badw(w1A, w2A) && bad_n == 0) bad_n = nA + 1;
        if (two && badw(w1B, w2B) && bad_n == 0) bad_n = nA + 2;
      }
      __syncwarp();
      if (own) {
        const double iw1A = rcp_nr(w1A), iw2A = rcp_nr(w2A);
        const double iw1B = rcp_nr(w1B), iw2B = rcp_nr(w2B);
        const double h1A = g1A * iw1A, h2A = g2A * iw2A;
        const double h1B = two ? g1B * iw1B : 0.0, h2B = two ? g2B * iw2B : 0.0;
        accd1 = fma(t1A, iw1A, accd1);
        accd2 = fma(t2A, iw2A, accd2);
        if (two) {
          accd1 = fma(t1B, iw1B, accd1);
          accd2 = fma(t2B, iw2B, accd2);
        }
#pragma unroll
        for (int so = 1; so <= NO; ++so) {
          if (so == NO && (I % 2) == 0 && !ov[so]) continue;  // the half-filled last slot
          const int cc = ob[so];
          const double2 zcA = sz[cc], ggA = sgg[cc], zcB = szB[cc], ggB = sggB[cc];
          const double xrA = fma(zrA, zcA.x, ziA * zcA.y), xiA = fma(ziA, zcA.x, -zrA * zcA.y);
          const double xrB = fma(zrB, zcB.x, ziB * zcB.y), xiB = fma(ziB, zcB.x, -zrB * zcB.y);
          const double k1A = h1A * ggA.x, k2A = h2A * ggA.y;
          const double k1B = h1B * ggB.x, k2B = h2B * ggB.y;  // 0 for a missing frame
          acc1[so] = fma(k1B, xrB, fma(k1A, xrA, acc1[so]));
          acc1i[so] = fma(k1B, xiB, fma(k1A, xiA, acc1i[so]));
          acc2[so] = fma(k2B, xrB, fma(k2A, xrA, acc2[so]));
          acc2i[so] = fma(k2B, xiB, fma(k2A, xiA, acc2i[so]));
        }
      }
      __syncwarp();  // the exchange buffers are rewritten by the next pair
    }
  } else {
#pragma unroll
  for (int k = 0; k < kStages - 1; ++k) {
    if (k < K) issue(k);
    cp_async_commit();
  }
#pragma unroll 1
  for (int64_t n = n0; n < n1; ++n) {
    const int k = (int)(n - n0);
    if (k + kStages - 1 < K) issue(k + kStages - 1);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    const unsigned char* slot = ring + (size_t)(k % kStages) * kStageStride;
    const double2 ycur = to_c128(*(const C*)slot);
    const double v1 = (double)*(const R*)(slot + YB);
    const double v2 = (double)*(const R*)(slot + YB + VB);
    if (own) sy[r] = ycur;
    __syncwarp();
    // channel r
    double zr = 0.0, zi = 0.0;
#pragma unroll
    for (int b = 0; b < I; ++b) {
      const double2 yb_ = sy[b];
      zr = fma(pc[b].x, yb_.x, fma(pc[b].y, yb_.y, zr));
      zi = fma(pc[b].x, yb_.y, fma(-pc[b].y, yb_.x, zi));
    }
    const double v1l = v1 * lam;
    const double den = v1l + v2;
    const double rden = rcp_nr(den);
    const double g1 = v1l * rden, g2 = v2 * rden;
    const double c = v2 * g1;
    const double pz = fma(zr, zr, zi * zi);
    const double t1 = fma(g1 * g1, pz, c);
    const double t2 = fma(g2 * g2, pz, c);
    if (LL && own) llacc += log(den) + pz * rden;
    if (own) {
      sz[r] = cmk(zr, zi);
      sgg[r] = cmk(g1, g2);
    }
    double w1 = 0.0, w2 = 0.0;
    if (UPDATE) {
      const double tr1 = group_sum<LB>(own ? t1 * il : 0.0);
      const double tr2 = group_sum<LB>(own ? t2 : 0.0);
      const double q1 = tr1 / I, q2 = tr2 / I;
      w1 = (q1 < fl) ? fl : q1;
      w2 = (q2 < fl) ? fl : q2;
      if (r == 0) {
        if (active) {
          vb[n * p.F] = (R)w1;
          vb[NF + n * p.F] = (R)w2;
        }
        const long long b1 = __double_as_longlong(w1), b2 = __double_as_longlong(w2);
        const bool bad = (((b1 >> 52) & 0x7ff) == 0x7ff) | (((b2 >> 52) & 0x7ff) == 0x7ff) |
                         (b1 <= 0) | (b2 <= 0);
        if (bad && bad_n == 0) bad_n = n + 1;
      }
    }
    __syncwarp();
    if (UPDATE && own) {
      const double iw1 = rcp_nr(w1), iw2 = rcp_nr(w2);
      const double h1 = g1 * iw1, h2 = g2 * iw2;
      accd1 = fma(t1, iw1, accd1);
      accd2 = fma(t2, iw2, accd2);
#pragma unroll
      for (int so = 1; so <= NO; ++so) {
        if (so == NO && (I % 2) == 0 && !ov[so]) continue;  // the half-filled last slot
        const int cc = ob[so];
        const double2 zc = sz[cc];
        const double xr = fma(zr, zc.x, zi * zc.y);   // z_r conj(z_c)
        const double xi = fma(zi, zc.x, -zr * zc.y);
        const double2 gg = sgg[cc];
        const double k1 = h1 * gg.x, k2 = h2 * gg.y;
        acc1[so] = fma(k1, xr, acc1[so]);
        acc1i[so] = fma(k1, xi, acc1i[so]);
        acc2[so] = fma(k2, xr, acc2[so]);
        acc2i[so] = fma(k2, xi, acc2i[so]);
      }
    }
    if (MU && own && active) {
      C* mo = (C*)p.mu_out;
      C o1, o2;
      if (p.mu_back) {
        double sx = 0.0, sy_ = 0.0;
#pragma unroll
        for (int b = 0; b < I; ++b) {
          const double2 zb = sz[b];
          const double gb = sgg[b].x;
          const double mx = gb * zb.x, my = gb * zb.y;
          sx = fma(wr[b].x, mx, fma(-wr[b].y, my, sx));
          sy_ = fma(wr[b].x, my, fma(wr[b].y, mx, sy_));
        }
        o1.x = sx;
        o1.y = sy_;
        o2.x = ycur.x - sx;  // partition mu_1 + mu_2 = y
        o2.y = ycur.y - sy_;
      } else {
        o1.x = zr * g1;
        o1.y = zi * g1;
        o2.x = zr * g2;
        o2.y = zi * g2;
      }
      mo[(((m * 2 + 0) * p.N + n) * p.F + f) * I + r] = o1;
      mo[(((m * 2 + 1) * p.N + n) * p.F + f) * I + r] = o2;
    }
    __syncwarp();  // sy / sz are rewritten by the next frame
  }
  }
  cp_async_wait_all();
  if (bad_n && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));
  if (LL) llacc = group_sum<LB>(llacc);
  if (!active) return;
  const int64_t ch = blockIdx.y;
  if (UPDATE && own) {
    double* sp = p.Spart + (size_t)ch * 2 * NP * G + g;
    FFCA_CHECK(ch < p.nchunk);
    sp[(size_t)r * G] = accd1;
    sp[(size_t)(NP + r) * G] = accd2;
#pragma unroll
    for (int so = 1; so <= NO; ++so) {
      if (!ov[so]) continue;
      // stored entry (a, b), a < b: the slot's (r, c) or its conjugate
      const int cc = ob[so];
      const bool flip = r > cc;
      const int a = flip ? cc : r, b = flip ? r : cc;
      const double s = flip ? -1.0 : 1.0;
      sp[(size_t)Herm<I>::re(a, b) * G] = acc1[so];
      sp[(size_t)Herm<I>::im(a, b) * G] = s * acc1i[so];
      sp[(size_t)(NP + Herm<I>::re(a, b)) * G] = acc2[so];
      sp[(size_t)(NP + Herm<I>::im(a, b)) * G] = s * acc2i[so];
    }
  }
  if (LL && r == 0) p.llbin[(size_t)ch * G + g] = llacc;
}

template <int I, typename R, bool UPDATE, bool LL, bool MU>
static cudaError_t launch_fast_par_v(const FastIterParams& p, cudaStream_t s) {
  constexpr bool PAIR = FFCA_K3P_PAIR && UPDATE && !LL && !MU;
  using Lay = FastParLayout<I, PAIR>;
  dim3 grid((unsigned)((window_end(p.g1, p.G) - p.g0 + Lay::BPB - 1) / Lay::BPB),
            (unsigned)p.nchunk);
  return launch_ex(fast_par_kernel<I, R, UPDATE, LL, MU, PAIR>, grid, dim3(Lay::WARPS * 32),
                   Lay::SMEM, s, p.pdl != 0, 0, p);
}

template <int I, typename R>
static cudaError_t launch_fast_par_t(const FastIterParams& p, cudaStream_t s) {
  const bool ll = p.llbin != nullptr;
  const bool mu = p.mu_out != nullptr;
  if (p.update) {
    if (!ll && !mu) return launch_fast_par_v<I, R, true, false, false>(p, s);
    if (ll && !mu) return launch_fast_par_v<I, R, true, true, false>(p, s);
    if (!ll && mu) return launch_fast_par_v<I, R, true, false, true>(p, s);
    return launch_fast_par_v<I, R, true, true, true>(p, s);
  }
  if (ll && !mu) return launch_fast_par_v<I, R, false, true, false>(p, s);
  if (!ll && mu) return launch_fast_par_v<I, R, false, false, true>(p, s);
  if (ll && mu) return launch_fast_par_v<I, R, false, true, true>(p, s);
  return cudaSuccess;
}

cudaError_t launch_fast_par(const FastIterParams& p, int I, int dtype, cudaStream_t s) {
  const bool f32 = dtype == FFCA_C64;
  switch (I) {
    case 5: return f32 ? launch_fast_par_t<5, float>(p, s) : launch_fast_par_t<5, double>(p, s);
    case 6: return f32 ? launch_fast_par_t<6, float>(p, s) : launch_fast_par_t<6, double>(p, s);
    case 7: return f32 ? launch_fast_par_t<7, float>(p, s) : launch_fast_par_t<7, double>(p, s);
    case 8: return f32 ? launch_fast_par_t<8, float>(p, s) : launch_fast_par_t<8, double>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

int fast_par_blocks_per_sm(int I, int dtype) {
  int n = 0;
  const bool f32 = dtype == FFCA_C64;
  switch (I) {
#define FFCA_OCC(II)                                                                            \
  case II:                                                                                      \
    if (f32)                                                                                    \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                            \
          &n, fast_par_kernel<II, float, true, false, false, FFCA_K3P_PAIR>,                    \
          FastParLayout<II>::WARPS * 32, FastParLayout<II, FFCA_K3P_PAIR>::SMEM);               \
    else                                                                                        \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                            \
          &n, fast_par_kernel<II, double, true, false, false, FFCA_K3P_PAIR>,                   \
          FastParLayout<II>::WARPS * 32, FastParLayout<II, FFCA_K3P_PAIR>::SMEM);               \
    break;
    FFCA_OCC(5)
    FFCA_OCC(6)
    FFCA_OCC(7)
    FFCA_OCC(8)
#undef FFCA_OCC
  }
  return n > 0 ? n : 1;
}

int fast_par_bins_per_cta() { return FastParLayout<8>::BPB; }

}  // namespace ffca
