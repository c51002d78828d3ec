// K4p — conventional FCA pass for large orders (5 <= I <= 8), lane-parallel.
//
// A point's frame-wise inverse (reference _kernels_numba.py:246-325) needs
// I x I complex matrices: at I = 8 ~1 KB each, so the per-thread kernel
// (ffca_fca.cu) spills heavily. Here a group of 8 lanes owns one bin and
// streams its frames; lane r owns row r of the per-point matrices:
//   R = v1 S1 + v2 S2 -> Rinv by Gauss-Jordan (pivot rows published through
//   shared memory, rows eliminated in registers), x = Rinv y,
//   Rinv and x x^H entries, traces, w_j, v update,
//   B_j += v_j^2/w_j x x^H, X_j += v1 v2/w_j Rinv  (as fca_em_kernel: the
//   I x I products of Phi_j are applied once per bin in fca_finish_kernel).
// The I(I+1)/2 Hermitian entries are dealt to the lanes circulantly: lane r
// owns (r, r + s mod I) for s = 0..I/2 (the s = I/2 diagonal of an even order
// to the lower half of the lanes), so every lane has ceil or floor of
// (I+1)/2 entries instead of a triangular row. Per-bin S1, S2 stay in shared
// memory (packed Hermitian). Partial sums per (chunk, bin) in the K4 layout.
#include "ffca_pencil_par.cuh"

namespace ffca {

namespace {

template <int I>
struct FcaParLayout {
  static constexpr int LB = 8;
  static constexpr int WARPS = 2;
  static constexpr int BPB = WARPS * 32 / LB;  // bins (groups) per CTA
  static constexpr int LD = (I % 2) ? I + 2 : I + 1;
  static constexpr int NS = I / 2 + 1;          // entry slots per lane
  static constexpr int MATD = I * LD * 2;       // doubles per padded complex matrix
  // per group: S1, S2 unpacked (2 MATD) + 1 matrix (rows of Rinv) + 3 vectors
  // (2I each) + misc (2) + pivot row and its inverse row (4I), rounded to an
  // odd number of 16-B units
  static constexpr int RAW = 3 * MATD + 6 * I + 2 + 4 * I;
  static constexpr int U16 = (RAW + 1) / 2;
  static constexpr int GROUP_DOUBLES = 2 * ((U16 % 2) ? U16 : U16 + 1);
  static constexpr size_t SMEM = (size_t)BPB * GROUP_DOUBLES * sizeof(double);
};


}  // namespace

template <int I, typename R>
#ifndef FCA_PAR_MINB
#define FCA_PAR_MINB 6  // CTAs per SM the lane-parallel FCA pass is register-budgeted for
#endif
__global__ void __launch_bounds__(FcaParLayout<I>::WARPS * 32, FCA_PAR_MINB) fca_par_kernel(const FcaIterParams p) {
  using Lay = FcaParLayout<I>;
  using C = typename CplxOf<R>::type;
  constexpr int NP = I * I;
  constexpr int LB = Lay::LB;
  constexpr int NS = Lay::NS;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane % LB;
  const int grp = warp * (32 / LB) + lane / LB;
  const int64_t G = p.G;
  int64_t g = (int64_t)blockIdx.x * Lay::BPB + grp;
  const bool active = g < G;
  if (!active) g = G - 1;
  const bool own = r < I;
  const int rr = own ? r : 0;
  const int64_t m = (unsigned)g / (unsigned)p.F, f = g - m * p.F;  // (32-bit division)
  double* base = sm + (size_t)grp * Lay::GROUP_DOUBLES;
  double2* SF = (double2*)base;             // [2][I][LD]: S1, S2 unpacked (row reads, no branches)
  double2* Lm = SF + 2 * I * Lay::LD;       // rows of Rinv
  double2* vy = Lm + I * Lay::LD;           // y
  double2* vx = vy + I;                     // R^-1 y (vy + 2I: spare)
  double* misc = (double*)(vx + I);
  double2* prow = (double2*)(misc + 2);     // published pivot row of R
  double2* pinv = prow + I;                 // and of the inverse
  auto at = [&](int a, int b) -> double2& { return Lm[a * Lay::LD + b]; };

  if (own) {  // row r of both covariances from the packed SoA copy
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < I; ++c) {
        const double* bj = p.Sp + (size_t)j * NP * G + g;
        double2 e;
        if (c == r)
          e = cmk(bj[(size_t)r * G], 0.0);
        else if (r < c)
          e = cmk(bj[(size_t)Herm<I>::re(r, c) * G], bj[(size_t)Herm<I>::im(r, c) * G]);
        else
          e = cmk(bj[(size_t)Herm<I>::re(c, r) * G], -bj[(size_t)Herm<I>::im(c, r) * G]);
        SF[(j * I + r) * Lay::LD + c] = e;
      }
  }
  __syncwarp();
  auto S1 = [&](int a, int b) -> double2 { return SF[a * Lay::LD + b]; };
  auto S2 = [&](int a, int b) -> double2 { return SF[(I + a) * Lay::LD + b]; };
  // this lane's entry slots: (a0, b0) = (r, r + s mod I)
  int sb[NS];
  bool sv[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    sb[s] = (rr + s) % I;
    sv[s] = own && (s < I / 2 || (I % 2) == 1 || rr < I / 2);
  }
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  const C* __restrict__ yb = (const C*)p.y + (m * p.N * p.F + f) * I;
  R* vb = (R*)p.v + m * 2 * NF + f;  // no __restrict__: may alias vr (in place)
  const R* vr = (p.v_src ? (const R*)p.v_src : (const R*)p.v) + m * 2 * NF + f;
  const double fl = p.floor[g];
  const bool do_ll = p.llbin != nullptr;

  // accumulators per slot, oriented (a0, b0): B1, B2, X1, X2
  double2 acc[kFcaParts][NS];
#pragma unroll
  for (int j = 0; j < kFcaParts; ++j)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[j][s] = cmk(0.0, 0.0);
  double llacc = 0.0;
  int64_t bad_n = 0;

  // one frame of prefetch in registers
  double2 ynext = cmk(0.0, 0.0);
  double v1n = 0.0, v2n = 0.0;
  if (n0 < n1) {
    if (own) ynext = to_c128(yb[n0 * p.F * I + r]);
    v1n = (double)vr[n0 * p.F];
    v2n = (double)vr[NF + n0 * p.F];
  }
#pragma unroll 1
  for (int64_t n = n0; n < n1; ++n) {
    const double2 ycur = ynext;
    const double v1 = v1n, v2 = v2n;
    if (n + 1 < n1) {
      if (own) ynext = to_c128(yb[(n + 1) * p.F * I + r]);
      v1n = (double)vr[(n + 1) * p.F];
      v2n = (double)vr[NF + (n + 1) * p.F];
    }
    // R = v1 S1 + v2 S2: row r in registers, with the row of the inverse
    double2 rrow[I], irow[I];
    if (own) {
      vy[r] = ycur;
#pragma unroll
      for (int c = 0; c < I; ++c) {
        const double2 s1 = S1(r, c), s2 = S2(r, c);
        rrow[c] = cmk(v1 * s1.x + v2 * s2.x, v1 * s1.y + v2 * s2.y);
        irow[c] = cmk(c == r ? 1.0 : 0.0, 0.0);
      }
    }
    // Frame-wise inverse by Gauss-Jordan elimination without pivoting (R is
    // Hermitian positive definite: the pivots are its LDL^H pivots d_p, all
    // > 0 iff R is PD — the reference's singular-mixture test). Step p: lane p
    // publishes its (unnormalised) pivot row, every other lane eliminates
    // column p from its row in registers (I complex MACs, independent across
    // columns); each row is scaled by 1/d_r at the end. One warp barrier per
    // step instead of the column-sequential Cholesky + triangular inverse +
    // L^-H L^-1 chain.
    bool okc = true;
    double dr = 1.0;
#pragma unroll
    for (int q = 0; q < I; ++q) {
      if (own && r == q) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          if (c >= q) prow[c] = rrow[c];
          if (c <= q) pinv[c] = irow[c];
        }
      }
      __syncwarp();
      const double d = prow[q].x;
      okc = okc && d > 0.0;
      if (own) {
        if (r == q) {
          dr = d;
        } else {
          const double2 fct = cscale(rrow[q], rcp_fast(d));
#pragma unroll
          for (int c = 0; c < I; ++c) {
            if (c > q) rrow[c] = cmsub(rrow[c], fct, prow[c]);
            if (c <= q) irow[c] = cmsub(irow[c], fct, pinv[c]);
          }
        }
      }
      __syncwarp();  // prow / pinv are rewritten by the next pivot
    }
    if (!okc && bad_n == 0) bad_n = n + 1;
    // row r of Rinv (into shared memory for the slot reads), x = Rinv y
    double2 ri[NS];
    double lquad = 0.0;
    if (own) {
      const double idr = rcp_fast(dr);
      double2 xr = cmk(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < I; ++c) {
        irow[c] = cscale(irow[c], idr);
        at(r, c) = irow[c];
        xr = cmac(xr, irow[c], vy[c]);
      }
      vx[r] = xr;
      lquad = ycur.x * xr.x + ycur.y * xr.y;  // Re conj(y_r) x_r
#pragma unroll
      for (int s = 0; s < NS; ++s) ri[s] = at(r, sb[s]);
    }
    __syncwarp();
    // log det R + y^H Rinv y = sum_r log d_r + Re y^H x
    if (do_ll) llacc += group_sum<LB>(own ? log(dr) + lquad : 0.0);
    if (p.mu_out != nullptr && active && own) {
      // mu_j = v_j S_j x (row r; the image pass only)
      double2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) {
        s1 = cmac(s1, S1(r, k), vx[k]);
        s2 = cmac(s2, S2(r, k), vx[k]);
      }
      C* mo = (C*)p.mu_out;
      mo[(((m * 2 + 0) * p.N + n) * p.F + f) * I + r] = from_c128<R>(cscale(s1, v1));
      mo[(((m * 2 + 1) * p.N + n) * p.F + f) * I + r] = from_c128<R>(cscale(s2, v2));
    }
    if (p.update) {
      // tr(A B) of Hermitian A, B over this lane's slots (weight 2 off the
      // diagonal): qf_j = tr(S_j x x^H), tR_j = tr(Rinv S_j)
      double2 xe[NS];
      double qf1 = 0.0, qf2 = 0.0, tR1 = 0.0, tR2 = 0.0;
      const double2 xr = vx[rr];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double2 xb = vx[sb[s]];
        xe[s] = cmulc(xr, xb);  // x_a0 conj(x_b0)
        if (s == 0) xe[s].y = 0.0;
        const double wgt = sv[s] ? (s == 0 ? 1.0 : 2.0) : 0.0;
        const double2 s1 = S1(rr, sb[s]), s2 = S2(rr, sb[s]);
        qf1 += wgt * (s1.x * xe[s].x + s1.y * xe[s].y);
        qf2 += wgt * (s2.x * xe[s].x + s2.y * xe[s].y);
        tR1 += wgt * (s1.x * ri[s].x + s1.y * ri[s].y);
        tR2 += wgt * (s2.x * ri[s].x + s2.y * ri[s].y);
      }
      const double vv = v1 * v2;
      const double t1 = group_sum<LB>(v1 * v1 * qf1 + vv * tR2);
      const double t2 = group_sum<LB>(v2 * v2 * qf2 + vv * tR1);
      const double q1 = t1 / I, q2 = t2 / I;
      const double w1 = (q1 < fl) ? fl : q1;
      const double w2 = (q2 < fl) ? fl : q2;
      if (active && r == 0) {
        vb[n * p.F] = (R)w1;
        vb[NF + n * p.F] = (R)w2;
      }
      const double iw1 = rcp_fast(w1), iw2 = rcp_fast(w2);
      const double cb1 = v1 * v1 * iw1, cb2 = v2 * v2 * iw2, cx1 = vv * iw1, cx2 = vv * iw2;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        acc[0][s].x = fma(cb1, xe[s].x, acc[0][s].x);
        acc[0][s].y = fma(cb1, xe[s].y, acc[0][s].y);
        acc[1][s].x = fma(cb2, xe[s].x, acc[1][s].x);
        acc[1][s].y = fma(cb2, xe[s].y, acc[1][s].y);
        acc[2][s].x = fma(cx1, ri[s].x, acc[2][s].x);
        acc[2][s].y = fma(cx1, ri[s].y, acc[2][s].y);
        acc[3][s].x = fma(cx2, ri[s].x, acc[3][s].x);
        acc[3][s].y = fma(cx2, ri[s].y, acc[3][s].y);
      }
    }
    __syncwarp();  // smem buffers are reused by the next frame
  }
  if (bad_n && active && r == 0 && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MIXTURE,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));
  if (!active) return;
  const int64_t ch = blockIdx.y;
  if (p.update) {
    double* sp = p.Spart + (size_t)ch * kFcaParts * NP * G + g;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (!sv[s]) continue;
      const int b0 = sb[s];
      if (s == 0) {
#pragma unroll
        for (int j = 0; j < kFcaParts; ++j) sp[(size_t)(j * NP + rr) * G] = acc[j][s].x;
      } else {
        // stored entry (a, b), a < b: the slot's (a0, b0) or its conjugate
        const bool flip = rr > b0;
        const int a = flip ? b0 : rr, b = flip ? rr : b0;
        const int ire = Herm<I>::re(a, b), iim = Herm<I>::im(a, b);
#pragma unroll
        for (int j = 0; j < kFcaParts; ++j) {
          sp[(size_t)(j * NP + ire) * G] = acc[j][s].x;
          sp[(size_t)(j * NP + iim) * G] = flip ? -acc[j][s].y : acc[j][s].y;
        }
      }
    }
  }
  if (do_ll && r == 0) p.llbin[(size_t)ch * G + g] = llacc;
}

// K4b — per-bin FCA steps, lane-parallel (LB lanes per bin, lane r owns
// row r; LB = the order rounded up to a power of two):
//  * finish: sums the chunk partials of the pass (fixed chunk order) and forms
//      out_j = (S_j B_j S_j + S1 X_j S2) / N, Hermitian part
//    with row-parallel products in shared memory, then either writes S_raw
//    (stage API) or regularises (modelops.py:29-39: + 1e-9 tr/I) and writes
//    the model / history S;
//  * prepare (S_in set): takes the initial model S instead;
// then packs S for the next pass and checks each S_j is positive definite
// (the reference factors every S_j per iteration: _cholesky_inverse,
// conventional.py:98-101) with a column-sequential Cholesky.
namespace {
template <int I>
struct BinParLayout {
  static constexpr int LB = I <= 1 ? 1 : I <= 2 ? 2 : I <= 4 ? 4 : 8;
  static constexpr int GROUPS = 64 / LB;  // bins per CTA
  static constexpr int LD = (I % 2) ? I + 2 : I + 1;
  static constexpr int MATD = I * LD * 2;
  static constexpr int RAW = 4 * MATD + 2;  // S1, S2, A (B / X / M), T
  static constexpr int U16 = (RAW + 1) / 2;
  static constexpr int GROUP_DOUBLES = 2 * ((U16 % 2) ? U16 : U16 + 1);
  static constexpr size_t SMEM = (size_t)GROUPS * GROUP_DOUBLES * sizeof(double);
};
}  // namespace

template <int I>
__global__ void __launch_bounds__(64)
    fca_bin_par_kernel(const double* __restrict__ Spart, int nchunk, int64_t N, int64_t G,
                       int64_t F, double* Sp, double2* S_model, double2* S_hist,
                       const double* llbin, double* llg, double2* S_raw,
                       const double2* __restrict__ S_in, ffca_status_dev* st, int iter) {
  using Lay = BinParLayout<I>;
  constexpr int NP = I * I;
  constexpr int LB = Lay::LB;
  constexpr int LD = Lay::LD;
  constexpr int NS = I / 2 + 1;
  // chained plain schedule: every thread waits for the streaming pass this
  // launch may programmatically depend on (a no-op otherwise) before the
  // CTA releases the next pass (launch_dependents counts per CTA)
  pdl_wait_primary();
  pdl_release_dependents();
  extern __shared__ __align__(16) double sm[];
  const int r = threadIdx.x % LB;
  const int grp = threadIdx.x / LB;
  int64_t g = (int64_t)blockIdx.x * Lay::GROUPS + grp;
  const bool active = g < G;
  if (!active) g = G - 1;
  const bool own = r < I;
  const int rr = own ? r : 0;
  const int64_t m = (unsigned)g / (unsigned)F, f = g - m * F;  // (32-bit division)
  double2* mS1 = (double2*)(sm + (size_t)grp * Lay::GROUP_DOUBLES);
  double2* mS2 = mS1 + I * LD;
  double2* mA = mS2 + I * LD;
  double2* mT = mA + I * LD;
  double* misc = (double*)(mT + I * LD);
  auto S1 = [&](int a, int b) -> double2& { return mS1[a * LD + b]; };
  auto S2 = [&](int a, int b) -> double2& { return mS2[a * LD + b]; };
  auto A = [&](int a, int b) -> double2& { return mA[a * LD + b]; };
  auto T = [&](int a, int b) -> double2& { return mT[a * LD + b]; };
  double2 out[2][I];
  if (S_in) {
    // prepare: the initial model (M,2,F,I,I)
    if (own) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int c = 0; c < I; ++c) out[j][c] = S_in[((m * 2 + j) * F + f) * NP + r * I + c];
    }
  } else {
    auto packed = [&](const double* base, int a, int b) -> double2 {  // base[e * G + g]
      if (a == b) return cmk(base[(size_t)a * G + g], 0.0);
      if (a < b)
        return cmk(base[(size_t)Herm<I>::re(a, b) * G + g],
                   base[(size_t)Herm<I>::im(a, b) * G + g]);
      return cmk(base[(size_t)Herm<I>::re(b, a) * G + g],
                 -base[(size_t)Herm<I>::im(b, a) * G + g]);
    };
    if (own) {
#pragma unroll
      for (int c = 0; c < I; ++c) {
        S1(r, c) = packed(Sp, r, c);
        S2(r, c) = packed(Sp + (size_t)NP * G, r, c);
      }
    }
    if (llg && r == 0 && active) llg[g] = -ordered_sum(llbin + g, nchunk, (size_t)G);
    __syncwarp();
    const double invN = 1.0 / (double)N;
    // chunk sums of this lane's circulant slots (r, r + s mod I) of all four
    // parts, in one pass over the chunks (all loads of a chunk in flight;
    // per-entry chunk order fixed)
    int ire[NS], iim[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int b0 = (rr + s) % I;
      const int a = rr < b0 ? rr : b0, b = rr < b0 ? b0 : rr;
      ire[s] = a == b ? a : Herm<I>::re(a, b);
      iim[s] = a == b ? a : Herm<I>::im(a, b);
    }
    double2 sums[kFcaParts][NS];
#pragma unroll
    for (int q = 0; q < kFcaParts; ++q)
#pragma unroll
      for (int s = 0; s < NS; ++s) sums[q][s] = cmk(0.0, 0.0);
    if (own) {
      // CB chunks per batch: all their loads issued before the (ordered) adds
      constexpr int NL = kFcaParts * NS * 2;
      constexpr int CB = NL >= 64 ? 1 : 64 / NL;
#pragma unroll 1
      for (int c0 = 0; c0 < nchunk; c0 += CB) {
        double t[CB][kFcaParts][NS][2];
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          if (c0 + cb >= nchunk) break;
#pragma unroll
          for (int q = 0; q < kFcaParts; ++q) {
            const double* sp = Spart + ((size_t)(c0 + cb) * kFcaParts + q) * NP * G + g;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
              t[cb][q][s][0] = sp[(size_t)ire[s] * G];
              t[cb][q][s][1] = sp[(size_t)iim[s] * G];
            }
          }
        }
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          if (c0 + cb >= nchunk) break;
#pragma unroll
          for (int q = 0; q < kFcaParts; ++q)
#pragma unroll
            for (int s = 0; s < NS; ++s) {
              sums[q][s].x += t[cb][q][s][0];
              sums[q][s].y += t[cb][q][s][1];
            }
        }
      }
    }
    // part `part` into the full matrix A
    auto gather = [&](int part) {
      if (!own) return;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (!(s < I / 2 || (I % 2) == 1 || rr < I / 2)) continue;
        const int b0 = (rr + s) % I;
        const int a = rr < b0 ? rr : b0, b = rr < b0 ? b0 : rr;
        const double sr = sums[part][s].x, si = a == b ? 0.0 : sums[part][s].y;
        A(a, b) = cmk(sr, si);
        A(b, a) = cmk(sr, -si);
      }
    };
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      // T = B_j S_j (row r), then M = S_j T (row r, registers)
      gather(j);
      __syncwarp();
      if (own) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 t = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) t = cmac(t, A(r, k), j == 0 ? S1(k, c) : S2(k, c));
          T(r, c) = t;
        }
      }
      __syncwarp();
      double2 mrow[I];
      if (own) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 t = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) t = cmac(t, j == 0 ? S1(r, k) : S2(r, k), T(k, c));
          mrow[c] = t;
        }
      }
      __syncwarp();
      // + S1 (X_j S2)
      gather(2 + j);
      __syncwarp();
      if (own) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 t = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) t = cmac(t, A(r, k), S2(k, c));
          T(r, c) = t;
        }
      }
      __syncwarp();
      if (own) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 t = mrow[c];
#pragma unroll
          for (int k = 0; k < I; ++k) t = cmac(t, S1(r, k), T(k, c));
          A(r, c) = t;  // M row r (A is free: every lane has read X_j)
        }
      }
      __syncwarp();
      // Hermitian part, / N (reference hermitize, modelops.py:24-26)
      if (own) {
#pragma unroll
        for (int c = 0; c < I; ++c) {
          const double2 u = A(r, c), w = A(c, r);
          out[j][c] = cmk(0.5 * (u.x + w.x) * invN, 0.5 * (u.y - w.y) * invN);
        }
      }
      __syncwarp();
    }
    if (S_raw) {
      if (active && own)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int c = 0; c < I; ++c)
            S_raw[((size_t)j * G + g) * NP + r * I + c] =
                c == r ? cmk(out[j][c].x, 0.0) : out[j][c];
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (!S_in) {
      // regularize_covariances: Hermitian diagonal + 1e-9 tr/I
      double dg = 0.0;
#pragma unroll
      for (int c = 0; c < I; ++c)
        if (c == r) dg = out[j][c].x;
      const double tr = group_sum<LB>(own ? dg : 0.0);
      const double eps = kCovEps * tr / I;
#pragma unroll
      for (int c = 0; c < I; ++c)
        if (c == r) out[j][c] = cmk(out[j][c].x + eps, 0.0);
      if (active && own) {
        double2* dst = S_model + ((m * 2 + j) * F + f) * NP + r * I;
        double2* hst = S_hist ? S_hist + ((m * 2 + j) * F + f) * NP + r * I : nullptr;
#pragma unroll
        for (int c = 0; c < I; ++c) {
          dst[c] = out[j][c];
          if (hst) hst[c] = out[j][c];
        }
      }
    }
    if (active && own) {
      double* dp = Sp + (size_t)j * NP * G + g;  // packed for the next pass (row r, c >= r)
#pragma unroll
      for (int c = 0; c < I; ++c) {
        if (c < r) continue;
        if (c == r) {
          dp[(size_t)r * G] = out[j][c].x;
        } else {
          dp[(size_t)Herm<I>::re(r, c) * G] = out[j][c].x;
          dp[(size_t)Herm<I>::im(r, c) * G] = out[j][c].y;
        }
      }
    }
    // positive-definiteness (Cholesky in A, column-sequential)
    __syncwarp();
    if (own) {
#pragma unroll
      for (int c = 0; c < I; ++c) A(r, c) = out[j][c];
    }
    __syncwarp();
    bool ok = true;
#pragma unroll
    for (int q = 0; q < I; ++q) {
      if (own && r == q) {
        double d = A(q, q).x;
#pragma unroll
        for (int k = 0; k < q; ++k) d -= cabs2(A(q, k));
        misc[0] = d;
        A(q, q) = cmk(sqrt(fmax(d, 0.0)), 0.0);
      }
      __syncwarp();
      ok = ok && misc[0] > 0.0;
      if (own && r > q) {
        double2 t = A(r, q);
#pragma unroll
        for (int k = 0; k < q; ++k) t = cmsubc(t, A(r, k), A(q, k));
        A(r, q) = cscale(t, 1.0 / A(q, q).x);
      }
      __syncwarp();
    }
    if (!ok && active && r == 0 && st)
      report_error(st, S_in ? iter : iter + 1, FFCA_ERR_NOT_PD, (unsigned long long)g);
  }
}

template <int I>
static cudaError_t launch_fca_bin_par_t(const double* Spart, int nchunk, int64_t N, int64_t G,
                                        int64_t F, double* Sp, double2* S_model,
                                        double2* S_hist, const double* llbin, double* llg,
                                        double2* S_raw, const double2* S_in, ffca_status_dev* st,
                                        int iter, cudaStream_t s, int pdl) {
  using Lay = BinParLayout<I>;
  const unsigned nb = (unsigned)((G + Lay::GROUPS - 1) / Lay::GROUPS);
  return launch_ex(fca_bin_par_kernel<I>, dim3(nb), dim3(64), Lay::SMEM, s, pdl != 0, 0, Spart,
                   nchunk, N, G, F, Sp, S_model, S_hist, llbin, llg, S_raw, S_in, st, iter);
}

cudaError_t launch_fca_bin_par(const double* Spart, int nchunk, int64_t N, int64_t G, int64_t F,
                               double* Sp, double2* S_model, double2* S_hist,
                               const double* llbin, double* llg, double2* S_raw,
                               const double2* S_in, int I, ffca_status_dev* st, int iter,
                               cudaStream_t s, int pdl) {
  switch (I) {
#define FFCA_CASE(II)                                                                         \
  case II:                                                                                    \
    return launch_fca_bin_par_t<II>(Spart, nchunk, N, G, F, Sp, S_model, S_hist, llbin, llg, \
                                    S_raw, S_in, st, iter, s, pdl);
    FFCA_CASE(1)
    FFCA_CASE(2)
    FFCA_CASE(3)
    FFCA_CASE(4)
    FFCA_CASE(5)
    FFCA_CASE(6)
    FFCA_CASE(7)
    FFCA_CASE(8)
#undef FFCA_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

template <int I, typename R>
cudaError_t launch_fca_par_t(const FcaIterParams& p, cudaStream_t s) {
  using Lay = FcaParLayout<I>;
  auto kern = fca_par_kernel<I, R>;
  if (cudaError_t e = ensure_smem<fca_par_kernel<I, R>>(Lay::SMEM)) return e;
  dim3 grid((unsigned)((p.G + Lay::BPB - 1) / Lay::BPB), (unsigned)p.nchunk);
  kern<<<grid, Lay::WARPS * 32, Lay::SMEM, s>>>(p);
  return cudaGetLastError();
}

template <int I, typename R>
int fca_par_bpsm_t() {
  using Lay = FcaParLayout<I>;
  auto kern = fca_par_kernel<I, R>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::SMEM);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, Lay::WARPS * 32, Lay::SMEM);
  return n > 0 ? n : 1;
}

cudaError_t launch_fca_par(const FcaIterParams& p, int I, int dtype, cudaStream_t s) {
  const bool f32 = dtype == FFCA_C64;
  switch (I) {
    case 5: return f32 ? launch_fca_par_t<5, float>(p, s) : launch_fca_par_t<5, double>(p, s);
    case 6: return f32 ? launch_fca_par_t<6, float>(p, s) : launch_fca_par_t<6, double>(p, s);
    case 7: return f32 ? launch_fca_par_t<7, float>(p, s) : launch_fca_par_t<7, double>(p, s);
    case 8: return f32 ? launch_fca_par_t<8, float>(p, s) : launch_fca_par_t<8, double>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

int fca_par_blocks_per_sm(int I, int dtype) {
  const bool f32 = dtype == FFCA_C64;
  switch (I) {
    case 5: return f32 ? fca_par_bpsm_t<5, float>() : fca_par_bpsm_t<5, double>();
    case 6: return f32 ? fca_par_bpsm_t<6, float>() : fca_par_bpsm_t<6, double>();
    case 7: return f32 ? fca_par_bpsm_t<7, float>() : fca_par_bpsm_t<7, double>();
    case 8: return f32 ? fca_par_bpsm_t<8, float>() : fca_par_bpsm_t<8, double>();
    default: return 1;
  }
}

int fca_par_bins_per_cta(int I) {
  (void)I;
  return FcaParLayout<8>::BPB;
}

}  // namespace ffca
