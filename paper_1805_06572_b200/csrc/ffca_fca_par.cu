// K4p — conventional FCA pass for large orders (5 <= I <= 8), lane-parallel.
//
// A point's frame-wise inverse and I x I products (reference
// _kernels_numba.py:246-325) need several I x I complex matrices: at I = 8
// that is ~1 KB each, so the per-thread kernel (ffca_fca.cu) spills heavily.
// Here a group of 8 lanes owns one bin and streams its frames; lane r owns row
// r (or column r) of every per-point matrix, which lives in shared memory:
//   R = v1 S1 + v2 S2 -> Cholesky L (column-sequential, row-parallel)
//   L^-1 (column-parallel)      u = L^-1 y, x = L^-H u = R^-1 y
//   mu_j = v_j S_j x            T = L^-H (L^-1 S2) = R^-1 S2
//   cross = v1 v2 S1 T (row r in registers; Hermitian, so its column r is
//   the conjugate of its row r)  tr_j = Re tr(S_j^-1 Phi_j) by group sum
//   w_j, v update, S_j rows accumulated in registers (upper triangle).
// Per-bin S1, S2, S1^-1, S2^-1 stay in shared memory (packed Hermitian).
// Partial sums per (chunk, bin) in the same Spart layout as K4.
#include "ffca_pencil_par.cuh"

namespace ffca {

namespace {

template <int I>
struct FcaParLayout {
  static constexpr int LB = 8;
  static constexpr int WARPS = 2;
  static constexpr int BPB = WARPS * 32 / LB;  // bins (groups) per CTA
  static constexpr int LD = (I % 2) ? I + 2 : I + 1;
  static constexpr int NP = I * I;
  static constexpr int MATD = I * LD * 2;  // doubles per padded complex matrix
  // per group: 4 packed S (4 NP) + 3 matrices (L/Y2, Li, T) + 5 vectors (2I each)
  // + misc (8), rounded to an odd number of 16-B units
  static constexpr int RAW = 4 * NP + 3 * MATD + 10 * I + 8;
  static constexpr int U16 = (RAW + 1) / 2;
  static constexpr int GROUP_DOUBLES = 2 * ((U16 % 2) ? U16 : U16 + 1);
  static constexpr size_t SMEM = (size_t)BPB * GROUP_DOUBLES * sizeof(double);
};

template <int I>
FFCA_DEV double2 packed_get(const double* S, int a, int b) {
  if (a == b) return cmk(S[a], 0.0);
  if (a < b) return cmk(S[Herm<I>::re(a, b)], S[Herm<I>::im(a, b)]);
  return cmk(S[Herm<I>::re(b, a)], -S[Herm<I>::im(b, a)]);
}

}  // namespace

template <int I, typename R>
__global__ void __launch_bounds__(FcaParLayout<I>::WARPS * 32) fca_par_kernel(const FcaIterParams p) {
  using Lay = FcaParLayout<I>;
  using C = typename CplxOf<R>::type;
  constexpr int NP = I * I;
  constexpr int LB = Lay::LB;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane % LB;
  const int grp = warp * (32 / LB) + lane / LB;
  const int64_t G = p.G;
  int64_t g = (int64_t)blockIdx.x * Lay::BPB + grp;
  const bool active = g < G;
  if (!active) g = G - 1;
  const bool own = r < I;
  const int64_t m = g / p.F, f = g - m * p.F;
  double* base = sm + (size_t)grp * Lay::GROUP_DOUBLES;
  double* Sp = base;                         // [4][NP] packed: S1, S2, S1^-1, S2^-1
  double2* Lm = (double2*)(base + 4 * NP);   // R / L, later Y2 = L^-1 S2
  double2* Li = Lm + I * Lay::LD;            // L^-1
  double2* Tm = Li + I * Lay::LD;            // R^-1 S2
  double2* vy = Tm + I * Lay::LD;            // y
  double2* vu = vy + I;                      // L^-1 y
  double2* vx = vu + I;                      // R^-1 y
  double2* vm1 = vx + I;                     // mu_1
  double2* vm2 = vm1 + I;                    // mu_2
  double* misc = (double*)(vm2 + I);
  auto at = [&](double2* M, int a, int b) -> double2& { return M[a * Lay::LD + b]; };

  for (int e = r; e < 4 * NP; e += LB) Sp[e] = p.Sp[(size_t)e * G + g];
  __syncwarp();
  const double* S1 = Sp;
  const double* S2 = Sp + NP;
  const double* Si1 = Sp + 2 * NP;
  const double* Si2 = Sp + 3 * NP;
  const int64_t n0 = (int64_t)blockIdx.y * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  const C* __restrict__ yb = (const C*)p.y + (m * p.N * p.F + f) * I;
  R* __restrict__ vb = (R*)p.v + m * 2 * NF + f;
  const double fl = p.floor[g];
  const bool do_ll = p.llbin != nullptr;

  double2 acc1[I], acc2[I];  // row r of the S_j sums (entries c >= r used)
#pragma unroll
  for (int c = 0; c < I; ++c) acc1[c] = acc2[c] = cmk(0.0, 0.0);
  double llacc = 0.0;
  int64_t bad_n = 0;

  // one frame of prefetch in registers
  double2 ynext = cmk(0.0, 0.0);
  double v1n = 0.0, v2n = 0.0;
  if (n0 < n1) {
    if (own) ynext = to_c128(yb[n0 * p.F * I + r]);
    v1n = (double)vb[n0 * p.F];
    v2n = (double)vb[NF + n0 * p.F];
  }
#pragma unroll 1
  for (int64_t n = n0; n < n1; ++n) {
    const double2 ycur = ynext;
    const double v1 = v1n, v2 = v2n;
    if (n + 1 < n1) {
      if (own) ynext = to_c128(yb[(n + 1) * p.F * I + r]);
      v1n = (double)vb[(n + 1) * p.F];
      v2n = (double)vb[NF + (n + 1) * p.F];
    }
    if (own) {
      vy[r] = ycur;
#pragma unroll
      for (int c = 0; c < I; ++c) {
        const double2 s1 = packed_get<I>(S1, r, c), s2 = packed_get<I>(S2, r, c);
        at(Lm, r, c) = cmk(v1 * s1.x + v2 * s2.x, v1 * s1.y + v2 * s2.y);
      }
    }
    __syncwarp();
    // Cholesky in place (lower), column-sequential. Every loop below is
    // unrolled over compile-time indices with the triangular bounds as
    // predicates: independent products interleave (ILP) instead of forming
    // one dependent chain of shared-memory loads per loop.
    bool okc = true;
#pragma unroll
    for (int j = 0; j < I; ++j) {
      if (own && r == j) {
        double d = at(Lm, j, j).x;
#pragma unroll
        for (int k = 0; k < j; ++k) d -= cabs2(at(Lm, j, k));
        misc[0] = d;
        at(Lm, j, j) = cmk(sqrt(fmax(d, 0.0)), 0.0);
      }
      __syncwarp();
      okc = okc && misc[0] > 0.0;
      if (own && r > j) {
        double2 s = at(Lm, r, j);
#pragma unroll
        for (int k = 0; k < j; ++k) s = csub(s, cmulc(at(Lm, r, k), at(Lm, j, k)));
        at(Lm, r, j) = cscale(s, 1.0 / at(Lm, j, j).x);
      }
      __syncwarp();
    }
    if (!okc && bad_n == 0) bad_n = n + 1;
    // L^-1, column-parallel: lane c keeps its column in registers
    if (own) {
      double2 col[I];
#pragma unroll
      for (int rr = 0; rr < I; ++rr) {
        double2 sacc = cmk(rr == r ? 1.0 : 0.0, 0.0);
#pragma unroll
        for (int k = 0; k < rr; ++k)
          if (k >= r) sacc = csub(sacc, cmul(at(Lm, rr, k), col[k]));
        col[rr] = (rr >= r) ? cscale(sacc, 1.0 / at(Lm, rr, rr).x) : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int rr = 0; rr < I; ++rr) at(Li, rr, r) = col[rr];
    }
    __syncwarp();
    // u = L^-1 y (row r), likelihood terms
    double lquad = 0.0, llog = 0.0;
    if (own) {
      double2 sacc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k)
        if (k <= r) sacc = cadd(sacc, cmul(at(Li, r, k), vy[k]));
      vu[r] = sacc;
      lquad = cabs2(sacc);
      llog = log(at(Lm, r, r).x);
    }
    __syncwarp();
    if (do_ll) {
      const double t = group_sum<LB>(2.0 * llog + lquad);
      llacc += t;
    }
    // x = L^-H u = R^-1 y; Y2 = L^-1 S2 into Lm (L no longer needed)
    double2 y2row[I];
    if (own) {
      double2 sacc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k)
        if (k >= r) sacc = cadd(sacc, cconjmul(at(Li, k, r), vu[k]));
      vx[r] = sacc;
      double2 lrow[I];
#pragma unroll
      for (int k = 0; k < I; ++k) lrow[k] = at(Li, r, k);
#pragma unroll
      for (int c = 0; c < I; ++c) {
        double2 t = cmk(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < I; ++k)
          if (k <= r) t = cadd(t, cmul(lrow[k], packed_get<I>(S2, k, c)));
        y2row[c] = t;
      }
    }
    __syncwarp();  // everyone done reading Lm (diag) before Y2 overwrites it
    if (own) {
#pragma unroll
      for (int c = 0; c < I; ++c) at(Lm, r, c) = y2row[c];
    }
    __syncwarp();
    // mu_j = v_j S_j x (row r); T = L^-H Y2 (row r)
    if (own) {
      double2 s1 = cmk(0.0, 0.0), s2 = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) {
        s1 = cadd(s1, cmul(packed_get<I>(S1, r, k), vx[k]));
        s2 = cadd(s2, cmul(packed_get<I>(S2, r, k), vx[k]));
      }
      vm1[r] = cscale(s1, v1);
      vm2[r] = cscale(s2, v2);
      double2 lcol[I];  // column r of Li: conj -> row r of Li^H
#pragma unroll
      for (int k = 0; k < I; ++k) lcol[k] = at(Li, k, r);
#pragma unroll
      for (int c = 0; c < I; ++c) {
        double2 t = cmk(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < I; ++k)
          if (k >= r) t = cadd(t, cconjmul(lcol[k], at(Lm, k, c)));
        at(Tm, r, c) = t;
      }
    }
    __syncwarp();
    if (p.mu_out != nullptr && active && own) {
      C* mo = (C*)p.mu_out;
      mo[(((m * 2 + 0) * p.N + n) * p.F + f) * I + r] = from_c128<R>(vm1[r]);
      mo[(((m * 2 + 1) * p.N + n) * p.F + f) * I + r] = from_c128<R>(vm2[r]);
    }
    if (p.update) {
      // cross row r = v1 v2 S1 T; traces against S_j^-1 (column r of Phi_j)
      double2 cr[I];
      double t1 = 0.0, t2 = 0.0;
      if (own) {
        const double vv = v1 * v2;
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 s = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) s = cadd(s, cmul(packed_get<I>(S1, r, k), at(Tm, k, c)));
          cr[c] = cscale(s, vv);
          if (c == r) cr[c].y = 0.0;  // compile-time index only: cr stays in registers
        }
        const double2 m1r = vm1[r], m2r = vm2[r];
#pragma unroll
        for (int b = 0; b < I; ++b) {
          // Phi_j[b][r] = mu_j[b] conj(mu_j[r]) + conj(cross[r][b])
          const double2 ph1 = cadd(cmulc(vm1[b], m1r), cconj(cr[b]));
          const double2 ph2 = cadd(cmulc(vm2[b], m2r), cconj(cr[b]));
          const double2 a1 = packed_get<I>(Si1, r, b), a2 = packed_get<I>(Si2, r, b);
          t1 += a1.x * ph1.x - a1.y * ph1.y;
          t2 += a2.x * ph2.x - a2.y * ph2.y;
        }
      }
      t1 = group_sum<LB>(t1);
      t2 = group_sum<LB>(t2);
      const double q1 = t1 / I, q2 = t2 / I;
      const double w1 = (q1 < fl) ? fl : q1;
      const double w2 = (q2 < fl) ? fl : q2;
      if (active && r == 0) {
        vb[n * p.F] = (R)w1;
        vb[NF + n * p.F] = (R)w2;
      }
      if (own) {
        const double iw1 = 1.0 / w1, iw2 = 1.0 / w2;
        const double2 m1r = vm1[r], m2r = vm2[r];
#pragma unroll
        for (int c = 0; c < I; ++c) {
          if (c < r) continue;
          const double2 p1 = cadd(cmulc(m1r, vm1[c]), cr[c]);
          const double2 p2 = cadd(cmulc(m2r, vm2[c]), cr[c]);
          acc1[c] = cadd(acc1[c], cscale(p1, iw1));
          acc2[c] = cadd(acc2[c], cscale(p2, iw2));
        }
      }
    }
    __syncwarp();  // smem buffers are reused by the next frame
  }
  if (bad_n && active && r == 0 && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MIXTURE,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));
  if (!active) return;
  const int64_t ch = blockIdx.y;
  if (p.update && own) {
    double* sp = p.Spart + (size_t)ch * 2 * NP * G + g;
#pragma unroll
    for (int c = 0; c < I; ++c) {
      if (c < r) continue;
      if (c == r) {
        sp[(size_t)r * G] = acc1[c].x;
        sp[(size_t)(NP + r) * G] = acc2[c].x;
      } else {
        sp[(size_t)Herm<I>::re(r, c) * G] = acc1[c].x;
        sp[(size_t)Herm<I>::im(r, c) * G] = acc1[c].y;
        sp[(size_t)(NP + Herm<I>::re(r, c)) * G] = acc2[c].x;
        sp[(size_t)(NP + Herm<I>::im(r, c)) * G] = acc2[c].y;
      }
    }
  }
  if (do_ll && r == 0) p.llbin[(size_t)ch * G + g] = llacc;
}

template <int I, typename R>
cudaError_t launch_fca_par_t(const FcaIterParams& p, cudaStream_t s) {
  using Lay = FcaParLayout<I>;
  auto kern = fca_par_kernel<I, R>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
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
