// K1p kernels: lane-parallel pencil refresh and initial pencil (see
// ffca_pencil_par.cuh). Same inputs/outputs as pencil_update_kernel /
// initial_pencil_kernel (ffca_pencil.cu).
#include "ffca_pencil_par.cuh"

namespace ffca {

// packed-Hermitian entry e (0 .. I*I-1) -> (a, b, component); component 0 =
// real diagonal, 1 = real part of (a<b), 2 = imaginary part of (a<b)
template <int I>
FFCA_DEV void packed_to_ab(int e, int& a, int& b, int& comp) {
  if (e < I) {
    a = b = e;
    comp = 0;
    return;
  }
  int idx = (e - I) >> 1;
  comp = 1 + ((e - I) & 1);
  int row = 0;
  while (idx >= I - row - 1) {
    idx -= I - row - 1;
    ++row;
  }
  a = row;
  b = row + 1 + idx;
}

template <int I>
__global__ void __launch_bounds__(ParLayout<I>::WARPS * 32) pencil_par_kernel(const PencilParams p) {
  using Lay = ParLayout<I>;
  constexpr int NP = I * I;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane % Lay::LB;
  const int bb = warp * Lay::BPW + lane / Lay::LB;
  const int64_t G = p.G;
  int64_t g = p.g0 + (int64_t)blockIdx.x * Lay::BPB + bb;
  const bool active = g < G;
  if (!active) g = G - 1;
  const bool own = r < I;
  const bool wr = own && active;  // may write global memory
  double* binb = sm + (size_t)bb * Lay::BIN_DOUBLES;
  const BinView<I> v{(double2*)binb, binb + Lay::NMAT * Lay::MAT * 2};
  const int64_t m = (unsigned)g / (unsigned)p.F, f = g - m * p.F;  // (32-bit division)

  // 1. chunk partials -> S~1, S~2 (full Hermitian); entries split over lanes
  bool fin = true;
  // every entry of this lane accumulates in one pass over the chunks (all
  // its loads of a chunk in flight together; per-entry chunk order kept,
  // bitwise equal to ordered_sum)
  constexpr int EPL = (2 * NP + Lay::LB - 1) / Lay::LB;  // entries per lane
  double part[EPL];
#pragma unroll
  for (int t = 0; t < EPL; ++t) part[t] = 0.0;
  constexpr int CB = EPL >= 64 ? 1 : 64 / EPL;  // chunks per batch of loads
#pragma unroll 1
  for (int c0 = 0; c0 < p.nchunk; c0 += CB) {
    double ld[CB][EPL];
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      if (c0 + cb >= p.nchunk) break;
      const double* sp = p.Spart + (size_t)(c0 + cb) * 2 * NP * G + g;
#pragma unroll
      for (int t = 0; t < EPL; ++t)
        ld[cb][t] = (r + Lay::LB * t < 2 * NP) ? sp[(size_t)(r + Lay::LB * t) * G] : 0.0;
    }
#pragma unroll
    for (int cb = 0; cb < CB; ++cb) {
      if (c0 + cb >= p.nchunk) break;
#pragma unroll
      for (int t = 0; t < EPL; ++t) part[t] += ld[cb][t];
    }
  }
#pragma unroll
  for (int t = 0; t < EPL; ++t) {
    const int e = r + Lay::LB * t;
    if (e >= 2 * NP) continue;
    double sacc = part[t] * (1.0 / (double)p.N);
    fin = fin && isfinite(sacc);
    const int j = e < NP ? 0 : 1;
    int a, b, comp;
    packed_to_ab<I>(e - j * NP, a, b, comp);
    const int M = j == 0 ? kS1 : kS2;
    if (comp == 0) {
      v.at(M, a, a) = cmk(sacc, 0.0);
    } else if (comp == 1) {
      v.at(M, a, b).x = sacc;
      v.at(M, b, a).x = sacc;
    } else {
      v.at(M, a, b).y = sacc;
      v.at(M, b, a).y = -sacc;
    }
  }
  if (!fin && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX, (unsigned long long)g);
  if (p.llg && active && r == 0) {
    const double sacc = ordered_sum(p.llbin + g, p.nchunk, (size_t)G);
    p.llg[g] = (double)p.N * p.logdet2[g] - sacc;
  }
  // 2. P_e -> kP, W_e -> kX (row r)
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c) {
      v.at(kP, r, c) = p.P[g * NP + r * I + c];
      v.at(kX, r, c) = p.W[g * NP + r * I + c];
    }
  }
  __syncwarp();
  // 3. tr(gram^-1 S~_j) with gram^-1 = W^H W (lane r: row r of S, column r of H)
  double t1 = 0.0, t2 = 0.0;
  if (own) {
#pragma unroll
    for (int b = 0; b < I; ++b) {
      double2 h = cmk(0.0, 0.0);  // H[b][r] = sum_k conj(W[k][b]) W[k][r]
#pragma unroll
      for (int k = 0; k < I; ++k) h = cmac_cj(h, v.at(kX, k, b), v.at(kX, k, r));
      const double2 s1 = v.at(kS1, r, b), s2 = v.at(kS2, r, b);
      t1 += s1.x * h.x - s1.y * h.y;
      t2 += s2.x * h.x - s2.y * h.y;
    }
  }
  t1 = group_sum<Lay::LB>(t1);
  t2 = group_sum<Lay::LB>(t2);
  const double eps1 = kCovEps * t1 / I, eps2 = kCovEps * t2 / I;
  __syncwarp();
  // 4. S_t = S~ + eps gram (upper from row owners, then mirrored)
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c) {
      if (c < r) continue;
      double2 gr = cmk(0.0, 0.0);  // gram[r][c] = sum_k conj(P[k][r]) P[k][c]
#pragma unroll
      for (int k = 0; k < I; ++k) gr = cmac_cj(gr, v.at(kP, k, r), v.at(kP, k, c));
      double2 a1 = cadd(v.at(kS1, r, c), cscale(gr, eps1));
      double2 a2 = cadd(v.at(kS2, r, c), cscale(gr, eps2));
      if (c == r) {
        a1.y = 0.0;
        a2.y = 0.0;
      }
      v.at(kS1, r, c) = a1;
      v.at(kS2, r, c) = a2;
    }
  }
  __syncwarp();
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c)
      if (c < r) {
        v.at(kS1, r, c) = cconj(v.at(kS1, c, r));
        v.at(kS2, r, c) = cconj(v.at(kS2, c, r));
      }
  }
  __syncwarp();
  // 5. model / history covariance W S_t W^H (only when read)
  if (p.S_model || p.S_hist) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int Sm = j == 0 ? kS1 : kS2;
      if (own) {  // kT[r][c] = sum_k S[r][k] conj(W[c][k])
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 acc = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) acc = cadd(acc, cmulc(v.at(Sm, r, k), v.at(kX, c, k)));
          v.at(kT, r, c) = acc;
        }
      }
      __syncwarp();
      if (wr) {
        double2* dst = p.S_model ? p.S_model + ((m * 2 + j) * p.F + f) * NP : nullptr;
        double2* hst = p.S_hist ? p.S_hist + ((m * 2 + j) * p.F + f) * NP : nullptr;
#pragma unroll
        for (int c = 0; c < I; ++c) {
          double2 acc = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < I; ++k) acc = cmac(acc, v.at(kX, r, k), v.at(kT, k, c));
          if (dst) dst[r * I + c] = acc;
          if (hst) hst[r * I + c] = acc;
        }
      }
      __syncwarp();
    }
  }
  // 6. GEVD of (S_t1, S_t2): eigenvalues -> scal, eigenvectors -> kA
  double msig = 0.0;
  const int rc = par_gevd<I>(v, r, own, &msig);
  if (rc != 0 && active && r == 0 && p.st) {
    report_error(p.st, p.iter, rc, (unsigned long long)g);
    report_min_value(p.st, msig);
  }
  // 7. P_next = P_e Q -> kT and global
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < I; ++k) acc = cmac(acc, v.at(kP, r, k), v.at(kA, k, c));
      v.at(kT, r, c) = acc;
      if (wr) p.P[g * NP + r * I + c] = acc;
    }
    if (wr) p.lam[g * I + r] = v.scal[6 * Lay::NPAIR + r];
  }
  __syncwarp();
  // 8. W_next = P_next^{-H}, log|det P_next|^2
  bool ok = true;
  const double lad = par_lu_inverse<I>(v, kT, r, own, &ok);
  if (wr) {
#pragma unroll
    for (int c = 0; c < I; ++c) p.W[g * NP + r * I + c] = cconj(v.at(kInv, c, r));
    if (r == 0) p.logdet2[g] = 2.0 * lad;
  }
}

template <int I>
__global__ void __launch_bounds__(ParLayout<I>::WARPS * 32)
    initial_par_kernel(const double2* __restrict__ S0, double2* P, double2* W, double* lam,
                       double* logdet2, int64_t G, int64_t F, ffca_status_dev* st) {
  using Lay = ParLayout<I>;
  constexpr int NP = I * I;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane % Lay::LB;
  const int bb = warp * Lay::BPW + lane / Lay::LB;
  int64_t g = (int64_t)blockIdx.x * Lay::BPB + bb;
  const bool active = g < G;
  if (!active) g = G - 1;
  const bool own = r < I;
  const bool wr = own && active;
  double* binb = sm + (size_t)bb * Lay::BIN_DOUBLES;
  const BinView<I> v{(double2*)binb, binb + Lay::NMAT * Lay::MAT * 2};
  const int64_t m = (unsigned)g / (unsigned)F, f = g - m * F;  // (32-bit division)
  const double2* s1 = S0 + ((m * 2 + 0) * F + f) * NP;
  const double2* s2 = S0 + ((m * 2 + 1) * F + f) * NP;
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c) {
      v.at(kS1, r, c) = s1[r * I + c];
      v.at(kS2, r, c) = s2[r * I + c];
    }
  }
  __syncwarp();
  // _check_hermitian (pencil.py:40-51) on both matrices
  double sc1 = 0.0, sc2 = 0.0, as1 = 0.0, as2 = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c) {
      sc1 = fmax(sc1, sqrt(cabs2(v.at(kS1, r, c))));
      sc2 = fmax(sc2, sqrt(cabs2(v.at(kS2, r, c))));
      as1 = fmax(as1, sqrt(cabs2(csub(v.at(kS1, r, c), cconj(v.at(kS1, c, r))))));
      as2 = fmax(as2, sqrt(cabs2(csub(v.at(kS2, r, c), cconj(v.at(kS2, c, r))))));
    }
  }
#pragma unroll
  for (int o = Lay::LB / 2; o > 0; o >>= 1) {
    sc1 = fmax(sc1, __shfl_xor_sync(0xffffffffu, sc1, o));
    sc2 = fmax(sc2, __shfl_xor_sync(0xffffffffu, sc2, o));
    as1 = fmax(as1, __shfl_xor_sync(0xffffffffu, as1, o));
    as2 = fmax(as2, __shfl_xor_sync(0xffffffffu, as2, o));
  }
  if ((as1 > kHermRtol * fmax(sc1, 1e-300) || as2 > kHermRtol * fmax(sc2, 1e-300)) && active &&
      r == 0 && st)
    report_error(st, 0, FFCA_ERR_NON_HERMITIAN, (unsigned long long)g);
  double msig = 0.0;
  const int rc = par_gevd<I>(v, r, own, &msig);
  if (rc != 0 && active && r == 0 && st) {
    report_error(st, 0, rc, (unsigned long long)g);
    report_min_value(st, msig);
  }
  if (wr) {
#pragma unroll
    for (int c = 0; c < I; ++c) P[g * NP + r * I + c] = v.at(kA, r, c);
    lam[g * I + r] = v.scal[6 * Lay::NPAIR + r];
  }
  __syncwarp();
  bool ok = true;
  const double lad = par_lu_inverse<I>(v, kA, r, own, &ok);
  if (wr) {
#pragma unroll
    for (int c = 0; c < I; ++c) W[g * NP + r * I + c] = cconj(v.at(kInv, c, r));
    if (r == 0) logdet2[g] = 2.0 * lad;
  }
}

template <int I>
static cudaError_t launch_par_t(const PencilParams& p, cudaStream_t s) {
  using Lay = ParLayout<I>;
  if (cudaError_t e = ensure_smem<pencil_par_kernel<I>>(Lay::SMEM)) return e;
  const unsigned nb = (unsigned)((window_end(p.g1, p.G) - p.g0 + Lay::BPB - 1) / Lay::BPB);
  if (cudaError_t e = launch_ex(pencil_par_kernel<I>, dim3(nb), dim3(Lay::WARPS * 32), Lay::SMEM,
                                s, false, p.prio, p))
    return e;
  return cudaGetLastError();
}

template <int I>
static cudaError_t launch_init_par_t(const double2* S0, double2* P, double2* W, double* lam,
                                     double* logdet2, int64_t G, int64_t F, ffca_status_dev* st,
                                     cudaStream_t s) {
  using Lay = ParLayout<I>;
  if (cudaError_t e = ensure_smem<initial_par_kernel<I>>(Lay::SMEM)) return e;
  const unsigned nb = (unsigned)((G + Lay::BPB - 1) / Lay::BPB);
  initial_par_kernel<I><<<nb, Lay::WARPS * 32, Lay::SMEM, s>>>(S0, P, W, lam, logdet2, G, F, st);
  return cudaGetLastError();
}

#define FFCA_PAR_SWITCH(I, CALL) \
  switch (I) {                   \
    case 1: return CALL(1);      \
    case 2: return CALL(2);      \
    case 3: return CALL(3);      \
    case 4: return CALL(4);      \
    case 5: return CALL(5);      \
    case 6: return CALL(6);      \
    case 7: return CALL(7);      \
    case 8: return CALL(8);      \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_pencil_par(const PencilParams& p, int I, cudaStream_t s) {
#define FFCA_CALL(II) launch_par_t<II>(p, s)
  FFCA_PAR_SWITCH(I, FFCA_CALL)
#undef FFCA_CALL
}

cudaError_t launch_initial_par(const double2* S0, double2* P, double2* W, double* lam,
                               double* logdet2, int64_t G, int64_t F, int I, ffca_status_dev* st,
                               cudaStream_t s) {
#define FFCA_CALL(II) launch_init_par_t<II>(S0, P, W, lam, logdet2, G, F, st, s)
  FFCA_PAR_SWITCH(I, FFCA_CALL)
#undef FFCA_CALL
}

}  // namespace ffca
