// K1's per-bin code (pencil_prep + pencil_update_body), shared by the
// one-thread-per-bin refresh kernel (ffca_pencil.cu) and the persistent EM
// kernel (ffca_persist.cuh).
#pragma once

#include <type_traits>

#include "ffca_internal.cuh"

namespace ffca {

// Steps shared by the fused (I <= 4) and split (I >= 5) pencil updates:
// chunk partials -> S~ (/N), ridge with eps*gram, model / history covariances,
// likelihood collect. Leaves S_t in S1/S2 and P_e in Pe.
struct NoPreSum {
  FFCA_DEV const double* operator()() const { return nullptr; }
};
// stand-alone refresh launched programmatically behind the streaming pass:
// wait for it, then release the next pass
struct PdlGateSum {
  bool on;
  FFCA_DEV const double* operator()() const {
    if (on) {
      pdl_wait_primary();
      pdl_release_dependents();
    }
    return nullptr;
  }
};
// `pre` (persistent kernel): called after this bin's P and W loads are issued
// and before the chunk partials are read — the wait for the tile's chunk CTAs.
// It may return a shared-memory copy of the tile's partials,
// [chunk][entry][32 bins] (the CTA's warps fetch it in one round trip), which
// the ordered sums then read instead of global memory.
template <int I, bool COH = false, class PreSum = NoPreSum>
FFCA_DEV bool pencil_prep(const PencilParams& p, int64_t g, double2 (&S1)[I][I],
                          double2 (&S2)[I][I], double2 (&Pe)[I][I], PreSum pre = PreSum()) {
  constexpr int NP = I * I;
  const int64_t G = p.G;
  const int64_t m = (unsigned)g / (unsigned)p.F, f = g - m * p.F;  // (32-bit division)

  // the basis of the pass being finished (this bin's P_e, W_e): requested
  // first, so that their latency overlaps the partials' (or the wait)
  // (stand-alone — also behind a programmatic wait — the 2 I^2 complex registers
  // are not affordable during the partial sums: loaded after them)
  constexpr bool kEarly = !std::is_same<PreSum, NoPreSum>::value && !std::is_same<PreSum, PdlGateSum>::value;
  double2 We[I][I];
  auto load_basis = [&]() {
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = 0; b < I; ++b) {
        Pe[a][b] = p.P[g * NP + a * I + b];
        We[a][b] = p.W[g * NP + a * I + b];
      }
  };
  if (kEarly) load_basis();
  const double* staged = pre();


  // 1. reduce partials
  {
    double s[2][NP];
#pragma unroll
    for (int e = 0; e < NP; ++e) s[0][e] = s[1][e] = 0.0;
    // CB chunks per batch: all their loads are issued before the adds, which
    // keep the chunk order (bitwise identical sums)
    // loads in flight per batch: ~64 (I = 4: register bound), ~108 at I = 3
    // (with the basis already in registers, half the batch at I = 3)
    constexpr int CB = I == 3 ? (kEarly ? 3 : 6)
                              : (2 * NP >= 64 ? 1 : (64 / (2 * NP) > 8 ? 8 : 64 / (2 * NP)));
#pragma unroll 1
    for (int c0 = 0; c0 < p.nchunk; c0 += CB) {
      double ld[CB][2 * NP];
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        if (c0 + cb >= p.nchunk) break;
        const double* sp = p.Spart + (size_t)(c0 + cb) * 2 * NP * G + g;
#pragma unroll
        for (int e = 0; e < 2 * NP; ++e)
          ld[cb][e] = staged ? staged[((c0 + cb) * 2 * NP + e) * 32 + (threadIdx.x & 31)]
                             : (COH ? __ldcg(sp + (size_t)e * G) : sp[(size_t)e * G]);
      }
#pragma unroll
      for (int cb = 0; cb < CB; ++cb) {
        if (c0 + cb >= p.nchunk) break;
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          s[0][e] += ld[cb][e];
          s[1][e] += ld[cb][NP + e];
        }
      }
    }
    const double invN = 1.0 / (double)p.N;
    bool fin = true;
#pragma unroll
    for (int e = 0; e < NP; ++e) {
      s[0][e] *= invN;
      s[1][e] *= invN;
      fin = fin && isfinite(s[0][e]) && isfinite(s[1][e]);
    }
    if (!fin && p.st) report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX, (unsigned long long)g);
    unpack_herm<I>(s[0], S1);
    unpack_herm<I>(s[1], S2);
  }
  // likelihood of the model this pass used (P_e, logdet2(P_e))
  if (p.llg) {
    const double s = ordered_sum(p.llbin + g, p.nchunk, (size_t)G);
    p.llg[g] = (double)p.N * p.logdet2[g] - s;
  }

  if (!kEarly) load_basis();

  // 2. ridge eps_j = 1e-9 tr(gram^{-1} S~_j)/I with gram^{-1} = W^H W
  //    (W = P^{-H}), then S_t = S~ + eps_j gram (fast.py:80-90).
  double eps[2];
  {
    double2 H[I][I];
    matmul_hn<I>(We, We, H);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double2(&Sj)[I][I] = j == 0 ? S1 : S2;
      double tr = 0.0;
#pragma unroll
      for (int a = 0; a < I; ++a) {
        tr += Sj[a][a].x * H[a][a].x;
#pragma unroll
        for (int b = a + 1; b < I; ++b)  // S_ab H_ba + S_ba H_ab = 2 Re(S_ab H_ba)
          tr += 2.0 * (Sj[a][b].x * H[b][a].x - Sj[a][b].y * H[b][a].y);
      }
      eps[j] = kCovEps * tr / I;
    }
  }
  {
    double2 gram[I][I];
    matmul_hn<I>(Pe, Pe, gram);
#pragma unroll
    for (int a = 0; a < I; ++a)
#pragma unroll
      for (int b = a; b < I; ++b) {
        // upper triangle of gram, mirrored: S_t stays exactly Hermitian
        S1[a][b] = cadd(S1[a][b], cscale(gram[a][b], eps[0]));
        S2[a][b] = cadd(S2[a][b], cscale(gram[a][b], eps[1]));
        if (b > a) {
          S1[b][a] = cconj(S1[a][b]);
          S2[b][a] = cconj(S2[a][b]);
        } else {
          S1[a][a].y = 0.0;
          S2[a][a].y = 0.0;
        }
      }
  }
  // model / history covariance back in the original basis: W S_t W^H
  // (fast.py:144-148), only when someone reads it
  if (p.S_model || p.S_hist) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double2 T[I][I], Sb[I][I];
      matmul_nh<I>(j == 0 ? S1 : S2, We, T);
      matmul<I>(We, T, Sb);
      double2* dst = p.S_model ? p.S_model + ((m * 2 + j) * p.F + f) * NP : nullptr;
      double2* hst = p.S_hist ? p.S_hist + ((m * 2 + j) * p.F + f) * NP : nullptr;
#pragma unroll
      for (int a = 0; a < I; ++a)
#pragma unroll
        for (int b = 0; b < I; ++b) {
          if (dst) dst[a * I + b] = Sb[a][b];
          if (hst) hst[a * I + b] = Sb[a][b];
        }
    }
  }

  return true;
}

// The refresh of bin g (K1's thread): GEVD of the regularised transformed
// pencil, P <- P Q, W = P^-H, log|det P|^2. COH: the chunk partials were
// written by other CTAs of the SAME kernel (persistent EM kernel) and are
// read with L2 loads.
struct NoPublish {
  FFCA_DEV void operator()() const {}
};
// `publish` (persistent kernel): called as soon as the bin's P_next and lambda
// are stored — all the next update pass reads — so that W = P_next^-H and
// log|det P|^2 (needed by the NEXT refresh's ridge, the image pass and the
// likelihood only) are computed while that pass is already streaming.
template <int I, bool COH = false, class PreSum = NoPreSum, class Publish = NoPublish>
FFCA_DEV void pencil_update_body(const PencilParams& p, const int64_t g, PreSum pre = PreSum(),
                                 Publish publish = Publish()) {
  constexpr int NP = I * I;
  double2 S1[I][I], S2[I][I], Pe[I][I];
  pencil_prep<I, COH, PreSum>(p, g, S1, S2, Pe, pre);

  // 3. GEVD of the transformed pencil, P <- P Q
  double lam[I];
  double2 Q[I][I];
  double msig = 0.0;
  const int rc = gevd_hpd<I>(S1, S2, lam, Q, &msig);
  if (rc != 0 && p.st) {
    report_error(p.st, p.iter, rc, (unsigned long long)g);
    report_min_value(p.st, msig);
  }
  double2 Pn[I][I];
  matmul<I>(Pe, Q, Pn);
#pragma unroll
  for (int a = 0; a < I; ++a) {
    p.lam[g * I + a] = lam[a];
#pragma unroll
    for (int b = 0; b < I; ++b) p.P[g * NP + a * I + b] = Pn[a][b];
  }
  publish();
  double2 Inv[I][I];
  double lad = 0.0;
  lu_inverse<I>(Pn, Inv, &lad);
#pragma unroll
  for (int a = 0; a < I; ++a)
#pragma unroll
    for (int b = 0; b < I; ++b) p.W[g * NP + a * I + b] = cconj(Inv[b][a]);
  p.logdet2[g] = 2.0 * lad;
}

}  // namespace ffca
