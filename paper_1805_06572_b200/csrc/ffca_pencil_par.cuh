// K1p — lane-parallel per-bin pencil refresh (all I <= 8).
//
// The per-thread K1 (ffca_pencil.cu) runs every small dense step of a bin's
// update serially in one thread: latency-bound when there are few bins
// (configs 0/1/2/4: 257-1025 bins) and a register-spilling monster at I = 8.
// Here a group of LB >= I lanes owns one bin; lane r owns row r (and, where
// an algorithm wants it, column r) of every I x I matrix, which live in
// shared memory with a padded row stride. Matrix products are row-parallel,
// the Cholesky factor is column-sequential with row-parallel updates, the
// triangular inverse is column-parallel, Gauss-Jordan is pivot-sequential /
// row-parallel, and the Hermitian Jacobi eigensolver uses the round-robin
// (Brent-Luk) ordering: I/2 disjoint rotations per round, column updates by
// row owners, row updates by column owners.
//
// Arithmetic and conventions match gevd_hpd / pencil_update_kernel:
// Cholesky-whitened GEVD (zhegv style), Demmel-Veselic Jacobi threshold,
// descending eigenvalues, largest-entry-real-positive column phases
// (reference pencil.py:76-135), ridge eps = 1e-9 tr(gram^-1 S~)/I with
// gram^-1 = W^H W (fast.py:80-90), P <- P Q (fast.py:107-113), W = P^-H and
// log|det P|^2 by pivoted Gauss-Jordan (fast.py:151-153).
#pragma once

#include "ffca_internal.cuh"

namespace ffca {

// Bank-conflict-free bin stride (in 16-B units): the lanes of a quarter warp
// (8 x 16 B = one 128-B shared-memory wavefront) belong to 8/LB bins and read
// entry (r, c) of their bin (row owners: r*LD + c) or (c, r) (column owners:
// c*LD + r); pick the padding of the bin stride S that keeps every
// quarter-warp on distinct 16-B slots.
constexpr int par_conflicts(int I, int LB, int LD, int S) {
  int worst = 0;
  for (int q = 0; q < 4; ++q)
    for (int pat = 0; pat < 2; ++pat) {
      int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int l = q * 8; l < q * 8 + 8; ++l) {
        const int b = l / LB, r = l % LB;
        if (r >= I) continue;
        const int off = b * S + (pat == 0 ? r * LD : r);
        const int c = ++cnt[off % 8];
        worst = c > worst ? c : worst;
      }
    }
  return worst;
}
constexpr int par_stride16(int I, int LB, int LD, int base16) {
  int best = base16, bw = 1 << 20;
  for (int S = base16; S < base16 + 16; ++S) {
    const int w = par_conflicts(I, LB, LD, S);
    if (w < bw) {
      bw = w;
      best = S;
    }
  }
  return best;
}

template <int I>
struct ParLayout {
  static constexpr int LB = I <= 2 ? 2 : (I <= 4 ? 4 : 8);  // lanes per bin
  static constexpr int BPW = 32 / LB;                       // bins per warp
  static constexpr int WARPS = 2;
  static constexpr int BPB = BPW * WARPS;     // bins per CTA
  static constexpr int LD = (I % 2) ? I + 2 : I + 1;  // odd padded row stride (complex)
  static constexpr int MAT = I * LD;          // complex entries per matrix
  static constexpr int NMAT = 8;
  static constexpr int NPAIR = (I + 1) / 2;  // rotations per round
  // per-bin scalars: rotation params (6 doubles x NPAIR), phases (2 x I),
  // eigenvalues (I), misc (8)
  static constexpr int NSCAL = (6 * NPAIR + 3 * I + 8 + 1) / 2 * 2;
  static constexpr int BASE16 = (NMAT * MAT * 2 + NSCAL) / 2;
  static constexpr int BIN_DOUBLES = 2 * par_stride16(I, LB, LD, BASE16);
  static constexpr size_t SMEM = (size_t)BPB * BIN_DOUBLES * sizeof(double);
};

// matrix slots
enum { kS1 = 0, kS2, kP, kX, kT, kA, kV, kInv };

template <int I>
struct BinView {
  using Lay = ParLayout<I>;
  double2* base;
  double* scal;
  FFCA_DEV double2* m(int which) const { return base + which * Lay::MAT; }
  FFCA_DEV double2& at(int which, int r, int c) const { return base[which * Lay::MAT + r * Lay::LD + c]; }
};

// group reductions over the LB lanes of one bin (lanes are contiguous)
template <int LB>
FFCA_DEV double group_sum(double x) {
#pragma unroll
  for (int o = LB / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
template <int LB>
FFCA_DEV bool group_any(bool x) {
  unsigned v = x ? 1u : 0u;
#pragma unroll
  for (int o = LB / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v != 0;
}

// round-robin (circle method) pairing for n = I (even) or I+1 (odd, with a
// dummy player): round k, pair i -> (p, q); q == I means "no rotation"
template <int I>
FFCA_DEV void rr_pair(int k, int i, int& p, int& q) {
  constexpr int n = (I % 2 == 0) ? I : I + 1;
  int a, b;
  if (i == 0) {
    a = n - 1;
    b = k;
  } else {
    a = (k + i) % (n - 1);
    b = (k - i + (n - 1)) % (n - 1);
  }
  p = a < b ? a : b;
  q = a < b ? b : a;
}

// C (row r) = A * B for an owner lane r < I (all operands in smem)
template <int I>
FFCA_DEV void row_matmul(const BinView<I>& v, int A, int B, int Cm, int r) {
  double2 out[I];
#pragma unroll
  for (int c = 0; c < I; ++c) {
    double2 acc = cmk(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < I; ++k) acc = cmac(acc, v.at(A, r, k), v.at(B, k, c));
    out[c] = acc;
  }
#pragma unroll
  for (int c = 0; c < I; ++c) v.at(Cm, r, c) = out[c];
}

// Cyclic Jacobi on the Hermitian matrix M (in place, smem) accumulating the
// eigenvectors in V (set to the identity here), round-robin ordering: in each
// round the NPAIR lanes of a bin compute the rotations of disjoint pairs,
// then row owners apply the column updates and column owners the row
// updates. Demmel-Veselic threshold; sweeps continue while any bin of the
// warp rotates. `act` predicates the bin's lanes (warp-synchronous).
// Returns false (on every lane of the warp) when kJacobiSweeps sweeps left a
// rotation pending in some bin of the warp whose `act` lanes are still rotating
// (reported by the callers as FFCA_ERR_NO_CONVERGENCE for those bins).
template <int I>
FFCA_DEV bool par_jacobi(const BinView<I>& v, int M, int V, int r, bool act) {
  using Lay = ParLayout<I>;
  if (act) {
#pragma unroll
    for (int c = 0; c < I; ++c) v.at(V, r, c) = cmk(r == c ? 1.0 : 0.0, 0.0);
  }
  __syncwarp();
  if (I == 1) return true;
  constexpr int n_rounds = (I % 2 == 0) ? I - 1 : I;
  constexpr double kTol2 = FFCA_JACOBI_TOL2;
  double* rot = v.scal;  // [NPAIR][6]: c, s, emi.x, emi.y, -, flag
  bool rotated = false;
#pragma unroll 1
  for (int sweep = 0; sweep < kJacobiSweeps; ++sweep) {
    rotated = false;
#pragma unroll 1
    for (int k = 0; k < n_rounds; ++k) {
      if (r < Lay::NPAIR) {  // identity unless this lane's pair rotates
        rot[6 * r + 0] = 1.0;
        rot[6 * r + 1] = 0.0;
        rot[6 * r + 2] = 1.0;
        rot[6 * r + 3] = 0.0;
        rot[6 * r + 5] = 0.0;
      }
      bool did = false;  // this lane's pair rotates this round
      if (act && r < Lay::NPAIR) {
        int p, q;
        rr_pair<I>(k, r, p, q);
        double* rp = rot + 6 * r;
        if (q < I) {
          const double2 apq = v.at(M, p, q);
          const double mag2 = cabs2(apq);
          const double app = v.at(M, p, p).x, aqq = v.at(M, q, q).x;
          if (mag2 > kTol2 * fabs(app * aqq) && mag2 > 0.0) {
            // MUFU seeds + Newton (as jacobi_herm)
            const double rmag = rsqrt_fast(mag2);
            const double theta = (aqq - app) * (0.5 * rmag);
            double t;
            if (fabs(theta) > 1e150) {
              t = 0.5 / theta;
            } else {
              const double h = fma(theta, theta, 1.0);
              t = rcp_fast(fabs(theta) + h * rsqrt_fast(h));
              if (theta < 0.0) t = -t;
            }
            const double c = rsqrt_fast(fma(t, t, 1.0));
            rp[0] = c;
            rp[1] = t * c;
            rp[2] = apq.x * rmag;
            rp[3] = -apq.y * rmag;
            rp[5] = 1.0;
            did = true;
          }
        }
      }
      __syncwarp();
      // a round in which no pair of any bin of the warp rotates (most rounds
      // of the late sweeps, all of the final checking sweep) skips both
      // update phases and their barriers
      if (!__any_sync(0xffffffffu, did)) continue;
      bool any = false;
      if (act) {  // column update by row owner r: M[r][p], M[r][q], V[r][p], V[r][q]
#pragma unroll
        for (int i = 0; i < Lay::NPAIR; ++i) {  // branch-free: a still pair applies the identity
          const double* rp = rot + 6 * i;
          any = any || rp[5] != 0.0;
          int p, q;
          rr_pair<I>(k, i, p, q);
          if ((I % 2) && q >= I) continue;  // the odd order's resting player
          const double c = rp[0], sn = rp[1];
          const double2 emi = cmk(rp[2], rp[3]);
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int X = w == 0 ? M : V;
            const double2 xp = v.at(X, r, p);
            const double2 xq = cmul(v.at(X, r, q), emi);
            v.at(X, r, p) = cmk(c * xp.x - sn * xq.x, c * xp.y - sn * xq.y);
            v.at(X, r, q) = cmk(sn * xp.x + c * xq.x, sn * xp.y + c * xq.y);
          }
        }
      }
      __syncwarp();
      if (act) {  // row update by column owner r: M[p][r], M[q][r]
#pragma unroll
        for (int i = 0; i < Lay::NPAIR; ++i) {
          const double* rp = rot + 6 * i;
          const bool pin = rp[5] != 0.0;
          int p, q;
          rr_pair<I>(k, i, p, q);
          if ((I % 2) && q >= I) continue;  // the odd order's resting player
          const double c = rp[0], sn = rp[1];
          const double2 epi = cmk(rp[2], -rp[3]);  // conj(emi)
          const double2 xp = v.at(M, p, r);
          const double2 xq = cmul(v.at(M, q, r), epi);
          double2 np_ = cmk(c * xp.x - sn * xq.x, c * xp.y - sn * xq.y);
          double2 nq_ = cmk(sn * xp.x + c * xq.x, sn * xp.y + c * xq.y);
          // pin the rotated 2x2 block here (its column owners are p and q):
          // off-diagonal exactly zero, diagonal exactly real
          if (pin && r == p) {
            np_.y = 0.0;
            nq_ = cmk(0.0, 0.0);
          } else if (pin && r == q) {
            np_ = cmk(0.0, 0.0);
            nq_.y = 0.0;
          }
          v.at(M, p, r) = np_;
          v.at(M, q, r) = nq_;
        }
      }
      rotated = rotated || any;
      __syncwarp();
    }
    if (act) {  // keep M exactly Hermitian (upper mirrored to lower)
      for (int c = 0; c < r; ++c) v.at(M, r, c) = cconj(v.at(M, c, r));
    }
    __syncwarp();
    if (!__any_sync(0xffffffffu, rotated)) return true;
  }
  return !group_any<Lay::LB>(rotated);  // this bin's verdict (its lanes agree)
}

// Parallel Hermitian-definite GEVD of (Phi = S1, Psi = S2) in the bin's smem.
// On exit: eigenvalues (descending) in scal[lam..], eigenvectors (phase
// pinned) in matrix kA. Returns FFCA_OK / FFCA_ERR_DEFINITENESS (min_sigma).
// Whitening by Cholesky (zhegv style) when 1/||L^-1||_F^2 certifies the
// definiteness floor; otherwise by the eigen-decomposition of Psi, exactly
// as the reference (pencil.py:113-134), which also decides definiteness.
// All lanes of the warp must call it (warp-synchronous).
template <int I>
FFCA_DEV int par_gevd(const BinView<I>& v, int r, bool own, double* min_sigma) {
  using Lay = ParLayout<I>;
  constexpr int LB = Lay::LB;
  double* lamv = v.scal + 6 * Lay::NPAIR;  // I
  double* phv = lamv + I;                   // 2 I (phases; also isq in path B)
  double* misc = phv + 2 * I;               // 8
  double tr = 0.0;
  for (int a = 0; a < I; ++a) tr += v.at(kS2, a, a).x;
  const double thr = kDefFloor * tr / I;
  // ---- Cholesky of Psi (lower) into kX, column-sequential ----
  bool chol_ok = true;
#pragma unroll 1
  for (int j = 0; j < I; ++j) {
    if (own && r == j) {
      double d = v.at(kS2, j, j).x;
      for (int k = 0; k < j; ++k) d -= cabs2(v.at(kX, j, k));
      misc[0] = d;
      misc[1] = rsqrt_fast(fmax(d, 0.0));  // 1 / L_jj (MUFU seed + Newton)
      v.at(kX, j, j) = cmk(fmax(d, 0.0) * misc[1], 0.0);
    }
    __syncwarp();
    chol_ok = chol_ok && (misc[0] > 0.0);
    if (own && r > j) {
      double2 sacc = v.at(kS2, r, j);
      for (int k = 0; k < j; ++k) sacc = cmsubc(sacc, v.at(kX, r, k), v.at(kX, j, k));
      v.at(kX, r, j) = cscale(sacc, misc[1]);
    }
    if (own && r < j) v.at(kX, r, j) = cmk(0.0, 0.0);
    __syncwarp();
  }
  // ---- Li = L^{-1} into kT, column-parallel (lane r owns column r) ----
  double fro = 0.0;
  if (own) {
    const int c = r;
#pragma unroll 1
    for (int rr = 0; rr < I; ++rr) {
      if (rr < c) {
        v.at(kT, rr, c) = cmk(0.0, 0.0);
        continue;
      }
      double2 sacc = cmk(rr == c ? 1.0 : 0.0, 0.0);
      for (int k = c; k < rr; ++k) sacc = cmsub(sacc, v.at(kX, rr, k), v.at(kT, k, c));
      const double2 val = cscale(sacc, rcp_fast(v.at(kX, rr, rr).x));
      v.at(kT, rr, c) = val;
      fro += cabs2(val);
    }
  }
  fro = group_sum<LB>(fro);
  const bool fb = !(chol_ok && (1.0 / fro) > thr);  // uniform over the bin's lanes
  __syncwarp();
  int rc = FFCA_OK;
  double smin = 0.0;
  if (!fb && own) {
    // ---- path A: Wh = Li Phi Li^H -> kS2; B = Li^H -> kX ----
    for (int c = 0; c < I; ++c) {  // kA row r = Li row r * Phi
      double2 acc = cmk(0.0, 0.0);
      for (int k = 0; k <= r; ++k) acc = cmac(acc, v.at(kT, r, k), v.at(kS1, k, c));
      v.at(kA, r, c) = acc;
    }
  }
  __syncwarp();
  if (!fb && own) {
    for (int c = r; c < I; ++c) {  // upper of row r: sum_k A[r][k] conj(Li[c][k])
      double2 acc = cmk(0.0, 0.0);
      for (int k = 0; k <= c; ++k) acc = cadd(acc, cmulc(v.at(kA, r, k), v.at(kT, c, k)));
      if (c == r) acc.y = 0.0;
      v.at(kS2, r, c) = acc;
    }
    for (int c = 0; c < I; ++c) v.at(kX, r, c) = c >= r ? cconj(v.at(kT, c, r)) : cmk(0.0, 0.0);
  }
  __syncwarp();
  if (!fb && own)
    for (int c = 0; c < r; ++c) v.at(kS2, r, c) = cconj(v.at(kS2, c, r));
  __syncwarp();
  if (__any_sync(0xffffffffu, fb)) {
    // ---- path B (rare): eig(Psi) = U diag(sig) U^H decides definiteness ----
    if (fb && own)
      for (int c = 0; c < I; ++c) v.at(kA, r, c) = v.at(kS2, r, c);
    __syncwarp();
    const bool conv_b = par_jacobi<I>(v, kA, kV, r, fb && own);
    smin = 1e308;
    for (int a = 0; a < I; ++a) smin = fmin(smin, v.at(kA, a, a).x);
    if (fb && !conv_b) rc = FFCA_ERR_NO_CONVERGENCE;
    else if (fb && !(smin > thr)) rc = FFCA_ERR_DEFINITENESS;
    const bool go = fb && own && rc == FFCA_OK;
    if (go) {  // B = U diag(sig^-1/2) -> kX
      for (int c = 0; c < I; ++c) v.at(kX, r, c) = cscale(v.at(kV, r, c), 1.0 / sqrt(v.at(kA, c, c).x));
    }
    __syncwarp();
    if (go) {  // kT = Phi B
      for (int c = 0; c < I; ++c) {
        double2 acc = cmk(0.0, 0.0);
        for (int k = 0; k < I; ++k) acc = cmac(acc, v.at(kS1, r, k), v.at(kX, k, c));
        v.at(kT, r, c) = acc;
      }
    }
    __syncwarp();
    if (go) {  // Wh = B^H (Phi B), re-symmetrised from the upper triangle
      for (int c = r; c < I; ++c) {
        double2 acc = cmk(0.0, 0.0);
        for (int k = 0; k < I; ++k) acc = cmac_cj(acc, v.at(kX, k, r), v.at(kT, k, c));
        if (c == r) acc.y = 0.0;
        v.at(kS2, r, c) = acc;
      }
    }
    __syncwarp();
    if (go)
      for (int c = 0; c < r; ++c) v.at(kS2, r, c) = cconj(v.at(kS2, c, r));
    __syncwarp();
  }
  const bool act = own && rc == FFCA_OK;
  // ---- eig(Wh): Jacobi into kV ----
  if (!par_jacobi<I>(v, kS2, kV, r, act) && act) rc = FFCA_ERR_NO_CONVERGENCE;
  // ---- sort descending: Qs[r][rank(c)] = V[r][c] (kX free? no: B) -> use kA as staging ----
  if (act) {
    for (int c = 0; c < I; ++c) v.at(kA, r, c) = v.at(kV, r, c);
  }
  __syncwarp();
  if (act) {
    for (int c = 0; c < I; ++c) {
      const double lc = v.at(kS2, c, c).x;
      int rk = 0;
      for (int k = 0; k < I; ++k) {
        const double lk = v.at(kS2, k, k).x;
        rk += (lk > lc) || (lk == lc && k < c);
      }
      v.at(kV, r, rk) = v.at(kA, r, c);
      if (r == 0) lamv[rk] = lc;
    }
  }
  __syncwarp();
  // ---- P_gevd = B Qs -> kA ----
  if (act) {
    for (int c = 0; c < I; ++c) {
      double2 acc = cmk(0.0, 0.0);
      for (int k = 0; k < I; ++k) acc = cmac(acc, v.at(kX, r, k), v.at(kV, k, c));
      v.at(kA, r, c) = acc;
    }
  }
  __syncwarp();
  // ---- column phases: lane c pins its column's largest entry real positive ----
  if (act) {
    const int c = r;
    double best = cabs2(v.at(kA, 0, c));
    double2 lead = v.at(kA, 0, c);
    for (int i = 1; i < I; ++i) {
      const double mm = cabs2(v.at(kA, i, c));
      if (mm > best) {
        best = mm;
        lead = v.at(kA, i, c);
      }
    }
    const double mag = sqrt(best);
    phv[2 * c] = mag > 0.0 ? lead.x / mag : 1.0;
    phv[2 * c + 1] = mag > 0.0 ? -lead.y / mag : 0.0;
  }
  __syncwarp();
  if (act) {
    for (int c = 0; c < I; ++c) v.at(kA, r, c) = cmul(v.at(kA, r, c), cmk(phv[2 * c], phv[2 * c + 1]));
  }
  __syncwarp();
  *min_sigma = smin;
  return rc;
}

// Gauss-Jordan inverse of matrix Msrc (copied to kX) into kInv, row-parallel;
// returns log|det| on all lanes; *ok false on a zero / non-finite pivot.
template <int I>
FFCA_DEV double par_lu_inverse(const BinView<I>& v, int Msrc, int r, bool own, bool* ok) {
  using Lay = ParLayout<I>;
  constexpr int LB = Lay::LB;
  double* misc = v.scal + 6 * Lay::NPAIR + 3 * I;
  if (own) {
#pragma unroll
    for (int c = 0; c < I; ++c) {
      v.at(kX, r, c) = v.at(Msrc, r, c);
      v.at(kInv, r, c) = cmk(r == c ? 1.0 : 0.0, 0.0);
    }
  }
  __syncwarp();
  double lad = 0.0;
  bool good = true;
#pragma unroll 1
  for (int k = 0; k < I; ++k) {
    // pivot: argmax |M[i][k]|^2 over i >= k (first maximum)
    double mv = (own && r >= k) ? cabs2(v.at(kX, r, k)) : -1.0;
    int mi = r;
#pragma unroll
    for (int o = LB / 2; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, mv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      if (ov > mv || (ov == mv && oi < mi)) {
        mv = ov;
        mi = oi;
      }
    }
    const int pr = mi;
    const double best = mv;
    good = good && (best > 0.0) && isfinite(best);
    lad += 0.5 * log(best);
    // swap rows k and pr (both M and Inv)
    double2 rowM[I], rowI[I];
    const int src = (r == k) ? pr : ((r == pr) ? k : r);
    if (own) {
#pragma unroll
      for (int c = 0; c < I; ++c) {
        rowM[c] = v.at(kX, src, c);
        rowI[c] = v.at(kInv, src, c);
      }
    }
    __syncwarp();
    if (own) {
#pragma unroll
      for (int c = 0; c < I; ++c) {
        v.at(kX, r, c) = rowM[c];
        v.at(kInv, r, c) = rowI[c];
      }
    }
    __syncwarp();
    if (own && r == k) {
      const double2 pv = v.at(kX, k, k);  // 1 / pv = conj(pv) / |pv|^2
      const double ib = rcp_fast(cabs2(pv));
      const double2 ip = cmk(pv.x * ib, -pv.y * ib);
#pragma unroll
      for (int c = 0; c < I; ++c) {
        v.at(kX, k, c) = cmul(v.at(kX, k, c), ip);
        v.at(kInv, k, c) = cmul(v.at(kInv, k, c), ip);
      }
    }
    __syncwarp();
    if (own && r != k) {
      const double2 fct = v.at(kX, r, k);
#pragma unroll
      for (int c = 0; c < I; ++c) {
        v.at(kX, r, c) = csub(v.at(kX, r, c), cmul(fct, v.at(kX, k, c)));
        v.at(kInv, r, c) = csub(v.at(kInv, r, c), cmul(fct, v.at(kInv, k, c)));
      }
    }
    __syncwarp();
  }
  (void)misc;
  *ok = good;
  return lad;
}

}  // namespace ffca
