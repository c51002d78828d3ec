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

#include <type_traits>

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

#ifndef FFCA_RCP_BATCH
#define FFCA_RCP_BATCH 0  // measured slower on config 3 (longer dependent chain)
#endif
#ifndef FFCA_RCP_NR
#define FFCA_RCP_NR 1  // Newton steps after rcp.approx.f64 in the streaming pass (1: ~1e-14 rel.)
#endif
// reciprocal for the streaming pass: MUFU.RCP64H seed + FFCA_RCP_NR Newton steps
FFCA_DEV double rcp_pass(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
  for (int i = 0; i < FFCA_RCP_NR; ++i) {
    const double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
  }
  return r;
}
// r[a] = 1 / d[a] for all a with ONE reciprocal (Montgomery's trick:
// prefix products, one rcp, back-substitution; ~2 ulp), falling back to
// per-element reciprocals when the product leaves the safe exponent range
template <int I>
FFCA_DEV void rcp_batch(const double (&d)[I], double (&r)[I]) {
  if constexpr (I == 1 || !FFCA_RCP_BATCH) {
#pragma unroll
    for (int a = 0; a < I; ++a) r[a] = rcp_pass(d[a]);
  } else {
    double pre[I];
    pre[0] = d[0];
#pragma unroll
    for (int a = 1; a < I; ++a) pre[a] = pre[a - 1] * d[a];
    const double all = pre[I - 1];
    if (all > 1e-280 && all < 1e280) {
      double inv = rcp_nr(all);
#pragma unroll
      for (int a = I - 1; a > 0; --a) {
        r[a] = inv * pre[a - 1];
        inv = inv * d[a];
      }
      r[0] = inv;
    } else {
#pragma unroll
      for (int a = 0; a < I; ++a) r[a] = rcp_nr(d[a]);
    }
  }
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

// ---- TMA bulk copies + mbarrier (sm_90+; the frame ring of the update pass) ----
FFCA_DEV unsigned smem_u32(const void* ptr) { return (unsigned)__cvta_generic_to_shared(ptr); }
FFCA_DEV void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
FFCA_DEV void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
FFCA_DEV void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
FFCA_DEV bool mbar_try_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
FFCA_DEV void mbar_wait(unsigned bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy completing on `bar` (16-B aligned, size % 16 == 0)
FFCA_DEV void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// order this thread's earlier generic-proxy shared-memory accesses before
// later async-proxy (bulk copy) writes to the same memory
FFCA_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Compute precision follows the streaming precision: complex128 runs the
// per-point math in FP64; complex64 runs it in FP32 (B200's 2x-wider FP32
// pipe) with FP64 per-bin state and FP64 accumulators fed by FP32 partial
// sums over blocks of kF32Block frames (fp32 streaming with
// fp64 per-bin accumulation reaches ~1e-6 of the complex128 oracle; the
// complex64 tolerance is 1e-4).
constexpr int kF32Block = 16;
template <typename R>
struct Math;
template <>
struct Math<double> {
  using T = double;
  using T2 = double2;
  static constexpr bool kBlocked = false;
  static FFCA_DEV double rcp(double x) { return rcp_nr(x); }
  template <int I>
  static FFCA_DEV void rcp_n(const double (&d)[I], double (&r)[I]) { rcp_batch<I>(d, r); }
  static FFCA_DEV double2 c2(double2 a) { return a; }
};
template <>
struct Math<float> {
  using T = float;
  using T2 = float2;
  static constexpr bool kBlocked = true;
  static FFCA_DEV float rcp(float x) { return __frcp_rn(x); }
  template <int I>
  static FFCA_DEV void rcp_n(const float (&d)[I], float (&r)[I]) {
#pragma unroll
    for (int a = 0; a < I; ++a) r[a] = __frcp_rn(d[a]);
  }
  static FFCA_DEV float2 c2(double2 a) { return make_float2((float)a.x, (float)a.y); }
};

// One ring stage of one warp = one frame of its 32 bins: the frame's y row
// of the 32 bins (32 * YB contiguous bytes in HBM) in Q units of UB bytes
// per bin, then v1[32] and v2[32]. The warp copies it cooperatively: copy c
// of lane l moves unit u = 32 c + l of the row, so every cp.async instruction
// reads one contiguous 32*UB-byte run of HBM (full sectors) and writes a
// contiguous run of shared memory; a bin's Q units are rotated by a
// bin-dependent amount (sw) so that the consumer reads (lane = bin, one unit
// each) hit distinct banks. (Per-lane 80-byte slots made every 16-B cp.async
// a ~30-way bank conflict and read half-used sectors.)
// ---- packed FP32 (sm_100 FFMA2 / FMUL2 / FADD2) ------------------------------
// Two FP32 lanes per instruction; ptxas folds scalar broadcasts, half swaps
// and half negations of the operands into operand modifiers (checked in
// SASS), so (a.x, a.x) or (a.y, -a.x) cost no moves. Used by the complex64
// pass at even orders, which is issue-bound in scalar FP32.
namespace f2 {
FFCA_DEV unsigned long long pk(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
FFCA_DEV float2 up(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
FFCA_DEV float2 fma(float2 a, float2 b, float2 c) {  // a * b + c
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return up(r);
}
FFCA_DEV float2 mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return up(r);
}
FFCA_DEV float2 add(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return up(r);
}
FFCA_DEV float2 bc(float a) { return make_float2(a, a); }
FFCA_DEV float rcp(float x) {  // MUFU.RCP (~1 ulp), no IEEE slow path
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
}  // namespace f2

template <int I, typename R>
struct RingSlot {
  using C = typename CplxOf<R>::type;
  static constexpr int YB = I * (int)sizeof(C);
  static constexpr int VB = (int)sizeof(R);
  static constexpr int UB = (YB % 16 == 0) ? 16 : 8;  // unit bytes
  static constexpr int Q = YB / UB;                   // units per bin
  static constexpr int WARP_BYTES = 32 * (YB + 2 * VB);
  static_assert(WARP_BYTES % 16 == 0, "stage alignment");
  // unit a of bin b sits at unit Q b + (a ^ sw(b)): for a power-of-two Q the
  // xor spreads the 8 (UB = 16) or 16 (UB = 8) consecutive bins that read
  // the same a over distinct banks; an odd Q needs no swizzle. Copy c of lane
  // l (unit 32 c + l) then lands at pos(first unit) + 32 c UB, and the reads
  // of bin b are at rbase(b) ^ (a UB) (Q even) or rbase(b) + a UB (Q odd).
  static constexpr bool kXor = UB == 16 && Q % 2 == 0;
  static FFCA_DEV constexpr int sw(int b) { return kXor ? (b * Q / 8) % Q : 0; }
  static FFCA_DEV constexpr int pos(int b, int a) { return (Q * b + (a ^ sw(b))) * UB; }
  static FFCA_DEV constexpr int rbase(int b) { return (Q * b + sw(b)) * UB; }
  static FFCA_DEV constexpr int rpos(int rb, int a) { return kXor ? (rb ^ (a * UB)) : rb + a * UB; }
};

// TMA ring stage of one warp (update pass, complex128): the frame's y row of
// the warp's 32 bins copied by ONE elected lane with cp.async.bulk (one copy,
// or two when the tile crosses into the next mixture) and v1, v2 as 16-B
// aligned supersets of their runs (a frame row of v is only 8-B aligned when
// F is odd). The row lands linearly (bin b at b*YB); lanes read their Q units
// in the rotated order (k + sw(b)) mod Q — the RingSlot swizzle moved from the
// write side to the read side, undone by storing P's rows in the same
// rotation — so the reads stay bank-conflict free.
template <int I, typename R>
struct BulkSlot {
  using RS = RingSlot<I, R>;
  static constexpr int YB = RS::YB, VB = RS::VB, Q = RS::Q;
  static constexpr int VA = ((32 * VB + 64) + 15) / 16 * 16;  // v run + alignment slack, 2 runs
  static constexpr int WARP_BYTES = 32 * YB + 2 * VA;
  static constexpr bool kOk = (YB % 16 == 0) && VB == 8;  // complex128
};

// The RingSlot scheme as a reusable object (used by the FCA pass, K4): a
// warp's frames n = nfirst + k * WARPS stream through a STAGES-deep ring at
// `base` (STAGES * WARPS * WARP_BYTES bytes per CTA). Same copies, swizzle and
// synchronisation as fast_em2_kernel's inline ring.
template <int I, typename R, int WARPS, int STAGES>
struct FrameRing {
  using Slot = RingSlot<I, R>;
  using C = typename CplxOf<R>::type;
  static constexpr int kStride = WARPS * Slot::WARP_BYTES;
  static constexpr size_t BYTES = (size_t)STAGES * kStride;
  unsigned char* wslots;
  const unsigned char* ynext;  // row of the next frame to issue (frames go in order)
  const R* vnext;
  int64_t ystep, vstep, NF;
  int64_t ycorr[Slot::Q];
  int spos0, rb, lane, issue_stage, read_stage;
  bool contiguous;

  FFCA_DEV void init(unsigned char* base, int warp, int lane_, int64_t tile0, int64_t G,
                     int64_t N, int64_t F, const void* y, const R* vrow, int64_t nfirst) {
    lane = lane_;
    wslots = base + (size_t)warp * Slot::WARP_BYTES;
    contiguous = (tile0 + 31 < G) && ((unsigned)tile0 / (unsigned)F == (unsigned)(tile0 + 31) / (unsigned)F);
    spos0 = Slot::pos(lane / Slot::Q, lane % Slot::Q);
    rb = Slot::rbase(lane);
    auto unit_off = [&](int c) -> int64_t {
      const int u = 32 * c + lane, b = u / Slot::Q, a = u % Slot::Q;
      int64_t gb = tile0 + b;
      if (gb >= G) gb = G - 1;
      const int64_t mb = (unsigned)gb / (unsigned)F, fb = gb - mb * F;
      return ((mb * N) * F + fb) * Slot::YB + a * Slot::UB;
    };
    const int64_t ybase = unit_off(0);
#pragma unroll
    for (int c = 0; c < Slot::Q; ++c)
      ycorr[c] = contiguous ? 0 : unit_off(c) - ybase - 32 * c * Slot::UB;
    ynext = (const unsigned char*)y + ybase + nfirst * F * Slot::YB;
    ystep = (int64_t)WARPS * F * Slot::YB;
    vnext = vrow + nfirst * F;
    vstep = (int64_t)WARPS * F;
    NF = N * F;
    issue_stage = read_stage = 0;
  }
  FFCA_DEV void issue() {  // the next frame of this warp
    unsigned char* slot = wslots + issue_stage;
    issue_stage = issue_stage + kStride == STAGES * kStride ? 0 : issue_stage + kStride;
    const unsigned char* yrow = ynext;
    ynext += ystep;
    unsigned char* dst = slot + spos0;
#pragma unroll
    for (int c = 0; c < Slot::Q; ++c) {
      const unsigned char* src = yrow + 32 * c * Slot::UB + (contiguous ? 0 : ycorr[c]);
      if constexpr (Slot::UB == 16)
        cp_async16(dst + 32 * c * Slot::UB, src);
      else
        cp_async8(dst + 32 * c * Slot::UB, src);
    }
    unsigned char* vs = slot + 32 * Slot::YB;
    if constexpr (sizeof(R) == 8) {
      cp_async8(vs + 8 * lane, vnext);
      cp_async8(vs + 256 + 8 * lane, vnext + NF);
    } else {
      cp_async4(vs + 4 * lane, vnext);
      cp_async4(vs + 128 + 4 * lane, vnext + NF);
    }
    vnext += vstep;
  }
  // this lane's bin of the next stage, widened to complex128 / float64
  unsigned char* cur = nullptr;  // stage of the frame last loaded (free until the next issue)
  FFCA_DEV void load(double2 (&yv)[I], double& v1, double& v2) {
    const unsigned char* slot = wslots + read_stage;
    cur = wslots + read_stage;
    read_stage = read_stage + kStride == STAGES * kStride ? 0 : read_stage + kStride;
    constexpr int PER = Slot::UB / (int)sizeof(C);
#pragma unroll
    for (int a = 0; a < Slot::Q; ++a) {
      const unsigned char* src = slot + Slot::rpos(rb, a);
      if constexpr (PER == 2) {
        const float4 q = *(const float4*)src;
        yv[2 * a] = cmk(q.x, q.y);
        yv[2 * a + 1] = cmk(q.z, q.w);
      } else {
        yv[a] = to_c128(*(const C*)src);
      }
    }
    const unsigned char* vs = slot + 32 * Slot::YB;
    v1 = (double)((const R*)vs)[lane];
    v2 = (double)((const R*)(vs + 32 * sizeof(R)))[lane];
  }
  // the same in two steps (K4: the observation is not needed, and not kept
  // in registers, while R is inverted): powers first, y from `cur` later
  FFCA_DEV void load_v(double& v1, double& v2) {
    cur = wslots + read_stage;
    read_stage = read_stage + kStride == STAGES * kStride ? 0 : read_stage + kStride;
    const unsigned char* vs = cur + 32 * Slot::YB;
    v1 = (double)((const R*)vs)[lane];
    v2 = (double)((const R*)(vs + 32 * sizeof(R)))[lane];
  }
  FFCA_DEV void load_y(double2 (&yv)[I]) const {
    constexpr int PER = Slot::UB / (int)sizeof(C);
#pragma unroll
    for (int a = 0; a < Slot::Q; ++a) {
      const unsigned char* src = cur + Slot::rpos(rb, a);
      if constexpr (PER == 2) {
        const float4 q = *(const float4*)src;
        yv[2 * a] = cmk(q.x, q.y);
        yv[2 * a + 1] = cmk(q.z, q.w);
      } else {
        yv[a] = to_c128(*(const C*)src);
      }
    }
  }
};

// Warp-cooperative store of one frame's posterior means (images) of the
// warp's 32 bins, (M,2,N,F,I) layout, through a ring stage the warp has
// consumed (free until the next issue refills it): every lane puts its bin's
// row in the ring's swizzled slot layout, then copy c of lane l stores unit
// 32 c + l of the 32-bin row — one contiguous 32*UB-byte run per store
// instruction instead of a lane stride of I*sizeof(C) bytes, which writes
// half sectors (2x the L2 store traffic of the image pass; ncu: 50% of the
// image pass's global store sectors excessive).
template <int I, typename R>
struct ImageRowStore {
  using Slot = RingSlot<I, R>;
  using C = typename CplxOf<R>::type;
  int64_t row0;              // byte offset of tile0's row at source 0, frame 0
  int64_t corr[Slot::Q];     // per-copy correction of a tile across a mixture boundary
  bool valid[Slot::Q];       // the copy's bin exists
  int64_t NF, F;
  int spos0, lane;
  bool contiguous;

  FFCA_DEV void init(int64_t tile0, int64_t G, int64_t N, int64_t F_, int lane_) {
    lane = lane_;
    F = F_;
    NF = N * F_;
    contiguous = (tile0 + 31 < G) && ((unsigned)tile0 / (unsigned)F_ == (unsigned)(tile0 + 31) / (unsigned)F_);
    spos0 = Slot::pos(lane / Slot::Q, lane % Slot::Q);
    const int64_t m0 = (unsigned)tile0 / (unsigned)F_, f0 = tile0 - m0 * F_;
    row0 = (m0 * 2 * NF + f0) * Slot::YB;
#pragma unroll
    for (int c = 0; c < Slot::Q; ++c) {
      const int u = 32 * c + lane, b = u / Slot::Q, a = u % Slot::Q;
      int64_t gb = tile0 + b;
      valid[c] = gb < G;
      if (gb >= G) gb = G - 1;
      const int64_t mb = (unsigned)gb / (unsigned)F_, fb = gb - mb * F_;
      corr[c] = contiguous ? 0 : (mb * 2 * NF + fb) * Slot::YB + a * Slot::UB - row0 -
                                     (int64_t)u * Slot::UB;
    }
  }
  // o[j][a]: source j, channel a of this lane's bin at frame n; `slot` the
  // consumed stage. Warp-synchronous (all lanes call it).
  template <typename CC>
  FFCA_DEV void store(void* mu_out, unsigned char* slot, int64_t n, const CC (&o)[2][I]) const {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      __syncwarp();  // (j = 0: every lane read the stage; j = 1: source 1 stored)
#pragma unroll
      for (int a = 0; a < Slot::Q; ++a) {
        unsigned char* d = slot + Slot::pos(lane, a);
        if constexpr (sizeof(C) == 16)
          *(double2*)d = make_double2((double)o[j][a].x, (double)o[j][a].y);
        else if constexpr (Slot::UB == 16)
          *(float4*)d = make_float4((float)o[j][2 * a].x, (float)o[j][2 * a].y,
                                    (float)o[j][2 * a + 1].x, (float)o[j][2 * a + 1].y);
        else
          *(float2*)d = make_float2((float)o[j][a].x, (float)o[j][a].y);
      }
      __syncwarp();
      unsigned char* row = (unsigned char*)mu_out + row0 + (j * NF + n * F) * Slot::YB;
#pragma unroll
      for (int c = 0; c < Slot::Q; ++c) {
        if (!valid[c]) continue;
        unsigned char* dst = row + (32 * c + lane) * Slot::UB + (contiguous ? 0 : corr[c]);
        const unsigned char* src = slot + spos0 + 32 * c * Slot::UB;
        if constexpr (Slot::UB == 16)
          *(uint4*)dst = *(const uint4*)src;
        else
          *(uint2*)dst = *(const uint2*)src;
      }
    }
  }
};

// complex64 update pass at even orders: its FP64 S~ accumulators live in
// shared memory (fed every kF32Block frames from the packed FP32 block sums),
// which frees 64 registers for a 4th CTA per SM (the pass is issue-bound)
template <int I, typename R, bool UPDATE, bool LL, bool MU>
struct SmemAcc {
  static constexpr bool value = std::is_same<R, float>::value && (I % 2 == 0) && UPDATE && !LL && !MU;
};

template <int I, typename R, int WARPS, int STAGES, bool MU = false, bool SACC = false,
          bool BULK = false>
struct Fast2Smem {
  static constexpr int NE = 2 * I * I + 1;
  static constexpr size_t RING =
      (size_t)STAGES * WARPS * (BULK ? BulkSlot<I, R>::WARP_BYTES : RingSlot<I, R>::WARP_BYTES);
  static constexpr size_t RED = (size_t)(WARPS - 1) * NE * 32 * sizeof(double);
  // P tile, rows of kTileStride (33) entries: the coalesced copy (consecutive
  // threads = consecutive entries of one bin) then hits distinct banks
  static constexpr size_t PB = (size_t)I * I * 33 * sizeof(typename Math<R>::T2);
  static constexpr size_t WB = MU ? PB : 0;                           // W tile, after P
  static constexpr size_t ACC = SACC ? (size_t)2 * I * I * WARPS * 32 * sizeof(double) : 0;
  static constexpr size_t BARS = BULK ? (size_t)STAGES * WARPS * 8 : 0;  // one mbarrier per stage
  static constexpr size_t MAIN = RING + PB + WB + ACC + BARS;  // accumulators after the tiles
  static constexpr size_t BYTES = MAIN > RED ? MAIN : RED;
};

#ifndef FFCA_K3_RING_FIRST
#define FFCA_K3_RING_FIRST 0  // 1: issue the frame ring before loading the P tile
#endif
#ifndef FFCA_K3_PCOAL
#define FFCA_K3_PCOAL 1  // coalesced copy of the tile's P / W blocks into shared memory
#endif
#ifndef FAST2_MINB
#define FAST2_MINB 3  // CTAs per SM the update pass is register-budgeted for
#endif
#ifndef FAST2_MU_STAGES
#define FAST2_MU_STAGES 6  // ring depth of the image-writing (last) pass
#endif
#ifndef FAST2_MU_MINB
#define FAST2_MU_MINB 2  // CTAs per SM the image-writing pass is budgeted for
#endif
#ifndef FAST2_STAGES
#define FAST2_STAGES 6  // cp.async ring depth (frames per thread)
#endif
#ifndef FAST2_UNROLL
#define FAST2_UNROLL 1  // frames per loop trip (ILP experiments)
#endif
#ifndef FAST2_SACC_STAGES
#define FAST2_SACC_STAGES 3  // ring depth of the complex64 pass with shared accumulators
#endif
template <int I, typename R, bool UPDATE, bool LL, bool MU>
constexpr int fast2_stages() {
  return MU ? FAST2_MU_STAGES : (SmemAcc<I, R, UPDATE, LL, MU>::value ? FAST2_SACC_STAGES : FAST2_STAGES);
}
template <int I, typename R, bool UPDATE, bool LL, bool MU>
constexpr int fast2_minb() {
  return MU ? FAST2_MU_MINB : (SmemAcc<I, R, UPDATE, LL, MU>::value ? 4 : FAST2_MINB);
}

// 16-byte L2 (cache-global) load of a complex128
__device__ __forceinline__ double2 ldcg2(const double2* p) { return __ldcg(p); }

// The pass of one CTA: bin tile `bx` of the launch window, frame chunk `by`.
// A device function so that the persistent EM kernel (ffca_persist.cuh) runs
// the same code for every iteration of a resident (tile, chunk). The per-bin
// state another CTA may have rewritten during the same kernel (P, W, lambda)
// is read with L2 loads (__ldcg), never through L1.
struct NoPreTile {  // (nothing to wait for)
  __device__ __forceinline__ bool operator()() const { return true; }
};
// stand-alone pass: with `on` (FastIterParams::pdl_wait) wait for the kernel
// this launch programmatically depends on, then release the next one
struct PdlGate {
  bool on;
  __device__ __forceinline__ bool operator()() const {
    if (on) {
      pdl_wait_primary();
      pdl_release_dependents();
    }
    return true;
  }
};
// `pre` (persistent kernel): called once the frame ring's first stages are in
// flight and before any per-bin state (P, W, lambda) is read — the wait for
// the tile's pencil refresh, overlapped with the y / v prefetch; false = the
// run was aborted (the CTA drains its copies and returns).
template <int I, typename R, int WARPS, int STAGES, bool UPDATE, bool LL, bool MU,
          bool BULK = false, class PreTile = NoPreTile>
__device__ __forceinline__ void fast_em2_body(const FastIterParams& p, const unsigned bx,
                                              const unsigned by, PreTile pre = PreTile()) {
  constexpr bool kRingFirst = FFCA_K3_RING_FIRST || !std::is_same<PreTile, NoPreTile>::value;
  using C = typename CplxOf<R>::type;
  using Slot = RingSlot<I, R>;
  using T = typename Math<R>::T;    // per-point compute type
  using T2 = typename Math<R>::T2;
  constexpr bool kBlk = Math<R>::kBlocked;
  // complex64 at even orders: the per-point math in packed FP32 (f2::)
  constexpr bool kF2 = kBlk && (I % 2 == 0);
  constexpr int NP = I * I;
  constexpr int NE = 2 * NP + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t G = p.G;
  const int64_t tile0 = p.g0 + (int64_t)bx * 32;  // (window edges are tile edges)
  int64_t g = tile0 + lane;
  const bool active = g < G;
  if (!active) g = G - 1;
  const int64_t m = g / p.F;
  const int64_t f = g - m * p.F;
  const int64_t n0 = (int64_t)by * p.chunk_frames;
  const int64_t n1 = min(p.N, n0 + p.chunk_frames);
  const int64_t NF = p.N * p.F;
  R* vb = (R*)p.v + m * 2 * NF + f;  // no __restrict__: may alias vr (in place)
  const R* vr = (p.v_src ? (const R*)p.v_src : (const R*)p.v) + m * 2 * NF + f;
  constexpr bool kSacc = SmemAcc<I, R, UPDATE, LL, MU>::value;
  using Sm = Fast2Smem<I, R, WARPS, STAGES, MU, kSacc, BULK>;
  using BS = BulkSlot<I, R>;
  static_assert(!BULK || (BS::kOk && UPDATE && !LL && !MU), "bulk ring: complex128 update pass");

  double acc[2][kSacc ? 1 : NP];  // (kSacc: in shared memory, accS)
  // accS[(j NP + e) * WARPS * 32 + tid]: thread-minor, conflict-free
  double* accS = (double*)(smem_raw + Sm::RING + Sm::PB + Sm::WB) + threadIdx.x;
  constexpr int kAccStride = WARPS * 32;
  if constexpr (kSacc) {
#pragma unroll
    for (int e = 0; e < 2 * NP; ++e) accS[e * kAccStride] = 0.0;
  }
  T accb[2][kBlk ? NP : 1];  // FP32 block sums (complex64 only)
#pragma unroll
  for (int j = 0; j < 2; ++j) {
#pragma unroll
    for (int e = 0; e < (kSacc ? 1 : NP); ++e) acc[j][e] = 0.0;
#pragma unroll
    for (int e = 0; e < (kBlk ? NP : 1); ++e) accb[j][e] = T(0);
  }
  float2 acc2[2][kF2 ? NP / 2 : 1];  // packed FP32 block sums (kF2): entries (2i, 2i+1)
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < (kF2 ? NP / 2 : 1); ++e) acc2[j][e] = make_float2(0.f, 0.f);
  auto accum = [&](int j, int e, T a, T b) {  // acc[j][e] += a * b
    if constexpr (kBlk)
      accb[j][e] = fma(a, b, accb[j][e]);
    else
      acc[j][e] = fma((double)a, (double)b, acc[j][e]);
  };
  auto flush = [&]() {
    if constexpr (kSacc) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < NP / 2; ++e) {
          accS[(j * NP + 2 * e) * kAccStride] += (double)acc2[j][e].x;
          accS[(j * NP + 2 * e + 1) * kAccStride] += (double)acc2[j][e].y;
          acc2[j][e] = make_float2(0.f, 0.f);
        }
    } else if constexpr (kF2) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < NP / 2; ++e) {
          acc[j][2 * e] += (double)acc2[j][e].x;
          acc[j][2 * e + 1] += (double)acc2[j][e].y;
          acc2[j][e] = make_float2(0.f, 0.f);
        }
    } else if constexpr (kBlk) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < NP; ++e) {
          acc[j][e] += (double)accb[j][e];
          accb[j][e] = T(0);
        }
    }
  };
  double llacc = 0.0;
  int64_t bad_n = 0;

  unsigned char* wslots = smem_raw + (size_t)warp * Slot::WARP_BYTES;
  constexpr size_t kStageStride = (size_t)WARPS * Slot::WARP_BYTES;
  const int64_t nfirst = n0 + warp;
  const int K = nfirst < n1 ? (int)((n1 - nfirst + WARPS - 1) / WARPS) : 0;
  // this lane's share of the warp's row copies: unit u = 32 c + lane belongs
  // to bin b = u / Q of the tile (clamped like g), unit a = u % Q. When the
  // tile's 32 bins lie in one mixture (and none is clamped) the row is one
  // contiguous run and copy c reads ybase + 32 c UB; a tile across a mixture
  // boundary (or the last, partial tile) adds a per-copy correction.
  const bool contiguous = (tile0 + 31 < G) && (tile0 / p.F == (tile0 + 31) / p.F);
  const int spos0 = Slot::pos(lane / Slot::Q, lane % Slot::Q);
  const int rb = Slot::rbase(lane);
  auto unit_off = [&](int c) -> int64_t {  // byte offset (frame 0) of copy c
    const int u = 32 * c + lane, b = u / Slot::Q, a = u % Slot::Q;
    int64_t gb = tile0 + b;
    if (gb >= G) gb = G - 1;
    const int64_t mb = gb / p.F, fb = gb - mb * p.F;
    return ((mb * p.N) * p.F + fb) * Slot::YB + a * Slot::UB;
  };
  const int64_t ybase = unit_off(0);
  int64_t ycorr[Slot::Q];  // unit_off(c) - ybase - 32 c UB (non-contiguous tiles)
#pragma unroll
  for (int c = 0; c < Slot::Q; ++c)
    ycorr[c] = contiguous ? 0 : unit_off(c) - ybase - 32 * c * Slot::UB;
  const unsigned char* ybytes = (const unsigned char*)p.y + ybase;
  const int64_t frame_bytes = p.F * Slot::YB;
  int issue_stage = 0, read_stage = 0;  // byte offsets of the next stages

  // frames are issued and consumed in order: running row pointers instead of
  // 64-bit n * F products per frame
  const unsigned char* ynext = ybytes + nfirst * frame_bytes;
  const R* vnext = vr + nfirst * p.F;
  const int64_t ystep = (int64_t)WARPS * frame_bytes, vstep = (int64_t)WARPS * p.F;
  auto issue = [&](int) {
    unsigned char* slot = wslots + issue_stage;
    issue_stage = (issue_stage + (int)kStageStride == STAGES * (int)kStageStride)
                      ? 0 : issue_stage + (int)kStageStride;
    const unsigned char* yrow = ynext;
    ynext += ystep;
    unsigned char* dst = slot + spos0;
    if (contiguous) {  // one base, compile-time offsets
#pragma unroll
      for (int c = 0; c < Slot::Q; ++c) {
        if constexpr (Slot::UB == 16)
          cp_async16(dst + 32 * c * Slot::UB, yrow + 32 * c * Slot::UB);
        else
          cp_async8(dst + 32 * c * Slot::UB, yrow + 32 * c * Slot::UB);
      }
    } else {
#pragma unroll
      for (int c = 0; c < Slot::Q; ++c) {
        const unsigned char* src = yrow + 32 * c * Slot::UB + ycorr[c];
        if constexpr (Slot::UB == 16)
          cp_async16(dst + 32 * c * Slot::UB, src);
        else
          cp_async8(dst + 32 * c * Slot::UB, src);
      }
    }
    unsigned char* vs = slot + 32 * Slot::YB;
    if constexpr (sizeof(R) == 8) {
      cp_async8(vs + 8 * lane, vnext);
      cp_async8(vs + 256 + 8 * lane, vnext + NF);
    } else {
      cp_async4(vs + 4 * lane, vnext);
      cp_async4(vs + 128 + 4 * lane, vnext + NF);
    }
    vnext += vstep;
  };

  // P lives in shared memory (bin-minor SoA after the frame ring): the 4
  // warps of the CTA work on the same 32 bins, so one 16*I*I-byte column per
  // lane serves all of them and frees the registers for the accumulators.
  constexpr int kTS = 33;  // P / W tile row stride (entries)
  T2* sP = (T2*)(smem_raw + Sm::RING);
  // W = P^{-H} for the image write (last pass only), same bin-minor tile layout
  T2* sW = sP + NP * kTS;
  auto load_tile = [&]() {
    if (FFCA_K3_PCOAL || BULK) {
      // the tile's P block (32 consecutive bins x NP entries) is one
      // contiguous run: thread t copies 16-B units t, t + 128, ... (bin
      // b = u / NP of the tile, clamped like g; entry e = u % NP)
      for (int u = threadIdx.x; u < 32 * NP; u += WARPS * 32) {
        const int b = u / NP, e = u - (u / NP) * NP;
        int64_t gb = tile0 + b;
        if (gb >= G) gb = G - 1;
        int es = e;
        if constexpr (BULK) {  // row r of P where the lane's rotated unit order reads y_r
          const int row = e / I;
          es = ((row - Slot::sw(b) + Slot::Q) % Slot::Q) * I + (e - row * I);
        }
        sP[es * kTS + b] = Math<R>::c2(ldcg2(p.P + gb * NP + e));
        if (MU && p.mu_back) sW[e * kTS + b] = Math<R>::c2(ldcg2(p.W + gb * NP + e));
      }
    } else {
      for (int e = warp; e < NP; e += WARPS) sP[e * kTS + lane] = Math<R>::c2(ldcg2(p.P + g * NP + e));
      if (MU && p.mu_back)
        for (int e = warp; e < NP; e += WARPS) sW[e * kTS + lane] = Math<R>::c2(ldcg2(p.W + g * NP + e));
    }
    __syncthreads();
  };
  // lambda (and the floor) are requested before the P tile's copy, so that
  // the two L2 round trips overlap
  double lam_g[I];
  double fl_g = 0.0;
  auto load_lam = [&]() {
#pragma unroll
    for (int a = 0; a < I; ++a) lam_g[a] = __ldcg(p.lam + g * I + a);
    fl_g = p.floor[g];
  };
  if (!kRingFirst) {
    load_lam();
    load_tile();
  }
  constexpr int kAhead = STAGES - 1;  // frames issued ahead
  // ---- TMA bulk ring (BULK): one elected lane per warp issues the copies ----
  // the tile's valid bins and the split into two mixtures (F >= 32: at most
  // two), per-segment source pointers at this warp's next frame, the 16-B
  // aligned v supersets (their alignment is a per-warp constant: a warp's
  // frames step by WARPS F v-elements = 32 F bytes), this lane's v offsets
  [[maybe_unused]] int b_nval = 0, b_s = 0;
  [[maybe_unused]] const unsigned char* b_y[2] = {nullptr, nullptr};
  [[maybe_unused]] const unsigned char* b_v[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  [[maybe_unused]] unsigned b_len[2][2] = {{0u, 0u}, {0u, 0u}};
  [[maybe_unused]] unsigned b_d2 = 0, b_bytes = 0, b_bar0 = 0;
  [[maybe_unused]] int b_off[2] = {0, 0};
  [[maybe_unused]] int b_rot = 0, b_ist = 0, b_rst = 0;
  [[maybe_unused]] unsigned b_ph = 0;
  auto b_stage = [&](int st) -> unsigned char* {
    return smem_raw + ((size_t)st * WARPS + warp) * BS::WARP_BYTES;
  };
  if constexpr (BULK) {
    b_nval = (int)min((int64_t)32, G - tile0);
    const int64_t m0 = tile0 / p.F, f0 = tile0 - m0 * p.F;
    b_s = (int)min((int64_t)b_nval, p.F - f0);
    b_y[0] = (const unsigned char*)p.y + ((m0 * p.N + nfirst) * p.F + f0) * BS::YB;
    b_y[1] = (const unsigned char*)p.y + (((m0 + 1) * p.N + nfirst) * p.F) * BS::YB;
    const unsigned char* vbase = (const unsigned char*)(p.v_src ? p.v_src : p.v);
    const int64_t va[2] = {(m0 * 2 * NF + nfirst * p.F + f0) * BS::VB,
                           ((m0 + 1) * 2 * NF + nfirst * p.F) * BS::VB};
    const int cnt[2] = {b_s, b_nval - b_s};
    b_d2 = (unsigned)((16 + b_s * BS::VB + 15) / 16 * 16);
#pragma unroll
    for (int j = 0; j < 2; ++j)  // v1, v2
#pragma unroll
      for (int q = 0; q < 2; ++q) {  // segments
        const uintptr_t a = (uintptr_t)(vbase + va[q] + (int64_t)j * NF * BS::VB);
        const uintptr_t lo = a & ~(uintptr_t)15;
        const uintptr_t hi = (a + (uintptr_t)cnt[q] * BS::VB + 15) & ~(uintptr_t)15;
        b_v[j][q] = (const unsigned char*)lo;
        b_len[j][q] = cnt[q] > 0 ? (unsigned)(hi - lo) : 0u;
        if ((lane < b_s) == (q == 0))
          b_off[j] = (q == 0 ? 0 : (int)b_d2) + (int)(a - lo) +
                     (q == 0 ? lane : lane - b_s) * BS::VB;
      }
    if (lane >= b_nval) b_off[0] = b_off[1] = 0;  // clamped bins read bin 0's slot
    b_bytes = (unsigned)(b_nval * BS::YB) + b_len[0][0] + b_len[0][1] + b_len[1][0] + b_len[1][1];
    b_rot = Slot::sw(lane);
    b_bar0 = smem_u32(smem_raw + Sm::RING + Sm::PB + Sm::WB + Sm::ACC) + warp * 8;
    if (lane == 0) {
      for (int st = 0; st < STAGES; ++st) mbar_init(b_bar0 + st * WARPS * 8, 1);
      mbar_init_fence();
    }
    __syncwarp();
  }
  auto bissue = [&]() {  // lane 0: this warp's next frame into stage b_ist
    const unsigned bar = b_bar0 + b_ist * WARPS * 8;
    unsigned char* dst = b_stage(b_ist);
    b_ist = b_ist + 1 == STAGES ? 0 : b_ist + 1;
    fence_proxy_async_smem();  // the stage's earlier generic reads before the async writes
    mbar_expect_tx(bar, b_bytes);
    bulk_g2s(smem_u32(dst), b_y[0], (unsigned)(b_s * BS::YB), bar);
    if (b_nval > b_s)
      bulk_g2s(smem_u32(dst + b_s * BS::YB), b_y[1], (unsigned)((b_nval - b_s) * BS::YB), bar);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      unsigned char* vd = dst + 32 * BS::YB + j * BS::VA;
      bulk_g2s(smem_u32(vd), b_v[j][0], b_len[j][0], bar);
      if (b_len[j][1]) bulk_g2s(smem_u32(vd + b_d2), b_v[j][1], b_len[j][1], bar);
    }
    const int64_t ys = (int64_t)WARPS * p.F * BS::YB, vs = (int64_t)WARPS * p.F * BS::VB;
    b_y[0] += ys;
    b_y[1] += ys;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      b_v[j][0] += vs;
      b_v[j][1] += vs;
    }
  };
  if constexpr (BULK) {
    if (lane == 0)
      for (int s = 0; s < kAhead; ++s)
        if (s < K) bissue();
  } else {
#pragma unroll
    for (int s = 0; s < kAhead; ++s) {
      if (s < K) issue(s);
      cp_async_commit();
    }
  }
  if (kRingFirst) {
    if (!pre()) {
      cp_async_wait_all();
      return;
    }
    load_lam();
    load_tile();
  }
  T lam[I], il[I];  // il = 1 / (I lam): the 1/I of v1 = tr1 / I folded in
#pragma unroll
  for (int a = 0; a < I; ++a) {
    lam[a] = (T)lam_g[a];
    il[a] = (T)rcp_nr((double)I * lam_g[a]);  // (MUFU seed + 2 Newton: ~1 ulp; no IEEE division)
  }
  const T fl = (T)fl_g;
  constexpr T invI = T(1) / I;

  R* vwrite = vb + nfirst * p.F;  // v of the frame being processed (advanced per frame)
  const unsigned char* cur_slot = wslots;  // ring stage of the frame being processed
  ImageRowStore<I, R> img;  // image rows (MU pass)
  if constexpr (MU) img.init(tile0, G, p.N, p.F, lane);
  // per-frame E+M body once z = P^H y is known
  auto frame = [&](int k, int64_t n, const T2 (&yv)[I], T v1, T v2, const T2 (&z)[I]) {
    T g1[I], g2[I], t1[I], t2[I];
    T tr1 = 0, tr2 = 0;  // already divided by I (folded into ilI / invI)
    double lprod = 1.0, quad = 0.0;
    bool bad = false;
    T v1l[I], den[I], rden[I];
    if constexpr (kF2) {
      // the same per-channel scalars, two channels per packed instruction
      float2 tr1p = make_float2(0.f, 0.f), tr2p = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < I / 2; ++q) {
        const int a = 2 * q;
        const float2 v1l2 = f2::mul(f2::bc(v1), make_float2(lam[a], lam[a + 1]));
        const float2 den2 = f2::add(v1l2, f2::bc(v2));
        const float2 rd2 = make_float2(f2::rcp(den2.x), f2::rcp(den2.y));
        const float2 g12 = f2::mul(v1l2, rd2), g22 = f2::mul(f2::bc(v2), rd2);
        const float2 pz2 = make_float2(fmaf(z[a].x, z[a].x, z[a].y * z[a].y),
                                       fmaf(z[a + 1].x, z[a + 1].x, z[a + 1].y * z[a + 1].y));
        const float2 t12 = f2::mul(g12, f2::fma(g12, pz2, f2::bc(v2)));
        const float2 t22 = f2::mul(g22, f2::fma(g22, pz2, v1l2));
        tr1p = f2::fma(t12, make_float2(il[a], il[a + 1]), tr1p);
        tr2p = f2::fma(t22, f2::bc(invI), tr2p);
        v1l[a] = v1l2.x, v1l[a + 1] = v1l2.y;
        den[a] = den2.x, den[a + 1] = den2.y;
        rden[a] = rd2.x, rden[a + 1] = rd2.y;
        g1[a] = g12.x, g1[a + 1] = g12.y;
        g2[a] = g22.x, g2[a + 1] = g22.y;
        t1[a] = t12.x, t1[a + 1] = t12.y;
        t2[a] = t22.x, t2[a + 1] = t22.y;
        if (LL) {
          lprod *= (double)den2.x * (double)den2.y;
          quad = fma((double)pz2.x, (double)rd2.x, quad);
          quad = fma((double)pz2.y, (double)rd2.y, quad);
        }
      }
      tr1 = tr1p.x + tr1p.y;
      tr2 = tr2p.x + tr2p.y;
    } else {
#pragma unroll
      for (int a = 0; a < I; ++a) {
        v1l[a] = v1 * lam[a];
        den[a] = v1l[a] + v2;
      }
      Math<R>::template rcp_n<I>(den, rden);
#pragma unroll
      for (int a = 0; a < I; ++a) {
        g1[a] = v1l[a] * rden[a];
        g2[a] = v2 * rden[a];
        const T pz = fma(z[a].x, z[a].x, z[a].y * z[a].y);
        // t_j = g_j^2 |z|^2 + c with c = v2 g1 = v1 lam g2 (reference
        // _kernels_numba.py:359-363), factored to save one multiply each
        t1[a] = g1[a] * fma(g1[a], pz, v2);
        t2[a] = g2[a] * fma(g2[a], pz, v1l[a]);
        tr1 = fma(t1[a], il[a], tr1);
        tr2 = fma(t2[a], invI, tr2);
        if (LL) {
          lprod *= (double)den[a];
          quad = fma((double)pz, (double)rden[a], quad);
        }
        // den == 0 needs no test: rcp(0) poisons w below (inf * 0 / NaN)
      }
    }
    if (LL) llacc += log(lprod) + quad;
    if (UPDATE) {
      const T q1 = tr1, q2 = tr2;
      const T w1 = (q1 < fl) ? fl : q1;  // NaN propagates like np.maximum
      const T w2 = (q2 < fl) ? fl : q2;
      if (active) {
        vwrite[0] = (R)w1;
        vwrite[NF] = (R)w2;
      }
      {  // non-finite or non-positive w (integer tests keep the FP pipes free)
        const double dw1 = w1, dw2 = w2;
        const long long b1 = __double_as_longlong(dw1), b2 = __double_as_longlong(dw2);
        bad |= (((b1 >> 52) & 0x7ff) == 0x7ff) | (((b2 >> 52) & 0x7ff) == 0x7ff) | (b1 <= 0) |
               (b2 <= 0);
      }
      if constexpr (kF2) {
        const float iw1 = f2::rcp(w1), iw2 = f2::rcp(w2);
        float h1[I], h2[I];
#pragma unroll
        for (int q = 0; q < I / 2; ++q) {  // diagonal entries (2q, 2q+1)
          const int a = 2 * q;
          acc2[0][q] = f2::fma(make_float2(t1[a], t1[a + 1]), f2::bc(iw1), acc2[0][q]);
          acc2[1][q] = f2::fma(make_float2(t2[a], t2[a + 1]), f2::bc(iw2), acc2[1][q]);
          const float2 h12 = f2::mul(make_float2(g1[a], g1[a + 1]), f2::bc(iw1));
          const float2 h22 = f2::mul(make_float2(g2[a], g2[a + 1]), f2::bc(iw2));
          h1[a] = h12.x, h1[a + 1] = h12.y;
          h2[a] = h22.x, h2[a + 1] = h22.y;
        }
#pragma unroll
        for (int a = 0; a < I; ++a) {
#pragma unroll
          for (int b = a + 1; b < I; ++b) {
            // (re, im) of z_a conj(z_b) in one pair, shared by both sources
            const float2 x = f2::fma(z[a], f2::bc(z[b].x),
                                     f2::mul(make_float2(z[a].y, -z[a].x), f2::bc(z[b].y)));
            const int e = Herm<I>::re(a, b) / 2;  // (re, im) = entries (2e, 2e+1)
            acc2[0][e] = f2::fma(f2::bc(h1[a] * g1[b]), x, acc2[0][e]);
            acc2[1][e] = f2::fma(f2::bc(h2[a] * g2[b]), x, acc2[1][e]);
          }
        }
        if ((k % kF32Block) == kF32Block - 1) flush();
      } else {
      T wv[2] = {w1, w2}, iw[2];
      Math<R>::template rcp_n<2>(wv, iw);
      const T iw1 = iw[0], iw2 = iw[1];
      T h1[I], h2[I];
#pragma unroll
      for (int a = 0; a < I; ++a) {
        accum(0, a, t1[a], iw1);
        accum(1, a, t2[a], iw2);
        h1[a] = g1[a] * iw1;
        h2[a] = g2[a] * iw2;
      }
#pragma unroll
      for (int a = 0; a < I; ++a) {
#pragma unroll
        for (int b = a + 1; b < I; ++b) {
          // z_a conj(z_b), shared by both sources
          const T zr = fma(z[a].x, z[b].x, z[a].y * z[b].y);
          const T zi = fma(z[a].y, z[b].x, -z[a].x * z[b].y);
          const T k1 = h1[a] * g1[b];
          const T k2 = h2[a] * g2[b];
          accum(0, Herm<I>::re(a, b), k1, zr);
          accum(0, Herm<I>::im(a, b), k1, zi);
          accum(1, Herm<I>::re(a, b), k2, zr);
          accum(1, Herm<I>::im(a, b), k2, zi);
        }
      }
      if (kBlk && ((k % kF32Block) == kF32Block - 1)) flush();
      }
    }
    if constexpr (MU) {
      // posterior means of this frame, both sources
      C o[2][I];
      if (p.mu_back) {
        // images (fast.py:133-141): mu_1 = P^{-H} (g1 z); mu_2 = y - mu_1, the
        // posterior partition mu_1 + mu_2 = y (g1 + g2 = 1, P^{-H} P^H = I),
        // exact up to rounding (reference test_fast.py:247-252)
#pragma unroll
        for (int a = 0; a < I; ++a) {
          T sx = 0, sy = 0;
#pragma unroll
          for (int b = 0; b < I; ++b) {
            const T2 w = sW[(a * I + b) * kTS + lane];
            const T mx = g1[b] * z[b].x, my = g1[b] * z[b].y;
            sx = fma(w.x, mx, fma(-w.y, my, sx));
            sy = fma(w.x, my, fma(w.y, mx, sy));
          }
          o[0][a].x = sx;
          o[0][a].y = sy;
          o[1][a].x = yv[a].x - sx;
          o[1][a].y = yv[a].y - sy;
        }
      } else {
#pragma unroll
        for (int a = 0; a < I; ++a) {
          o[0][a].x = z[a].x * g1[a];
          o[0][a].y = z[a].y * g1[a];
          o[1][a].x = z[a].x * g2[a];
          o[1][a].y = z[a].y * g2[a];
        }
      }
      img.store(p.mu_out, (unsigned char*)cur_slot, n, o);
    }
    if (bad && bad_n == 0) bad_n = n + 1;
  };
  auto load_frame = [&](int k, T2 (&yv)[I], T& v1, T& v2) {
    const unsigned char* slot = wslots + read_stage;
    cur_slot = slot;
    read_stage = (read_stage + (int)kStageStride == STAGES * (int)kStageStride)
                     ? 0 : read_stage + (int)kStageStride;
    constexpr int PER = Slot::UB / (int)sizeof(T2);  // channels per unit
#pragma unroll
    for (int a = 0; a < Slot::Q; ++a) {
      const T2* src = (const T2*)(slot + Slot::rpos(rb, a));
      if constexpr (PER == 2) {
        const float4 q = *(const float4*)src;  // two complex64 channels
        yv[2 * a] = T2{(T)q.x, (T)q.y};
        yv[2 * a + 1] = T2{(T)q.z, (T)q.w};
      } else {
        yv[a] = *src;
      }
    }
    const unsigned char* vs = slot + 32 * Slot::YB;
    v1 = ((const R*)vs)[lane];
    v2 = ((const R*)(vs + 32 * sizeof(R)))[lane];
  };
  auto bload = [&](T2 (&yv)[I], T& v1, T& v2) {  // BULK: the stage of frame k
    const unsigned bar = b_bar0 + b_rst * WARPS * 8;
    mbar_wait(bar, b_ph);
    const unsigned char* slot = b_stage(b_rst);
    if (++b_rst == STAGES) {
      b_rst = 0;
      b_ph ^= 1u;
    }
    const unsigned char* row = slot + lane * BS::YB;
#pragma unroll
    for (int k = 0; k < Slot::Q; ++k)  // unit (k + rot) mod Q (P's rows stored to match)
      yv[k] = *(const T2*)(row + 16 * ((k + b_rot) % Slot::Q));
    v1 = *(const R*)(slot + 32 * BS::YB + b_off[0]);
    v2 = *(const R*)(slot + 32 * BS::YB + BS::VA + b_off[1]);
  };

  {
    constexpr int kUnroll = FAST2_UNROLL;
#pragma unroll kUnroll
    for (int k = 0; k < K; ++k) {
      __syncwarp();  // every lane is done with the stage the next copy overwrites
      T2 yv[I];
      T v1, v2;
      if constexpr (BULK) {
        if (lane == 0 && k + STAGES - 1 < K) bissue();
        bload(yv, v1, v2);
      } else {
        if (k + STAGES - 1 < K) issue(k + STAGES - 1);
        cp_async_commit();
        cp_async_wait<STAGES - 1>();
        __syncwarp();  // the other lanes' copies of this stage are visible
        load_frame(k, yv, v1, v2);
      }
      T2 z[I];
      if constexpr (kF2) {
        // z_a = sum_b conj(P_ba) y_b: p.x (y.x, y.y) + p.y (y.y, -y.x), packed
#pragma unroll
        for (int a = 0; a < I; ++a) {
          const T2 p0 = sP[(0 * I + a) * kTS + lane];
          float2 za = f2::fma(f2::bc(p0.y), make_float2(yv[0].y, -yv[0].x),
                              f2::mul(f2::bc(p0.x), yv[0]));
#pragma unroll
          for (int b = 1; b < I; ++b) {
            const T2 pb = sP[(b * I + a) * kTS + lane];
            za = f2::fma(f2::bc(pb.x), yv[b], za);
            za = f2::fma(f2::bc(pb.y), make_float2(yv[b].y, -yv[b].x), za);
          }
          z[a] = za;
        }
      } else
#pragma unroll
      for (int a = 0; a < I; ++a) {
        const T2 p0 = sP[(0 * I + a) * kTS + lane];
        T zr = p0.x * yv[0].x + p0.y * yv[0].y;
        T zi = p0.x * yv[0].y - p0.y * yv[0].x;
#pragma unroll
        for (int b = 1; b < I; ++b) {
          const T2 pb = sP[(b * I + a) * kTS + lane];
          zr = fma(pb.x, yv[b].x, fma(pb.y, yv[b].y, zr));
          zi = fma(pb.x, yv[b].y, fma(-pb.y, yv[b].x, zi));
        }
        z[a].x = zr;
        z[a].y = zi;
      }
      frame(k, nfirst + (int64_t)k * WARPS, yv, v1, v2, z);
      vwrite += vstep;
    }
  }
  flush();
  cp_async_wait_all();
  if (bad_n && active && p.st)
    report_error(p.st, p.iter, FFCA_ERR_SINGULAR_MATRIX,
                 (unsigned long long)((m * p.N + (bad_n - 1)) * p.F + f));

  if (!UPDATE && !LL) return;
  if constexpr (kSacc) {
    // --- cross-warp reduction straight from the shared accumulators ---
    __syncthreads();
    if (warp != 0 || !active) return;
    double* sp = p.Spart + (size_t)by * 2 * NP * G + g;
#pragma unroll
    for (int e = 0; e < 2 * NP; ++e) {
      double t = accS[e * kAccStride];
#pragma unroll
      for (int w = 1; w < WARPS; ++w) t += accS[e * kAccStride + w * 32];
      sp[(size_t)e * G] = t;
    }
    return;
  } else {
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
  const int64_t c = by;
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
}

template <int I, typename R, int WARPS, int STAGES, bool UPDATE, bool LL, bool MU,
          bool BULK = false>
__global__ void __launch_bounds__(WARPS * 32, (fast2_minb<I, R, UPDATE, LL, MU>())) fast_em2_kernel(const FastIterParams p) {
  // (split-phase windows: dependents cover other bins and are released on entry;
  // chained plain schedule: released inside the pass, after its own wait)
  if (!p.pdl_wait) pdl_release_dependents();
  fast_em2_body<I, R, WARPS, STAGES, UPDATE, LL, MU, BULK>(p, blockIdx.x, blockIdx.y,
                                                          PdlGate{p.pdl_wait != 0});
}

// TMA bulk-copy frame ring for the complex128 update pass (off: measured
// slower). Correct (the whole GPU suite passes with it on), but at one warp
// per 32-bin tile every warp-frame is 3-6 small bulk copies (a 2 KB y row,
// two ~256 B v runs, doubled across a mixture boundary) issued by one lane:
// the copies serialise on the SM's TMA unit, each needs its operands moved
// to uniform registers (a waterfall loop in SASS) and the ring state costs
// registers (spills at 168): config-3 update pass 2.09 ms vs 1.55 ms with the
// cooperative cp.async ring, config 4 0.563 vs 0.412 ms (same session).
#ifndef FFCA_K3_BULK
#define FFCA_K3_BULK 0
#endif
// The bulk ring needs every tile within two mixtures (F >= 32) and 16-B
// aligned y / v bases; other calls take the cp.async ring.
template <int I, typename R, bool UPDATE, bool LL, bool MU>
constexpr bool fast2_bulk_capable() {
  return FFCA_K3_BULK && BulkSlot<I, R>::kOk && UPDATE && !LL && !MU &&
         !SmemAcc<I, R, UPDATE, LL, MU>::value;
}

template <int I, typename R, bool UPDATE, bool LL, bool MU, bool BULK>
cudaError_t launch_fast2_kern(const FastIterParams& p, cudaStream_t s) {
  constexpr int WARPS = kWarps;
  constexpr int STAGES = fast2_stages<I, R, UPDATE, LL, MU>();
  using Sm = Fast2Smem<I, R, WARPS, STAGES, MU, SmemAcc<I, R, UPDATE, LL, MU>::value, BULK>;
  auto kern = fast_em2_kernel<I, R, WARPS, STAGES, UPDATE, LL, MU, BULK>;
  if (cudaError_t e = ensure_smem<fast_em2_kernel<I, R, WARPS, STAGES, UPDATE, LL, MU, BULK>>(Sm::BYTES))
    return e;
  dim3 grid((unsigned)((window_end(p.g1, p.G) - p.g0 + 31) / 32), (unsigned)p.nchunk);
  return launch_ex(kern, grid, dim3(WARPS * 32), Sm::BYTES, s, p.pdl != 0 || p.pdl_wait != 0, 0, p);
}

template <int I, typename R, bool UPDATE, bool LL, bool MU>
cudaError_t launch_fast2_variant(const FastIterParams& p, cudaStream_t s) {
  if constexpr (fast2_bulk_capable<I, R, UPDATE, LL, MU>()) {
    const void* vb = p.v_src ? p.v_src : p.v;
    if (p.F >= 32 && ((uintptr_t)p.y % 16) == 0 && ((uintptr_t)vb % 16) == 0)
      return launch_fast2_kern<I, R, UPDATE, LL, MU, true>(p, s);
  }
  return launch_fast2_kern<I, R, UPDATE, LL, MU, false>(p, s);
}

template <int I, typename R>
int fast2_blocks_per_sm() {
  constexpr int STAGES = fast2_stages<I, R, true, false, false>();
  using Sm = Fast2Smem<I, R, kWarps, STAGES, false, SmemAcc<I, R, true, false, false>::value>;
  auto kern = fast_em2_kernel<I, R, kWarps, STAGES, true, false, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sm::BYTES);
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, Sm::BYTES);
  return n > 0 ? n : 1;
}

// K3t (ffca_fast_tma.cuh): the complex128 update pass with a CTA-wide TMA
// ring over 128-bin tiles; needs every tile within two mixtures (F >= 128)
// and 16-B aligned y / v bases. Off by default: correct (GPU suite green with
// it on) but slower than the cooperative cp.async ring — config-3 update pass
// 1.68 ms vs 1.56 ms, config 4 0.488 vs 0.412 ms (same session): the 128-bin
// P tile (32 KB) leaves room for only 4 ring stages at 3 CTAs/SM, i.e. ~90 KB
// in flight per SM against ~150 KB for the per-warp 6-stage ring, and the 4
// warps of a CTA run in lockstep on the shared stages.
#ifndef FFCA_K3T
#define FFCA_K3T 0
#endif
template <int I>
cudaError_t launch_fast_tma(const FastIterParams& p, cudaStream_t s);
template <int I, typename R>
bool fast_tma_applies(const FastIterParams& p) {
  if constexpr (!FFCA_K3T || !std::is_same<R, double>::value) {
    return false;
  } else {
    const void* vb = p.v_src ? p.v_src : p.v;
    return p.update && !p.llbin && !p.mu_out && p.F >= 128 && ((uintptr_t)p.y % 16) == 0 &&
           ((uintptr_t)vb % 16) == 0;
  }
}

template <int I, typename R>
cudaError_t launch_fast2(const FastIterParams& p, cudaStream_t s) {
  const bool ll = p.llbin != nullptr;
  const bool mu = p.mu_out != nullptr;
  if (fast_tma_applies<I, R>(p)) return launch_fast_tma<I>(p, s);
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
