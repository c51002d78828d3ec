// KP — persistent FastFCA EM kernel for problems whose whole update-pass grid
// is resident at once (configs 0 / 1: a few hundred bins). The plain schedule
// runs two launches per iteration (streaming pass K3, per-bin refresh K1) and
// on these sizes each is a few microseconds of latency-bound work behind a
// kernel boundary. Here ONE cooperative launch runs `iters` full iterations
// (reference fast.py:200-223, the loop body of fastfca_run):
//
//   * one CTA per (32-bin tile, frame chunk) stays resident: every iteration
//     it runs K3's pass (fast_em2_body, the same code as the stand-alone
//     kernel: same chunking, same arithmetic, same partial layout), then
//     takes a ticket on the tile's arrival counter;
//   * the LAST chunk CTA of a tile to arrive refreshes the tile (LAR): warps
//     1-3 sum the tile's partials in chunk order into shared memory, warp 0
//     (lane = bin) runs K1's per-bin refresh (pencil_update_body) on the sums
//     and publishes the tile's iteration number; the others wait for it.
//     (FFCA_PERSIST_LAR=0: dedicated refresher warps, one per tile, poll the
//     arrival counter instead — slower, kept for comparison.)
//
// Tiles never wait for each other: the only synchronisation is per tile,
// through two words in global memory (release: __threadfence + atomic;
// acquire: relaxed polling loads + one fence), and the per-bin state crossing
// CTAs (partials, P, lambda) is read from L2 (__ldcg), never through L1. The launch is
// cooperative only for its co-residency guarantee (a CTA that spins on a
// tile's flag needs that tile's other CTAs to be running); the waits are
// bounded (kSpinLimitNs) and report FFCA_ERR_CUDA instead of hanging.
#pragma once

#include "ffca_fast2.cuh"
#include "ffca_pencil_body.cuh"

namespace ffca {

constexpr unsigned long long kSpinLimitNs = 4000000000ull;  // 4 s

// Polling load: relaxed at gpu scope (served by L2, no L1 invalidation per
// poll — an acquire load compiles to the load plus a CCTL.IVALL, which on an
// SM shared with a refresher warp keeps flushing that warp's L1-resident
// spill slots). The acquire fence is issued once, after the wait.
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// spin until *flag >= target; false when the run was aborted / timed out
__device__ __forceinline__ bool wait_ge(const int* flag, int target, int* abort) {
  unsigned spins = 0;
  unsigned long long t0 = 0;
  while (ld_relaxed_gpu(flag) < target) {
    if ((++spins & 255u) == 0) {
      if (ld_relaxed_gpu(abort)) return false;
      const unsigned long long t = global_ns();
      if (t0 == 0) t0 = t;
      if (t - t0 > kSpinLimitNs) {
        atomicExch(abort, 1);
        return false;
      }
    }
  }
  fence_acquire_gpu();
  return true;
}

template <int I>
struct PersistCfg {
  static constexpr int WARPS = kWarps;
  static constexpr int STAGES = fast2_stages<I, double, true, false, false>();
  using Sm = Fast2Smem<I, double, WARPS, STAGES, false, false, false>;
};

#ifndef FFCA_PERSIST_LAR_EARLY
#define FFCA_PERSIST_LAR_EARLY 0  // LAR: publish a tile before W is stored (second generation word)
#endif
#ifndef FFCA_PERSIST_MINB
#define FFCA_PERSIST_MINB 2  // CTAs per SM: the refresher role (K1's per-bin code) needs the
                             // full register budget (at 3 per SM it spills ~0.7-2.7 KB and
                             // config 1 drops from 17.2 to 12.9 G)
#endif

template <int I>
__global__ void __launch_bounds__(kWarps * 32, FFCA_PERSIST_MINB)
    fast_persist_kernel(FastIterParams fp, PencilParams pp, const PersistCtl ctl) {
  using Cfg = PersistCfg<I>;
  const int nstream = ctl.tiles * ctl.nchunk;
  if ((int)blockIdx.x < nstream) {
    // ---- streaming role: tile-major so that a tile's chunks start together
    const unsigned tile = blockIdx.x % (unsigned)ctl.tiles;
    const unsigned chunk = blockIdx.x / (unsigned)ctl.tiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int s_ok, s_ticket;
    // (LAR) the tile's summed partials, [2 I^2][32 bins], beyond the pass's shared memory
    extern __shared__ __align__(16) unsigned char kp_smem[];
    double* stage = (double*)(kp_smem + Cfg::Sm::BYTES);
    constexpr int NE2 = 2 * I * I;
    const int64_t g = pp.g0 + (int64_t)tile * 32 + lane;
    const bool active = g < pp.G;
    auto cta_barrier = []() { asm volatile("barrier.sync 1, %0;" ::"n"(kWarps * 32) : "memory"); };
    for (int l = 0; l < ctl.iters; ++l) {
      fp.iter = l + 1;
      if (l > 0) fp.v_src = nullptr;
      // the wait for the tile's refresh of iteration l - 1 runs inside the
      // pass, after its y / v prefetch is in flight and before P / lambda
      auto pre = [&]() -> bool {
        if (l == 0) return true;
        if (threadIdx.x < 32) {
          const bool ok = wait_ge(ctl.ready + tile, l, ctl.abort);
          if (threadIdx.x == 0) s_ok = ok;
        }
        __syncthreads();
        return s_ok != 0;
      };
      fast_em2_body<I, double, Cfg::WARPS, Cfg::STAGES, true, false, false, false>(fp, tile, chunk,
                                                                                  pre);
      if (l > 0 && !s_ok) return;  // aborted inside the pass (CTA-uniform)
      // (LAR) the tile's W generation, read while the fence below drains: the
      // acquire fence after the ticket orders the later W loads behind it
      const int wseen = (ctl.lar && warp == 0) ? ld_relaxed_gpu(ctl.wready + tile) : 0;
      __threadfence();   // this thread's v and partial stores, device-wide
      __syncthreads();   // (also: the body's shared memory is free for the next iteration)
      if (!ctl.lar) {
        if (threadIdx.x == 0) atomicAdd(ctl.arrive + tile, 1);
        continue;
      }
      // ---- LAR: the LAST chunk CTA of the tile to arrive refreshes the tile.
      // Its four warps sum the tile's chunk partials (fixed chunk order, every
      // load in flight at once) into shared memory, warp 0 runs K1's per-bin
      // code on the sums and publishes the tile; warps 1-3 go on to the next
      // pass's prefetch. No refresher CTAs, one flag hop per iteration.
      if (threadIdx.x == 0) s_ticket = atomicAdd(ctl.arrive + tile, 1);
      __syncthreads();
      if (s_ticket != ctl.nchunk * (l + 1) - 1) continue;  // (CTA-uniform)
      fence_acquire_gpu();  // the other chunk CTAs' partials (released before their arrival)
      // (warps 1-3 reduce; warp 0 already holds its bins' P / W in registers and only waits)
      constexpr int RT = (kWarps - 1) * 32;  // reducing threads
      auto staged = [&]() -> const double* {
        cta_barrier();  // (per-thread: warp 0's lanes arrive from inside the per-bin code)
        return stage;
      };
      auto reduce = [&]() {
        const int rt = (int)threadIdx.x - 32;
        constexpr int PPT = (NE2 * 32 + RT - 1) / RT;  // (entry, bin) pairs per thread
        constexpr int CB = NE2 >= 18 ? 8 : 16;  // chunks per batch (register budget)
        double sum[PPT];
#pragma unroll
        for (int j = 0; j < PPT; ++j) sum[j] = 0.0;
#pragma unroll 1
        for (int c0 = 0; c0 < ctl.nchunk; c0 += CB) {
          double buf[PPT][CB];
#pragma unroll
          for (int j = 0; j < PPT; ++j) {
            const int idx = rt + RT * j;
            const int e = idx >> 5, b = idx & 31;
            int64_t gb = pp.g0 + (int64_t)tile * 32 + b;
            if (gb >= pp.G) gb = pp.G - 1;
            const double* sp = pp.Spart + (size_t)e * pp.G + gb;
#pragma unroll
            for (int k = 0; k < CB; ++k)
              buf[j][k] = (idx < NE2 * 32 && c0 + k < ctl.nchunk)
                              ? __ldcg(sp + (size_t)(c0 + k) * NE2 * pp.G)
                              : 0.0;
          }
#pragma unroll
          for (int j = 0; j < PPT; ++j)
#pragma unroll
            for (int k = 0; k < CB; ++k)
              if (c0 + k < ctl.nchunk) sum[j] += buf[j][k];
        }
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          const int idx = rt + RT * j;
          if (idx < NE2 * 32) stage[idx] = sum[j];
        }
        cta_barrier();
      };
      if (warp != 0) {
        reduce();
        continue;
      }
      PencilParams q = pp;
      q.iter = l + 1;
      q.nchunk = 1;  // (the staged sums are one "chunk")
#if FFCA_PERSIST_LAR_EARLY
      // publish after P / lambda, W later under its own generation word (the
      // tile's next refresh may run on another CTA). Measured no faster: the
      // refreshing CTA starts its next pass late by the W computation and is
      // the tile's last arriver again, so the tile's iteration is the same.
      auto publish = [&]() {
        __threadfence();  // P, lambda of this bin, device-wide
        asm volatile("barrier.sync 2, 32;" ::: "memory");
        if (lane == 0) atomicExch(ctl.ready + tile, l + 1);
      };
      const bool wok = wseen >= l || wait_ge(ctl.wready + tile, l, ctl.abort);
      if (active)
        pencil_update_body<I, true>(q, g, staged, publish);
      else {
        staged();
        publish();
      }
      __threadfence();  // W, log|det P|^2 of this bin, device-wide
      asm volatile("barrier.sync 2, 32;" ::: "memory");
      if (lane == 0) atomicExch(ctl.wready + tile, l + 1);
      if (!__all_sync(0xffffffffu, wok) && lane == 0 && pp.st)
        report_error(pp.st, l + 1, FFCA_ERR_CUDA, (unsigned long long)tile);
#else
      // the whole per-bin state (P, lambda, W, log|det P|^2) is stored before
      // the tile is published: the tile's next refresh may run on another CTA
      // and reads all of it behind this one release
      (void)wseen;
      if (active)
        pencil_update_body<I, true>(q, g, staged);
      else
        staged();
      __threadfence();
      asm volatile("barrier.sync 2, 32;" ::: "memory");
      if (lane == 0) atomicExch(ctl.ready + tile, l + 1);
#endif
    }
  } else {
    // ---- refresher role: warp 0 of the CTA, lane = bin of the tile.
    // (Staging the tile's partials in shared memory with all four warps —
    // every load in flight at once — measured slower: config 1 15.9-17.2 G
    // against 19.3 G for the one-warp refresher below.)
    // FFCA_PERSIST_RTILES tiles per refresher CTA (one per warp): warps that
    // run the same ~64 KB of straight-line per-bin code on one SM share its
    // instruction-cache fills (the stand-alone K1 is instruction-fetch bound)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp >= FFCA_PERSIST_RTILES) return;
    const int tile = ((int)blockIdx.x - nstream) * FFCA_PERSIST_RTILES + warp;
    if (tile >= ctl.tiles) return;
    const int64_t g = pp.g0 + (int64_t)tile * 32 + lane;
    const bool active = g < pp.G;
    for (int l = 0; l < ctl.iters; ++l) {
      pp.iter = l + 1;
      bool ok = true;
      // the wait for the tile's chunk CTAs runs inside the per-bin code, after
      // the bin's P / W loads are issued
      auto pre = [&]() -> const double* {
        ok = wait_ge(ctl.arrive + tile, ctl.nchunk * (l + 1), ctl.abort);
        return nullptr;
      };
      // the tile's generation is published once every lane has stored P and
      // lambda; W and log|det P|^2 follow while the next pass streams (a lane's
      // own loads of them in the next refresh are in program order; the image
      // pass reads them after the kernel)
      auto publish = [&]() {
        __threadfence();  // P, lambda of this bin, device-wide
        // (per-thread barrier of this warp's 32 lanes: inactive lanes arrive below)
        asm volatile("barrier.sync %0, 32;" ::"r"(2 + warp) : "memory");
        if (lane == 0 && ok) atomicExch(ctl.ready + tile, l + 1);
      };
      if (active)
        pencil_update_body<I, true>(pp, g, pre, publish);
      else {
        pre();
        publish();
      }
      if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0 && pp.st)
          report_error(pp.st, l + 1, FFCA_ERR_CUDA, (unsigned long long)tile);
        return;
      }
    }
  }
}

// Dynamic shared memory: the streaming role's ring + tile
template <int I>
size_t persist_smem(int) {  // the pass's ring + tile, then LAR's staged sums [2 I^2][32]
  return PersistCfg<I>::Sm::BYTES + (size_t)2 * I * I * 32 * sizeof(double);
}
template <int I>
cudaError_t persist_attr() {
  return ensure_smem<fast_persist_kernel<I>>(persist_smem<I>(0));
}

// CTAs of the persistent kernel that can be resident at once on this device
template <int I>
int persist_slots() {
  auto kern = fast_persist_kernel<I>;
  if (persist_attr<I>() != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, persist_smem<I>(0)) !=
      cudaSuccess)
    return 0;
  return n * sm_count();
}
template <int I>
int persist_max_chunks() {
  return 1 << 20;  // (no per-chunk resource in the kernel)
}

template <int I>
cudaError_t launch_persist(const FastIterParams& fp, const PencilParams& pp, const PersistCtl& ctl,
                           cudaStream_t s) {
  if (cudaError_t e = persist_attr<I>()) return e;
  if (ctl.nchunk > persist_max_chunks<I>()) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ctl.tiles * ctl.nchunk + (ctl.lar ? 0 : (int)persist_refreshers(ctl.tiles))));
  cfg.blockDim = dim3(kWarps * 32);
  cfg.dynamicSmemBytes = persist_smem<I>(ctl.nchunk);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fast_persist_kernel<I>, fp, pp, ctl);
}

}  // namespace ffca
