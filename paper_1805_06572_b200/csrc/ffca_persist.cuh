// KP — persistent FastFCA EM kernel for problems whose whole update-pass grid
// is resident at once (configs 0 / 1: a few hundred bins). The plain schedule
// runs two launches per iteration (streaming pass K3, per-bin refresh K1) and
// on these sizes each is a few microseconds of latency-bound work behind a
// kernel boundary. Here ONE cooperative launch runs `iters` full iterations
// (reference fast.py:200-223, the loop body of fastfca_run):
//
//   * streaming CTAs, one per (32-bin tile, frame chunk): every iteration
//     they run K3's pass (fast_em2_body, the same code as the stand-alone
//     kernel: same chunking, same arithmetic, same partial layout), then
//     bump the tile's arrival counter;
//   * one refresher warp per tile (lane = bin; four to a CTA): waits until
//     all of the tile's chunk CTAs have arrived, runs K1's per-bin refresh
//     (pencil_update_body) and publishes the tile's iteration number.
//
// Tiles never wait for each other: the only synchronisation is per tile,
// through two words in global memory (release: __threadfence + atomic;
// acquire: relaxed polling loads + one fence), and the per-bin state crossing CTAs (partials, P,
// W, lambda) is read from L2 (__ldcg), never through L1. The launch is
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
    __shared__ int s_ok;
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
      __threadfence();   // this thread's v and partial stores, device-wide
      __syncthreads();   // (also: the body's shared memory is free for the next iteration)
      if (threadIdx.x == 0) atomicAdd(ctl.arrive + tile, 1);
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
size_t persist_smem(int) {
  return PersistCfg<I>::Sm::BYTES;
}
template <int I>
cudaError_t persist_attr() {
  return ensure_smem<fast_persist_kernel<I>>(PersistCfg<I>::Sm::BYTES);
}

// CTAs of the persistent kernel that can be resident at once on this device
template <int I>
int persist_slots() {
  auto kern = fast_persist_kernel<I>;
  if (persist_attr<I>() != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kWarps * 32, PersistCfg<I>::Sm::BYTES) !=
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
  cfg.gridDim = dim3((unsigned)(ctl.tiles * ctl.nchunk + (int)persist_refreshers(ctl.tiles)));
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
