// K3 dispatch + likelihood bookkeeping + frame chunking.
// (The fused pass itself lives in ffca_fast2.cuh for I <= 4 and in
// ffca_fast_par.cu for I >= 5.) Original design notes of the pass:
// K3 — fused FastFCA iteration: z = P^H y, diagonal posterior, v update,
// per-bin transformed covariance accumulation, optional log-likelihood and
// optional posterior-mean / separated-image write, in ONE streaming pass.
//
// Reference: _kernels_numba.py:328-391 (_fast_iteration) fused with
// _kernels_numba.py:220-243 (_fast_log_likelihood) and fast.py:133-141
// (back_transform_images, via W = P^{-H}).
//
// Thread mapping: lane <-> global bin g = m*F + f (32 consecutive bins per
// warp, so every frame row of y and v is a coalesced load), warps <-> frame
// slices. Each thread keeps its bin's P, lambda and the packed Hermitian
// accumulators of both sources in registers and streams its frames; the
// per-bin sums are reduced across the CTA's warps in shared memory and
// written as one partial per (frame chunk, bin). Reduction order is fixed, so
// results are deterministic and independent of how bins are sharded.
#include <cstdlib>

#include "ffca_fast2.cuh"  // FFCA_K3T

namespace ffca {

// v2 kernels for I <= 4 (ffca_fast2.cuh, instantiated in ffca_fast_i<I>.cu)
template <int I, typename R>
cudaError_t launch_fast2(const FastIterParams& p, cudaStream_t s);
template <int I, typename R>
int fast2_blocks_per_sm();
cudaError_t launch_fast_par(const FastIterParams& p, int I, int dtype, cudaStream_t s);
int fast_par_blocks_per_sm(int I, int dtype);
int fast_par_bins_per_cta();

int fast_blocks_per_sm(int I, int dtype) {
  static int cache[2][9] = {};
  const int d = dtype == FFCA_C64 ? 1 : 0;
  if (I < 1 || I > 8) return 1;
  if (cache[d][I]) return cache[d][I];
  int n = 1;
  switch (I) {
    case 1:
      n = d ? fast2_blocks_per_sm<1, float>() : fast2_blocks_per_sm<1, double>();
      break;
    case 2:
      n = d ? fast2_blocks_per_sm<2, float>() : fast2_blocks_per_sm<2, double>();
      break;
    case 3:
      n = d ? fast2_blocks_per_sm<3, float>() : fast2_blocks_per_sm<3, double>();
      break;
    case 4:
      n = d ? fast2_blocks_per_sm<4, float>() : fast2_blocks_per_sm<4, double>();
      break;
    default:
      n = fast_par_blocks_per_sm(I, dtype);
      break;
  }

  cache[d][I] = n;
  return n;
}


template <int I>
int fast_tma_blocks_per_sm();  // ffca_fast_i<I>.cu

// the update pass's CTA tile and residency: K3t (128-bin tiles, complex128,
// I <= 4) when enabled, else the cp.async ring kernel (32-bin tiles) / K3p
bool fast_tma_tiles(int I, int dtype) { return FFCA_K3T && dtype == FFCA_C128 && I >= 1 && I <= 4; }
int fast_tile_bins(int I, int dtype) {
  if (I >= 5) return fast_par_bins_per_cta();
  return fast_tma_tiles(I, dtype) ? 128 : 32;
}
int fast_update_blocks_per_sm(int I, int dtype) {
  if (!fast_tma_tiles(I, dtype)) return I >= 5 ? fast_par_blocks_per_sm(I, dtype) : fast_blocks_per_sm(I, dtype);
  static int cache[5] = {};
  if (!cache[I]) {
    switch (I) {
      case 1: cache[I] = fast_tma_blocks_per_sm<1>(); break;
      case 2: cache[I] = fast_tma_blocks_per_sm<2>(); break;
      case 3: cache[I] = fast_tma_blocks_per_sm<3>(); break;
      default: cache[I] = fast_tma_blocks_per_sm<4>(); break;
    }
  }
  return cache[I];
}

int bin_window_granularity(int I, int dtype) {
  const int t = fast_tile_bins(I, dtype);  // K3 32 / K3t 128 / K3p 8; K1p 8-32
  return t > 32 ? t : 32;
}

// KP (persistent EM kernel) applies
// to complex128 I <= 4 problems of at most FFCA_PERSIST_MAXPTS (default 4 Mi)
// TF-bins whose tiles * (nchunk + 1) CTAs are resident at once.
static int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return e && *e ? atoll(e) : dflt;
}
// FFCA_PERSIST: 0 never, 1 whenever the shape fits, unset: the measured-win
// region (fast_persist_auto)
bool pdl_chain_enabled() {
  static const int v = (int)env_i64("FFCA_PDL_CHAIN", 1);
  return v != 0;
}
bool fast_persist_lar() {
  static const int v = (int)env_i64("FFCA_PERSIST_LAR", 1);
  return v != 0;
}
int fast_persist_env() {
  static const int v = (int)env_i64("FFCA_PERSIST", -1);
  return v;
}
bool fast_persist_shape(int64_t G, int64_t N, int I, int dtype) {
  static const int64_t maxpts = env_i64("FFCA_PERSIST_MAXPTS", (int64_t)4 << 20);
  if (I < 1 || I > 4 || dtype != FFCA_C128 || G * N > maxpts) return false;
  const int64_t tiles = (G + 31) / 32;
  return tiles * 3 <= fast_persist_slots(I);
}
// Shapes on which KP measured faster than the plain schedule
// (profiles/r02_persist_sweep_lar.jsonl, 48 shapes, each schedule with its own
// chunk plan): I = 3 up to 33 tiles (+2..37%, one shape -3%), I = 2 up to 9
// tiles with >= 500k TF-bins (+17..35%; smaller or wider I = 2 problems are
// within +-6%). At I = 4 the plain schedule's lane-parallel K1p beats the
// one-thread-per-bin refresh (KP 0.67-0.92x).
bool fast_persist_auto(int64_t G, int64_t N, int I, int dtype) {
  if (!fast_persist_shape(G, N, I, dtype) || G * N < 32768) return false;
  const int64_t tiles = (G + 31) / 32;
  return (I == 3 && tiles <= 33) || (I == 2 && tiles <= 9 && G * N >= 500000);
}
// whether a run with these flags takes the KP path (given that its chunking fits)
bool fast_persist_wanted(unsigned flags, int64_t G, int64_t N, int I, int dtype) {
  if (flags & (FFCA_FLAG_NO_PERSIST | FFCA_FLAG_LIKELIHOOD | FFCA_FLAG_HISTORY)) return false;
  const int env = fast_persist_env();
  if (env == 0) return false;
  if ((flags & FFCA_FLAG_PERSIST) || env > 0) return fast_persist_shape(G, N, I, dtype);
  return fast_persist_auto(G, N, I, dtype);
}
// KP's chunk plan: one resident wave with room for the tiles' refresher CTAs,
// the finest chunking of >= FFCA_PERSIST_MINF frames (default 8 per warp)
bool plan_persist_chunks(int64_t G, int64_t N, int I, int dtype, int64_t* chunk_frames,
                         int* nchunk) {
  if (!fast_persist_shape(G, N, I, dtype)) return false;
  static const int64_t minf = env_i64("FFCA_PERSIST_MINF", 8 * kWarps);
  const int64_t tiles = (G + 31) / 32;
  int64_t ncmax = (fast_persist_slots(I) - persist_refreshers(tiles)) / tiles;
  if (ncmax > fast_persist_max_chunks(I)) ncmax = fast_persist_max_chunks(I);
  for (int64_t nc = ncmax; nc >= 1; --nc) {
    const int64_t cf = (N + nc - 1) / nc;
    if (cf < minf && nc > 1) continue;
    *chunk_frames = cf;
    *nchunk = (int)((N + cf - 1) / cf);
    return true;
  }
  return false;
}

// I >= 5 problems of a few hundred to a few thousand bins: the lane-parallel
// refresh K1p is one short latency-bound wave (config 2: 79 of 221 us per
// iteration), so the driver runs two bin windows, window B's pass overlapping
// window A's refresh (config 2 FastFCA 4.64 -> 5.3 G; three windows lose).
// FFCA_PAR_SPLIT=0 turns the rule off.
bool fast_par_split_shape(int64_t G, int64_t N, int I) {
  static const int on = (int)env_i64("FFCA_PAR_SPLIT", 1);
  return on && I >= 5 && G >= 256 && G <= 4096 && G * N >= ((int64_t)1 << 19);
}

void plan_fast_chunks(int64_t G, int64_t N, int I, int dtype, int64_t* chunk_frames,
                      int* nchunk) {
  if (I >= 5 && fast_par_split_shape(G, N, I)) {
    // two bin windows (split-phase schedule): each window's pass should fill
    // the GPU by itself, with chunks of >= 48 frames (config 2: 41 chunks of
    // 49 frames; sweep in profiles/r02_split_phase.txt)
    plan_chunks((G + 1) / 2, N, fast_par_blocks_per_sm(I, dtype), chunk_frames, nchunk,
                fast_par_bins_per_cta(), 48);
    return;
  }
  if (I >= 5)
    plan_chunks(G, N, fast_par_blocks_per_sm(I, dtype), chunk_frames, nchunk,
                fast_par_bins_per_cta(), 16);
  else
    // I <= 3: at most 17 chunks. The one-thread-per-bin refresh K1 reads every
    // chunk's partials in dependent batches, which the wave model does not
    // see: on single small mixtures 13-17 chunks beat the slot-filling 26-34
    // by 8-20% (profiles/r02_chunk_probe.jsonl; config 1 17.4 -> 19.9 G)
    plan_chunks(G, N, fast_update_blocks_per_sm(I, dtype), chunk_frames, nchunk,
                fast_tile_bins(I, dtype), 8 * kWarps, I <= 3 ? 17 : 0);
}

cudaError_t launch_fast_em(const FastIterParams& p, int I, int dtype, cudaStream_t s) {
  if (I >= 5) return launch_fast_par(p, I, dtype, s);  // lane-parallel (ffca_fast_par.cu)
#define FFCA_CASE2(II)                                                      \
  case II:                                                                  \
    return dtype == FFCA_C64 ? launch_fast2<II, float>(p, s)                \
                             : launch_fast2<II, double>(p, s);
  switch (I) {
    FFCA_CASE2(1)
    FFCA_CASE2(2)
    FFCA_CASE2(3)
    FFCA_CASE2(4)
    default:
      return cudaErrorInvalidValue;
  }
#undef FFCA_CASE2
}

// ---- KP dispatch (ffca_persist_i<I>.cu) ---------------------------------------
template <int I>
int persist_slots();
template <int I>
int persist_max_chunks();
int fast_persist_max_chunks(int I) {
  switch (I) {
    case 1: return persist_max_chunks<1>();
    case 2: return persist_max_chunks<2>();
    case 3: return persist_max_chunks<3>();
    case 4: return persist_max_chunks<4>();
    default: return 0;
  }
}
template <int I>
cudaError_t launch_persist(const FastIterParams& fp, const PencilParams& pp, const PersistCtl& ctl,
                           cudaStream_t s);

int fast_persist_slots(int I) {
  static int cache[5] = {-1, -1, -1, -1, -1};
  if (I < 1 || I > 4) return 0;
  if (cache[I] < 0) {
    switch (I) {
      case 1: cache[I] = persist_slots<1>(); break;
      case 2: cache[I] = persist_slots<2>(); break;
      case 3: cache[I] = persist_slots<3>(); break;
      default: cache[I] = persist_slots<4>(); break;
    }
  }
  return cache[I];
}

cudaError_t launch_fast_persist(const FastIterParams& fp, const PencilParams& pp, int* sync,
                                int tiles, int iters, int I, cudaStream_t s) {
  PersistCtl ctl{sync, sync + tiles, sync + 2 * tiles, sync + 3 * tiles, tiles, fp.nchunk, iters,
                 fast_persist_lar() ? 1 : 0};
  switch (I) {
    case 1: return launch_persist<1>(fp, pp, ctl, s);
    case 2: return launch_persist<2>(fp, pp, ctl, s);
    case 3: return launch_persist<3>(fp, pp, ctl, s);
    case 4: return launch_persist<4>(fp, pp, ctl, s);
    default: return cudaErrorInvalidValue;
  }
}

// ---- likelihood bookkeeping ------------------------------------------------
__global__ void ll_collect_kernel(const double* __restrict__ llbin, int nchunk,
                                  const double* __restrict__ logdet2, int64_t N, int64_t G,
                                  double* __restrict__ llg) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  const double s = ordered_sum(llbin + g, nchunk, (size_t)G);
  const double ld = logdet2 ? (double)N * logdet2[g] : 0.0;
  llg[g] = ld - s;
}

cudaError_t launch_ll_collect(const double* llbin, int nchunk, const double* logdet2, int64_t N,
                              int64_t G, double* llg, cudaStream_t s) {
  ll_collect_kernel<<<(unsigned)((G + 255) / 256), 256, 0, s>>>(llbin, nchunk, logdet2, N, G,
                                                                llg);
  return cudaGetLastError();
}

// one CTA per (m, level): fixed-order tree over bins
__global__ void ll_reduce_kernel(const double* __restrict__ llg, int64_t M, int64_t F, int64_t N,
                                 int I, int Lp1, double* __restrict__ loglik) {
  const int64_t m = blockIdx.x;
  const int l = blockIdx.y;
  const int64_t G = M * F;
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) s += llg[(size_t)l * G + m * F + f];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    loglik[m * Lp1 + l] = sh[0] - (double)N * (double)F * (double)I * kLogPi;
}

cudaError_t launch_ll_reduce(const double* llg, int64_t M, int64_t F, int64_t N, int I, int nlev,
                             int Lp1, double* loglik, cudaStream_t s) {
  dim3 grid((unsigned)M, (unsigned)nlev);
  ll_reduce_kernel<<<grid, 256, 0, s>>>(llg, M, F, N, I, Lp1, loglik);
  return cudaGetLastError();
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

void plan_chunks(int64_t G, int64_t N, int blocks_per_sm, int64_t* chunk_frames, int* nchunk,
                 int tile_bins, int64_t min_frames, int64_t max_chunks) {
  // Pick the frame chunking that minimises the modelled makespan
  //   waves(tiles * nchunk / resident CTAs) * (frames per chunk + per-CTA overhead)
  // so that the grid does not end on a mostly idle last wave (config 4:
  // 33 bin tiles; config 3: 2056). >= 16 frames per warp per chunk.
  const int64_t tiles = (G + tile_bins - 1) / tile_bins;
  const int64_t slots = (int64_t)sm_count() * (blocks_per_sm > 0 ? blocks_per_sm : 1);
  int64_t max_nc = (N + min_frames - 1) / min_frames;
  if (max_nc < 1) max_nc = 1;
  if (max_nc > 4096) max_nc = 4096;
  if (max_chunks > 0 && max_nc > max_chunks) max_nc = max_chunks;
  constexpr int64_t kOverhead = 24;  // frames-equivalent: P/W load, ring fill, reduction
  int64_t best_cf = N, best_cost = -1;
  for (int64_t nc = 1; nc <= max_nc; ++nc) {
    const int64_t cf = (N + nc - 1) / nc;
    const int64_t ncv = (N + cf - 1) / cf;
    if (ncv != nc) continue;  // same chunking as a smaller nc
    const int64_t waves = (tiles * ncv + slots - 1) / slots;
    const int64_t cost = waves * (cf + kOverhead);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_cf = cf;
    }
  }
  *chunk_frames = best_cf;
  *nchunk = (int)((N + best_cf - 1) / best_cf);
}

}  // namespace ffca
