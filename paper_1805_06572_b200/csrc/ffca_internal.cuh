// Internal launch interfaces shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>

#include "ffca_common.cuh"

namespace ffca {

// Opt a kernel into > 48 KB of dynamic shared memory on the CURRENT device.
// The attribute is per (function, device context), so the "done" record is a
// per-device bit (atomic: several host threads may launch concurrently); a
// process that drives a second GPU sets it again there.
template <auto Kern>
inline cudaError_t ensure_smem(size_t bytes) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

constexpr int kWarps = 4;  // warps per CTA in the frame-streaming kernels
// FCA per-(chunk, bin) partial sums: packed Hermitian B1, B2, X1, X2 with
// sum_n Phi_j / w_j = S_j B_j S_j + S1 X_j S2 (see fca_em_kernel)
constexpr int kFcaParts = 4;

// ---- K3: fused FastFCA transform + E + M (+ likelihood, + images) ----------
struct FastIterParams {
  const void* y;        // (M,N,F,I) complex R
  void* v;              // (M,2,N,F) R, read (and written when update)
  const void* v_src;    // powers read instead of v (null: v), e.g. the caller's init
  const double2* P;     // (G,I,I)
  const double2* W;     // (G,I,I) = P^{-H}; needed when mu_back
  const double* lam;    // (G,I)
  const double* floor;  // (G)
  double* Spart;        // [nchunk][2*I*I][G] partial sums (update)
  double* llbin;        // [nchunk][G] sum_n sum_i log den + |z|^2/den, or null
  void* mu_out;         // (M,2,N,F,I) complex R or null
  int mu_back;          // 1: write W m (images); 0: write m (transformed posterior mean)
  int update;           // v update + S accumulation
  int64_t M, N, F, G;
  int64_t chunk_frames;
  int nchunk;
  ffca_status_dev* st;
  int iter;
  // bin window [g0, g1) of this launch (g1 = 0: to G). g0 is a multiple of
  // the pass's bin tile and g1 is one too or G (bin_window_granularity)
  int64_t g0, g1;
  // launch with programmatic stream serialisation: this pass may start while
  // the previous kernel on the stream (a pass over OTHER bins) drains
  int pdl;
  // plain schedule chained with programmatic dependent launch: the pass was
  // launched while the previous per-bin refresh may still run; it prefetches
  // its first frames, then waits for that kernel (griddepcontrol.wait) before
  // it reads P / lambda, and only then releases its own dependent
  int pdl_wait;
};
// every CTA of a streaming pass releases its programmatic dependents on entry:
// a pass over other bins launched after it with FastIterParams::pdl fills
// the SM slots of its last partial wave instead of waiting for its drain
__device__ __forceinline__ void pdl_release_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// wait until the kernel this one programmatically depends on has completed
// and its memory is visible (a no-op for a normally launched kernel)
__device__ __forceinline__ void pdl_wait_primary() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// whether the plain FastFCA schedule chains its launches (FFCA_PDL_CHAIN=0: off)
bool pdl_chain_enabled();
// kernel launch with the optional programmatic-serialisation attribute
// and an optional scheduling priority (0: the stream's; else a value in the
// device's stream-priority range, lower = more urgent; kept in graph nodes)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, bool pdl, int prio, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (prio) {
    attr[n].id = cudaLaunchAttributePriority;
    attr[n].val.priority = prio;
    ++n;
  }
  cfg.attrs = n ? attr : nullptr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// bins per window step: every window edge is a tile edge of the update pass
// (K3 / K3t / K3p) and of the pencil refresh (K1 / K1p)
int bin_window_granularity(int I, int dtype);
__host__ __device__ inline int64_t window_end(int64_t g1, int64_t G) { return g1 > 0 ? g1 : G; }
cudaError_t launch_fast_em(const FastIterParams& p, int I, int dtype, cudaStream_t s);

// ---- K4: fused conventional FCA iteration (+ likelihood, + mu) -------------
struct FcaIterParams {
  const void* y;        // (M,N,F,I)
  void* v;              // (M,2,N,F)
  const void* v_src;    // powers read instead of v (null: v)
  const double* Sp;     // [2][I*I][G] packed S1, S2 (SoA)
  const double* floor;  // (G)
  double* Spart;        // [nchunk][kFcaParts*I*I][G]: B1, B2, X1, X2 packed
  double* llbin;        // [nchunk][G] sum log det R + y^H R^-1 y, or null
  void* mu_out;         // (M,2,N,F,I) or null
  int update;
  int64_t M, N, F, G;
  int64_t chunk_frames;
  int nchunk;
  ffca_status_dev* st;
  int iter;
  // chained plain schedule (as FastIterParams::pdl_wait): prefetch the first
  // frames, wait for the per-bin finish, release the next finish, load S1 / S2
  int pdl_wait;
};
cudaError_t launch_fca_em(const FcaIterParams& p, int I, int dtype, cudaStream_t s);

// ---- K1: per-bin pencil update ----------------------------------------------
struct PencilParams {
  const double* Spart;  // [nchunk][2*I*I][G]
  int nchunk;
  int64_t N, G;
  double2* P;        // (G,I,I) in: P_e, out: P_next
  double2* W;        // (G,I,I) in: P_e^{-H}, out: P_next^{-H}
  double* lam;       // (G,I) out
  double* logdet2;   // (G) in: logdet2(P_e), out: logdet2(P_next)
  double2* S_model;  // (M,2,F,I,I) out: back-transformed regularised S (model S)
  double2* S_hist;   // (M,2,F,I,I) slice for this iteration or null
  const double* llbin;  // [nchunk][G] or null
  double* llg;          // (G) out or null: N logdet2(P_e) - sum llbin
  int64_t F;
  ffca_status_dev* st;
  int iter;
  double2* St;  // [2][G][I][I] scratch for the split path (I >= 5)
  int64_t g0, g1;  // bin window (g1 = 0: to G), as FastIterParams
  int prio;        // launch priority (0: the stream's), see launch_ex
  int pdl_wait;    // launched programmatically behind the streaming pass (K1, I <= 4): wait
                   // for it before the partials are read, then release the next pass
};
// whether launch_pencil_update honours a bin window (the 3-kernel I >= 5
// path, FFCA_K1=thread, does not)
bool pencil_window_capable(int64_t G, int I);
// whether the refresh is the one-thread-per-bin K1 (honours PencilParams::pdl_wait)
bool pencil_thread_kernel(int64_t G, int I);
cudaError_t launch_pencil_update(const PencilParams& p, int I, cudaStream_t s);

// ---- KP: persistent FastFCA EM kernel (ffca_persist.cuh) ---------------------
// One cooperative launch that runs `iters` whole iterations (pass + refresh)
// of a complex128 I <= 4 problem whose tiles * (nchunk + 1) CTAs are resident
// at once. `sync` = 3 * tiles + 1 zeroed ints (arrival counters, tile
// generations, W generations, abort word). fast_persist_slots: CTAs resident at once (0:
// not available for this order).
struct PersistCtl {
  int* arrive;  // [tiles] chunk CTAs that finished a pass of the tile (cumulative over iterations)
  int* ready;   // [tiles] iterations whose refresh has published P and lambda
  int* wready;  // [tiles] iterations whose refresh has stored W and log|det P|^2 (LAR)
  int* abort;   // [1] a wait timed out
  int tiles, nchunk;
  int iters;    // iterations run inside the kernel (numbered 1..iters as the plain loop's p.iter)
  int lar;      // 1: the last chunk CTA of a tile to arrive refreshes it (no refresher CTAs)
};

#ifndef FFCA_PERSIST_RTILES
#define FFCA_PERSIST_RTILES 4  // tiles (warps) per refresher CTA of KP, 1..4
#endif
bool fast_persist_lar();  // FFCA_PERSIST_LAR (default 1)
inline int64_t persist_refreshers(int64_t tiles) {
  return fast_persist_lar() ? 0 : (tiles + FFCA_PERSIST_RTILES - 1) / FFCA_PERSIST_RTILES;
}
int fast_persist_slots(int I);
int fast_persist_max_chunks(int I);  // (the refresher stages the tile's partials in shared memory)
// shape test of the KP path (order, dtype, size); a run also needs
// tiles * (nchunk + 1) <= fast_persist_slots and no likelihood / history / events.
// fast_persist_wanted: the run's flags (FFCA_FLAG_PERSIST / _NO_PERSIST), the
// FFCA_PERSIST environment override and the measured-win region decide
bool fast_persist_shape(int64_t G, int64_t N, int I, int dtype);
bool fast_persist_wanted(unsigned flags, int64_t G, int64_t N, int I, int dtype);
bool plan_persist_chunks(int64_t G, int64_t N, int I, int dtype, int64_t* chunk_frames,
                         int* nchunk);
cudaError_t launch_fast_persist(const FastIterParams& fp, const PencilParams& pp, int* sync,
                                int tiles, int iters, int I, cudaStream_t s);

// initial pencil from S0 (M,2,F,I,I): P, W, lam, logdet2 (fast.py:127-130)
cudaError_t launch_initial_pencil(const double2* S0, double2* P, double2* W, double* lam,
                                  double* logdet2, int64_t G, int64_t F, int I,
                                  ffca_status_dev* st, cudaStream_t s);

// ---- FCA per-bin steps ------------------------------------------------------
// pack S (M,2,F,I,I) -> Sp [4][I*I][G] with S1,S2 and their Cholesky inverses
cudaError_t launch_fca_prepare(const double2* S, double* Sp, int64_t G, int64_t F, int I,
                               ffca_status_dev* st, int iter, cudaStream_t s);
// reduce partials, regularise (modelops.py:29-39), write S_model (+hist), and
// refresh Sp (S and S^{-1}) for the next iteration; llg (G) collect.
// per-bin FCA prepare (S_in) / finish / stage sums (S_raw), lane-parallel
// (fca_bin_par_kernel, ffca_fca_par.cu)
cudaError_t launch_fca_bin_par(const double* Spart, int nchunk, int64_t N, int64_t G, int64_t F,
                               double* Sp, double2* S_model, double2* S_hist,
                               const double* llbin, double* llg, double2* S_raw,
                               const double2* S_in, int I, ffca_status_dev* st, int iter,
                               cudaStream_t s, int pdl = 0);
// stage API: S_raw (2,G,I,I) = sum_n Phi_j / w_j / N from the chunk partials
cudaError_t launch_fca_sraw(const double* Spart, int nchunk, int64_t N, int64_t G,
                            const double* Sp, double2* S_raw, int I, cudaStream_t s);
cudaError_t launch_fca_finish(const double* Spart, int nchunk, int64_t N, int64_t G, int64_t F,
                              double* Sp, double2* S_model, double2* S_hist,
                              const double* llbin, double* llg, int I, ffca_status_dev* st,
                              int iter, cudaStream_t s, int pdl = 0);
// (pdl: launched programmatically behind the streaming pass, see fca_enqueue; the
// kernel waits for its primary before anything else, then releases its dependent)

// ---- likelihood bookkeeping -------------------------------------------------
// llg[g] = coef_logdet * N * logdet2[g] - sum_c llbin[c][g]   (logdet2 may be null)
cudaError_t launch_ll_collect(const double* llbin, int nchunk, const double* logdet2, int64_t N,
                              int64_t G, double* llg, cudaStream_t s);
// loglik[m*(L+1)+l] = sum_f llg[l][m*F+f] - N F I log(pi)
cudaError_t launch_ll_reduce(const double* llg, int64_t M, int64_t F, int64_t N, int I,
                             int nlev, int Lp1, double* loglik, cudaStream_t s);

// chunking of the frame axis so that the grid fills the GPU without a
// mostly idle last wave; blocks_per_sm = resident CTAs of the streaming kernel
void plan_chunks(int64_t G, int64_t N, int blocks_per_sm, int64_t* chunk_frames, int* nchunk,
                 int tile_bins = 32, int64_t min_frames = 8 * kWarps, int64_t max_chunks = 0);
int fast_blocks_per_sm(int I, int dtype);
// the FastFCA update pass's CTA tile (bins) and resident CTAs per SM
int fast_tile_bins(int I, int dtype);
int fast_update_blocks_per_sm(int I, int dtype);
int fca_blocks_per_sm(int I, int dtype);
// FCA plan: the lane-parallel kernel (I >= 5) tiles fewer bins per CTA and
// streams every frame of a chunk in one lane group
void plan_fca_chunks(int64_t G, int64_t N, int I, int dtype, int64_t* chunk_frames, int* nchunk);
void plan_fast_chunks(int64_t G, int64_t N, int I, int dtype, int64_t* chunk_frames, int* nchunk);
// I >= 5: shapes the driver runs as two bin windows (split-phase, no PDL)
bool fast_par_split_shape(int64_t G, int64_t N, int I);

int sm_count();

}  // namespace ffca
