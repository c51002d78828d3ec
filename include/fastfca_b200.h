/*
 * fastfca_b200.h — C ABI of the B200-native FCA / FastFCA EM library
 * (libfastfca_b200.so, built from paper_1805_06572_b200/csrc/ for sm_100a).
 *
 * Drop-in boundary. The reference package `fastfca` 0.1.0 exposes its hot path
 * at two levels, and this header replaces both:
 *
 *   1. the kernel-backend plugin `_backend.kernels()`
 *      (reference pkg/src/fastfca/_backend.py:57-61), a module exporting the
 *      11 per-(n, f) functions of pkg/src/fastfca/_kernels_numpy.py:19-193 /
 *      _kernels_numba.py:69-391 -> the `ffca_<name>` stage entry points below;
 *   2. the run-level engines `fastfca_run` (pkg/src/fastfca/fast.py:156-260)
 *      and `fca_run` (pkg/src/fastfca/conventional.py:104-164)
 *      -> ffca_fastfca_run / ffca_fca_run, which keep the whole EM loop on the
 *      device (one H2D before, one D2H after; no host round trip per iteration).
 *
 * Conventions
 *   - Plain pointers and sizes only; every array pointer is DEVICE memory
 *     unless its comment says "host".
 *   - complex128 arrays are interleaved (re, im) doubles; complex64 arrays are
 *     interleaved floats. Layouts are the reference's (types.py:1-8,
 *     _kernels_numpy.py:3-13), with a leading mixture axis M for batches:
 *       y (M,N,F,I)   v (M,2,N,F)   S (M,2,F,I,I)   P (M*F,I,I)
 *       lam (M*F,I)   v_floor (M,F)   images / mu (M,2,N,F,I)
 *   - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default);
 *     functions return before the GPU finishes unless stated otherwise.
 *   - Return value: FFCA_OK or FFCA_ERR_INVALID / FFCA_ERR_CUDA for launch-time
 *     failures. Numerical failures found by the kernels (the reference's
 *     exceptions) are written to a device status word and decoded by
 *     ffca_status_read.
 *   - Supported channel counts: 1 <= I <= 8 (BASELINE configs use 2, 3, 4, 8).
 */
#ifndef FASTFCA_B200_H
#define FASTFCA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: map 1:1 onto reference errors.py ------------------- */
#define FFCA_OK 0
#define FFCA_ERR_SINGULAR_MATRIX 1  /* SingularMatrixError, fast.py:39-55 (collapsed powers) */
#define FFCA_ERR_SINGULAR_MIXTURE 2 /* SingularMixtureError(frame, bin), conventional.py:27-38 */
#define FFCA_ERR_DEFINITENESS 3     /* DefinitenessError(min_eigenvalue), pencil.py:114-122 */
#define FFCA_ERR_NON_HERMITIAN 4    /* NonHermitianError, pencil.py:40-51 */
#define FFCA_ERR_SINGULAR_BASIS 5   /* SingularMatrixError, fast.py:137-140 (basis solve) */
#define FFCA_ERR_NOT_PD 6           /* numpy LinAlgError from cholesky, conventional.py:98-101 */
#define FFCA_ERR_NO_CONVERGENCE 7   /* numpy LinAlgError from eigh (heevd did not converge),
                                       pencil.py:72,113,130; here: Jacobi sweep limit */
#define FFCA_ERR_INVALID 10         /* bad argument (shape, dtype, NULL pointer) */
#define FFCA_ERR_CUDA 11            /* CUDA runtime failure */

#define FFCA_C128 0 /* complex128 streaming (the reference's only precision) */
#define FFCA_C64 1  /* complex64 streaming, float64 per-bin state */

/* run flags */
#define FFCA_FLAG_LIKELIHOOD 1u /* fill loglik (reference compute_likelihood) */
#define FFCA_FLAG_HISTORY 2u    /* fill S_hist / v_hist (reference record_history) */
#define FFCA_FLAG_IMAGES 4u     /* write the separated images */
#define FFCA_FLAG_GRAPH 8u      /* capture the run's launch sequence as a CUDA graph on the
                                 * first call with these exact arguments and replay it on
                                 * later identical calls (repeated runs on fixed buffers);
                                 * ignored when iter_events / kernel_events are given */
#define FFCA_FLAG_PERSIST 16u   /* FastFCA: use the persistent EM kernel whenever the run fits it
                                 * (complex128, I <= 4, no likelihood / history / events, the
                                 * whole pass grid resident): the first L-1 iterations in ONE
                                 * cooperative launch (streaming + refresher CTAs, per-tile
                                 * flags). Without the flag it is used on the shapes where it
                                 * measured faster; same arithmetic as the plain schedule */
#define FFCA_FLAG_NO_PERSIST 32u /* never use the persistent EM kernel */

/* Device-side status word (lives in the run workspace, or caller-allocated
 * for the stage entry points). Zero-initialise with ffca_status_reset. */
typedef struct ffca_status_dev {
  unsigned long long first; /* min over (iteration<<48 | code<<44 | index) */
  double value;             /* definiteness: worst minimum eigenvalue */
} ffca_status_dev;

/* Host-side decoded status. */
typedef struct ffca_status {
  int code;        /* FFCA_OK or FFCA_ERR_* */
  int iteration;   /* EM iteration that failed (-1 = initial pencil / pre-loop) */
  long long index; /* flat (m, n, f) point or (m, f) bin, per code */
  double value;    /* min eigenvalue for FFCA_ERR_DEFINITENESS */
} ffca_status;

/* Run-level arguments for ffca_fastfca_run / ffca_fca_run. */
typedef struct ffca_run_args {
  int64_t M, N, F; /* mixtures, frames, bins */
  int I;           /* channels */
  int dtype;       /* FFCA_C128 | FFCA_C64 (y, v, images, v_hist) */
  int iterations;  /* L >= 0 */
  unsigned flags;  /* FFCA_FLAG_* */
  const void* y;   /* (M,N,F,I) complex */
  void* v;         /* (M,2,N,F) real: init powers in, final powers out (in place) */
  const double* S0;      /* (M,2,F,I,I) complex128 init covariances */
  const double* v_floor; /* (M,F) float64 */
  void* images;          /* (M,2,N,F,I) complex out (FFCA_FLAG_IMAGES) */
  double* S_out;         /* (M,2,F,I,I) complex128 out: final model S */
  double* loglik;        /* (M, L+1) float64 out (FFCA_FLAG_LIKELIHOOD) */
  double* S_hist;        /* (L,M,2,F,I,I) complex128 or NULL */
  void* v_hist;          /* (L,M,2,N,F) real or NULL */
  void* workspace;       /* >= ffca_*_workspace_size bytes, 256-B aligned */
  size_t workspace_bytes;
  void* const* iter_events; /* optional cudaEvent_t[L+1] recorded at iteration edges */
  int64_t chunk_frames;     /* frames per reduction chunk; 0 = auto (ffca_plan_chunks).
                               Runs with equal chunk_frames give bitwise-identical per-bin
                               results however the bins / mixtures are sharded. */
  void* const* kernel_events; /* optional cudaEvent_t[2L]: before/after each fused streaming
                                 pass (the dominant kernel), for roofline timing */
  const void* v_in; /* optional (M,2,N,F) initial powers, read only: the first pass reads
                       them here and writes `v` (which then need not be initialised);
                       NULL = `v` holds the initial powers (in place) */
  int bin_parts;    /* FastFCA split-phase schedule: the bins in this many windows; window
                       i's per-bin pencil refresh runs on a second (per-thread, per-device)
                       stream while window i+1 streams, the passes chained with
                       programmatic serialisation. 0 = auto (ffca_plan_parts), 1 = one
                       window (plain schedule; also forced with FFCA_FLAG_HISTORY).
                       Results are bitwise independent of it. */
} ffca_run_args;

/* ---- library info ------------------------------------------------------ */
const char* ffca_version(void);
int ffca_device_arch(void); /* compiled SM arch, e.g. 100 */

/* ---- run level (fast.py:156-260, conventional.py:104-164) -------------- */
/* Frame-axis chunking the drivers use for G = M*F bins and N frames
 * (algorithm 0 = FastFCA, 1 = FCA; needs a device for the occupancy query). */
int ffca_plan_chunks(int64_t G, int64_t N, int I, int dtype, int algorithm,
                     int64_t* chunk_frames, int* nchunk);
/* Grid of the streaming pass for that plan (chunk_frames 0 = the auto plan):
 * *ctas = bin tiles x frame chunks, *slots = resident CTAs on the whole device
 * (SM count x CTAs per SM); ctas / slots = waves. Needs a device. */
/* Bin windows the FastFCA driver pipelines (bin_parts = 0): 1 = none.
 * Needs a device. */
int ffca_plan_parts(int64_t G, int64_t N, int I, int dtype, int algorithm);
int ffca_plan_grid(int64_t G, int64_t N, int I, int dtype, int algorithm, int64_t chunk_frames,
                   int64_t* ctas, int64_t* slots);
size_t ffca_fastfca_workspace_size(int64_t M, int64_t N, int64_t F, int I, int iterations,
                                   unsigned flags, int64_t chunk_frames);
int ffca_fastfca_run(const ffca_run_args* args, void* stream);
size_t ffca_fca_workspace_size(int64_t M, int64_t N, int64_t F, int I, int iterations,
                               unsigned flags, int64_t chunk_frames);
int ffca_fca_run(const ffca_run_args* args, void* stream);
/* Decode the status word kept in a run workspace; synchronises `stream`. */
/* release every cached run graph (FFCA_FLAG_GRAPH) */
int ffca_graph_cache_clear(void);
int ffca_run_status(const void* workspace, void* stream, ffca_status* out);

/* ---- status words for the stage entry points --------------------------- */
int ffca_status_reset(ffca_status_dev* st, void* stream);
/* Synchronises `stream`, copies and decodes. */
int ffca_status_read(const ffca_status_dev* st, void* stream, ffca_status* out);
/* Decode a status word that is already in HOST memory (e.g. copied
 * asynchronously out of a run workspace before the workspace is reused). */
int ffca_status_decode(const ffca_status_dev* host_word, ffca_status* out);

/* ---- kernel-module contract (_kernels_numpy.py:19-193; M = 1) ---------- */
/* fast_transform: yt = P^H y  (_kernels_numba.py:147-162) */
int ffca_fast_transform(const double* y, const double* P, double* yt, int64_t N, int64_t F,
                        int I, void* stream);
/* fast_e_step: (mu, Phi) in the diagonal basis (_kernels_numba.py:165-193) */
int ffca_fast_e_step(const double* yt, const double* v, const double* lam, double* mu,
                     double* Phi, int64_t N, int64_t F, int I, void* stream);
/* fast_v_update: v from diag(Phi) (_kernels_numba.py:196-213), unfloored */
int ffca_fast_v_update(const double* Phi, const double* lam, double* v, int64_t N, int64_t F,
                       int I, void* stream);
/* fast_S_update / fca_S_update: (1/N) sum_n Phi / v (_kernels_numba.py:98-113,216-217) */
int ffca_S_update(const double* Phi, const double* v, double* S, int64_t N, int64_t F, int I,
                  void* stream);
/* fast_log_likelihood -> *out (device scalar) (_kernels_numba.py:220-243) */
int ffca_fast_log_likelihood(const double* yt, const double* v, const double* lam,
                             const double* logdet2, double* out, int64_t N, int64_t F, int I,
                             void* stream);
/* fast_iteration: fused transform+E+M (_kernels_numba.py:328-391) */
int ffca_fast_iteration(const double* y, const double* P, const double* v, const double* lam,
                        const double* v_floor, double* mu, double* v_new, double* S_raw,
                        int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream);
/* fca_e_step: frame-wise inverse posterior (_kernels_numba.py:12-72) */
int ffca_fca_e_step(const double* y, const double* v, const double* S, double* mu, double* Phi,
                    int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream);
/* fca_v_update: tr(S_prev^{-1} Phi)/I (_kernels_numba.py:75-95), unfloored */
int ffca_fca_v_update(const double* Phi, const double* S_prev, double* v, int64_t N, int64_t F,
                      int I, ffca_status_dev* st, void* stream);
/* fca_log_likelihood -> *out (device scalar) (_kernels_numba.py:116-144) */
int ffca_fca_log_likelihood(const double* y, const double* v, const double* S, double* out,
                            int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream);
/* fca_iteration: fused conventional E+M (_kernels_numba.py:246-325) */
int ffca_fca_iteration(const double* y, const double* v, const double* S, const double* Sinv,
                       const double* v_floor, double* mu, double* v_new, double* S_raw,
                       int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream);

/* ---- per-bin linear algebra (pencil.py, fast.py:107-153, conventional.py:98-101) */
/* gevd_hpd over a batch of pencils (pencil.py:85-135): lam (B,D) desc, P (B,D,D) */
int ffca_gevd_hpd(const double* Phi, const double* Psi, double* lam, double* P, int64_t batch,
                  int D, int check_hermitian, ffca_status_dev* st, void* stream);
/* propagate_pencil (fast.py:107-124): P_next = P_prev Q, lam */
int ffca_propagate_pencil(const double* St1, const double* St2, const double* P_prev,
                          double* P_next, double* lam, int64_t batch, int D,
                          ffca_status_dev* st, void* stream);
/* S^{-1} = L^{-H} L^{-1} (conventional.py:98-101) */
int ffca_cholesky_inverse(const double* S, double* Sinv, int64_t batch, int D,
                          ffca_status_dev* st, void* stream);
/* solve_hermitian_system (pencil.py:138-157): X = A^{-1} B per batch entry by LU with
 * partial pivoting (np.linalg.solve / zgesv); A (batch,D,D), B and X (batch,D,K) complex128;
 * norms (batch,2) float64 out: ||A X - B||^2 and ||B||^2 of each entry. An exactly
 * singular A reports FFCA_ERR_SINGULAR_MATRIX (index = batch entry). */
int ffca_solve(const double* A, const double* B, double* X, double* norms, int64_t batch,
               int D, int64_t K, ffca_status_dev* st, void* stream);
/* hermitize + 1e-9 tr/D ridge (modelops.py:29-39) */
int ffca_regularize_covariances(const double* S, double* out, int64_t batch, int D,
                                void* stream);
/* hermitize + eps*gram ridge, eps = 1e-9 tr(gram^{-1} S)/D (fast.py:80-90);
 * gram == NULL -> eps = 1e-9 tr(S)/D with an identity ridge */
int ffca_regularize_transformed(const double* S_raw, const double* gram, double* out,
                                int64_t batch, int D, void* stream);
/* solve P^H mu = mu_t per bin (fast.py:133-141); mu_t, out: (Src,N,F,I) */
int ffca_back_transform_images(const double* mu_t, const double* P, double* out, int64_t Src,
                               int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream);
/* (P^H)^{-1} S_t P^{-1} per bin (fast.py:144-148); S_t, out: (Src,F,I,I) */
int ffca_back_transform_covariances(const double* S_t, const double* P, double* out,
                                    int64_t Src, int64_t F, int I, ffca_status_dev* st,
                                    void* stream);
/* 2 log|det P| per bin (fast.py:151-153) */
int ffca_logdet2(const double* P, double* out, int64_t batch, int D, void* stream);
/* init_random powers/floor from y (initializers.py:20-39, modelops.py:12-21):
 * v (M,2,N,F) = max(||y||^2/(2I), floor), v_floor (M,F) */
int ffca_init_powers(const void* y, void* v, double* v_floor, int64_t M, int64_t N, int64_t F,
                     int I, int dtype, void* stream);

/* ---- mask-clustering initial model (reference initializers.py:42-143) -----
 * y (M,N,F,I) complex128 -> v (M,2,N,F) f64, S (M,2,F,I,I) c128, v_floor (M,F):
 * per-bin deterministic 2-means of the phase-aligned unit observations, unit-
 * trace group covariances + 1e-2 ridge, cross-bin label alignment, masked
 * floored powers. Needs N >= 2 I (the reference falls back to init_random(y, 0)
 * below that; the caller does too). */
size_t ffca_init_masks_workspace_size(int64_t M, int64_t N, int64_t F, int I);
int ffca_init_masks(const double* y, double* v, double* S, double* v_floor, int64_t M, int64_t N,
                    int64_t F, int I, void* workspace, size_t workspace_bytes, void* stream);

/* ---- STFT front / back end (reference stft.py:9-107) ----------------------
 * Square-root periodic Hann window, frame_shift = frame_length / 2, half a
 * frame of leading zeros; frame_length a power of two in [2, 8192].
 * frames = max((length - 1) / shift + 2, 2)   (stft.py:30-32, num_frames) */
int64_t ffca_stft_frames(int64_t length, int frame_shift);
/* stft_analyze (stft.py:35-70): x (batch, channels, length) f64 ->
 * spec (batch, frames, frame_length/2 + 1, channels) c128 */
int ffca_stft_analyze(const double* x, double* spec, int64_t batch, int channels, int64_t length,
                      int frame_length, void* stream);
/* stft_synthesize (stft.py:73-107): spec (batch, frames, frame_length/2 + 1,
 * channels) c128 -> out (batch, channels, length) f64, DC / Nyquist taken as
 * real, overlap-add trimmed to [shift, shift + length); length <= frames * shift */
int ffca_stft_synthesize(const double* spec, double* out, int64_t batch, int channels,
                         int64_t frames, int frame_length, int64_t length, void* stream);

/* ---- separation quality (reference metrics.py) ---------------------------
 * sdr (metrics.py:27-60, _channel_sdr): for each signal pair p of est, ref
 * (pairs, length) f64 (device), the least-squares projection of est onto ref
 * delayed by 0..max_shift samples (max_shift <= 63); sdr_db[p] =
 * 10 log10(target / max(noise, 1e-30 target)), -300 for a zero projection.
 * flags[p]: bit 0 = silent reference (MetricError), bit 1 = numerically
 * rank-deficient delay basis (dependent delays dropped). pairs <= 65535.
 * Deterministic (fixed-order reductions). */
size_t ffca_sdr_workspace_size(int64_t pairs, int64_t length, int max_shift);
int ffca_sdr(const double* est, const double* ref, int64_t pairs, int64_t length, int max_shift,
             double* sdr_db, int* flags, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FASTFCA_B200_H */
