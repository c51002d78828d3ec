// extern "C" entry points: the device-resident EM drivers (the native runtime
// of the hot path) and the per-bin batched routines.
//
// ffca_fastfca_run mirrors fastfca_run (reference fast.py:156-260) and
// ffca_fca_run mirrors fca_run (conventional.py:104-164): same iteration
// structure, same likelihood / history / image semantics, but every step is
// a kernel on one stream and nothing returns to the host inside the loop.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <mutex>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "ffca_internal.cuh"

namespace ffca {
cudaError_t launch_gevd_batch(const double2* Phi, const double2* Psi, double* lam, double2* P,
                              const double2* Pprev, int64_t B, int I, int check,
                              ffca_status_dev* st, cudaStream_t s);
cudaError_t launch_cholinv(const double2* S, double2* Sinv, int64_t B, int I, ffca_status_dev* st,
                           cudaStream_t s);
cudaError_t launch_regularize(const double2* S, double2* out, int64_t B, int I, cudaStream_t s);
cudaError_t launch_solve(const double2* A, const double2* B, double2* X, double* norms,
                         int64_t batch, int I, int64_t K, ffca_status_dev* st, cudaStream_t s);
cudaError_t launch_reg_transformed(const double2* S, const double2* gram, double2* out,
                                   int64_t B, int I, cudaStream_t s);
cudaError_t launch_inverse_h(const double2* P, double2* W, double* logdet2, int64_t B, int I,
                             ffca_status_dev* st, cudaStream_t s);
cudaError_t launch_apply_w(const double2* mu_t, const double2* W, double2* out, int64_t Src,
                           int64_t N, int64_t F, int I, cudaStream_t s);
cudaError_t launch_conj_w(const double2* S, const double2* W, double2* out, int64_t Src,
                          int64_t F, int I, cudaStream_t s);
cudaError_t launch_init_powers(const void* y, void* v, double* floor, int64_t M, int64_t N,
                               int64_t F, int I, int dtype, cudaStream_t s);
int fast_par_blocks_per_sm(int I, int dtype);
int fast_par_bins_per_cta();
int fca_par_blocks_per_sm(int I, int dtype);
int fca_par_bins_per_cta(int I);
}  // namespace ffca

using namespace ffca;

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* b) : base((char*)b) {}
  template <typename T>
  T* take(size_t count) {
    T* p = base ? (T*)(base + off) : nullptr;
    off += align_up(count * sizeof(T));
    return p;
  }
};

struct FastWs {
  ffca_status_dev* st;
  double2 *P, *W, *St;
  double *lam, *logdet2, *Spart, *llbin, *llg;
  int* sync;  // KP: 3 * tiles + 1 ints (arrival counters, tile / W generations, abort word)
  int64_t chunk_frames;
  int nchunk;
  size_t bytes;
};

bool chunk_override(int64_t N, int64_t cf_req, int64_t* cf, int* nc) {
  if (cf_req <= 0) return false;
  *cf = cf_req < N ? cf_req : N;
  *nc = (int)((N + *cf - 1) / *cf);
  return true;
}

FastWs carve_fast(void* base, int64_t M, int64_t N, int64_t F, int I, int L, unsigned flags,
                  int64_t cf_req, int dtype) {
  FastWs w{};
  const int64_t G = M * F;
  if (!chunk_override(N, cf_req, &w.chunk_frames, &w.nchunk)) {
    if (!(fast_persist_wanted(flags, G, N, I, dtype) &&
          plan_persist_chunks(G, N, I, dtype, &w.chunk_frames, &w.nchunk)))
      plan_fast_chunks(G, N, I, dtype, &w.chunk_frames, &w.nchunk);
  }
  Carve c(base);
  w.st = c.take<ffca_status_dev>(1);
  w.P = c.take<double2>(G * I * I);
  w.W = c.take<double2>(G * I * I);
  w.lam = c.take<double>(G * I);
  w.logdet2 = c.take<double>(G);
  w.Spart = c.take<double>((size_t)w.nchunk * 2 * I * I * G);
  w.sync = c.take<int>(3 * ((G + 31) / 32) + 1);
  const bool ll = flags & FFCA_FLAG_LIKELIHOOD;
  w.llbin = ll ? c.take<double>((size_t)w.nchunk * G) : nullptr;
  w.llg = ll ? c.take<double>((size_t)(L + 1) * G) : nullptr;
  w.St = I >= 5 ? c.take<double2>((size_t)2 * G * I * I) : nullptr;
  w.bytes = c.off;
  return w;
}

struct FcaWs {
  ffca_status_dev* st;
  double *Sp, *Spart, *llbin, *llg;
  int64_t chunk_frames;
  int nchunk;
  size_t bytes;
};

FcaWs carve_fca(void* base, int64_t M, int64_t N, int64_t F, int I, int L, unsigned flags,
                int64_t cf_req, int dtype) {
  FcaWs w{};
  const int64_t G = M * F;
  if (!chunk_override(N, cf_req, &w.chunk_frames, &w.nchunk))
    plan_fca_chunks(G, N, I, dtype, &w.chunk_frames, &w.nchunk);
  Carve c(base);
  w.st = c.take<ffca_status_dev>(1);
  w.Sp = c.take<double>((size_t)2 * I * I * G);
  w.Spart = c.take<double>((size_t)w.nchunk * kFcaParts * I * I * G);
  const bool ll = flags & FFCA_FLAG_LIKELIHOOD;
  w.llbin = ll ? c.take<double>((size_t)w.nchunk * G) : nullptr;
  w.llg = ll ? c.take<double>((size_t)(L + 1) * G) : nullptr;
  w.bytes = c.off;
  return w;
}

int check_args(const ffca_run_args* a) {
  if (!a || a->M < 1 || a->N < 1 || a->F < 1 || a->I < 1 || a->I > kMaxOrder ||
      a->iterations < 0 || a->iterations > 65000 || a->chunk_frames < 0 || !a->y || !a->v || !a->S0 || !a->v_floor ||
      !a->S_out || !a->workspace)
    return FFCA_ERR_INVALID;
  if (a->dtype != FFCA_C128 && a->dtype != FFCA_C64) return FFCA_ERR_INVALID;
  // bin indices are split into (mixture, bin) with 32-bit divisions in the kernels
  if (a->M * a->F >= 0x7fffffff || a->N * a->F >= ((int64_t)1 << 40)) return FFCA_ERR_INVALID;
  if ((a->flags & FFCA_FLAG_IMAGES) && !a->images) return FFCA_ERR_INVALID;
  if ((a->flags & FFCA_FLAG_LIKELIHOOD) && !a->loglik) return FFCA_ERR_INVALID;
  if (((size_t)a->workspace) % kAlign) return FFCA_ERR_INVALID;
  return FFCA_OK;
}

inline int cu(cudaError_t e) { return e == cudaSuccess ? FFCA_OK : FFCA_ERR_CUDA; }
// FFCA_DEBUG_SYNC=1: synchronise after every launch and name the failing step
inline bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FFCA_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
inline cudaError_t checked(cudaError_t e, const char* what, int line) {
  if (e == cudaSuccess && debug_sync()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess && debug_sync())
    fprintf(stderr, "ffca: %s (capi line %d) failed: %s\n", what, line, cudaGetErrorString(e));
  return e;
}
#define FFCA_TRY(expr)                                   \
  do {                                                   \
    int _rc = cu(checked((expr), #expr, __LINE__));      \
    if (_rc != FFCA_OK) return _rc;                      \
  } while (0)

inline size_t real_size(int dtype) { return dtype == FFCA_C64 ? 4 : 8; }

void decode(const ffca_status_dev& d, ffca_status* out) {
  if (d.first == ~0ull) {
    out->code = FFCA_OK;
    out->iteration = 0;
    out->index = -1;
    out->value = 0.0;
    return;
  }
  out->iteration = (int)((d.first >> 48) & 0xffff) - 1;
  out->code = (int)((d.first >> 44) & 0xf);
  out->index = (long long)(d.first & ((1ull << 44) - 1));
  out->value = d.value;
}

__global__ void status_init_kernel(ffca_status_dev* st) {
  st->first = ~0ull;
  st->value = 1e308;
}

int reset_status(ffca_status_dev* st, cudaStream_t s) {
  status_init_kernel<<<1, 1, 0, s>>>(st);
  return cu(cudaGetLastError());
}

}  // namespace

extern "C" {
static int fastfca_enqueue(const ffca_run_args* a, cudaStream_t s);
static int fca_enqueue(const ffca_run_args* a, cudaStream_t s);
}

namespace {

// ---- run graphs (FFCA_FLAG_GRAPH) -------------------------------------------
// The launch sequence of a run is a pure function of its arguments (and the
// device), so it is captured once into a CUDA graph and replayed: one graph
// launch instead of 2L+3 kernel launches, and graph-internal dependencies
// instead of stream launch gaps (~6 us each on the small configs).
struct GraphEntry {
  std::string key;
  cudaGraphExec_t exec;
};
std::mutex g_graph_mu;
std::list<GraphEntry> g_graphs;  // most recently used first
constexpr size_t kGraphCacheMax = 64;

int run_graph(int algorithm, const ffca_run_args* a, cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FFCA_ERR_CUDA;
  std::string key((const char*)a, sizeof(*a));
  key.push_back((char)algorithm);
  key.append((const char*)&dev, sizeof(dev));
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it) {
    if (it->key == key) {
      g_graphs.splice(g_graphs.begin(), g_graphs, it);
      return cu(cudaGraphLaunch(g_graphs.front().exec, s));
    }
  }
  cudaStream_t cs = nullptr;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return FFCA_ERR_CUDA;
  int rc = cu(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
  if (rc == FFCA_OK) {
    rc = algorithm ? fca_enqueue(a, cs) : fastfca_enqueue(a, cs);
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (rc == FFCA_OK && e != cudaSuccess) rc = FFCA_ERR_CUDA;
    cudaGraphExec_t exec = nullptr;
    if (rc == FFCA_OK) rc = cu(cudaGraphInstantiate(&exec, graph, 0));
    if (graph) cudaGraphDestroy(graph);
    if (rc == FFCA_OK) {
      if (g_graphs.size() >= kGraphCacheMax) {
        cudaGraphExecDestroy(g_graphs.back().exec);
        g_graphs.pop_back();
      }
      g_graphs.push_front(GraphEntry{std::move(key), exec});
      rc = cu(cudaGraphLaunch(exec, s));
    }
  }
  cudaStreamDestroy(cs);
  return rc;
}

// NVTX range around a run's enqueue (header-only NVTX v3: free without a
// tool attached; named with the run's shape for nsys / ncu --nvtx filters)
struct NvtxRun {
  NvtxRun(const char* what, const ffca_run_args* a) {
    char buf[160];
    snprintf(buf, sizeof buf, "%s M=%lld N=%lld F=%lld I=%d L=%d %s%s", what, (long long)a->M,
             (long long)a->N, (long long)a->F, a->I, a->iterations,
             a->dtype == FFCA_C64 ? "c64" : "c128",
             (a->flags & FFCA_FLAG_GRAPH) ? " graph" : "");
    nvtxRangePushA(buf);
  }
  ~NvtxRun() { nvtxRangePop(); }
};

struct NvtxIter {  // one EM iteration's launches
  explicit NvtxIter(int l) {
    char buf[32];
    snprintf(buf, sizeof buf, "em iteration %d", l);
    nvtxRangePushA(buf);
  }
  ~NvtxIter() { nvtxRangePop(); }
};

// the stream the split-phase schedule runs the pencil refreshes on: one per
// (host thread, device), high priority so the refresh CTAs are placed ahead
// of the queued streaming-pass CTAs as SM slots free up
cudaStream_t side_stream() {
  thread_local cudaStream_t ss[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!ss[dev]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&ss[dev], cudaStreamNonBlocking, hi) != cudaSuccess)
      ss[dev] = nullptr;
  }
  return ss[dev];
}

// FFCA_PDL=0: split-phase passes launched without programmatic serialisation
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FFCA_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// bin windows of the split-phase FastFCA schedule. The per-bin pencil refresh
// (K1 / K1p) is latency bound (one thread / lane group per bin, a serial GEVD)
// and in the plain schedule the GPU idles behind it every iteration (config
// 4: K1p 45 of 500 us). With k windows, window i's refresh runs on a second
// stream while window i+1 streams (the next pass launched with programmatic
// serialisation, so it also fills the previous pass's last wave).
// Measured (profiles/r02_split_phase.txt): config 4 +6% at k = 3-4; config 3
// +-1% (K1 holds the whole register file while it runs: a throughput cost,
// not a latency one); configs 0-2 lose (their passes are latency bound per
// CTA, so a window's pass takes as long as a full one). The auto plan splits
// only large single-mixture problems at I <= 4. FFCA_PARTS=k overrides.
int auto_parts(int64_t M, int64_t F, int64_t N, int I, int dtype) {
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("FFCA_PARTS");
    env = e ? atoi(e) : -1;
  }
  const int64_t G = M * F;
  int k = env > 0 ? env : ((M == 1 && I <= 4 && G * N >= ((int64_t)4 << 20)) ? 3 : 1);
  if (env <= 0 && fast_par_split_shape(G, N, I)) k = 2;
  const int64_t maxk = G / bin_window_granularity(I, dtype);  // windows of >= one tile
  if (k > maxk) k = (int)(maxk > 1 ? maxk : 1);
  return k < 1 ? 1 : k;
}

int plan_parts(const ffca_run_args* a) {
  const int64_t G = a->M * a->F;
  if (a->flags & FFCA_FLAG_HISTORY) return 1;  // per-iteration v snapshots need a join
  if (!pencil_window_capable(G, a->I)) return 1;
  int k = a->bin_parts > 0 ? a->bin_parts : auto_parts(a->M, a->F, a->N, a->I, a->dtype);
  const int64_t maxk = G / bin_window_granularity(a->I, a->dtype);
  if (k > maxk) k = (int)(maxk > 1 ? maxk : 1);
  return k < 1 ? 1 : (k > 16 ? 16 : k);
}

// largest run (TF-bins) whose plain schedule is chained with programmatic
// dependent launch (see fastfca_enqueue / fca_enqueue)
// (measured per shape, profiles/r02_pdl_chain_probe.txt: I = 2 gains 6-12% up to
// ~600k TF-bins and loses up to 9% at 1-2M; I = 3 gains nothing beyond 300k and
// loses up to 11% at 1-2M; FFCA_PDL_CHAIN_MAX overrides)
int64_t pdl_chain_max_points(int I) {
  static int64_t v = -2;
  if (v == -2) {
    const char* e = getenv("FFCA_PDL_CHAIN_MAX");
    v = (e && *e) ? atoll(e) : -1;
  }
  if (v >= 0) return v;
  return I <= 2 ? 600000 : 300000;
}

bool graph_mode(const ffca_run_args* a) {
  return (a->flags & FFCA_FLAG_GRAPH) && !a->iter_events && !a->kernel_events && !debug_sync();
}

}  // namespace

extern "C" {

const char* ffca_version(void) { return "fastfca_b200 0.1.0 (sm_100a)"; }

int ffca_device_arch(void) { return 100; }

int ffca_plan_chunks(int64_t G, int64_t N, int I, int dtype, int algorithm,
                     int64_t* chunk_frames, int* nchunk) {
  if (G < 1 || N < 1 || I < 1 || I > kMaxOrder || !chunk_frames || !nchunk)
    return FFCA_ERR_INVALID;
  if (algorithm)
    plan_fca_chunks(G, N, I, dtype, chunk_frames, nchunk);
  else
    plan_fast_chunks(G, N, I, dtype, chunk_frames, nchunk);
  return FFCA_OK;
}

int ffca_plan_parts(int64_t G, int64_t N, int I, int dtype, int algorithm) {
  if (G < 1 || N < 1 || I < 1 || I > kMaxOrder) return FFCA_ERR_INVALID;
  if (algorithm || !pencil_window_capable(G, I)) return 1;
  return auto_parts(1, G, N, I, dtype);
}

int ffca_plan_grid(int64_t G, int64_t N, int I, int dtype, int algorithm, int64_t chunk_frames,
                   int64_t* ctas, int64_t* slots) {
  if (G < 1 || N < 1 || I < 1 || I > kMaxOrder || !ctas || !slots) return FFCA_ERR_INVALID;
  int64_t cf = chunk_frames;
  int nc = 0;
  if (cf <= 0) {
    if (algorithm)
      plan_fca_chunks(G, N, I, dtype, &cf, &nc);
    else
      plan_fast_chunks(G, N, I, dtype, &cf, &nc);
  }
  if (cf > N) cf = N;
  nc = (int)((N + cf - 1) / cf);
  int bpsm, tile;
  if (algorithm) {
    bpsm = I >= 5 ? fca_par_blocks_per_sm(I, dtype) : fca_blocks_per_sm(I, dtype);
    tile = I >= 5 ? fca_par_bins_per_cta(I) : 32;
  } else {
    bpsm = fast_update_blocks_per_sm(I, dtype);
    tile = fast_tile_bins(I, dtype);
  }
  *ctas = (G + tile - 1) / tile * nc;
  *slots = (int64_t)sm_count() * bpsm;
  return FFCA_OK;
}

size_t ffca_fastfca_workspace_size(int64_t M, int64_t N, int64_t F, int I, int iterations,
                                   unsigned flags, int64_t chunk_frames) {
  if (M < 1 || N < 1 || F < 1 || I < 1 || I > kMaxOrder || iterations < 0) return 0;
  // chunk count is largest for the most-occupant dtype: size for both
  const size_t a = carve_fast(nullptr, M, N, F, I, iterations, flags, chunk_frames, FFCA_C128).bytes;
  const size_t b = carve_fast(nullptr, M, N, F, I, iterations, flags, chunk_frames, FFCA_C64).bytes;
  return a > b ? a : b;
}

int ffca_graph_cache_clear(void) {
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (auto& g : g_graphs) cudaGraphExecDestroy(g.exec);
  g_graphs.clear();
  return FFCA_OK;
}

int ffca_fastfca_run(const ffca_run_args* a, void* stream) {
  const int rc = check_args(a);
  if (rc) return rc;
  const NvtxRun range("ffca_fastfca_run", a);
  if (graph_mode(a)) return run_graph(0, a, (cudaStream_t)stream);
  return fastfca_enqueue(a, (cudaStream_t)stream);
}

int ffca_fca_run(const ffca_run_args* a, void* stream) {
  const int rc = check_args(a);
  if (rc) return rc;
  const NvtxRun range("ffca_fca_run", a);
  if (graph_mode(a)) return run_graph(1, a, (cudaStream_t)stream);
  return fca_enqueue(a, (cudaStream_t)stream);
}

size_t ffca_fca_workspace_size(int64_t M, int64_t N, int64_t F, int I, int iterations,
                               unsigned flags, int64_t chunk_frames) {
  if (M < 1 || N < 1 || F < 1 || I < 1 || I > kMaxOrder || iterations < 0) return 0;
  const size_t a = carve_fca(nullptr, M, N, F, I, iterations, flags, chunk_frames, FFCA_C128).bytes;
  const size_t b = carve_fca(nullptr, M, N, F, I, iterations, flags, chunk_frames, FFCA_C64).bytes;
  return a > b ? a : b;
}

// Split-phase EM loop (L >= 1, no history): the bins in k windows [e_i, e_i+1)
// with tile-aligned edges. Main stream: pass(0, l), pass(1, l), ..., each
// after its window's previous refresh; side stream: refresh(i, l) after
// pass(i, l). So refresh(i, l) overlaps pass(i+1, l) (and the next
// iteration's first passes), and every per-bin quantity sees exactly the
// plain schedule's sequence of kernels (bitwise-identical results: the
// windows only restrict which bins a launch covers). On return the main
// stream has joined the side stream.
static int fastfca_split_loop(const ffca_run_args* a, const FastWs& w, FastIterParams p, int k,
                              cudaStream_t s) {
  const int64_t G = a->M * a->F;
  const int I = a->I, L = a->iterations;
  const unsigned fl = a->flags;
  const bool ll = fl & FFCA_FLAG_LIKELIHOOD;
  const bool vin = a->v_in && a->v_in != a->v;
  cudaEvent_t* ev = (cudaEvent_t*)a->iter_events;
  cudaEvent_t* kev = (cudaEvent_t*)a->kernel_events;
  const int gran = bin_window_granularity(I, a->dtype);
  int64_t edge[17];
  const int64_t tiles = (G + gran - 1) / gran;
  int nw = 0;
  edge[0] = 0;
  for (int i = 1; i <= k; ++i) {
    int64_t e = (i == k) ? G : ((tiles * i + k / 2) / k) * gran;
    if (e > G) e = G;
    if (e > edge[nw]) edge[++nw] = e;
  }
  cudaStream_t side = side_stream();
  if (!side) return FFCA_ERR_CUDA;
  int lo_prio = 0, hi_prio = 0;  // the refreshes are dispatched ahead of queued pass CTAs
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  // events: fork, pass_done[i], ref_done[i] (re-recorded every iteration;
  // each wait binds to the latest record enqueued before it)
  cudaEvent_t evs[1 + 2 * 16];
  int ne = 0;
  int rc = FFCA_OK;
  for (; ne < 1 + 2 * nw; ++ne)
    if (cudaEventCreateWithFlags(&evs[ne], cudaEventDisableTiming) != cudaSuccess) {
      rc = FFCA_ERR_CUDA;
      break;
    }
  cudaEvent_t* pass_done = evs + 1;
  cudaEvent_t* ref_done = evs + 1 + nw;
#define FFCA_TRY_S(expr)                                  \
  do {                                                    \
    rc = cu(checked((expr), #expr, __LINE__));            \
    if (rc != FFCA_OK) goto done;                         \
  } while (0)
  if (rc != FFCA_OK) goto done;
  FFCA_TRY_S(cudaEventRecord(evs[0], s));
  FFCA_TRY_S(cudaStreamWaitEvent(side, evs[0], 0));
  for (int l = 0; l < L; ++l) {
    const NvtxIter nvtx_it(l);
    if (ev) FFCA_TRY_S(cudaEventRecord(ev[l], s));
    const bool last = (l == L - 1);
    for (int i = 0; i < nw; ++i) {
      if (l > 0) FFCA_TRY_S(cudaStreamWaitEvent(s, ref_done[i], 0));
      if (kev && i == 0) FFCA_TRY_S(cudaEventRecord(kev[2 * l], s));
      p.update = 1;
      p.mu_out = (last && (fl & FFCA_FLAG_IMAGES)) ? a->images : nullptr;
      p.mu_back = 1;
      p.iter = l + 1;
      p.v_src = (vin && l == 0) ? a->v_in : nullptr;
      p.g0 = edge[i];
      p.g1 = edge[i + 1];
      // passes over different windows are independent: each may start while
      // the previous one (the last pass on the stream) drains
      // (I >= 5: programmatic launch of the lane-parallel pass over the other
      // window's tail measured slower, 3.6 vs 5.0 G at config 2)
      p.pdl = (l > 0 || i > 0) && pdl_enabled() && I <= 4;
      FFCA_TRY_S(launch_fast_em(p, I, a->dtype, s));
      if (kev && i == nw - 1) FFCA_TRY_S(cudaEventRecord(kev[2 * l + 1], s));
      FFCA_TRY_S(cudaEventRecord(pass_done[i], s));
      FFCA_TRY_S(cudaStreamWaitEvent(side, pass_done[i], 0));
      PencilParams q{};
      q.Spart = w.Spart;
      q.nchunk = w.nchunk;
      q.N = a->N;
      q.G = G;
      q.F = a->F;
      q.P = w.P;
      q.W = w.W;
      q.lam = w.lam;
      q.logdet2 = w.logdet2;
      q.S_model = last ? (double2*)a->S_out : nullptr;
      q.S_hist = nullptr;
      q.llbin = ll ? w.llbin : nullptr;
      q.llg = ll ? w.llg + (size_t)l * G : nullptr;
      q.st = w.st;
      q.iter = l + 1;
      q.St = w.St;
      q.g0 = edge[i];
      q.g1 = edge[i + 1];
      q.prio = hi_prio;
      FFCA_TRY_S(launch_pencil_update(q, I, side));
      FFCA_TRY_S(cudaEventRecord(ref_done[i], side));
    }
  }
  for (int i = 0; i < nw; ++i) FFCA_TRY_S(cudaStreamWaitEvent(s, ref_done[i], 0));
#undef FFCA_TRY_S
done:
  for (int i = 0; i < ne; ++i) cudaEventDestroy(evs[i]);
  return rc;
}

static int fastfca_enqueue(const ffca_run_args* a, cudaStream_t s) {
  int rc = 0;
  const int64_t M = a->M, N = a->N, F = a->F, G = M * F;
  const int I = a->I, L = a->iterations;
  const unsigned fl = a->flags;
  FastWs w = carve_fast(a->workspace, M, N, F, I, L, fl, a->chunk_frames, a->dtype);
  if (w.bytes > a->workspace_bytes) return FFCA_ERR_INVALID;
  const bool ll = fl & FFCA_FLAG_LIKELIHOOD;
  const bool hist = (fl & FFCA_FLAG_HISTORY) != 0;
  const size_t Sslice = (size_t)M * 2 * F * I * I;  // complex entries per S snapshot
  const size_t vslice = (size_t)M * 2 * N * F;      // real entries per v snapshot
  cudaEvent_t* ev = (cudaEvent_t*)a->iter_events;
  cudaEvent_t* kev = (cudaEvent_t*)a->kernel_events;

  if ((rc = reset_status(w.st, s))) return rc;
  FFCA_TRY(launch_initial_pencil((const double2*)a->S0, w.P, w.W, w.lam, w.logdet2, G, F, I,
                                 w.st, s));
  FastIterParams p{};
  p.y = a->y;
  p.v = a->v;
  p.P = w.P;
  p.W = w.W;
  p.lam = w.lam;
  p.floor = a->v_floor;
  p.Spart = w.Spart;
  p.llbin = ll ? w.llbin : nullptr;
  p.M = M;
  p.N = N;
  p.F = F;
  p.G = G;
  p.chunk_frames = w.chunk_frames;
  p.nchunk = w.nchunk;
  p.st = w.st;
  // v_in: the first pass reads the initial powers there and writes v (no copy)
  const bool vin = a->v_in && a->v_in != a->v;
  if (vin && L == 0)
    FFCA_TRY(cudaMemcpyAsync(a->v, a->v_in, vslice * real_size(a->dtype),
                             cudaMemcpyDeviceToDevice, s));

  if (L == 0) {
    if (ev) FFCA_TRY(cudaEventRecord(ev[0], s));
    p.update = 0;
    p.mu_out = (fl & FFCA_FLAG_IMAGES) ? a->images : nullptr;
    p.mu_back = 1;
    p.iter = 0;
    if (p.mu_out || p.llbin) FFCA_TRY(launch_fast_em(p, I, a->dtype, s));
    if (ll) FFCA_TRY(launch_ll_collect(w.llbin, w.nchunk, w.logdet2, N, G, w.llg, s));
    FFCA_TRY(cudaMemcpyAsync(a->S_out, a->S0, Sslice * sizeof(double2),
                             cudaMemcpyDeviceToDevice, s));
  } else if (plan_parts(a) > 1) {
    if ((rc = fastfca_split_loop(a, w, p, plan_parts(a), s))) return rc;
    if (ev) FFCA_TRY(cudaEventRecord(ev[L], s));
    if (ll) {
      p.update = 0;
      p.mu_out = nullptr;
      p.iter = L + 1;
      FFCA_TRY(launch_fast_em(p, I, a->dtype, s));
      FFCA_TRY(launch_ll_collect(w.llbin, w.nchunk, w.logdet2, N, G, w.llg + (size_t)L * G, s));
    }
  } else {
    // KP: the first L - 1 iterations of a small problem in one persistent
    // launch (the last pass writes the images: a stand-alone launch)
    int l0 = 0;
    const int64_t tiles = (G + 31) / 32;
    if (L >= 3 && !ev && !kev && fast_persist_wanted(fl, G, N, I, a->dtype) &&
        tiles * w.nchunk + persist_refreshers(tiles) <= fast_persist_slots(I) &&
        w.nchunk <= fast_persist_max_chunks(I)) {
      FFCA_TRY(cudaMemsetAsync(w.sync, 0, (3 * tiles + 1) * sizeof(int), s));
      p.update = 1;
      p.mu_out = nullptr;
      p.mu_back = 1;
      p.v_src = vin ? a->v_in : nullptr;
      PencilParams q{};
      q.Spart = w.Spart;
      q.nchunk = w.nchunk;
      q.N = N;
      q.G = G;
      q.F = F;
      q.P = w.P;
      q.W = w.W;
      q.lam = w.lam;
      q.logdet2 = w.logdet2;
      q.st = w.st;
      q.St = w.St;
      const NvtxIter nvtx_it(0);
      // a cooperative launch the device cannot place at once (SMs taken by
      // another context) is refused up front: fall back to the plain schedule
      const cudaError_t ke = launch_fast_persist(p, q, w.sync, (int)tiles, L - 1, I, s);
      if (ke == cudaSuccess) {
        p.v_src = nullptr;
        l0 = L - 1;
      } else if (ke == cudaErrorCooperativeLaunchTooLarge || ke == cudaErrorLaunchOutOfResources) {
        cudaGetLastError();
      } else {
        FFCA_TRY(ke);
      }
    }
    // Plain schedule chained with programmatic dependent launch (I <= 4 pass +
    // one-thread-per-bin refresh, nothing else on the stream in between): the
    // next kernel is launched while the current one runs, prefetches what
    // does not depend on it (the pass: its first y / v frames) and waits
    // (griddepcontrol.wait) before it reads the other's output; each kernel
    // releases its dependent only after its own wait, so a pass never
    // overlaps the previous pass and a refresh never the previous refresh.
    // Measured: config 0 (128k TF-bins) 11.1-11.5 -> 13.1 G; no change at config 1
    // (513k) and above, where the launch latency is a small share: small runs only.
    const bool chain = pdl_chain_enabled() && !hist && !ev && !kev && I <= 4 &&
                       G * N <= pdl_chain_max_points(I) && pencil_thread_kernel(G, I);
    for (int l = l0; l < L; ++l) {
      const NvtxIter nvtx_it(l);
      if (ev) FFCA_TRY(cudaEventRecord(ev[l], s));
      p.update = 1;
      p.pdl_wait = chain ? 1 : 0;
      const bool last = (l == L - 1);
      p.mu_out = (last && (fl & FFCA_FLAG_IMAGES)) ? a->images : nullptr;
      p.mu_back = 1;
      p.iter = l + 1;
      p.v_src = (vin && l == 0) ? a->v_in : nullptr;
      if (kev) FFCA_TRY(cudaEventRecord(kev[2 * l], s));
      FFCA_TRY(launch_fast_em(p, I, a->dtype, s));
      p.v_src = nullptr;
      if (kev) FFCA_TRY(cudaEventRecord(kev[2 * l + 1], s));
      if (hist && a->v_hist)
        FFCA_TRY(cudaMemcpyAsync((char*)a->v_hist + (size_t)l * vslice * real_size(a->dtype),
                                 a->v, vslice * real_size(a->dtype), cudaMemcpyDeviceToDevice,
                                 s));
      PencilParams q{};
      q.Spart = w.Spart;
      q.nchunk = w.nchunk;
      q.N = N;
      q.G = G;
      q.F = F;
      q.P = w.P;
      q.W = w.W;
      q.lam = w.lam;
      q.logdet2 = w.logdet2;
      q.S_model = (l == L - 1) ? (double2*)a->S_out : nullptr;  // model S = last iteration's
      q.S_hist = (hist && a->S_hist) ? (double2*)a->S_hist + (size_t)l * Sslice : nullptr;
      q.llbin = ll ? w.llbin : nullptr;
      q.llg = ll ? w.llg + (size_t)l * G : nullptr;
      q.st = w.st;
      q.iter = l + 1;
      q.St = w.St;
      q.pdl_wait = chain ? 1 : 0;
      FFCA_TRY(launch_pencil_update(q, I, s));
    }
    p.pdl_wait = 0;
    if (ev) FFCA_TRY(cudaEventRecord(ev[L], s));
    if (ll) {
      p.update = 0;
      p.mu_out = nullptr;
      p.iter = L + 1;
      FFCA_TRY(launch_fast_em(p, I, a->dtype, s));
      FFCA_TRY(launch_ll_collect(w.llbin, w.nchunk, w.logdet2, N, G, w.llg + (size_t)L * G, s));
    }
  }
  if (ll) FFCA_TRY(launch_ll_reduce(w.llg, M, F, N, I, L + 1, L + 1, a->loglik, s));
  return FFCA_OK;
}

static int fca_enqueue(const ffca_run_args* a, cudaStream_t s) {
  int rc = 0;
  const int64_t M = a->M, N = a->N, F = a->F, G = M * F;
  const int I = a->I, L = a->iterations;
  const unsigned fl = a->flags;
  FcaWs w = carve_fca(a->workspace, M, N, F, I, L, fl, a->chunk_frames, a->dtype);
  if (w.bytes > a->workspace_bytes) return FFCA_ERR_INVALID;
  const bool ll = fl & FFCA_FLAG_LIKELIHOOD;
  const bool hist = (fl & FFCA_FLAG_HISTORY) != 0;
  const size_t Sslice = (size_t)M * 2 * F * I * I;
  const size_t vslice = (size_t)M * 2 * N * F;
  cudaEvent_t* ev = (cudaEvent_t*)a->iter_events;
  cudaEvent_t* kev = (cudaEvent_t*)a->kernel_events;

  if ((rc = reset_status(w.st, s))) return rc;
  FFCA_TRY(launch_fca_prepare((const double2*)a->S0, w.Sp, G, F, I, w.st, 0, s));
  FcaIterParams p{};
  p.y = a->y;
  p.v = a->v;
  p.Sp = w.Sp;
  p.floor = a->v_floor;
  p.Spart = w.Spart;
  p.llbin = ll ? w.llbin : nullptr;
  p.M = M;
  p.N = N;
  p.F = F;
  p.G = G;
  p.chunk_frames = w.chunk_frames;
  p.nchunk = w.nchunk;
  p.st = w.st;
  const bool vin = a->v_in && a->v_in != a->v;
  if (vin && L == 0)
    FFCA_TRY(cudaMemcpyAsync(a->v, a->v_in, vslice * real_size(a->dtype),
                             cudaMemcpyDeviceToDevice, s));
  if (L == 0) {
    if (ev) FFCA_TRY(cudaEventRecord(ev[0], s));
    p.update = 0;
    p.mu_out = (fl & FFCA_FLAG_IMAGES) ? a->images : nullptr;
    p.iter = 0;
    if (p.mu_out || p.llbin) FFCA_TRY(launch_fca_em(p, I, a->dtype, s));
    if (ll) FFCA_TRY(launch_ll_collect(w.llbin, w.nchunk, nullptr, N, G, w.llg, s));
    FFCA_TRY(cudaMemcpyAsync(a->S_out, a->S0, Sslice * sizeof(double2),
                             cudaMemcpyDeviceToDevice, s));
  } else {
    // plain schedule chained with programmatic dependent launch, as FastFCA's
    // (I <= 4 pass K4 + lane-parallel finish K4b, nothing else on the stream)
    // (config 0 9.7 -> 10.3 G; config 1 loses, 18.3 -> 16.3 G: small runs only)
    const bool chain = pdl_chain_enabled() && !hist && !ev && !kev && I <= 4 &&
                       G * N <= pdl_chain_max_points(3);  // (measured at config 0 / 1 only)
    for (int l = 0; l < L; ++l) {
      const NvtxIter nvtx_it(l);
      if (ev) FFCA_TRY(cudaEventRecord(ev[l], s));
      p.update = 1;
      p.pdl_wait = chain ? 1 : 0;
      const bool last = (l == L - 1);
      p.mu_out = (last && (fl & FFCA_FLAG_IMAGES)) ? a->images : nullptr;
      p.iter = l + 1;
      p.v_src = (vin && l == 0) ? a->v_in : nullptr;
      if (kev) FFCA_TRY(cudaEventRecord(kev[2 * l], s));
      FFCA_TRY(launch_fca_em(p, I, a->dtype, s));
      p.v_src = nullptr;
      if (kev) FFCA_TRY(cudaEventRecord(kev[2 * l + 1], s));
      if (hist && a->v_hist)
        FFCA_TRY(cudaMemcpyAsync((char*)a->v_hist + (size_t)l * vslice * real_size(a->dtype),
                                 a->v, vslice * real_size(a->dtype), cudaMemcpyDeviceToDevice,
                                 s));
      // the finish's only check is the Cholesky of the new S, which the
      // reference does at the start of the NEXT iteration (conventional.py:131,
      // 98-101): after the last iteration nothing inverts S, so a
      // final non-PD model returns normally there -> no status word
      FFCA_TRY(launch_fca_finish(
          w.Spart, w.nchunk, N, G, F, w.Sp, (double2*)a->S_out,
          (hist && a->S_hist) ? (double2*)a->S_hist + (size_t)l * Sslice : nullptr,
          ll ? w.llbin : nullptr, ll ? w.llg + (size_t)l * G : nullptr, I,
          (l == L - 1) ? nullptr : w.st, l + 1, s, chain ? 1 : 0));
    }
    p.pdl_wait = 0;
    if (ev) FFCA_TRY(cudaEventRecord(ev[L], s));
    if (ll) {
      p.update = 0;
      p.mu_out = nullptr;
      p.iter = L + 1;
      FFCA_TRY(launch_fca_em(p, I, a->dtype, s));
      FFCA_TRY(launch_ll_collect(w.llbin, w.nchunk, nullptr, N, G, w.llg + (size_t)L * G, s));
    }
  }
  if (ll) FFCA_TRY(launch_ll_reduce(w.llg, M, F, N, I, L + 1, L + 1, a->loglik, s));
  return FFCA_OK;
}

int ffca_run_status(const void* workspace, void* stream, ffca_status* out) {
  if (!workspace || !out) return FFCA_ERR_INVALID;
  return ffca_status_read((const ffca_status_dev*)workspace, stream, out);
}

int ffca_status_decode(const ffca_status_dev* host_word, ffca_status* out) {
  if (!host_word || !out) return FFCA_ERR_INVALID;
  decode(*host_word, out);
  return FFCA_OK;
}

int ffca_status_reset(ffca_status_dev* st, void* stream) {
  if (!st) return FFCA_ERR_INVALID;
  return reset_status(st, (cudaStream_t)stream);
}

int ffca_status_read(const ffca_status_dev* st, void* stream, ffca_status* out) {
  if (!st || !out) return FFCA_ERR_INVALID;
  ffca_status_dev h;
  cudaStream_t s = (cudaStream_t)stream;
  FFCA_TRY(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  FFCA_TRY(cudaStreamSynchronize(s));
  decode(h, out);
  return FFCA_OK;
}

// ---- per-bin batched routines ---------------------------------------------
int ffca_gevd_hpd(const double* Phi, const double* Psi, double* lam, double* P, int64_t batch,
                  int D, int check_hermitian, ffca_status_dev* st, void* stream) {
  if (!Phi || !Psi || !lam || !P || batch < 0 || D < 1 || D > kMaxOrder) return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_gevd_batch((const double2*)Phi, (const double2*)Psi, lam, (double2*)P, nullptr,
                              batch, D, check_hermitian, st, (cudaStream_t)stream));
}

int ffca_propagate_pencil(const double* St1, const double* St2, const double* P_prev,
                          double* P_next, double* lam, int64_t batch, int D,
                          ffca_status_dev* st, void* stream) {
  if (!St1 || !St2 || !P_prev || !P_next || !lam || batch < 0 || D < 1 || D > kMaxOrder)
    return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_gevd_batch((const double2*)St1, (const double2*)St2, lam, (double2*)P_next,
                              (const double2*)P_prev, batch, D, 1, st, (cudaStream_t)stream));
}

int ffca_cholesky_inverse(const double* S, double* Sinv, int64_t batch, int D,
                          ffca_status_dev* st, void* stream) {
  if (!S || !Sinv || batch < 0 || D < 1 || D > kMaxOrder) return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_cholinv((const double2*)S, (double2*)Sinv, batch, D, st,
                           (cudaStream_t)stream));
}

int ffca_solve(const double* A, const double* B, double* X, double* norms, int64_t batch,
               int D, int64_t K, ffca_status_dev* st, void* stream) {
  if (!A || !B || !X || !norms || batch < 0 || D < 1 || D > kMaxOrder || K < 0)
    return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_solve((const double2*)A, (const double2*)B, (double2*)X, norms, batch, D, K, st,
                         (cudaStream_t)stream));
}

int ffca_regularize_covariances(const double* S, double* out, int64_t batch, int D,
                                void* stream) {
  if (!S || !out || batch < 0 || D < 1 || D > kMaxOrder) return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_regularize((const double2*)S, (double2*)out, batch, D, (cudaStream_t)stream));
}

int ffca_regularize_transformed(const double* S_raw, const double* gram, double* out,
                                int64_t batch, int D, void* stream) {
  if (!S_raw || !out || batch < 0 || D < 1 || D > kMaxOrder) return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_reg_transformed((const double2*)S_raw, (const double2*)gram, (double2*)out,
                                   batch, D, (cudaStream_t)stream));
}

int ffca_logdet2(const double* P, double* out, int64_t batch, int D, void* stream) {
  if (!P || !out || batch < 0 || D < 1 || D > kMaxOrder) return FFCA_ERR_INVALID;
  if (batch == 0) return FFCA_OK;
  return cu(launch_inverse_h((const double2*)P, nullptr, out, batch, D, nullptr,
                             (cudaStream_t)stream));
}

int ffca_back_transform_images(const double* mu_t, const double* P, double* out, int64_t Src,
                               int64_t N, int64_t F, int I, ffca_status_dev* st, void* stream) {
  if (!mu_t || !P || !out || Src < 0 || N < 0 || F < 1 || I < 1 || I > kMaxOrder)
    return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  double2* W = nullptr;
  FFCA_TRY(cudaMallocAsync((void**)&W, (size_t)F * I * I * sizeof(double2), s));
  int rc = cu(launch_inverse_h((const double2*)P, W, nullptr, F, I, st, s));
  if (rc == FFCA_OK && Src * N > 0)
    rc = cu(launch_apply_w((const double2*)mu_t, W, (double2*)out, Src, N, F, I, s));
  cudaFreeAsync(W, s);
  return rc;
}

int ffca_back_transform_covariances(const double* S_t, const double* P, double* out,
                                    int64_t Src, int64_t F, int I, ffca_status_dev* st,
                                    void* stream) {
  if (!S_t || !P || !out || Src < 0 || F < 1 || I < 1 || I > kMaxOrder) return FFCA_ERR_INVALID;
  cudaStream_t s = (cudaStream_t)stream;
  double2* W = nullptr;
  FFCA_TRY(cudaMallocAsync((void**)&W, (size_t)F * I * I * sizeof(double2), s));
  int rc = cu(launch_inverse_h((const double2*)P, W, nullptr, F, I, st, s));
  if (rc == FFCA_OK && Src > 0)
    rc = cu(launch_conj_w((const double2*)S_t, W, (double2*)out, Src, F, I, s));
  cudaFreeAsync(W, s);
  return rc;
}

int ffca_init_powers(const void* y, void* v, double* v_floor, int64_t M, int64_t N, int64_t F,
                     int I, int dtype, void* stream) {
  if (!y || !v || !v_floor || M < 1 || N < 1 || F < 1 || I < 1) return FFCA_ERR_INVALID;
  return cu(launch_init_powers(y, v, v_floor, M, N, F, I, dtype, (cudaStream_t)stream));
}

}  // extern "C"
