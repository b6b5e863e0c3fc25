// pxg_main.cu — libpxg: pass orchestration on two CUDA streams and the C ABI (include/pxg.h).
//
// Per pass (proj/src/proxy.cpp:683-827): Stage 1 (pool walks -> priority selection ->
// entries -> probes -> bounds -> reciprocal rounds -> finish) runs on `stream1` one pass
// ahead of Stage 2 (eye/light wavefronts -> connections -> proxy connection -> gate + film
// -> gamma) on `stream`. Stage 1 of pass p+1 reads and writes only the subspace statistics
// and its own pool slot, never the film, the grid shares or gamma, so overlapping it with
// Stage 2 of pass p leaves every result identical to the sequential order.
#include <dlfcn.h>

#include <fstream>
#include <mutex>
#include <utility>

#include "pxg_stage_kernels.cuh"
#include "pxg_pt.cuh"

// ------------------------------------------------------------------ context
// Pool state of one pass, double-buffered: Stage 1 of pass p+1 (stream s1) fills one slot
// while Stage 2 of pass p (stream s2) reads the other.
struct PoolSlot {
  IncHdr* inc = nullptr;
  PV* prefix = nullptr;
  int* kept = nullptr;
  int* label_start = nullptr;
  int* label_list = nullptr;
  PassState* ps = nullptr;
  double* snap_sum = nullptr;  // SubspaceStats snapshot after Stage 1 of this pass
  double* snap_sq = nullptr;
  long long* snap_cnt = nullptr;
  cudaEvent_t s1_done = nullptr;  // Stage 1 wrote the slot
  cudaEvent_t s2_done = nullptr;  // Stage 2 finished reading it
  cudaEvent_t t0 = nullptr, t1 = nullptr, r0 = nullptr, r1 = nullptr;  // Stage-1 timing
  double* bound = nullptr;      // B per entry used by this pass's reciprocal runs
  long long* diag = nullptr;    // [4000*5] Stage-1 diagnostics of this pass
  int* diag_touched = nullptr;  // [4000]
  double* snap_max = nullptr;
  long long* snap_rcnt = nullptr;
  int pass = -1;
  int batch_end = 0;  // first pass after the Stage-1 batch this slot belongs to
  bool timing_pending = false;
};

// Process-wide cache of pinned host staging buffers: page-locking and unlocking host memory
// (cudaMallocHost / cudaFreeHost) costs up to hundreds of ms and would otherwise be paid by
// every context create / destroy (the per-call render_proxy_bdpt path).
namespace {
std::mutex g_pinned_mu;
std::vector<std::pair<size_t, void*>> g_pinned_free;

void* pinned_acquire(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    for (size_t i = 0; i < g_pinned_free.size(); ++i)
      if (g_pinned_free[i].first == bytes) {
        void* p = g_pinned_free[i].second;
        g_pinned_free.erase(g_pinned_free.begin() + static_cast<long>(i));
        return p;
      }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) throw CudaErr{"cudaMallocHost failed"};
  return p;
}

void pinned_release(void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  if (g_pinned_free.size() >= 8) {  // bounded: free the oldest
    cudaFreeHost(g_pinned_free.front().second);
    g_pinned_free.erase(g_pinned_free.begin());
  }
  g_pinned_free.emplace_back(bytes, p);
}
}  // namespace

// ---- parity entry point of the production traversal kernels (pxg_trace_rays)
// Queue fill with the production conventions: closest-hit rays as given (tmax or 1e30);
// any-hit segments a -> b as conn_eval_one / occluded() build them (unit direction sd/dist,
// tmax = dist * (1 - 1e-6)); a segment shorter than kRayEps is never occluded (tmax 0).
__global__ void k_fill_trace_queue(int n, const double* rays, const double* tmax, int any, RayQueue Q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* r = rays + 6 * static_cast<size_t>(i);
  V3 o = v3(r[0], r[1], r[2]), d;
  double tm;
  if (any) {
    const V3 sd = v3(r[3], r[4], r[5]) - o;
    const double dist = length(sd);
    if (dist < kRayEps) {
      d = v3(1.0, 0.0, 0.0);
      tm = 0.0;
    } else {
      d = sd / dist;
      tm = dist * (1.0 - 1e-6);
    }
  } else {
    d = v3(r[3], r[4], r[5]);
    tm = tmax ? tmax[i] : 1e30;
  }
  Q.ray[2 * i] = make_double4(o.x, o.y, o.z, d.x);
  Q.ray[2 * i + 1] = make_double4(d.y, d.z, tm, 0.0);
  Q.path[i] = i;
  if (i == 0) *Q.count = n;
}

// The reciprocal node wavefront's traversal (k_recip_eval_wave: rw_trace) on the queue's
// rays, one lane per ray.
template <bool kAny>
__global__ void k_wave_trace(SceneView S, RayQueue Q, const double* rays, int any_segments) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = *Q.count;
  bool has = j < n;
  TravState ts;
  if (has) {
    trav_init(ts, Q, j);
    if (kAny && !(ts.t_best > 0.0)) has = false;  // a segment shorter than kRayEps: never occluded
  }
  const bool occ = rw_trace<kAny>(S, ts, has);
  if (j >= n) return;
  if (kAny) {
    Q.hit_prim[j] = occ ? 1 : 0;
  } else {
    Q.hit_prim[j] = ts.best;
    Q.hit_t[j] = ts.t_best;
  }
}

// sin / cos of the draws k (u = k * 2^-32, phi = 2*pi*u) with the device code path of the
// samplers (pxg_sincos_2pi parity entry point).
__global__ void k_sincos_2pi(int n, const uint32_t* k, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s, c;
  sincos_2pi(static_cast<double>(k[i]) * 0x1p-32, s, c);
  out[2 * i] = s;
  out[2 * i + 1] = c;
}

// glibc agreement table of the device sin / cos (include/pxg_sincos.h), built next to
// libpxg.so by the build (csrc/pxg_sincos_gen.cpp, from the host's libm). Loaded once per
// process and uploaded once per device; a missing table is an error, never a silent switch
// to CUDA's sin / cos.
namespace {
std::mutex g_sc_mu;
std::vector<char> g_sc_file;
bool g_sc_device[64] = {};

std::string sincos_table_path() {
  if (const char* e = std::getenv("PXG_SINCOS_TABLE")) return e;
  Dl_info info{};
  if (dladdr(reinterpret_cast<void*>(&pxg_abi_version), &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const size_t slash = so.rfind('/');
    return (slash == std::string::npos ? std::string(".") : so.substr(0, slash)) + "/pxg_sincos_glibc.bin";
  }
  return "pxg_sincos_glibc.bin";
}

void ensure_sincos_table(int device);
}  // namespace

// A finalised scene (the analogue of the reference's Scene after load_scene -> finalize,
// proj/src/scene.cpp:234-252): the flattened description (owned copies), the host BVH
// (pxg_host.cpp) and the device-ready arrays. Immutable; any number of contexts, on any
// device, are created from it without rebuilding the BVH.
struct pxg_scene {
  std::vector<int> shape, material, emitter_prim;
  std::vector<double> a, b, c, radius, materials, emitter_radiance;
  pxg_scene_desc desc{};  // pointers into the vectors above
  SceneHost host;
  std::vector<std::pair<void*, size_t>> pinned;  // page-locked host arrays (fast per-context upload)
  ~pxg_scene() {
    for (auto& pr : pinned) cudaHostUnregister(pr.first);
  }
};

struct pxg_ctx {
  std::string err;
  int device = 0;
  cudaStream_t stream = nullptr;   // Stage 2 (and everything else)
  cudaStream_t stream1 = nullptr;  // Stage 1 of the next pass
  cudaStream_t stream_t = nullptr;  // Stage 2a: eye + light sub-path traces, one pass ahead
  // sub-path vertex pools, double-buffered by pass parity so the traces of pass p+1 run
  // while the connections / proxy connection of pass p read pass p's pools
  PV* eye_buf[2] = {nullptr, nullptr};
  PV* light_buf[2] = {nullptr, nullptr};
  int* neye_buf[2] = {nullptr, nullptr};
  int* nlight_buf[2] = {nullptr, nullptr};
  cudaEvent_t trace_done[2] = {nullptr, nullptr};  // Stage 2a of the buffer's pass finished
  cudaEvent_t paths_free[2] = {nullptr, nullptr};  // Stage 2b finished reading the buffer
  RayQueue qP, qQ;  // proxy-wavefront queues (qA / qB belong to the traces)
  RayQueue qPS;     // proxy-connection shadow rays (qS belongs to the connections)
  PathCache pcache_buf[2];  // per-sub-path MIS step caches, double-buffered like the pools
  cudaStream_t stream_p = nullptr;  // Stage 2b': proxy connection, forked from the pass
  cudaEvent_t proxy_done = nullptr, gamma_done = nullptr;
  cudaEvent_t x_in = nullptr, x_out = nullptr;  // pxg_accum_to_device_async: caller <-> context ordering
  pxg_params P{};
  pxg_shard shard{};
  uint64_t seed = 0;
  int width = 0, height = 0, max_depth = 0, n = 0, n_px_total = 0, row0 = 0, rows = 0;
  // Stage-2 row tiles: a pass runs Stage 2 over [row0_ctx, row0_ctx + rows_ctx) in tiles of
  // tile_rows rows (a multiple of the 10-row gate grid) so the per-pixel working set of a
  // 4K depth-16 image fits in HBM. Per-pixel state that outlives a tile (RNG counters, film,
  // the pass values and gamma contributions in pixel order, the gate grid) is full-size; the
  // vertex pools, connection slots and queues are tile-size. n / row0 / rows / n_cells and the
  // full-size pointers below describe the active tile while Stage 2 is enqueued, the whole
  // context otherwise (activate_tile / activate_ctx).
  int n_ctx = 0, row0_ctx = 0, rows_ctx = 0, n_cells_ctx = 0, tile_rows = 0, ntiles = 1;
  long long tile_step = 0;  // (pass, tile) steps enqueued: parity selects the vertex-pool buffer
  struct FullView {
    unsigned* ctr;
    double *bdpt, *val, *acc, *gval, *grid_total, *grid_proxy;
    ProxRec* prox;
    int *pflags, *gbin, *eye_prims, *light_prims;
  } full{};
  int light_walks = 0;
  int grid_w = 0, grid_h = 0, n_cells = 0;
  bool proxy_on = false;
  int passes_done = 0;
  int pass_limit = -1;  // no Stage-1 lookahead at or beyond this pass (pxg_set_pass_limit)
  std::vector<void*> allocs;

  SceneView S{};
  Mapper M{};
  // stage 2
  PV* d_eye = nullptr;
  PV* d_light = nullptr;
  int *d_neye = nullptr, *d_nlight = nullptr;
  unsigned* d_ctr = nullptr;
  double *d_bdpt = nullptr, *d_val = nullptr, *d_acc = nullptr;
  ProxRec* d_prox = nullptr;
  PV* d_scratch = nullptr;
  double *d_grid_total = nullptr, *d_grid_proxy = nullptr;
  int *d_gbin = nullptr, *d_gbin_sorted = nullptr;
  double *d_gval = nullptr, *d_gval_sorted = nullptr;
  int* d_gsort_tmp = nullptr;  // stable_bin_sort scratch (pxg_prims.cuh)
  int* d_pflags = nullptr;
  int *d_eye_prims = nullptr, *d_light_prims = nullptr;
  // stats (live, written by Stage 1 only)
  double *d_max_ratio = nullptr, *d_sum_est = nullptr, *d_sum_sq = nullptr;
  long long *d_ratio_cnt = nullptr, *d_est_cnt = nullptr;
  int* d_touched = nullptr;
  // gamma: rows and accumulators on the device; learning state is host bookkeeping
  bool gamma_learning = true;
  int gamma_iter = 0;
  double* d_gamma = nullptr;
  double* d_gamma_accum = nullptr;
  // pool (Stage 1 working buffers)
  int cand_cap = 0;
  unsigned long long* d_ckey = nullptr;
  unsigned* d_cval = nullptr;
  int* d_ccount = nullptr;
  unsigned* d_sel = nullptr;
  double* d_probe = nullptr;
  int* d_probe_ok = nullptr;
  double* d_bound = nullptr;
  double* d_run_est = nullptr;
  long long* d_run_cost = nullptr;
  int* d_run_trunc = nullptr;
  RecipFrame* d_frames = nullptr;
  RunState* d_rstate = nullptr;
  double* d_rg = nullptr;
  long long* d_rn = nullptr;
  int* d_re = nullptr;
  int* d_ract[2] = {nullptr, nullptr};
  int* d_rnact = nullptr;
  int recip_rounds = 0;
  static constexpr int kBatchMax = kBatchSetMax;  // passes per Stage-1 batch (PXG_BATCH, default kBatchDefault)
  static constexpr int kBatchDefault = 8;
  static constexpr int kRing = 3;      // pool slots = kRing batches: Stage 1 up to ~2 batches ahead
  PoolSlot slot[kRing * kBatchMax];   // ring of kRing * batch slots (the rest unallocated)
  int batch = kBatchMax;               // passes per batch (<= kBatchMax)
  int next_batch = 0;                  // first pass without a launched Stage 1
  int ring() const { return kRing * batch; }
  PoolSlot& slot_of(int pass) { return slot[pass % ring()]; }
  int* d_err = nullptr;
  // diagnostics
  long long* d_diag = nullptr;  // [4000*5]: cols 2..4 written by k_pool_finish
  unsigned long long *d_diag_attempt = nullptr, *d_diag_accept = nullptr;
  unsigned long long* d_kept_total = nullptr;
  int* d_diag_touched = nullptr;
  // wavefront queues and buffers
  RayQueue qA{}, qB{}, qS{};  // qA/qB: Stage 2 bounces; qS: shadow rays
  RayQueue wA{}, wB{};        // Stage-1 pool-walk bounces (own queues: runs concurrently)
  ConnBuf conn{};
  PathCache pcache{};
  double *d_ebeta = nullptr, *d_epdf = nullptr, *d_lbeta = nullptr, *d_lpdf = nullptr;
  int* d_scan_tmp = nullptr;  // exclusive_sum scratch (pxg_prims.cuh)
  int max_slots = 0;
  PV* d_wpool = nullptr;
  int* d_wnv = nullptr;
  unsigned* d_wctr = nullptr;
  double *d_wbeta = nullptr, *d_wpdf = nullptr;
  int n_walks = 0;
  // timing (Stage 2 events on `stream`)
  cudaEvent_t ev[8];
  cudaEvent_t ev_call[3];
  double stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long launches = 0;
  ProxWave pw{};
  static constexpr int kSnap = PXG_SNAPSHOT_SLOTS;
  double* d_snap[kSnap] = {};  // running-mean snapshots for the pipelined pass_done loop
  cudaEvent_t snap_ev[kSnap] = {};
  int snap_passes[kSnap] = {};
  double* h_pinned = nullptr;              // pinned staging for read-backs (process-wide cache)
  size_t pinned_bytes = 0;
  int* h_err = nullptr;                    // [kSnap] pinned error flags of the snapshots
  int trav_blocks = 0;        // persistent traversal grid (SMs x resident blocks)
  int trav_minb = 6;          // resident blocks per SM of the traversal variant (6 or 8)
  bool trav_post = false;     // postponed leaf tests (scenes with quantised nodes)
  int gs_blocks = 0;          // grid of the grid-stride slot kernels (SMs x 256 blocks of 128; 16 / 64 measured slower)
  int eval_blocks = 0;        // grid-stride reciprocal node evaluation grid
  int wave_blocks = 0;        // k_recip_eval_wave grid (0: the thread-per-node k_recip_eval)
  PV* d_rw_scratch = nullptr; // candidate vertices of k_recip_eval_wave: [wave_blocks][kRW][4]
  // global reciprocal wavefront (pxg_recip_queue.cuh): per-node scratch + its ray queues
  RqView rq{nullptr, nullptr, 0};
  RayQueue rqA, rqB, rqS;
  unsigned long long* d_node_stat = nullptr;  // reciprocal tree nodes evaluated / consumed, finished runs
  int* shade_perm[2] = {nullptr, nullptr};    // k_shade_order's per-tile class order: [0] Stage-2 traces, [1] Stage-1 walks
  double* d_rw_ends = nullptr; // its visibility segment endpoints: [wave_blocks][kRW][10][6]
  int dfs_blocks = 0;         // grid-stride warp-DFS grid
  int sel_cap = 0;            // shared-memory capacity (entries) of the pool selection
  size_t sel_smem = 0;
  size_t fin_smem = 0;        // pool finish shared memory
  int* d_trav_next = nullptr;  // [8] ray fetch counters (per stream use)
  // traversal roofline measurement (pxg_measure_traversal)
  bool measure = false;
  unsigned long long* d_tcnt = nullptr;  // closest {rays, nodes, prims}, any-hit {rays, nodes, prims}
  struct TimedLaunch {
    cudaEvent_t a, b;
    int kind;  // 0 closest, 1 any-hit
  };
  std::vector<TimedLaunch> tl;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  cudaEvent_t take_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }

  template <typename T>
  T* alloc(size_t n_) {
    // stream-ordered allocator on a process-wide pool that keeps freed memory (release
    // threshold = max): creating and destroying contexts does not map/unmap GBs each time
    T* p = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n_, 1) * sizeof(T), stream));
    allocs.push_back(p);
    return p;
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));  // v may be a temporary
    return p;
  }
  // upload of host data that outlives the call (the pxg_scene's arrays): no synchronisation
  template <typename T>
  T* upload_async(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, stream));
    return p;
  }
  template <typename T>
  T* zeros(size_t n_) {
    T* p = alloc<T>(n_);
    CK(cudaMemsetAsync(p, 0, std::max<size_t>(n_, 1) * sizeof(T), stream));
    return p;
  }
  ~pxg_ctx() {
    if (stream) cudaStreamSynchronize(stream);
    if (stream1) cudaStreamSynchronize(stream1);
    if (stream_t) cudaStreamSynchronize(stream_t);
    if (stream_p) cudaStreamSynchronize(stream_p);
    for (void* p : allocs) cudaFreeAsync(p, stream);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    for (auto& e : ev_call) if (e) cudaEventDestroy(e);
    for (auto& e : ev_pool) cudaEventDestroy(e);
    for (auto& e : snap_ev) if (e) cudaEventDestroy(e);
    if (h_pinned) pinned_release(h_pinned, pinned_bytes);
    if (h_err) pinned_release(h_err, kSnap * sizeof(int));
    for (auto& sl : slot)
      for (cudaEvent_t e : {sl.s1_done, sl.s2_done, sl.t0, sl.t1, sl.r0, sl.r1})
        if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (stream1) cudaStreamDestroy(stream1);
    if (stream_t) cudaStreamDestroy(stream_t);
    if (stream_p) cudaStreamDestroy(stream_p);
    for (cudaEvent_t e : {proxy_done, gamma_done, x_in, x_out})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {trace_done[0], trace_done[1], paths_free[0], paths_free[1]})
      if (e) cudaEventDestroy(e);
  }
};

namespace {

void raise_err(int e) {
  if (!e) return;
  const char* what = e == kErrIntegrand ? "reciprocal: integrand must be finite and non-negative"
                     : e == kErrSupport ? "reciprocal: support pdf must be finite and positive"
                     : e == kErrSplit   ? "stochastic_split: bad ratio"
                     : e == kErrPool    ? "pool: candidate selection failed (buffer overflow or key ties)"
                                        : "update_ratio: ratio must be finite and non-negative";
  throw RuntimeErr{what};
}

void check_err(pxg_ctx* c, cudaStream_t st) {
  int e = 0;
  CK(cudaMemcpyAsync(&e, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  raise_err(e);
}

// PXG_PROFILE=1: synchronise and print host-side stage timestamps (debugging aid).
struct HostProbe {
  cudaStream_t st;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit HostProbe(cudaStream_t s) : st(s), on(std::getenv("PXG_PROFILE") != nullptr) {
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pxg] %-14s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

#ifndef PXG_TRAV_HI
#define PXG_TRAV_HI 8  // resident blocks per SM of the high-occupancy traversal variant (A/B: 10, 12)
#endif
// Persistent traversal of queue q (closest hit or any hit) with the context's occupancy variant.
template <bool kAny, int kL>
void launch_trav_layout(pxg_ctx* c, const RayQueue& q, int* fetch, cudaStream_t st) {
  if (c->trav_minb == 8) {
    if (c->trav_post)
      k_trav_persistent<kAny, PXG_TRAV_HI, true, kL><<<c->trav_blocks, 128, 0, st>>>(c->S, q, fetch);
    else
      k_trav_persistent<kAny, PXG_TRAV_HI, false, kL><<<c->trav_blocks, 128, 0, st>>>(c->S, q, fetch);
  } else {
    if (c->trav_post)
      k_trav_persistent<kAny, 6, true, kL><<<c->trav_blocks, 128, 0, st>>>(c->S, q, fetch);
    else
      k_trav_persistent<kAny, 6, false, kL><<<c->trav_blocks, 128, 0, st>>>(c->S, q, fetch);
  }
}

// The node layout is a template parameter of the kernels (no per-visit test of S.nodeq).
template <bool kAny>
void launch_trav(pxg_ctx* c, const RayQueue& q, int* fetch, cudaStream_t st) {
  if (c->S.nodeq)
    launch_trav_layout<kAny, 1>(c, q, fetch, st);
  else
    launch_trav_layout<kAny, 0>(c, q, fetch, st);
}

RayQueue make_queue(pxg_ctx* c, size_t cap) {
  RayQueue q;
  q.ray = c->alloc<double4>(2 * cap);
  q.path = c->alloc<int>(cap);
  q.hit_prim = c->alloc<int>(cap);
  q.hit_t = c->alloc<double>(cap);
  q.count = c->zeros<int>(1);
  q.cap = static_cast<int>(cap);
  return q;
}

// Sub-path wavefront: start kernel, then one (closest-hit, shade) pair per bounce.
void trace_paths(pxg_ctx* c, const PathSet& P, RayQueue in, RayQueue out, cudaStream_t st) {
  CK(cudaMemsetAsync(in.count, 0, sizeof(int), st));
  const int T = 128;
  if (P.eye)
    k_eye_start<<<blocks(P.n, T), T, 0, st>>>(c->S, P, in, c->row0);
  else
    k_light_start<<<blocks(P.n, T), T, 0, st>>>(c->S, P, in);
  ++c->launches;
  for (int b = 0; b + 1 < P.max_vertices; ++b) {
    int* fetch = c->d_trav_next + (st == c->stream1 ? 1 : 0);
    CK(cudaMemsetAsync(fetch, 0, sizeof(int), st));
    if (c->measure) {
      pxg_ctx::TimedLaunch t{c->take_event(), c->take_event(), 0};
      CK(cudaEventRecord(t.a, st));
      launch_trav<false>(c, in, fetch, st);
      CK(cudaEventRecord(t.b, st));
      k_closest_count<<<blocks(P.n, T), T, 0, st>>>(c->S, in, c->d_tcnt);
      c->tl.push_back(t);
    } else {
      launch_trav<false>(c, in, fetch, st);
    }
    CK(cudaMemsetAsync(out.count, 0, sizeof(int), st));
    if (c->shade_perm[0]) {
      int* perm = c->shade_perm[st == c->stream1 ? 1 : 0];
      k_shade_order<<<blocks(P.n, kOrderT), kOrderT, 0, st>>>(c->S, in, perm);
      k_shade_perm<<<blocks(P.n, 128), 128, 0, st>>>(c->S, P, in, out, perm);
      ++c->launches;
    } else {
      k_shade<<<blocks(P.n, PXG_SHADE_T), PXG_SHADE_T, 0, st>>>(c->S, P, in, out);
    }
    c->launches += 2;
    std::swap(in, out);
  }
}

// Standard strategies of every pixel (weighted_bdpt_value, proxy.cpp:621-643).
void connections(pxg_ctx* c, bool use_stats, const PoolSlot& sl) {
  const int n = c->n, D = c->max_depth, T = 128;
  cudaStream_t st = c->stream;
  ConnBuf& C = c->conn;
  k_conn_count<<<blocks(n, T), T, 0, st>>>(c->d_neye, c->d_nlight, n, D, C.count);
  c->launches += exclusive_sum(C.count, C.offset, n + 1, c->d_scan_tmp, st);
  k_conn_enum<<<blocks(n, T), T, 0, st>>>(c->d_neye, c->d_nlight, n, D, C);
  CK(cudaMemsetAsync(c->qS.count, 0, sizeof(int), st));
  CK(cudaMemsetAsync(C.n_live, 0, sizeof(int), st));
  const long long slots = static_cast<long long>(n) * c->max_slots;
  const int gs = static_cast<int>(std::min<long long>(c->gs_blocks, blocks(slots, T)));
  k_conn_eval<<<gs, T, 0, st>>>(c->S, c->d_eye, c->d_light, n, C, c->qS);
  int* fetch = c->d_trav_next + 2;
  CK(cudaMemsetAsync(fetch, 0, sizeof(int), st));
  if (c->measure) {
    pxg_ctx::TimedLaunch t{c->take_event(), c->take_event(), 1};
    CK(cudaEventRecord(t.a, st));
    launch_trav<true>(c, c->qS, fetch, st);
    CK(cudaEventRecord(t.b, st));
    k_anyhit_count<<<blocks(slots, T), T, 0, st>>>(c->S, c->qS, c->d_tcnt + 3);
    c->tl.push_back(t);
  } else {
    launch_trav<true>(c, c->qS, fetch, st);
  }
  k_conn_visibility<<<gs, T, 0, st>>>(c->qS, C);
  k_conn_mis<<<gs, T, 0, st>>>(c->S, c->M,
                                             StatsView{c->d_max_ratio, sl.snap_sum, sl.snap_sq, sl.snap_cnt},
                                             use_stats ? 1 : 0, c->d_eye, c->d_light, n, C, c->pcache);
  k_conn_sum<<<blocks(n, T), T, 0, st>>>(n, C, c->d_bdpt);
  c->launches += 9;
}

// The reciprocal runs of a batch: rounds of (parallel node evaluation, DFS resume); round r
// evaluates the next chunk_r = min(first * grow^r, 16384) nodes of every active run. The
// round count is fixed on the host (the smallest R with chunk_0 + ... + chunk_{R-1} >= cap,
// after which every run has finished), and the kernels read the active count on the device,
// so no round waits for the host; a round with no active run costs two empty launches.
template <typename Eval>
int recip_rounds(cudaStream_t stream, long long cap, int* nact, Eval&& eval_and_dfs) {
  static const int first = std::getenv("PXG_RECIP_CHUNK") ? std::atoi(std::getenv("PXG_RECIP_CHUNK")) : 16;
  static const int grow = std::getenv("PXG_RECIP_GROW") ? std::atoi(std::getenv("PXG_RECIP_GROW")) : 2;
  static const bool verbose = std::getenv("PXG_PROFILE") != nullptr;
  int cur = 0, chunk = std::max(first, 1), rounds = 0;
  long long covered = 0;
  do {
    if (verbose) {
      int count = 0;
      CK(cudaMemcpyAsync(&count, nact + cur, sizeof(int), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      std::fprintf(stderr, "[pxg]   round %d: %d runs x %d nodes\n", rounds, count, chunk);
    }
    CK(cudaMemsetAsync(nact + (1 - cur), 0, sizeof(int), stream));
    // every active run has the same nodes evaluated so far (`covered`): the last round's chunk
    // stops at the cap, so no thread or scratch slot is spent on nodes past it
    eval_and_dfs(cur, static_cast<int>(std::max<long long>(1, std::min<long long>(chunk, cap - covered))));
    cur = 1 - cur;
    covered += chunk;
    chunk = static_cast<int>(std::min<long long>(static_cast<long long>(chunk) * std::max(grow, 1), 16384));
    ++rounds;
  } while (covered < cap);
  return rounds;
}

void read_stage1_timing(pxg_ctx* c, PoolSlot& sl) {
  if (!sl.timing_pending) return;
  sl.timing_pending = false;
  if (cudaEventQuery(sl.t1) != cudaSuccess) {  // never block the host for diagnostics
    cudaGetLastError();
    return;
  }
  float a = 0.f, b = 0.f;
  if (cudaEventElapsedTime(&a, sl.t0, sl.t1) != cudaSuccess) a = 0.f;
  if (cudaEventElapsedTime(&b, sl.r0, sl.r1) != cudaSuccess) b = 0.f;
  cudaGetLastError();
  c->stage_ms[0] += a;
  c->stage_ms[1] += b;
  sl.timing_pending = false;
}

// Stage 1 of `pass` into `sl` on stream1 (proxy.cpp:684-736). Host synchronisation here
// only waits for stream1, so Stage 2 of the previous pass keeps running on `stream`.
// Stage-1 front of `pass` into `sl` on stream1: pool walks, priority selection, entries,
// probes and bounds (proxy.cpp:684-714, 389-395). Bounds of pass p see the bucket maxima
// after pass p-1's probes, so fronts run in pass order on the one stream.
void stage1_fronts(pxg_ctx* c, int p0, int L) {
  cudaStream_t st = c->stream1;
  HostProbe hp(st);
  for (int b = 0; b < L; ++b) {
    PoolSlot& sl = c->slot_of(p0 + b);
    CK(cudaStreamWaitEvent(st, sl.s2_done, 0));  // Stage 2 of the slot's previous pass is done
    sl.pass = p0 + b;
  }
  CK(cudaEventRecord(c->slot_of(p0).t0, st));
  for (int b = 0; b < L; ++b) {
    PoolSlot& sl = c->slot_of(p0 + b);
    CK(cudaMemsetAsync(sl.diag, 0, sizeof(long long) * kBuckets * 5, st));
    CK(cudaMemsetAsync(sl.diag_touched, 0, sizeof(int) * kBuckets, st));
  }
  const int walks = c->n_walks;
  CK(cudaMemsetAsync(c->d_ccount, 0, sizeof(int) * L, st));
  if (walks > 0) {
    // the pool walks of all L passes as one wavefront: walk w of pass p on (POOL_WALK, p<<32|w)
    const int nw = L * walks;
    CK(cudaMemsetAsync(c->d_wctr, 0, sizeof(unsigned) * nw, st));
    PathSet W{c->d_wpool, c->d_wnv, c->d_wctr, c->d_wbeta, c->d_wpdf, c->seed,
              (static_cast<uint64_t>(p0) << 32) + static_cast<uint64_t>(c->shard.walk_begin),
              PXG_KIND_POOL_WALK, nw, c->max_depth - 1, 0, walks};
    trace_paths(c, W, c->wA, c->wB, st);
    k_pool_keys<<<blocks(nw, 128), 128, 0, st>>>(c->d_wpool, c->d_wnv, walks, L, c->seed, p0, c->shard.walk_begin,
                                                 c->d_ckey, c->d_cval, c->d_ccount, c->cand_cap);
    ++c->launches;
    hp.mark("walks");
  }
  // priority selection, entry count, raw count and kappa of every pass on the device
  const int budget = c->P.pool_budget;
  const int B1 = std::max(budget, 1);
  FrontSet fs{};
  fs.n = L;
  for (int b = 0; b < L; ++b) {
    PoolSlot& sl = c->slot_of(p0 + b);
    fs.ps[b] = sl.ps;
    fs.inc[b] = sl.inc;
    fs.prefix[b] = sl.prefix;
  }
  k_pool_select<<<L, 1024, c->sel_smem, st>>>(c->d_ckey, c->d_cval, c->d_ccount, c->cand_cap, budget, c->sel_cap,
                                              c->d_sel, fs, c->d_err);
  ++c->launches;
  hp.mark("select");
  if (budget > 0) {
    const int R = c->P.recip_repeats;
    // entries and probes are independent across passes: one launch each for the batch
    k_pool_entries<<<dim3(blocks(budget, 64), L), 64, 0, st>>>(c->M, fs, c->d_sel, B1, c->d_wpool, L * walks,
                                                               walks, c->shard.walk_begin);
    k_pool_probes<<<dim3(blocks(4 * budget, 64), L), 64, 0, st>>>(c->S, c->seed, p0, fs, c->d_probe,
                                                                  c->d_probe_ok, 4 * B1, R);
    c->launches += 2;
  }
  // bounds in pass order: B of pass p sees the bucket maxima after pass p-1's probes
  for (int b = 0; b < L; ++b) {
    PoolSlot& sl = c->slot_of(p0 + b);
    if (budget > 0) {
      k_pool_bounds<<<1, 512, (6 * sizeof(double) + 5 * sizeof(int)) * budget, st>>>(
          sl.ps, sl.inc, c->d_probe + static_cast<size_t>(b) * 4 * B1,
          c->d_probe_ok + static_cast<size_t>(b) * 4 * B1, c->d_max_ratio, c->d_ratio_cnt, c->d_touched, sl.bound,
          c->d_err);
      ++c->launches;
    }
    // ratio statistics as of this pass (reported by pxg_read_stats; Stage 2 does not read them)
    CK(cudaMemcpyAsync(sl.snap_max, c->d_max_ratio, sizeof(double) * kBuckets, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(sl.snap_rcnt, c->d_ratio_cnt, sizeof(long long) * kBuckets, cudaMemcpyDeviceToDevice, st));
  }
  hp.mark("entries+bounds");
}

// One reciprocal round on stream `st`: evaluate nodes [avail, avail + chunk) of every active
// run (global wavefront, its overflow and the thread-per-node variant), then resume the DFS.
void recip_round(pxg_ctx* c, cudaStream_t st, const BatchSet& bs, int R, int stride, long long cap, int cur,
                 int chunk) {
  if (c->wave_blocks > 0) {
    int served = 0;
    if (c->rq.cap > 0) {
      // the global wavefront takes the first `served` runs of the list (all of them unless the
      // round outgrows the scratch); the block-local kernel takes the rest (usually none)
      served = c->rq.cap / chunk;
      int* fetch = c->d_trav_next + 1;
      RayQueue qa = c->rqA, qb = c->rqB;
      const int gsb = c->gs_blocks;
      CK(cudaMemsetAsync(qa.count, 0, sizeof(int), st));
      CK(cudaMemsetAsync(c->rqS.count, 0, sizeof(int), st));
      k_rq_setup<<<gsb, 128, 0, st>>>(c->S, c->seed, R, stride, cap, bs, c->d_ract[cur], c->d_rnact + cur, served,
                                      chunk, c->d_rstate, c->rq, qa);
      for (int step = 0; step < 4; ++step) {  // support_sample's chain: u <= 4 vertices
        CK(cudaMemsetAsync(fetch, 0, sizeof(int), st));
        launch_trav<false>(c, qa, fetch, st);
        CK(cudaMemsetAsync(qb.count, 0, sizeof(int), st));
        k_rq_glue<<<gsb / 2, kGlueT, 0, st>>>(c->S, c->seed, R, stride, bs, c->rq, qa, qb);
        std::swap(qa, qb);
      }
      k_rq_record<<<gsb / 2, kGlueT, 0, st>>>(c->S, R, stride, bs, c->d_rnact + cur, served, chunk, c->rq, c->rqS);
      CK(cudaMemsetAsync(fetch, 0, sizeof(int), st));
      launch_trav<true>(c, c->rqS, fetch, st);
      k_rq_vis<<<gsb, 256, 0, st>>>(c->rqS, c->rq);
      k_rq_finish<<<gsb, 128, 0, st>>>(c->seed, R, stride, cap, bs, c->d_rnact + cur, served, chunk, c->rq,
                                       c->d_rg, c->d_rn, c->d_re);
      c->launches += 13;
    }
    k_recip_eval_wave<<<c->wave_blocks, kRW, 0, st>>>(c->S, c->seed, R, stride, cap, bs, c->d_ract[cur],
                                                      c->d_rnact + cur, chunk, c->d_rstate, c->d_rg, c->d_rn,
                                                      c->d_re, c->d_rw_scratch, c->d_rw_ends, served);
  } else
    k_recip_eval<<<c->eval_blocks, 64, 0, st>>>(
        c->S, c->seed, R, stride, cap, bs, c->d_ract[cur], c->d_rnact + cur, chunk, c->d_rstate, c->d_rg,
        c->d_rn, c->d_re);
  k_recip_dfs_warp<128><<<c->dfs_blocks, 128, 0, st>>>(R, stride, cap, bs, 0.0, c->d_ract[cur],
                                                c->d_rnact + cur, chunk, c->d_rstate, c->d_rg, c->d_rn, c->d_re, c->d_frames,
                                                c->d_run_est, c->d_run_cost, c->d_run_trunc, c->d_ract[1 - cur],
                                                c->d_rnact + (1 - cur), c->d_err, c->d_node_stat);
  c->launches += 2;
}

// Stage 1 of passes [p0, p0 + L): the fronts in pass order, ONE set of reciprocal rounds
// for all L x budget x repeats runs (the long-run tail is paid once per batch), then the
// finishes in pass order (bucket estimate sums are sequential across passes).
void run_stage1_batch(pxg_ctx* c, int p0, int L) {
  cudaStream_t st = c->stream1;
  HostProbe hp(st);
  BatchSet bs{};
  bs.n = L;
  stage1_fronts(c, p0, L);
  for (int b = 0; b < L; ++b) {
    PoolSlot& sl = c->slot_of(p0 + b);
    bs.p[b] = BatchPass{sl.inc, sl.prefix, sl.bound, sl.ps, p0 + b};
  }
  const int R = c->P.recip_repeats;
  const int stride = std::max(c->P.pool_budget, 1) * std::max(R, 1);
  PoolSlot& s0 = c->slot_of(p0);
  CK(cudaEventRecord(s0.r0, st));
  if (R >= 1) {
    const int runs = L * stride;
    const long long cap = c->P.recursion_cap;
    CK(cudaMemsetAsync(c->d_rnact, 0, 2 * sizeof(int), st));
    k_recip_init<<<blocks(runs, 128), 128, 0, st>>>(runs, R, stride, bs, c->d_rstate, c->d_ract[0], c->d_rnact,
                                                   c->d_run_est, c->d_run_cost, c->d_run_trunc);
    c->recip_rounds = recip_rounds(st, cap, c->d_rnact, [&](int cur, int chunk) {
      recip_round(c, st, bs, R, stride, cap, cur, chunk);
    });
    c->launches += 1;
    if (std::getenv("PXG_PROFILE")) {  // run-cost distribution of this batch
      std::vector<long long> cost(runs);
      CK(cudaMemcpyAsync(cost.data(), c->d_run_cost, sizeof(long long) * runs, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::sort(cost.begin(), cost.end());
      long long sum = 0, live = 0;
      for (long long v : cost) sum += v, live += v > 0;
      auto q = [&](double f) { return cost[std::min<size_t>(runs - 1, static_cast<size_t>(f * runs))]; };
      std::fprintf(stderr, "[pxg] recip batch: runs %d live %lld nodes %lld p50 %lld p90 %lld p99 %lld p999 %lld max %lld\n",
                   runs, live, sum, q(0.5), q(0.9), q(0.99), q(0.999), cost[runs - 1]);
    }
  }
  CK(cudaEventRecord(s0.r1, st));
  hp.mark("recip");
  for (int b = 0; b < L; ++b) {
    PoolSlot& sl = c->slot_of(p0 + b);
    const size_t o = static_cast<size_t>(b) * stride;
    k_pool_finish<<<1, 1024, c->fin_smem, st>>>(
        R, sl.inc, sl.bound, c->d_run_est + o, c->d_run_trunc + o, c->d_sum_est, c->d_sum_sq, c->d_est_cnt,
        c->d_touched, sl.diag, sl.diag_touched, sl.kept, sl.label_start, sl.label_list, sl.ps, sl.snap_sum,
        sl.snap_sq, sl.snap_cnt);
    ++c->launches;
    CK(cudaEventRecord(sl.t1, st));
    CK(cudaEventRecord(sl.s1_done, st));
    sl.timing_pending = b == 0;
    sl.batch_end = p0 + L;
  }
  c->next_batch = p0 + L;
  hp.mark("finish");
}

// Stage 2 of `pass` on `stream` (proxy.cpp:738-827), reading pool slot `sl`.
// Stage 2 of `pass`, split in two stream-ordered halves (proj/src/proxy.cpp:738-827):
//   2a on stream_t: eye then light sub-paths of every pixel (the pixel's Rng stream continues
//      from pass to pass, so traces run in pass order on their own stream; they never read
//      Stage 1), into the vertex pools of buffer pass & 1;
//   2b on stream:   connections + MIS, proxy connection, gate + film, gamma, in pass order.
// 2a(p+1) overlaps 2b(p); 2a(p+2) waits until 2b(p) has released the buffer.
void activate_view(pxg_ctx* c, int row0, int rows) {
  const size_t off = static_cast<size_t>(row0 - c->row0_ctx) * c->width;
  const int cell_off = (row0 - c->row0_ctx) / 10 * c->grid_w;
  c->row0 = row0;
  c->rows = rows;
  c->n = rows * c->width;
  c->grid_h = (rows + 9) / 10;
  c->n_cells = c->grid_w * c->grid_h;
  const pxg_ctx::FullView& f = c->full;
  c->d_ctr = f.ctr + off;
  c->d_bdpt = f.bdpt + 3 * off;
  c->d_val = f.val + 3 * off;
  c->d_acc = f.acc + 3 * off;
  c->d_prox = f.prox + off;
  c->d_pflags = f.pflags + off;
  c->d_gbin = f.gbin + off;
  c->d_gval = f.gval + off;
  c->d_eye_prims = f.eye_prims + off * (c->max_depth + 1);
  c->d_light_prims = f.light_prims + off * std::max(c->max_depth - 1, 1);
  c->d_grid_total = f.grid_total + cell_off;
  c->d_grid_proxy = f.grid_proxy + cell_off;
  for (PathCache& pc : c->pcache_buf) pc.n = c->n;
  c->pcache.n = c->n;
}

void activate_tile(pxg_ctx* c, int t) {
  const int r0 = c->row0_ctx + t * c->tile_rows;
  activate_view(c, r0, std::min(c->tile_rows, c->row0_ctx + c->rows_ctx - r0));
}

void activate_ctx(pxg_ctx* c) { activate_view(c, c->row0_ctx, c->rows_ctx); }

void enqueue_stage2_tile(pxg_ctx* c, int pass, PoolSlot& sl, bool record_prims, bool first_tile, bool last_tile);

// Stage 2 of `pass` over the context's row tiles (one tile unless the image is too large for
// one working set), then the gamma update over the whole context in pixel order.
void enqueue_stage2(pxg_ctx* c, int pass, PoolSlot& sl, bool record_prims) {
  for (int t = 0; t < c->ntiles; ++t) {
    activate_tile(c, t);
    enqueue_stage2_tile(c, pass, sl, record_prims, t == 0, t == c->ntiles - 1);
  }
  activate_ctx(c);
  cudaStream_t st = c->stream;
  if (c->proxy_on && c->gamma_learning) {
    // record_contribution in pixel order: a stable sort by bin keeps pixel order per bin
    c->launches += stable_bin_sort(c->d_gbin, c->d_gval, c->n, c->d_gbin_sorted, c->d_gval_sorted, c->d_gsort_tmp, st);
    k_gamma_update<<<blocks(kT * kS, 128), 128, 0, st>>>(c->n, c->d_gbin_sorted, c->d_gval_sorted, c->d_gamma_accum,
                                                         c->d_gamma, 1);
    k_gamma_rows<<<1, 32, 0, st>>>(c->d_gamma_accum, c->d_gamma);
    c->launches += 2;
    ++c->gamma_iter;
    if (c->gamma_iter >= c->P.freeze_iteration) c->gamma_learning = false;
  }
  CK(cudaEventRecord(c->gamma_done, st));
  CK(cudaEventRecord(c->ev[7], st));
  CK(cudaEventRecord(sl.s2_done, st));
}

void enqueue_stage2_tile(pxg_ctx* c, int pass, PoolSlot& sl, bool record_prims, bool first_tile, bool last_tile) {
  cudaStream_t st = c->stream, tt = c->stream_t;
  const int T = 128;
  const int b = static_cast<int>(c->tile_step++ & 1);
  c->d_eye = c->eye_buf[b];
  c->d_light = c->light_buf[b];
  c->d_neye = c->neye_buf[b];
  c->d_nlight = c->nlight_buf[b];
  c->pcache = c->pcache_buf[b];
  HostProbe hp(st);
  // ---- 2a
  if (c->measure) CK(cudaStreamSynchronize(st));  // measurement: no 2a / 2b overlap
  CK(cudaStreamWaitEvent(tt, c->paths_free[b], 0));
  CK(cudaEventRecord(c->ev[1], tt));
  {
    PathSet E{c->d_eye, c->d_neye, c->d_ctr, c->d_ebeta, c->d_epdf, c->seed,
              static_cast<uint64_t>(c->row0) * c->width, PXG_KIND_REF, c->n, c->max_depth + 1, 1};
    PathSet L{c->d_light, c->d_nlight, c->d_ctr, c->d_lbeta, c->d_lpdf, c->seed,
              static_cast<uint64_t>(c->row0) * c->width, PXG_KIND_REF, c->n, c->max_depth - 1, 0};
    trace_paths(c, E, c->qA, c->qB, tt);
    trace_paths(c, L, c->qA, c->qB, tt);
    if (record_prims) {
      k_record_prims<<<blocks(c->n, T), T, 0, tt>>>(c->d_eye, c->d_neye, c->d_light, c->d_nlight, c->n,
                                                   c->max_depth, c->d_eye_prims, c->d_light_prims);
      ++c->launches;
    }
    // sub-path-only MIS step densities (used by the connections of this pass)
    k_path_factors<<<blocks((PXG_PF_MERGE ? 2ll : 4ll) * c->n, T), T, 0, tt>>>(c->S, c->d_eye, c->d_neye, c->d_light, c->d_nlight, c->n,
                                                  c->pcache);
    ++c->launches;
  }
  CK(cudaEventRecord(c->ev[4], tt));
  CK(cudaEventRecord(c->trace_done[b], tt));
  // ---- 2b
  CK(cudaEventRecord(c->ev[0], st));
  if (c->proxy_on) {
    CK(cudaStreamWaitEvent(st, sl.s1_done, 0));
    if (first_tile) {  // the pass's Stage-1 diagnostics, once
      k_fold_diag<<<blocks(kBuckets, 128), 128, 0, st>>>(sl.diag, sl.diag_touched, sl.ps, c->d_diag,
                                                         c->d_diag_touched, c->d_kept_total);
      ++c->launches;
    }
  }
  CK(cudaStreamWaitEvent(st, c->trace_done[b], 0));
  hp.mark("trace");
  // ---- 2b': the proxy connection forks here (it reads the eye sub-paths, the pool slot and
  // gamma, never the connections) and joins before the gate
  cudaStream_t sp = c->stream_p;
  if (c->proxy_on) {
    CK(cudaEventRecord(c->proxy_done, st));  // fork point: s1_done and trace_done already waited
    CK(cudaStreamWaitEvent(sp, c->proxy_done, 0));
    CK(cudaStreamWaitEvent(sp, c->gamma_done, 0));  // gamma of the previous pass
  }
  connections(c, c->proxy_on, sl);
  CK(cudaEventRecord(c->ev[5], st));
  hp.mark("connect");
  if (c->proxy_on) {
    if (c->measure) CK(cudaStreamWaitEvent(sp, c->ev[5], 0));  // measurement: no overlap with timed launches
    ProxCtx C{c->S, c->M, StatsView{c->d_max_ratio, sl.snap_sum, sl.snap_sq, sl.snap_cnt}, c->d_eye, c->d_neye,
              c->n, c->row0, c->width, c->max_depth, c->seed, sl.inc, sl.prefix, sl.label_start, sl.label_list,
              c->d_gamma, sl.ps};
    ProxWave& W = c->pw;
    RayQueue in = c->qP, out = c->qQ;
    CK(cudaMemsetAsync(in.count, 0, sizeof(int), sp));
    k_pxw_select<<<blocks(c->n, T), T, 0, sp>>>(C, W, pass, c->n_px_total, c->d_prox, in);
    for (int step = 0; step < 4; ++step) {
      int* fetch = c->d_trav_next + 3;
      CK(cudaMemsetAsync(fetch, 0, sizeof(int), sp));
      launch_trav<false>(c, in, fetch, sp);
      CK(cudaMemsetAsync(out.count, 0, sizeof(int), sp));
      k_pxw_retrace<<<blocks(c->n, T), T, 0, sp>>>(C, W, pass, c->n_px_total, in, out);
      std::swap(in, out);
    }
    CK(cudaMemsetAsync(c->qPS.count, 0, sizeof(int), sp));
    k_pxw_value<<<blocks(c->n, T), T, 0, sp>>>(C, W, c->qPS, c->d_prox);
    {
      int* fetch = c->d_trav_next + 4;
      CK(cudaMemsetAsync(fetch, 0, sizeof(int), sp));
      launch_trav<true>(c, c->qPS, fetch, sp);
    }
    k_pxw_occlusion<<<blocks(static_cast<long long>(c->n) * kMaxLight, T), T, 0, sp>>>(W, c->qPS);
    k_pxw_mis<<<blocks(c->n, T), T, 0, sp>>>(C, W, c->d_prox);
    c->launches += 13;
    CK(cudaEventRecord(c->ev[6], sp));
    CK(cudaEventRecord(c->proxy_done, sp));
    CK(cudaStreamWaitEvent(st, c->proxy_done, 0));  // join
  }
  CK(cudaEventRecord(c->paths_free[b], st));  // last reader of this pass's vertex pools
  if (!c->proxy_on) CK(cudaEventRecord(c->ev[6], st));
  hp.mark("proxy");
  k_gate<<<blocks(c->n_cells, 64), 64, 0, st>>>(
      c->n_cells, c->grid_w, c->row0, c->rows, c->width, pass, c->P.gate_high, c->P.gate_low, c->P.gate_threshold,
      static_cast<double>(c->light_walks), c->proxy_on ? 1 : 0, sl.ps, c->d_bdpt, c->d_prox, c->d_acc, c->d_val,
      c->d_grid_total, c->d_grid_proxy, c->d_gbin, c->d_gval, c->d_pflags, c->d_diag_attempt, c->d_diag_accept,
      c->d_diag_touched);
  ++c->launches;
  (void)last_tile;
  hp.mark("gate");
}

void read_stage2_timing(pxg_ctx* c) {
  auto el = [&](int a, int b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    return static_cast<double>(ms);
  };
  c->stage_ms[2] += el(1, 4);
  c->stage_ms[3] += el(4, 5);
  c->stage_ms[4] += el(5, 6);
  c->stage_ms[5] += el(6, 7);
}

// Renders `npass` passes. Stage 1 runs in batches of c->batch passes on stream1; while
// the GPU renders Stage 2 of one batch (enqueued without host synchronisation), the host
// drives Stage 1 of the next batch, so the two overlap.
void render_passes_impl(pxg_ctx* c, int npass, bool record_last, bool wait = true) {
  for (int k = 0; k < 8; ++k) c->stage_ms[k] = 0.0;
  c->launches = 0;
  CK(cudaEventRecord(c->ev_call[0], c->stream));
  if (wait) {  // a timed call: its work starts after the call's start event on every stream
    CK(cudaStreamWaitEvent(c->stream1, c->ev_call[0], 0));
    CK(cudaStreamWaitEvent(c->stream_t, c->ev_call[0], 0));
  }  // (asynchronous calls must not serialise the streams: one call per pass in the pipeline)
  // Pipeline fill: the first batches of a context grow geometrically (passes [0,1), [1,3),
  // [3,7), [7,15), then c->batch at a time), so Stage 2 starts after one pass of Stage 1
  // instead of a whole batch (the per-call render_proxy_bdpt path). Batch composition does
  // not change any result.
  auto batch_len = [&](int p0) {
    int L = p0 < c->batch ? std::min(c->batch, p0 + 1) : c->batch;
    if (c->pass_limit >= 0) L = std::min(L, std::max(1, c->pass_limit - p0));
    return L;
  };
  // Look-ahead: after every Stage-2 enqueue, Stage 1 is launched for every batch that fits in
  // the slot ring (within the pass limit), so each batch has one to two batches of Stage-2
  // time to finish even when the host runs only a few passes ahead (the pipelined pass_done
  // loop). Launched batches never reach passes_done + ring - 1: the ring keeps the last
  // rendered pass's slot for the dump / diagnostics readers.
  auto launch_ahead = [&]() {
    if (!c->proxy_on) return;
    for (;;) {
      const int q = c->passes_done, nb = c->next_batch;
      if (c->pass_limit >= 0 && nb >= c->pass_limit) break;
      const int L = batch_len(nb);
      if (nb + L > q + c->ring() - 1) break;  // a whole batch, as far ahead as the ring allows
      for (int i = 0; i < L; ++i) read_stage1_timing(c, c->slot_of(nb + i));
      run_stage1_batch(c, nb, L);
    }
  };
  static const bool overlap = std::getenv("PXG_NO_OVERLAP") == nullptr;
  for (int k = 0; k < npass; ++k) {
    const int p = c->passes_done;
    if (c->proxy_on && c->slot_of(p).pass != p) {  // first call, or the look-ahead stopped at the limit
      c->next_batch = p;
      run_stage1_batch(c, p, batch_len(p));
    }
    if (overlap && !c->measure) launch_ahead();
    // measurement mode: the streams are serialised so every timed traversal launch has the
    // GPU to itself (its duration is the kernel's, not a share of the Stage-1 overlap)
    if (c->measure) CK(cudaStreamSynchronize(c->stream1));
    enqueue_stage2(c, p, c->slot_of(p), record_last && k == npass - 1);
    CK(cudaGetLastError());
    ++c->passes_done;
    if (!overlap || c->measure) {
      CK(cudaStreamSynchronize(c->stream));
      launch_ahead();
    } else {
      launch_ahead();
    }
  }
  if (wait) {
    CK(cudaEventSynchronize(c->ev[7]));
    read_stage2_timing(c);  // the last pass of the call
  }
  if (!wait) return;  // asynchronous: the caller synchronises (snapshot / read)
  CK(cudaEventRecord(c->ev_call[2], c->stream1));
  CK(cudaStreamWaitEvent(c->stream, c->ev_call[2], 0));
  CK(cudaEventRecord(c->ev_call[1], c->stream));
  CK(cudaEventSynchronize(c->ev_call[1]));
  float total = 0.f;
  CK(cudaEventElapsedTime(&total, c->ev_call[0], c->ev_call[1]));
  c->stage_ms[6] = total;
  for (int i = 0; i < c->ring(); ++i) read_stage1_timing(c, c->slot[i]);
  check_err(c, c->stream);
}

int fail(pxg_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_global_err = msg;
  return code;
}

// Restores the caller's current device on exit (a host thread driving several GPUs keeps its
// own device selection across libpxg calls).
struct DeviceRestore {
  int dev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      cudaGetLastError();
      dev = -1;
    }
  }
  ~DeviceRestore() {
    if (dev >= 0) cudaSetDevice(dev);
  }
};

template <typename F>
int guarded(pxg_ctx* c, F&& f) {
  DeviceRestore keep;
  try {
    if (c) CK(cudaSetDevice(c->device));
    f();
    return PXG_OK;
  } catch (const CudaErr& e) {
    return fail(c, PXG_E_CUDA, e.msg);
  } catch (const InvalidErr& e) {
    return fail(c, PXG_E_INVALID, e.msg);
  } catch (const RuntimeErr& e) {
    return fail(c, PXG_E_RUNTIME, e.msg);
  } catch (const std::exception& e) {
    return fail(c, PXG_E_INVALID, e.what());
  }
}

void ensure_sincos_table(int device) {
  std::lock_guard<std::mutex> lk(g_sc_mu);
  if (device < 0 || device >= 64) throw InvalidErr{"pxg: device index out of range"};
  if (g_sc_device[device]) return;
  if (g_sc_file.empty()) {
    const std::string path = sincos_table_path();
    std::ifstream f(path, std::ios::binary);
    if (!f) throw InvalidErr{"pxg: sin/cos table " + path + " missing (run the build: python -m paper_2503_23412_b200.build)"};
    std::vector<char> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    uint32_t hdr[2] = {0, 0};
    if (buf.size() >= sizeof(hdr)) std::memcpy(hdr, buf.data(), sizeof(hdr));
    const size_t want = sizeof(hdr) + sizeof(double) * 2 * PXG_SC_RANGES + sizeof(uint32_t) * (PXG_SC_BUCKETS + 1) +
                        sizeof(uint16_t) * static_cast<size_t>(hdr[1]);
    if (hdr[0] != PXG_SC_MAGIC || buf.size() != want) throw InvalidErr{"pxg: sin/cos table " + path + " is corrupt"};
    g_sc_file.swap(buf);
  }
  const char* p = g_sc_file.data() + 2 * sizeof(uint32_t);
  const size_t bytes = g_sc_file.size() - 2 * sizeof(uint32_t);
  char* d = nullptr;
  CK(cudaMalloc(&d, bytes));  // process lifetime, shared by every context on the device
  CK(cudaMemcpy(d, p, bytes, cudaMemcpyHostToDevice));
  pxg_sincos_table t;
  t.thr = reinterpret_cast<const double*>(d);
  t.offset = reinterpret_cast<const uint32_t*>(d + sizeof(double) * 2 * PXG_SC_RANGES);
  t.entry = reinterpret_cast<const uint16_t*>(d + sizeof(double) * 2 * PXG_SC_RANGES + sizeof(uint32_t) * (PXG_SC_BUCKETS + 1));
  CK(cudaMemcpyToSymbol(pxg::g_sincos, &t, sizeof(t)));
  g_sc_device[device] = true;
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

void pxg_default_params(pxg_params* p) {
  p->enabled = 1;
  p->pool_budget = 400;
  p->recip_repeats = 5;
  p->freeze_iteration = 40;
  p->recursion_cap = 10000;
  p->pretrace_paths = 20000;
  p->light_walks = 0;
  p->gate_high = 1.0;
  p->gate_low = 0.2;
  p->gate_threshold = 0.05;
}

int pxg_abi_version(void) { return PXG_ABI_VERSION; }

int pxg_node_bytes(const pxg_ctx* c) {
  if (!c) return -1;
  return c->S.nodeq ? static_cast<int>(sizeof(BvhNode4Q)) : static_cast<int>(sizeof(BvhNode4));
}

int pxg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char* pxg_last_error(const pxg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_global_err.c_str(); }

void pxg_destroy(pxg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  delete ctx;
}

namespace {
void scene_build(const pxg_scene_desc* sd, pxg_scene* s) {
  const int n = sd->n_prims, nm = sd->n_materials, ne = sd->n_emitters;
  if (n < 0 || nm < 0 || ne < 0) throw InvalidErr{"scene: negative count"};
  s->shape.assign(sd->shape, sd->shape + n);
  s->material.assign(sd->material, sd->material + n);
  s->a.assign(sd->a, sd->a + 3 * static_cast<size_t>(n));
  s->b.assign(sd->b, sd->b + 3 * static_cast<size_t>(n));
  s->c.assign(sd->c, sd->c + 3 * static_cast<size_t>(n));
  s->radius.assign(sd->radius, sd->radius + n);
  s->materials.assign(sd->materials, sd->materials + 7 * static_cast<size_t>(nm));
  s->emitter_prim.assign(sd->emitter_prim, sd->emitter_prim + ne);
  s->emitter_radiance.assign(sd->emitter_radiance, sd->emitter_radiance + 3 * static_cast<size_t>(ne));
  s->desc = *sd;
  s->desc.shape = s->shape.data();
  s->desc.material = s->material.data();
  s->desc.a = s->a.data();
  s->desc.b = s->b.data();
  s->desc.c = s->c.data();
  s->desc.radius = s->radius.data();
  s->desc.materials = s->materials.data();
  s->desc.emitter_prim = s->emitter_prim.data();
  s->desc.emitter_radiance = s->emitter_radiance.data();
  if (sd->max_depth < 1) throw InvalidErr{"scene: max_depth must be at least 1"};
  if (sd->max_depth + 1 > kMaxPath - 2 || sd->max_depth - 1 > kMaxLight - 1)
    throw InvalidErr{"pxg: max_depth above 16 is not supported"};
  finalize_scene(s->desc, s->host);
  s->host.nodes.clear();  // the binary tree is only the input of the 4-wide collapse
  s->host.nodes.shrink_to_fit();
  // page-lock the large arrays once, so every context uploads them at full PCIe speed
  auto pin = [&](void* p, size_t bytes) {
    if (bytes < (1u << 20)) return;
    if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) == cudaSuccess)
      s->pinned.emplace_back(p, bytes);
    else
      cudaGetLastError();  // not fatal: the upload falls back to staged copies
  };
  SceneHost& h = s->host;
  pin(h.nodes4.data(), h.nodes4.size() * sizeof(HostNode4));
  pin(h.nodes4q.data(), h.nodes4q.size() * sizeof(HostNode4Q));
  pin(h.recs.data(), h.recs.size() * sizeof(HostRec));
  pin(h.prim_abc.data(), h.prim_abc.size() * sizeof(double));
  pin(h.prim_geo.data(), h.prim_geo.size() * sizeof(double));
  pin(h.prim_center.data(), h.prim_center.size() * sizeof(double));
}

int create_impl(const pxg_scene* scn, const pxg_params* params, uint64_t seed, int device, const pxg_shard* shard,
                pxg_ctx** out);
}  // namespace

int pxg_scene_create(const pxg_scene_desc* sd, pxg_scene** out) {
  if (!sd || !out) return fail(nullptr, PXG_E_INVALID, "pxg_scene_create: null argument");
  *out = nullptr;
  auto* s = new pxg_scene();
  const int rc = guarded(nullptr, [&]() { scene_build(sd, s); });
  if (rc != PXG_OK) {
    delete s;
    return rc;
  }
  *out = s;
  return PXG_OK;
}

void pxg_scene_destroy(pxg_scene* s) { delete s; }

long long pxg_scene_device_bytes(const pxg_scene* s) {
  if (!s) return -1;
  const SceneHost& h = s->host;
  return static_cast<long long>(h.nodes4.size() * sizeof(HostNode4) + h.nodes4q.size() * sizeof(HostNode4Q) +
                                h.recs.size() * sizeof(HostRec) +
                                (h.prim_mat.size() + h.prim_emitter.size() + h.prim_shape.size()) * sizeof(int) +
                                (h.prim_geo.size() + h.prim_center.size() + h.prim_abc.size() + h.emitter_cum.size() +
                                 s->emitter_radiance.size()) * sizeof(double) +
                                s->emitter_prim.size() * sizeof(int) + s->materials.size() * sizeof(double));
}

int pxg_create_from_scene(const pxg_scene* scene, const pxg_params* params, uint64_t seed, int device,
                          const pxg_shard* shard, pxg_ctx** out) {
  if (!scene || !out) return fail(nullptr, PXG_E_INVALID, "pxg_create_from_scene: null argument");
  return create_impl(scene, params, seed, device, shard, out);
}

int pxg_create(const pxg_scene_desc* sd, const pxg_params* params, uint64_t seed, int device,
               const pxg_shard* shard, pxg_ctx** out) {
  if (!sd || !out) return fail(nullptr, PXG_E_INVALID, "pxg_create: null argument");
  *out = nullptr;
  if (pxg_device_count() <= 0) return fail(nullptr, PXG_E_NODEVICE, "pxg_create: no CUDA device");
  pxg_scene* s = nullptr;
  int rc = pxg_scene_create(sd, &s);
  if (rc != PXG_OK) return rc;
  rc = create_impl(s, params, seed, device, shard, out);
  pxg_scene_destroy(s);  // the context holds device copies only
  return rc;
}

namespace {
int create_impl(const pxg_scene* scn, const pxg_params* params, uint64_t seed, int device, const pxg_shard* shard,
                pxg_ctx** out) {
  const pxg_scene_desc* sd = &scn->desc;
  *out = nullptr;
  if (pxg_device_count() <= 0) return fail(nullptr, PXG_E_NODEVICE, "pxg_create: no CUDA device");
  auto* c = new pxg_ctx();
  c->device = device;
  int rc = guarded(c, [&]() {
    // PXG_PROFILE: host timestamps of the creation phases (debugging aid)
    static const bool prof = std::getenv("PXG_PROFILE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (!prof) return;
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
      std::fprintf(stderr, "[pxg] create %-12s %8.2f ms\n", what, ms);
    };
    if (params) c->P = *params; else pxg_default_params(&c->P);
    c->seed = seed;
    CK(cudaSetDevice(device));
    ensure_sincos_table(device);
    {
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = ~0ull;
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    {
      // Stage 1 is a chain of small latency-bound launches (reciprocal rounds): give it the
      // highest priority so its blocks are scheduled ahead of Stage 2's wide kernels.
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&c->stream1, cudaStreamNonBlocking, hi));
      CK(cudaStreamCreateWithFlags(&c->stream_t, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&c->stream_p, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->proxy_done, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->gamma_done, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->x_in, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->x_out, cudaEventDisableTiming));
    }
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    for (auto& e : c->ev_call) CK(cudaEventCreate(&e));
    mark("streams");
    const SceneHost& h = scn->host;
    c->width = sd->width;
    c->height = sd->height;
    c->max_depth = sd->max_depth;
    c->n_px_total = sd->width * sd->height;
    c->light_walks = c->P.light_walks > 0 ? c->P.light_walks : c->n_px_total;
    if (shard) {
      c->shard = *shard;
    } else {
      c->shard = pxg_shard{0, sd->height, 0, c->light_walks};
    }
    if (c->shard.row_begin < 0 || c->shard.row_end > sd->height || c->shard.row_begin >= c->shard.row_end ||
        (c->shard.row_begin % 10) != 0 || c->shard.walk_begin < 0 || c->shard.walk_end > c->light_walks ||
        c->shard.walk_begin > c->shard.walk_end)
      throw InvalidErr{"pxg_create: invalid shard"};
    c->row0 = c->shard.row_begin;
    c->rows = c->shard.row_end - c->shard.row_begin;
    c->n = c->rows * c->width;
    c->row0_ctx = c->row0;
    c->rows_ctx = c->rows;
    c->n_ctx = c->n;
    bool any_spec = false;
    std::vector<Material> mats(sd->n_materials);
    for (int m = 0; m < sd->n_materials; ++m) {
      const double* q = sd->materials + 7 * m;
      Material& M = mats[m];
      M.base_color = v3(q[0], q[1], q[2]);
      M.metallic = q[3];
      M.roughness = q[4];
      M.transmission = q[5];
      M.ior = q[6];
      M.specular = ((M.metallic >= 0.5 || M.transmission >= 0.5) && M.roughness < 0.2) ? 1 : 0;
      M.pad = 0;
      any_spec = any_spec || M.specular;
    }
    c->proxy_on = c->P.enabled != 0;
    (void)any_spec;
    // device scene
    SceneView& S = c->S;
    S.nodes = nullptr;  // the binary tree stays on the host (pxg_scene)
    S.nodes4 = reinterpret_cast<const BvhNode4*>(c->upload_async(h.nodes4));
    if (reinterpret_cast<uintptr_t>(S.nodes4) % 32 != 0) throw CudaErr{"pxg_create: node array not 32-byte aligned"};
    S.nodes4q = h.nodeq ? reinterpret_cast<const BvhNode4Q*>(c->upload_async(h.nodes4q)) : nullptr;
    S.nodeq = PXG_NODEQ && h.nodeq;  // chosen per scene in finalize_scene (pxg_host.cpp)
    if (reinterpret_cast<uintptr_t>(S.nodes4q) % 32 != 0) throw CudaErr{"pxg_create: node array not 32-byte aligned"};
    S.recs = reinterpret_cast<const PrimRec*>(c->upload_async(h.recs));
    S.prim_mat = c->upload_async(h.prim_mat);
    S.prim_emitter = c->upload_async(h.prim_emitter);
    S.prim_geo = c->upload_async(h.prim_geo);
    S.prim_center = c->upload_async(h.prim_center);
    S.prim_shape = c->upload_async(h.prim_shape);
    S.prim_abc = c->upload_async(h.prim_abc);
    S.materials = c->upload(mats);
    S.emitter_prim = c->upload_async(scn->emitter_prim);
    S.emitter_rad = c->upload_async(scn->emitter_radiance);
    S.emitter_cum = c->upload_async(h.emitter_cum);
    S.n_prims = sd->n_prims;
    S.n_emit = sd->n_emitters;
    S.n_nodes = static_cast<int>(h.nodes4.size());
    S.n_mat = sd->n_materials;
    S.total_emitter_area = h.total_emitter_area;
    S.bbox_min = v3(h.bbox_min[0], h.bbox_min[1], h.bbox_min[2]);
    S.bbox_max = v3(h.bbox_max[0], h.bbox_max[1], h.bbox_max[2]);
    S.cam_pos = v3(h.cam[0], h.cam[1], h.cam[2]);
    S.cam_fwd = v3(h.cam[3], h.cam[4], h.cam[5]);
    S.cam_right = v3(h.cam[6], h.cam[7], h.cam[8]);
    S.cam_up = v3(h.cam[9], h.cam[10], h.cam[11]);
    S.tan_half = h.tan_half;
    S.aspect = h.aspect;
    S.width = sd->width;
    S.height = sd->height;
    S.max_depth = sd->max_depth;
    c->M.bmin = S.bbox_min;
    c->M.bmax = S.bbox_max;
    // stage-2 buffers: full-size per-pixel state, tile-size working set (see pxg_ctx::tile_rows)
    {
      int ms = 0;
      for (int t = 2; t <= c->max_depth + 1; ++t) ms += 1 + std::min(c->max_depth - 1, c->max_depth + 1 - t);
      c->max_slots = ms;
      const double D = c->max_depth;
      // bytes per pixel of the tile-size working set: 2 eye + 2 light vertex pools, proxy
      // scratch, connection slots + their shadow queue, step caches, queues
      const double per_px = 128.0 * (2 * (D + 1) + 2 * (D - 1) + kMaxLight) + ms * (40.0 + 80.0) +
                            2.0 * 4 * kMaxPath * 8 + kMaxLight * 80.0 + 4 * 80.0 + 256.0;
      const char* tb = std::getenv("PXG_TILE_BUDGET_GB");
      const double budget = (tb ? std::atof(tb) : 64.0) * 1e9;
      int tr = c->rows_ctx;
      if (static_cast<double>(c->n_ctx) * per_px > budget)
        tr = std::max(10, static_cast<int>(budget / per_px / c->width) / 10 * 10);
      if (const char* e = std::getenv("PXG_TILE_ROWS")) tr = std::max(10, std::atoi(e) / 10 * 10);
      c->tile_rows = std::min(tr, c->rows_ctx);
      c->ntiles = (c->rows_ctx + c->tile_rows - 1) / c->tile_rows;
      if (c->ntiles > 1 && (c->row0_ctx % 10) != 0) throw InvalidErr{"pxg_create: tiled shard must start on the gate grid"};
    }
    const size_t nc = c->n_ctx;
    const size_t n = static_cast<size_t>(c->tile_rows) * c->width;  // tile-size working set
    c->full.ctr = c->zeros<unsigned>(nc);
    c->full.bdpt = c->zeros<double>(3 * nc);
    c->full.val = c->zeros<double>(3 * nc);
    c->full.acc = c->zeros<double>(3 * nc);
    c->full.prox = c->zeros<ProxRec>(nc);
    c->full.pflags = c->zeros<int>(nc);
    c->full.gbin = c->zeros<int>(nc);
    c->full.gval = c->zeros<double>(nc);
    c->full.eye_prims = c->zeros<int>(nc * (c->max_depth + 1));
    c->full.light_prims = c->zeros<int>(nc * std::max(c->max_depth - 1, 1));
    for (int k = 0; k < 2; ++k) {
      c->eye_buf[k] = c->alloc<PV>(n * (c->max_depth + 1));
      c->light_buf[k] = c->alloc<PV>(n * std::max(c->max_depth - 1, 1));
      c->neye_buf[k] = c->zeros<int>(n);
      c->nlight_buf[k] = c->zeros<int>(n);
      CK(cudaEventCreateWithFlags(&c->trace_done[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->paths_free[k], cudaEventDisableTiming));
    }
    c->d_eye = c->eye_buf[0];
    c->d_light = c->light_buf[0];
    c->d_neye = c->neye_buf[0];
    c->d_nlight = c->nlight_buf[0];
    c->d_scratch = c->alloc<PV>(n * kMaxLight);
    c->pw.entry = c->zeros<int>(n);
    c->pw.tp = c->zeros<int>(n);
    c->pw.ctr = c->zeros<unsigned>(n);
    c->pw.step = c->zeros<int>(n);
    c->pw.state = c->zeros<int>(n);
    c->pw.density = c->zeros<double>(n);
    c->pw.pdf = c->zeros<double>(n);
    c->pw.value = c->zeros<double>(3 * n);
    c->pw.occl = c->zeros<int>(n);
    c->pw.lv = c->d_scratch;
    for (int k = 0; k < pxg_ctx::kSnap; ++k) {
      c->d_snap[k] = c->alloc<double>(3 * nc);
      CK(cudaEventCreateWithFlags(&c->snap_ev[k], cudaEventDisableTiming));
    }
    c->pinned_bytes = sizeof(double) * 3 * nc;
    c->h_pinned = static_cast<double*>(pinned_acquire(c->pinned_bytes));
    c->h_err = static_cast<int*>(pinned_acquire(pxg_ctx::kSnap * sizeof(int)));
    for (int k = 0; k < pxg_ctx::kSnap; ++k) c->h_err[k] = 0;
    c->d_ebeta = c->zeros<double>(3 * n);
    c->d_epdf = c->zeros<double>(n);
    c->d_lbeta = c->zeros<double>(3 * n);
    c->d_lpdf = c->zeros<double>(n);
    const size_t slots = n * static_cast<size_t>(c->max_slots);
    c->conn.count = c->zeros<int>(n + 1);
    c->conn.offset = c->zeros<int>(n + 1);
    c->conn.desc = c->alloc<int2>(slots);
    c->conn.value = c->alloc<double>(3 * slots);
    c->conn.state = c->zeros<int>(slots);
    c->conn.total = c->zeros<int>(1);
    c->conn.live = c->alloc<int>(slots);
    c->conn.n_live = c->zeros<int>(1);
    {
      const size_t L = static_cast<size_t>(kMaxPath);
      for (PathCache& pc : c->pcache_buf) {
        pc.LF = c->zeros<double>(L * n);
        pc.LR = c->zeros<double>(L * n);
        pc.EF = c->zeros<double>(L * n);
        pc.ER = c->zeros<double>(L * n);
        pc.ld = c->zeros<double>(n);
        pc.ld_ok = c->zeros<int>(n);
        pc.n = static_cast<int>(n);
      }
      c->pcache = c->pcache_buf[0];
    }
    c->qS = make_queue(c, slots);
    c->n_walks = c->shard.walk_end - c->shard.walk_begin;
    c->qA = make_queue(c, n);
    c->qB = make_queue(c, n);
    c->qP = make_queue(c, n);
    c->qQ = make_queue(c, n);
    c->qPS = make_queue(c, n * kMaxLight);
    {
      c->d_scan_tmp = c->alloc<int>(scan_tiles(static_cast<long long>(n) + 1));
    }
    {
      const char* eb = std::getenv("PXG_BATCH");
      c->batch = std::max(1, std::min(pxg_ctx::kBatchMax, eb ? std::atoi(eb) : pxg_ctx::kBatchDefault));
      if (!eb && c->proxy_on && c->n_walks > 0) {
        // a batch holds the vertex pools of all its passes' walks: cap it to a memory budget
        // (4M walks at depth 16 take 8 GB per pass). Batch composition changes no result.
        const double per_pass = static_cast<double>(c->n_walks) *
                                (128.0 * std::max(c->max_depth - 1, 1) + 2 * 80.0 + 48.0 + 12.0 * c->max_depth);
        const char* wb = std::getenv("PXG_WALK_BUDGET_GB");
        const double budget = (wb ? std::atof(wb) : 32.0) * 1e9;
        c->batch = std::max(1, std::min(c->batch, static_cast<int>(budget / per_pass)));
      }
    }
    if (!std::getenv("PXG_SHADE_PERM") || std::atoi(std::getenv("PXG_SHADE_PERM")) != 0) {  // 0: one-kernel k_shade (A/B)
      const size_t w = (c->proxy_on && c->n_walks > 0) ? static_cast<size_t>(c->n_walks) * c->batch : 0;
      c->shade_perm[0] = c->alloc<int>(n + kOrderT);
      c->shade_perm[1] = c->alloc<int>(w + kOrderT);
    }
    if (c->proxy_on && c->n_walks > 0) {
      const size_t w = static_cast<size_t>(c->n_walks) * c->batch;  // the walks of a whole batch
      c->wA = make_queue(c, w);
      c->wB = make_queue(c, w);
      c->d_wpool = c->alloc<PV>(w * std::max(c->max_depth - 1, 1));
      c->d_wnv = c->zeros<int>(w);
      c->d_wctr = c->zeros<unsigned>(w);
      c->d_wbeta = c->zeros<double>(3 * w);
      c->d_wpdf = c->zeros<double>(w);
    }
    c->grid_w = (c->width + 9) / 10;
    c->n_cells_ctx = c->grid_w * ((c->rows_ctx + 9) / 10);
    c->full.grid_total = c->zeros<double>(c->n_cells_ctx);
    c->full.grid_proxy = c->zeros<double>(c->n_cells_ctx);
    c->d_gbin_sorted = c->zeros<int>(nc);
    c->d_gval_sorted = c->zeros<double>(nc);
    {
      c->d_gsort_tmp = c->alloc<int>(sort_tmp_ints(static_cast<int>(nc)));
    }
    activate_ctx(c);
    // stats
    c->d_max_ratio = c->zeros<double>(kBuckets);
    c->d_sum_est = c->zeros<double>(kBuckets);
    c->d_sum_sq = c->zeros<double>(kBuckets);
    c->d_ratio_cnt = c->zeros<long long>(kBuckets);
    c->d_est_cnt = c->zeros<long long>(kBuckets);
    c->d_touched = c->zeros<int>(kBuckets);
    c->gamma_learning = c->P.freeze_iteration > 0;  // GammaMatrix::uniform (subspace.cpp:130-141)
    c->gamma_iter = 0;
    c->d_gamma = c->upload(std::vector<double>(kT * kS, 1.0 / kS));
    c->d_gamma_accum = c->zeros<double>(kT * kS);
    // pool
    const int walks = c->shard.walk_end - c->shard.walk_begin;
    c->cand_cap = std::max(1, walks) * std::max(1, c->max_depth - 2);
    c->d_ckey = c->alloc<unsigned long long>(static_cast<size_t>(c->cand_cap) * c->batch);
    c->d_cval = c->alloc<unsigned>(static_cast<size_t>(c->cand_cap) * c->batch);
    c->d_ccount = c->zeros<int>(c->batch);
    if (c->P.pool_budget > 3072) throw InvalidErr{"pxg: pool_budget above 3072 is not supported"};
    {
      // device priority selection: 2 x budget expected keys below the first threshold
      int cap = 1024;
      while (cap < 4 * c->P.pool_budget) cap <<= 1;
      c->sel_cap = cap;
      c->sel_smem = static_cast<size_t>(cap) * (sizeof(unsigned long long) + sizeof(unsigned));
      CK(cudaFuncSetAttribute(k_pool_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(c->sel_smem)));
      const int b = std::max(c->P.pool_budget, 0);
      CK(cudaFuncSetAttribute(k_pool_bounds, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>((6 * sizeof(double) + 5 * sizeof(int)) * b)));
      int n2 = 1;
      while (n2 < b) n2 <<= 1;
      c->fin_smem = sizeof(unsigned long long) * n2 + (sizeof(double) + 2 * sizeof(int)) * b +
                    sizeof(int) * (kS + 1024);
      CK(cudaFuncSetAttribute(k_pool_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(c->fin_smem)));
    }
    const int B = std::max(c->P.pool_budget, 1);
    const int R = std::max(c->P.recip_repeats, 1);
    c->d_sel = c->alloc<unsigned>(static_cast<size_t>(B) * c->batch);
    c->d_probe = c->zeros<double>(4 * static_cast<size_t>(B) * c->batch);
    c->d_probe_ok = c->zeros<int>(4 * static_cast<size_t>(B) * c->batch);
    for (int si = 0; si < c->ring(); ++si) {
      PoolSlot& sl = c->slot[si];
      sl.inc = c->zeros<IncHdr>(B);
      sl.prefix = c->alloc<PV>(static_cast<size_t>(B) * kMaxLight);
      sl.kept = c->zeros<int>(B);
      sl.label_start = c->zeros<int>(kS + 1);
      sl.label_list = c->zeros<int>(B);
      sl.ps = c->zeros<PassState>(1);
      sl.bound = c->zeros<double>(B);
      sl.diag = c->zeros<long long>(kBuckets * 5);
      sl.diag_touched = c->zeros<int>(kBuckets);
      sl.snap_sum = c->zeros<double>(kBuckets);
      sl.snap_sq = c->zeros<double>(kBuckets);
      sl.snap_cnt = c->zeros<long long>(kBuckets);
      sl.snap_max = c->zeros<double>(kBuckets);
      sl.snap_rcnt = c->zeros<long long>(kBuckets);
      for (cudaEvent_t* e : {&sl.s1_done, &sl.s2_done, &sl.t0, &sl.t1, &sl.r0, &sl.r1}) CK(cudaEventCreate(e));
    }
    const size_t NR = static_cast<size_t>(B) * R * c->batch;  // reciprocal runs of one Stage-1 batch
    c->d_run_est = c->zeros<double>(NR);
    c->d_run_cost = c->zeros<long long>(NR);
    c->d_run_trunc = c->zeros<int>(NR);
    if (c->P.recursion_cap > (1 << 20) || c->P.recip_repeats > 255)
      throw InvalidErr{"pxg: recursion_cap above 2^20 or recip_repeats above 255 is not supported"};
    if (c->proxy_on && c->P.recursion_cap > 0) {
      const size_t rc = NR * static_cast<size_t>(c->P.recursion_cap);
      c->d_frames = c->alloc<RecipFrame>(rc);
      c->d_rg = c->alloc<double>(rc);
      c->d_rn = c->alloc<long long>(rc);
      c->d_re = c->alloc<int>(rc);
    }
    c->d_rstate = c->alloc<RunState>(NR);
    c->d_ract[0] = c->alloc<int>(NR);
    c->d_ract[1] = c->alloc<int>(NR);
    c->d_rnact = c->zeros<int>(2);
    c->d_err = c->zeros<int>(1);
    c->d_kept_total = c->zeros<unsigned long long>(2);  // kept, raw
    c->d_tcnt = c->zeros<unsigned long long>(6);
    c->d_trav_next = c->zeros<int>(8);
    {
      int sms = 0, per_sm = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      c->trav_minb = c->S.nodeq ? 8 : 6;
      if (const char* e = std::getenv("PXG_TRAV_MINB")) c->trav_minb = std::atoi(e) == 8 ? 8 : 6;
      c->trav_post = c->S.nodeq != 0;
      if (const char* e = std::getenv("PXG_TRAV_POSTPONE")) c->trav_post = std::atoi(e) != 0;
      if (c->trav_minb == 8)
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trav_persistent<false, PXG_TRAV_HI, true, 1>, 128, 0));
      else
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trav_persistent<false, 6, false, 0>, 128, 0));
      c->trav_blocks = std::max(1, sms * std::max(per_sm, 1));
      c->gs_blocks = sms * (std::getenv("PXG_GS_PER_SM") ? std::atoi(std::getenv("PXG_GS_PER_SM")) : 256);
      int pe = 0, pd = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pe, k_recip_eval, 64, 0));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pd, k_recip_dfs_warp<128>, 128, 0));
      c->eval_blocks = std::max(1, sms * std::max(pe, 1));
      c->dfs_blocks = std::max(1, sms * std::max(pd, 1));
      // PXG_RECIP_WAVE=0 selects the thread-per-node evaluation (A/B experiments)
      static const bool wave = !std::getenv("PXG_RECIP_WAVE") || std::atoi(std::getenv("PXG_RECIP_WAVE")) != 0;
      if (wave && c->proxy_on) {
        int pw = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pw, k_recip_eval_wave, kRW, 0));
        c->wave_blocks = std::max(1, sms * std::max(pw, 1));
        c->d_rw_scratch = c->alloc<PV>(static_cast<size_t>(c->wave_blocks) * kRW * 4);
        c->d_rw_ends = c->alloc<double>(static_cast<size_t>(c->wave_blocks) * kRW * 60);
        // PXG_RECIP_QUEUE=0: block-local wavefront only (A/B); PXG_RQ_ITEMS: scratch capacity in nodes
        static const bool queue = !std::getenv("PXG_RECIP_QUEUE") || std::atoi(std::getenv("PXG_RECIP_QUEUE")) != 0;
        if (queue && c->P.recursion_cap > 0 && NR > 0) {
          const long long want = std::getenv("PXG_RQ_ITEMS") ? std::atoll(std::getenv("PXG_RQ_ITEMS")) : (4ll << 20);
          const long long most = static_cast<long long>(NR) * std::min<long long>(c->P.recursion_cap, 16384);
          const size_t items = static_cast<size_t>(std::max<long long>(1024, std::min(want, most)));
          c->rq.item = c->alloc<RqItem>(items);
          c->rq.gv = c->alloc<PV>(items * 4);
          c->rq.cap = static_cast<int>(items);
          c->rqA = make_queue(c, items);
          c->rqB = make_queue(c, items);
          c->rqS = make_queue(c, items * 10);  // <= 10 visibility segments per node
        }
      }
      c->d_node_stat = c->zeros<unsigned long long>(4);
    }
    c->d_diag = c->zeros<long long>(kBuckets * 5);
    c->d_diag_attempt = c->zeros<unsigned long long>(kBuckets);
    c->d_diag_accept = c->zeros<unsigned long long>(kBuckets);
    c->d_diag_touched = c->zeros<int>(kBuckets);
    mark("buffers");
    if (c->proxy_on) {
      const int np = std::max(c->P.pretrace_paths, 1000);
      k_pretrace<<<blocks(np, 64), 64, 0, c->stream>>>(c->S, c->M, c->seed, np, c->d_max_ratio, c->d_ratio_cnt,
                                                       c->d_touched, c->d_err);
      CK(cudaGetLastError());
      check_err(c, c->stream);
    }
    CK(cudaDeviceSynchronize());
    mark("pretrace");
  });
  if (rc != PXG_OK) {
    g_global_err = c->err;
    delete c;
    return rc;
  }
  *out = c;
  return PXG_OK;
}
}  // namespace

int pxg_render_passes(pxg_ctx* c, int npass) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() { render_passes_impl(c, npass, false); });
}

int pxg_render_pass(pxg_ctx* c) { return pxg_render_passes(c, 1); }

int pxg_render_pass_traced(pxg_ctx* c) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() { render_passes_impl(c, 1, true); });
}

int pxg_measure_traversal(pxg_ctx* c, int npass, double* out) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() {
    CK(cudaMemset(c->d_tcnt, 0, 6 * sizeof(unsigned long long)));
    c->tl.clear();
    c->ev_used = 0;
    c->measure = true;
    try {
      render_passes_impl(c, npass, false);
    } catch (...) {
      c->measure = false;
      throw;
    }
    c->measure = false;
    CK(cudaDeviceSynchronize());
    double ms[2] = {0.0, 0.0};
    long long nl[2] = {0, 0};
    for (const auto& t : c->tl) {
      float e = 0.f;
      CK(cudaEventElapsedTime(&e, t.a, t.b));
      ms[t.kind] += e;
      nl[t.kind] += 1;
    }
    unsigned long long h[6];
    CK(cudaMemcpy(h, c->d_tcnt, sizeof(h), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 2; ++k) {
      out[5 * k + 0] = ms[k];
      out[5 * k + 1] = static_cast<double>(nl[k]);
      out[5 * k + 2] = static_cast<double>(h[3 * k + 0]);
      out[5 * k + 3] = static_cast<double>(h[3 * k + 1]);
      out[5 * k + 4] = static_cast<double>(h[3 * k + 2]);
    }
  });
}

int pxg_render_passes_async(pxg_ctx* c, int npass) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() { render_passes_impl(c, npass, false, false); });
}

int pxg_snapshot_mean(pxg_ctx* c, int slot) {
  if (!c || slot < 0 || slot >= pxg_ctx::kSnap) return fail(c, PXG_E_INVALID, "pxg_snapshot_mean: bad slot");
  return guarded(c, [&]() {
    CK(cudaMemcpyAsync(c->d_snap[slot], c->d_acc, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToDevice, c->stream));
    // the error flag as of these passes (Stage-1 errors of a pass are visible once its
    // Stage 2, which waits for them, has run), read without waiting for the look-ahead
    CK(cudaMemcpyAsync(c->h_err + slot, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaEventRecord(c->snap_ev[slot], c->stream));
    c->snap_passes[slot] = c->passes_done;
  });
}

int pxg_read_snapshot(pxg_ctx* c, int slot, double* rgb, int* passes) {
  if (!c || slot < 0 || slot >= pxg_ctx::kSnap) return fail(c, PXG_E_INVALID, "pxg_read_snapshot: bad slot");
  return guarded(c, [&]() {
    CK(cudaEventSynchronize(c->snap_ev[slot]));
    CK(cudaMemcpy(c->h_pinned, c->d_snap[slot], sizeof(double) * 3 * c->n, cudaMemcpyDeviceToHost));
    const double inv = 1.0 / static_cast<double>(c->snap_passes[slot] > 0 ? c->snap_passes[slot] : 1);
    for (size_t i = 0; i < 3 * static_cast<size_t>(c->n); ++i) rgb[i] = c->h_pinned[i] * inv;
    if (passes) *passes = c->snap_passes[slot];
    raise_err(c->h_err[slot]);
  });
}

int pxg_set_pass_limit(pxg_ctx* c, int limit) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  c->pass_limit = limit;
  return PXG_OK;
}

int pxg_synchronize(pxg_ctx* c) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() {
    for (cudaStream_t st : {c->stream_t, c->stream_p, c->stream1, c->stream}) CK(cudaStreamSynchronize(st));
    check_err(c, c->stream);  // a deferred estimator error of the enqueued passes
  });
}

int pxg_read_accum(pxg_ctx* c, double* rgb, int* passes) {
  return guarded(c, [&]() {
    CK(cudaMemcpyAsync(rgb, c->d_acc, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (passes) *passes = c->passes_done;
  });
}

int pxg_accum_to_device_async(pxg_ctx* c, double* dst, void* stream, int* passes) {
  return guarded(c, [&]() {
    if (!dst) throw InvalidErr{"pxg_accum_to_device_async: null destination"};
    cudaStream_t caller = static_cast<cudaStream_t>(stream);
    // dst is free once the caller's earlier work on it (e.g. the previous round's in-place
    // all-reduce) has run; the copy sees every pass enqueued so far (stream order on c->stream)
    CK(cudaEventRecord(c->x_in, caller));
    CK(cudaStreamWaitEvent(c->stream, c->x_in, 0));
    CK(cudaMemcpyAsync(dst, c->d_acc, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaEventRecord(c->x_out, c->stream));
    CK(cudaStreamWaitEvent(caller, c->x_out, 0));  // the caller's next work (the reduce) follows the copy
    if (passes) *passes = c->passes_done;
  });
}

int pxg_accum_to_device(pxg_ctx* c, double* dst, int* passes) {
  const int rc = pxg_accum_to_device_async(c, dst, nullptr, passes);
  if (rc != PXG_OK) return rc;
  return guarded(c, [&]() { CK(cudaEventSynchronize(c->x_out)); });
}

int pxg_read_mean(pxg_ctx* c, double* rgb, int* passes) {
  return guarded(c, [&]() {
    CK(cudaMemcpyAsync(rgb, c->d_acc, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const double d = static_cast<double>(c->passes_done > 0 ? c->passes_done : 1);
    for (size_t i = 0; i < 3 * static_cast<size_t>(c->n); ++i) rgb[i] = rgb[i] * (1.0 / d);
    if (passes) *passes = c->passes_done;
  });
}

int pxg_read_diag(pxg_ctx* c, long long* rows, int* touched, long long* pool) {
  return guarded(c, [&]() {
    CK(cudaStreamSynchronize(c->stream));
    std::vector<long long> d(kBuckets * 5);
    std::vector<unsigned long long> at(kBuckets), ac(kBuckets);
    std::vector<int> tc(kBuckets);
    unsigned long long kept[2] = {0, 0};
    CK(cudaMemcpy(d.data(), c->d_diag, sizeof(long long) * kBuckets * 5, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(at.data(), c->d_diag_attempt, sizeof(unsigned long long) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ac.data(), c->d_diag_accept, sizeof(unsigned long long) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tc.data(), c->d_diag_touched, sizeof(int) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(kept, c->d_kept_total, sizeof(kept), cudaMemcpyDeviceToHost));
    for (int k = 0; k < kBuckets; ++k) {
      d[k * 5 + 0] = static_cast<long long>(at[k]);
      d[k * 5 + 1] = static_cast<long long>(ac[k]);
    }
    if (rows) std::memcpy(rows, d.data(), sizeof(long long) * kBuckets * 5);
    if (touched) std::memcpy(touched, tc.data(), sizeof(int) * kBuckets);
    if (pool) {
      pool[0] = static_cast<long long>(kept[1]);
      pool[1] = static_cast<long long>(kept[0]);
    }
  });
}

int pxg_read_stats(pxg_ctx* c, double* stats3, long long* counts2, double* gamma_rows) {
  return guarded(c, [&]() {
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->stream1));
    // after pass p the statistics are the snapshot Stage 2 of pass p used (a look-ahead
    // Stage 1 may already have advanced the live tables)
    const double *pmax = c->d_max_ratio, *psum = c->d_sum_est, *psq = c->d_sum_sq;
    const long long *prc = c->d_ratio_cnt, *pec = c->d_est_cnt;
    if (c->proxy_on && c->passes_done > 0) {
      const PoolSlot& sl = c->slot_of(c->passes_done - 1);
      pmax = sl.snap_max;
      psum = sl.snap_sum;
      psq = sl.snap_sq;
      prc = sl.snap_rcnt;
      pec = sl.snap_cnt;
    }
    std::vector<double> a(kBuckets), b(kBuckets), s(kBuckets);
    std::vector<long long> rc(kBuckets), ec(kBuckets);
    CK(cudaMemcpy(a.data(), pmax, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), psum, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(s.data(), psq, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rc.data(), prc, sizeof(long long) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ec.data(), pec, sizeof(long long) * kBuckets, cudaMemcpyDeviceToHost));
    for (int k = 0; k < kBuckets; ++k) {
      if (stats3) {
        stats3[3 * k] = a[k];
        stats3[3 * k + 1] = b[k];
        stats3[3 * k + 2] = s[k];
      }
      if (counts2) {
        counts2[2 * k] = rc[k];
        counts2[2 * k + 1] = ec[k];
      }
    }
    if (gamma_rows) CK(cudaMemcpy(gamma_rows, c->d_gamma, sizeof(double) * kT * kS, cudaMemcpyDeviceToHost));
  });
}

int pxg_dump_pass(pxg_ctx* c, double* val, double* bdpt, double* cc, int* flags) {
  return guarded(c, [&]() {
    CK(cudaStreamSynchronize(c->stream));
    const size_t n = c->n;
    if (val) CK(cudaMemcpy(val, c->d_val, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (bdpt) CK(cudaMemcpy(bdpt, c->d_bdpt, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (cc) {
      std::vector<ProxRec> pr(n);
      CK(cudaMemcpy(pr.data(), c->d_prox, sizeof(ProxRec) * n, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) cc[3 * i + k] = c->proxy_on ? pr[i].c[k] : 0.0;
    }
    if (flags) CK(cudaMemcpy(flags, c->d_pflags, sizeof(int) * n, cudaMemcpyDeviceToHost));
  });
}

static_assert(sizeof(pxg_vertex) == sizeof(PV), "pxg_vertex mirrors PV");
static_assert(PXG_MAX_LIGHT == kMaxLight, "repaired light sub-path capacity");
static_assert(sizeof(pxg_path_record) == 184, "pxg_path_record layout (render.PATH_RECORD_DTYPE)");

int pxg_dump_paths(pxg_ctx* c, int px_begin, int px_end, pxg_path_record* rec, pxg_vertex* eye, pxg_vertex* light,
                   pxg_vertex* proxy, double* stats) {
  return guarded(c, [&]() {
    if (c->ntiles > 1) throw InvalidErr{"pxg_dump_paths: not available for Stage-2 row-tiled contexts"};
    if (px_begin < 0 || px_end > c->n || px_begin > px_end) throw InvalidErr{"pxg_dump_paths: pixel range"};
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->stream1));
    const int m = px_end - px_begin;
    const size_t n = c->n;
    const int de = c->max_depth + 1, dl = std::max(c->max_depth - 1, 1);
    // vertex-major device pools [k][pixel] -> pixel-major host rows, one strided copy per vertex index
    if (eye)
      for (int k = 0; k < de; ++k)
        CK(cudaMemcpy2D(eye + k, sizeof(PV) * de, c->d_eye + k * n + px_begin, sizeof(PV), sizeof(PV), m,
                        cudaMemcpyDeviceToHost));
    if (light)
      for (int k = 0; k < dl; ++k)
        CK(cudaMemcpy2D(light + k, sizeof(PV) * dl, c->d_light + k * n + px_begin, sizeof(PV), sizeof(PV), m,
                        cudaMemcpyDeviceToHost));
    std::vector<int> ne(m), nl(m);
    if (m) {
      CK(cudaMemcpy(ne.data(), c->d_neye + px_begin, sizeof(int) * m, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(nl.data(), c->d_nlight + px_begin, sizeof(int) * m, cudaMemcpyDeviceToHost));
    }
    std::vector<double> val(3 * m), bdpt(3 * m);
    if (m) {
      CK(cudaMemcpy(val.data(), c->d_val + 3 * px_begin, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(bdpt.data(), c->d_bdpt + 3 * px_begin, sizeof(double) * 3 * m, cudaMemcpyDeviceToHost));
    }
    std::vector<ProxRec> pr;
    std::vector<int> entry, tp;
    std::vector<double> dens;
    std::vector<PV> lv;
    std::vector<IncHdr> inc;
    std::vector<PV> pre;
    const bool px_on = c->proxy_on && c->passes_done > 0;
    if (px_on && m) {
      pr.resize(m);
      entry.resize(m);
      tp.resize(m);
      dens.resize(m);
      lv.resize(static_cast<size_t>(m) * kMaxLight);
      CK(cudaMemcpy(pr.data(), c->d_prox + px_begin, sizeof(ProxRec) * m, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(entry.data(), c->pw.entry + px_begin, sizeof(int) * m, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(tp.data(), c->pw.tp + px_begin, sizeof(int) * m, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(dens.data(), c->pw.density + px_begin, sizeof(double) * m, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(lv.data(), c->pw.lv + static_cast<size_t>(px_begin) * kMaxLight, sizeof(PV) * kMaxLight * m,
                    cudaMemcpyDeviceToHost));
      const PoolSlot& sl = c->slot_of(c->passes_done - 1);
      PassState ps;
      CK(cudaMemcpy(&ps, sl.ps, sizeof(PassState), cudaMemcpyDeviceToHost));
      if (ps.n_ent > 0) {
        inc.resize(ps.n_ent);
        pre.resize(static_cast<size_t>(ps.n_ent) * kMaxLight);
        CK(cudaMemcpy(inc.data(), sl.inc, sizeof(IncHdr) * ps.n_ent, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(pre.data(), sl.prefix, sizeof(PV) * kMaxLight * ps.n_ent, cudaMemcpyDeviceToHost));
      }
      if (stats) {
        std::vector<double> s(kBuckets), q(kBuckets);
        std::vector<long long> cnt(kBuckets);
        CK(cudaMemcpy(s.data(), sl.snap_sum, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(q.data(), sl.snap_sq, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cnt.data(), sl.snap_cnt, sizeof(long long) * kBuckets, cudaMemcpyDeviceToHost));
        for (int k = 0; k < kBuckets; ++k) {
          stats[3 * k] = s[k];
          stats[3 * k + 1] = q[k];
          stats[3 * k + 2] = static_cast<double>(cnt[k]);
        }
      }
    } else if (stats) {
      for (int k = 0; k < 3 * kBuckets; ++k) stats[k] = 0.0;
    }
    for (int i = 0; i < m; ++i) {
      pxg_path_record r;
      std::memset(&r, 0, sizeof(r));
      r.n_eye = ne[i];
      r.n_light = nl[i];
      r.entry = -1;
      for (int k = 0; k < 3; ++k) {
        r.val[k] = val[3 * i + k];
        r.bdpt[k] = bdpt[3 * i + k];
      }
      pxg_vertex* pv = proxy ? proxy + static_cast<size_t>(i) * kMaxLight : nullptr;
      if (pv) std::memset(pv, 0, sizeof(pxg_vertex) * kMaxLight);
      if (px_on) {
        const ProxRec& o = pr[i];
        r.flags = o.flags;
        r.q_sel = o.q_sel;
        for (int k = 0; k < 3; ++k) r.c[k] = o.c[k];
        if (o.flags & 1) r.tp = tp[i];
        if ((o.flags & 4) && entry[i] >= 0 && entry[i] < static_cast<int>(inc.size())) {
          const int e = entry[i];
          const IncHdr& h = inc[e];
          r.entry = e;
          r.u = h.u;
          r.n_prefix = h.n_prefix;
          r.has_cdir = h.has_cdir;
          r.c_label = h.c_label;
          r.s_label = h.s_label;
          r.key = h.key;
          r.cdir[0] = h.cdir.x;
          r.cdir[1] = h.cdir.y;
          r.cdir[2] = h.cdir.z;
          r.prefix_pdf = h.prefix_pdf;
          r.inverse_p = h.inverse_p;
          r.inverse_p_m2 = h.inverse_p_m2;
          if (o.flags & 16) r.retrace_density = dens[i];
          if (pv) {
            std::memcpy(pv, &pre[static_cast<size_t>(e) * kMaxLight], sizeof(PV) * h.n_prefix);
            if (o.flags & 16)  // device slot n_prefix + (u-1-j) holds g[j]
              for (int j = 0; j < h.u; ++j)
                std::memcpy(pv + h.n_prefix + j, &lv[static_cast<size_t>(i) * kMaxLight + h.n_prefix + (h.u - 1 - j)],
                            sizeof(PV));
            std::memcpy(pv + h.n_prefix + h.u, &h.spec_end, sizeof(PV));
          }
        }
      }
      if (rec) rec[i] = r;
    }
  });
}

int pxg_dump_prims(pxg_ctx* c, int* eye, int* light) {
  return guarded(c, [&]() {
    CK(cudaStreamSynchronize(c->stream));
    const size_t n = c->n;
    if (eye) CK(cudaMemcpy(eye, c->d_eye_prims, sizeof(int) * n * (c->max_depth + 1), cudaMemcpyDeviceToHost));
    if (light)
      CK(cudaMemcpy(light, c->d_light_prims, sizeof(int) * n * std::max(c->max_depth - 1, 1), cudaMemcpyDeviceToHost));
  });
}

int pxg_dump_pool(pxg_ctx* c, int cap, int* n_out, long long* raw, int* walk, int* end, int* key, double* inv_p,
                  double* inv_p_m2, double* bound) {
  return guarded(c, [&]() {
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamSynchronize(c->stream1));
    if (c->passes_done == 0 || !c->proxy_on) {
      if (n_out) *n_out = 0;
      if (raw) *raw = 0;
      return;
    }
    const PoolSlot& sl = c->slot_of(c->passes_done - 1);
    PassState ps;
    CK(cudaMemcpy(&ps, sl.ps, sizeof(PassState), cudaMemcpyDeviceToHost));
    const int n_ent = ps.n_ent;
    std::vector<IncHdr> inc(n_ent);
    std::vector<int> kept(std::max(ps.n_kept, 0));
    std::vector<double> bd(n_ent);
    if (n_ent) {
      CK(cudaMemcpy(inc.data(), sl.inc, sizeof(IncHdr) * n_ent, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(bd.data(), sl.bound, sizeof(double) * n_ent, cudaMemcpyDeviceToHost));
    }
    if (ps.n_kept > 0) CK(cudaMemcpy(kept.data(), sl.kept, sizeof(int) * ps.n_kept, cudaMemcpyDeviceToHost));
    const int m = std::min(cap, ps.n_kept);
    for (int i = 0; i < m; ++i) {
      const IncHdr& h = inc[kept[i]];
      if (walk) walk[i] = h.walk;
      if (end) end[i] = h.end;
      if (key) key[i] = h.key;
      if (inv_p) inv_p[i] = h.inverse_p;
      if (inv_p_m2) inv_p_m2[i] = h.inverse_p_m2;
      if (bound) bound[i] = bd[kept[i]];
    }
    if (n_out) *n_out = ps.n_kept;
    if (raw) *raw = ps.raw;
  });
}

int pxg_intersect(pxg_ctx* c, int n, const double* rays, const double* tmax, int* prim, double* t) {
  return guarded(c, [&]() {
    if (n <= 0) return;
    double* dr = dupload(rays, static_cast<size_t>(n) * 6);
    double* dt = tmax ? dupload(tmax, n) : nullptr;
    int* dp = dalloc<int>(n);
    double* dtt = dalloc<double>(n);
    k_intersect<<<blocks(n, 128), 128, 0, c->stream>>>(c->S, n, dr, dt, dp, dtt);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(prim, dp, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(t, dtt, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(dr);
    if (dt) cudaFree(dt);
    cudaFree(dp);
    cudaFree(dtt);
  });
}

int pxg_proxy_probe(pxg_ctx* c, int n_walk, const pxg_vertex* walk, int n_cand, const pxg_vertex* cand, int n_draws,
                    uint64_t seed, int* info, double* prefix_pdf, double* q, double* f, pxg_vertex* draw_cand,
                    double* draw_q, int* draw_escaped) {
  return guarded(c, [&]() {
    static_assert(sizeof(pxg_vertex) == sizeof(PV), "pxg_vertex is the device vertex record");
    if (!walk || !info || !prefix_pdf || n_walk < 1 || n_walk > kMaxLight)
      throw InvalidErr{"pxg_proxy_probe: walk of 1..16 vertices required"};
    if ((n_cand > 0 && (!cand || !q || !f)) || (n_draws > 0 && (!draw_cand || !draw_q || !draw_escaped)))
      throw InvalidErr{"pxg_proxy_probe: null output"};
    cudaStream_t st = c->stream;
    PV* dw = dupload(reinterpret_cast<const PV*>(walk), n_walk);
    IncHdr* dh = dalloc<IncHdr>(1);
    PV* dpre = dalloc<PV>(kMaxLight);
    int* dinfo = dalloc<int>(8);
    double* dpp = dalloc<double>(1);
    CK(cudaMemsetAsync(dinfo, 0, sizeof(int) * 8, st));
    CK(cudaMemsetAsync(dpp, 0, sizeof(double), st));
    k_probe_dropout<<<1, 32, 0, st>>>(c->M, dw, n_walk, dh, dpre, dinfo, dpp);
    CK(cudaMemcpyAsync(info, dinfo, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(prefix_pdf, dpp, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int u = info[0] ? info[1] : 0;
    if (u > 0 && n_cand > 0) {
      PV* dc = dupload(reinterpret_cast<const PV*>(cand), static_cast<size_t>(n_cand) * u);
      double* dq = dalloc<double>(n_cand);
      double* df = dalloc<double>(n_cand);
      k_probe_densities<<<blocks(n_cand, 64), 64, 0, st>>>(c->S, dh, dpre, n_cand, dc, dq, df);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(q, dq, sizeof(double) * n_cand, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(f, df, sizeof(double) * n_cand, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      cudaFree(dc), cudaFree(dq), cudaFree(df);
    }
    if (u > 0 && n_draws > 0) {
      PV* dc = dalloc<PV>(static_cast<size_t>(n_draws) * u);
      double* dq = dalloc<double>(n_draws);
      int* de = dalloc<int>(n_draws);
      CK(cudaMemsetAsync(dc, 0, sizeof(PV) * static_cast<size_t>(n_draws) * u, st));
      k_probe_samples<<<blocks(n_draws, 64), 64, 0, st>>>(c->S, seed, dh, dpre, n_draws, dc, dq, de);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(draw_cand, dc, sizeof(PV) * static_cast<size_t>(n_draws) * u, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(draw_q, dq, sizeof(double) * n_draws, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(draw_escaped, de, sizeof(int) * n_draws, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      cudaFree(dc), cudaFree(dq), cudaFree(de);
    }
    cudaFree(dw), cudaFree(dh), cudaFree(dpre), cudaFree(dinfo), cudaFree(dpp);
  });
}

int pxg_proxy_recip(pxg_ctx* c, int n_walk, const pxg_vertex* walk, double bound, int n_runs, double* est,
                    long long* cost, int* truncated) {
  return guarded(c, [&]() {
    if (!walk || !est || !cost || !truncated || n_walk < 1 || n_walk > kMaxLight || n_runs < 1)
      throw InvalidErr{"pxg_proxy_recip: walk of 1..16 vertices and output arrays required"};
    if (!(bound > 0.0)) throw RuntimeErr{"reciprocal: bound must be positive"};
    if (!c->proxy_on || c->P.recursion_cap <= 0 || !c->d_rg)
      throw InvalidErr{"pxg_proxy_recip: the context has proxy sampling off"};
    const int R = 255;  // runs per (pass, entry): pxg_recip_stream packs the run index in 8 bits
    const int L = (n_runs + R - 1) / R;
    const size_t NR = static_cast<size_t>(std::max(c->P.pool_budget, 1)) * std::max(c->P.recip_repeats, 1) * c->batch;
    if (L > kBatchSetMax || static_cast<size_t>(L) * R > NR)
      throw InvalidErr{"pxg_proxy_recip: more runs than the context's reciprocal buffers hold"};
    CK(cudaDeviceSynchronize());  // the run buffers belong to Stage 1: nothing of it may be in flight
    cudaStream_t st = c->stream1;
    PV* dw = dupload(reinterpret_cast<const PV*>(walk), n_walk);
    IncHdr* dh = dalloc<IncHdr>(1);
    PV* dpre = dalloc<PV>(kMaxLight);
    int* dinfo = dalloc<int>(8);
    double* dpp = dalloc<double>(1);
    double* db = dupload(&bound, 1);
    PassState hps{};
    hps.n_ent = 1;
    PassState* dps = dupload(&hps, 1);
    k_probe_dropout<<<1, 32, 0, st>>>(c->M, dw, n_walk, dh, dpre, dinfo, dpp);
    int info0 = 0;
    CK(cudaMemcpyAsync(&info0, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!info0) {
      cudaFree(dw), cudaFree(dh), cudaFree(dpre), cudaFree(dinfo), cudaFree(dpp), cudaFree(db), cudaFree(dps);
      throw InvalidErr{"pxg_proxy_recip: dropout rejects the walk"};
    }
    BatchSet bs{};
    bs.n = L;
    for (int b = 0; b < L; ++b) bs.p[b] = BatchPass{dh, dpre, db, dps, 0x700000 + b};  // passes no render uses
    const int runs = L * R;
    const long long cap = c->P.recursion_cap;
    CK(cudaMemsetAsync(c->d_rnact, 0, 2 * sizeof(int), st));
    k_recip_init<<<blocks(runs, 128), 128, 0, st>>>(runs, R, R, bs, c->d_rstate, c->d_ract[0], c->d_rnact, c->d_run_est,
                                                   c->d_run_cost, c->d_run_trunc);
    recip_rounds(st, cap, c->d_rnact, [&](int cur, int chunk) { recip_round(c, st, bs, R, R, cap, cur, chunk); });
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(est, c->d_run_est, sizeof(double) * n_runs, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(cost, c->d_run_cost, sizeof(long long) * n_runs, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(truncated, c->d_run_trunc, sizeof(int) * n_runs, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(dw), cudaFree(dh), cudaFree(dpre), cudaFree(dinfo), cudaFree(dpp), cudaFree(db), cudaFree(dps);
    check_err(c, st);
  });
}

int pxg_trace_rays(pxg_ctx* c, int kernel, int any_hit, int n, const double* rays, const double* tmax, int* prim,
                   double* t) {
  return guarded(c, [&]() {
    if (n <= 0) return;
    if (!rays || !prim || (!any_hit && !t)) throw InvalidErr{"pxg_trace_rays: null argument"};
    if (kernel < 0 || kernel > 2) throw InvalidErr{"pxg_trace_rays: kernel must be 0, 1 or 2"};
    if (kernel == 0) {  // the single-ray paths (Scene::intersect / Scene::occluded)
      const int rc = any_hit ? pxg_occluded(c, n, rays, prim) : pxg_intersect(c, n, rays, tmax, prim, t);
      if (rc == PXG_E_INVALID) throw InvalidErr{c->err};
      if (rc != PXG_OK) throw CudaErr{c->err};
      return;
    }
    cudaStream_t st = c->stream;
    double* dr = dupload(rays, static_cast<size_t>(n) * 6);
    double* dt = (!any_hit && tmax) ? dupload(tmax, n) : nullptr;
    RayQueue q;
    q.ray = dalloc<double4>(2 * static_cast<size_t>(n));
    q.path = dalloc<int>(n);
    q.hit_prim = dalloc<int>(n);
    q.hit_t = dalloc<double>(n);
    q.count = dalloc<int>(1);
    q.cap = n;
    int* fetch = dalloc<int>(1);
    CK(cudaMemsetAsync(fetch, 0, sizeof(int), st));
    k_fill_trace_queue<<<blocks(n, 128), 128, 0, st>>>(n, dr, dt, any_hit, q);
    if (kernel == 1) {  // the production persistent kernels, the context's node layout
      if (any_hit)
        launch_trav<true>(c, q, fetch, st);
      else
        launch_trav<false>(c, q, fetch, st);
    } else if (any_hit) {
      k_wave_trace<true><<<blocks(n, 128), 128, 0, st>>>(c->S, q, dr, 1);
    } else {
      k_wave_trace<false><<<blocks(n, 128), 128, 0, st>>>(c->S, q, dr, 0);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(prim, q.hit_prim, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
    if (!any_hit) CK(cudaMemcpyAsync(t, q.hit_t, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (void* p : {static_cast<void*>(dr), static_cast<void*>(dt), static_cast<void*>(q.ray),
                    static_cast<void*>(q.path), static_cast<void*>(q.hit_prim), static_cast<void*>(q.hit_t),
                    static_cast<void*>(q.count), static_cast<void*>(fetch)})
      if (p) cudaFree(p);
    if (!any_hit)
      for (int i = 0; i < n; ++i)
        if (prim[i] < 0) t[i] = 0.0;  // pxg_intersect's convention for a miss
  });
}

int pxg_render_pt(pxg_ctx* c, int spp, uint64_t seed, int chunks, double* rgb) {
  return guarded(c, [&]() {
    if (!rgb) throw InvalidErr{"pxg_render_pt: null output"};
    if (chunks < 1) throw InvalidErr{"pxg_render_pt: chunks must be >= 1"};
    // render_image's `spp <= 0 -> scene.settings.spp` (transport.cpp:358) is resolved by the
    // caller: pxg_scene_desc carries no Settings::spp
    if (spp <= 0) throw InvalidErr{"pxg_render_pt: spp must be >= 1"};
    const int n = c->n;
    const size_t per = static_cast<size_t>(n) * 3;
    double* dparts = dalloc<double>(per * chunks);
    double* dout = dalloc<double>(per);
    const long long threads = static_cast<long long>(n) * chunks;
    k_render_pt<<<static_cast<unsigned>((threads + 127) / 128), 128, 0, c->stream>>>(c->S, c->max_depth, c->row0, n,
                                                                                       chunks, spp, seed, dparts);
    CK(cudaGetLastError());
    k_pt_reduce<<<blocks(static_cast<long long>(per), 256), 256, 0, c->stream>>>(n, chunks, dparts, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(rgb, dout, sizeof(double) * per, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(dparts);
    cudaFree(dout);
  });
}

int pxg_occluded(pxg_ctx* c, int n, const double* segs, int* occ) {
  return guarded(c, [&]() {
    if (n <= 0) return;
    double* ds = dupload(segs, static_cast<size_t>(n) * 6);
    int* dout = dalloc<int>(n);
    k_occluded<<<blocks(n, 128), 128, 0, c->stream>>>(c->S, n, ds, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(occ, dout, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(ds);
    cudaFree(dout);
  });
}

int pxg_recip_twopoint(int n, double bound, long long cap, uint64_t seed, double* est, long long* cost,
                       int* truncated) {
  return guarded(nullptr, [&]() {
    if (!(bound > 0.0)) throw RuntimeErr{"reciprocal: bound must be positive"};
    if (n <= 0) return;
    if (cap < 0 || cap > (1 << 20)) throw InvalidErr{"pxg_recip_twopoint: cap out of range"};
    const long long capa = std::max<long long>(cap, 1);
    cudaStream_t st = nullptr;
    std::vector<void*> tmp;
    auto A = [&](size_t bytes) {
      void* p = nullptr;
      CK(cudaMalloc(&p, std::max<size_t>(bytes, 1)));
      tmp.push_back(p);
      return p;
    };
    try {
      const size_t nc = static_cast<size_t>(n) * capa;
      auto* de = static_cast<double*>(A(sizeof(double) * n));
      auto* dc = static_cast<long long*>(A(sizeof(long long) * n));
      auto* dt = static_cast<int*>(A(sizeof(int) * n));
      auto* rs = static_cast<RunState*>(A(sizeof(RunState) * n));
      auto* g = static_cast<double*>(A(sizeof(double) * nc));
      auto* ns = static_cast<long long*>(A(sizeof(long long) * nc));
      auto* ne = static_cast<int*>(A(sizeof(int) * nc));
      auto* fr = static_cast<RecipFrame*>(A(sizeof(RecipFrame) * nc));
      int* act[2] = {static_cast<int*>(A(sizeof(int) * n)), static_cast<int*>(A(sizeof(int) * n))};
      auto* nact = static_cast<int*>(A(sizeof(int) * 2));
      auto* derr = static_cast<int*>(A(sizeof(int)));
      CK(cudaMemset(nact, 0, 2 * sizeof(int)));
      CK(cudaMemset(derr, 0, sizeof(int)));
      const BatchSet none{};  // n == 0: every run live, fixed bound
      k_recip_init<<<blocks(n, 128), 128>>>(n, 1, 1, none, rs, act[0], nact, de, dc, dt);
      recip_rounds(st, cap, nact, [&](int cur, int chunk) {
        k_twopoint_eval<<<4 * 148, 128>>>(seed, bound, cap, act[cur],
                                                                                     nact + cur, chunk, rs, g, ns, ne);
        // a small frame window so the spill / reload paths are exercised by the fixture
        k_recip_dfs_warp<4><<<8 * 148, 128>>>(1, 1, cap, none, bound, act[cur], nact + cur, chunk, rs, g,
                                                       ns, ne, fr, de, dc, dt, act[1 - cur], nact + (1 - cur), derr);
      });
      CK(cudaGetLastError());
      CK(cudaMemcpy(est, de, sizeof(double) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(cost, dc, sizeof(long long) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(truncated, dt, sizeof(int) * n, cudaMemcpyDeviceToHost));
    } catch (...) {
      for (void* p : tmp) cudaFree(p);
      throw;
    }
    for (void* p : tmp) cudaFree(p);
  });
}

int pxg_rng_draws(uint64_t seed, unsigned kind, unsigned sub, uint64_t stream, int n, unsigned* out) {
  return guarded(nullptr, [&]() {
    if (n <= 0) return;
    unsigned* d = dalloc<unsigned>(n);
    k_rng<<<1, 1>>>(seed, kind, sub, stream, n, d);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

int pxg_sincos_2pi(int device, int n, const uint32_t* k, double* s, double* c) {
  return guarded(nullptr, [&]() {
    if (n <= 0) return;
    if (!k || !s || !c) throw InvalidErr{"pxg_sincos_2pi: null argument"};
    CK(cudaSetDevice(device));
    ensure_sincos_table(device);
    uint32_t* dk = dupload(k, static_cast<size_t>(n));
    double* ds = dalloc<double>(2 * static_cast<size_t>(n));
    k_sincos_2pi<<<blocks(n, 256), 256>>>(n, dk, ds);
    CK(cudaGetLastError());
    std::vector<double> h(2 * static_cast<size_t>(n));
    CK(cudaMemcpy(h.data(), ds, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
      s[i] = h[2 * static_cast<size_t>(i)];
      c[i] = h[2 * static_cast<size_t>(i) + 1];
    }
    cudaFree(dk);
    cudaFree(ds);
  });
}

int pxg_read_timing(pxg_ctx* c, double* t, long long* counts) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  for (int k = 0; k < 8; ++k) t[k] = c->stage_ms[k];
  if (counts) {
    counts[0] = c->launches;
    counts[1] = 0;
  }
  return PXG_OK;
}

int pxg_read_recip_counts(pxg_ctx* c, long long* out) {
  return guarded(c, [&]() {
    if (!out) throw InvalidErr{"pxg_read_recip_counts: null output"};
    unsigned long long h[4] = {0, 0, 0, 0};
    if (c->d_node_stat) {
      CK(cudaStreamSynchronize(c->stream1));
      CK(cudaMemcpy(h, c->d_node_stat, sizeof(h), cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < 3; ++k) out[k] = static_cast<long long>(h[k]);
  });
}

}  // extern "C"
