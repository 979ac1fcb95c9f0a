// Host runtime of the B200-native ASADMM iteration loop: owns device state,
// drives the sm_100a kernels of kernels.cuh, and exports the C ABI declared
// in include/radmm_b200.h.
//
// Reference mapping (paths under /root/reference/proj/include/radmm):
//   radmm_run            <- run()                  admm.hpp:357-445
//   Sensor::* state      <- SensorCore             admm.hpp:88-192
//   fusion_kernel        <- FusionCore::round      admm.hpp:236-258
//   refactor()/GJ        <- LocalSolveCache        solver_core.hpp:30-58
//   screen_all()         <- SensorCore::screen     admm.hpp:134-159
//   NCCL exchange        <- run_inproc/run_tcp gather+broadcast (runtime.hpp:362-766)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>
#include <type_traits>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#ifndef RADMM_EXPERIMENTAL
#define RADMM_EXPERIMENTAL 0
#endif
#include "../../include/radmm_b200.h"
#include "kernels.cuh"

using namespace radmm_dev;

namespace {

thread_local std::string g_last_error;

struct Failure : std::exception {
  int code;
  std::string msg;
  Failure(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Failure(code, msg); }

void check_cuda(cudaError_t e, const char* what, int line) {
  if (e == cudaSuccess) return;
  const int code = (e == cudaErrorMemoryAllocation) ? RADMM_OUT_OF_MEMORY : RADMM_CUDA;
  fail(code, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " (radmm_b200.cu:" +
                 std::to_string(line) + ")");
}
#define CK(x) check_cuda((x), #x, __LINE__)

int env_int(const char* name, int dflt);

// ---------------------------------------------------------------------------
// Tuning switches (RADMM_* names: A/B knobs and build-only paths, defaults in
// DESIGN.md section 10).  Nothing reads the environment on a launch path:
// every ABI call refreshes one snapshot of the environment (tune_refresh,
// from guarded()), radmm_set_tuning() overrides it programmatically, and
// env_int() only looks the snapshot up.
// ---------------------------------------------------------------------------
struct TuneEntry {
  std::string name;
  bool env_set = false, api_set = false;
  int env_val = 0, api_val = 0;
};
std::mutex g_tune_mu;
std::vector<TuneEntry> g_tune;  // grows as switches are first consulted
std::atomic<unsigned> g_tune_gen{1};  // bumped by every refresh / override

TuneEntry& tune_entry(const char* name) {  // caller holds g_tune_mu
  for (TuneEntry& t : g_tune)
    if (t.name == name) return t;
  g_tune.push_back(TuneEntry{name});
  TuneEntry& t = g_tune.back();
  const char* e = std::getenv(name);
  t.env_set = e != nullptr;
  t.env_val = e ? std::atoi(e) : 0;
  return t;
}

void tune_refresh() {
  std::lock_guard<std::mutex> lk(g_tune_mu);
  bool changed = false;
  for (TuneEntry& t : g_tune) {
    const char* e = std::getenv(t.name.c_str());
    const bool set = e != nullptr;
    const int val = e ? std::atoi(e) : 0;
    changed = changed || set != t.env_set || val != t.env_val;
    t.env_set = set;
    t.env_val = val;
  }
  if (changed) g_tune_gen.fetch_add(1, std::memory_order_release);
}

template <class F>
int guarded(F&& f) {
  try {
    tune_refresh();
    f();
    return RADMM_OK;
  } catch (const Failure& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return RADMM_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RADMM_CUDA;
  }
}

// One non-blocking stream per device for allocation-time work (DArr).
cudaStream_t alloc_stream() {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!streams[dev]) {  // highest priority: its fills go ahead of queued CTAs of long kernels
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, hi));
  }
  return streams[dev];
}

template <typename T>
struct DArr {
  T* p = nullptr;
  size_t n = 0;
  bool own = true;  // false: a view of memory owned elsewhere (frame contexts share operators)
  DArr() = default;
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  DArr(DArr&& o) noexcept : p(o.p), n(o.n), own(o.own) { o.p = nullptr; o.n = 0; o.own = true; }
  DArr& operator=(DArr&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; own = o.own; o.p = nullptr; o.n = 0; o.own = true; }
    return *this;
  }
  void view(T* ptr, size_t count) {
    release();
    p = ptr;
    n = count;
    own = false;
  }
  ~DArr() { release(); }
  // Device memory comes from the device's stream-ordered pool (see
  // configure_pool): freed blocks stay reserved up to a retention threshold,
  // so the next context on this device allocates without driver calls.
  // Context streams are non-blocking, so frees wait for the device first.
  void release() {
    if (p && own) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, alloc_stream());
    }
    p = nullptr;
    n = 0;
    own = true;
  }
  void alloc(size_t count, bool zero = true) {
    release();
    if (count == 0) return;
    // allocation-side work on a private non-blocking stream: the legacy
    // default stream made these waits include the context stream's running
    // work (config 3: every upload waited for the previous sensor's Gram)
    cudaStream_t as = alloc_stream();
    CK(cudaMallocAsync(&p, count * sizeof(T), as));
    n = count;
    if (zero) CK(cudaMemsetAsync(p, 0, count * sizeof(T), as));
    CK(cudaStreamSynchronize(as));  // usable (and zeroed) from any stream from here on
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
};

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (only sharded contexts need it).
// ---------------------------------------------------------------------------
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm;
// ncclConfig_t as of NCCL 2.27 (versioned by size/version: newer libraries
// accept it); only `blocking` is set -- a non-blocking communicator, so the
// host can poll ncclCommGetAsyncError and enforce a timeout instead of
// hanging in a collective when a peer dies (runtime.hpp:540-545, 739-760).
struct nccl_config {
  size_t size;
  unsigned int magic;
  unsigned int version;
  int blocking, cgaClusterSize, minCTAs, maxCTAs;
  const char* netName;
  int splitShare, trafficClass;
  const char* commName;
  int collnetEnable, CTAPolicy, shrinkShare, nvlsCTAs;
};
constexpr int kNcclInProgress = 7;
struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(nccl_uid*) = nullptr;
  int (*CommInitRank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  int (*CommInitRankConfig)(nccl_comm*, int, nccl_uid, int, nccl_config*) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
  int (*CommDestroy)(nccl_comm) = nullptr;
  int (*CommAbort)(nccl_comm) = nullptr;
  int (*GetAsyncError)(nccl_comm, int*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  void load() {
    if (h) return;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) fail(RADMM_TRANSPORT, "cannot load libnccl.so.2");
    GetUniqueId = (int (*)(nccl_uid*))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (int (*)(nccl_comm*, int, nccl_uid, int))dlsym(h, "ncclCommInitRank");
    AllGather = (int (*)(const void*, void*, size_t, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllGather");
    CommDestroy = (int (*)(nccl_comm))dlsym(h, "ncclCommDestroy");
    CommInitRankConfig = (int (*)(nccl_comm*, int, nccl_uid, int, nccl_config*))dlsym(h, "ncclCommInitRankConfig");
    CommAbort = (int (*)(nccl_comm))dlsym(h, "ncclCommAbort");
    GetAsyncError = (int (*)(nccl_comm, int*))dlsym(h, "ncclCommGetAsyncError");
    GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllGather || !CommDestroy)
      fail(RADMM_TRANSPORT, "libnccl is missing required symbols");
  }
  void check(int r, const char* what) {
    if (r != 0 && r != kNcclInProgress)
      fail(RADMM_TRANSPORT, std::string("NCCL error in ") + what + ": " +
                                (GetErrorString ? GetErrorString(r) : std::to_string(r)));
  }
  // Wait until a non-blocking communicator leaves ncclInProgress (after init
  // or an enqueue); abort it and raise RADMM_TRANSPORT on an error or after
  // timeout_ms -- the reference's TransportError / receive timeout.
  void settle(nccl_comm comm, const char* what, int timeout_ms) {
    if (!GetAsyncError) return;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      int st = 0;
      const int r = GetAsyncError(comm, &st);
      if (r != 0) st = r;
      if (st == 0) return;
      if (st != kNcclInProgress) {
        if (CommAbort) CommAbort(comm);
        fail(RADMM_TRANSPORT, std::string("NCCL error in ") + what + ": " +
                                  (GetErrorString ? GetErrorString(st) : std::to_string(st)));
      }
      if (std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() > timeout_ms) {
        if (CommAbort) CommAbort(comm);
        fail(RADMM_TRANSPORT, std::string("NCCL timeout in ") + what + " after " + std::to_string(timeout_ms) +
                                  " ms (a peer is gone or stalled)");
      }
      std::this_thread::yield();
    }
  }
};
Nccl g_nccl;
constexpr int kNcclDouble = 8;  // ncclFloat64

// ---------------------------------------------------------------------------
// Device state
// ---------------------------------------------------------------------------
// forward CTA width: 256 threads (512-row tiles) up to kFwdTallRows, then
// RADMM_FWD_TALL_THREADS (1024 default: config 3 forward 21.6 -> 20.2 ms; 512)
int env_int(const char* name, int dflt);
int fwd_threads(int64_t ld) {
  if (ld <= kFwdTallRows) return 256;
  static const int tall = env_int("RADMM_FWD_TALL_THREADS", 1024) == 512 ? 512 : 1024;
  return tall;
}

struct Sensor {
  int rows = 0;
  int64_t ld = 0;  // roundup(rows, 64)
  bool has_op = false, has_y = false;
  DArr<float2> A;
  DArr<double2> y, y_eff;
  // active set + SensorCore state
  int n_act = 0;
  bool primal = false;
  bool stalled = false;
  DArr<int> J, Jnew, keep_pos, rem_pix, rem_pos, blk_cnt, blk_off, totals;
  DArr<unsigned char> keep;
  DArr<double2> x_full, x_hat, x_hat_new, data, data_new, rhs;
  DArr<double> ring;
  // cached inverse of the capacitance (dual) or Gram (primal) matrix
  DArr<double2> G, G2;
  // cached factor of the full active set (depends on A, mu, beta only, not on
  // y): reused by the next run on this resident problem (frames sharing A)
  DArr<double2> G0;
  bool g0_valid = false, g0_primal = false;
  double g0_mu = 0, g0_beta = 0;
  // G itself still holds the full-set factor of (base_mu, base_beta) (no
  // downdate, fold or rebuild since): the next run reuses it in place, and G0
  // is written only just before G is first modified (snapshot_base)
  bool g_is_base = false;
  double base_mu = 0, base_beta = 0;
  int64_t g0_ld = 0;
  int g0_n = 0;
  size_t g0_elems = 0;
  int64_t ldg = 0;
  int g_n = 0;
  // forward partials / KM-space vectors
  DArr<double2> part, v, w;
  int part_chunks = 0;  // capacity of part in chunks of ld
  int removed_now = 0;
  bool v_ready = false;  // v = A_J rhs for the coming iteration left by the fused sweep
  // Lagged data term (dual form): data holds mu A_J^H y_eff_s; the true data
  // term is data - mu A_J^H z with z = y_eff_s - y_eff (frozen echo since the
  // snapshot).  Then w = G (v_s + beta z) and x = (rhs_s - mu A_J^H w)/beta is
  // exactly the reference update, so an elimination event needs no data pass.
  DArr<double2> y_eff_s, bz;
  bool data_lag = false;
  // Hermitian G-apply partials (dot: nb x groups x 64, ax: nb(nb-1)/2 x 64)
  DArr<double2> hdot, hax;
  DArr<double2> apart;  // row-segmented adjoint partials (nseg x N)
  // Lazy Woodbury downdates (dual form, see lazy_dot_kernel): G stays the
  // factor of the base active set; the eliminated columns D accumulate in
  // P = G A_D (ld x kLazyMax) with Sinv = (I - mu A_D^H P)^{-1}, and are
  // folded into G only when kLazyMax is reached.
  // raw full-set Gram A A^H computed right after the operator upload (overlaps
  // the next sensor's upload); the run's first factorization scales it
  bool raw_gram = false;
  bool raw_packed = false;  // the raw Gram sits in Cp (packed factor) instead of G
  int lz_d = 0;    // |D|
  int lz_new = 0;  // 1-3: the last lz_new columns of P are formed by the next G-apply (extra right-hand sides)
  int lz_r = 0;    // columns added by the last event (bordered Sinv update pending)
  DArr<double2> lz_P, lz_R, lz_S, lz_t, lz_B;
  DArr<int> lz_pix;
  // KM-space refinement of the dual solve (refine(), kernels_batched.cuh):
  // the capacitance C of G's base set in packed lower tiles (Cp; Cp0 next to
  // the cached factor G0), residual rho and correction dw
  DArr<double2> Cp, Cp0, rho, dw;
  bool cp_valid = false, cp0_valid = false;
  // dual factor stored as packed lower tiles (herm_packed_tile) instead of a
  // full ld x rows matrix: half the HBM (config 3 fits with C next to it) and
  // tile-contiguous reads for the Hermitian apply; g0_packed: G0's layout
  bool gpacked = false, g0_packed = false;
  // complex64 copy of a packed G for the refinement's correction pass (half
  // its bytes); re-derived lazily whenever G changes (g32_valid)
  DArr<float2> G32;
  bool g32_valid = false;
};

constexpr int kFlagCap = 4 * kMaxBatch;  // pinned pivot-flag slots

struct Scratch {
  DArr<char> buf;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    const size_t bytes = round_up((int64_t)(count * sizeof(T)), 256);
    if (off + bytes > buf.n) fail(RADMM_OUT_OF_MEMORY, "scratch arena exhausted");
    T* p = reinterpret_cast<T*>(buf.p + off);
    off += bytes;
    return p;
  }
  void reserve(size_t bytes) {
    if (bytes > buf.n) {
      CK(cudaDeviceSynchronize());
      buf.alloc(bytes, false);
    }
    off = 0;
  }
};

}  // namespace

// Process-wide free list of mapped pinned host blocks (size classes of
// powers of two from 64 KB).  Never returned to the driver.
size_t pinned_class(size_t bytes) {
  size_t c = 64 << 10;
  while (c < bytes) c <<= 1;
  return c;
}
std::mutex g_pinned_mu;
std::vector<std::pair<size_t, char*>> g_pinned_free;
char* pinned_get(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    for (size_t i = 0; i < g_pinned_free.size(); ++i)
      if (g_pinned_free[i].first == bytes) {
        char* p = g_pinned_free[i].second;
        g_pinned_free.erase(g_pinned_free.begin() + i);
        return p;
      }
  }
  char* p = nullptr;
  CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  return p;
}
void pinned_put(char* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back({bytes, p});
}

struct radmm_ctx {
  int device = 0;
  int N = 0;
  int Q = 0;        // local sensors
  int Q_total = 0;
  int q_begin = 0;
  int rank = 0, world = 1;
  bool sharded = false;  // NCCL exchange active (world > 1, or forced at world 1 by RADMM_FORCE_NCCL)
  int q_max_local = 0;
  int sm_count = 148;
  int fwd_per_sm = 4;  // resident forward-kernel CTAs per SM (occupancy API), 256-thread variant
  int fwd_per_sm_tall = 2;  // the 512-thread variant (operators taller than kFwdTallRows)
  int sweep_clusters = 0;  // clusters of the last fused sweep (= partial chunks it left)
  cudaStream_t stream = nullptr;
  cudaStream_t up_stream = nullptr;  // operator uploads (overlap the previous sensor's Gram)
  cudaEvent_t up_event = nullptr;
  std::vector<cudaEvent_t> gram_evs;  // per sensor: its eager Gram (a re-upload waits for it)
  std::vector<Sensor> sensors;
  DArr<double2> s, xg, sigma, sigma_pre, gap;
  DArr<double> fpart;
  DArr<unsigned int> fcounter;
  DArr<FusionScalars> fs_dev;
  FusionScalars* fs_host = nullptr;
  FusionScalars* fs_host_dev = nullptr;
  DArr<const double2*> contrib;
  char* pinned_block = nullptr;  // mapped pinned block holding fs_host, h_totals, h_flags (pinned_get)
  size_t pinned_bytes = 0;
  int* h_totals = nullptr;   // mapped pinned, 3 slots x local sensors (kept counts; see enqueue_screen)
  int* d_totals = nullptr;   // device alias of h_totals
  int* h_flags = nullptr;    // pinned, kFlagCap (deferred pivot flags accumulate)
  Scratch scratch;
  DArr<int> fail_flags;
  // sharded exchange
  nccl_comm comm = nullptr;
  DArr<double2> send_buf, gathered;
  DArr<double> size_send, size_recv;
  int nccl_timeout_ms = 60000;     // transport timeout (radmm_set_transport_timeout)
  bool sync_meta = false;          // observer runs: per-iteration metadata all-gather (else once at run end)
  double* meta_host = nullptr;     // pinned, 2 slots of (2 q_max_local + 1) doubles (sync_meta)
  size_t meta_bytes = 0;
  std::vector<double> shard_meta;  // per completed iteration: local n_act, stalled flags, notice bytes
  // results of the last run
  std::vector<radmm_iteration_record> records;
  std::vector<int32_t> active_log;
  std::vector<int32_t> removal_log;
  radmm_run_summary summary{};
  bool have_result = false;
  int64_t launches = 0;
  int64_t rebuilds = 0, downdates = 0;
  int64_t factor_cache_hits = 0;
  int W = 5;
  int upd = 0;  // local updates performed in the current run
  // device timing: per-iteration CUDA events (always), per-phase events
  // (profiling mode) -- all on this context's stream.
  cudaEvent_t ev_it0 = nullptr, ev_it1 = nullptr;
  std::vector<double> iter_ms;       // per-step device wall time (incl. host round trip)
  std::vector<double> iter_busy_ms;  // per-step device time from first to last kernel
  std::vector<cudaEvent_t> ev_steps;
  std::vector<cudaEvent_t> ev_ends;  // recorded after each round's fusion
  DArr<int> go_flags;                // speculation guards, alternating per round
  DArr<unsigned> lazy_cnt;           // lazy_dot_kernel arrival counters (one per job)
  DArr<int> sgo_flags;               // "next round screens" flags, alternating per round
  bool pdl = false;                  // programmatic dependent launch: on inside the iteration loop (RADMM_PDL)
  bool refine = true;                // KM-space refinement of the dual solves (radmm_run_options.skip_refinement)
  double trace_us[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // RADMM_TRACE_HOST: host time of the event stages
  int trace_n = 0;
  int oz_eager = -1;                 // upload-time Grams on the Ozaki path (-1: not decided yet, see eager_gram)
  int64_t refine_skipped = 0;        // dual sensors whose packed C did not fit (solved unrefined)
  DArr<unsigned> screen_sync;        // screen_fused_kernel arrival ticket + changed flag (zero between launches)
  bool pre_screened[2] = {false, false};  // screening enqueued behind round k (slot k & 1)
  DArr<double2> split_ws;            // split-K partial tiles
  DArr<uint64_t> herm_items;         // Hermitian G-apply work items (largest first)
  std::vector<int64_t> herm_sig;     // (batch position, order) the items were built for
  int herm_n_items = 0;
  bool defer_fail_check = false;     // downdates: pivot check folded into the iteration sync
  int pending_fail = 0;              // deferred pivot flags waiting in h_flags
  // removal log kept on the device during a run (one D2H at the end)
  DArr<int> dlog;
  struct LogSeg { int k, q, count; int64_t off; };
  std::vector<LogSeg> log_segs;
  int64_t log_used = 0;
  std::vector<int64_t> iter_launches;
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  int ev_used = 0;  // events handed out since the last flush
  struct Mark { int cat; int ev0, ev1; double bytes; int64_t launches; };
  std::vector<Mark> marks;
  double prof_ms[RADMM_PHASE_COUNT] = {};
  double prof_bytes[RADMM_PHASE_COUNT] = {};
  int64_t prof_launches[RADMM_PHASE_COUNT] = {};
  int64_t prof_calls[RADMM_PHASE_COUNT] = {};
  // Multi-frame batches (BASELINE config 5): one child context per frame,
  // sharing this context's operators (views) and stream.
  std::vector<std::unique_ptr<radmm_ctx>> frames;
  radmm_ctx* parent = nullptr;
  bool own_stream = true;
  // frame-batched contractions: job tables + split-K partials (parent only)
  DArr<FrameBatchJob> fb_jobs;
  DArr<FrameReduceJob> fb_red;
  DArr<FrameRhsJob> fb_rhs;
  DArr<double2> fb_part;
  std::vector<DArr<double2>> gtmp;    // full rows x rows temporaries: Gram + Gauss-Jordan of packed factors
  std::vector<DArr<double2>> fb_g;    // full copies of packed factors for the frame-batched DMMA passes
  std::vector<DArr<double2>> fb_cap;  // full capacitances for the batched refinement pass
  bool fb_cap_ok = false;             // fb_cap holds this run's base C (reset per run_frames)
  bool fb_g_ok = false;               // fb_g holds this run's unpacked base factors
  double fb_g_mu = 0, fb_g_beta = 0;
  double fb_cap_mu = 0, fb_cap_beta = 0;
  DArr<GramJob> gram_jobs;
  // Ozaki-sliced Gram scratch (kernels_ozaki.cuh): row maxima, slices, pair blocks
  DArr<unsigned> oz_rowmax;
  DArr<int8_t> oz_P, oz_Q;
  DArr<int32_t> oz_R;
  // fused sweep v4 control (tile arrival counters / flags / norm partials)
  DArr<unsigned> s4_cnt, s4_flag, s4_done;
  DArr<double> s4_norms;
  unsigned s4_seq = 0;
  DArr<double2> xg_alt, sigma_alt;  // v5 writes the new x_G / sigma here, then they swap

  ~radmm_ctx() {
    const bool tr = env_int("RADMM_TRACE_DESTROY", 0) != 0;
    auto t = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (!tr) return;
      const auto n = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[radmm ~ctx] %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
      t = n;
    };
    if (device >= 0) cudaSetDevice(device);
    frames.clear();  // children use this context's stream and operators
    if (ev_it0) cudaEventDestroy(ev_it0);
    if (ev_it1) cudaEventDestroy(ev_it1);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_steps) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_ends) cudaEventDestroy(e);
    mark("events");
    if (comm && g_nccl.CommDestroy) g_nccl.CommDestroy(comm);
    if (meta_host) pinned_put(reinterpret_cast<char*>(meta_host), meta_bytes);
    pinned_put(pinned_block, pinned_bytes);  // fs_host / h_totals / h_flags live in it
    mark("host");
    if (stream && own_stream) cudaStreamDestroy(stream);
    if (up_stream) cudaStreamDestroy(up_stream);
    if (up_event) cudaEventDestroy(up_event);
    for (cudaEvent_t e : gram_evs)
      if (e) cudaEventDestroy(e);
    mark("streams");
    scratch.buf.release();
    mark("scratch");
    for (DArr<double2>* v : {&s, &xg, &sigma, &sigma_pre, &gap, &send_buf, &gathered, &split_ws, &fb_part, &xg_alt,
                             &sigma_alt})
      v->release();
    mark("vectors");
  }
};

namespace {

constexpr size_t kColdotSmemMax = 200 * 1024;
constexpr int kDefaultCpw = 2;
constexpr int kDowndateMatvecMax = 8;  // removed columns handled as Hermitian matvecs
constexpr size_t kColdotBigSmem = 96 * 1024;
constexpr int kMaxChunk = 2048;  // forward columns per CTA (shared-memory coefficient slab)

// ---- device-time accounting (CUDA events on the context stream) -------------
cudaEvent_t take_event(radmm_ctx* c, int& idx) {
  if (c->ev_used >= (int)c->ev_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->ev_pool.push_back(e);
  }
  idx = c->ev_used++;
  return c->ev_pool[idx];
}

struct PhaseScope {
  radmm_ctx* c;
  int cat;
  double bytes;
  int e0 = -1;
  int64_t l0 = 0;
  PhaseScope(radmm_ctx* ctx, int category, double algorithmic_bytes) : c(ctx), cat(category), bytes(algorithmic_bytes) {
    if (!c->profiling) return;
    CK(cudaEventRecord(take_event(c, e0), c->stream));
    l0 = c->launches;
  }
  ~PhaseScope() {
    if (!c->profiling || e0 < 0) return;
    int e1;
    if (c->ev_used >= (int)c->ev_pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return;
      c->ev_pool.push_back(e);
    }
    e1 = c->ev_used++;
    if (cudaEventRecord(c->ev_pool[e1], c->stream) != cudaSuccess) return;
    c->marks.push_back({cat, e0, e1, bytes, c->launches - l0});
  }
};

// Called after a stream synchronize: fold the recorded phases into the stats.
void flush_marks(radmm_ctx* c) {
  for (const auto& m : c->marks) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev_pool[m.ev0], c->ev_pool[m.ev1]));
    c->prof_ms[m.cat] += ms;
    c->prof_bytes[m.cat] += m.bytes;
    c->prof_launches[m.cat] += m.launches;
    c->prof_calls[m.cat] += 1;
  }
  c->marks.clear();
  c->ev_used = 0;
}

void set_device(radmm_ctx* c) { CK(cudaSetDevice(c->device)); }

// Keep up to RADMM_POOL_KEEP_GB (default 16) of freed device memory reserved
// in the device's default pool between contexts (0: release at every sync).
// Returning a context's memory to the driver is slow and erratic (config 3:
// 172 GB, measured 0.9-5.4 s inside radmm_ctx_destroy when the pool trimmed at
// every synchronisation of the teardown).  So the pool never trims by itself
// (release threshold = max): a destroyed context's blocks go back to the pool
// at once -- the next context reuses them without driver calls -- and the
// pool is trimmed down to RADMM_POOL_KEEP_GB by one background thread per
// teardown, off the caller's critical path.  The thread is joined before the
// next context is created (memory estimates must not race it), by
// radmm_pool_trim() and at process exit.  RADMM_POOL_ASYNC_TRIM=0 restores the
// synchronous behaviour (threshold = RADMM_POOL_KEEP_GB, trimming inside the
// teardown's synchronisations).
struct PoolReaper {
  std::mutex mu;
  std::thread th;
};
PoolReaper& pool_reaper() {
  static PoolReaper* r = new PoolReaper;  // never destroyed: joined by the atexit hook instead
  return *r;
}
void pool_reaper_join() {
  PoolReaper& r = pool_reaper();
  std::lock_guard<std::mutex> lk(r.mu);
  if (r.th.joinable()) r.th.join();
}
uint64_t pool_keep_bytes() { return (uint64_t)std::max(0, env_int("RADMM_POOL_KEEP_GB", 16)) << 30; }
bool pool_async_trim() { return env_int("RADMM_POOL_ASYNC_TRIM", 1) != 0; }

void configure_pool(int device) {
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = pool_async_trim() ? ~0ull : pool_keep_bytes();
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
}

void pool_trim_async(int device) {
  if (!pool_async_trim()) return;
  pool_reaper_join();
  static std::once_flag once;
  std::call_once(once, [] { std::atexit([] { pool_reaper_join(); }); });
  const size_t keep = (size_t)pool_keep_bytes();
  PoolReaper& r = pool_reaper();
  std::lock_guard<std::mutex> lk(r.mu);
  r.th = std::thread([device, keep] {
    cudaMemPool_t pool;
    if (cudaSetDevice(device) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess)
      cudaMemPoolTrimTo(pool, keep);
  });
}

// Bytes an allocation can still get: free device memory plus what the
// stream-ordered pool holds reserved but unused (freed blocks it keeps up to
// the release threshold -- invisible to cudaMemGetInfo).
size_t mem_available(int device) {
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
      free_b += (size_t)(reserved - used);
  }
  return free_b;
}

int occupancy(const void* func, int threads, size_t smem);
void set_smem_attr(const void* func, int bytes);

void init_ctx(radmm_ctx* c, int device, int n_pixels, int q_local) {
  pool_reaper_join();  // a previous context's memory is back with the driver (or kept by the pool)
  c->device = device;
  CK(cudaSetDevice(device));
  configure_pool(device);
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    fail(RADMM_CUDA, "radmm_b200 requires an sm_100 (Blackwell) GPU; found " + std::string(prop.name));
  }
  CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  c->fwd_per_sm = occupancy((const void*)fwd_kernel<MODE_RHS, 256>, 256, 16 * 1024);
  c->fwd_per_sm = std::max(1, c->fwd_per_sm);
  if (fwd_threads(1 << 30) == 1024)
    c->fwd_per_sm_tall = occupancy((const void*)fwd_kernel<MODE_RHS, 1024>, 1024, 16 * 1024);
  else
    c->fwd_per_sm_tall = occupancy((const void*)fwd_kernel<MODE_RHS, 512>, 512, 16 * 1024);
  c->fwd_per_sm_tall = std::max(1, c->fwd_per_sm_tall);
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->N = n_pixels;
  c->Q = q_local;
  c->sensors.resize(q_local);
  const int N = n_pixels;
  c->s.alloc(N); c->xg.alloc(N); c->sigma.alloc(N); c->sigma_pre.alloc(N); c->gap.alloc(N);
  const int fblocks = (N + kFusionThreads - 1) / kFusionThreads;
  c->fpart.alloc((size_t)fblocks * 5);
  c->fcounter.alloc(1);
  c->fs_dev.alloc(1);
  // one mapped pinned block for the host-visible scalars, from a process-wide
  // free list: cudaFreeHost can stall for hundreds of ms, so blocks are reused
  // across contexts instead of freed
  const size_t off_tot = round_up(2 * sizeof(FusionScalars), 256);
  const size_t off_flags = off_tot + round_up(sizeof(int) * 3 * std::max(1, q_local), 256);
  c->pinned_bytes = pinned_class(off_flags + sizeof(int) * kFlagCap);
  c->pinned_block = pinned_get(c->pinned_bytes);
  std::memset(c->pinned_block, 0, c->pinned_bytes);
  c->fs_host = reinterpret_cast<FusionScalars*>(c->pinned_block);
  std::memset(c->fs_host, 0, 2 * sizeof(FusionScalars));
  c->go_flags.alloc(2);
  c->sgo_flags.alloc(2);
  c->screen_sync.alloc(2);
  CK(cudaHostGetDevicePointer((void**)&c->fs_host_dev, c->fs_host, 0));
  c->h_totals = reinterpret_cast<int*>(c->pinned_block + off_tot);
  CK(cudaHostGetDevicePointer((void**)&c->d_totals, c->h_totals, 0));
  c->h_flags = reinterpret_cast<int*>(c->pinned_block + off_flags);
  c->fail_flags.alloc(kMaxBatch);
  for (int q = 0; q < q_local; ++q) {
    Sensor& S = c->sensors[q];
    S.J.alloc(N); S.Jnew.alloc(N); S.keep_pos.alloc(N); S.rem_pix.alloc(N); S.rem_pos.alloc(N);
    S.keep.alloc(N);
    const int nb = (N + kScanBlock - 1) / kScanBlock;
    S.blk_cnt.alloc(nb); S.blk_off.alloc(nb); S.totals.alloc(1);
    S.x_full.alloc(N); S.x_hat.alloc(N); S.x_hat_new.alloc(N); S.data.alloc(N); S.data_new.alloc(N);
    S.rhs.alloc(N);
  }
}

Sensor& sensor_at(radmm_ctx* c, int q) {
  if (!c) fail(RADMM_INVALID_ARGUMENT, "null context");
  if (q < 0 || q >= c->Q) fail(RADMM_INVALID_ARGUMENT, "sensor index out of range");
  return c->sensors[q];
}

void prepare_operator(radmm_ctx* c, Sensor& S, int rows) {
  if (rows < 1) fail(RADMM_INVALID_ARGUMENT, "ForwardOperator: rows must be >= 1");
  if (c->parent) fail(RADMM_INVALID_ARGUMENT, "frame contexts share their parent's operators");
  if (!c->frames.empty()) {  // frame contexts view the old operators
    CK(cudaStreamSynchronize(c->stream));
    c->frames.clear();
  }
  S.rows = rows;
  S.ld = round_up(rows, 64);
  if (S.A.n != (size_t)S.ld * c->N) S.A.alloc((size_t)S.ld * c->N, false);
  if (S.ld > rows)  // zero padding rows (ordered before the upload on the context stream)
    CK(cudaMemset2DAsync(S.A.p + rows, S.ld * sizeof(float2), 0, (S.ld - rows) * sizeof(float2), c->N,
                         c->stream));
  // no zero fill: a fill is a kernel, and behind an eager Gram that occupies
  // every SM it would wait for the Gram (begin_run writes y_eff; v, w, bz,
  // y_eff_s are written before they are read)
  if (S.y_eff.n != (size_t)S.ld) S.y_eff.alloc(S.ld, false);
  if (S.y_eff_s.n != (size_t)S.ld) S.y_eff_s.alloc(S.ld, false);
  if (S.bz.n != (size_t)S.ld) S.bz.alloc(S.ld, false);
  if (S.v.n != (size_t)S.ld) S.v.alloc(S.ld, false);
  if (S.w.n != (size_t)S.ld) S.w.alloc(S.ld, false);
  const int tile = 2 * fwd_threads(S.ld);
  const int tiles = (int)((S.ld + tile - 1) / tile);
  const int per_sm = fwd_threads(S.ld) > 256 ? c->fwd_per_sm_tall : c->fwd_per_sm;
  S.part_chunks = std::max(std::max(1, c->sm_count * per_sm / tiles), (c->N + kMaxChunk - 1) / kMaxChunk) + 1;
  S.part.alloc((size_t)S.part_chunks * S.ld, false);
  S.has_op = true;
  S.g0_valid = false;  // a new operator invalidates the cached factor
  S.g_is_base = false;
  S.raw_gram = false;
  S.raw_packed = false;
  S.cp_valid = S.cp0_valid = false;
  S.has_y = false;
}

// Kernel attribute / occupancy queries cost microseconds of host time each;
// the per-iteration launch path (and the host-bound elimination rounds) asks
// the same questions every time, so the answers are cached per process.
std::mutex g_attr_mu;
std::vector<std::pair<const void*, int>> g_smem_attr;
std::vector<std::pair<std::pair<const void*, int64_t>, int>> g_occ;

void set_smem_attr(const void* func, int bytes) {
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto& e : g_smem_attr)
      if (e.first == func) {
        if (e.second >= bytes) return;
        break;
      }
  }
  CK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  for (auto& e : g_smem_attr)
    if (e.first == func) {
      e.second = std::max(e.second, bytes);
      return;
    }
  g_smem_attr.push_back({func, bytes});
}

int occupancy(const void* func, int threads, size_t smem) {
  const int64_t key = (int64_t)threads << 32 | (int64_t)smem;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto& e : g_occ)
      if (e.first.first == func && e.first.second == key) return e.second;
  }
  int v = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, func, threads, smem));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  g_occ.push_back({{func, key}, v});
  return v;
}

#define LAUNCH_PLAIN(c, kern, grid, block, smem, ...)                        \
  do {                                                                        \
    kern<<<(grid), (block), (smem), (c)->stream>>>(__VA_ARGS__);              \
    CK(cudaGetLastError());                                                   \
    ++(c)->launches;                                                          \
  } while (0)

// Every kernel opens with pdl_enter() (griddepcontrol.wait, then
// launch_dependents; kernels_async.cuh), so inside the iteration loop
// (c->pdl, see do_run) context-stream launches use programmatic stream
// serialisation: a kernel's CTAs are scheduled while its predecessor drains,
// hiding the launch gaps between the forward, G-apply, reduce, adjoint,
// fusion, screening, lazy-correction and event kernels.  RADMM_PDL=0 turns it
// off; outside the loop the wait is a no-op.
#define LAUNCH(c, kern, grid, block, smem, ...)                                       \
  do {                                                                                \
    if ((c)->pdl) {                                                                   \
      cudaLaunchConfig_t cfg_{};                                                      \
      cfg_.gridDim = dim3(grid);                                                      \
      cfg_.blockDim = dim3(block);                                                    \
      cfg_.dynamicSmemBytes = (smem);                                                 \
      cfg_.stream = (c)->stream;                                                      \
      cudaLaunchAttribute at_[1];                                                     \
      at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                 \
      at_[0].val.programmaticStreamSerializationAllowed = 1;                          \
      cfg_.attrs = at_;                                                               \
      cfg_.numAttrs = 1;                                                              \
      CK(cudaLaunchKernelEx(&cfg_, kern, __VA_ARGS__));                               \
      ++(c)->launches;                                                                \
    } else {                                                                          \
      LAUNCH_PLAIN(c, kern, grid, block, smem, __VA_ARGS__);                          \
    }                                                                                 \
  } while (0)

// ---- column-dot launches --------------------------------------------------
// One full wave of resident CTAs split evenly over the batch (occupancy API);
// every warp then owns a balanced contiguous range of columns.
template <typename T, int EPI, bool SMEM, int CPW, int THREADS = 256>
void coldot_launch(radmm_ctx* c, const Pack<ColDotJob>& pk, size_t nb, int n_max, size_t smem, double mu,
                   double beta, const int* go) {
  auto kern = coldot_kernel<T, EPI, SMEM, CPW, THREADS>;
  if (SMEM && smem > 48 * 1024)
    set_smem_attr((const void*)kern, (int)(227 * 1024));
  int per_sm = 1;
  per_sm = occupancy((const void*)kern, THREADS, SMEM ? smem : 0);
  const int target = c->sm_count * std::max(1, per_sm);
  constexpr int kWarps = THREADS / 32;
  const int gx =
      std::max(1, std::min((n_max + kWarps * CPW - 1) / (kWarps * CPW), (int)((target + nb - 1) / nb)));
  LAUNCH(c, kern, dim3(gx, (unsigned)nb), THREADS, SMEM ? smem : 0, pk, mu, beta, go);
}

// CTAs per job for a batch of nb jobs on `slots` resident CTA slots: the
// smallest count whose total fills whole waves (< 3% idle in the last wave),
// so a large batch (the segmented config-3 adjoint: 64 jobs) has no
// nearly-empty tail wave.  At most gmax (the columns to go round).
int wave_grid(int slots, int nb, int gmax) {
  int best = std::max(1, std::min(gmax, (slots + nb - 1) / nb));
  for (int gx = 1; gx <= std::min(gmax, 64 * slots); ++gx) {
    const int64_t total = (int64_t)gx * nb, waves = (total + slots - 1) / slots;
    if (waves * slots - total <= (waves * slots) * 3 / 100 && total >= slots) return gx;
  }
  return best;
}

template <int EPI>
void coldot_pipe_launch(radmm_ctx* c, const Pack<ColDotJob>& pk, size_t nb, int n_max, size_t smem, double mu,
                        double beta, const int* go) {
  const int minb = env_int("RADMM_PIPE_MINB", 2);  // measured: 2 CTAs/SM (128 regs) streams best
  const int cpw = env_int("RADMM_PIPE_CPW", 4) == 2 ? 2 : 4;  // 4 columns per warp: adjoint 0.346 -> 0.343 ms
  auto kern = cpw == 4 ? coldot_pipe_kernel<EPI, 256, 2, 4>
              : minb >= 4 ? coldot_pipe_kernel<EPI, 256, 4> : minb == 2 ? coldot_pipe_kernel<EPI, 256, 2>
                                                                       : coldot_pipe_kernel<EPI, 256, 3>;
  if (smem > 48 * 1024) set_smem_attr((const void*)kern, (int)(227 * 1024));
  int per_sm = 1;
  per_sm = occupancy((const void*)kern, 256, smem);
  const int slots = c->sm_count * std::max(1, per_sm);
  const int gmax = std::max(1, (n_max + 8 * cpw - 1) / (8 * cpw));
  LAUNCH(c, kern, dim3(wave_grid(slots, (int)nb, gmax), (unsigned)nb), 256, smem, pk, mu, beta, go);
}

int coldot_cpw() {
  const int x = env_int("RADMM_CPW", 0);
  return (x == 1 || x == 2 || x == 4) ? x : 0;
}

template <typename T, int EPI>
void coldot(radmm_ctx* c, const std::vector<ColDotJob>& jobs, double mu, double beta, const int* go = nullptr) {
  if (jobs.empty()) return;
  for (size_t b0 = 0; b0 < jobs.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, jobs.size() - b0);
    Pack<ColDotJob> pk;
    int64_t ld_max = 0;
    int n_max = 0;
    for (size_t i = 0; i < nb; ++i) {
      pk.j[i] = jobs[b0 + i];
      ld_max = std::max(ld_max, pk.j[i].vld ? pk.j[i].vld : pk.j[i].ld);
      n_max = std::max(n_max, pk.j[i].n_out);
    }
    if (n_max == 0) continue;
    const size_t smem = (size_t)ld_max * sizeof(double2);
    if (smem > kColdotSmemMax) {
      coldot_launch<T, EPI, false, 1>(c, pk, nb, n_max, 0, mu, beta, go);
      continue;
    }
    const int cpw = coldot_cpw() ? coldot_cpw() : kDefaultCpw;
    if (smem > (size_t)env_int("RADMM_COLDOT_WIDE_BYTES", (int)kColdotBigSmem)) {  // one CTA per SM: go wide
      coldot_launch<T, EPI, true, 2, 1024>(c, pk, nb, n_max, smem, mu, beta, go);
      continue;
    }
    bool even = true;  // the pipelined kernel streams 64-row steps in fours
    for (size_t i = 0; i < nb; ++i) even = even && ((pk.j[i].len + 63) / 64) % 4 == 0;
    if (std::is_same<T, float2>::value && EPI != EPI_XPRIMAL && cpw == 2 && even && env_int("RADMM_COLDOT_PIPE", 1))
      coldot_pipe_launch<EPI>(c, pk, nb, n_max, smem, mu, beta, go);
    else if (cpw == 1) coldot_launch<T, EPI, true, 1>(c, pk, nb, n_max, smem, mu, beta, go);
    else if (cpw == 2) coldot_launch<T, EPI, true, 2>(c, pk, nb, n_max, smem, mu, beta, go);
    else coldot_launch<T, EPI, true, 4>(c, pk, nb, n_max, smem, mu, beta, go);
  }
}

// ---- Hermitian G-apply (dual form): w = G v from the lower block triangle ----
bool herm_enabled() { return env_int("RADMM_HERM", 1) != 0; }

// algorithmic bytes of one G-apply: the Hermitian triangle (or the full matrix)
double gapply_bytes(int n) {
  return herm_enabled() && n >= env_int("RADMM_HERM_MIN_ROWS", 512) ? 8.0 * n * (n + 1.0) : 16.0 * n * (double)n;
}

// Job table for the listed (dual) sensors: v = S.v -> w = S.w, plus the work
// item list, rebuilt only when the batch signature changes.
int herm_pack(radmm_ctx* c, const std::vector<int>& qs, Pack<HermJob>& pk) {
  std::vector<int64_t> sig;
  int nb_max = 0;
  for (size_t i = 0; i < qs.size(); ++i) {
    Sensor& S = c->sensors[qs[i]];
    HermJob h{};
    h.G = S.G.p; h.ld = S.gpacked ? kHermTile : S.ldg; h.packed = S.gpacked ? 1 : 0; h.n = S.rows;
    h.nb = (S.rows + kHermTile - 1) / kHermTile;
    h.groups = (h.nb + kHermStrip - 1) / kHermStrip;
    const size_t nd = (size_t)h.nb * h.groups * kHermTile,
                 na = std::max<size_t>((size_t)h.nb * (h.nb - 1) / 2 * kHermTile, 1);
    if (S.hdot.n < 4 * nd) S.hdot.alloc(4 * nd, false);  // up to four right-hand sides
    if (S.hax.n < 4 * na) S.hax.alloc(4 * na, false);
    h.v = S.v.p; h.w = S.w.p; h.dotp = S.hdot.p; h.axp = S.hax.p;
    h.dstride = (int64_t)nd; h.astride = (int64_t)na;
    pk.j[i] = h;
    nb_max = std::max(nb_max, h.nb);
    sig.push_back(h.n);
  }
  if (sig != c->herm_sig) {
    std::vector<uint64_t> items;
    for (int nt = kHermStrip; nt >= 1; --nt)  // largest strips first (tail balance)
      for (size_t i = 0; i < qs.size(); ++i) {
        const int nb = pk.j[i].nb;
        for (int J = 0; J < nb; ++J)
          for (int I0 = J; I0 < nb; I0 += kHermStrip)
            if (std::min(kHermStrip, nb - I0) == nt) items.push_back(herm_item((int)i, J, I0, nt));
      }
    if (c->herm_items.n < items.size()) {
      CK(cudaStreamSynchronize(c->stream));  // queued launches may still read the old table
      c->herm_items.alloc(items.size(), false);
    }
    // ordered in the context stream: launches already queued (a speculative
    // iteration) read the previous table before it is overwritten
    CK(cudaMemcpyAsync(c->herm_items.p, items.data(), items.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                       c->stream));
    c->herm_n_items = (int)items.size();
    c->herm_sig = sig;
  }
  return nb_max;
}

// nr = 2 when some job carries a second right-hand side (v1 -> w1).
void herm_launch(radmm_ctx* c, const Pack<HermJob>& pk, size_t nq, int nb_max, int nr, const int* go,
                 bool packed = false) {
  for (size_t i = 0; i < nq; ++i) packed = packed || pk.j[i].packed;  // only the persistent kernel reads tiles
#if RADMM_EXPERIMENTAL  // superseded variants (TMA ring, one CTA per item), measured slower
  if (nr == 1 && !packed && env_int("RADMM_HERM", 1) == 2) {
    set_smem_attr((const void*)herm_gapply_tma_kernel, (int)((int)kHermTmaSmem));
    const int grid = std::min(c->herm_n_items, c->sm_count);
    LAUNCH(c, herm_gapply_tma_kernel, dim3((unsigned)grid), 288, kHermTmaSmem, pk, c->herm_items.p,
           c->herm_n_items, go);
  } else if (nr == 1 && !packed && !env_int("RADMM_HERM_PERSIST", 1)) {
    LAUNCH(c, herm_gapply_kernel<1>, dim3((unsigned)c->herm_n_items), 256, 0, pk, c->herm_items.p, go);
  } else
#endif
  {
    nr = nr <= 1 ? 1 : nr == 2 ? 2 : 4;
    auto kern = nr == 1 ? herm_gapply_persist_kernel<1> : nr == 2 ? herm_gapply_persist_kernel<2>
                                                                   : herm_gapply_persist_kernel<4>;
    const size_t smem = herm_persist_smem(nr);
    set_smem_attr((const void*)kern, (int)((int)smem));
    int per_sm = 1;
    per_sm = occupancy((const void*)kern, 256, smem);
    const int grid = std::min(c->herm_n_items, c->sm_count * std::max(1, per_sm));
    LAUNCH(c, kern, dim3((unsigned)grid), 256, smem, pk, c->herm_items.p, c->herm_n_items, go);
  }
  LAUNCH(c, herm_reduce_kernel, dim3((unsigned)nb_max, (unsigned)nq, (unsigned)nr), kHermRedSlices * kHermTile, 0,
         pk, go);
}

// Below this order the triangle's few long strips (one CTA each) are
// latency-bound: the full-matrix column-dot apply spreads over more CTAs.
constexpr int kHermMinRows = 512;

void gapply(radmm_ctx* c, const std::vector<int>& qs, const int* go = nullptr) {
  if (qs.empty()) return;
  int rows_max = 0;
  for (int q : qs) rows_max = std::max(rows_max, c->sensors[q].rows);
  if (!herm_enabled() || qs.size() > (size_t)kMaxBatch || rows_max < env_int("RADMM_HERM_MIN_ROWS", kHermMinRows)) {
    std::vector<ColDotJob> gj;
    for (int q : qs) {
      Sensor& S = c->sensors[q];
      ColDotJob g{};
      g.M = S.G.p; g.ld = S.ldg; g.len = S.rows; g.n_out = S.rows; g.vec = S.v.p; g.out = S.w.p; g.scale = 1.0;
      gj.push_back(g);
      for (int u = 0; u < S.lz_new; ++u) {  // pending lazy-downdate columns P[:, d-new+u] = G a_u
        g.vec = S.lz_R.p + (size_t)u * S.ld; g.out = S.lz_P.p + (size_t)(S.lz_d - S.lz_new + u) * S.ld;
        gj.push_back(g);
      }
    }
    coldot<double2, EPI_STORE>(c, gj, 1.0, 1.0, go);
    return;
  }
  Pack<HermJob> pk;
  const int nb_max = herm_pack(c, qs, pk);
  int nr = 1;
  for (size_t i = 0; i < qs.size(); ++i) {
    Sensor& S = c->sensors[qs[i]];
    if (!S.lz_new) continue;
    // this event's removed columns ride the pass as extra right-hand sides
    HermJob& hj = pk.j[i];
    const double2* vs[3] = {nullptr, nullptr, nullptr};
    double2* ws[3] = {nullptr, nullptr, nullptr};
    for (int u = 0; u < S.lz_new && u < 3; ++u) {
      vs[u] = S.lz_R.p + (size_t)u * S.ld;
      ws[u] = S.lz_P.p + (size_t)(S.lz_d - S.lz_new + u) * S.ld;
    }
    hj.v1 = vs[0]; hj.w1 = ws[0]; hj.v2 = vs[1]; hj.w2 = ws[1]; hj.v3 = vs[2]; hj.w3 = ws[2];
    nr = std::max(nr, 1 + S.lz_new);
  }
  herm_launch(c, pk, qs.size(), nb_max, nr, go);
}

// ---- forward (axpy) launches ------------------------------------------------
template <int MODE>
void forward(radmm_ctx* c, const std::vector<FwdJob>& jobs, const std::vector<ReduceJob>& red, double beta,
             const int* go = nullptr) {
  for (size_t b0 = 0; b0 < jobs.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, jobs.size() - b0);
    Pack<FwdJob> pk;
    Pack<ReduceJob> rp;
    int max_chunks = 0, max_len = 0;
    int64_t ld_max = 0;
    for (size_t i = 0; i < nb; ++i) {
      pk.j[i] = jobs[b0 + i];
      rp.j[i] = red[b0 + i];
      max_chunks = std::max(max_chunks, pk.j[i].n_chunks);
      max_len = std::max(max_len, pk.j[i].chunk_len);
      ld_max = std::max(ld_max, pk.j[i].ld);
    }
    if (max_chunks > 0) {
      const size_t smem = (size_t)max_len * (sizeof(double2) + sizeof(int));
      const int threads = fwd_threads(ld_max);
      auto kern = threads == 1024 ? fwd_kernel<MODE, 1024> : threads == 512 ? fwd_kernel<MODE, 512> : fwd_kernel<MODE, 256>;
      if (smem > 48 * 1024) set_smem_attr((const void*)kern, (int)(227 * 1024));
      dim3 grid((unsigned)((ld_max + 2 * threads - 1) / (2 * threads)), max_chunks, (unsigned)nb);
      LAUNCH(c, kern, grid, threads, smem, pk, c->gap.p, c->sigma.p, beta, go);
    }
    dim3 rg((unsigned)((ld_max + 255) / 256), (unsigned)nb);
    LAUNCH(c, reduce_parts_kernel, rg, 256, 0, rp, go);
  }
}

// chunking so one forward launch is exactly one full wave of resident CTAs
void plan_chunks(radmm_ctx* c, const Sensor& S, int n, int batch, int& n_chunks, int& chunk_len) {
  const int tile = 2 * fwd_threads(S.ld);
  const int tiles = (int)((S.ld + tile - 1) / tile);
  const int target = c->sm_count * (fwd_threads(S.ld) > 256 ? c->fwd_per_sm_tall : c->fwd_per_sm);
  const int chunks = std::min(S.part_chunks, std::max(1, target / std::max(1, tiles * batch)));
  chunk_len = (int)std::min<int64_t>(kMaxChunk, round_up(std::max<int64_t>(32, (n + chunks - 1) / chunks), 8));
  n_chunks = (n + chunk_len - 1) / chunk_len;
}

// ---- GEMM launches -----------------------------------------------------------
template <int EPI>
void gemm(radmm_ctx* c, const std::vector<GemmJob>& jobs) {
  for (size_t b0 = 0; b0 < jobs.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, jobs.size() - b0);
    Pack<GemmJob> pk;
    int mm = 0, nn = 0;
    for (size_t i = 0; i < nb; ++i) {
      pk.j[i] = jobs[b0 + i];
      mm = std::max(mm, pk.j[i].m);
      nn = std::max(nn, pk.j[i].n);
    }
    if (mm == 0 || nn == 0) continue;
    const int tiles = ((nn + kGB - 1) / kGB) * ((mm + kGB - 1) / kGB);
    int kmax = 0, herm = 0;
    for (size_t i = 0; i < nb; ++i) {
      kmax = std::max(kmax, pk.j[i].k);
      herm |= pk.j[i].herm;
    }
    // skinny products (rank-r downdates): split K so the grid fills the GPU
    int nsplit = 1;
    // (>= 32 k-steps per split, aim for ~4 CTAs per SM)
    if (EPI == GEPI_PLAIN && !herm && tiles * (int)nb < 4 * c->sm_count && kmax >= 64 * kGK) {
      nsplit = std::min(kmax / (32 * kGK), (4 * c->sm_count + tiles * (int)nb - 1) / (tiles * (int)nb));
      nsplit = std::max(1, nsplit);
    }
    if (nsplit > 1) {
      const size_t need = (size_t)nsplit * nb * (size_t)mm * nn;
      if (c->split_ws.n < need) c->split_ws.alloc(need, false);
      dim3 grid((nn + kGB - 1) / kGB, (mm + kGB - 1) / kGB, (unsigned)(nb * nsplit));
      const int64_t stride = (int64_t)mm * nn;  // uniform per (job, split) slot
      LAUNCH(c, gemm_kernel<GEPI_SPLIT>, grid, 256, 0, pk, nsplit, c->split_ws.p, stride);
      dim3 rg((unsigned)(((int64_t)mm * nn + 255) / 256), (unsigned)nb);
      LAUNCH(c, gemm_split_reduce, rg, 256, 0, pk, nsplit, c->split_ws.p, stride);
      continue;
    }
    if (EPI != GEPI_SPLIT && mm >= 256 && nn >= 256 && env_int("RADMM_GEMM_BIG", 2) == 2) {
      set_smem_attr((const void*)gemm_dmma_kernel<EPI>, (int)((int)kGemmDmmaSmem));
      dim3 grid((nn + kDmBN - 1) / kDmBN, (mm + kDmBM - 1) / kDmBM, (unsigned)nb);
      LAUNCH(c, gemm_dmma_kernel<EPI>, grid, 256, kGemmDmmaSmem, pk);
      continue;
    }
    if (EPI != GEPI_SPLIT && mm >= 256 && nn >= 256 && env_int("RADMM_GEMM_BIG", 2)) {
      set_smem_attr((const void*)gemm_big_kernel<EPI>, (int)((int)kGemmBigSmem));
      dim3 grid((nn + kBigBN - 1) / kBigBN, (mm + kBigBM - 1) / kBigBM, (unsigned)nb);
      LAUNCH(c, gemm_big_kernel<EPI>, grid, 256, kGemmBigSmem, pk);
      continue;
    }
    dim3 grid((nn + kGB - 1) / kGB, (mm + kGB - 1) / kGB, (unsigned)nb);
    LAUNCH(c, gemm_kernel<EPI>, grid, 256, 0, pk, 1, (double2*)nullptr, (int64_t)0);
  }
}

MatRef mref(const void* p, int64_t ld, bool c64, bool trans = false, bool conj = false,
            const int* ridx = nullptr, const int* cidx = nullptr) {
  MatRef m;
  m.p = p; m.ld = ld; m.ridx = ridx; m.cidx = cidx;
  m.c64 = c64 ? 1 : 0; m.trans = trans ? 1 : 0; m.conj = conj ? 1 : 0;
  return m;
}

GemmJob gjob(int m, int n, int k, MatRef a, MatRef b, double2* cp, int64_t ldc, double alpha,
             double beta0, double diag_add = 0.0) {
  GemmJob g;
  g.m = m; g.n = n; g.k = k; g.a = a; g.b = b; g.c = cp; g.ldc = ldc;
  g.alpha = alpha; g.beta0 = beta0; g.diag_add = diag_add; g.k0 = 0; g.kb = 0; g.herm = 0;
  return g;
}

// ---- batched in-place Gauss-Jordan inverse of HPD matrices --------------------
struct InvTarget {
  double2* M;
  int64_t ld;
  int n;
};

constexpr int kGJB = 64;

void check_deferred(radmm_ctx* c);

// Inverts every target in place; raises RADMM_NUMERICAL if a pivot fails.
// herm = true: the Hermitian sweep (kernels_dense.cuh, gj_hpanel_kernel): the
// targets are HPD with a valid lower triangle (and diagonal 64-blocks); only
// lower tiles are updated -- half the work -- and the result is written
// exactly Hermitian (no projection pass needed).  Needs one more n x 64 panel
// of scratch per target.
void gj_invert(radmm_ctx* c, const std::vector<InvTarget>& targets, const char* what, bool herm = false) {
  if (targets.empty()) return;
  if (targets.size() > kMaxBatch) fail(RADMM_INVALID_ARGUMENT, "too many matrices in one batch");
  const size_t T = targets.size();
  // scratch: P (64x64), F (n x 64), R (64 x n) (+ T = F P, n x 64) per target
  size_t need = 0;
  for (const auto& t : targets)
    need += (64 * 64 + (herm ? 3 : 2) * (size_t)round_up(t.n, 64) * 64) * sizeof(double2) + 4 * 256;
  Scratch& sc = c->scratch;
  const size_t base_off = sc.off;
  if (sc.off + need > sc.buf.n) {
    // grow: preserve nothing (callers take scratch before gj only for inputs they own)
    fail(RADMM_OUT_OF_MEMORY, "scratch arena too small for Gauss-Jordan inverse");
  }
  std::vector<double2*> P(T), F(T), R(T), TP(T);
  std::vector<int64_t> ldf(T);
  int n_max = 0;
  for (size_t i = 0; i < T; ++i) {
    const int64_t nn = round_up(targets[i].n, 64);
    P[i] = sc.take<double2>(64 * 64);
    F[i] = sc.take<double2>((size_t)nn * 64);
    R[i] = sc.take<double2>((size_t)nn * 64);
    TP[i] = herm ? sc.take<double2>((size_t)nn * 64) : nullptr;
    ldf[i] = nn;
    n_max = std::max(n_max, targets[i].n);
  }
  if (herm && n_max <= kGJB) herm = false;  // single pivot block: the in-shared-memory inverse below
  CK(cudaMemsetAsync(c->fail_flags.p, 0, sizeof(int) * kMaxBatch, c->stream));
  set_smem_attr((const void*)gj_diag_kernel, (int)(kGjSmem));
  if (n_max <= kGJB) {
    // every matrix is a single pivot block (the r x r downdate systems):
    // one in-shared-memory Gauss-Jordan, written back in place
    Pack<DiagJob> dj;
    for (size_t i = 0; i < T; ++i) {
      DiagJob d{};
      d.M = targets[i].M; d.ld = targets[i].ld; d.n = targets[i].n; d.k0 = 0; d.kb = targets[i].n;
      d.P = targets[i].M; d.ldp = targets[i].ld;
      d.fail = c->fail_flags.p + i;
      dj.j[i] = d;
    }
    LAUNCH(c, gj_diag_kernel, dim3((unsigned)T), 1024, kGjSmem, dj);
    n_max = 0;  // skip the blocked sweep below
  }
  for (int k0 = 0; k0 < n_max; k0 += kGJB) {
    Pack<DiagJob> dj;
    std::vector<GemmJob> rjobs, ujobs;
    int live = 0;
    int64_t panel_max = 0;
    for (size_t i = 0; i < T; ++i) {
      DiagJob d;
      d.M = targets[i].M; d.ld = targets[i].ld; d.n = targets[i].n; d.k0 = k0;
      d.kb = std::max(0, std::min(kGJB, targets[i].n - k0));
      d.P = P[i]; d.ldp = 64; d.F = F[i]; d.ldf = ldf[i]; d.R = R[i]; d.ldr = 64;
      d.fail = c->fail_flags.p + i;
      d.herm = herm ? 1 : 0;
      dj.j[i] = d;
      if (d.kb <= 0) continue;
      ++live;
      panel_max = std::max<int64_t>(panel_max, (int64_t)d.n * d.kb);
      // R' = P * M[K, :]
      rjobs.push_back(gjob(d.kb, d.n, d.kb, mref(P[i], 64, false),
                           mref(targets[i].M + k0, targets[i].ld, false), R[i], 64, 1.0, 0.0));
      GemmJob u = gjob(d.n, d.n, d.kb, mref(F[i], ldf[i], false), mref(R[i], 64, false),
                       targets[i].M, targets[i].ld, 1.0, 0.0);
      u.k0 = k0;
      u.kb = d.kb;
      ujobs.push_back(u);
    }
    if (!live) break;
    set_smem_attr((const void*)gj_diag_kernel, (int)(kGjSmem));
    LAUNCH(c, gj_diag_kernel, dim3((unsigned)T), 1024, kGjSmem, dj);
    const int pblocks = (int)std::min<int64_t>(1024, (panel_max + 255) / 256);
    if (herm) {
      // F = M[:, K] (from the lower triangle), R = F^H; T = F P; M -= T R on
      // the lower tiles; then the pivot rows / columns and -P
      LAUNCH(c, gj_hpanel_kernel, dim3(pblocks, (unsigned)T), 256, 0, dj);
      std::vector<GemmJob> tjobs;
      Pack<DiagJob> fx = dj;
      Pack<GjUpdJob> up;
      int nu = 0, nmax = 0;
      for (size_t i = 0; i < T; ++i) {
        const DiagJob& d = dj.j[i];
        fx.j[i].F = TP[i];
        if (d.kb <= 0) continue;
        tjobs.push_back(gjob(d.n, d.kb, d.kb, mref(F[i], ldf[i], false), mref(P[i], 64, false), TP[i], ldf[i], 1.0,
                             0.0));
        up.j[nu++] = GjUpdJob{targets[i].M, targets[i].ld, d.n, TP[i], ldf[i], R[i], k0, d.kb};
        nmax = std::max(nmax, d.n);
      }
      gemm<GEPI_PLAIN>(c, tjobs);
      set_smem_attr((const void*)gj_update_kernel<true>, (int)((int)kGjuSmem));
      LAUNCH(c, gj_update_kernel<true>,
             dim3((unsigned)((nmax + kGjuBN - 1) / kGjuBN), (unsigned)((nmax + kGjuBM - 1) / kGjuBM), (unsigned)nu), 256,
             kGjuSmem, up);
      LAUNCH(c, gj_hfix_kernel, dim3(pblocks, (unsigned)T), 256, 0, fx);
      continue;
    }
    LAUNCH(c, gj_panel_kernel, dim3(pblocks, (unsigned)T), 256, 0, dj);
    gemm<GEPI_PLAIN>(c, rjobs);
    LAUNCH(c, gj_fix_kernel, dim3((unsigned)T), 256, 0, dj);
    if (env_int("RADMM_GJ_UPDATE", 1) && ujobs.size() <= (size_t)kMaxBatch) {
      // rank-kb update with both operands resident in shared memory
      Pack<GjUpdJob> up;
      int nmax = 0;
      for (size_t u = 0; u < ujobs.size(); ++u) {
        const GemmJob& g = ujobs[u];
        up.j[u] = GjUpdJob{g.c, g.ldc, g.m, reinterpret_cast<const double2*>(g.a.p), g.a.ld,
                           reinterpret_cast<const double2*>(g.b.p), g.k0, g.kb};
        nmax = std::max(nmax, g.m);
      }
      set_smem_attr((const void*)gj_update_kernel<false>, (int)((int)kGjuSmem));
      LAUNCH(c, gj_update_kernel<false>, dim3((unsigned)((nmax + kGjuBN - 1) / kGjuBN), (unsigned)((nmax + kGjuBM - 1) / kGjuBM),
                                       (unsigned)ujobs.size()), 256, kGjuSmem, up);
    } else {
      gemm<GEPI_GJ>(c, ujobs);
    }
  }
  if (herm)  // M = -inv: negate the lower triangle and mirror it
    for (size_t i = 0; i < T; ++i) {
      const int nt = (targets[i].n + 31) / 32;
      LAUNCH(c, gj_hfinish_kernel, dim3((unsigned)((int64_t)nt * (nt + 1) / 2)), 256, 0, targets[i].M, targets[i].ld,
             targets[i].n);
    }
  // flags land after any still-unchecked deferred ones
  if (c->pending_fail + T > (size_t)kFlagCap) {
    CK(cudaStreamSynchronize(c->stream));
    check_deferred(c);
  }
  const int off = c->pending_fail;
  CK(cudaMemcpyAsync(c->h_flags + off, c->fail_flags.p, sizeof(int) * T, cudaMemcpyDeviceToHost, c->stream));
  sc.off = base_off;
  if (c->defer_fail_check) {  // checked after the iteration's own sync (check_deferred)
    c->pending_fail = off + (int)T;
    return;
  }
  CK(cudaStreamSynchronize(c->stream));
  for (size_t i = 0; i < T; ++i)
    if (c->h_flags[off + i]) fail(RADMM_NUMERICAL, std::string(what) + ": Cholesky failed");
}

// Deferred pivot check of the last downdate (the stream has been synchronised).
void check_deferred(radmm_ctx* c) {
  const int t = c->pending_fail;
  c->pending_fail = 0;
  for (int i = 0; i < t; ++i)
    if (c->h_flags[i]) fail(RADMM_NUMERICAL, "factorize: Cholesky failed");
}

// ---------------------------------------------------------------------------
// Factorization: LocalSolveCache (solver_core.hpp:34-45) realised as the
// explicit inverse of the smaller of the two equivalent systems.
// ---------------------------------------------------------------------------
void ensure_g(Sensor& S, int dim, int64_t ld) {
  const size_t need = (size_t)ld * dim;
  if (S.G.n < need) S.G.alloc(need);
}

// Hermitian projection of the dual factors (see herm_symmetrize_kernel): the
// lower-triangle G-apply then uses exactly the matrix the full apply would.
void symmetrize(radmm_ctx* c, const std::vector<int>& qs) {
  if (env_int("RADMM_SYMM", 1) == 0) return;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    if (S.primal || S.gpacked || S.g_n <= 0) continue;  // packed: the lower tiles define G
    const int nt = (S.g_n + 31) / 32;
    LAUNCH(c, herm_symmetrize_kernel, dim3((unsigned)((int64_t)nt * (nt + 1) / 2)), 256, 0, S.G.p, S.ldg, S.g_n);
  }
}

// ---- Ozaki-sliced Gram on the int8 tensor cores (tcgen05, kernels_ozaki.cuh) ----
bool ozaki_enabled() { return env_int("RADMM_OZAKI", 1) != 0; }

// The slices are large for tall operators (config 3: 18.5 GB per sensor); only
// small scratch (<= 2 GB, config 2: 1.2 GB) is kept between Grams.
void release_ozaki_scratch(radmm_ctx* c) {
  const size_t bytes = c->oz_P.n + c->oz_Q.n + c->oz_R.n * 4;
  if (bytes == 0) return;
  // small scratch is kept for the next Gram -- unless the device is nearly
  // full (config 3 on one GPU), where every GB goes back before the run
  if (bytes <= (2ull << 30) && mem_available(c->device) > (12ull << 30)) return;
  c->oz_P.release();
  c->oz_Q.release();
  c->oz_R.release();
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D int8 map over rows x kdim bytes, 128 x 128-byte boxes, SWIZZLE_128B
bool slice_tensor_map(CUtensorMap* map, const int8_t* base, int64_t rows, int64_t kdim) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kdim};
  const cuuint32_t box[2] = {(cuuint32_t)radmm_oz::kOzBK, (cuuint32_t)radmm_oz::kOzBM};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Scratch of one Ozaki Gram (slices, pair blocks, row maxima) in bytes.
double ozaki_scratch_bytes(int rows, int n) {
  using namespace radmm_oz;
  const int T = (rows + kOzBM - 1) / kOzBM, tiles = T * (T + 1) / 2;
  const double rows_pad = (double)T * kOzBM, kdim = 2.0 * round_up(n, 64);
  return 2.0 * kOzSlices * rows_pad * kdim + 4.0 * tiles * kOzPairs * 2 * kOzBM * kOzBN + 4.0 * rows_pad;
}

// Scratch of the chunked Gram: the P slices of one pixel chunk + row maxima.
double ozaki_chunk_scratch_bytes(int rows, int n) {
  using namespace radmm_oz;
  const double rows_pad = (double)round_up(rows, kOzBM);
  const double half = (double)std::min<int64_t>(kOzChunk, round_up(n, kOzBK));
  return kOzSlices * rows_pad * 2.0 * half + 4.0 * rows_pad;
}

// RADMM_OZ_CHUNK: 0 = one-pass Gram only, 1 (default) = chunked Gram when the
// one-pass scratch does not fit, 2 = always chunked (tests).
int ozaki_chunk_mode() { return env_int("RADMM_OZ_CHUNK", 1); }

// The chunked Gram (kernels_ozaki.cuh, oz_gram_chunk_kernel): C must be zeroed
// by the caller (it holds the fp64 accumulators between chunks).
bool ozaki_gram_chunked(radmm_ctx* c, Sensor& S, const int* J, int n, double2* C, int64_t ldc, double mu, double beta) {
  using namespace radmm_oz;
  const int rows = S.rows;
  const int T = (rows + kOzBM - 1) / kOzBM, tiles = T * (T + 1) / 2;
  const int64_t rows_pad = (int64_t)T * kOzBM;
  const int half = (int)std::min<int64_t>(kOzChunk, round_up(n, kOzBK));  // slice columns per part
  const size_t pbytes = (size_t)kOzSlices * rows_pad * 2 * half;
  if (c->oz_P.n < pbytes || c->oz_rowmax.n < (size_t)rows_pad) {
    const size_t free_b = mem_available(c->device);
    const size_t held = c->oz_P.n + c->oz_Q.n + c->oz_R.n * 4;
    if (free_b + held < pbytes + rows_pad * 4 + (3ull << 30)) return false;
    if (c->oz_P.n < pbytes) {
      c->oz_Q.release();
      c->oz_R.release();
      c->oz_P.alloc(pbytes, false);
    }
    if (c->oz_rowmax.n < (size_t)rows_pad) c->oz_rowmax.alloc(rows_pad, false);
  }
  CUtensorMap tP;
  if (!slice_tensor_map(&tP, c->oz_P.p, (int64_t)kOzSlices * rows_pad, 2 * (int64_t)half)) return false;
  CK(cudaMemsetAsync(c->oz_rowmax.p, 0, sizeof(unsigned) * rows_pad, c->stream));
  CK(cudaMemsetAsync(c->oz_P.p, 0, pbytes, c->stream));  // padding rows / columns are zero slices
  const int split = std::max(1, std::min(64, n / 256));
  LAUNCH(c, oz_rowmax_kernel, dim3((unsigned)((rows + 255) / 256), (unsigned)split), 256, 0, S.A.p, S.ld, rows, J, n,
         c->oz_rowmax.p);
  set_smem_attr((const void*)oz_gram_chunk_kernel, (int)((int)kOzCSmem));
  const int64_t slice = rows_pad * 2 * half;
  for (int c0 = 0; c0 < n; c0 += half) {
    const int cn = std::min(half, n - c0);
    if (cn < half && c0 > 0)  // a short last chunk: the columns past it must read as zero
      CK(cudaMemsetAsync(c->oz_P.p, 0, pbytes, c->stream));
    LAUNCH(c, oz_slice_kernel, dim3((unsigned)((cn + 31) / 32), (unsigned)((rows + 63) / 64)), 256, 0, S.A.p, S.ld,
           rows, J, cn, half, c->oz_rowmax.p, c->oz_P.p, (int8_t*)nullptr, slice, c0);
    LAUNCH(c, oz_gram_chunk_kernel, dim3((unsigned)tiles), kOzCThreads, kOzCSmem, tP, (int)rows_pad, half, rows, C,
           ldc);
  }
  LAUNCH(c, oz_gram_finish_kernel, dim3((unsigned)((rows + 255) / 256), (unsigned)rows), 256, 0, c->oz_rowmax.p, rows,
         C, ldc, mu, beta);
  return true;
}

// C = beta I + mu A_J A_J^H (rows x rows, lower tiles + exact mirror) for one
// sensor; returns false (caller falls back to the fp64 DMMA Gram) when the
// slices do not fit next to the resident problem or the shape is out of range.
// C arrives zeroed.
bool ozaki_gram(radmm_ctx* c, Sensor& S, const int* J, int n, double2* C, int64_t ldc, double mu, double beta) {
  using namespace radmm_oz;
  if (!ozaki_enabled() || n < 1 || n > 65536) return false;
  const int chunk_mode = ozaki_chunk_mode();
  if (chunk_mode == 2) return ozaki_gram_chunked(c, S, J, n, C, ldc, mu, beta);
  const int rows = S.rows;
  const int T = (rows + kOzBM - 1) / kOzBM, tiles = T * (T + 1) / 2;
  const int64_t rows_pad = (int64_t)T * kOzBM, npad = round_up(n, 64), kdim = 2 * npad;
  const size_t slice = (size_t)rows_pad * kdim, pq = (size_t)kOzSlices * slice;
  const size_t rblk = (size_t)tiles * kOzPairs * 2 * kOzBM * kOzBN;
  const size_t need = 2 * pq + rblk * 4 + rows_pad * 4;
  if (c->oz_P.n < pq || c->oz_Q.n < pq || c->oz_R.n < rblk || c->oz_rowmax.n < (size_t)rows_pad) {
    const size_t free_b = mem_available(c->device);
    const size_t held = c->oz_P.n + c->oz_Q.n + c->oz_R.n * 4;
    if (free_b + held < need + (4ull << 30))
      return chunk_mode == 1 && ozaki_gram_chunked(c, S, J, n, C, ldc, mu, beta);
    if (c->oz_P.n < pq) c->oz_P.alloc(pq, false);
    if (c->oz_Q.n < pq) c->oz_Q.alloc(pq, false);
    if (c->oz_R.n < rblk) c->oz_R.alloc(rblk, false);
    if (c->oz_rowmax.n < (size_t)rows_pad) c->oz_rowmax.alloc(rows_pad, false);
  }
  CK(cudaMemsetAsync(c->oz_rowmax.p, 0, sizeof(unsigned) * rows_pad, c->stream));
  CK(cudaMemsetAsync(c->oz_P.p, 0, pq, c->stream));  // padding rows / columns are zero slices
  CK(cudaMemsetAsync(c->oz_Q.p, 0, pq, c->stream));
  const int split = std::max(1, std::min(64, n / 256));
  LAUNCH(c, oz_rowmax_kernel, dim3((unsigned)((rows + 255) / 256), (unsigned)split), 256, 0, S.A.p, S.ld, rows, J, n,
         c->oz_rowmax.p);
  LAUNCH(c, oz_slice_kernel, dim3((unsigned)((n + 31) / 32), (unsigned)((rows + 63) / 64)), 256, 0, S.A.p, S.ld, rows,
         J, n, (int)npad, c->oz_rowmax.p, c->oz_P.p, c->oz_Q.p, (int64_t)slice, 0);
  CUtensorMap tP, tQ;
  if (env_int("RADMM_OZ_TMA", 1) && slice_tensor_map(&tP, c->oz_P.p, (int64_t)kOzSlices * rows_pad, kdim) &&
      slice_tensor_map(&tQ, c->oz_Q.p, (int64_t)kOzSlices * rows_pad, kdim)) {
    set_smem_attr((const void*)oz_gram_pairs_tma_kernel, (int)((int)kOzTSmem));
    LAUNCH(c, oz_gram_pairs_tma_kernel, dim3((unsigned)tiles, (unsigned)kOzPairs), 128, kOzTSmem, tP, tQ,
           (int)rows_pad, (int)kdim, c->oz_R.p);
  } else {
    set_smem_attr((const void*)oz_gram_pairs_kernel, (int)((int)kOzSmem));
    LAUNCH(c, oz_gram_pairs_kernel, dim3((unsigned)tiles, (unsigned)kOzPairs), 128, kOzSmem, c->oz_P.p, c->oz_Q.p,
           (int64_t)slice, rows, (int)kdim, c->oz_R.p);
  }
  LAUNCH(c, oz_combine_kernel, dim3((unsigned)(kOzBM * kOzBN / 256), (unsigned)tiles), 256, 0, c->oz_R.p,
         c->oz_rowmax.p, rows, C, ldc, mu, beta);
  return true;
}

// ---- KM-space refinement of the dual solve (see kernels_batched.cuh) --------
size_t cap_tiles(int n) {
  const size_t nb = (size_t)(n + kHermTile - 1) / kHermTile;
  return nb * (nb + 1) / 2;
}

// Keep C = beta I + mu A_J A_J^H of a dual sensor (in S.G, lower tiles valid,
// right before the in-place inversion) as packed lower tiles.  Skipped --
// and the sensor solved unrefined, counted in refine_skipped -- only when the
// tiles would not fit next to 1 GB of free HBM.
void cap_keep(radmm_ctx* c, Sensor& S, const double2* C, int64_t ldc) {
  S.cp_valid = false;
  if (S.primal) return;
  const size_t need = cap_tiles(S.rows) * kHermTile * kHermTile;
  if (S.Cp.n < need) {
    const size_t free_b = mem_available(c->device);
    if (free_b < need * sizeof(double2) + (1ull << 30)) {
      ++c->refine_skipped;
      return;
    }
    S.Cp.alloc(need, false);
  }
  LAUNCH(c, cap_pack_kernel, dim3((unsigned)cap_tiles(S.rows)), 256, 0, C, ldc, S.rows, S.Cp.p);
  S.cp_valid = true;
}

// Elements of G's storage (packed lower tiles or a full ldg x g_n matrix).
size_t g_elems(const Sensor& S) {
  return S.gpacked ? cap_tiles(S.rows) * kHermTile * kHermTile : (size_t)S.ldg * S.g_n;
}

// A dual factor of this sensor is stored packed (callers check dual-ness).
bool use_gpacked(const radmm_ctx* c, const Sensor& S) {
  return herm_enabled() && S.rows >= env_int("RADMM_HERM_MIN_ROWS", kHermMinRows) && c->Q <= kMaxBatch &&
         env_int("RADMM_GPACK", 1) != 0;
}

// Full rows x rows temporaries for `count` packed factorizations at once.
void gtmp_reserve(radmm_ctx* c, int count, size_t elems) {
  if ((int)c->gtmp.size() < count) c->gtmp.resize(count);
  for (int i = 0; i < count; ++i)
    if (c->gtmp[i].n < elems) c->gtmp[i].alloc(elems, false);
}

void gtmp_release(radmm_ctx* c) {
  size_t held = 0;
  for (auto& t : c->gtmp) held += t.n * sizeof(double2);
  if (held <= (2ull << 30)) return;
  c->gtmp.clear();
}

// C <- C - mu A_R A_R^H for the packed capacitances (fold / eager downdate):
// pix lists the removed columns of each job.
void cap_update(radmm_ctx* c, const std::vector<CapJob>& jobs, double mu) {
  for (size_t b0 = 0; b0 < jobs.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, jobs.size() - b0);
    Pack<CapJob> pk;
    size_t tiles = 0;
    for (size_t i = 0; i < nb; ++i) {
      pk.j[i] = jobs[b0 + i];
      tiles = std::max(tiles, cap_tiles(pk.j[i].n));
    }
    LAUNCH(c, cap_update_kernel, dim3((unsigned)tiles, (unsigned)nb), 256, 0, pk, mu);
  }
}

// G <- G + alpha X Y^H on packed factors (lazy fold / eager downdate).
void packed_update(radmm_ctx* c, const std::vector<PackedUpdJob>& jobs, double alpha) {
  for (size_t b0 = 0; b0 < jobs.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, jobs.size() - b0);
    Pack<PackedUpdJob> pk;
    size_t tiles = 0;
    for (size_t i = 0; i < nb; ++i) {
      pk.j[i] = jobs[b0 + i];
      tiles = std::max(tiles, cap_tiles(pk.j[i].n));
    }
    LAUNCH(c, herm_packed_update_kernel, dim3((unsigned)tiles, (unsigned)nb), 256, 0, pk, alpha);
  }
}

void lazy_correct(radmm_ctx* c, const std::vector<int>& qs, double mu, const int* go, bool on_dw = false);
// The lazy terms in one cluster launch (RADMM_LAZY_FUSED=0: dot + axpy launches).
bool lazy_fused(int rows_max) { return rows_max <= kLazyFusedRows && env_int("RADMM_LAZY_FUSED", 1) != 0; }

// rho += mu A_D (A_D^H w) for sensors with accumulated lazy columns: the
// residual against C_D = C - mu A_D A_D^H, the capacitance the lazy inverse
// (G + P Sinv P^H terms) inverts.
void lazy_resid(radmm_ctx* c, const std::vector<int>& qs, double mu, const int* go) {
  Pack<LazyJob> pk;
  int nb = 0, dmax = 0, rmax = 0;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    if (S.primal || S.lz_d == 0) continue;
    if (nb >= kMaxBatch) fail(RADMM_INVALID_ARGUMENT, "too many sensors in one lazy-downdate batch");
    if (c->lazy_cnt.n < (size_t)kMaxBatch) c->lazy_cnt.alloc(kMaxBatch);
    LazyJob j{S.A.p, S.ld, S.rows, S.lz_pix.p, S.lz_d, S.lz_P.p, S.lz_S.p, kLazyMax, S.w.p, S.lz_t.p,
              c->lazy_cnt.p + nb};
    j.ident = 1;
    j.dst = S.rho.p;
    pk.j[nb++] = j;
    dmax = std::max(dmax, S.lz_d);
    rmax = std::max(rmax, S.rows);
  }
  if (!nb) return;
  if (lazy_fused(rmax)) {  // one cluster launch per batch (kernels_batched.cuh)
    LAUNCH(c, lazy_fused_kernel, dim3(kLazyCluster, (unsigned)nb), 256, 0, pk, mu, go);
    return;
  }
  LAUNCH(c, lazy_dot_kernel, dim3((unsigned)dmax, (unsigned)nb), 256, 0, pk, mu, go);
  LAUNCH(c, lazy_resid_axpy_kernel, dim3((unsigned)((rmax + 255) / 256), (unsigned)nb), 256, 0, pk, go);
}

// Re-derive the complex64 copy of a packed G after it changed (memory
// permitting; RADMM_G32=0 keeps the correction in fp64).  The correction
// pass's input is the residual, ~eps cond(C) of v, so fp32 factor entries
// cost nothing measurable (C2 single solve: 1.8e-9 vs 6.7e-10).
bool g32_refresh(radmm_ctx* c, Sensor& S) {
  if (!S.gpacked || env_int("RADMM_G32", 1) == 0) return false;
  if (S.g32_valid) return true;
  const size_t n = cap_tiles(S.rows) * kHermTile * kHermTile;
  if (S.G32.n < n) {
    if (mem_available(c->device) < n * sizeof(float2) + (4ull << 30)) return false;
    S.G32.alloc(n, false);
  }
  LAUNCH(c, pack_to_c64_kernel, dim3((unsigned)std::min<size_t>((n + 255) / 256, 4096)), 256, 0, S.G.p, S.G32.p,
         (int64_t)n);
  S.g32_valid = true;
  return true;
}

// One step of fixed-precision iterative refinement of w = C_D^{-1} v for the
// listed dual sensors (after gapply + lazy_correct left w1 in S.w):
//   rho = v - C w1 + mu A_D A_D^H w1     (packed C, Hermitian apply)
//   dw  = G rho + lazy terms             (the same apply as w1's)
//   w   = w1 + dw
// It makes the explicit-inverse solve backward stable: C2 5.7e-6 -> 2.5e-10
// against the primal-Cholesky solution.  Algorithmic
// bytes: one more pass over C's and G's lower triangles.
void refine(radmm_ctx* c, const std::vector<int>& gq, double mu, const int* go) {
  if (!c->refine) return;
  std::vector<int> qs;
  for (int q : gq)
    if (!c->sensors[q].primal && c->sensors[q].cp_valid) qs.push_back(q);
  for (size_t b0 = 0; b0 < qs.size(); b0 += kMaxBatch) {
    const std::vector<int> part(qs.begin() + b0, qs.begin() + std::min(qs.size(), b0 + kMaxBatch));
    int rows_max = 0;
    bool any_lazy = false;
    for (int q : part) {
      Sensor& S = c->sensors[q];
      if (S.rho.n < (size_t)S.ld) S.rho.alloc(S.ld);
      if (S.dw.n < (size_t)S.ld) S.dw.alloc(S.ld);
      rows_max = std::max(rows_max, S.rows);
      any_lazy = any_lazy || S.lz_d > 0;
    }
    // rho = v - C w1
    Pack<HermJob> pk;
    const int nb_max = herm_pack(c, part, pk);
    for (size_t i = 0; i < part.size(); ++i) {
      Sensor& S = c->sensors[part[i]];
      HermJob& h = pk.j[i];
      h.G = S.Cp.p; h.ld = kHermTile; h.packed = 1;
      h.v = S.w.p; h.w = S.rho.p; h.v1 = nullptr; h.w1 = nullptr;
      h.base = S.v.p; h.sgn = -1.0;
    }
    herm_launch(c, pk, part.size(), nb_max, 1, go, true);
    if (any_lazy) lazy_resid(c, part, mu, go);
    // dw = C_D^{-1} rho (w += dw directly when no lazy terms follow), through
    // the complex64 copy of a packed G where it fits (g32_refresh)
    const bool herm = herm_enabled() && rows_max >= env_int("RADMM_HERM_MIN_ROWS", kHermMinRows);
    if (herm) {
      Pack<HermJob> pg;
      herm_pack(c, part, pg);
      for (size_t i = 0; i < part.size(); ++i) {
        Sensor& S = c->sensors[part[i]];
        HermJob& h = pg.j[i];
        h.G32 = g32_refresh(c, S) ? S.G32.p : nullptr;
        h.v = S.rho.p; h.v1 = nullptr; h.w1 = nullptr;
        if (S.lz_d > 0) { h.w = S.dw.p; h.base = nullptr; }
        else { h.w = S.w.p; h.base = S.w.p; h.sgn = 1.0; }
      }
      herm_launch(c, pg, part.size(), nb_max, 1, go);
    } else {
      std::vector<ColDotJob> gj;
      for (int q : part) {
        Sensor& S = c->sensors[q];
        ColDotJob g{};
        g.M = S.G.p; g.ld = S.ldg; g.len = S.rows; g.n_out = S.rows; g.vec = S.rho.p; g.out = S.dw.p; g.scale = 1.0;
        gj.push_back(g);
      }
      coldot<double2, EPI_STORE>(c, gj, 1.0, 1.0, go);
    }
    if (any_lazy) lazy_correct(c, part, mu, go, true);
    Pack<VaddJob> va;
    int nva = 0;
    for (int q : part) {
      Sensor& S = c->sensors[q];
      if (herm && S.lz_d == 0) continue;  // already folded into the reduce
      if (S.lz_d > 0) continue;           // folded into the lazy term (lazy_correct, sum_into)
      va.j[nva++] = VaddJob{S.w.p, S.dw.p, S.rows};
    }
    if (nva) LAUNCH(c, vadd_kernel, dim3((unsigned)((rows_max + 255) / 256), (unsigned)nva), 256, 0, va, go);
  }
}

// Full rebuild for the listed sensors (batched): data term + factor.
void release_ozaki_scratch(radmm_ctx* c);

void rebuild_packed(radmm_ctx* c, const std::vector<int>& qs, double mu, double beta);

void full_rebuild(radmm_ctx* c, const std::vector<int>& qs0, double mu, double beta) {
  if (qs0.empty()) return;
  std::vector<int> qs, packed;
  for (int q : qs0) {
    Sensor& S = c->sensors[q];
    S.primal = S.n_act <= S.rows;
    (!S.primal && use_gpacked(c, S) ? packed : qs).push_back(q);
  }
  rebuild_packed(c, packed, mu, beta);
  if (qs.empty()) return;
  std::vector<GemmJob> jobs;
  std::vector<GramJob> grams;
  std::vector<InvTarget> inv;
  for (int q : qs) {  // every factor's storage first: the Ozaki scratch is sized against what is left
    Sensor& S = c->sensors[q];
    const bool primal = S.n_act <= S.rows;
    const int dim = primal ? S.n_act : S.rows;
    ensure_g(S, dim, primal ? round_up(dim, 32) : S.ld);
  }
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    S.primal = S.n_act <= S.rows;
    S.lz_d = S.lz_new = 0;  // a fresh factor of the current set
    const int dim = S.primal ? S.n_act : S.rows;
    const int64_t ldg = S.primal ? round_up(dim, 32) : S.ld;
    const bool raw = S.raw_gram && !S.raw_packed && !S.primal && S.n_act == c->N && S.ldg == ldg && !S.gpacked;
    if (S.gpacked) S.G.release();  // was packed (layout switch): a full matrix now
    S.gpacked = false;
    ensure_g(S, dim, ldg);
    S.ldg = ldg;
    S.g_n = dim;
    if (!raw) CK(cudaMemsetAsync(S.G.p, 0, sizeof(double2) * (size_t)ldg * dim, c->stream));
    if (S.primal) {
      // Gram mu A_J^H A_J + beta I (solver_core.hpp:39-40)
      jobs.push_back(gjob(dim, dim, S.rows, mref(S.A.p, S.ld, true, true, true, nullptr, S.J.p),
                          mref(S.A.p, S.ld, true, false, false, nullptr, S.J.p), S.G.p, ldg, mu, 0.0, beta));
      jobs.back().herm = 1;  // Hermitian: lower tiles + mirror
    } else if (raw) {
      // the full-set Gram was formed at upload (eager_gram): scale it in place
      // (same roundings as forming beta I + mu A A^H directly)
      LAUNCH(c, gram_scale_kernel, dim3((unsigned)((int64_t)dim * dim + 255) / 256), 256, 0, S.G.p, ldg, dim, mu,
             beta);
    } else if (env_int("RADMM_GRAM", 1) && ozaki_gram(c, S, S.J.p, S.n_act, S.G.p, ldg, mu, beta)) {
      // capacitance beta I + mu A_J A_J^H from int8 slices on the tcgen05 tensor cores
    } else if (env_int("RADMM_GRAM", 1)) {
      // capacitance beta I + mu A_J A_J^H on the fp64 tensor cores
      grams.push_back(GramJob{S.A.p, S.ld, S.J.p, S.n_act, S.rows, S.G.p, ldg});
    } else {
      // capacitance beta I + mu A_J A_J^H (Woodbury form of the same system)
      jobs.push_back(gjob(dim, dim, S.n_act, mref(S.A.p, S.ld, true, false, false, nullptr, S.J.p),
                          mref(S.A.p, S.ld, true, true, true, nullptr, S.J.p), S.G.p, ldg, mu, 0.0, beta));
      jobs.back().herm = 1;
    }
    inv.push_back({S.G.p, ldg, dim});
    S.raw_gram = false;  // G now holds (becomes) the factor
    ++c->rebuilds;
  }
  if (!grams.empty()) {
    if (c->gram_jobs.n < grams.size()) c->gram_jobs.alloc(grams.size(), false);
    CK(cudaMemcpyAsync(c->gram_jobs.p, grams.data(), sizeof(GramJob) * grams.size(), cudaMemcpyHostToDevice,
                       c->stream));
    int mmax = 0;
    for (const auto& g : grams) mmax = std::max(mmax, g.m);
    set_smem_attr((const void*)gram_dmma_kernel, (int)((int)kGramSmem));
    LAUNCH(c, gram_dmma_kernel, dim3((unsigned)((mmax + kGrBN - 1) / kGrBN), (unsigned)((mmax + kGrBM - 1) / kGrBM),
                                     (unsigned)grams.size()),
           256, kGramSmem, c->gram_jobs.p, mu, beta);
  }
  gemm<GEPI_PLAIN>(c, jobs);
  release_ozaki_scratch(c);
  for (int q : qs) cap_keep(c, c->sensors[q], c->sensors[q].G.p, c->sensors[q].ldg);  // C, before the in-place inversion
  size_t need = 0;
  for (const auto& t : inv) need += (64 * 64 + 2 * (size_t)round_up(t.n, 64) * 64) * sizeof(double2) + 1024;
  c->scratch.reserve(need);
  gj_invert(c, inv, "factorize");
  symmetrize(c, qs);
}

// Dual factors in packed lower tiles: per chunk of sensors, the capacitance
// is formed in full temporaries (upload-time raw Gram unpacked and scaled, or
// a fresh Ozaki / DMMA Gram), kept packed (Cp, refinement), inverted in place
// by Gauss-Jordan and packed into S.G.  Chunks are sized so the temporaries
// fit next to everything resident (config 3 on one GPU: 171 GB).
void rebuild_packed(radmm_ctx* c, const std::vector<int>& qs, double mu, double beta) {
  if (qs.empty()) return;
  size_t full = 0;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    S.lz_d = S.lz_new = 0;
    const size_t ge = cap_tiles(S.rows) * kHermTile * kHermTile;
    if (!S.gpacked || S.G.n < ge) {
      S.G.release();
      S.G.alloc(ge, false);
    }
    S.gpacked = true;
    S.g32_valid = false;
    S.ldg = kHermTile;
    S.g_n = S.rows;
    full = std::max(full, (size_t)S.ld * S.rows);
  }
  for (int q : qs) {  // C's packed tiles before the temporaries take what is left
    Sensor& S = c->sensors[q];
    const size_t cn = cap_tiles(S.rows) * kHermTile * kHermTile;
    if (S.Cp.n < cn && mem_available(c->device) >= cn * sizeof(double2) + (4ull << 30)) S.Cp.alloc(cn, false);
  }
  const size_t free_b = mem_available(c->device);
  size_t held = 0;
  for (auto& t : c->gtmp) held += t.n * sizeof(double2);
  const size_t room = free_b + held > (6ull << 30) ? free_b + held - (6ull << 30) : 0;
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>(qs.size(), room / (full * sizeof(double2))));
  gtmp_reserve(c, chunk, full);
  for (size_t b0 = 0; b0 < qs.size(); b0 += chunk) {
    const size_t nb = std::min<size_t>(chunk, qs.size() - b0);
    std::vector<GemmJob> jobs;
    std::vector<GramJob> grams;
    std::vector<InvTarget> inv;
    for (size_t i = 0; i < nb; ++i) {
      Sensor& S = c->sensors[qs[b0 + i]];
      double2* T = c->gtmp[i].p;
      const int64_t ldt = S.ld;
      const int dim = S.rows;
      if (S.raw_gram && S.raw_packed && S.cp_valid && S.n_act == c->N) {
        // the raw full-set Gram A A^H formed at upload (eager_gram, packed in Cp)
        CK(cudaMemsetAsync(T, 0, sizeof(double2) * (size_t)ldt * dim, c->stream));
        LAUNCH(c, cap_unpack_kernel, dim3((unsigned)cap_tiles(dim)), 256, 0, S.Cp.p, dim, T, ldt);
        LAUNCH(c, gram_scale_kernel, dim3((unsigned)((int64_t)dim * dim + 255) / 256), 256, 0, T, ldt, dim, mu,
               beta);
      } else {
        CK(cudaMemsetAsync(T, 0, sizeof(double2) * (size_t)ldt * dim, c->stream));
        if (env_int("RADMM_GRAM", 1) && ozaki_gram(c, S, S.J.p, S.n_act, T, ldt, mu, beta)) {
        } else if (env_int("RADMM_GRAM", 1)) {
          grams.push_back(GramJob{S.A.p, S.ld, S.J.p, S.n_act, S.rows, T, ldt});
        } else {
          jobs.push_back(gjob(dim, dim, S.n_act, mref(S.A.p, S.ld, true, false, false, nullptr, S.J.p),
                              mref(S.A.p, S.ld, true, true, true, nullptr, S.J.p), T, ldt, mu, 0.0, beta));
          jobs.back().herm = 1;
        }
      }
      inv.push_back({T, ldt, dim});
      S.raw_gram = false;
      ++c->rebuilds;
    }
    if (!grams.empty()) {
      if (c->gram_jobs.n < grams.size()) c->gram_jobs.alloc(grams.size(), false);
      CK(cudaMemcpyAsync(c->gram_jobs.p, grams.data(), sizeof(GramJob) * grams.size(), cudaMemcpyHostToDevice,
                         c->stream));
      int mmax = 0;
      for (const auto& g : grams) mmax = std::max(mmax, g.m);
      set_smem_attr((const void*)gram_dmma_kernel, (int)((int)kGramSmem));
      LAUNCH(c, gram_dmma_kernel,
             dim3((unsigned)((mmax + kGrBN - 1) / kGrBN), (unsigned)((mmax + kGrBM - 1) / kGrBM),
                  (unsigned)grams.size()),
             256, kGramSmem, c->gram_jobs.p, mu, beta);
    }
    gemm<GEPI_PLAIN>(c, jobs);
    for (size_t i = 0; i < nb; ++i) {
      Sensor& S = c->sensors[qs[b0 + i]];
      cap_keep(c, S, c->gtmp[i].p, S.ld);
    }
    size_t need = 0;
    for (const auto& t : inv) need += (64 * 64 + 3 * (size_t)round_up(t.n, 64) * 64) * sizeof(double2) + 1024;
    c->scratch.reserve(need);
    // Hermitian sweep (RADMM_GJ_HERM=0: the general sweep + projection): the
    // capacitances are HPD and only their lower tiles are kept
    const bool hsweep = env_int("RADMM_GJ_HERM", 1) != 0;
    gj_invert(c, inv, "factorize", hsweep);
    for (size_t i = 0; i < nb; ++i) {
      Sensor& S = c->sensors[qs[b0 + i]];
      // Hermitian projection first (see symmetrize): the packed apply reads the
      // diagonal tiles whole, so they must be the projected factor's (the
      // Hermitian sweep's result is exactly Hermitian already)
      if (!hsweep && env_int("RADMM_SYMM", 1) != 0) {
        const int nt = (S.rows + 31) / 32;
        LAUNCH(c, herm_symmetrize_kernel, dim3((unsigned)((int64_t)nt * (nt + 1) / 2)), 256, 0, c->gtmp[i].p, S.ld,
               S.rows);
      }
      LAUNCH(c, cap_pack_kernel, dim3((unsigned)cap_tiles(S.rows)), 256, 0, c->gtmp[i].p, S.ld, S.rows, S.G.p);
    }
  }
  release_ozaki_scratch(c);
  gtmp_release(c);
}

// Data term mu A_J^H y_eff for the listed sensors (admm.hpp:177).
void data_terms(radmm_ctx* c, const std::vector<int>& qs, double mu) {
  std::vector<ColDotJob> jobs;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    ColDotJob j{};
    j.M = S.A.p; j.ld = S.ld; j.len = S.rows; j.n_out = S.n_act; j.cols = S.J.p;
    j.vec = S.y_eff.p; j.out = S.data.p; j.scale = mu;
    jobs.push_back(j);
  }
  coldot<float2, EPI_STORE>(c, jobs, mu, 1.0);
  for (int q : qs) {  // the data term is exact again: snapshot y_eff, no lag
    Sensor& S = c->sensors[q];
    CK(cudaMemcpyAsync(S.y_eff_s.p, S.y_eff.p, sizeof(double2) * S.ld, cudaMemcpyDeviceToDevice, c->stream));
    S.data_lag = false;
  }
}

// One batched bookkeeping launch per event (see event_prep_kernel).
void event_prep(radmm_ctx* c, const std::vector<EventJob>& jobs) {
  for (size_t b0 = 0; b0 < jobs.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, jobs.size() - b0);
    Pack<EventJob> pk;
    int64_t work = 1;
    for (size_t i = 0; i < nb; ++i) {
      const EventJob& j = jobs[b0 + i];
      pk.j[i] = j;
      work = std::max<int64_t>(work, std::max<int64_t>(j.r, (j.lz_R ? j.ld * j.r : 0) + (j.bz ? j.ld : 0)));
    }
    const unsigned blocks = (unsigned)std::min<int64_t>(1024, (work + 255) / 256);
    LAUNCH(c, event_prep_kernel, dim3(blocks, (unsigned)nb), 256, 0, pk);
  }
}

// ---- lazy Woodbury downdates (dual form) ------------------------------------
bool fused_enabled();
bool lazy_enabled() { return env_int("RADMM_LAZY", 1) != 0 && !fused_enabled(); }
// RADMM_LAZY_MAX (<= kLazyMax) lowers the fold point (tests force folds)
int lazy_max() { return std::min(kLazyMax, std::max(1, env_int("RADMM_LAZY_MAX", kLazyMax))); }

// Removed columns per event that ride the iteration's G-apply as extra
// right-hand sides (1: the two-RHS kernel; 2-3: the four-RHS kernel, one CTA
// per SM); larger events form their columns in extra passes, two per pass.
int lazy_ride() { return std::max(0, std::min(3, env_int("RADMM_LAZY_RIDE", 3))); }

void lazy_reserve(Sensor& S) {
  if (S.lz_P.n < (size_t)S.ld * kLazyMax) {
    S.lz_P.alloc((size_t)S.ld * kLazyMax, false);
    S.lz_R.alloc((size_t)S.ld * kLazyMax, false);
    S.lz_S.alloc((size_t)kLazyMax * kLazyMax, false);
    S.lz_t.alloc(2 * kLazyMax, false);
    S.lz_pix.alloc(kLazyMax, false);
    S.lz_B.alloc((size_t)kLazyMax * kBorderMax, false);
  }
}

// Sinv <- (I - mu A_D^H P)^{-1} for the listed sensors, whose last lz_r
// columns of P were just formed: bordered update (lazy_border_*_kernel), two
// launches for all sensors.  Pivots are checked at the iteration's sync, like
// the eager path's.
void lazy_finish(radmm_ctx* c, const std::vector<int>& qs, double mu) {
  if (qs.empty()) return;
  if (qs.size() > (size_t)kMaxBatch) fail(RADMM_INVALID_ARGUMENT, "too many sensors in one lazy-downdate batch");
  Pack<BorderJob> pk;
  int dmax = 0;
  for (size_t i = 0; i < qs.size(); ++i) {
    Sensor& S = c->sensors[qs[i]];
    pk.j[i] = BorderJob{S.A.p, S.ld, S.rows, S.lz_pix.p, S.lz_d - S.lz_r, S.lz_r, S.lz_P.p, S.lz_B.p, S.lz_S.p,
                        c->fail_flags.p + i};
    dmax = std::max(dmax, S.lz_d);
  }
  const unsigned nb = (unsigned)qs.size();
  LAUNCH(c, lazy_border_dots_kernel, dim3((unsigned)dmax, nb), 256, 0, pk);
  set_smem_attr((const void*)lazy_border_inv_kernel, (int)((int)kBorderSmem));
  LAUNCH(c, lazy_border_inv_kernel, dim3(nb), 256, kBorderSmem, pk, mu);
  if (c->pending_fail + (int)nb > kFlagCap) {
    CK(cudaStreamSynchronize(c->stream));
    check_deferred(c);
  }
  CK(cudaMemcpyAsync(c->h_flags + c->pending_fail, c->fail_flags.p, sizeof(int) * nb, cudaMemcpyDeviceToHost,
                     c->stream));
  c->pending_fail += (int)nb;
}

// Fold the accumulated columns into G: G <- G + mu P Sinv P^H (Hermitian,
// lower tiles + exact mirror), D <- {}.
void lazy_fold(radmm_ctx* c, const std::vector<int>& qs, double mu) {
  if (qs.empty()) return;
  size_t need = 0;
  for (int q : qs) need += (size_t)c->sensors[q].ld * kLazyMax * sizeof(double2) + 1024;
  c->scratch.reserve(need);
  std::vector<GemmJob> st3, st4;
  std::vector<CapJob> cj;
  std::vector<PackedUpdJob> pu;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    const int m = S.rows, d = S.lz_d;
    double2* T = c->scratch.take<double2>((size_t)S.ld * kLazyMax);
    st3.push_back(gjob(m, d, d, mref(S.lz_P.p, S.ld, false), mref(S.lz_S.p, kLazyMax, false), T, S.ld, 1.0, 0.0));
    if (S.gpacked) {
      S.g32_valid = false;
      pu.push_back(PackedUpdJob{S.G.p, T, S.lz_P.p, S.ld, m, d});
    } else {
      st4.push_back(gjob(m, m, d, mref(T, S.ld, false), mref(S.lz_P.p, S.ld, false, true, true), S.G.p, S.ldg, mu,
                         1.0));
      st4.back().herm = 1;
    }
    if (S.cp_valid) cj.push_back(CapJob{S.Cp.p, S.A.p, S.ld, S.rows, S.lz_pix.p, d});
    S.lz_d = 0;
    S.lz_new = 0;
  }
  gemm<GEPI_PLAIN>(c, st3);
  gemm<GEPI_PLAIN>(c, st4);
  packed_update(c, pu, mu);
  cap_update(c, cj, mu);  // the base capacitance follows G's base set
}

// Append this event's removed columns to D.  A single column rides the next
// iteration's G-apply as a second right-hand side (no extra pass over G);
// more columns are formed now, two per pass of G's lower triangle.
void lazy_append(radmm_ctx* c, const std::vector<int>& qs, double mu) {
  if (qs.empty()) return;
  auto clk = [] { return std::chrono::steady_clock::now(); };
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  const auto l0 = clk();
  std::vector<int> now;
  int passes = 0;
  std::vector<EventJob> ej;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    const int r = S.removed_now;
    lazy_reserve(S);
    EventJob e{};
    e.rem_pix = S.rem_pix.p; e.r = r; e.lz_pix_dst = S.lz_pix.p + S.lz_d; e.A = S.A.p; e.ld = S.ld; e.lz_R = S.lz_R.p;
    ej.push_back(e);
    S.lz_d += r;
    S.lz_r = r;
    if (r <= lazy_ride() && herm_enabled()) {
      S.lz_new = r;  // formed by the next iteration's G-apply (gapply), no extra pass over G
    } else {
      now.push_back(q);
      passes = std::max(passes, (r + 1) / 2);
    }
    ++c->downdates;
  }
  event_prep(c, ej);
  const auto l1 = clk();
  c->trace_us[3] += us(l0, l1);
  if (now.empty()) return;
  std::vector<int> dual;  // the iteration's G-apply batch (same item table)
  for (int q = 0; q < c->Q; ++q)
    if (!c->sensors[q].primal) dual.push_back(q);
  if (!herm_enabled() || dual.size() > (size_t)kMaxBatch) {
    std::vector<ColDotJob> gj;
    for (int q : now) {
      Sensor& S = c->sensors[q];
      const int r = S.removed_now, d0 = S.lz_d - r;
      for (int u = 0; u < r; ++u) {
        ColDotJob g{};
        g.M = S.G.p; g.ld = S.ldg; g.len = S.rows; g.n_out = S.rows; g.scale = 1.0;
        g.vec = S.lz_R.p + (size_t)u * S.ld; g.out = S.lz_P.p + (size_t)(d0 + u) * S.ld;
        gj.push_back(g);
      }
    }
    coldot<double2, EPI_STORE>(c, gj, 1.0, 1.0);
  } else {
    Pack<HermJob> pk;
    const int nb_max = herm_pack(c, dual, pk);
    c->trace_us[4] += us(l1, clk());
    for (int p = 0; p < passes; ++p) {
      for (size_t i = 0; i < dual.size(); ++i) {
        Sensor& S = c->sensors[dual[i]];
        HermJob& h = pk.j[i];
        h.v = h.v1 = nullptr;
        h.w = h.w1 = nullptr;
        if (std::find(now.begin(), now.end(), dual[i]) == now.end()) continue;
        const int r = S.removed_now, d0 = S.lz_d - r;
        for (int t = 0; t < 2; ++t) {
          const int u = 2 * p + t;
          if (u >= r) break;
          (t ? h.v1 : h.v) = S.lz_R.p + (size_t)u * S.ld;
          (t ? h.w1 : h.w) = S.lz_P.p + (size_t)(d0 + u) * S.ld;
        }
      }
      herm_launch(c, pk, dual.size(), nb_max, 2, nullptr);
    }
  }
  const auto l2 = clk();
  c->trace_us[5] += us(l1, l2);
  lazy_finish(c, now, mu);
  c->trace_us[6] += us(l2, clk());
}

// w <- C_D^{-1} v from u = G v for every listed sensor with accumulated columns.
void lazy_correct(radmm_ctx* c, const std::vector<int>& qs, double mu, const int* go, bool on_dw) {
  Pack<LazyJob> pk;
  int nb = 0, dmax = 0, rmax = 0;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    if (S.primal || S.lz_d == 0) continue;
    if (nb >= kMaxBatch) fail(RADMM_INVALID_ARGUMENT, "too many sensors in one lazy-downdate batch");
    pk.j[nb] = LazyJob{S.A.p, S.ld, S.rows, S.lz_pix.p, S.lz_d, S.lz_P.p, S.lz_S.p, kLazyMax,
                       on_dw ? S.dw.p : S.w.p, S.lz_t.p, c->lazy_cnt.p + nb};
    // the refinement's correction: w += dw + lazy term in the same kernel (no separate w += dw)
    if (on_dw) pk.j[nb].sum_into = S.w.p;
    ++nb;
    dmax = std::max(dmax, S.lz_d);
    rmax = std::max(rmax, S.rows);
  }
  if (!nb) return;
  if (c->lazy_cnt.n < (size_t)kMaxBatch) c->lazy_cnt.alloc(kMaxBatch);  // zeroed; the last blocks re-zero
  for (int i = 0; i < nb; ++i) pk.j[i].cnt = c->lazy_cnt.p + i;
  if (lazy_fused(rmax)) {
    LAUNCH(c, lazy_fused_kernel, dim3(kLazyCluster, (unsigned)nb), 256, 0, pk, mu, go);
    return;
  }
  LAUNCH(c, lazy_dot_kernel, dim3((unsigned)dmax, (unsigned)nb), 256, 0, pk, mu, go);
  LAUNCH(c, lazy_axpy_kernel, dim3((unsigned)((rmax + 255) / 256), (unsigned)nb), 256, 0, pk, mu, go);
}

void eager_downdate(radmm_ctx* c, const std::vector<int>& qs, double mu);
void snapshot_base(radmm_ctx* c, Sensor& S, bool modify);

// Downdates after screening removed rem_q columns: dual sensors accumulate
// them lazily (up to kLazyMax, then fold); primal sensors and large removals
// take the eager path.
void downdate(radmm_ctx* c, const std::vector<int>& qs, double mu) {
  if (qs.empty()) return;
  std::vector<int> lazy, fold, eager;
  const bool lz = lazy_enabled();
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    const int cap = lazy_max();
    const bool use_lazy = lz && !S.primal && S.removed_now <= std::min(cap, kBorderMax);
    if (!S.primal && S.lz_d > 0 && (!use_lazy || S.lz_d + S.removed_now > cap)) fold.push_back(q);
    (use_lazy ? lazy : eager).push_back(q);
  }
  for (int q : fold) snapshot_base(c, c->sensors[q], true);
  for (int q : eager) snapshot_base(c, c->sensors[q], true);
  lazy_fold(c, fold, mu);
  lazy_append(c, lazy, mu);
  eager_downdate(c, eager, mu);
}

// Low-rank downdates after screening removed rem_q columns.
//   dual:   G <- G + mu P (I - mu R^H P)^{-1} P^H,  P = G R   (Woodbury)
//   primal: Hinv_KK <- Hinv_KK - Hinv_KD inv(Hinv_DD) Hinv_DK (inverse of a
//           principal submatrix), written compacted into G2 then swapped.
void eager_downdate(radmm_ctx* c, const std::vector<int>& qs, double mu) {
  if (qs.empty()) return;
  size_t need = 0;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    const size_t r = S.removed_now;
    const size_t dimr = round_up(r, 64);
    if (S.primal) need += (dimr * dimr + (size_t)round_up(S.n_act, 64) * dimr) * sizeof(double2);
    else need += (3 * (size_t)S.ld * dimr + dimr * dimr) * sizeof(double2);
    need += (64 * 64 + 2 * dimr * 64) * sizeof(double2) + 4096;
  }
  c->scratch.reserve(need);
  std::vector<GemmJob> st1, st2, st3, st4;
  std::vector<std::vector<ColDotJob>> p_by_col;  // P[:, u] = G a_u jobs, by column u
  std::vector<InvTarget> inv;
  Pack<SubJob> sub;
  int nsub = 0;
  int64_t sub_max = 0;
  std::vector<double2*> Pm(qs.size()), Tm(qs.size()), Sm(qs.size());
  std::vector<CapJob> capj;
  std::vector<PackedUpdJob> pupd;
  std::vector<int> hp_q;                 // packed dual sensors: P = G R by Hermitian applies
  std::vector<double2*> hp_R, hp_P;
  for (size_t t = 0; t < qs.size(); ++t) {
    Sensor& S = c->sensors[qs[t]];
    const int r = S.removed_now;
    const int64_t ldr = round_up(r, 32);
    Sm[t] = c->scratch.take<double2>((size_t)ldr * r);
    CK(cudaMemsetAsync(Sm[t], 0, sizeof(double2) * (size_t)ldr * r, c->stream));
    if (!S.primal) {
      const int m = S.rows;
      Pm[t] = c->scratch.take<double2>((size_t)S.ld * r);
      Tm[t] = c->scratch.take<double2>((size_t)S.ld * r);
      // P = G R: few columns -> r Hermitian matvecs G a_t through the streaming
      // column-dot kernel (G read once per removed column, all sensors batched);
      // many columns -> tiled GEMM; packed factors -> Hermitian applies, two
      // columns per pass over the lower tiles
      if (S.gpacked) {
        double2* Rb = c->scratch.take<double2>((size_t)S.ld * r);
        LAUNCH(c, gather_cols_c128_kernel, dim3((unsigned)((S.ld * r + 255) / 256)), 256, 0, S.A.p, S.ld,
               S.rem_pix.p, r, Rb);
        hp_q.push_back(qs[t]);
        hp_R.push_back(Rb);
        hp_P.push_back(Pm[t]);
      } else if (r <= env_int("RADMM_DD_MATVEC", kDowndateMatvecMax)) {
        double2* Rb = c->scratch.take<double2>((size_t)S.ld * r);
        LAUNCH(c, gather_cols_c128_kernel, dim3((unsigned)((S.ld * r + 255) / 256)), 256, 0, S.A.p, S.ld,
               S.rem_pix.p, r, Rb);
        for (int u = 0; u < r; ++u) {
          ColDotJob j{};
          j.M = S.G.p; j.ld = S.ldg; j.len = S.rows; j.n_out = S.rows; j.vec = Rb + (size_t)u * S.ld;
          j.out = Pm[t] + (size_t)u * S.ld; j.scale = 1.0;
          if ((int)p_by_col.size() <= u) p_by_col.resize(u + 1);
          p_by_col[u].push_back(j);
        }
      } else {
        st1.push_back(gjob(m, r, m, mref(S.G.p, S.ldg, false),
                           mref(S.A.p, S.ld, true, false, false, nullptr, S.rem_pix.p), Pm[t], S.ld, 1.0, 0.0));
      }
      // S = I - mu R^H P
      st2.push_back(gjob(r, r, m, mref(S.A.p, S.ld, true, true, true, nullptr, S.rem_pix.p),
                         mref(Pm[t], S.ld, false), Sm[t], ldr, -mu, 0.0, 1.0));
      inv.push_back({Sm[t], ldr, r});
      // T = P Sinv
      st3.push_back(gjob(m, r, r, mref(Pm[t], S.ld, false), mref(Sm[t], ldr, false), Tm[t], S.ld, 1.0, 0.0));
      // G += mu T P^H: a Hermitian rank-r update, applied to the lower tiles
      // with an exact conjugate mirror -- G stays exactly Hermitian (no
      // projection pass needed after a downdate)
      if (S.gpacked) {
        S.g32_valid = false;
        pupd.push_back(PackedUpdJob{S.G.p, Tm[t], Pm[t], S.ld, m, r});
      } else {
        st4.push_back(gjob(m, m, r, mref(Tm[t], S.ld, false), mref(Pm[t], S.ld, false, true, true), S.G.p,
                           S.ldg, mu, 1.0));
        st4.back().herm = 1;
      }
      if (S.cp_valid) capj.push_back(CapJob{S.Cp.p, S.A.p, S.ld, S.rows, S.rem_pix.p, r});
    } else {
      const int nn = S.n_act;  // kept
      const int64_t ld_new = round_up(nn, 32);
      if (S.G2.n < (size_t)ld_new * nn) S.G2.alloc((size_t)ld_new * nn);
      CK(cudaMemsetAsync(S.G2.p, 0, sizeof(double2) * (size_t)ld_new * nn, c->stream));
      Tm[t] = c->scratch.take<double2>((size_t)round_up(nn, 64) * r);
      // S = Hinv[D, D]
      SubJob sj;
      sj.M = S.G.p; sj.ld = S.ldg; sj.ridx = S.rem_pos.p; sj.cidx = S.rem_pos.p; sj.m = r; sj.n = r;
      sj.out = Sm[t]; sj.ldo = ldr;
      sub.j[nsub++] = sj;
      sub_max = std::max<int64_t>(sub_max, (int64_t)r * r);
      SubJob sk;
      sk.M = S.G.p; sk.ld = S.ldg; sk.ridx = S.keep_pos.p; sk.cidx = S.keep_pos.p; sk.m = nn; sk.n = nn;
      sk.out = S.G2.p; sk.ldo = ld_new;
      sub.j[nsub++] = sk;
      sub_max = std::max<int64_t>(sub_max, (int64_t)nn * nn);
      inv.push_back({Sm[t], ldr, r});
      // T = Hinv[K, D] Sinv
      st3.push_back(gjob(nn, r, r, mref(S.G.p, S.ldg, false, false, false, S.keep_pos.p, S.rem_pos.p),
                         mref(Sm[t], ldr, false), Tm[t], round_up(nn, 64), 1.0, 0.0));
      // G2 -= T Hinv[D, K]
      st4.push_back(gjob(nn, nn, r, mref(Tm[t], round_up(nn, 64), false),
                         mref(S.G.p, S.ldg, false, false, false, S.rem_pos.p, S.keep_pos.p), S.G2.p, ld_new,
                         -1.0, 1.0));
    }
    ++c->downdates;
  }
  if (nsub) {
    const int blocks = (int)std::min<int64_t>(2048, (sub_max + 255) / 256);
    LAUNCH(c, gather_sub_kernel, dim3(std::max(1, blocks), nsub), 256, 0, sub);
  }
  for (const auto& jobs : p_by_col) coldot<double2, EPI_STORE>(c, jobs, mu, 1.0);
  if (!hp_q.empty()) {
    Pack<HermJob> pk;
    const int nb_max = herm_pack(c, hp_q, pk);
    int rmax = 0;
    for (int q : hp_q) rmax = std::max(rmax, c->sensors[q].removed_now);
    for (int u0 = 0; u0 < rmax; u0 += 2) {
      for (size_t i = 0; i < hp_q.size(); ++i) {
        Sensor& S = c->sensors[hp_q[i]];
        HermJob& h = pk.j[i];
        h.v = h.v1 = nullptr;
        h.w = h.w1 = nullptr;
        h.base = nullptr;
        for (int tcol = 0; tcol < 2; ++tcol) {
          const int u = u0 + tcol;
          if (u >= S.removed_now) break;
          (tcol ? h.v1 : h.v) = hp_R[i] + (size_t)u * S.ld;
          (tcol ? h.w1 : h.w) = hp_P[i] + (size_t)u * S.ld;
        }
      }
      herm_launch(c, pk, hp_q.size(), nb_max, 2, nullptr);
    }
  }
  gemm<GEPI_PLAIN>(c, st1);
  gemm<GEPI_PLAIN>(c, st2);
  c->defer_fail_check = true;  // the r x r pivots are checked after the iteration's sync
  gj_invert(c, inv, "factorize");
  c->defer_fail_check = false;
  gemm<GEPI_PLAIN>(c, st3);
  gemm<GEPI_PLAIN>(c, st4);
  packed_update(c, pupd, mu);
  cap_update(c, capj, mu);
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    if (S.primal) {
      std::swap(S.G, S.G2);
      S.ldg = round_up(S.n_act, 32);
      S.g_n = S.n_act;
    }
  }
}


// Frozen-echo update y_eff -= A[:, removed] x_full[removed] (admm.hpp:174-176;
// incremental: frozen values never change once frozen).
void update_y_eff(radmm_ctx* c, const std::vector<int>& qs) {
  std::vector<FwdJob> jobs;
  std::vector<ReduceJob> red;
  for (int q : qs) {
    Sensor& S = c->sensors[q];
    FwdJob f{};
    f.A = S.A.p; f.ld = S.ld; f.n = S.removed_now; f.J = S.rem_pix.p; f.src = S.x_full.p;
    f.part = S.part.p;
    plan_chunks(c, S, S.removed_now, (int)qs.size(), f.n_chunks, f.chunk_len);
    jobs.push_back(f);
    ReduceJob r{S.part.p, f.n_chunks, S.ld, S.rows, S.y_eff.p, S.y_eff.p, -1.0};
    red.push_back(r);
  }
  forward<MODE_GATHER>(c, jobs, red, 0.0);
}

// ---------------------------------------------------------------------------
// One run
// ---------------------------------------------------------------------------
void validate_hyper(const radmm_hyperparams* h) {
  if (!h) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: null");
  if (!(h->mu > 0.0)) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: mu must be > 0");
  if (!(h->lambda >= 0.0)) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: lambda must be >= 0");
  if (!(h->beta > 0.0)) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: beta must be > 0");
  if (!(h->eps_abs > 0.0)) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: eps_abs must be > 0");
  if (!(h->eps_rel > 0.0)) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: eps_rel must be > 0");
  if (h->screening_window < 2)
    fail(RADMM_INVALID_ARGUMENT, "Hyperparams: screening_window needs at least one successive pair");
  if (!(h->screening_tol >= 0.0)) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: screening_tol must be >= 0");
  if (h->max_iter < 1) fail(RADMM_INVALID_ARGUMENT, "Hyperparams: max_iter must be >= 1");
}

size_t contribution_size(size_t n) { return 1 + 4 + 8 + 4 + n * (4 + 16); }  // wire.hpp:54-56
size_t notice_size(size_t n) { return 1 + 4 + 8 + 4 + n * (4 + 16); }        // wire.hpp:60-62

void begin_run(radmm_ctx* c, const radmm_hyperparams* h) {
  const int N = c->N;
  c->W = h->screening_window;
  c->upd = 0;
  std::vector<int> all;
  for (int q = 0; q < c->Q; ++q) {
    Sensor& S = c->sensors[q];
    if (!S.has_op) fail(RADMM_INVALID_ARGUMENT, "Problem: sensor " + std::to_string(q) + " has no operator");
    if (!S.has_y) fail(RADMM_INVALID_ARGUMENT, "Problem: measurement length mismatch");
    S.n_act = N;
    S.stalled = false;
    S.removed_now = 0;
    S.v_ready = false;
    S.lz_d = S.lz_new = 0;
    LAUNCH(c, iota_kernel, dim3((N + 255) / 256), 256, 0, S.J.p, N);
    CK(cudaMemsetAsync(S.x_full.p, 0, sizeof(double2) * N, c->stream));
    CK(cudaMemsetAsync(S.x_hat.p, 0, sizeof(double2) * N, c->stream));
    if (S.ring.n != (size_t)c->W * N) S.ring.alloc((size_t)c->W * N);
    CK(cudaMemsetAsync(S.ring.p, 0, sizeof(double) * S.ring.n, c->stream));
    CK(cudaMemsetAsync(S.y_eff.p, 0, sizeof(double2) * S.ld, c->stream));
    CK(cudaMemcpyAsync(S.y_eff.p, S.y.p, sizeof(double2) * S.rows, cudaMemcpyDeviceToDevice, c->stream));
    all.push_back(q);
  }
  for (DArr<double2>* v : {&c->s, &c->xg, &c->sigma, &c->sigma_pre, &c->gap})
    CK(cudaMemsetAsync(v->p, 0, sizeof(double2) * N, c->stream));
  CK(cudaMemsetAsync(c->fcounter.p, 0, sizeof(unsigned), c->stream));
  data_terms(c, all, h->mu);
  std::vector<int> fresh;
  for (int q : all) {
    Sensor& S = c->sensors[q];
    // the layout this run would factor the full set in (a cached factor of
    // the other layout -- RADMM_HERM / RADMM_GPACK changed -- is refactored)
    const bool want_packed = c->N > S.rows && use_gpacked(c, S);
    if (S.g_is_base && S.base_mu == h->mu && S.base_beta == h->beta && S.gpacked == want_packed) {
      ++c->factor_cache_hits;  // G is untouched since its full-set factorization
    } else if (S.g0_valid && S.g0_mu == h->mu && S.g0_beta == h->beta && S.g0_packed == want_packed) {
      if (S.gpacked != S.g0_packed) S.G.release();
      S.g32_valid = false;
      if (S.G.n < S.g0_elems) S.G.alloc(S.g0_elems);
      CK(cudaMemcpyAsync(S.G.p, S.G0.p, sizeof(double2) * S.g0_elems, cudaMemcpyDeviceToDevice, c->stream));
      S.gpacked = S.g0_packed;
      S.primal = S.g0_primal;
      S.ldg = S.g0_ld;
      S.g_n = S.g0_n;
      S.cp_valid = false;
      if (!S.primal && S.cp0_valid) {
        const size_t cn = cap_tiles(S.rows) * kHermTile * kHermTile;
        if (S.Cp.n < cn) S.Cp.alloc(cn, false);
        CK(cudaMemcpyAsync(S.Cp.p, S.Cp0.p, cn * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
        S.cp_valid = true;
      } else if (!S.primal) {
        ++c->refine_skipped;
      }
      S.g_is_base = true;
      S.base_mu = h->mu;
      S.base_beta = h->beta;
      ++c->factor_cache_hits;
    } else {
      fresh.push_back(q);
    }
  }
  full_rebuild(c, fresh, h->mu, h->beta);
  for (int q : fresh) {
    Sensor& S = c->sensors[q];
    S.g_is_base = true;
    S.base_mu = h->mu;
    S.base_beta = h->beta;
  }
  // size the event-path scratch once (a 64-column downdate on every sensor)
  // so elimination rounds never stop to grow it
  {
    size_t need = 0;
    for (const Sensor& S : c->sensors) {
      const size_t dimr = 64, n64 = (size_t)round_up(std::max<int64_t>(S.n_act, S.rows), 64);
      need += (3 * (size_t)S.ld * dimr + dimr * dimr + n64 * dimr) * sizeof(double2);
      need += (64 * 64 + 2 * dimr * 64) * sizeof(double2) + 4096;
    }
    c->scratch.reserve(need);
  }
}

// Keep the full-set factor for the next run before G is first modified: copy
// G -> G0 when memory allows (always leaves >= 4 GB free).  `modify`: the
// caller is about to change G (downdate, fold, rebuild), so G stops being
// the base factor.
void snapshot_base(radmm_ctx* c, Sensor& S, bool modify) {
  if (!S.g_is_base) return;
  if (modify) S.g_is_base = false;
  if (S.g0_valid && S.g0_mu == S.base_mu && S.g0_beta == S.base_beta && S.g0_ld == S.ldg && S.g0_n == S.g_n &&
      S.g0_packed == S.gpacked)
    return;
  if (env_int("RADMM_FACTOR_CACHE", 1) == 0) return;
  if (!S.G0.own) S.G0.release();  // never write through a view of another context's factor
  const size_t bytes = sizeof(double2) * g_elems(S);
  if (S.G0.n < bytes / sizeof(double2)) {
    const size_t free_b = mem_available(c->device);
    if (free_b < bytes + (4ull << 30)) {
      S.g0_valid = false;
      return;
    }
    S.G0.alloc(bytes / sizeof(double2), false);
  }
  CK(cudaMemcpyAsync(S.G0.p, S.G.p, bytes, cudaMemcpyDeviceToDevice, c->stream));
  // the packed capacitance of the same base set travels with it (refinement)
  S.cp0_valid = false;
  if (S.cp_valid) {
    const size_t cn = cap_tiles(S.rows) * kHermTile * kHermTile;
    if (!S.Cp0.own) S.Cp0.release();
    bool ok = S.Cp0.n >= cn;
    if (!ok) {
      const size_t free_b = mem_available(c->device);
      if (free_b >= cn * sizeof(double2) + (4ull << 30)) {
        S.Cp0.alloc(cn, false);
        ok = true;
      }
    }
    if (ok) {
      CK(cudaMemcpyAsync(S.Cp0.p, S.Cp.p, cn * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
      S.cp0_valid = true;
    }
  }
  S.g0_valid = true;
  S.g0_primal = S.primal;
  S.g0_packed = S.gpacked;
  S.g0_elems = g_elems(S);
  S.g0_mu = S.base_mu;
  S.g0_beta = S.base_beta;
  S.g0_ld = S.ldg;
  S.g0_n = S.g_n;
}

// Adjoint + x-update.  When KM is so large that one shared copy of w per
// CTA leaves a single CTA per SM (KM > 6144, BASELINE config 3), the columns
// are dotted in row segments of kAdjSeg rows (2048: 32 KB of w per CTA, the
// config-2 occupancy) into partials, then summed in segment order.
constexpr int kAdjSeg = 2048;

void adjoint(radmm_ctx* c, const std::vector<ColDotJob>& aj, const std::vector<int>& aq, double mu, double beta,
             const int* go) {
  std::vector<ColDotJob> whole, segs;
  std::vector<XFinJob> fin;
  for (size_t t = 0; t < aj.size(); ++t) {
    const ColDotJob& a = aj[t];
    // RADMM_ADJ_SPLIT_ROWS / RADMM_ADJ_SEG override the switch point and the
    // segment (tests force several segments at oracle-sized problems)
    const int split_rows = env_int("RADMM_ADJ_SPLIT_ROWS", (int)(kColdotBigSmem / sizeof(double2)) + 1);
    const int seg = (int)round_up(std::max(64, env_int("RADMM_ADJ_SEG", kAdjSeg)), 64);
    if (a.len < split_rows) {
      whole.push_back(a);
      continue;
    }
    Sensor& S = c->sensors[aq[t]];
    const int nseg = (a.len + seg - 1) / seg;
    const size_t need = (size_t)nseg * c->N;
    if (S.apart.n < need) S.apart.alloc(need, false);
    for (int sg = 0; sg < nseg; ++sg) {
      ColDotJob j{};
      j.M = reinterpret_cast<const float2*>(a.M) + (int64_t)sg * seg;
      j.ld = a.ld;
      j.len = std::min(seg, a.len - sg * seg);
      j.vld = seg;
      j.n_out = a.n_out;
      j.cols = a.cols;
      j.vec = a.vec + (int64_t)sg * seg;
      j.out = S.apart.p + (size_t)sg * c->N;
      j.scale = 1.0;
      segs.push_back(j);
    }
    fin.push_back(XFinJob{a, S.apart.p, nseg, c->N});
  }
  if (!whole.empty()) coldot<float2, EPI_XDUAL>(c, whole, mu, beta, go);
  if (segs.empty()) return;
  coldot<float2, EPI_STORE>(c, segs, mu, beta, go);
  for (size_t b0 = 0; b0 < fin.size(); b0 += kMaxBatch) {
    const size_t nb = std::min<size_t>(kMaxBatch, fin.size() - b0);
    Pack<XFinJob> pk;
    int n_max = 0;
    for (size_t i = 0; i < nb; ++i) {
      pk.j[i] = fin[b0 + i];
      n_max = std::max(n_max, pk.j[i].a.n_out);
    }
    LAUNCH(c, xdual_finish_kernel, dim3((unsigned)((n_max + 255) / 256), (unsigned)nb), 256, 0, pk, mu, beta, go);
  }
}

// One synchronous Jacobi sweep of local updates (admm.hpp:389-390).
void local_updates(radmm_ctx* c, const radmm_hyperparams* h, const int* go = nullptr) {
  const int slot = c->upd % c->W;
  for (Sensor& S : c->sensors) S.v_ready = false;  // partial buffers are reused below
  std::vector<FwdJob> fj;
  std::vector<ReduceJob> rj;
  std::vector<ColDotJob> aj, pj;
  std::vector<int> gq;
  Pack<RhsJob> rh;
  int n_rhs = 0, rhs_max = 0;
  int n_dual = 0;
  double g_bytes = 0;
  for (int q = 0; q < c->Q; ++q) if (!c->sensors[q].primal) ++n_dual;
  for (int q = 0; q < c->Q; ++q) {
    Sensor& S = c->sensors[q];
    double* ring_slot = S.ring.p + (size_t)slot * c->N;
    if (!S.primal) {
      FwdJob f{};
      f.A = S.A.p; f.ld = S.ld; f.n = S.n_act; f.J = S.J.p; f.data = S.data.p; f.x_hat = S.x_hat.p;
      f.rhs_out = S.rhs.p; f.part = S.part.p;
      plan_chunks(c, S, S.n_act, n_dual, f.n_chunks, f.chunk_len);
      fj.push_back(f);
      // v = beta z + A_J rhs_s when the data term lags (see Sensor::data_lag)
      rj.push_back(ReduceJob{S.part.p, f.n_chunks, S.ld, S.rows, S.data_lag ? S.bz.p : nullptr, S.v.p, 1.0});
      gq.push_back(q);
      g_bytes += gapply_bytes(S.rows);
      if (c->refine && S.cp_valid)  // refinement: packed C pass + correction pass (complex64 G when it fits)
        g_bytes += 16.0 * cap_tiles(S.rows) * kHermTile * kHermTile +
                   (S.gpacked && S.g32_valid ? 8.0 * cap_tiles(S.rows) * kHermTile * kHermTile : gapply_bytes(S.rows));
      ColDotJob a{};
      a.M = S.A.p; a.ld = S.ld; a.len = S.rows; a.n_out = S.n_act; a.cols = S.J.p; a.pix = S.J.p;
      a.vec = S.w.p; a.rhs = S.rhs.p; a.x_hat = S.x_hat.p; a.x_full = S.x_full.p; a.ring_slot = ring_slot;
      aj.push_back(a);
    } else {
      if (n_rhs >= kMaxBatch) fail(RADMM_INVALID_ARGUMENT, "too many primal sensors in one batch");
      rh.j[n_rhs++] = RhsJob{S.n_act, S.J.p, S.data.p, S.x_hat.p, S.rhs.p};
      rhs_max = std::max(rhs_max, S.n_act);
      ColDotJob p{};
      p.M = S.G.p; p.ld = S.ldg; p.len = S.n_act; p.n_out = S.n_act; p.pix = S.J.p; p.vec = S.rhs.p;
      p.x_hat = S.x_hat.p; p.x_full = S.x_full.p; p.ring_slot = ring_slot;
      pj.push_back(p);
    }
  }
  double a_bytes = 0, p_bytes = 0;
  for (const auto& a : aj) a_bytes += 8.0 * a.len * a.n_out;
  for (const auto& p : pj) p_bytes += 16.0 * p.len * p.n_out;
  if (!fj.empty()) {
    {
      PhaseScope ps(c, RADMM_PHASE_FORWARD, a_bytes);
      forward<MODE_RHS>(c, fj, rj, h->beta, go);
    }
    {
      PhaseScope ps(c, RADMM_PHASE_GAPPLY, g_bytes);
      gapply(c, gq, go);
      std::vector<int> fin;  // lazy columns the G-apply just formed
      for (int q : gq)
        if (c->sensors[q].lz_new) {
          c->sensors[q].lz_new = 0;
          fin.push_back(q);
        }
      lazy_finish(c, fin, h->mu);
      lazy_correct(c, gq, h->mu, go);
      refine(c, gq, h->mu, go);
    }
    PhaseScope ps(c, RADMM_PHASE_ADJOINT, a_bytes);
    adjoint(c, aj, gq, h->mu, h->beta, go);  // gq lists the same dual sensors in the same order
  }
  if (n_rhs) {
    PhaseScope ps(c, RADMM_PHASE_PRIMAL, p_bytes);
    LAUNCH(c, rhs_kernel, dim3((rhs_max + 255) / 256, n_rhs), 256, 0, rh, c->gap.p, c->sigma.p, h->beta, go);
    coldot<double2, EPI_XPRIMAL>(c, pj, h->mu, h->beta, go);
  }
  ++c->upd;
}

// Sharded runs: every rank receives every sensor image (fixed global order)
// in ONE all-gather per iteration; the per-sensor active sizes, stall flags
// and notice bytes (records only) are gathered once at the end of the run
// (finish_sharded_records) -- or per iteration when an observer needs them.
// Images travel as complex128: s is a near-cancelling mean of the images in
// the degenerate BASELINE problems, so rounding them to
// complex64 would cost s its parity with the oracle.
void exchange(radmm_ctx* c, double notice_bytes, int k) {
  if (!c->sharded) return;
  const size_t N = c->N;
  PhaseScope ps(c, RADMM_PHASE_EXCHANGE, 16.0 * N * c->q_max_local * c->world);
  for (int q = 0; q < c->Q; ++q)
    CK(cudaMemcpyAsync(c->send_buf.p + (size_t)q * N, c->sensors[q].x_full.p, sizeof(double2) * N,
                       cudaMemcpyDeviceToDevice, c->stream));
  g_nccl.check(g_nccl.AllGather(c->send_buf.p, c->gathered.p, (size_t)c->q_max_local * N * 2, kNcclDouble, c->comm,
                                c->stream), "ncclAllGather(contributions)");
  g_nccl.settle(c->comm, "ncclAllGather(contributions)", c->nccl_timeout_ms);
  ++c->launches;
  if (!c->sync_meta) return;
  const size_t stride = 2 * (size_t)c->q_max_local + 1;
  double* meta = c->meta_host + (size_t)(k & 1) * stride;  // two slots: the copy of round k-1 may be in flight
  std::fill(meta, meta + stride, 0.0);
  for (int q = 0; q < c->Q; ++q) {
    meta[2 * q] = c->sensors[q].n_act;
    meta[2 * q + 1] = c->sensors[q].stalled ? 1.0 : 0.0;
  }
  meta[2 * c->q_max_local] = notice_bytes;
  CK(cudaMemcpyAsync(c->size_send.p, meta, sizeof(double) * stride, cudaMemcpyHostToDevice, c->stream));
  g_nccl.check(g_nccl.AllGather(c->size_send.p, c->size_recv.p, stride, kNcclDouble, c->comm, c->stream),
               "ncclAllGather(meta)");
  g_nccl.settle(c->comm, "ncclAllGather(meta)", c->nccl_timeout_ms);
  ++c->launches;
}

// Wait for a round's completion event; in sharded runs poll the NCCL
// communicator meanwhile, so a failed or vanished peer surfaces as
// RADMM_TRANSPORT within the timeout instead of a hang.
void wait_round(radmm_ctx* c, cudaEvent_t e) {
  if (!c->sharded || !g_nccl.GetAsyncError) {
    CK(cudaEventSynchronize(e));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t r = cudaEventQuery(e);
    if (r == cudaSuccess) return;
    if (r != cudaErrorNotReady) CK(r);
    int st = 0;
    if (g_nccl.GetAsyncError(c->comm, &st) != 0 || (st != 0 && st != kNcclInProgress)) {
      if (g_nccl.CommAbort) g_nccl.CommAbort(c->comm);
      c->comm = nullptr;
      fail(RADMM_TRANSPORT, std::string("NCCL asynchronous error during the iteration: ") +
                                (g_nccl.GetErrorString ? g_nccl.GetErrorString(st) : std::to_string(st)));
    }
    if (std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() >
        c->nccl_timeout_ms) {
      if (g_nccl.CommAbort) g_nccl.CommAbort(c->comm);
      c->comm = nullptr;
      fail(RADMM_TRANSPORT, "iteration did not complete within " + std::to_string(c->nccl_timeout_ms) +
                                " ms (a peer rank is gone or stalled)");
    }
    std::this_thread::yield();
  }
}

FusionArgs fusion_args(radmm_ctx* c, const radmm_hyperparams* h, int k);

void run_fusion(radmm_ctx* c, const radmm_hyperparams* h, int k, const int* go = nullptr,
                int* go_next = nullptr, int stop_on_converge = 1, int screen_next_possible = 0,
                int* screen_go = nullptr) {
  FusionArgs a = fusion_args(c, h, k);
  a.go = go;
  a.go_next = go_next;
  a.stop_on_converge = stop_on_converge;
  a.screen_next_possible = screen_next_possible;
  a.screen_go = screen_go;
  PhaseScope ps(c, RADMM_PHASE_FUSION, 16.0 * c->N * (c->Q_total + 7));
  LAUNCH(c, fusion_kernel, dim3((c->N + kFusionThreads - 1) / kFusionThreads), kFusionThreads, 0, a);
}

bool fused_enabled();

// SensorCore::screen for every local sensor (admm.hpp:134-159, run :380-386),
// device part: zeta, keep flags, compaction into the *_new buffers and the
// kept counts (mapped host slot `slot`).  Guarded (go, sgo) when it is
// enqueued behind a fusion round; go_next lets the next round run when no
// active set changes.  Returns false if the history is still short.
bool enqueue_screen(radmm_ctx* c, const radmm_hyperparams* h, int slot, const int* go, const int* sgo,
                    int* go_next) {
  if (c->upd < c->W) return false;  // history shorter than W+1 (admm.hpp:137)
  Pack<ScreenJob> pk;
  int n_max = 0;
  if (c->Q > kMaxBatch) fail(RADMM_INVALID_ARGUMENT, "too many sensors per GPU for screening batch");
  for (int q = 0; q < c->Q; ++q) {
    Sensor& S = c->sensors[q];
    ScreenJob j;
    j.n = S.n_act; j.J = S.J.p; j.ring = S.ring.p; j.ring_stride = c->N; j.first_slot = c->upd % c->W;
    j.keep = S.keep.p; j.block_counts = S.blk_cnt.p; j.block_offsets = S.blk_off.p; j.totals = S.totals.p;
    j.Jnew = S.Jnew.p; j.keep_pos = S.keep_pos.p; j.rem_pix = S.rem_pix.p; j.rem_pos = S.rem_pos.p;
    j.x_hat = S.x_hat.p; j.x_hat_new = S.x_hat_new.p;
    j.data = S.data.p; j.data_new = S.data_new.p;
    pk.j[q] = j;
    n_max = std::max(n_max, S.n_act);
  }
  const int nb = (n_max + kScanBlock - 1) / kScanBlock;
  double sb = 0;
  for (int q = 0; q < c->Q; ++q) sb += (double)c->sensors[q].n_act * (8.0 * c->W + 4 + 1 + 4 + 4 + 32);
  PhaseScope ps(c, RADMM_PHASE_SCREEN, sb);
  // one cluster launch (RADMM_SCREEN_FUSED=0 selects the three-kernel path)
  if (n_max <= kScreenCluster * kScanBlock * kScreenMaxE && env_int("RADMM_SCREEN_FUSED", 1) != 0) {
    LAUNCH(c, screen_fused_kernel, dim3(kScreenCluster, c->Q), kScanBlock, 0, pk, c->Q, c->W, h->screening_tol, go,
           sgo, c->d_totals + (size_t)slot * c->Q, go_next, c->screen_sync.p);
    return true;
  }
  LAUNCH(c, screen_flags_kernel, dim3(nb, c->Q), kScanBlock, 0, pk, c->W, h->screening_tol, go, sgo);
  LAUNCH(c, screen_scan_kernel, dim3(1), 256, 0, pk, c->Q, go, sgo, c->d_totals + (size_t)slot * c->Q, go_next);
  LAUNCH(c, screen_scatter_kernel, dim3(nb, c->Q), kScanBlock, 0, pk, go, sgo);
  return true;
}

// Host part, after the kept counts of slot `slot` are visible: stall flags,
// active-set swaps, removal log, then rebuild() (admm.hpp:171-179) as frozen
// echo + lagged data term + downdates.  Returns the notice bytes of the round.
uint64_t apply_screen(radmm_ctx* c, const radmm_hyperparams* h, int k, int slot) {
  const volatile int* tot = c->h_totals + (size_t)slot * c->Q;
  uint64_t notice = 0;
  std::vector<int> changed;
  int64_t log_need = c->log_used;
  for (int q = 0; q < c->Q; ++q) {
    Sensor& S = c->sensors[q];
    const int kept = tot[q];
    const int removed = S.n_act - kept;
    if (removed == 0) continue;
    if (kept == 0) {  // admm.hpp:148-151
      S.stalled = true;
      continue;
    }
    log_need += removed;
  }
  if (c->dlog.n < (size_t)log_need) {  // the removal log stays on the device until the run ends
    const size_t cap = std::max<size_t>((size_t)c->Q * c->N, (size_t)log_need);
    DArr<int> grown;
    grown.alloc(cap, false);
    if (c->log_used)
      CK(cudaMemcpyAsync(grown.p, c->dlog.p, sizeof(int) * c->log_used, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->dlog = std::move(grown);
  }
  std::vector<EventJob> ej;
  for (int q = 0; q < c->Q; ++q) {
    Sensor& S = c->sensors[q];
    const int kept = tot[q];
    const int removed = S.n_act - kept;
    if (removed == 0 || kept == 0) continue;
    S.removed_now = removed;
    S.v_ready = false;  // the speculative v was formed over the old active set
    std::swap(S.J, S.Jnew);
    std::swap(S.x_hat, S.x_hat_new);
    std::swap(S.data, S.data_new);
    S.n_act = kept;
    changed.push_back(q);
    notice += notice_size((size_t)removed);
    EventJob e{};
    e.rem_pix = S.rem_pix.p; e.r = removed; e.log_dst = c->dlog.p + c->log_used;
    ej.push_back(e);
    c->log_segs.push_back({k, c->q_begin + q, removed, c->log_used});
    c->log_used += removed;
  }
  if (changed.empty()) return notice;
  double rb = 0;
  for (int q : changed) {
    const Sensor& S = c->sensors[q];
    rb += 8.0 * S.rows * (S.n_act + S.removed_now) + (S.primal ? 32.0 * S.n_act * S.n_act : 48.0 * S.rows * S.rows);
  }
  PhaseScope ps(c, RADMM_PHASE_REFACTOR, rb);
  const bool trace = env_int("RADMM_TRACE_HOST", 0) != 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
  const auto h0 = now();
  update_y_eff(c, changed);
  const auto h1 = now();
  // dual sensors that stay dual keep a lagged data term (no full pass);
  // primal sensors (and the experimental fused sweeps) recompute it
  std::vector<int> exact;
  for (size_t t = 0; t < changed.size(); ++t) {
    Sensor& S = c->sensors[changed[t]];
    const bool stays_dual = !S.primal && S.n_act > S.rows;
    if (stays_dual && !fused_enabled()) {
      ej[t].bz = S.bz.p; ej[t].y_eff_s = S.y_eff_s.p; ej[t].y_eff = S.y_eff.p; ej[t].ld = S.ld; ej[t].beta = h->beta;
      S.data_lag = true;
    } else {
      exact.push_back(changed[t]);
    }
  }
  event_prep(c, ej);
  data_terms(c, exact, h->mu);
  const auto h2 = now();
  std::vector<int> rebuild, down;
  for (int q : changed) {
    Sensor& S = c->sensors[q];
    const bool now_primal = S.n_act <= S.rows;
    if (S.primal) {
      (S.removed_now <= S.n_act ? down : rebuild).push_back(q);
    } else if (now_primal) {
      rebuild.push_back(q);
    } else {
      (S.removed_now <= S.rows ? down : rebuild).push_back(q);
    }
  }
  for (int q : rebuild) snapshot_base(c, c->sensors[q], true);
  full_rebuild(c, rebuild, h->mu, h->beta);
  downdate(c, down, h->mu);
  if (trace) {
    const auto h3 = now();
    c->trace_us[0] += us(h0, h1);
    c->trace_us[1] += us(h1, h2);
    c->trace_us[2] += us(h2, h3);
    ++c->trace_n;
  }
  return notice;
}

// Synchronous screening (observer / sharded / fused / profiling runs).
uint64_t screen_all(radmm_ctx* c, const radmm_hyperparams* h, int k) {
  if (!enqueue_screen(c, h, 2, nullptr, nullptr, nullptr)) return 0;
  CK(cudaStreamSynchronize(c->stream));
  return apply_screen(c, h, k, 2);
}

// Stall flags of a screening round whose active sets did not change.
void note_stalls(radmm_ctx* c, int slot) {
  const volatile int* tot = c->h_totals + (size_t)slot * c->Q;
  for (int q = 0; q < c->Q; ++q)
    if (tot[q] == 0 && c->sensors[q].n_act > 0) c->sensors[q].stalled = true;
}

// ---- single-pass fused sweep (one GPU, all sensors dual, Q <= 8) ------------
int env_int(const char* name, int dflt) {
  // launch paths call this a few dozen times per round: a per-thread cache
  // keyed by the name literal's address answers without the lock while the
  // switch table is unchanged (generation counter)
  struct Hit { const char* name; int dflt; unsigned gen; int value; };
  thread_local Hit cache[64];
  thread_local int used = 0;
  const unsigned gen = g_tune_gen.load(std::memory_order_acquire);
  for (int i = 0; i < used; ++i)
    if (cache[i].name == name && cache[i].dflt == dflt) {
      if (cache[i].gen == gen) return cache[i].value;
      break;
    }
  int value;
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    const TuneEntry& t = tune_entry(name);
    value = t.api_set ? t.api_val : t.env_set ? t.env_val : dflt;
  }
  for (int i = 0; i < used; ++i)
    if (cache[i].name == name && cache[i].dflt == dflt) {
      cache[i].gen = gen;
      cache[i].value = value;
      return value;
    }
  if (used < 64) cache[used++] = Hit{name, dflt, gen, value};
  return value;
}

FusionArgs fusion_args(radmm_ctx* c, const radmm_hyperparams* h, int k) {
  FusionArgs a;
  a.contrib = c->contrib.p;
  a.Q = c->Q_total;
  a.N = c->N;
  a.s = c->s.p; a.xg = c->xg.p; a.sigma = c->sigma.p; a.sigma_pre = c->sigma_pre.p; a.gap = c->gap.p;
  a.beta = h->beta;
  a.kappa = h->lambda / h->beta;
  a.root_n_eps_abs = std::sqrt((double)c->N) * h->eps_abs;
  a.eps_rel = h->eps_rel;
  a.has_prev = k > 1 ? 1 : 0;
  a.iteration = k;
  a.partials = c->fpart.p;
  a.counter = c->fcounter.p;
  a.out_dev = c->fs_dev.p;
  a.out_host = c->fs_host_dev + (k & 1);  // two slots: round k+1 may finish before the host reads round k
  a.go = nullptr;
  a.go_next = nullptr;
  a.stop_on_converge = 1;
  a.screen_next_possible = 0;
  a.screen_go = nullptr;
  return a;
}

#if RADMM_EXPERIMENTAL
// ---- parked experiment: single-pass fused sweeps ------
// Compiled only with -DRADMM_EXPERIMENTAL=1 (__graft_entry__.build(experimental=True));
// every variant measured slower than the two-pass default, none carries the
// KM-space refinement, and the product library does not ship them.
constexpr int kDefaultSweepTile = 16;

// RADMM_FUSED: 0 = two-pass local updates (default), 1 = synchronous cluster
// sweep (v1), 2 = asynchronous warp-specialised sweep (v2).
int fused_version() { return env_int("RADMM_FUSED", 0); }

bool fused_enabled() { return fused_version() != 0; }

bool sweep3_eligible(radmm_ctx* c);

bool sweep4_eligible(radmm_ctx* c) {
  if (c->N % kS4P != 0 || c->sm_count / c->Q < 1) return false;
  for (const Sensor& S : c->sensors)
    if (S.n_act != c->N || S.primal || S.ld != c->sensors[0].ld || S.ld > 2048) return false;
  return true;
}

bool fused_eligible(radmm_ctx* c) {
  if (fused_version() == 4 || fused_version() == 5) return !c->sharded && sweep4_eligible(c);
  if (!fused_enabled() || c->sharded || c->Q < 1 || c->Q > 8) return false;
  if (fused_version() == 3 && !sweep3_eligible(c)) return false;
  for (const Sensor& S : c->sensors)
    if (S.primal || S.ld > 4 * 512) return false;
  return true;
}

template <int RPT>
void launch_sweep(radmm_ctx* c, const Pack<SweepJob>& pk, const FusionArgs& fa, const radmm_hyperparams* h,
                  size_t smem) {
  auto kern = fused_sweep_kernel<RPT>;
  if (smem > 48 * 1024) set_smem_attr((const void*)kern, (int)((int)smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)c->Q;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kSweepThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)c->Q);
  int clusters = 0;
  CK(cudaOccupancyMaxActiveClusters(&clusters, (void*)kern, &cfg));
  clusters = std::max(1, clusters);
  const int cap = env_int("RADMM_SWEEP_CLUSTERS", 0);
  if (cap > 0) clusters = std::min(clusters, cap);
  for (const Sensor& S : c->sensors) clusters = std::min(clusters, S.part_chunks);
  const int tile = std::max(8, std::min(kSweepTile, env_int("RADMM_SWEEP_TILE", kDefaultSweepTile)));
  const int prefetch = env_int("RADMM_SWEEP_PREFETCH", 1);
  const int range = (int)round_up((c->N + clusters - 1) / clusters, tile);
  clusters = (c->N + range - 1) / range;
  cfg.gridDim = dim3((unsigned)(c->Q * clusters));
  // the fusion partials hold one slot per block of the grid
  if (c->fpart.n < (size_t)5 * c->Q * clusters) c->fpart.alloc((size_t)5 * c->Q * clusters);
  FusionArgs a = fa;
  a.partials = c->fpart.p;
  if (env_int("RADMM_DEBUG", 0))
    std::fprintf(stderr, "[radmm] sweep1: clusters=%d grid=%d smem=%zu range=%d tile=%d\n", clusters,
                 c->Q * clusters, smem, range, tile);
  CK(cudaLaunchKernelEx(&cfg, kern, pk, a, h->mu, h->beta, clusters, range, tile, prefetch));
  ++c->launches;
  c->sweep_clusters = clusters;
}

template <int RPT>
void launch_sweep2(radmm_ctx* c, const Pack<SweepJob>& pk, const FusionArgs& fa, const radmm_hyperparams* h,
                   int64_t ld_max) {
  auto kern = fused_sweep2_kernel<RPT>;
  const int tile = std::max(2, std::min(64, env_int("RADMM_SWEEP_TILE", 16)));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)c->Q;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kS2Threads);
  cfg.stream = c->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3((unsigned)c->Q);
  // smem: w (ld complex) + tile table of the largest range (one cluster: N)
  size_t smem = (size_t)ld_max * sizeof(double2) + sizeof(int) * ((size_t)c->N / tile + 2);
  set_smem_attr((const void*)kern, (int)((int)std::min<size_t>(smem, 200 * 1024)));
  cfg.dynamicSmemBytes = std::min<size_t>(smem, 200 * 1024);
  int clusters = 0;
  CK(cudaOccupancyMaxActiveClusters(&clusters, (void*)kern, &cfg));
  clusters = std::max(1, clusters);
  const int cap = env_int("RADMM_SWEEP_CLUSTERS", 0);
  if (cap > 0) clusters = std::min(clusters, cap);
  for (const Sensor& S : c->sensors) clusters = std::min(clusters, S.part_chunks);
  const int range = (int)round_up((c->N + clusters - 1) / clusters, tile);
  clusters = (c->N + range - 1) / range;
  smem = (size_t)ld_max * sizeof(double2) + sizeof(int) * ((size_t)range / tile + 2);
  if (smem > 200 * 1024) fail(RADMM_INVALID_ARGUMENT, "fused sweep: tile table exceeds shared memory");
  set_smem_attr((const void*)kern, (int)((int)smem));
  cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3((unsigned)(c->Q * clusters));
  if (c->fpart.n < (size_t)5 * c->Q * clusters) c->fpart.alloc((size_t)5 * c->Q * clusters);
  FusionArgs a = fa;
  a.partials = c->fpart.p;
  if (env_int("RADMM_DEBUG", 0))
    std::fprintf(stderr, "[radmm] sweep2: clusters=%d grid=%d block=%d smem=%zu range=%d tile=%d\n", clusters,
                 c->Q * clusters, kS2Threads, smem, range, tile);
  CK(cudaLaunchKernelEx(&cfg, kern, pk, a, h->mu, h->beta, range, tile));
  ++c->launches;
  c->sweep_clusters = clusters;
}

bool sweep3_eligible(radmm_ctx* c) {
  if (c->Q > kS3Q) return false;
  for (const Sensor& S : c->sensors) {
    if (S.primal || S.ld != c->sensors[0].ld) return false;
    if (S.ld % kS3R != 0 || S.ld / kS3R > kS3Threads || S.ld / kS3R < 64) return false;
  }
  return true;
}

void launch_sweep4(radmm_ctx* c, const Pack<SweepJob>& sp, const FusionArgs& fa, const radmm_hyperparams* h) {
  const int64_t ld = c->sensors[0].ld;
  const int ntiles = c->N / kS4P;
  int chunks = std::max(1, c->sm_count / c->Q);
  for (const Sensor& S : c->sensors) chunks = std::min(chunks, S.part_chunks);
  const int tpc = (ntiles + chunks - 1) / chunks;
  chunks = (ntiles + tpc - 1) / tpc;
  if (c->s4_cnt.n < (size_t)ntiles) {
    c->s4_cnt.alloc(ntiles);
    c->s4_flag.alloc(ntiles);
    c->s4_norms.alloc((size_t)5 * ntiles, false);
  }
  if (c->s4_done.n < 1) c->s4_done.alloc(1);
  Pack<Sweep4Job> pk;
  for (int q = 0; q < c->Q; ++q) {
    const SweepJob& j = sp.j[q];
    pk.j[q] = Sweep4Job{j.A, j.w, j.data, j.rhs, j.x_hat, j.x_full, j.ring_slot, j.part};
  }
  const bool v5 = fused_version() == 5;
  if (v5 && c->xg_alt.n < (size_t)c->N) {
    c->xg_alt.alloc(c->N);
    c->sigma_alt.alloc(c->N);
  }
  Sweep4Ctl ctl{c->s4_cnt.p, c->s4_flag.p, c->s4_norms.p, c->s4_done.p, ++c->s4_seq, tpc,
                v5 ? c->xg_alt.p : nullptr, v5 ? c->sigma_alt.p : nullptr};
  const size_t smem = (size_t)ld * sizeof(double2) + (size_t)kS4Slots * kS4P * ld * sizeof(float2) +
                      kS4Slots * sizeof(uint64_t);
  set_smem_attr((const void*)fused_sweep4_kernel, (int)((int)smem));
  double mu = h->mu, beta = h->beta;
  int64_t ldv = ld;
  void* args[] = {(void*)&pk, (void*)&fa, (void*)&ctl, (void*)&mu, (void*)&beta, (void*)&ldv};
  if (env_int("RADMM_DEBUG", 0))
    std::fprintf(stderr, "[radmm] sweep4: chunks=%d tiles/chunk=%d grid=%dx%d smem=%zu\n", chunks, tpc, chunks,
                 c->Q, smem);
  if (fused_version() == 5) {
    const size_t smem5 = (size_t)ld * sizeof(double2) + (size_t)kS5Slots * kS4P * ld * sizeof(float2) +
                         2 * kS5Slots * sizeof(uint64_t);
    set_smem_attr((const void*)fused_sweep5_kernel, (int)((int)smem5));
    CK(cudaLaunchCooperativeKernel((void*)fused_sweep5_kernel, dim3((unsigned)chunks, (unsigned)c->Q),
                                   dim3(kS5Threads), args, smem5, c->stream));
    std::swap(c->xg, c->xg_alt);  // the round's new x_G / sigma
    std::swap(c->sigma, c->sigma_alt);
  } else {
    CK(cudaLaunchCooperativeKernel((void*)fused_sweep4_kernel, dim3((unsigned)chunks, (unsigned)c->Q),
                                   dim3(kS4Threads), args, smem, c->stream));
  }
  ++c->launches;
  c->sweep_clusters = chunks;
}

void launch_sweep3(radmm_ctx* c, const Pack<SweepJob>& sp, const FusionArgs& fa, const radmm_hyperparams* h) {
  const int64_t ld = c->sensors[0].ld;
  const int sl = (int)(ld / kS3R);
  Pack<Sweep3Job> pk;
  for (int q = 0; q < c->Q; ++q) {
    const SweepJob& s = sp.j[q];
    pk.j[q] = Sweep3Job{s.A, s.J, s.n_act, s.w, s.data, s.rhs, s.x_hat, s.x_full, s.ring_slot, s.part};
  }
  const size_t base = 2ull * kS3Cols * sl * sizeof(float2) + (size_t)c->Q * sl * sizeof(double2);
  // per-sensor tile tables: sized for >= 8 clusters, re-checked below
  const size_t tab_est = sizeof(int) * (size_t)c->Q * ((c->N + 8 * kS3P - 1) / (8 * kS3P) + 2);
  size_t smem = base + tab_est;
  set_smem_attr((const void*)fused_sweep3_kernel, (int)((int)smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kS3R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kS3Threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(kS3R);
  int clusters = 0;
  CK(cudaOccupancyMaxActiveClusters(&clusters, (void*)fused_sweep3_kernel, &cfg));
  clusters = std::max(1, clusters);
  const int cap = env_int("RADMM_SWEEP_CLUSTERS", 0);
  if (cap > 0) clusters = std::min(clusters, cap);
  for (const Sensor& S : c->sensors) clusters = std::min(clusters, S.part_chunks);
  const int range = (int)round_up((c->N + clusters - 1) / clusters, kS3P);
  clusters = (c->N + range - 1) / range;
  const size_t tab = sizeof(int) * (size_t)c->Q * (range / kS3P + 2);
  if (tab > tab_est) {
    smem = base + tab;
    if (smem > 227 * 1024) fail(RADMM_INVALID_ARGUMENT, "fused sweep v3: tile tables exceed shared memory");
    set_smem_attr((const void*)fused_sweep3_kernel, (int)((int)smem));
    cfg.dynamicSmemBytes = smem;
  }
  cfg.gridDim = dim3((unsigned)(kS3R * clusters));
  if (c->fpart.n < (size_t)5 * kS3R * clusters) c->fpart.alloc((size_t)5 * kS3R * clusters);
  FusionArgs a = fa;
  a.partials = c->fpart.p;
  if (env_int("RADMM_DEBUG", 0))
    std::fprintf(stderr, "[radmm] sweep3: clusters=%d grid=%d smem=%zu range=%d sl=%d\n", clusters,
                 kS3R * clusters, smem, range, sl);
  CK(cudaLaunchKernelEx(&cfg, fused_sweep3_kernel, pk, a, h->mu, h->beta, ld, range));
  ++c->launches;
  c->sweep_clusters = clusters;
}


// One iteration on the fused path: v for every sensor (left by the previous
// sweep, or a fresh forward pass after an active-set change / at k = 1), the
// capacitance-inverse apply, then the sweep (x-update, fusion, next forward).
void fused_iteration(radmm_ctx* c, const radmm_hyperparams* h, int k) {
  const int slot = c->upd % c->W;
  std::vector<FwdJob> fj;
  std::vector<ReduceJob> rj_fwd;
  Pack<ReduceJob> rj_sweep;
  int n_ready = 0;
  int64_t ld_max = 0;
  std::vector<int> gq;
  Pack<SweepJob> sp;
  double a_bytes = 0, g_bytes = 0, f_bytes = 0;
  for (int q = 0; q < c->Q; ++q) {
    Sensor& S = c->sensors[q];
    ld_max = std::max(ld_max, S.ld);
    if (!S.v_ready) {
      FwdJob f{};
      f.A = S.A.p; f.ld = S.ld; f.n = S.n_act; f.J = S.J.p; f.data = S.data.p; f.x_hat = S.x_hat.p;
      f.rhs_out = S.rhs.p; f.part = S.part.p;
      plan_chunks(c, S, S.n_act, c->Q, f.n_chunks, f.chunk_len);
      fj.push_back(f);
      rj_fwd.push_back(ReduceJob{S.part.p, f.n_chunks, S.ld, S.rows, nullptr, S.v.p, 1.0});
      f_bytes += 8.0 * S.rows * S.n_act;
    } else {
      rj_sweep.j[n_ready++] = ReduceJob{S.part.p, c->sweep_clusters, S.ld, S.rows, nullptr, S.v.p, 1.0};
    }
    gq.push_back(q);
    g_bytes += gapply_bytes(S.rows);
    a_bytes += 8.0 * S.rows * S.n_act;
    sp.j[q] = SweepJob{S.A.p, S.ld, S.n_act, S.J.p, S.w.p, S.data.p, S.rhs.p, S.x_hat.p, S.x_full.p,
                       S.ring.p + (size_t)slot * c->N, S.part.p};
  }
  {
    PhaseScope ps(c, RADMM_PHASE_FORWARD, f_bytes);
    if (!fj.empty()) forward<MODE_RHS>(c, fj, rj_fwd, h->beta);
    if (n_ready)
      LAUNCH(c, reduce_parts_kernel, dim3((unsigned)((ld_max + 255) / 256), n_ready), 256, 0, rj_sweep, nullptr);
  }
  {
    PhaseScope ps(c, RADMM_PHASE_GAPPLY, g_bytes);
    gapply(c, gq);
  }
  {
    PhaseScope ps(c, RADMM_PHASE_SWEEP, a_bytes + 16.0 * c->N * (c->Q + 7));
    const size_t smem = (size_t)ld_max * sizeof(double2) + kSweepTile * (sizeof(double2) + sizeof(int));
    const FusionArgs fa = fusion_args(c, h, k);
    if (fused_version() == 4 || fused_version() == 5) {
      launch_sweep4(c, sp, fa, h);
    } else if (fused_version() == 3) {
      launch_sweep3(c, sp, fa, h);
    } else if (fused_version() == 2) {
      if (ld_max <= 256) launch_sweep2<1>(c, sp, fa, h, ld_max);
      else if (ld_max <= 512) launch_sweep2<2>(c, sp, fa, h, ld_max);
      else if (ld_max <= 1024) launch_sweep2<4>(c, sp, fa, h, ld_max);
      else launch_sweep2<8>(c, sp, fa, h, ld_max);
    } else if (ld_max <= 512) {
      launch_sweep<1>(c, sp, fa, h, smem);
    } else if (ld_max <= 1024) {
      launch_sweep<2>(c, sp, fa, h, smem);
    } else {
      launch_sweep<4>(c, sp, fa, h, smem);
    }
  }
  for (Sensor& S : c->sensors) S.v_ready = true;
  ++c->upd;
}

#else
bool fused_enabled() { return false; }
bool fused_eligible(radmm_ctx*) { return false; }
void fused_iteration(radmm_ctx*, const radmm_hyperparams*, int) {
  fail(RADMM_INVALID_ARGUMENT, "fused sweeps are an experiment: build with RADMM_EXPERIMENTAL=1");
}
#endif  // RADMM_EXPERIMENTAL

void build_contrib(radmm_ctx* c) {
  std::vector<const double2*> ptrs(c->Q_total);
  if (!c->sharded) {
    for (int q = 0; q < c->Q; ++q) ptrs[q] = c->sensors[q].x_full.p;
  } else {
    for (int g = 0; g < c->Q_total; ++g) {
      int r = 0;
      while (r + 1 < c->world && (int64_t)(r + 1) * c->Q_total / c->world <= g) ++r;
      const int begin = (int)((int64_t)r * c->Q_total / c->world);
      ptrs[g] = c->gathered.p + ((size_t)r * c->q_max_local + (g - begin)) * c->N;
    }
  }
  if (c->contrib.n != ptrs.size()) c->contrib.alloc(ptrs.size());
  CK(cudaMemcpyAsync(c->contrib.p, ptrs.data(), sizeof(void*) * ptrs.size(), cudaMemcpyHostToDevice, c->stream));
}

// Record one round (admm.hpp:397-420): residuals, per-sensor active sizes
// (after this round's screening), bytes_sent, active_fraction, stall flag.
void record_round(radmm_ctx* c, int k, const FusionScalars& f, uint64_t notice, radmm_run_summary& sm,
                  std::vector<int32_t>& sizes, std::vector<double>& meta_all,
                  std::chrono::steady_clock::time_point t1) {
  radmm_iteration_record rec{};
  rec.iteration = k;
  rec.pri_res = f.pri_res;
  rec.dual_res = f.dual_res;
  rec.eps_pri = f.eps_pri;
  rec.eps_dual = f.eps_dual;
  uint64_t bytes = notice;
  bool stalled_any = false;
  if (!c->sharded) {
    for (int q = 0; q < c->Q; ++q) {
      sizes[q] = c->sensors[q].n_act;
      stalled_any = stalled_any || c->sensors[q].stalled;
    }
  } else if (!c->sync_meta) {
    // local view now (rank-local sensors), the global records at the end of
    // the run (finish_sharded_records): no per-iteration host round trip
    const size_t stride = 2 * (size_t)c->q_max_local + 1;
    const size_t base = c->shard_meta.size();
    c->shard_meta.resize(base + stride, 0.0);
    for (int q = 0; q < c->Q; ++q) {
      c->shard_meta[base + 2 * q] = c->sensors[q].n_act;
      c->shard_meta[base + 2 * q + 1] = c->sensors[q].stalled ? 1.0 : 0.0;
    }
    c->shard_meta[base + 2 * c->q_max_local] = (double)notice;
    rec.bytes_sent = notice;
    rec.ms_elapsed = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
    c->records.push_back(rec);
    return;
  } else {
    // observer runs: this round's metadata all-gather completed with END(k)
    const int stride = 2 * c->q_max_local + 1;
    meta_all.resize((size_t)stride * c->world);
    CK(cudaMemcpyAsync(meta_all.data(), c->size_recv.p, sizeof(double) * meta_all.size(), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    bytes = 0;
    for (int r = 0; r < c->world; ++r) {
      const int begin = (int)((int64_t)r * c->Q_total / c->world);
      const int end = (int)((int64_t)(r + 1) * c->Q_total / c->world);
      for (int g = begin; g < end; ++g) {
        sizes[g] = (int32_t)meta_all[(size_t)r * stride + 2 * (g - begin)];
        stalled_any = stalled_any || meta_all[(size_t)r * stride + 2 * (g - begin) + 1] != 0.0;
      }
      bytes += (uint64_t)meta_all[(size_t)r * stride + 2 * c->q_max_local];
    }
  }
  int max_active = 0;
  for (int g = 0; g < c->Q_total; ++g) {
    const size_t cb = contribution_size((size_t)sizes[g]);
    bytes += cb;
    max_active = std::max(max_active, sizes[g]);
    sm.total_active_solves += (uint64_t)sizes[g];
    c->active_log.push_back(sizes[g]);
  }
  rec.bytes_sent = bytes;
  rec.active_fraction = (double)max_active / c->N;
  rec.ms_elapsed = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
  sm.total_bytes += bytes;
  c->records.push_back(rec);
  sm.screening_stalled = stalled_any ? 1 : 0;
}

// Sharded runs without an observer: one all-gather of every rank's
// per-iteration metadata at the end of the run, then the records' global
// fields (admm.hpp:397-420) exactly as the per-iteration path computes them.
void finish_sharded_records(radmm_ctx* c, radmm_run_summary& sm) {
  if (!c->sharded || c->sync_meta) return;
  const size_t stride = 2 * (size_t)c->q_max_local + 1, K = c->records.size();
  if (K == 0) return;
  DArr<double> dsend, drecv;
  dsend.alloc(K * stride, false);
  drecv.alloc(K * stride * c->world, false);
  CK(cudaMemcpyAsync(dsend.p, c->shard_meta.data(), sizeof(double) * K * stride, cudaMemcpyHostToDevice, c->stream));
  g_nccl.check(g_nccl.AllGather(dsend.p, drecv.p, K * stride, kNcclDouble, c->comm, c->stream),
               "ncclAllGather(records)");
  g_nccl.settle(c->comm, "ncclAllGather(records)", c->nccl_timeout_ms);
  std::vector<double> all(K * stride * c->world);
  CK(cudaMemcpyAsync(all.data(), drecv.p, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->active_log.clear();
  sm.total_active_solves = 0;
  sm.total_bytes = 0;
  bool stalled_any = false;
  for (size_t k = 0; k < K; ++k) {
    uint64_t bytes = 0;
    int max_active = 0;
    for (int r = 0; r < c->world; ++r) {
      const double* m = all.data() + ((size_t)r * K + k) * stride;
      const int begin = (int)((int64_t)r * c->Q_total / c->world);
      const int end = (int)((int64_t)(r + 1) * c->Q_total / c->world);
      bytes += (uint64_t)m[2 * c->q_max_local];
      for (int g = begin; g < end; ++g) {
        const int32_t sz = (int32_t)m[2 * (g - begin)];
        stalled_any = stalled_any || m[2 * (g - begin) + 1] != 0.0;
        bytes += contribution_size((size_t)sz);
        max_active = std::max(max_active, (int)sz);
        sm.total_active_solves += (uint64_t)sz;
        c->active_log.push_back(sz);
      }
    }
    c->records[k].bytes_sent = bytes;
    c->records[k].active_fraction = (double)max_active / c->N;
    sm.total_bytes += bytes;
  }
  sm.screening_stalled = stalled_any ? 1 : 0;
}

// Removal log: one D2H of the device log at the end of a run, expanded into
// (iteration, sensor, pixel) triples.
void finish_removal_log(radmm_ctx* c) {
  if (c->log_used) {
    std::vector<int> pix((size_t)c->log_used);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(pix.data(), c->dlog.p, sizeof(int) * pix.size(), cudaMemcpyDeviceToHost));
    for (const auto& sg : c->log_segs)
      for (int i = 0; i < sg.count; ++i) {
        c->removal_log.push_back(sg.k);
        c->removal_log.push_back(sg.q);
        c->removal_log.push_back(pix[(size_t)sg.off + i]);
      }
  }
  c->log_segs.clear();
  c->log_used = 0;
}

void do_run(radmm_ctx* c, const radmm_hyperparams* h, const radmm_run_options* o, radmm_run_summary* out) {
  validate_hyper(h);
  set_device(c);
  const bool asadmm = o && o->mode == RADMM_MODE_ASADMM;
  const bool disable = o && o->disable_screening;
  const bool fixed = o && o->fixed_iterations;
  c->records.clear();
  c->active_log.clear();
  c->removal_log.clear();
  c->log_segs.clear();
  c->log_used = 0;
  c->pending_fail = 0;
  c->have_result = false;
  c->launches = 0;
  c->rebuilds = c->downdates = 0;
  c->refine = !(o && o->skip_refinement);
  c->refine_skipped = 0;
  c->iter_ms.clear();
  c->iter_launches.clear();
  c->marks.clear();
  c->ev_used = 0;
  for (int i = 0; i < RADMM_PHASE_COUNT; ++i) {
    c->prof_ms[i] = c->prof_bytes[i] = 0;
    c->prof_launches[i] = c->prof_calls[i] = 0;
  }
  if (!c->ev_it0) {
    CK(cudaEventCreate(&c->ev_it0));
    CK(cudaEventCreate(&c->ev_it1));
  }
  radmm_run_summary sm{};
  const auto t0 = std::chrono::steady_clock::now();
  build_contrib(c);
  begin_run(c, h);
  CK(cudaStreamSynchronize(c->stream));
  const auto t1 = std::chrono::steady_clock::now();
  sm.setup_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  std::vector<double> hx, hs, hsig;
  std::vector<int32_t> sizes(c->Q_total);
  std::vector<double> meta_all;
  if (o && o->observer) { hx.resize(2 * (size_t)c->N); hs.resize(2 * (size_t)c->N); hsig.resize(2 * (size_t)c->N); }
  bool staged_trigger = false;
  FusionScalars f{};
  // step boundaries: STEP(k-1) is recorded when iteration k starts, so
  // elapsed(STEP(k-1), STEP(k)) is the device-clock wall time of iteration k
  // including the host round trip before iteration k+1.  Both live in small
  // rings (creating an event per possible iteration cost ~0.1 s per run);
  // iteration k's time is read one iteration later, when both are complete.
  constexpr int kEvRing = 4;
  while (c->ev_steps.size() < (size_t)kEvRing) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->ev_steps.push_back(e);
  }
  c->iter_busy_ms.clear();
  while (c->ev_ends.size() < (size_t)kEvRing) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->ev_ends.push_back(e);
  }
  auto STEP = [&](int i) { return c->ev_steps[i % kEvRing]; };
  auto END = [&](int i) { return c->ev_ends[i % kEvRing]; };
  auto step_time = [&](int it) {  // iteration it (>= 1): STEP(it-1) .. STEP(it), both complete
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, STEP(it - 1), STEP(it)));
    c->iter_ms.push_back(ms);
  };
  // Device-guarded speculation: while iteration k runs, iteration k+1 is
  // already enqueued; its kernels run only if fusion_k set go[(k+1)&1] (not
  // converged, and no screening staged).  Otherwise they exit at entry and
  // the host re-issues k+1 after screening.  Off for observers / profiling /
  // sharded or fused runs.
  // Sharded runs speculate too: every host decision below depends only on the
  // fusion scalars, which are bitwise identical on all ranks, so every rank
  // issues the same rounds (one all-gather each) -- except the pre-enqueued
  // screening, whose "did any set change" is rank-local: sharded runs screen
  // the synchronous way (screen_all) instead.
  const bool spec = !(o && o->observer) && !fused_enabled() && !c->profiling && env_int("RADMM_SPECULATE", 1) != 0;
  c->sync_meta = c->sharded && o && o->observer;
  if (c->sync_meta && !c->meta_host) {
    c->meta_bytes = pinned_class(2 * sizeof(double) * (2 * (size_t)c->q_max_local + 1));
    c->meta_host = reinterpret_cast<double*>(pinned_get(c->meta_bytes));
  }
  c->shard_meta.clear();
  auto screen_next_possible = [&]() { return (asadmm && !disable && c->upd >= c->W) ? 1 : 0; };
  // issue one round: local updates (+ exchange) + fusion; go == nullptr = unconditional
  // With speculation the next round's screening is enqueued right behind this
  // round's fusion, guarded by the flag the fusion writes; the host then reads
  // the kept counts at the same sync as the round's scalars (no extra round
  // trip), and a screening round that changes no active set does not even
  // cancel the speculative round.
  constexpr double kPreScreenRatio = 8.0;
  bool trigger_seen = false;
  double last_ratio = 1e300;  // pri_res / eps_pri of the last completed round
  auto issue = [&](int kk, const int* go, uint64_t notice) {
    int* go_next = spec ? c->go_flags.p + ((kk + 1) & 1) : nullptr;
    c->pre_screened[kk & 1] = false;
    if (fused_eligible(c)) {
      fused_iteration(c, h, kk);
    } else {
      local_updates(c, h, go);
      exchange(c, (double)notice, kk);
      const int snp = screen_next_possible();
      // the guarded screening is enqueued only when the trigger is near: the
      // last observed primal residual within kPreScreenRatio of its
      // threshold, or the trigger seen already.  Otherwise (C2's long
      // approach) the three guarded launches are skipped; if the trigger does
      // fire, the speculative round is cancelled and screening runs the
      // synchronous way (screen_all) -- same result.
      const bool near = trigger_seen || last_ratio <= kPreScreenRatio;
      int* sgo = (spec && snp && near && !c->sharded) ? c->sgo_flags.p + (kk & 1) : nullptr;
      run_fusion(c, h, kk, go, go_next, fixed ? 0 : 1, snp, sgo);
      if (sgo) c->pre_screened[kk & 1] = enqueue_screen(c, h, kk & 1, go, sgo, go_next);
    }
    CK(cudaEventRecord(END(kk), c->stream));
  };
  // active sets changed by the screening enqueued behind round kk
  auto pre_changed = [&](int kk) {
    const volatile int* tot = c->h_totals + (size_t)(kk & 1) * c->Q;
    for (int q = 0; q < c->Q; ++q)
      if (tot[q] != 0 && tot[q] != c->sensors[q].n_act) return true;
    return false;
  };
  bool k_launched = false;   // iteration k already enqueued (speculatively)
  bool prev_event = false;   // the screening before the current round changed an active set
  const int spec_after_event = env_int("RADMM_SPEC_AFTER_EVENT", 0);
  const bool trace_host = env_int("RADMM_TRACE_HOST", 0) != 0;  // host time of re-issued rounds (stderr)
  double host_ev_us = 0, host_issue_us = 0;
  int host_n = 0;
  int64_t l_k = 0;           // launch counter when iteration k was enqueued
  uint64_t notice_k = 0;
  // PDL inside the iteration loop only (iterations, screening, events): the
  // setup kernels (Gram, Gauss-Jordan, Ozaki) measured ~2 ms slower with it
  struct PdlScope {
    radmm_ctx* c;
    explicit PdlScope(radmm_ctx* cc) : c(cc) { c->pdl = env_int("RADMM_PDL", 1) != 0; }
    ~PdlScope() { c->pdl = false; }
  } pdl_scope(c);
  for (int k = 1; k <= h->max_iter; ++k) {
    if (!k_launched) {
      const auto tt0 = std::chrono::steady_clock::now();
      l_k = c->launches;
      CK(cudaEventRecord(STEP(k - 1), c->stream));
      notice_k = 0;
      if (asadmm && !disable && staged_trigger)
        notice_k = c->pre_screened[(k - 1) & 1] ? apply_screen(c, h, k, (k - 1) & 1) : screen_all(c, h, k);
      prev_event = notice_k > 0;
      const auto tt1 = std::chrono::steady_clock::now();
      issue(k, nullptr, notice_k);
      if (trace_host) {
        const auto tt2 = std::chrono::steady_clock::now();
        host_ev_us += std::chrono::duration<double, std::micro>(tt1 - tt0).count();
        host_issue_us += std::chrono::duration<double, std::micro>(tt2 - tt1).count();
        ++host_n;
      }
    }
    const uint64_t notice = notice_k;
    const int64_t l0 = l_k;
    const int64_t l_end = c->launches;
    // Right after an elimination event the next screening most likely changes
    // a set again (C4: 382 of 400 rounds), and a speculative round would only
    // be cancelled -- a dozen no-op launches on the device.  Skip it then: the
    // pre-enqueued screening still runs behind this round's fusion.
    bool spec_next = spec && k < h->max_iter && !(prev_event && spec_after_event == 0);
    int upd_before_next = c->upd;
    if (spec_next) {
      l_k = c->launches;
      CK(cudaEventRecord(STEP(k), c->stream));
      issue(k + 1, c->go_flags.p + ((k + 1) & 1), 0);
    }
    wait_round(c, END(k));
    check_deferred(c);             // pivots of a downdate issued before iteration k
    if (k >= 2) step_time(k - 1);  // STEP(k-1) precedes iteration k's kernels: complete
    c->iter_launches.push_back(l_end - l0);
    flush_marks(c);
    f = c->fs_host[k & 1];
    k_launched = false;
    if (spec_next) {
      const bool screens = f.trigger && asadmm && !disable && upd_before_next >= c->W;
      // the screening behind round k ran on the device; it cancelled round
      // k+1 only if an active set changed
      const bool pre = screens && c->pre_screened[k & 1];
      const bool cancelled = (!fixed && f.converged) || (screens && (!pre || pre_changed(k)));
      if (cancelled) {
        // the cancelled round's kernels exit at entry; what the host enqueues
        // next runs after them in stream order
        c->upd = upd_before_next;  // the no-op round consumed no update
        for (Sensor& S : c->sensors) S.v_ready = false;
      } else {
        if (pre) note_stalls(c, k & 1);
        k_launched = true;
        notice_k = 0;
      }
    }
    record_round(c, k, f, notice, sm, sizes, meta_all, t1);
    trigger_seen = trigger_seen || f.trigger;
    last_ratio = f.eps_pri > 0 ? f.pri_res / f.eps_pri : 1e300;
    if (o && o->observer) {
      CK(cudaMemcpy(hx.data(), c->xg.p, sizeof(double2) * c->N, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(hs.data(), c->s.p, sizeof(double2) * c->N, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(hsig.data(), c->sigma.p, sizeof(double2) * c->N, cudaMemcpyDeviceToHost));
      radmm_iteration_view view{k, hx.data(), hs.data(), hsig.data(), sizes.data(), f.converged, f.trigger};
      o->observer(o->observer_user, &view);
    }
    sm.iterations = k;
    if (f.converged && !fixed) {
      sm.converged = 1;
      break;
    }
    staged_trigger = f.trigger != 0;
  }
  if (fixed) sm.converged = f.converged;
  if (trace_host && host_n) {
    std::fprintf(stderr, "[radmm host] %d re-issued rounds: events %.1f us, issue %.1f us per round\n", host_n,
                 host_ev_us / host_n, host_issue_us / host_n);
    if (c->trace_n)
      std::fprintf(stderr,
                   "[radmm host] %d events: frozen echo %.1f us, bookkeeping launch %.1f us, downdates %.1f us "
                   "(lazy append: prep %.1f, item table %.1f, column passes %.1f, border %.1f)\n",
                   c->trace_n, c->trace_us[0] / c->trace_n, c->trace_us[1] / c->trace_n, c->trace_us[2] / c->trace_n,
                   c->trace_us[3] / c->trace_n, c->trace_us[4] / c->trace_n, c->trace_us[5] / c->trace_n,
                   c->trace_us[6] / c->trace_n);
    for (double& t : c->trace_us) t = 0;
    c->trace_n = 0;
  }
  CK(cudaEventRecord(STEP(sm.iterations), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  check_deferred(c);
  finish_removal_log(c);
  finish_sharded_records(c, sm);
  if (sm.iterations >= 1) step_time(sm.iterations);
  const auto t2 = std::chrono::steady_clock::now();
  sm.solve_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
  sm.kernel_launches = c->launches;
  sm.rebuilds = c->rebuilds;
  sm.downdates = c->downdates;
  sm.refine_skipped = c->refine ? c->refine_skipped : 0;
  c->summary = sm;
  c->have_result = true;
  if (out) *out = sm;
}

// ---- multi-frame batches (BASELINE config 5) ---------------------------------
// Frame f of a context is a child context that views the parent's operators
// (no copy) and uses the parent's stream; everything that depends on the
// frame's measurements (y, active sets, factor, ADMM state, records) is its
// own.  run_frames drives all frames in lockstep; each frame follows the
// reference loop (admm.hpp:357-445) to its own stopping rule, exactly as a
// run of that frame alone would.
radmm_ctx* frame_ctx(radmm_ctx* p, int f) {
  if (!p) fail(RADMM_INVALID_ARGUMENT, "null context");
  if (p->parent) fail(RADMM_INVALID_ARGUMENT, "frame contexts cannot hold frames");
  if (p->sharded) fail(RADMM_INVALID_ARGUMENT, "multi-frame batches need an unsharded context");
  if (f < 0 || f >= 4096) fail(RADMM_INVALID_ARGUMENT, "frame index out of range");
  while ((int)p->frames.size() <= f) {
    for (int q = 0; q < p->Q; ++q)
      if (!p->sensors[q].has_op)
        fail(RADMM_INVALID_ARGUMENT, "Problem: sensor " + std::to_string(q) + " has no operator");
    auto ch = std::make_unique<radmm_ctx>();
    init_ctx(ch.get(), p->device, p->N, p->Q);
    CK(cudaStreamDestroy(ch->stream));
    ch->stream = p->stream;
    ch->own_stream = false;
    ch->parent = p;
    ch->Q_total = p->Q_total;
    ch->q_begin = 0;
    ch->q_max_local = p->Q;
    for (int q = 0; q < p->Q; ++q) {
      Sensor& S = ch->sensors[q];
      Sensor& P = p->sensors[q];
      S.rows = P.rows;
      S.ld = P.ld;
      S.A.view(P.A.p, P.A.n);
      S.y_eff.alloc(S.ld);
      S.y_eff_s.alloc(S.ld);
      S.bz.alloc(S.ld);
      S.v.alloc(S.ld);
      S.w.alloc(S.ld);
      S.part_chunks = P.part_chunks;
      S.part.alloc((size_t)S.part_chunks * S.ld, false);
      S.has_op = true;
    }
    p->frames.push_back(std::move(ch));
  }
  return p->frames[f].get();
}

// Point frame f's factor cache at a full-set factor computed elsewhere (the
// parent's, or frame 0's): the frame's begin_run then copies it instead of
// refactorising (the factor depends on A, mu, beta only).
void share_factor(radmm_ctx* dst, radmm_ctx* src, double mu, double beta) {
  for (int q = 0; q < dst->Q; ++q) {
    Sensor& D = dst->sensors[q];
    Sensor& S = src->sensors[q];
    if (S.g_is_base && S.base_mu == mu && S.base_beta == beta) snapshot_base(src, S, false);
    if (!S.g0_valid || S.g0_mu != mu || S.g0_beta != beta) continue;
    if (D.g0_valid && D.g0_mu == mu && D.g0_beta == beta && D.g0_packed == S.g0_packed) continue;
    D.G0.view(S.G0.p, S.G0.n);
    D.cp0_valid = S.cp0_valid;
    if (S.cp0_valid) D.Cp0.view(S.Cp0.p, S.Cp0.n);
    D.g0_valid = true;
    D.g0_primal = S.g0_primal;
    D.g0_packed = S.g0_packed;
    D.g0_elems = S.g0_elems;
    D.g0_mu = mu;
    D.g0_beta = beta;
    D.g0_ld = S.g0_ld;
    D.g0_n = S.g0_n;
  }
}

// A frame rides the batched contractions while it has never eliminated a
// pixel in this run: full active set (J = identity), dual form, and the
// factor still the shared full-set one (no downdate or rebuild can have
// happened without an elimination).
bool frame_attached(const radmm_ctx* c) {
  for (const Sensor& S : c->sensors)
    if (S.n_act != c->N || S.primal || S.data_lag) return false;
  return true;
}

int split_for(const radmm_ctx* p, int tiles) {
  const int want = (3 * p->sm_count + tiles - 1) / std::max(1, tiles);
  return std::max(1, std::min(16, want));
}

// One synchronous Jacobi sweep (admm.hpp:389-390) for up to kFB attached
// frames: rhs, V = A RHS, W = G V, X = (RHS - mu A^H W)/beta with the
// history / scatter epilogue -- every operator column read once for all
// frames.  fs: frame contexts (same mu, beta; identical factors).
void frame_batch_updates(radmm_ctx* p, const std::vector<radmm_ctx*>& fs, double mu, double beta) {
  const int Q = p->Q, nf = (int)fs.size();
  const int N = p->N;
  if (nf < 1 || nf > kFB) fail(RADMM_INVALID_ARGUMENT, "frame batch size");
  int64_t ld_max = 0;
  int rows_max = 0;
  for (const Sensor& S : p->sensors) {
    ld_max = std::max(ld_max, S.ld);
    rows_max = std::max(rows_max, S.rows);
  }
  const int mt_rows = (rows_max + kFbBM - 1) / kFbBM;
  const int sp_fwd = split_for(p, mt_rows * Q);
  const int sp_gap = split_for(p, mt_rows * Q);
  const int sp_max = std::max(sp_fwd, sp_gap);
  const size_t part_per = (size_t)sp_max * kFB * ld_max;
  if (p->fb_part.n < part_per * Q) p->fb_part.alloc(part_per * Q, false);
  if (p->fb_jobs.n < (size_t)Q) p->fb_jobs.alloc(Q, false);
  if (p->fb_red.n < (size_t)Q) p->fb_red.alloc(Q, false);
  if (p->fb_rhs.n < (size_t)Q * kFB) p->fb_rhs.alloc((size_t)Q * kFB, false);
  // rhs for every (sensor, frame)
  std::vector<FrameRhsJob> rj((size_t)Q * nf);
  for (int q = 0; q < Q; ++q)
    for (int f = 0; f < nf; ++f) {
      Sensor& S = fs[f]->sensors[q];
      rj[(size_t)q * nf + f] = FrameRhsJob{N, S.data.p, S.x_hat.p, fs[f]->gap.p, fs[f]->sigma.p, S.rhs.p};
    }
  CK(cudaMemcpyAsync(p->fb_rhs.p, rj.data(), sizeof(FrameRhsJob) * rj.size(), cudaMemcpyHostToDevice, p->stream));
  LAUNCH(p, frame_rhs_kernel, dim3((unsigned)((N + 255) / 256), (unsigned)(Q * nf)), 256, 0, p->fb_rhs.p, beta);
  std::vector<FrameBatchJob> jobs(Q);
  std::vector<FrameReduceJob> red(Q);
  auto run_pass = [&](int mode, int nsplit) {
    CK(cudaMemcpyAsync(p->fb_jobs.p, jobs.data(), sizeof(FrameBatchJob) * Q, cudaMemcpyHostToDevice, p->stream));
    int mmax = 0;
    for (const auto& j : jobs) mmax = std::max(mmax, j.m);
    const dim3 grid((unsigned)((mmax + kFbBM - 1) / kFbBM), (unsigned)nsplit, (unsigned)Q);
    const int sm = (int)kFbSmem;
    const bool v2 = env_int("RADMM_FRAME_KERNEL", 2) == 2;
    if (mode != FB_GAP && v2) {  // operator passes: cp.async multistage pipeline
      if (mode == FB_FWD) {
        set_smem_attr((const void*)frame_batch2_kernel<FB_FWD>, (int)((int)kFb2Smem));
        LAUNCH(p, frame_batch2_kernel<FB_FWD>, grid, 256, kFb2Smem, p->fb_jobs.p, nsplit, mu, beta);
      } else {
        set_smem_attr((const void*)frame_batch2_kernel<FB_ADJ>, (int)((int)kFb2Smem));
        LAUNCH(p, frame_batch2_kernel<FB_ADJ>, grid, 256, kFb2Smem, p->fb_jobs.p, nsplit, mu, beta);
      }
    } else if (mode == FB_FWD) {
      set_smem_attr((const void*)frame_batch_kernel<FB_FWD>, (int)(sm));
      LAUNCH(p, frame_batch_kernel<FB_FWD>, grid, 256, kFbSmem, p->fb_jobs.p, nsplit, mu, beta);
    } else if (mode == FB_GAP) {
      set_smem_attr((const void*)frame_batch_kernel<FB_GAP>, (int)(sm));
      LAUNCH(p, frame_batch_kernel<FB_GAP>, grid, 256, kFbSmem, p->fb_jobs.p, nsplit, mu, beta);
    } else {
      set_smem_attr((const void*)frame_batch_kernel<FB_ADJ>, (int)(sm));
      LAUNCH(p, frame_batch_kernel<FB_ADJ>, grid, 256, kFbSmem, p->fb_jobs.p, nsplit, mu, beta);
    }
    if (mode == FB_ADJ) return;
    CK(cudaMemcpyAsync(p->fb_red.p, red.data(), sizeof(FrameReduceJob) * Q, cudaMemcpyHostToDevice, p->stream));
    LAUNCH(p, frame_reduce_kernel, dim3((unsigned)((mmax + 255) / 256), (unsigned)nf, (unsigned)Q), 256, 0,
           p->fb_red.p);
  };
  // V = A RHS
  for (int q = 0; q < Q; ++q) {
    const Sensor& P = p->sensors[q];
    FrameBatchJob j{};
    j.A = P.A.p; j.lda = P.ld; j.m = P.rows; j.k = N; j.nf = nf;
    j.part = p->fb_part.p + (size_t)q * part_per; j.ldp = ld_max;
    FrameReduceJob r{};
    r.part = j.part; r.ldp = ld_max; r.m = P.rows; r.nf = nf; r.nsplit = sp_fwd;
    for (int f = 0; f < nf; ++f) {
      j.B[f] = fs[f]->sensors[q].rhs.p;
      r.out[f] = fs[f]->sensors[q].v.p;
    }
    jobs[q] = j;
    red[q] = r;
  }
  {
    PhaseScope ps(p, RADMM_PHASE_FORWARD, 8.0 * ld_max * N * Q);
    run_pass(FB_FWD, sp_fwd);
  }
  // W = G V on the shared factor (a packed factor is unpacked once per run
  // into a full matrix for the DMMA pass)
  if (p->fb_g.size() < (size_t)Q) p->fb_g.resize(Q);
  const bool fb_g_fresh = !(p->fb_g_ok && p->fb_g_mu == mu && p->fb_g_beta == beta);
  for (int q = 0; q < Q; ++q) {
    const Sensor& H = fs[0]->sensors[q];
    if (!H.gpacked || !fb_g_fresh) continue;
    DArr<double2>& Gf = p->fb_g[q];
    if (Gf.n < (size_t)H.ld * H.rows) Gf.alloc((size_t)H.ld * H.rows, false);
    LAUNCH(p, cap_unpack_kernel, dim3((unsigned)cap_tiles(H.rows)), 256, 0, H.G.p, H.rows, Gf.p, H.ld);
  }
  p->fb_g_ok = true;
  p->fb_g_mu = mu;
  p->fb_g_beta = beta;
  auto g_full = [&](int q) -> const double2* { return fs[0]->sensors[q].gpacked ? p->fb_g[q].p : fs[0]->sensors[q].G.p; };
  auto g_ld = [&](int q) -> int64_t { return fs[0]->sensors[q].gpacked ? fs[0]->sensors[q].ld : fs[0]->sensors[q].ldg; };
  for (int q = 0; q < Q; ++q) {
    const Sensor& H = fs[0]->sensors[q];
    FrameBatchJob& j = jobs[q];
    j.A = g_full(q); j.lda = g_ld(q); j.m = H.rows; j.k = H.rows;
    FrameReduceJob& r = red[q];
    r.nsplit = sp_gap;
    for (int f = 0; f < nf; ++f) {
      j.B[f] = fs[f]->sensors[q].v.p;
      r.out[f] = fs[f]->sensors[q].w.p;
    }
  }
  {
    PhaseScope ps(p, RADMM_PHASE_GAPPLY, 16.0 * ld_max * ld_max * Q * (fs[0]->refine ? 3 : 1));
    run_pass(FB_GAP, sp_gap);
    // KM-space refinement for every frame (see refine()): R = V - C W, then
    // W += G R -- two more DMMA passes over the frames' right-hand sides,
    // with C unpacked once per run into a full matrix (frame 0's base C).
    bool can = fs[0]->refine;
    for (int q = 0; q < Q && can; ++q) can = fs[0]->sensors[q].cp_valid && !fs[0]->sensors[q].primal;
    if (can) {
      if (p->fb_cap.size() < (size_t)Q) p->fb_cap.resize(Q);
      for (int q = 0; q < Q; ++q) {
        const Sensor& H = fs[0]->sensors[q];
        DArr<double2>& Cf = p->fb_cap[q];
        if (!p->fb_cap_ok || p->fb_cap_mu != mu || p->fb_cap_beta != beta || Cf.n < (size_t)H.ld * H.rows) {
          if (Cf.n < (size_t)H.ld * H.rows) Cf.alloc((size_t)H.ld * H.rows, false);
          LAUNCH(p, cap_unpack_kernel, dim3((unsigned)cap_tiles(H.rows)), 256, 0, H.Cp.p, H.rows, Cf.p, H.ld);
        }
      }
      p->fb_cap_ok = true;
      p->fb_cap_mu = mu;
      p->fb_cap_beta = beta;
      for (int q = 0; q < Q; ++q) {  // R = V - C W  (into rho)
        FrameBatchJob& j = jobs[q];
        j.A = p->fb_cap[q].p;
        j.lda = fs[0]->sensors[q].ld;
        FrameReduceJob& r = red[q];
        for (int f = 0; f < nf; ++f) {
          j.B[f] = fs[f]->sensors[q].w.p;
          if (fs[f]->sensors[q].rho.n < (size_t)fs[f]->sensors[q].ld) fs[f]->sensors[q].rho.alloc(fs[f]->sensors[q].ld);
          r.out[f] = fs[f]->sensors[q].rho.p;
          r.base[f] = fs[f]->sensors[q].v.p;
        }
        r.sgn = -1.0;
      }
      run_pass(FB_GAP, sp_gap);
      for (int q = 0; q < Q; ++q) {  // W = W + G R
        FrameBatchJob& j = jobs[q];
        j.A = g_full(q);
        j.lda = g_ld(q);
        FrameReduceJob& r = red[q];
        for (int f = 0; f < nf; ++f) {
          j.B[f] = fs[f]->sensors[q].rho.p;
          r.out[f] = fs[f]->sensors[q].w.p;
          r.base[f] = fs[f]->sensors[q].w.p;
        }
        r.sgn = 1.0;
      }
      run_pass(FB_GAP, sp_gap);
      for (int q = 0; q < Q; ++q)
        for (int f = 0; f < nf; ++f) red[q].base[f] = nullptr;
    }
  }
  // X = (RHS - mu A^H W) / beta + epilogue
  for (int q = 0; q < Q; ++q) {
    const Sensor& P = p->sensors[q];
    FrameBatchJob& j = jobs[q];
    j.A = P.A.p; j.lda = P.ld; j.m = N; j.k = P.rows;
    for (int f = 0; f < nf; ++f) {
      Sensor& S = fs[f]->sensors[q];
      j.B[f] = S.w.p;
      j.rhs[f] = S.rhs.p;
      j.x_hat[f] = S.x_hat.p;
      j.x_full[f] = S.x_full.p;
      j.ring[f] = S.ring.p + (size_t)(fs[f]->upd % fs[f]->W) * N;
    }
  }
  {
    PhaseScope ps(p, RADMM_PHASE_ADJOINT, 8.0 * ld_max * N * Q);
    run_pass(FB_ADJ, 1);
  }
  for (radmm_ctx* c : fs) {
    ++c->upd;
    for (Sensor& S : c->sensors) S.v_ready = false;
  }
}

void run_frames(radmm_ctx* p, int F, const radmm_hyperparams* hs, const radmm_run_options* o,
                radmm_run_summary* outs) {
  if (F < 1 || !hs) fail(RADMM_INVALID_ARGUMENT, "run_frames: need at least one frame");
  if (o && o->observer) fail(RADMM_INVALID_ARGUMENT, "run_frames: observers are not supported");
  for (int f = 0; f < F; ++f) validate_hyper(&hs[f]);
  set_device(p);
  const bool asadmm = o && o->mode == RADMM_MODE_ASADMM;
  const bool disable = o && o->disable_screening;
  const bool fixed = o && o->fixed_iterations;
  // frame-batched contractions (RADMM_FRAME_BATCH=0: per-frame kernels only)
  const bool batched = env_int("RADMM_FRAME_BATCH", 1) != 0;
  std::vector<radmm_ctx*> ch(F);
  for (int f = 0; f < F; ++f) {
    ch[f] = frame_ctx(p, f);
    for (int q = 0; q < p->Q; ++q)
      if (!ch[f]->sensors[q].has_y)
        fail(RADMM_INVALID_ARGUMENT, "run_frames: frame " + std::to_string(f) + " sensor " + std::to_string(q) +
                                         " has no measurement");
  }
  std::vector<radmm_run_summary> sm(F);
  p->fb_cap_ok = false;
  p->fb_g_ok = false;
  p->marks.clear();
  p->ev_used = 0;
  for (int i = 0; i < RADMM_PHASE_COUNT; ++i) {  // parent stats = this call's batched passes
    p->prof_ms[i] = p->prof_bytes[i] = 0;
    p->prof_launches[i] = p->prof_calls[i] = 0;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (int f = 0; f < F; ++f) {
    radmm_ctx* c = ch[f];
    c->records.clear();
    c->active_log.clear();
    c->removal_log.clear();
    c->log_segs.clear();
    c->log_used = 0;
    c->pending_fail = 0;
    c->have_result = false;
    c->launches = 0;
    c->rebuilds = c->downdates = 0;
    c->refine = !(o && o->skip_refinement);
    c->refine_skipped = 0;
    c->iter_ms.clear();
    c->iter_launches.clear();
    c->marks.clear();
    c->ev_used = 0;
    share_factor(c, p, hs[f].mu, hs[f].beta);
    if (f > 0) share_factor(c, ch[0], hs[f].mu, hs[f].beta);
    build_contrib(c);
    begin_run(c, &hs[f]);
  }
  CK(cudaStreamSynchronize(p->stream));
  const auto t1 = std::chrono::steady_clock::now();
  const double setup_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  int max_iter = 0;
  for (int f = 0; f < F; ++f) max_iter = std::max(max_iter, hs[f].max_iter);
  std::vector<char> done(F, 0), staged(F, 0);
  std::vector<uint64_t> notice(F, 0);
  std::vector<FusionScalars> last(F);
  std::vector<int32_t> sizes(p->Q_total);
  std::vector<double> meta_all;
  std::vector<int> live;
  for (int k = 1; k <= max_iter; ++k) {
    live.clear();
    for (int f = 0; f < F; ++f)
      if (!done[f] && k <= hs[f].max_iter) live.push_back(f);
    if (live.empty()) break;
    for (int f : live) notice[f] = (asadmm && !disable && staged[f]) ? screen_all(ch[f], &hs[f], k) : 0;
    // attached frames with equal (mu, beta) share the batched contractions
    std::vector<int> single;
    std::vector<std::vector<int>> groups;
    for (int f : live) {
      if (!batched || !frame_attached(ch[f])) {
        single.push_back(f);
        continue;
      }
      bool placed = false;
      for (auto& g : groups)
        if ((int)g.size() < kFB && hs[g[0]].mu == hs[f].mu && hs[g[0]].beta == hs[f].beta) {
          g.push_back(f);
          placed = true;
          break;
        }
      if (!placed) groups.push_back({f});
    }
    for (auto& g : groups) {
      if (g.size() == 1) {
        single.push_back(g[0]);
        continue;
      }
      std::vector<radmm_ctx*> fc;
      for (int f : g) fc.push_back(ch[f]);
      frame_batch_updates(p, fc, hs[g[0]].mu, hs[g[0]].beta);
    }
    for (int f : single) local_updates(ch[f], &hs[f]);
    // all frames' fusion rounds in one launch (FusionCore::round, admm.hpp:236-258)
    for (size_t b0 = 0; b0 < live.size(); b0 += kMaxBatch) {
      const size_t nb = std::min<size_t>(kMaxBatch, live.size() - b0);
      Pack<FusionArgs> fp;
      for (size_t i = 0; i < nb; ++i) {
        const int f = live[b0 + i];
        FusionArgs a = fusion_args(ch[f], &hs[f], k);
        a.stop_on_converge = fixed ? 0 : 1;
        fp.j[i] = a;
      }
      PhaseScope ps(p, RADMM_PHASE_FUSION, 16.0 * p->N * (p->Q_total + 7) * nb);
      LAUNCH(p, fusion_frames_kernel, dim3((unsigned)((p->N + kFusionThreads - 1) / kFusionThreads), (unsigned)nb),
             kFusionThreads, 0, fp);
      for (size_t i = 0; i < nb; ++i) ++ch[live[b0 + i]]->launches;
    }
    CK(cudaStreamSynchronize(p->stream));
    for (int f : live) check_deferred(ch[f]);
    flush_marks(p);  // batched-pass phase events (profiling mode) live on the parent
    const auto now = std::chrono::steady_clock::now();
    for (int f : live) {
      const FusionScalars fs = ch[f]->fs_host[k & 1];
      record_round(ch[f], k, fs, notice[f], sm[f], sizes, meta_all, t1);
      sm[f].iterations = k;
      last[f] = fs;
      staged[f] = fs.trigger != 0;
      if ((fs.converged && !fixed) || k == hs[f].max_iter) {
        if (fs.converged && !fixed) sm[f].converged = 1;
        done[f] = 1;
        sm[f].solve_ms = std::chrono::duration<double, std::milli>(now - t1).count();
      }
    }
  }
  for (int f = 0; f < F; ++f) {
    radmm_ctx* c = ch[f];
    finish_removal_log(c);
    if (fixed) sm[f].converged = last[f].converged;
    sm[f].setup_ms = setup_ms;
    sm[f].kernel_launches = c->launches;
    sm[f].rebuilds = c->rebuilds;
    sm[f].downdates = c->downdates;
    sm[f].refine_skipped = c->refine ? c->refine_skipped : 0;
    c->summary = sm[f];
    c->have_result = true;
    if (outs) outs[f] = sm[f];
  }
}

void copy_out(radmm_ctx* c, const void* dev, void* host, size_t bytes) {
  if (!host) fail(RADMM_INVALID_ARGUMENT, "null output buffer");
  set_device(c);
  CK(cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost));
}

void need_result(radmm_ctx* c) {
  if (!c) fail(RADMM_INVALID_ARGUMENT, "null context");
  if (!c->have_result) fail(RADMM_INVALID_ARGUMENT, "no completed run on this context");
}

}  // namespace

struct radmm_solve_cache {
  radmm_ctx* ctx = nullptr;
  double mu = 0, beta = 0;
  int rows = 0, cols = 0;
  DArr<double2> x, tmp;
  DArr<double> ring;
  ~radmm_solve_cache() { delete ctx; }
};

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* radmm_last_error(void) { return g_last_error.c_str(); }
int radmm_version(void) { return 2; }

int radmm_build_features(void) { return RADMM_EXPERIMENTAL ? 1 : 0; }

int radmm_hyperparams_default(radmm_hyperparams* out) {
  return guarded([&] {
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    *out = radmm_hyperparams{3.0, 20.0, 100.0, 1e-4, 1e-2, 5, 1e-5, 1000};
  });
}

int radmm_hyperparams_validate(const radmm_hyperparams* h) {
  return guarded([&] { validate_hyper(h); });
}

int radmm_ctx_create(int device, int n_pixels, int n_sensors, radmm_ctx** out) {
  return guarded([&] {
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    if (n_sensors < 1) fail(RADMM_INVALID_ARGUMENT, "Problem: needs at least one sensor");
    if (n_pixels < 1) fail(RADMM_INVALID_ARGUMENT, "Problem: needs at least one pixel");
    auto c = std::make_unique<radmm_ctx>();
    init_ctx(c.get(), device, n_pixels, n_sensors);
    c->Q_total = n_sensors;
    c->q_begin = 0;
    c->q_max_local = n_sensors;
    *out = c.release();
  });
}

int radmm_ctx_destroy(radmm_ctx* ctx) {
  return guarded([&] {
    if (ctx && ctx->parent) fail(RADMM_INVALID_ARGUMENT, "frame contexts are owned by their parent context");
    if (ctx && env_int("RADMM_TRACE_DESTROY", 0)) {
      auto now = [] { return std::chrono::steady_clock::now(); };
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      const auto t0 = now();
      cudaSetDevice(ctx->device);
      cudaDeviceSynchronize();
      const auto t1 = now();
      ctx->frames.clear();
      const auto t2 = now();
      ctx->sensors.clear();
      const auto t3 = now();
      delete ctx;
      const auto t4 = now();
      std::fprintf(stderr, "[radmm destroy] sync %.2f ms, frames %.2f ms, sensors %.2f ms, rest %.2f ms\n", ms(t0, t1),
                   ms(t1, t2), ms(t2, t3), ms(t3, t4));
      return;
    }
    const int device = ctx ? ctx->device : -1;
    delete ctx;
    if (device >= 0) pool_trim_async(device);
  });
}

int radmm_pool_trim(int device) {
  return guarded([&] {
    pool_reaper_join();
    cudaMemPool_t pool;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemPoolTrimTo(pool, (size_t)pool_keep_bytes()));
  });
}

// Eager full-set Gram A A^H (dual sensors) on the context stream, ordered
// after `ev` (the operator upload): the tensor-core Gram of sensor q runs
// while sensor q+1 uploads.  The first run scales it (full_rebuild).
void eager_gram(radmm_ctx* c, Sensor& S, int q, cudaEvent_t ev) {
  if (c->parent || S.rows >= c->N || !env_int("RADMM_EAGER_GRAM", 1) || !env_int("RADMM_GRAM", 1)) return;
  if (ev) CK(cudaStreamWaitEvent(c->stream, ev, 0));
  if (use_gpacked(c, S)) {
    // packed factor: the raw Gram goes through one full temporary into Cp
    // (rebuild_packed unpacks and scales it)
    const size_t cn = cap_tiles(S.rows) * kHermTile * kHermTile;
    const size_t free_b = mem_available(c->device);
    const size_t tmp = (size_t)S.ld * S.rows;
    const size_t held = c->gtmp.empty() ? 0 : c->gtmp[0].n;
    if (free_b + held * sizeof(double2) < (tmp + (S.Cp.n < cn ? cn : 0)) * sizeof(double2) + (6ull << 30)) return;
    if (S.Cp.n < cn) S.Cp.alloc(cn, false);
    gtmp_reserve(c, 1, tmp);
    double2* T = c->gtmp[0].p;
    CK(cudaMemsetAsync(T, 0, sizeof(double2) * tmp, c->stream));
    // The Ozaki slices are only worth it if they can stay allocated across the
    // uploads: releasing a multi-GB scratch synchronises the device, which
    // would serialise every upload behind the previous sensor's Gram (config
    // 3: 0.6 s per sensor).  Project the whole problem's residency (every
    // sensor like this one) once per context; if the slices do not fit next to
    // it, the uploads use the fp64 DMMA Gram, which needs no scratch.
    if (c->oz_eager < 0) {
      size_t free_now = 0, total = 0;
      CK(cudaMemGetInfo(&free_now, &total));
      const double per_sensor = (double)S.ld * c->N * sizeof(float2) + 2.0 * cn * sizeof(double2) + 64.0 * c->N * 16;
      // 1: the one-pass Gram's scratch fits; 2: only the chunked Gram's does
      // (config 3: 0.94 GB instead of 26 GB); 0: neither (fp64 DMMA Gram)
      const double base = per_sensor * c->Q + tmp * 16.0 + (8.0 * (1ull << 30));
      const int mode = ozaki_chunk_mode();
      c->oz_eager = (mode != 2 && base + ozaki_scratch_bytes(S.rows, c->N) < (double)total) ? 1
                    : (mode >= 1 && base + ozaki_chunk_scratch_bytes(S.rows, c->N) < (double)total) ? 2 : 0;
    }
    const bool oz = (c->oz_eager == 1 && ozaki_gram(c, S, nullptr, c->N, T, S.ld, 1.0, 0.0)) ||
                    (c->oz_eager == 2 && ozaki_enabled() && c->N <= 65536 &&
                     ozaki_gram_chunked(c, S, nullptr, c->N, T, S.ld, 1.0, 0.0));
    if (!oz) {  // (the Ozaki scratch stays allocated for the next upload; the first run releases it)
      const GramJob g{S.A.p, S.ld, nullptr, c->N, S.rows, T, S.ld};
      set_smem_attr((const void*)gram_dmma1_kernel, (int)((int)kGramSmem));
      LAUNCH(c, gram_dmma1_kernel,
             dim3((unsigned)((S.rows + kGrBN - 1) / kGrBN), (unsigned)((S.rows + kGrBM - 1) / kGrBM), 1u), 256,
             kGramSmem, g, 1.0, 0.0);
    }
    LAUNCH(c, cap_pack_kernel, dim3((unsigned)cap_tiles(S.rows)), 256, 0, T, S.ld, S.rows, S.Cp.p);
    S.cp_valid = true;  // raw A A^H (raw_gram) until the first run scales it
    S.raw_gram = true;
    S.raw_packed = true;
    S.primal = false;
    if (c->gram_evs.size() < (size_t)c->Q) c->gram_evs.resize(c->Q, nullptr);
    if (!c->gram_evs[q]) CK(cudaEventCreateWithFlags(&c->gram_evs[q], cudaEventDisableTiming));
    CK(cudaEventRecord(c->gram_evs[q], c->stream));
    return;
  }
  if (S.gpacked) S.G.release();
  S.gpacked = false;
  S.raw_packed = false;
  ensure_g(S, S.rows, S.ld);
  S.ldg = S.ld;
  S.g_n = S.rows;
  S.primal = false;
  CK(cudaMemsetAsync(S.G.p, 0, sizeof(double2) * (size_t)S.ld * S.rows, c->stream));
  if (ozaki_gram(c, S, nullptr, c->N, S.G.p, S.ld, 1.0, 0.0)) {
    release_ozaki_scratch(c);
    S.raw_gram = true;
    if (c->gram_evs.size() < (size_t)c->Q) c->gram_evs.resize(c->Q, nullptr);
    if (!c->gram_evs[q]) CK(cudaEventCreateWithFlags(&c->gram_evs[q], cudaEventDisableTiming));
    CK(cudaEventRecord(c->gram_evs[q], c->stream));
    return;
  }
  // the job travels as a kernel parameter: a pageable job-table upload would
  // wait for the previous sensor's Gram and serialise the pipeline
  const GramJob g{S.A.p, S.ld, nullptr, c->N, S.rows, S.G.p, S.ld};
  set_smem_attr((const void*)gram_dmma1_kernel, (int)((int)kGramSmem));
  LAUNCH(c, gram_dmma1_kernel,
         dim3((unsigned)((S.rows + kGrBN - 1) / kGrBN), (unsigned)((S.rows + kGrBM - 1) / kGrBM), 1u), 256,
         kGramSmem, g, 1.0, 0.0);
  S.raw_gram = true;
  if (c->gram_evs.size() < (size_t)c->Q) c->gram_evs.resize(c->Q, nullptr);
  if (!c->gram_evs[q]) CK(cudaEventCreateWithFlags(&c->gram_evs[q], cudaEventDisableTiming));
  CK(cudaEventRecord(c->gram_evs[q], c->stream));
}

int radmm_set_operator_c64(radmm_ctx* ctx, int q, int rows, const float* a, int64_t lda, int ptr_kind) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (!a) fail(RADMM_INVALID_ARGUMENT, "null operator");
    if (lda < rows) fail(RADMM_INVALID_ARGUMENT, "lda < rows");
    set_device(ctx);
    const auto tp0 = std::chrono::steady_clock::now();
    prepare_operator(ctx, S, rows);
    const auto tp1 = std::chrono::steady_clock::now();
    const cudaMemcpyKind kind = ptr_kind == RADMM_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // host operators upload on their own stream (the data rows; the padding
    // rows are zeroed on the context stream), so the previous sensor's eager
    // Gram keeps running; the call returns once the host buffer is consumed
    const bool host = ptr_kind != RADMM_PTR_DEVICE && !ctx->parent;
    if (host && !ctx->up_stream) {
      CK(cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ctx->up_event, cudaEventDisableTiming));
    }
    cudaStream_t st = host ? ctx->up_stream : ctx->stream;
    if (host && (size_t)q < ctx->gram_evs.size() && ctx->gram_evs[q])  // a queued Gram may still read A_q
      CK(cudaStreamWaitEvent(st, ctx->gram_evs[q], 0));
    if (lda == S.ld && rows == S.ld)  // contiguous: one linear copy
      CK(cudaMemcpyAsync(S.A.p, a, sizeof(float2) * (size_t)rows * ctx->N, kind, st));
    else
      CK(cudaMemcpy2DAsync(S.A.p, S.ld * sizeof(float2), a, lda * sizeof(float2), rows * sizeof(float2), ctx->N,
                           kind, st));
    if (host) CK(cudaEventRecord(ctx->up_event, st));
    const auto tp2 = std::chrono::steady_clock::now();
    eager_gram(ctx, S, q, host ? ctx->up_event : nullptr);
    const auto tp3 = std::chrono::steady_clock::now();
    if (host) CK(cudaStreamSynchronize(st));
    else CK(cudaStreamSynchronize(ctx->stream));
    if (env_int("RADMM_DEBUG", 0)) {
      const auto tp4 = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "[radmm] set_operator q=%d: prepare %.2f ms, copy enqueue %.2f, eager gram %.2f, sync %.2f\n",
                   q, ms(tp0, tp1), ms(tp1, tp2), ms(tp2, tp3), ms(tp3, tp4));
    }
  });
}

int radmm_set_operator_c128(radmm_ctx* ctx, int q, int rows, const double* a, int64_t lda, int ptr_kind) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (!a) fail(RADMM_INVALID_ARGUMENT, "null operator");
    if (lda < rows) fail(RADMM_INVALID_ARGUMENT, "lda < rows");
    set_device(ctx);
    prepare_operator(ctx, S, rows);
    const int64_t chunk = std::max<int64_t>(1, (64ll << 20) / (rows * (int64_t)sizeof(double2)));
    DArr<double2> stage;
    stage.alloc((size_t)rows * std::min<int64_t>(chunk, ctx->N), false);
    for (int64_t c0 = 0; c0 < ctx->N; c0 += chunk) {
      const int64_t nc = std::min<int64_t>(chunk, ctx->N - c0);
      CK(cudaMemcpy2DAsync(stage.p, rows * sizeof(double2), a + 2 * c0 * lda, lda * sizeof(double2),
                           rows * sizeof(double2), nc,
                           ptr_kind == RADMM_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           ctx->stream));
      const int64_t total = rows * nc;
      LAUNCH(ctx, c128_to_c64_kernel, dim3((unsigned)((total + 255) / 256)), 256, 0, stage.p, (int64_t)rows,
             S.A.p + c0 * S.ld, S.ld, rows, (int)nc);
    }
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int radmm_set_frame_measurement(radmm_ctx* ctx, int frame, int q, const double* y, int ptr_kind) {
  return guarded([&] {
    radmm_ctx* fc = frame_ctx(ctx, frame);
    const int st = radmm_set_measurement(fc, q, y, ptr_kind);
    if (st != RADMM_OK) fail(st, g_last_error);
  });
}

int radmm_run_frames(radmm_ctx* ctx, int frames, const radmm_hyperparams* hypers, const radmm_run_options* opts,
                     radmm_run_summary* summaries) {
  return guarded([&] {
    if (!ctx) fail(RADMM_INVALID_ARGUMENT, "null context");
    run_frames(ctx, frames, hypers, opts, summaries);
  });
}

int radmm_frame(radmm_ctx* ctx, int frame, radmm_ctx** out) {
  return guarded([&] {
    if (!ctx || !out) fail(RADMM_INVALID_ARGUMENT, "null argument");
    if (frame < 0 || frame >= (int)ctx->frames.size()) fail(RADMM_INVALID_ARGUMENT, "frame index out of range");
    *out = ctx->frames[frame].get();
  });
}

int radmm_set_measurement(radmm_ctx* ctx, int q, const double* y, int ptr_kind) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (!S.has_op) fail(RADMM_INVALID_ARGUMENT, "set the operator before the measurement");
    if (!y) fail(RADMM_INVALID_ARGUMENT, "null measurement");
    set_device(ctx);
    S.y.alloc(S.ld);
    if (ptr_kind != RADMM_PTR_DEVICE && ctx->up_stream) {
      // on the upload stream (a queued eager Gram keeps running); the context
      // stream is ordered after it by an event
      CK(cudaMemcpyAsync(S.y.p, y, sizeof(double2) * S.rows, cudaMemcpyHostToDevice, ctx->up_stream));
      CK(cudaEventRecord(ctx->up_event, ctx->up_stream));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->up_event, 0));
      CK(cudaStreamSynchronize(ctx->up_stream));  // the caller may reuse y on return
    } else {
      CK(cudaMemcpyAsync(S.y.p, y, sizeof(double2) * S.rows,
                         ptr_kind == RADMM_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                         ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));  // the caller may reuse y on return
    }
    S.has_y = true;
  });
}

int radmm_generate_dechirp_operator(radmm_ctx* ctx, int q, int M, int K, const double* pix, const double* tx,
                                    const double* rx, const double* phi, double fc, double bw, double pulse) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (M < 1 || K < 1 || !pix || !tx || !rx || !phi) fail(RADMM_INVALID_ARGUMENT, "bad generator arguments");
    set_device(ctx);
    prepare_operator(ctx, S, M * K);
    const int N = ctx->N;
    DArr<double> dpix, dtx, drx, dphi;
    dpix.alloc(3 * (size_t)N, false); dtx.alloc(3, false); drx.alloc(3 * (size_t)M, false); dphi.alloc(N, false);
    CK(cudaMemcpyAsync(dpix.p, pix, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(dtx.p, tx, sizeof(double) * 3, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(drx.p, rx, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(dphi.p, phi, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
    const int64_t total = (int64_t)M * K * N;
    LAUNCH(ctx, dechirp_kernel, dim3((unsigned)((total + 255) / 256)), 256, 0, S.A.p, S.ld, M, K, N, dpix.p, dtx.p,
           drx.p, dphi.p, bw / pulse, fc, pulse / K, 299792458.0);
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int radmm_generate_echo_operator(radmm_ctx* ctx, int q, int M, int K, const double* pix, const double* tx,
                                 const double* rx, double fc, double sample_rate, double chirp_rate,
                                 double pulse_duration) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (M < 1 || K < 1 || !pix || !tx || !rx) fail(RADMM_INVALID_ARGUMENT, "bad generator arguments");
    if (!(sample_rate > 0.0) || !(pulse_duration > 0.0)) fail(RADMM_INVALID_ARGUMENT, "Waveform: bad parameters");
    set_device(ctx);
    prepare_operator(ctx, S, M * K);
    const int N = ctx->N;
    DArr<double> dpix, dtx, drx;
    dpix.alloc(3 * (size_t)N, false); dtx.alloc(3, false); drx.alloc(3 * (size_t)M, false);
    CK(cudaMemcpyAsync(dpix.p, pix, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(dtx.p, tx, sizeof(double) * 3, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(drx.p, rx, sizeof(double) * 3 * M, cudaMemcpyHostToDevice, ctx->stream));
    const int64_t total = (int64_t)M * K * N;
    LAUNCH(ctx, echo_kernel, dim3((unsigned)((total + 255) / 256)), 256, 0, S.A.p, S.ld, M, K, N, dpix.p, dtx.p,
           drx.p, fc, sample_rate, chirp_rate, pulse_duration, 299792458.0, 3.141592653589793238462643383279502884);
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

int radmm_get_operator_c64(radmm_ctx* ctx, int q, float* out) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (!S.has_op || !out) fail(RADMM_INVALID_ARGUMENT, "no operator");
    set_device(ctx);
    CK(cudaMemcpy2D(out, S.rows * sizeof(float2), S.A.p, S.ld * sizeof(float2), S.rows * sizeof(float2), ctx->N,
                    cudaMemcpyDeviceToHost));
  });
}

int radmm_run(radmm_ctx* ctx, const radmm_hyperparams* hyper, const radmm_run_options* opts,
              radmm_run_summary* summary) {
  return guarded([&] {
    if (!ctx) fail(RADMM_INVALID_ARGUMENT, "null context");
    do_run(ctx, hyper, opts, summary);
  });
}

int radmm_get_image(radmm_ctx* ctx, double* out) {
  return guarded([&] {
    need_result(ctx);
    DArr<double> img;
    img.alloc(ctx->N, false);
    LAUNCH(ctx, abs_kernel, dim3((ctx->N + 255) / 256), 256, 0, ctx->xg.p, ctx->N, img.p);
    CK(cudaStreamSynchronize(ctx->stream));
    copy_out(ctx, img.p, out, sizeof(double) * ctx->N);
  });
}

int radmm_get_vector(radmm_ctx* ctx, radmm_vector which, double* out) {
  return guarded([&] {
    need_result(ctx);
    const double2* src = nullptr;
    switch (which) {
      case RADMM_VEC_X_GLOBAL: src = ctx->xg.p; break;
      case RADMM_VEC_S: src = ctx->s.p; break;
      case RADMM_VEC_SIGMA: src = ctx->sigma.p; break;
      case RADMM_VEC_SIGMA_PRE_GLOBAL: src = ctx->sigma_pre.p; break;
      case RADMM_VEC_GAP: src = ctx->gap.p; break;
      default: fail(RADMM_INVALID_ARGUMENT, "unknown vector");
    }
    copy_out(ctx, src, out, sizeof(double2) * ctx->N);
  });
}

int radmm_get_sensor_image(radmm_ctx* ctx, int q, double* out) {
  return guarded([&] {
    need_result(ctx);
    Sensor& S = sensor_at(ctx, q);
    copy_out(ctx, S.x_full.p, out, sizeof(double2) * ctx->N);
  });
}

int radmm_get_record_count(radmm_ctx* ctx, int* count) {
  return guarded([&] {
    need_result(ctx);
    if (!count) fail(RADMM_INVALID_ARGUMENT, "null output");
    *count = (int)ctx->records.size();
  });
}

int radmm_get_records(radmm_ctx* ctx, radmm_iteration_record* out, int capacity) {
  return guarded([&] {
    need_result(ctx);
    if (!out || capacity < (int)ctx->records.size()) fail(RADMM_INVALID_ARGUMENT, "output too small");
    std::memcpy(out, ctx->records.data(), sizeof(radmm_iteration_record) * ctx->records.size());
  });
}

int radmm_get_active_sizes(radmm_ctx* ctx, int32_t* out, int capacity) {
  return guarded([&] {
    need_result(ctx);
    if (!out || capacity < (int)ctx->active_log.size()) fail(RADMM_INVALID_ARGUMENT, "output too small");
    std::memcpy(out, ctx->active_log.data(), sizeof(int32_t) * ctx->active_log.size());
  });
}

int radmm_get_active_set(radmm_ctx* ctx, int q, int32_t* out, int* count) {
  return guarded([&] {
    need_result(ctx);
    Sensor& S = sensor_at(ctx, q);
    if (!count) fail(RADMM_INVALID_ARGUMENT, "null output");
    *count = S.n_act;
    if (out) copy_out(ctx, S.J.p, out, sizeof(int) * S.n_act);
  });
}

int radmm_get_removal_log_size(radmm_ctx* ctx, int* entries) {
  return guarded([&] {
    need_result(ctx);
    if (!entries) fail(RADMM_INVALID_ARGUMENT, "null output");
    *entries = (int)(ctx->removal_log.size() / 3);
  });
}

int radmm_get_removal_log(radmm_ctx* ctx, int32_t* out, int capacity) {
  return guarded([&] {
    need_result(ctx);
    if (!out || capacity < (int)(ctx->removal_log.size() / 3)) fail(RADMM_INVALID_ARGUMENT, "output too small");
    std::memcpy(out, ctx->removal_log.data(), sizeof(int32_t) * ctx->removal_log.size());
  });
}

int radmm_factorize(int device, int rows, int cols, const double* a_hat, double mu, double beta,
                    radmm_solve_cache** out) {
  return guarded([&] {
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    if (!(mu > 0.0)) fail(RADMM_INVALID_ARGUMENT, "factorize: mu must be > 0");
    if (!(beta > 0.0)) fail(RADMM_INVALID_ARGUMENT, "factorize: beta must be > 0");
    if (rows < 1 || cols < 1 || !a_hat) fail(RADMM_INVALID_ARGUMENT, "factorize: empty matrix");
    for (int64_t i = 0; i < 2ll * rows * cols; ++i)
      if (!std::isfinite(a_hat[i])) fail(RADMM_INVALID_ARGUMENT, "factorize: matrix has non-finite entries");
    auto sc = std::make_unique<radmm_solve_cache>();
    sc->ctx = new radmm_ctx();
    radmm_ctx* c = sc->ctx;
    init_ctx(c, device, cols, 1);
    c->Q_total = 1;
    c->q_max_local = 1;
    Sensor& S = c->sensors[0];
    int st = radmm_set_operator_c128(c, 0, rows, a_hat, rows, RADMM_PTR_HOST);
    if (st != RADMM_OK) fail(st, g_last_error);
    S.n_act = cols;
    LAUNCH(c, iota_kernel, dim3((cols + 255) / 256), 256, 0, S.J.p, cols);
    full_rebuild(c, {0}, mu, beta);
    sc->mu = mu; sc->beta = beta; sc->rows = rows; sc->cols = cols;
    sc->x.alloc(cols); sc->tmp.alloc(cols); sc->ring.alloc(cols);
    *out = sc.release();
  });
}

int radmm_solve_local(radmm_solve_cache* sc, const double* rhs, double* x) {
  return guarded([&] {
    if (!sc || !rhs || !x) fail(RADMM_INVALID_ARGUMENT, "solve_local: null argument");
    radmm_ctx* c = sc->ctx;
    set_device(c);
    Sensor& S = c->sensors[0];
    CK(cudaMemcpyAsync(S.rhs.p, rhs, sizeof(double2) * sc->cols, cudaMemcpyHostToDevice, c->stream));
    if (S.primal) {
      ColDotJob j{};
      j.M = S.G.p; j.ld = S.ldg; j.len = sc->cols; j.n_out = sc->cols; j.vec = S.rhs.p; j.out = sc->x.p; j.scale = 1.0;
      coldot<double2, EPI_STORE>(c, {j}, sc->mu, sc->beta);
    } else {
      FwdJob f{};
      f.A = S.A.p; f.ld = S.ld; f.n = sc->cols; f.J = S.J.p; f.src = S.rhs.p; f.part = S.part.p;
      plan_chunks(c, S, sc->cols, 1, f.n_chunks, f.chunk_len);
      forward<MODE_GATHER>(c, {f}, {ReduceJob{S.part.p, f.n_chunks, S.ld, S.rows, nullptr, S.v.p, 1.0}}, 0.0);
      gapply(c, {0});
      refine(c, {0}, sc->mu, nullptr);
      ColDotJob a{};
      a.M = S.A.p; a.ld = S.ld; a.len = S.rows; a.n_out = sc->cols; a.cols = S.J.p; a.pix = S.J.p; a.vec = S.w.p;
      a.rhs = S.rhs.p; a.x_hat = sc->x.p; a.x_full = sc->tmp.p; a.ring_slot = sc->ring.p;
      adjoint(c, {a}, {0}, sc->mu, sc->beta, nullptr);
    }
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(x, sc->x.p, sizeof(double2) * sc->cols, cudaMemcpyDeviceToHost));
  });
}

int radmm_solve_cache_destroy(radmm_solve_cache* sc) {
  return guarded([&] {
    const int device = sc && sc->ctx ? sc->ctx->device : -1;
    delete sc;
    if (device >= 0) pool_trim_async(device);
  });
}

int radmm_soft_threshold(int device, const double* v, int64_t n, double kappa, double* out) {
  return guarded([&] {
    if (!(kappa >= 0.0)) fail(RADMM_INVALID_ARGUMENT, "soft_threshold: kappa must be >= 0");
    if (n < 0 || (n > 0 && (!v || !out))) fail(RADMM_INVALID_ARGUMENT, "soft_threshold: null buffer");
    if (n == 0) return;
    CK(cudaSetDevice(device));
    DArr<double2> dv, dout;
    dv.alloc(n, false);
    dout.alloc(n, false);
    CK(cudaMemcpy(dv.p, v, sizeof(double2) * n, cudaMemcpyHostToDevice));
    soft_threshold_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dv.p, n, kappa, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout.p, sizeof(double2) * n, cudaMemcpyDeviceToHost));
  });
}

int radmm_apply_operator(radmm_ctx* ctx, int q, const double* x, double* y) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (!S.has_op || !x || !y) fail(RADMM_INVALID_ARGUMENT, "ForwardOperator::apply: size mismatch");
    set_device(ctx);
    const int N = ctx->N;
    DArr<double2> dx;
    DArr<int> idx;
    dx.alloc(N, false);
    idx.alloc(N, false);
    CK(cudaMemcpyAsync(dx.p, x, sizeof(double2) * N, cudaMemcpyHostToDevice, ctx->stream));
    LAUNCH(ctx, iota_kernel, dim3((N + 255) / 256), 256, 0, idx.p, N);
    FwdJob f{};
    f.A = S.A.p; f.ld = S.ld; f.n = N; f.J = idx.p; f.src = dx.p; f.part = S.part.p;
    plan_chunks(ctx, S, N, 1, f.n_chunks, f.chunk_len);
    forward<MODE_GATHER>(ctx, {f}, {ReduceJob{S.part.p, f.n_chunks, S.ld, S.rows, nullptr, S.v.p, 1.0}}, 0.0);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(y, S.v.p, sizeof(double2) * S.rows, cudaMemcpyDeviceToHost));
  });
}

int radmm_apply_adjoint(radmm_ctx* ctx, int q, const double* y, double* x) {
  return guarded([&] {
    Sensor& S = sensor_at(ctx, q);
    if (!S.has_op || !x || !y) fail(RADMM_INVALID_ARGUMENT, "ForwardOperator::apply_adjoint: size mismatch");
    set_device(ctx);
    const int N = ctx->N;
    DArr<double2> dy, dx;
    DArr<int> idx;
    dy.alloc(S.ld);
    dx.alloc(N, false);
    idx.alloc(N, false);
    CK(cudaMemcpyAsync(dy.p, y, sizeof(double2) * S.rows, cudaMemcpyHostToDevice, ctx->stream));
    LAUNCH(ctx, iota_kernel, dim3((N + 255) / 256), 256, 0, idx.p, N);
    ColDotJob j{};
    j.M = S.A.p; j.ld = S.ld; j.len = S.rows; j.n_out = N; j.cols = idx.p; j.vec = dy.p; j.out = dx.p; j.scale = 1.0;
    coldot<float2, EPI_STORE>(ctx, {j}, 1.0, 1.0);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(x, dx.p, sizeof(double2) * N, cudaMemcpyDeviceToHost));
  });
}

int radmm_back_projection(radmm_ctx* ctx, double* image) {
  return guarded([&] {
    if (!ctx || !image) fail(RADMM_INVALID_ARGUMENT, "back_projection: null argument");
    for (const Sensor& S : ctx->sensors)
      if (!S.has_op || !S.has_y) fail(RADMM_INVALID_ARGUMENT, "back_projection: need one measurement per operator");
    set_device(ctx);
    radmm_ctx* c = ctx;
    const size_t N = c->N;
    // per-sensor adjoint images A_q^H y_q: into the exchange send buffer when
    // sharded (then all-gathered), else into a local Q x N buffer
    DArr<double2> local;
    double2* dst = c->sharded ? c->send_buf.p : nullptr;
    if (!dst) {
      local.alloc((size_t)c->Q * N, false);
      dst = local.p;
    }
    std::vector<ColDotJob> jobs;
    for (int q = 0; q < c->Q; ++q) {
      Sensor& S = c->sensors[q];
      ColDotJob j{};
      j.M = S.A.p; j.ld = S.ld; j.len = S.rows; j.n_out = (int)N; j.vec = S.y.p; j.out = dst + (size_t)q * N;
      j.scale = 1.0;
      jobs.push_back(j);
    }
    coldot<float2, EPI_STORE>(c, jobs, 1.0, 1.0);
    std::vector<const double2*> ptrs(c->Q_total);
    if (c->sharded) {
      g_nccl.check(g_nccl.AllGather(c->send_buf.p, c->gathered.p, (size_t)c->q_max_local * N * 2, kNcclDouble,
                                    c->comm, c->stream), "ncclAllGather(back_projection)");
      g_nccl.settle(c->comm, "ncclAllGather(back_projection)", c->nccl_timeout_ms);
      for (int g = 0; g < c->Q_total; ++g) {
        int r = 0;
        while (r + 1 < c->world && (int64_t)(r + 1) * c->Q_total / c->world <= g) ++r;
        const int begin = (int)((int64_t)r * c->Q_total / c->world);
        ptrs[g] = c->gathered.p + ((size_t)r * c->q_max_local + (g - begin)) * N;
      }
    } else {
      for (int q = 0; q < c->Q; ++q) ptrs[q] = dst + (size_t)q * N;
    }
    DArr<const double2*> dptrs;
    dptrs.alloc(ptrs.size(), false);
    CK(cudaMemcpyAsync(dptrs.p, ptrs.data(), sizeof(void*) * ptrs.size(), cudaMemcpyHostToDevice, c->stream));
    DArr<double> mag;
    mag.alloc(N, false);
    LAUNCH(c, bp_sum_kernel, dim3((unsigned)((N + 255) / 256)), 256, 0, dptrs.p, c->Q_total, (int)N, mag.p);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(image, mag.p, sizeof(double) * N, cudaMemcpyDeviceToHost));
    double peak = 0.0;
    for (size_t j = 0; j < N; ++j) peak = std::max(peak, image[j]);
    if (peak > 0.0)
      for (size_t j = 0; j < N; ++j) image[j] /= peak;  // an all-zero result stays all-zero
  });
}

int radmm_set_profiling(radmm_ctx* ctx, int enabled) {
  return guarded([&] {
    if (!ctx) fail(RADMM_INVALID_ARGUMENT, "null context");
    ctx->profiling = enabled != 0;
  });
}

int radmm_get_phase_stats(radmm_ctx* ctx, radmm_phase_stat* out) {
  return guarded([&] {
    // the last radmm_run, or (on a parent) the batched passes of the last radmm_run_frames
    if (!ctx) fail(RADMM_INVALID_ARGUMENT, "null context");
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    for (int i = 0; i < RADMM_PHASE_COUNT; ++i)
      out[i] = radmm_phase_stat{ctx->prof_calls[i], ctx->prof_launches[i], ctx->prof_ms[i], ctx->prof_bytes[i]};
  });
}

int radmm_get_iteration_stats(radmm_ctx* ctx, double* device_ms, int64_t* launches, int capacity) {
  return guarded([&] {
    need_result(ctx);
    if (capacity < (int)ctx->iter_ms.size()) fail(RADMM_INVALID_ARGUMENT, "output too small");
    if (device_ms) std::memcpy(device_ms, ctx->iter_ms.data(), sizeof(double) * ctx->iter_ms.size());
    if (launches) std::memcpy(launches, ctx->iter_launches.data(), sizeof(int64_t) * ctx->iter_launches.size());
  });
}

int radmm_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    if (bytes == 0) return;
    void* p = nullptr;
    const cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(RADMM_OUT_OF_MEMORY, std::string("radmm_host_alloc: ") + cudaGetErrorString(e));
    }
    *out = p;
  });
}

int radmm_host_free(void* p) {
  return guarded([&] {
    if (p) CK(cudaFreeHost(p));
  });
}

int radmm_set_tuning(const char* name, int value, int clear) {
  return guarded([&] {
    if (!name || std::strncmp(name, "RADMM_", 6) != 0) fail(RADMM_INVALID_ARGUMENT, "tuning switches are RADMM_*");
    std::lock_guard<std::mutex> lk(g_tune_mu);
    TuneEntry& t = tune_entry(name);
    t.api_set = clear == 0;
    t.api_val = value;
    g_tune_gen.fetch_add(1, std::memory_order_release);
  });
}

int radmm_set_transport_timeout(radmm_ctx* ctx, int timeout_ms) {
  return guarded([&] {
    if (!ctx) fail(RADMM_INVALID_ARGUMENT, "null context");
    if (timeout_ms < 1) fail(RADMM_INVALID_ARGUMENT, "transport timeout must be >= 1 ms");
    ctx->nccl_timeout_ms = timeout_ms;
  });
}

int radmm_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    g_nccl.load();
    nccl_uid id;
    g_nccl.check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
  });
}

int radmm_ctx_create_sharded(int device, int n_pixels, int q_total, int q_begin, int q_end, int rank,
                             int world_size, const uint8_t nccl_id[128], radmm_ctx** out) {
  return guarded([&] {
    if (!out) fail(RADMM_INVALID_ARGUMENT, "null output");
    if (world_size < 1 || rank < 0 || rank >= world_size) fail(RADMM_INVALID_ARGUMENT, "bad rank / world size");
    if (q_total < 1) fail(RADMM_INVALID_ARGUMENT, "Problem: at least one sensor");
    // Q < G: the ranks past the sensors hold none -- they join the exchange
    // with empty blocks and run the (redundant) fusion like every rank
    const int b = (int)((int64_t)rank * q_total / world_size);
    const int e = (int)((int64_t)(rank + 1) * q_total / world_size);
    if (q_begin != b || q_end != e)
      fail(RADMM_INVALID_ARGUMENT, "sensor range must be the contiguous block [r*Q/G, (r+1)*Q/G)");
    auto c = std::make_unique<radmm_ctx>();
    init_ctx(c.get(), device, n_pixels, e - b);
    c->Q_total = q_total;
    c->q_begin = b;
    c->rank = rank;
    c->world = world_size;
    c->q_max_local = (q_total + world_size - 1) / world_size;
    // a one-rank communicator exercises the very same exchange path on one GPU
    c->sharded = world_size > 1 || (nccl_id && env_int("RADMM_FORCE_NCCL", 0) != 0);
    if (c->sharded) {
      if (!nccl_id) fail(RADMM_INVALID_ARGUMENT, "null NCCL id");
      g_nccl.load();
      nccl_uid id;
      std::memcpy(id.internal, nccl_id, 128);
      c->nccl_timeout_ms = std::max(1000, env_int("RADMM_NCCL_TIMEOUT_MS", c->nccl_timeout_ms));
      if (g_nccl.CommInitRankConfig && g_nccl.GetAsyncError) {
        nccl_config cfg{sizeof(nccl_config), 0xcafebeef, 22703, 0 /* non-blocking */, INT32_MIN, INT32_MIN,
                        INT32_MIN, nullptr, INT32_MIN, INT32_MIN, nullptr, INT32_MIN, INT32_MIN, INT32_MIN, INT32_MIN};
        g_nccl.check(g_nccl.CommInitRankConfig(&c->comm, world_size, id, rank, &cfg), "ncclCommInitRankConfig");
        g_nccl.settle(c->comm, "ncclCommInitRankConfig", c->nccl_timeout_ms);
      } else {
        g_nccl.check(g_nccl.CommInitRank(&c->comm, world_size, id, rank), "ncclCommInitRank");
      }
      c->send_buf.alloc((size_t)c->q_max_local * n_pixels);
      c->gathered.alloc((size_t)c->q_max_local * n_pixels * world_size);
      c->size_send.alloc(2 * (size_t)c->q_max_local + 1);
      c->size_recv.alloc((2 * (size_t)c->q_max_local + 1) * world_size);
    }
    *out = c.release();
  });
}

}  // extern "C"
