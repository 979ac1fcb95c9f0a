/*
 * radmm_b200 -- C ABI of the B200-native ASADMM iteration loop.
 *
 * Drop-in boundary for the reference's solver entry points
 * (/root/reference/proj/include/radmm/..., cited per function below).  All
 * signatures are plain C: opaque handles, plain pointers and sizes, int
 * status codes, no exceptions and no torch types.  Complex numbers are
 * interleaved (re, im) pairs: complex128 = 2 doubles, complex64 = 2 floats.
 * Matrices are column-major (Eigen's default, forward_model.hpp:18-20),
 * row r = m*K + k, column n = pixel (forward_model.hpp:22-23,104-107).
 *
 * Error conventions: every call returns a radmm_status; on
 * failure radmm_last_error() holds a thread-local message.  The Python and
 * C++ shims re-raise the reference's exception types:
 *   RADMM_INVALID_ARGUMENT -> std::invalid_argument (admm.hpp:41-57,69-80;
 *                             solver_core.hpp:15-16,35-38,48-49)
 *   RADMM_NUMERICAL        -> std::runtime_error ("factorize: Cholesky
 *                             failed", solver_core.hpp:42-43)
 *   RADMM_TRANSPORT        -> TransportError (runtime.hpp:27-35; NCCL here)
 *   RADMM_CUDA / RADMM_OUT_OF_MEMORY -> std::runtime_error
 * Non-convergence is not an error (admm.hpp:427-431): summary.converged = 0.
 */
#ifndef RADMM_B200_H
#define RADMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RADMM_OK = 0,
  RADMM_INVALID_ARGUMENT = 1,
  RADMM_NUMERICAL = 2,
  RADMM_TRANSPORT = 3,
  RADMM_CUDA = 4,
  RADMM_OUT_OF_MEMORY = 5
} radmm_status;

/* Mode, admm.hpp:25. */
typedef enum { RADMM_MODE_SADMM = 0, RADMM_MODE_ASADMM = 1 } radmm_mode;

/* Hyperparams, admm.hpp:31-39 (same fields, same defaults). */
typedef struct {
  double mu;              /* 3.0   */
  double lambda;          /* 20.0  */
  double beta;            /* 100.0 */
  double eps_abs;         /* 1e-4  */
  double eps_rel;         /* 1e-2  */
  int32_t screening_window; /* 5   */
  double screening_tol;   /* 1e-5  */
  int32_t max_iter;       /* 1000  */
} radmm_hyperparams;

/* IterationRecord, admm.hpp:284-295 (per-sensor vectors via
 * radmm_get_active_sizes). */
typedef struct {
  int32_t iteration;
  double pri_res;
  double dual_res;
  double eps_pri;
  double eps_dual;
  double active_fraction;  /* max_q N_q / N after this round's screening */
  double ms_elapsed;       /* cumulative wall time */
  uint64_t bytes_sent;     /* notices + sum_q contribution_size(N_q) */
} radmm_iteration_record;

/* IterationView, admm.hpp:339-347: host copies valid during the callback. */
typedef struct {
  int32_t iteration;
  const double* x_global;   /* N complex128 */
  const double* s;          /* N complex128 */
  const double* sigma;      /* N complex128 */
  const int32_t* active_sizes; /* Q (local sensors) */
  int32_t converged;
  int32_t screening_trigger;
} radmm_iteration_view;

typedef void (*radmm_observer_fn)(void* user, const radmm_iteration_view* view);

/* Arguments of run() that are not Hyperparams (admm.hpp:357-359) plus the
 * build-only switches SURVEY 8b lists. */
typedef struct {
  radmm_mode mode;
  int32_t disable_screening;  /* must equal SADMM bitwise (test_admm.cpp:266-288) */
  int32_t fixed_iterations;   /* build-only: never stop on convergence */
  radmm_observer_fn observer; /* slow path: D2H of x_G, s, sigma per iteration */
  void* observer_user;
  /* build-only precision switch: 0 (default) = every dual (Woodbury) solve
   * takes one step of KM-space iterative refinement with the exact
   * capacitance, which makes it backward stable like the reference's
   * Cholesky (solver_core.hpp:41-51); 1 = the bare explicit-inverse apply
   * (faster, ~eps cond(C)^2 forward error -- DESIGN.md section 3). */
  int32_t skip_refinement;
} radmm_run_options;

/* RunResult scalars, admm.hpp:324-335 + ConvergenceReport totals :297-300. */
typedef struct {
  int32_t converged;
  int32_t screening_stalled;
  int32_t iterations;
  uint64_t total_active_solves;
  uint64_t total_bytes;
  double setup_ms;           /* upload + initial factorization */
  double solve_ms;           /* iteration loop */
  int64_t kernel_launches;   /* library kernels launched by the last run */
  int64_t rebuilds;          /* full refactorizations */
  int64_t downdates;         /* low-rank active-set downdates */
  int64_t refine_skipped;    /* dual sensors solved without refinement (packed C did not fit) */
} radmm_run_summary;

typedef enum {
  RADMM_VEC_X_GLOBAL = 0,
  RADMM_VEC_S = 1,
  RADMM_VEC_SIGMA = 2,
  RADMM_VEC_SIGMA_PRE_GLOBAL = 3,
  RADMM_VEC_GAP = 4
} radmm_vector;

typedef struct radmm_ctx radmm_ctx;
typedef struct radmm_solve_cache radmm_solve_cache;

/* Flag for pointers that already live in device memory. */
#define RADMM_PTR_HOST 0
#define RADMM_PTR_DEVICE 1

const char* radmm_last_error(void);
int radmm_version(void);
/* Tuning switches (RADMM_* names: A/B knobs and
 * build-only paths; defaults are the shipped configuration).  The environment
 * is read once per ABI call, never on a launch path; radmm_set_tuning
 * overrides it (clear != 0 removes the override). */
int radmm_set_tuning(const char* name, int value, int clear);
/* Bit 0: built with the parked experimental kernels (RADMM_EXPERIMENTAL). */
int radmm_build_features(void);

/* Hyperparams defaults / validate (admm.hpp:32-57). */
int radmm_hyperparams_default(radmm_hyperparams* out);
int radmm_hyperparams_validate(const radmm_hyperparams* h);

/* ---- Problem (admm.hpp:60-81) ------------------------------------------ */
/* A context owns one Problem on one GPU: n_sensors operators over
 * n_pixels.  For sharded runs (run_distributed, runtime.hpp:768-775) the
 * context owns sensors [q_begin, q_end) of q_total; see radmm_ctx_create_sharded. */
int radmm_ctx_create(int device, int n_pixels, int n_sensors, radmm_ctx** out);
int radmm_ctx_destroy(radmm_ctx* ctx);

/* ForwardOperator::from_matrix (forward_model.hpp:126-133).  q is the
 * 0-based LOCAL sensor slot; rows = K*M of that sensor (ragged allowed);
 * a points at a column-major rows x n_pixels matrix with leading
 * dimension lda >= rows.  The device copy is complex64.  Returns once the
 * host buffer has been consumed (the reference's copy semantics); the
 * sensor's full-set capacitance Gram then keeps running on the device,
 * overlapping the next sensor's upload (consumed by the first radmm_run). */
int radmm_set_operator_c64(radmm_ctx* ctx, int q, int rows, const float* a, int64_t lda, int ptr_kind);
int radmm_set_operator_c128(radmm_ctx* ctx, int q, int rows, const double* a, int64_t lda, int ptr_kind);
/* Measurement y_q (Problem::measurements), complex128, length rows. */
int radmm_set_measurement(radmm_ctx* ctx, int q, const double* y, int ptr_kind);
/* Device generator for the BASELINE dechirped-LFM operator of one sensor:
 * A[m*K+k, n] = exp(j 2 pi (alpha tau t_k + fc tau + phi_n)),
 * tau = (|tx - p_n| + |rx_m - p_n|)/c, t_k = k*T/K; phi_n in TURNS (cycles,
 * [0,1)).  pix: N x 3, rx: M x 3, tx: 3, phi: N (host arrays).  IEEE basic
 * operations only (portable sincos), bitwise equal to the host generator
 * scenario.baseline_operator on any machine. */
int radmm_generate_dechirp_operator(radmm_ctx* ctx, int q, int M, int K, const double* pix,
                                    const double* tx, const double* rx, const double* phi,
                                    double fc, double bw, double pulse);
/* Device assembly of the reference's own operator, EchoKernel::entry +
 * ForwardOperator::dense (forward_model.hpp:32-114): row m*K + k, pixel n,
 *   tau = (|tx - p_n| + |rx_m - p_n|)/c,  t = k/fs - tau,
 *   a = exp(j(-2 pi fc tau + pi alpha t^2)) for 0 <= t <= T, else 0,
 * stored as complex64.  pix: N x 3, rx: M x 3, tx: 3 (host arrays); K from
 * the reference's derive_sample_count (host side). */
int radmm_generate_echo_operator(radmm_ctx* ctx, int q, int M, int K, const double* pix, const double* tx,
                                 const double* rx, double fc, double sample_rate, double chirp_rate,
                                 double pulse_duration);
/* Copy a sensor's device operator back (complex64, column-major, ld = rows). */
int radmm_get_operator_c64(radmm_ctx* ctx, int q, float* out);

/* ---- run (admm.hpp:357-445) --------------------------------------------- */
int radmm_run(radmm_ctx* ctx, const radmm_hyperparams* hyper, const radmm_run_options* opts,
              radmm_run_summary* summary);

/* RunResult accessors (admm.hpp:324-335), valid after radmm_run. */
int radmm_get_image(radmm_ctx* ctx, double* out);                 /* N doubles |x_G| */
int radmm_get_vector(radmm_ctx* ctx, radmm_vector which, double* out); /* N complex128 */
int radmm_get_sensor_image(radmm_ctx* ctx, int q, double* out);   /* x_q, N complex128 */
int radmm_get_record_count(radmm_ctx* ctx, int* count);
int radmm_get_records(radmm_ctx* ctx, radmm_iteration_record* out, int capacity);
/* active_sizes[k*Q + q] for every recorded iteration k (local sensors). */
int radmm_get_active_sizes(radmm_ctx* ctx, int32_t* out, int capacity);
/* Current active set J_q (sorted pixel indices); *count receives N_q. */
int radmm_get_active_set(radmm_ctx* ctx, int q, int32_t* out, int* count);
/* Per-iteration per-sensor active-set history for mask parity: the active
 * set of sensor q after screening at iteration k is reconstructed from the
 * removal log: removed pixels of (k, q) in order. */
int radmm_get_removal_log_size(radmm_ctx* ctx, int* entries);
/* Each entry: iteration, sensor, pixel (3 int32 per entry). */
int radmm_get_removal_log(radmm_ctx* ctx, int32_t* out, int capacity);

/* ---- LocalSolveCache (solver_core.hpp:30-66) and soft_threshold (:14-23) */
/* factorize(a_hat, mu, beta): a_hat column-major rows x cols complex128
 * (stored complex64 on the device).  Forms the rows x rows capacitance or
 * the cols x cols Gram (whichever is smaller) and inverts it on the GPU. */
int radmm_factorize(int device, int rows, int cols, const double* a_hat, double mu, double beta,
                    radmm_solve_cache** out);
int radmm_solve_local(radmm_solve_cache* cache, const double* rhs, double* x);
int radmm_solve_cache_destroy(radmm_solve_cache* cache);
int radmm_soft_threshold(int device, const double* v, int64_t n, double kappa, double* out);

/* ---- operator application (forward_model.hpp:147-177) ------------------ */
/* y = A_q x (x: N complex128, y: rows complex128), host buffers. */
int radmm_apply_operator(radmm_ctx* ctx, int q, const double* x, double* y);
/* x = A_q^H y (y: rows complex128, x: N complex128), host buffers. */
int radmm_apply_adjoint(radmm_ctx* ctx, int q, const double* y, double* x);

/* ---- Multi-frame batches (BASELINE config 5) -------------------------------
 * F independent scenes observed through the same operators (the reference
 * solves them one after another: one run(problem_f, ...) per frame,
 * proj/include/radmm/admm.hpp:357-445).  Frame f is a child context that
 * views this context's operators (no copy) and owns everything that depends
 * on its measurements.  Setting an operator on the parent drops its frames. */
/* Measurement of sensor q in frame f (creates frames 0..f on first use). */
int radmm_set_frame_measurement(radmm_ctx* ctx, int frame, int q, const double* y, int ptr_kind);
/* Run frames 0..frames-1 in lockstep, frame f with hypers[f]; each frame stops
 * on its own rule exactly as run() on that frame alone would.  summaries:
 * frames entries (may be NULL).  Observers are not supported here. */
int radmm_run_frames(radmm_ctx* ctx, int frames, const radmm_hyperparams* hypers, const radmm_run_options* opts,
                     radmm_run_summary* summaries);
/* Borrowed handle of frame f: every radmm_get_* result getter works on it.
 * Owned by ctx (radmm_ctx_destroy refuses it). */
int radmm_frame(radmm_ctx* ctx, int frame, radmm_ctx** out);

/* Matched-filter image |sum_q A_q^H y_q| normalised to unit peak, on the
 * resident operators and measurements (an all-zero result stays all-zero).
 * Replaces back_projection(operators, measurements)
 * (proj/include/radmm/forward_model.hpp:201-220).  image: N doubles.
 * Sharded contexts: collective over all ranks (every rank gets the image). */
int radmm_back_projection(radmm_ctx* ctx, double* image);

/* ---- device-side measurement ------------------------------------------- */
/* Phases of one iteration, timed with CUDA events on the context's stream
 * when profiling is enabled; bytes are ALGORITHMIC bytes. */
typedef enum {
  RADMM_PHASE_FORWARD = 0,   /* v = A_J rhs (+ rhs prologue, partial reduce) */
  RADMM_PHASE_GAPPLY = 1,    /* w = G v (capacitance inverse apply)          */
  RADMM_PHASE_ADJOINT = 2,   /* x = (rhs - mu A_J^H w)/beta + scatter/ring   */
  RADMM_PHASE_PRIMAL = 3,    /* x = Hinv rhs (primal form sensors)           */
  RADMM_PHASE_EXCHANGE = 4,  /* NCCL all-gather of sensor images             */
  RADMM_PHASE_FUSION = 5,    /* average, threshold, dual, norms, stop rule   */
  RADMM_PHASE_SCREEN = 6,    /* zeta + ballot/prefix-sum compaction          */
  RADMM_PHASE_REFACTOR = 7,  /* frozen echo, data term, downdate / rebuild   */
  RADMM_PHASE_SWEEP = 8,     /* fused adjoint(k) + fusion(k) + forward(k+1)  */
  RADMM_PHASE_COUNT = 9
} radmm_phase;

typedef struct {
  int64_t calls;     /* times the phase ran */
  int64_t launches;  /* kernels launched by it */
  double total_ms;   /* device time (CUDA events) */
  double bytes;      /* algorithmic bytes moved */
} radmm_phase_stat;

/* Page-locked host memory for operator buffers (cudaHostAlloc, portable):
 * what a caller stages large problems in so the uploads run at PCIe/C2C
 * speed (config 3: 137 GB of operators).  Not part of the reference API. */
int radmm_host_alloc(size_t bytes, void** out);
int radmm_host_free(void* p);

/* radmm_ctx_destroy returns once the context's device memory is back in the
 * library's stream-ordered pool (the next context reuses it at once); the pool
 * gives everything above RADMM_POOL_KEEP_GB back to the driver from a
 * background thread (config 3: 172 GB, seconds of driver work).  This call
 * waits for that thread and trims synchronously -- for callers that want the
 * memory available to other allocators right away.  Not part of the reference
 * API (the reference's host memory is freed by its destructors). */
int radmm_pool_trim(int device);

int radmm_set_profiling(radmm_ctx* ctx, int enabled);
/* out[RADMM_PHASE_COUNT], accumulated over the last run. */
int radmm_get_phase_stats(radmm_ctx* ctx, radmm_phase_stat* out);
/* Device time (CUDA events) and kernel launches of each iteration of the
 * last run (screening + refactor + local updates + exchange + fusion). */
int radmm_get_iteration_stats(radmm_ctx* ctx, double* device_ms, int64_t* launches, int capacity);

/* ---- sharded runs over NCCL (runtime.hpp:768-775 analogue) ------------- */
/* 128-byte NCCL unique id, produced on rank 0 and broadcast by the caller. */
int radmm_nccl_unique_id(uint8_t out[128]);
/* Transport timeout of a sharded context (default 60000 ms; env
 * RADMM_NCCL_TIMEOUT_MS at creation): a collective or iteration that does not
 * complete in time aborts the communicator and returns RADMM_TRANSPORT -- the
 * reference's tcp_timeout_ms / TransportError (runtime.hpp:540-545,739-775). */
int radmm_set_transport_timeout(radmm_ctx* ctx, int timeout_ms);
int radmm_ctx_create_sharded(int device, int n_pixels, int q_total, int q_begin, int q_end,
                             int rank, int world_size, const uint8_t nccl_id[128],
                             radmm_ctx** out);

#ifdef __cplusplus
}
#endif
#endif /* RADMM_B200_H */
