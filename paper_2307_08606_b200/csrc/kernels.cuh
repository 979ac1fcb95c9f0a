// sm_100a kernels of the ASADMM iteration loop.
//
// Data layout in HBM:
//   * A_q        complex64, column-major, leading dimension ld_q =
//                roundup(rows_q, 64) (zero-padded rows), so every pixel's
//                column is a 512-B aligned contiguous run.  Never moved:
//                elimination compacts the index list J_q instead and every
//                matvec streams only the active columns A(:, J_q).
//   * G_q        complex128 inverse of the rows x rows capacitance
//                beta I + mu A_J A_J^H (dual form) or of the N_q x N_q
//                Gram mu A_J^H A_J + beta I (primal form), column-major.
//   * solver state (x_full, x_hat, rhs, data, s, x_G, sigma, gap) complex128;
//     screening ring of |x_k - x_{k-1}|, W x N doubles per sensor.
// Arithmetic: A is promoted to fp64 in registers; all products and sums are
// fp64 (the fp64 oracle sees the very same complex64 operator values).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace radmm_dev {

constexpr int kWarp = 32;
constexpr int kMaxBatch = 64;

// Per-sensor job descriptors travel as __grid_constant__ kernel parameters
// (no device-side descriptor arrays, no extra copies per launch).
template <typename T>
struct Pack {
  T j[kMaxBatch];
};

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_scale(double2 a, double s) {
  return make_double2(__dmul_rn(a.x, s), __dmul_rn(a.y, s));
}
__device__ __forceinline__ double c_abs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double c_norm2(double2 a) { return a.x * a.x + a.y * a.y; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// acc += conj(a) * v  (4 DFMA)
__device__ __forceinline__ void cfma_conj(double& re, double& im, double ar, double ai, double2 v) {
  re = fma(ar, v.x, re);
  re = fma(ai, v.y, re);
  im = fma(ar, v.y, im);
  im = fma(-ai, v.x, im);
}
// acc += a * c  (4 DFMA)
__device__ __forceinline__ void cfma(double& re, double& im, double ar, double ai, double2 c) {
  re = fma(ar, c.x, re);
  re = fma(-ai, c.y, re);
  im = fma(ar, c.y, im);
  im = fma(ai, c.x, im);
}

// ---------------------------------------------------------------------------
// Column-dot kernel: out_i = sum_r conj(M[r, col_i]) * vec[r] for the active
// columns, with a per-use epilogue.  One warp per column: each lane streams
// 16-B vector loads down the contiguous column, the vector sits in shared
// memory, and the warp reduces with shuffles.  Used for
//   * the adjoint matvec A_J^H w fused with the x-update (EPI_XDUAL),
//   * the capacitance/Gram-inverse apply G v (EPI_STORE, G Hermitian),
//   * the primal x-update Hinv rhs (EPI_XPRIMAL),
//   * the data term mu A_J^H y_eff on rebuild (EPI_STORE, scale mu).
// ---------------------------------------------------------------------------
enum { EPI_STORE = 0, EPI_XDUAL = 1, EPI_XPRIMAL = 2 };

struct ColDotJob {
  const void* M;       // float2* (A) or double2* (G / Hinv)
  int64_t ld;          // leading dimension in complex elements (multiple of 64 / 32)
  int len;             // rows participating (<= ld); vec is zero-padded to ld
  int n_out;           // number of output columns
  const int* cols;     // matrix column of output i (nullptr: identity)
  const int* pix;      // pixel index of output i for the x-update epilogue
  const double2* vec;  // input vector (len entries)
  double2* out;        // EPI_STORE destination
  double scale;        // EPI_STORE scale
  const double2* rhs;  // EPI_XDUAL: rhs_i
  double2* x_hat;      // x-update outputs (compacted)
  double2* x_full;     // x-update scatter target (N)
  double* ring_slot;   // screening ring row for this update (N doubles)
  int64_t vld;         // rows of vec staged in shared memory (0: ld); < ld for row segments
};

// Columns per warp (CPW): each vector element fetched from shared memory
// feeds CPW columns (CPW x fewer LDS per HBM byte) and each lane keeps
// 2*CPW independent 16-B loads in flight.
constexpr int kCPW = 4;  // upper bound (ColDot launch picks 1, 2 or 4)

template <typename T, int CPW>
struct ColLoad;

// complex64 operator columns.  The shared vector is stored split by row
// parity (sv_e[i] = vec[2i], sv_o[i] = vec[2i+1]) so a lane's two complex
// values for its float4 are two conflict-free 16-B loads.
template <int CPW>
struct ColLoad<float2, CPW> {
  static constexpr int kRowsPerStep = 64;
  __device__ static __forceinline__ void dot(const void* base, int64_t ld, const int (&col)[CPW], int steps,
                                             const double2* __restrict__ sv, int64_t half, int lane,
                                             double (&re)[CPW], double (&im)[CPW]) {
    const float4* p[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      p[c] = reinterpret_cast<const float4*>(reinterpret_cast<const float2*>(base) + (int64_t)col[c] * ld) + lane;
      re[c] = 0.0;
      im[c] = 0.0;
    }
    const double2* ve = sv + lane;
    const double2* vo = sv + half + lane;
    int s = 0;
#pragma unroll 1
    for (; s + 2 <= steps; s += 2) {
      float4 a0[CPW], a1[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) a0[c] = __ldg(p[c] + (s + 0) * 32);
#pragma unroll
      for (int c = 0; c < CPW; ++c) a1[c] = __ldg(p[c] + (s + 1) * 32);
      const double2 e0 = ve[(s + 0) * 32], o0 = vo[(s + 0) * 32];
      const double2 e1 = ve[(s + 1) * 32], o1 = vo[(s + 1) * 32];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        cfma_conj(re[c], im[c], a0[c].x, a0[c].y, e0);
        cfma_conj(re[c], im[c], a0[c].z, a0[c].w, o0);
        cfma_conj(re[c], im[c], a1[c].x, a1[c].y, e1);
        cfma_conj(re[c], im[c], a1[c].z, a1[c].w, o1);
      }
    }
    for (; s < steps; ++s) {
      const double2 e0 = ve[s * 32], o0 = vo[s * 32];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const float4 a0 = __ldg(p[c] + s * 32);
        cfma_conj(re[c], im[c], a0.x, a0.y, e0);
        cfma_conj(re[c], im[c], a0.z, a0.w, o0);
      }
    }
  }
  // smem layout: even rows then odd rows
  __device__ static __forceinline__ int64_t slot(int64_t r, int64_t half) { return (r & 1) ? half + (r >> 1) : (r >> 1); }
};

// complex128 matrices (capacitance inverse G, primal Hinv).
template <int CPW>
struct ColLoad<double2, CPW> {
  static constexpr int kRowsPerStep = 32;
  __device__ static __forceinline__ void dot(const void* base, int64_t ld, const int (&col)[CPW], int steps,
                                             const double2* __restrict__ sv, int64_t /*half*/, int lane,
                                             double (&re)[CPW], double (&im)[CPW]) {
    const double2* p[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      p[c] = reinterpret_cast<const double2*>(base) + (int64_t)col[c] * ld + lane;
      re[c] = 0.0;
      im[c] = 0.0;
    }
    const double2* v = sv + lane;
    int s = 0;
#pragma unroll 1
    for (; s + 2 <= steps; s += 2) {
      double2 a0[CPW], a1[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) a0[c] = __ldg(p[c] + (s + 0) * 32);
#pragma unroll
      for (int c = 0; c < CPW; ++c) a1[c] = __ldg(p[c] + (s + 1) * 32);
      const double2 v0 = v[(s + 0) * 32], v1 = v[(s + 1) * 32];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        cfma_conj(re[c], im[c], a0[c].x, a0[c].y, v0);
        cfma_conj(re[c], im[c], a1[c].x, a1[c].y, v1);
      }
    }
    for (; s < steps; ++s) {
      const double2 v0 = v[s * 32];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const double2 a0 = __ldg(p[c] + s * 32);
        cfma_conj(re[c], im[c], a0.x, a0.y, v0);
      }
    }
  }
  __device__ static __forceinline__ int64_t slot(int64_t r, int64_t) { return r; }
};

// Fallback dot for vectors too long for shared memory (rows > ~12k, e.g. the
// reference desk scenario's 24568-row operators): the vector is read through
// L1/L2 with a bounds check.  Only used on rebuild paths.
template <typename T>
__device__ __forceinline__ void dot_global(const void* base, int64_t ld, int col, int len, const double2* __restrict__ vec,
                                           int lane, double& re, double& im) {
  re = 0.0;
  im = 0.0;
  const T* p = reinterpret_cast<const T*>(base) + (int64_t)col * ld;
  for (int r = lane; r < len; r += 32) {
    const T a = p[r];
    cfma_conj(re, im, (double)a.x, (double)a.y, __ldg(vec + r));
  }
}

template <int EPI>
__device__ __forceinline__ void coldot_epilogue(const ColDotJob& jb, int i, double re, double im, double mu,
                                                double beta) {
  if (EPI == EPI_STORE) {
    jb.out[i] = make_double2(__dmul_rn(jb.scale, re), __dmul_rn(jb.scale, im));
  } else {
    double2 xh;
    if (EPI == EPI_XDUAL) {
      // x = (rhs - mu * A^H w) / beta  (Woodbury form of solver_core.hpp:47-51)
      const double2 r = jb.rhs[i];
      xh = make_double2(__ddiv_rn(__dsub_rn(r.x, __dmul_rn(mu, re)), beta),
                        __ddiv_rn(__dsub_rn(r.y, __dmul_rn(mu, im)), beta));
    } else {
      xh = make_double2(re, im);
    }
    const int p = jb.pix[i];
    const double2 old = jb.x_full[p];
    jb.ring_slot[p] = c_abs(c_sub(xh, old));  // |hist[h][j] - hist[h-1][j]| (admm.hpp:143)
    jb.x_full[p] = xh;                        // admm.hpp:121-122
    jb.x_hat[i] = xh;                         // admm.hpp:120
  }
}

// THREADS = 256 normally; 1024 when the shared vector is so large (KM = 8192:
// 128 KB) that only one CTA fits per SM, to keep enough loads in flight.
template <typename T, int EPI, bool SMEM_VEC, int CPW, int THREADS>
__global__ void __launch_bounds__(THREADS) coldot_kernel(const __grid_constant__ Pack<ColDotJob> jobs, double mu, double beta,
                                                         const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  extern __shared__ double2 sv[];
  constexpr int kWarps = THREADS / 32;
  const ColDotJob& jb = jobs.j[blockIdx.y];
  const int n_out = jb.n_out;
  // balanced contiguous column range per warp (sizes differ by <= 1)
  const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const int i_begin = (int)(gw * n_out / nw);
  const int i_end = (int)((gw + 1) * n_out / nw);
  if ((int)((int64_t)blockIdx.x * kWarps * n_out / nw) >= n_out) return;  // whole CTA idle
  const int64_t ld = jb.ld;
  const int64_t vld = jb.vld ? jb.vld : ld;
  const int64_t half = vld >> 1;
  if (SMEM_VEC) {
    for (int r = threadIdx.x; r < vld; r += blockDim.x)
      sv[ColLoad<T, CPW>::slot(r, half)] = (r < jb.len) ? jb.vec[r] : make_double2(0.0, 0.0);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int steps = (int)((jb.len + ColLoad<T, CPW>::kRowsPerStep - 1) / ColLoad<T, CPW>::kRowsPerStep);
  for (int i0 = i_begin; i0 < i_end; i0 += CPW) {
    if (SMEM_VEC) {
      int col[CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int i = min(i0 + c, i_end - 1);
        col[c] = jb.cols ? jb.cols[i] : i;
      }
      double re[CPW], im[CPW];
      ColLoad<T, CPW>::dot(jb.M, ld, col, steps, sv, half, lane, re, im);
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        re[c] = warp_sum(re[c]);
        im[c] = warp_sum(im[c]);
      }
#pragma unroll
      for (int c = 0; c < CPW; ++c)
        if (lane == c && i0 + c < i_end) coldot_epilogue<EPI>(jb, i0 + c, re[c], im[c], mu, beta);
    } else {
      for (int c = 0; c < CPW && i0 + c < i_end; ++c) {
        const int i = i0 + c;
        const int col = jb.cols ? jb.cols[i] : i;
        double re, im;
        dot_global<T>(jb.M, ld, col, jb.len, jb.vec, lane, re, im);
        re = warp_sum(re);
        im = warp_sum(im);
        if (lane == 0) coldot_epilogue<EPI>(jb, i, re, im, mu, beta);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Forward kernel: v = sum_i A[:, J_i] * coef_i over a chunk of active columns
// (rows in 512-row tiles, 2 complex per thread via float4), with the
// coefficient prologue fused:
//   MODE_RHS:    coef_i = data_i + beta gap[J_i] + beta x_hat_i - sigma[J_i]
//                (rhs of admm.hpp:114-119, also written out for the x-update)
//   MODE_GATHER: coef_i = src[J_i]  (frozen-echo update of y_eff, admm.hpp:174-176)
// Partial sums per chunk are reduced by reduce_parts_kernel in fixed order.
// ---------------------------------------------------------------------------
enum { MODE_RHS = 0, MODE_GATHER = 1 };

struct FwdJob {
  const float2* A;
  int64_t ld;
  int n;               // columns in the list
  const int* J;        // column (pixel) list
  const double2* data; // MODE_RHS
  const double2* x_hat;
  double2* rhs_out;
  const double2* src;  // MODE_GATHER
  double2* part;       // [n_chunks][ld]
  int n_chunks;
  int chunk_len;
};

constexpr int kFwdThreads = 256;
constexpr int kFwdTile = 2 * kFwdThreads;

template <int MODE>
__global__ void __launch_bounds__(kFwdThreads) fwd_kernel(const __grid_constant__ Pack<FwdJob> jobs,
                                                          const double2* __restrict__ gap,
                                                          const double2* __restrict__ sigma, double beta,
                                                          const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  extern __shared__ unsigned char smem_raw[];
  const FwdJob& jb = jobs.j[blockIdx.z];
  const int chunk = blockIdx.x;
  if (chunk >= jb.n_chunks) return;
  const int64_t row0 = (int64_t)blockIdx.y * kFwdTile;
  if (row0 >= jb.ld) return;
  const int i0 = chunk * jb.chunk_len;
  const int cnt = min(jb.chunk_len, jb.n - i0);
  double2* coef = reinterpret_cast<double2*>(smem_raw);
  int* cidx = reinterpret_cast<int*>(coef + jb.chunk_len);
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
    const int i = i0 + t;
    const int c = jb.J[i];
    double2 v;
    if (MODE == MODE_RHS) {
      const double2 d = jb.data[i], g = gap[c], xh = jb.x_hat[i], sg = sigma[c];
      v.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
      v.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
      if (blockIdx.y == 0) jb.rhs_out[i] = v;
    } else {
      v = jb.src[c];
    }
    coef[t] = v;
    cidx[t] = c;
  }
  __syncthreads();
  const int64_t r = row0 + 2 * threadIdx.x;
  double a0r = 0, a0i = 0, a1r = 0, a1i = 0;
  double b0r = 0, b0i = 0, b1r = 0, b1i = 0;
  if (r < jb.ld) {
    const float2* A = jb.A + r;
    int t = 0;
#pragma unroll 1
    for (; t + 8 <= cnt; t += 8) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(A + (int64_t)cidx[t + u] * jb.ld));
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const double2 c0 = coef[t + u], c1 = coef[t + u + 1];
        cfma(a0r, a0i, x[u].x, x[u].y, c0); cfma(a1r, a1i, x[u].z, x[u].w, c0);
        cfma(b0r, b0i, x[u + 1].x, x[u + 1].y, c1); cfma(b1r, b1i, x[u + 1].z, x[u + 1].w, c1);
      }
    }
    for (; t < cnt; ++t) {
      const float4 x0 = __ldg(reinterpret_cast<const float4*>(A + (int64_t)cidx[t] * jb.ld));
      const double2 c0 = coef[t];
      cfma(a0r, a0i, x0.x, x0.y, c0); cfma(a1r, a1i, x0.z, x0.w, c0);
    }
    double2* out = jb.part + (int64_t)chunk * jb.ld + r;
    out[0] = make_double2(a0r + b0r, a0i + b0i);
    out[1] = make_double2(a1r + b1r, a1i + b1i);
  }
}

// out[r] = base[r] + sign * sum_c part[c][r]   (fixed chunk order)
struct ReduceJob {
  const double2* part;
  int n_chunks;
  int64_t ld;
  int len;
  const double2* base;  // may be nullptr
  double2* out;
  double sign;
};

__global__ void reduce_parts_kernel(const __grid_constant__ Pack<ReduceJob> jobs, const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  const ReduceJob& jb = jobs.j[blockIdx.y];
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= jb.ld) return;
  double sr = 0, si = 0;
  if (r < jb.len) {
    for (int c = 0; c < jb.n_chunks; ++c) {
      const double2 v = jb.part[(int64_t)c * jb.ld + r];
      sr += v.x;
      si += v.y;
    }
  }
  double2 o;
  if (jb.base) {
    const double2 b = (r < jb.len) ? jb.base[r] : make_double2(0, 0);
    o = make_double2(b.x + jb.sign * sr, b.y + jb.sign * si);
  } else {
    o = make_double2(jb.sign * sr, jb.sign * si);
  }
  jb.out[r] = (r < jb.len) ? o : make_double2(0, 0);
}

// rhs_i = data_i + beta gap[J_i] + beta x_hat_i - sigma[J_i] (primal sensors)
struct RhsJob {
  int n;
  const int* J;
  const double2* data;
  const double2* x_hat;
  double2* rhs;
};

__global__ void rhs_kernel(const __grid_constant__ Pack<RhsJob> jobs, const double2* __restrict__ gap,
                           const double2* __restrict__ sigma, double beta, const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  const RhsJob& jb = jobs.j[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= jb.n) return;
  const int c = jb.J[i];
  const double2 d = jb.data[i], g = gap[c], xh = jb.x_hat[i], sg = sigma[c];
  double2 v;
  v.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
  v.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
  jb.rhs[i] = v;
}

// ---------------------------------------------------------------------------
// Fusion: FusionCore::round (admm.hpp:236-258) for N pixels, then the five
// squared norms reduced deterministically (per-block partials, last block
// sums them in fixed order) and the stopping rule evaluated on the device.
// ---------------------------------------------------------------------------
struct FusionScalars {
  double pri_res, dual_res, eps_pri, eps_dual;
  double sq[5];
  int trigger, converged;
  int iteration;
  int pad;
};

struct FusionArgs {
  const double2* const* contrib;  // Q sensor images x_q (mirror == x_full)
  int Q;
  int N;
  double2* s;
  double2* xg;
  double2* sigma;
  double2* sigma_pre;
  double2* gap;
  double beta, kappa;
  double root_n_eps_abs, eps_rel;
  int has_prev;
  int iteration;
  double* partials;        // [gridDim.x * 5]
  unsigned int* counter;
  FusionScalars* out_dev;
  FusionScalars* out_host; // mapped pinned memory
  // device-guarded speculation: this round runs only if *go != 0; it then
  // decides whether the next (already enqueued) round may run
  const int* go;
  int* go_next;
  int stop_on_converge;     // !fixed_iterations
  int screen_next_possible; // ASADMM, screening enabled, history full after this round
};

constexpr int kFusionThreads = 256;

__device__ __forceinline__ double2 soft_threshold1(double2 v, double kappa) {
  const double mag = c_abs(v);  // std::abs(complex) (solver_core.hpp:18)
  if (mag > kappa) {
    const double f = __dsub_rn(1.0, __ddiv_rn(kappa, mag));
    return make_double2(__dmul_rn(v.x, f), __dmul_rn(v.y, f));
  }
  return make_double2(0.0, 0.0);
}

// FusionCore::round for one pixel j; accumulates the five squared norms.
// contrib(k) returns sensor k's image value at j.
template <typename Contrib>
__device__ __forceinline__ void fusion_pixel(const FusionArgs& a, int j, Contrib contrib, double (&q)[5]) {
  double2 s = make_double2(0.0, 0.0);
  for (int k = 0; k < a.Q; ++k) s = c_add(s, contrib(k));  // fixed sensor order (admm.hpp:239)
  s = make_double2(__ddiv_rn(s.x, (double)a.Q), __ddiv_rn(s.y, (double)a.Q));
  const double2 xgp = a.xg[j];
  const double2 sg = a.sigma[j];
  a.sigma_pre[j] = sg;
  const double2 v = make_double2(__dadd_rn(s.x, __ddiv_rn(sg.x, a.beta)), __dadd_rn(s.y, __ddiv_rn(sg.y, a.beta)));
  const double2 xg = soft_threshold1(v, a.kappa);
  const double2 eta = c_sub(s, xg);
  const double2 dx = c_sub(xg, xgp);
  const double2 sn = make_double2(__dadd_rn(sg.x, __dmul_rn(a.beta, eta.x)), __dadd_rn(sg.y, __dmul_rn(a.beta, eta.y)));
  a.s[j] = s;
  a.xg[j] = xg;
  a.sigma[j] = sn;
  a.gap[j] = c_sub(xg, s);
  q[0] += c_norm2(eta);
  q[1] += c_norm2(dx);
  q[2] += c_norm2(s);
  q[3] += c_norm2(xg);
  q[4] += c_norm2(sn);
}

// Block-reduce the five partial sums, publish them, and let the last block of
// the grid reduce all blocks in fixed order and evaluate the stopping rule
// (admm.hpp:244-256).  Deterministic for a fixed grid.
__device__ __forceinline__ void fusion_finish(const FusionArgs& a, double (&q)[5], int nblocks, int bid) {
  __shared__ double red[5][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const double w = warp_sum(q[t]);
    if (lane == 0) red[t][warp] = w;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double acc = 0;
    for (int w = 0; w < nwarps; ++w) acc += red[threadIdx.x][w];
    a.partials[bid * 5 + threadIdx.x] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(a.counter, 1u) == (unsigned)nblocks - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // all threads stage the block partials into shared memory in parallel, then
  // threads 0..4 add them in block order (the same order, bitwise, as a
  // sequential walk -- without its ~nblocks dependent L2 round trips)
  __shared__ double stage[5 * 64];
  double acc = 0.0;
  for (int b0 = 0; b0 < nblocks; b0 += 64) {
    const int nb = min(64, nblocks - b0);
    for (int e = threadIdx.x; e < 5 * nb; e += blockDim.x)
      stage[e] = ((volatile double*)a.partials)[b0 * 5 + e];
    __syncthreads();
    if (threadIdx.x < 5)
      for (int b = 0; b < nb; ++b) acc += stage[b * 5 + threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x < 5) red[threadIdx.x][0] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    FusionScalars f;
    for (int t = 0; t < 5; ++t) f.sq[t] = red[t][0];
    f.pri_res = sqrt(f.sq[0]);
    f.dual_res = a.beta * sqrt(f.sq[1]);
    f.eps_pri = a.root_n_eps_abs + a.eps_rel * fmax(sqrt(f.sq[2]), sqrt(f.sq[3]));
    f.eps_dual = a.root_n_eps_abs + a.eps_rel * sqrt(f.sq[4]);
    f.trigger = f.pri_res <= f.eps_pri;
    f.converged = a.has_prev && f.trigger && f.dual_res <= f.eps_dual;
    if (a.go_next)
      *a.go_next = !((a.stop_on_converge && f.converged) || (a.screen_next_possible && f.trigger));
    f.iteration = a.iteration;
    f.pad = 0;
    *a.out_dev = f;
    if (a.out_host) {
      volatile FusionScalars* h = a.out_host;
      h->pri_res = f.pri_res; h->dual_res = f.dual_res; h->eps_pri = f.eps_pri; h->eps_dual = f.eps_dual;
      for (int t = 0; t < 5; ++t) h->sq[t] = f.sq[t];
      h->trigger = f.trigger; h->converged = f.converged;
      __threadfence_system();
      h->iteration = f.iteration;
    }
    *a.counter = 0u;
  }
}

// whole grid = one fusion round
__device__ __forceinline__ void fusion_finish(const FusionArgs& a, double (&q)[5]) {
  fusion_finish(a, q, gridDim.x * gridDim.y * gridDim.z,
                blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
}

__global__ void __launch_bounds__(kFusionThreads) fusion_kernel(FusionArgs a) {
  if (a.go && __ldg(a.go) == 0) return;  // cancelled speculative iteration
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double q[5] = {0, 0, 0, 0, 0};
  if (j < a.N) fusion_pixel(a, j, [&](int k) { return a.contrib[k][j]; }, q);
  fusion_finish(a, q);
}

// One fusion round per frame of a multi-frame batch (blockIdx.y = frame);
// each frame reduces over its own row of blocks with its own counter.
__global__ void __launch_bounds__(kFusionThreads) fusion_frames_kernel(const __grid_constant__ Pack<FusionArgs> P) {
  const FusionArgs& a = P.j[blockIdx.y];
  if (a.go && __ldg(a.go) == 0) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double q[5] = {0, 0, 0, 0, 0};
  if (j < a.N) fusion_pixel(a, j, [&](int k) { return a.contrib[k][j]; }, q);
  fusion_finish(a, q, gridDim.x, blockIdx.x);
}

// ---------------------------------------------------------------------------
// Screening (SensorCore::screen, admm.hpp:134-159) as a warp-ballot /
// prefix-sum stream compaction of the active list.
//   zeta_i = (1/W) sum_{t=0}^{W-1} ring[(upd-W+t) mod W][J_i]  (oldest first)
//   keep   = zeta_i >= tol
// ---------------------------------------------------------------------------
constexpr int kScanBlock = 1024;

struct ScreenJob {
  int n;
  const int* J;
  const double* ring;     // W x N
  int64_t ring_stride;    // N
  int first_slot;         // (upd - W) mod W
  unsigned char* keep;    // n flags
  int* block_counts;      // ceil(n / kScanBlock)
  int* block_offsets;
  int* totals;            // [0] = kept
  int* Jnew;
  int* keep_pos;          // old compacted index of kept entry
  int* rem_pix;           // removed pixel indices (in order)
  int* rem_pos;           // removed old compacted positions
  const double2* x_hat;
  double2* x_hat_new;
  const double2* data;  // compacted with J: the (possibly lagged) data term
  double2* data_new;
};

__global__ void __launch_bounds__(kScanBlock) screen_flags_kernel(const __grid_constant__ Pack<ScreenJob> jobs, int W, double tol) {
  const ScreenJob& jb = jobs.j[blockIdx.y];
  __shared__ int wc[kScanBlock / 32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  if ((int)blockIdx.x * kScanBlock >= jb.n) return;
  bool k = false;
  if (i < jb.n) {
    const int c = jb.J[i];
    double z = 0.0;
    for (int t = 0; t < W; ++t) {
      const int slot = (jb.first_slot + t) % W;
      z += jb.ring[(int64_t)slot * jb.ring_stride + c];
    }
    z = z / (double)W;
    k = z >= tol;
    jb.keep[i] = k ? 1 : 0;
  }
  const unsigned b = __ballot_sync(0xffffffffu, k);
  if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) s += wc[w];
    jb.block_counts[blockIdx.x] = s;
  }
}

__global__ void screen_scan_kernel(const __grid_constant__ Pack<ScreenJob> jobs) {
  const ScreenJob& jb = jobs.j[blockIdx.x];
  if (threadIdx.x != 0) return;
  const int nb = (jb.n + kScanBlock - 1) / kScanBlock;
  int s = 0;
  for (int b = 0; b < nb; ++b) {
    jb.block_offsets[b] = s;
    s += jb.block_counts[b];
  }
  jb.totals[0] = s;
}

__global__ void __launch_bounds__(kScanBlock) screen_scatter_kernel(const __grid_constant__ Pack<ScreenJob> jobs) {
  const ScreenJob& jb = jobs.j[blockIdx.y];
  __shared__ int woff[kScanBlock / 32];
  if ((int)blockIdx.x * kScanBlock >= jb.n) return;
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const bool valid = i < jb.n;
  const bool k = valid && jb.keep[i];
  const unsigned b = __ballot_sync(0xffffffffu, k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) woff[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kScanBlock / 32; ++w) {
      const int c = woff[w];
      woff[w] = s;
      s += c;
    }
  }
  __syncthreads();
  if (!valid) return;
  const int kept_before = jb.block_offsets[blockIdx.x] + woff[warp] + __popc(b & ((1u << lane) - 1u));
  if (k) {
    jb.Jnew[kept_before] = jb.J[i];
    jb.keep_pos[kept_before] = i;
    jb.x_hat_new[kept_before] = jb.x_hat[i];  // x_full[J_new] (admm.hpp:153-156)
    jb.data_new[kept_before] = jb.data[i];
  } else {
    const int rpos = i - kept_before;
    jb.rem_pix[rpos] = jb.J[i];
    jb.rem_pos[rpos] = i;
  }
}

// ---------------------------------------------------------------------------
// fp64 complex GEMM, SIMT tiles (64 x 64 x 8, 256 threads, 4 x 4 per thread):
//   C = alpha * op(A) op(B) + beta0 * C  (+ diag) with gathered operands.
// op(M)(i, k): (r, c) = trans ? (k, i) : (i, k); r = ridx ? ridx[r] : r;
// c = cidx ? cidx[c] : c; value M[r + c*ld] (complex64 promoted or
// complex128), conjugated if conj.  Drives the factor builds and
// downdates of LocalSolveCache (solver_core.hpp:34-45) and the
// Gauss-Jordan inverse.
// ---------------------------------------------------------------------------
struct MatRef {
  const void* p;
  int64_t ld;
  const int* ridx;
  const int* cidx;
  int c64;
  int trans;
  int conj;
};

enum { GEPI_PLAIN = 0, GEPI_GJ = 1, GEPI_SPLIT = 2 };

struct GemmJob {
  int m, n, k;
  MatRef a, b;
  double2* c;
  int64_t ldc;
  double alpha, beta0;
  double diag_add;  // C[i,i] += diag_add
  int k0, kb;       // GEPI_GJ: pivot block rows/cols [k0, k0+kb); b = R' (kb x n)
  int herm;         // result is Hermitian: compute tiles with m0 >= n0, mirror conj
};

__device__ __forceinline__ double2 mat_load(const MatRef& m, int i, int k) {
  int r = m.trans ? k : i;
  int c = m.trans ? i : k;
  if (m.ridx) r = m.ridx[r];
  if (m.cidx) c = m.cidx[c];
  double2 v;
  if (m.c64) {
    const float2 f = reinterpret_cast<const float2*>(m.p)[r + (int64_t)c * m.ld];
    v = make_double2((double)f.x, (double)f.y);
  } else {
    v = reinterpret_cast<const double2*>(m.p)[r + (int64_t)c * m.ld];
  }
  if (m.conj) v.y = -v.y;
  return v;
}

constexpr int kGB = 64, kGK = 8;
constexpr int kGjSmem = (64 * 65 + 128) * 16;

// GEPI_SPLIT: split-K for skinny products (the rank-r downdates, r << KM):
// blockIdx.z = job * nsplit + split; each split accumulates its K range and
// stores the raw partial tile to ws[split][m][n]; gemm_split_reduce applies
// alpha / beta0 / diag in fixed split order.
template <int EPI>
__global__ void __launch_bounds__(256) gemm_kernel(const __grid_constant__ Pack<GemmJob> jobs, int nsplit,
                                                   double2* __restrict__ ws, int64_t ws_stride) {
  const int split = blockIdx.z % nsplit;
  const GemmJob& jb = jobs.j[blockIdx.z / nsplit];
  const int m0 = blockIdx.y * kGB, n0 = blockIdx.x * kGB;
  if (m0 >= jb.m || n0 >= jb.n) return;
  if (EPI == GEPI_PLAIN && jb.herm && m0 < n0) return;  // upper tiles come from the mirror
  __shared__ double2 As[2][kGK][kGB];
  __shared__ double2 Bs[2][kGK][kGB];
  const int tid = threadIdx.x;
  // thread (tx, ty) owns rows m0 + tx + 16a and columns n0 + ty + 16b: a warp
  // covers 16 consecutive rows of 2 columns, so the column-major epilogue
  // (the rank-r updates are read-modify-write bound) is coalesced.
  const int tx = tid & 15, ty = tid >> 4;
  double acc_r[4][4], acc_i[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc_r[a][b] = acc_i[a][b] = 0.0;

  const MatRef A = jb.a, B = jb.b;
  auto load_tile = [&](int buf, int kk0) {
    // A tile: kGB (i) x kGK (k)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int e = tid + t * 256;
      int ii, kk;
      if (!A.trans) { ii = e & 63; kk = e >> 6; } else { kk = e & 7; ii = e >> 3; }
      const int gi = m0 + ii, gk = kk0 + kk;
      As[buf][kk][ii] = (gi < jb.m && gk < jb.k) ? mat_load(A, gi, gk) : make_double2(0.0, 0.0);
    }
    // B tile: kGK (k) x kGB (j)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int e = tid + t * 256;
      int kk, jj;
      if (!B.trans) { kk = e & 7; jj = e >> 3; } else { jj = e & 63; kk = e >> 6; }
      const int gj = n0 + jj, gk = kk0 + kk;
      Bs[buf][kk][jj] = (gj < jb.n && gk < jb.k) ? mat_load(B, gk, gj) : make_double2(0.0, 0.0);
    }
  };

  const int nk_all = (jb.k + kGK - 1) / kGK;
  const int per = (nk_all + nsplit - 1) / nsplit;
  const int t0 = split * per;
  const int nk = max(0, min(nk_all, t0 + per) - t0);
  if (nk > 0) load_tile(0, t0 * kGK);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    if (t + 1 < nk) load_tile(cur ^ 1, (t0 + t + 1) * kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      double2 av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[cur][kk][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[cur][kk][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          acc_r[a][b] = fma(av[a].x, bv[b].x, acc_r[a][b]);
          acc_r[a][b] = fma(-av[a].y, bv[b].y, acc_r[a][b]);
          acc_i[a][b] = fma(av[a].x, bv[b].y, acc_i[a][b]);
          acc_i[a][b] = fma(av[a].y, bv[b].x, acc_i[a][b]);
        }
    }
    __syncthreads();
  }
  // read the C tile first (all 16 loads in flight) when it is accumulated into
  double2 cold[4][4];
  if (EPI == GEPI_PLAIN && jb.beta0 != 0.0) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = m0 + tx + 16 * a, j = n0 + ty + 16 * b;
        cold[a][b] = (i < jb.m && j < jb.n) ? jb.c[i + (int64_t)j * jb.ldc] : make_double2(0.0, 0.0);
      }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = m0 + tx + 16 * a;
    if (i >= jb.m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = n0 + ty + 16 * b;
      if (j >= jb.n) continue;
      double2* cp = jb.c + i + (int64_t)j * jb.ldc;
      if (EPI == GEPI_SPLIT) {
        ws[(int64_t)blockIdx.z * ws_stride + (int64_t)j * jb.m + i] = make_double2(acc_r[a][b], acc_i[a][b]);
      } else if (EPI == GEPI_PLAIN) {
        double2 o = make_double2(jb.alpha * acc_r[a][b], jb.alpha * acc_i[a][b]);
        if (jb.beta0 != 0.0) {
          o.x += jb.beta0 * cold[a][b].x;
          o.y += jb.beta0 * cold[a][b].y;
        }
        if (i == j) {
          o.x += jb.diag_add;
          if (jb.herm) o.y = 0.0;  // exact real diagonal of a Hermitian matrix
        }
        if (jb.herm && i < j) continue;  // written (bit-exactly) as the mirror of (j, i)
        *cp = o;
        if (jb.herm && i != j) jb.c[j + (int64_t)i * jb.ldc] = make_double2(o.x, -o.y);
      } else {
        // Gauss-Jordan sweep of pivot block K = [k0, k0+kb):
        //   i in K:      M[i,j] = R'[i-k0, j]
        //   i not in K:  M[i,j] = (j in K ? 0 : M[i,j]) - (F R')[i,j]
        const bool iK = i >= jb.k0 && i < jb.k0 + jb.kb;
        if (iK) {
          *cp = reinterpret_cast<const double2*>(jb.b.p)[(i - jb.k0) + (int64_t)j * jb.b.ld];
        } else {
          const bool jK = j >= jb.k0 && j < jb.k0 + jb.kb;
          const double2 c0 = jK ? make_double2(0.0, 0.0) : *cp;
          *cp = make_double2(c0.x - acc_r[a][b], c0.y - acc_i[a][b]);
        }
      }
    }
  }
}

// Large products (Gram / capacitance builds, Gauss-Jordan rank-64 updates):
// (16 TM) x (16 TN) tiles, TM x TN complex outputs per thread, the next K
// slice prefetched into registers while the current one is multiplied, shared
// rows padded by one element so transposed stores are conflict-free.  Every
// output accumulates over k in the same order with the same FMA sequence as
// gemm_kernel, so the two are bitwise identical.
constexpr int kBigTM = 8, kBigTN = 4;
constexpr int kBigBM = 16 * kBigTM, kBigBN = 16 * kBigTN;
constexpr size_t kGemmBigSmem = (size_t)2 * kGK * ((kBigBM + 1) + (kBigBN + 1)) * sizeof(double2);

template <int EPI>
__global__ void __launch_bounds__(256, 1) gemm_big_kernel(const __grid_constant__ Pack<GemmJob> jobs) {
  constexpr int TM = kBigTM, TN = kBigTN, BM = kBigBM, BN = kBigBN;
  constexpr int LA = BM * kGK / 256, LB = BN * kGK / 256;  // prefetched elements per thread
  const GemmJob& jb = jobs.j[blockIdx.z];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= jb.m || n0 >= jb.n) return;
  if (EPI == GEPI_PLAIN && jb.herm && m0 + BM <= n0) return;  // strictly-upper tiles come from the mirror
  extern __shared__ double2 gsm[];
  double2(*As)[kGK][BM + 1] = reinterpret_cast<double2(*)[kGK][BM + 1]>(gsm);
  double2(*Bs)[kGK][BN + 1] = reinterpret_cast<double2(*)[kGK][BN + 1]>(gsm + 2 * kGK * (BM + 1));
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  double acc_r[TM][TN], acc_i[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc_r[a][b] = acc_i[a][b] = 0.0;
  const MatRef A = jb.a, B = jb.b;
  double2 pa[LA], pb[LB];
  auto a_pos = [&](int e, int& ii, int& kk) {
    if (!A.trans) { ii = e % BM; kk = e / BM; } else { kk = e & 7; ii = e >> 3; }
  };
  auto b_pos = [&](int e, int& jj, int& kk) {
    if (!B.trans) { kk = e & 7; jj = e >> 3; } else { jj = e % BN; kk = e / BN; }
  };
  auto fetch = [&](int kk0) {
#pragma unroll
    for (int t = 0; t < LA; ++t) {
      int ii, kk;
      a_pos(tid + t * 256, ii, kk);
      const int gi = m0 + ii, gk = kk0 + kk;
      pa[t] = (gi < jb.m && gk < jb.k) ? mat_load(A, gi, gk) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int t = 0; t < LB; ++t) {
      int jj, kk;
      b_pos(tid + t * 256, jj, kk);
      const int gj = n0 + jj, gk = kk0 + kk;
      pb[t] = (gj < jb.n && gk < jb.k) ? mat_load(B, gk, gj) : make_double2(0.0, 0.0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int t = 0; t < LA; ++t) {
      int ii, kk;
      a_pos(tid + t * 256, ii, kk);
      As[buf][kk][ii] = pa[t];
    }
#pragma unroll
    for (int t = 0; t < LB; ++t) {
      int jj, kk;
      b_pos(tid + t * 256, jj, kk);
      Bs[buf][kk][jj] = pb[t];
    }
  };
  const int nk = (jb.k + kGK - 1) / kGK;
  if (nk > 0) {
    fetch(0);
    stash(0);
  }
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    if (t + 1 < nk) fetch((t + 1) * kGK);  // in flight during the multiply below
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      double2 av[TM], bv[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) av[a] = As[cur][kk][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < TN; ++b) bv[b] = Bs[cur][kk][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) {
          acc_r[a][b] = fma(av[a].x, bv[b].x, acc_r[a][b]);
          acc_r[a][b] = fma(-av[a].y, bv[b].y, acc_r[a][b]);
          acc_i[a][b] = fma(av[a].x, bv[b].y, acc_i[a][b]);
          acc_i[a][b] = fma(av[a].y, bv[b].x, acc_i[a][b]);
        }
    }
    if (t + 1 < nk) stash(cur ^ 1);  // that buffer's readers finished in the previous iteration
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int i = m0 + tx + 16 * a;
    if (i >= jb.m) continue;
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const int j = n0 + ty + 16 * b;
      if (j >= jb.n) continue;
      double2* cp = jb.c + i + (int64_t)j * jb.ldc;
      if (EPI == GEPI_PLAIN) {
        if (jb.herm && i < j) continue;  // written (bit-exactly) as the mirror of (j, i)
        double2 o = make_double2(jb.alpha * acc_r[a][b], jb.alpha * acc_i[a][b]);
        if (jb.beta0 != 0.0) {
          const double2 c0 = *cp;
          o.x += jb.beta0 * c0.x;
          o.y += jb.beta0 * c0.y;
        }
        if (i == j) {
          o.x += jb.diag_add;
          if (jb.herm) o.y = 0.0;
        }
        *cp = o;
        if (jb.herm && i != j) jb.c[j + (int64_t)i * jb.ldc] = make_double2(o.x, -o.y);
      } else {
        const bool iK = i >= jb.k0 && i < jb.k0 + jb.kb;
        if (iK) {
          *cp = reinterpret_cast<const double2*>(jb.b.p)[(i - jb.k0) + (int64_t)j * jb.b.ld];
        } else {
          const bool jK = j >= jb.k0 && j < jb.k0 + jb.kb;
          const double2 c0 = jK ? make_double2(0.0, 0.0) : *cp;
          *cp = make_double2(c0.x - acc_r[a][b], c0.y - acc_i[a][b]);
        }
      }
    }
  }
}

// fp64 tensor-core (DMMA) variant of the large products.  mma.sync m8n8k4
// f64 fragments (PTX ISA):  A 8x4 row: a = A[lane/4][lane%4];  B 4x8 col:
// b = B[lane%4][lane/4];  C 8x8: c[v] = C[lane/4][2 (lane%4) + v].
// A complex 8x8x4 block is four real MMAs (Cr += Ar Br - Ai Bi,
// Ci += Ar Bi + Ai Br).  CTA tile 128 x 64, BK = 8, 8 warps as 4 (m) x 2 (n),
// each warp a 32 x 32 block = 4 x 4 DMMA tiles.  Shared planes (real / imag,
// k-major) have pitches = 4 (mod 16) doubles: the fragment loads of a half
// warp hit 16 distinct banks.  Same register-prefetch pipeline and epilogues
// as gemm_big_kernel; products are exact fp64 (not bitwise equal to the SIMT
// kernels: the tensor core's accumulation order differs).
constexpr int kDmBM = 128, kDmBN = 64, kDmPA = 132, kDmPB = 68;
constexpr size_t kGemmDmmaSmem = (size_t)2 * 2 * kGK * (kDmPA + kDmPB) * sizeof(double);

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int EPI>
__global__ void __launch_bounds__(256, 1) gemm_dmma_kernel(const __grid_constant__ Pack<GemmJob> jobs) {
  constexpr int BM = kDmBM, BN = kDmBN, PA = kDmPA, PB = kDmPB;
  constexpr int LA = BM * kGK / 256, LB = BN * kGK / 256;
  const GemmJob& jb = jobs.j[blockIdx.z];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= jb.m || n0 >= jb.n) return;
  if (EPI == GEPI_PLAIN && jb.herm && m0 + BM <= n0) return;
  extern __shared__ double dsm[];
  // [buf][plane][kk][pitch]
  double* Ash = dsm;                            // 2 x 2 x kGK x PA
  double* Bsh = dsm + 2 * 2 * kGK * PA;         // 2 x 2 x kGK x PB
  auto As = [&](int buf, int pl, int kk) { return Ash + ((buf * 2 + pl) * kGK + kk) * PA; };
  auto Bs = [&](int buf, int pl, int kk) { return Bsh + ((buf * 2 + pl) * kGK + kk) * PB; };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;  // warp block origin in the tile
  const int fr = lane >> 2, fc = lane & 3;                // fragment row / k
  // 3M complex products: Re = P1 - P2, Im = P3 - P1 - P2 (see frame_batch2_kernel)
  double p1[4][4][2], p2[4][4][2], p3[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) p1[a][b][v] = p2[a][b][v] = p3[a][b][v] = 0.0;
  const MatRef A = jb.a, B = jb.b;
  double2 pa[LA], pb[LB];
  auto a_pos = [&](int e, int& ii, int& kk) {
    if (!A.trans) { ii = e % BM; kk = e / BM; } else { kk = e & 7; ii = e >> 3; }
  };
  auto b_pos = [&](int e, int& jj, int& kk) {
    if (!B.trans) { kk = e & 7; jj = e >> 3; } else { jj = e % BN; kk = e / BN; }
  };
  auto fetch = [&](int kk0) {
#pragma unroll
    for (int t = 0; t < LA; ++t) {
      int ii, kk;
      a_pos(tid + t * 256, ii, kk);
      const int gi = m0 + ii, gk = kk0 + kk;
      pa[t] = (gi < jb.m && gk < jb.k) ? mat_load(A, gi, gk) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int t = 0; t < LB; ++t) {
      int jj, kk;
      b_pos(tid + t * 256, jj, kk);
      const int gj = n0 + jj, gk = kk0 + kk;
      pb[t] = (gj < jb.n && gk < jb.k) ? mat_load(B, gk, gj) : make_double2(0.0, 0.0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int t = 0; t < LA; ++t) {
      int ii, kk;
      a_pos(tid + t * 256, ii, kk);
      As(buf, 0, kk)[ii] = pa[t].x;
      As(buf, 1, kk)[ii] = pa[t].y;
    }
#pragma unroll
    for (int t = 0; t < LB; ++t) {
      int jj, kk;
      b_pos(tid + t * 256, jj, kk);
      Bs(buf, 0, kk)[jj] = pb[t].x;
      Bs(buf, 1, kk)[jj] = pb[t].y;
    }
  };
  const int nk = (jb.k + kGK - 1) / kGK;
  if (nk > 0) {
    fetch(0);
    stash(0);
  }
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    if (t + 1 < nk) fetch((t + 1) * kGK);
#pragma unroll
    for (int k4 = 0; k4 < kGK; k4 += 4) {
      double ar[4], ai[4], as[4], br[4], bi[4], bs[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ar[a] = As(cur, 0, k4 + fc)[wm + 8 * a + fr];
        ai[a] = As(cur, 1, k4 + fc)[wm + 8 * a + fr];
        as[a] = ar[a] + ai[a];
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        br[b] = Bs(cur, 0, k4 + fc)[wn + 8 * b + fr];
        bi[b] = Bs(cur, 1, k4 + fc)[wn + 8 * b + fr];
        bs[b] = br[b] + bi[b];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dmma884(p1[a][b], ar[a], br[b]);
          dmma884(p2[a][b], ai[a], bi[b]);
          dmma884(p3[a][b], as[a], bs[b]);
        }
    }
    if (t + 1 < nk) stash(cur ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = m0 + wm + 8 * a + fr, j = n0 + wn + 8 * b + 2 * fc + v;
        if (i >= jb.m || j >= jb.n) continue;
        double2* cp = jb.c + i + (int64_t)j * jb.ldc;
        const double accr = p1[a][b][v] - p2[a][b][v], acci = p3[a][b][v] - p1[a][b][v] - p2[a][b][v];
        if (EPI == GEPI_PLAIN) {
          if (jb.herm && i < j) continue;
          double2 o = make_double2(jb.alpha * accr, jb.alpha * acci);
          if (jb.beta0 != 0.0) {
            const double2 c0 = *cp;
            o.x += jb.beta0 * c0.x;
            o.y += jb.beta0 * c0.y;
          }
          if (i == j) {
            o.x += jb.diag_add;
            if (jb.herm) o.y = 0.0;
          }
          *cp = o;
          if (jb.herm && i != j) jb.c[j + (int64_t)i * jb.ldc] = make_double2(o.x, -o.y);
        } else {
          const bool iK = i >= jb.k0 && i < jb.k0 + jb.kb;
          if (iK) {
            *cp = reinterpret_cast<const double2*>(jb.b.p)[(i - jb.k0) + (int64_t)j * jb.b.ld];
          } else {
            const bool jK = j >= jb.k0 && j < jb.k0 + jb.kb;
            const double2 c0 = jK ? make_double2(0.0, 0.0) : *cp;
            *cp = make_double2(c0.x - accr, c0.y - acci);
          }
        }
      }
}

// C = alpha * sum_s ws[job*nsplit + s] + beta0 * C (+ diag), fixed split order.
__global__ void gemm_split_reduce(const __grid_constant__ Pack<GemmJob> jobs, int nsplit,
                                  const double2* __restrict__ ws, int64_t ws_stride) {
  const GemmJob& jb = jobs.j[blockIdx.y];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)jb.m * jb.n) return;
  const int i = (int)(e % jb.m), j = (int)(e / jb.m);
  double sr = 0.0, si = 0.0;
  for (int s = 0; s < nsplit; ++s) {
    const double2 v = ws[(int64_t)(blockIdx.y * nsplit + s) * ws_stride + (int64_t)j * jb.m + i];
    sr += v.x;
    si += v.y;
  }
  double2* cp = jb.c + i + (int64_t)j * jb.ldc;
  double2 o = make_double2(jb.alpha * sr, jb.alpha * si);
  if (jb.beta0 != 0.0) {
    const double2 c0 = *cp;
    o.x += jb.beta0 * c0.x;
    o.y += jb.beta0 * c0.y;
  }
  if (i == j) o.x += jb.diag_add;
  *cp = o;
}

// In-place Gauss-Jordan inverse of one kb x kb HPD pivot block (kb <= 64)
// in shared memory: writes P = inv(M_KK) to P (ld = ldp) and raises *fail
// if a pivot is not a positive finite real (the Cholesky-failure analogue of
// solver_core.hpp:42-43).
struct DiagJob {
  const double2* M;
  int64_t ld;
  int n;          // matrix order
  int k0, kb;     // pivot block
  double2* P;     // kb x kb, ld = ldp
  int64_t ldp;
  double2* F;     // copy of M[:, K] (n x kb), ld = ldf
  int64_t ldf;
  double2* R;     // row panel R' (kb x n), ld = ldr
  int64_t ldr;
  int* fail;
};

__global__ void __launch_bounds__(1024) gj_diag_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  const DiagJob& jb = jobs.j[blockIdx.x];
  if (jb.k0 >= jb.n) return;
  extern __shared__ double2 gj_smem[];
  double2 (*S)[65] = reinterpret_cast<double2 (*)[65]>(gj_smem);
  double2* prow = gj_smem + 64 * 65;
  double2* pcol = prow + 64;
  const int kb = jb.kb;
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    S[r][c] = jb.M[(jb.k0 + r) + (int64_t)(jb.k0 + c) * jb.ld];
  }
  __syncthreads();
  for (int p = 0; p < kb; ++p) {
    const double2 piv = S[p][p];
    if (threadIdx.x == 0 && !(piv.x > 0.0 && isfinite(piv.x) && isfinite(piv.y))) atomicExch(jb.fail, 1);
    const double den = piv.x * piv.x + piv.y * piv.y;
    const double2 ip = make_double2(piv.x / den, -piv.y / den);
    if (threadIdx.x < kb) {
      const int c = threadIdx.x;
      const double2 v = S[p][c];
      prow[c] = (c == p) ? ip : make_double2(v.x * ip.x - v.y * ip.y, v.x * ip.y + v.y * ip.x);
      pcol[c] = S[c][p];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
      const int r = e % kb, c = e / kb;
      if (r == p) {
        S[r][c] = prow[c];
      } else {
        const double2 f = pcol[r];
        const double2 pr = prow[c];
        const double2 base = (c == p) ? make_double2(0.0, 0.0) : S[r][c];
        S[r][c] = make_double2(base.x - (f.x * pr.x - f.y * pr.y), base.y - (f.x * pr.y + f.y * pr.x));
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    jb.P[r + (int64_t)c * jb.ldp] = S[r][c];
  }
}

// F = M[:, K] (pivot column panel), grid-stride over n*kb per job.
__global__ void gj_panel_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  const DiagJob& jb = jobs.j[blockIdx.y];
  if (jb.k0 >= jb.n) return;
  const int64_t total = (int64_t)jb.n * jb.kb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % jb.n), c = (int)(e / jb.n);
    jb.F[r + (int64_t)c * jb.ldf] = jb.M[r + (int64_t)(jb.k0 + c) * jb.ld];
  }
}

// R'[:, K] = P (overwrite the pivot columns of the row panel).
__global__ void gj_fix_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  const DiagJob& jb = jobs.j[blockIdx.x];
  if (jb.k0 >= jb.n) return;
  for (int e = threadIdx.x; e < jb.kb * jb.kb; e += blockDim.x) {
    const int r = e % jb.kb, c = e / jb.kb;
    jb.R[r + (int64_t)(jb.k0 + c) * jb.ldr] = jb.P[r + (int64_t)c * jb.ldp];
  }
}

// out[i + j*ldo] = M[ridx[i] + cidx[j]*ld] (submatrix gather, grid-stride)
struct SubJob {
  const double2* M;
  int64_t ld;
  const int* ridx;
  const int* cidx;
  int m, n;
  double2* out;
  int64_t ldo;
};

__global__ void gather_sub_kernel(const __grid_constant__ Pack<SubJob> jobs) {
  const SubJob& jb = jobs.j[blockIdx.y];
  const int64_t total = (int64_t)jb.m * jb.n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % jb.m), j = (int)(e / jb.m);
    jb.out[i + (int64_t)j * jb.ldo] = jb.M[jb.ridx[i] + (int64_t)jb.cidx[j] * jb.ld];
  }
}

// Utility kernels -----------------------------------------------------------
__global__ void c128_to_c64_kernel(const double2* __restrict__ src, int64_t lds, float2* __restrict__ dst,
                                   int64_t ldd, int rows, int cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * cols) return;
  const int r = (int)(e % rows);
  const int64_t c = e / rows;
  const double2 v = src[r + c * lds];
  dst[r + c * ldd] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
}

__global__ void soft_threshold_kernel(const double2* __restrict__ v, int64_t n, double kappa, double2* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = soft_threshold1(v[i], kappa);
}

__global__ void abs_kernel(const double2* __restrict__ v, int n, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = c_abs(v[i]);
}

// out = beta * (a - b): the accumulated frozen echo z = y_eff_s - y_eff,
// scaled, that is folded into v when the stored data term lags (see
// local_updates in radmm_b200.cu).
__global__ void scaled_diff_kernel(double2* __restrict__ out, const double2* __restrict__ a,
                                   const double2* __restrict__ b, double beta, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double2(beta * (a[i].x - b[i].x), beta * (a[i].y - b[i].y));
}

// Rb[:, t] = A[:, rem_pix[t]] promoted to complex128 (zero-padded to ld).
__global__ void gather_cols_c128_kernel(const float2* __restrict__ A, int64_t ld, const int* __restrict__ pix,
                                        int r, double2* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ld * r) return;
  const int t = (int)(e / ld);
  const int64_t row = e % ld;
  const float2 v = A[row + (int64_t)pix[t] * ld];
  out[e] = make_double2((double)v.x, (double)v.y);
}

__global__ void iota_kernel(int* __restrict__ J, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) J[i] = i;
}

// Gather x_full[J] -> x_hat (and zero a vector) etc.
__global__ void gather_kernel(const double2* __restrict__ src, const int* __restrict__ idx, int n, double2* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// BASELINE dechirped-LFM operator generator (mirrors scenario.baseline_operator
// operation by operation, no FMA contraction).
__global__ void dechirp_kernel(float2* __restrict__ A, int64_t ld, int M, int K, int N,
                               const double* __restrict__ pix, const double* __restrict__ tx,
                               const double* __restrict__ rx, const double* __restrict__ phi,
                               double alpha, double fc, double t_step, double c_light, double two_pi) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = M * K;
  if (e >= (int64_t)rows * N) return;
  const int r = (int)(e % rows);
  const int n = (int)(e / rows);
  const int m = r / K, k = r % K;
  const double px = pix[3 * n], py = pix[3 * n + 1], pz = pix[3 * n + 2];
  double dx = __dsub_rn(tx[0], px), dy = __dsub_rn(tx[1], py), dz = __dsub_rn(tx[2], pz);
  const double dtx = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  dx = __dsub_rn(rx[3 * m], px); dy = __dsub_rn(rx[3 * m + 1], py); dz = __dsub_rn(rx[3 * m + 2], pz);
  const double drx = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  const double tau = __ddiv_rn(__dadd_rn(dtx, drx), c_light);
  const double tk = __dmul_rn((double)k, t_step);
  double cyc = __dadd_rn(__dmul_rn(__dmul_rn(alpha, tau), tk), __dmul_rn(fc, tau));
  cyc = __dsub_rn(cyc, floor(cyc));
  const double ang = __dadd_rn(__dmul_rn(two_pi, cyc), phi[n]);
  double s, c;
  sincos(ang, &s, &c);
  A[r + (int64_t)n * ld] = make_float2(__double2float_rn(c), __double2float_rn(s));
}

}  // namespace radmm_dev

namespace radmm_dev {

// ---------------------------------------------------------------------------
// Single-pass fused sweep (one GPU, all sensors in the dual form, Q <= 8).
//
// The two matvecs of consecutive iterations read the same operator columns:
// the adjoint of iteration k (x-update) and the forward of iteration k+1
// (v = A_J rhs).  Between them sits the fusion round, which couples all
// sensors at each pixel.  A thread-block cluster holds one CTA per sensor over
// a shared pixel range; per pixel tile:
//   (a) CTA q: u_i = A_q(:,J_i)^H w_q for its active columns of the tile and
//       the x-update epilogue (x_hat, x_full scatter, screening ring)   [HBM]
//   (b) cluster barrier (release/acquire); CTA q runs FusionCore::round on a
//       1/Q slice of the tile's pixels, reading every sensor's x_full (L2)
//   (c) cluster barrier; CTA q forms rhs_{k+1} for its tile columns
//   (d) CTA q accumulates v_{k+1} += A_q(:,J_i) rhs_i in registers     [L2]
// A is streamed from HBM once per iteration; the second touch hits L2.  Each
// CTA finally writes its KM-length partial of v_{k+1} (fixed-order reduce),
// and the grid's last block finishes the fusion norms / stopping rule.
// ---------------------------------------------------------------------------
struct SweepJob {
  const float2* A;
  int64_t ld;
  int n_act;
  const int* J;
  const double2* w;
  const double2* data;
  double2* rhs;
  double2* x_hat;
  double2* x_full;
  double* ring_slot;
  double2* part;  // [n_clusters][ld]
};

constexpr int kSweepThreads = 256;
constexpr int kSweepTile = 64;

__device__ __forceinline__ void cluster_sync_acqrel() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int lower_bound_dev(const int* J, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (J[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// u = A(:,col)^H w for two columns, 8 float4 loads in flight per lane.
__device__ __forceinline__ void sweep_dot2(const float2* __restrict__ A, int64_t ld, int c0, int c1, int steps,
                                           const double2* __restrict__ sv, int64_t half, int lane,
                                           double (&re)[2], double (&im)[2]) {
  const float4* p0 = reinterpret_cast<const float4*>(A + (int64_t)c0 * ld) + lane;
  const float4* p1 = reinterpret_cast<const float4*>(A + (int64_t)c1 * ld) + lane;
  const double2* ve = sv + lane;
  const double2* vo = sv + half + lane;
  re[0] = re[1] = im[0] = im[1] = 0.0;
  int s = 0;
#pragma unroll 1
  for (; s + 4 <= steps; s += 4) {
    float4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldg(p0 + (s + u) * 32);
#pragma unroll
    for (int u = 0; u < 4; ++u) b[u] = __ldg(p1 + (s + u) * 32);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 e = ve[(s + u) * 32], o = vo[(s + u) * 32];
      cfma_conj(re[0], im[0], a[u].x, a[u].y, e);
      cfma_conj(re[0], im[0], a[u].z, a[u].w, o);
      cfma_conj(re[1], im[1], b[u].x, b[u].y, e);
      cfma_conj(re[1], im[1], b[u].z, b[u].w, o);
    }
  }
  for (; s < steps; ++s) {
    const float4 a = __ldg(p0 + s * 32), b = __ldg(p1 + s * 32);
    const double2 e = ve[s * 32], o = vo[s * 32];
    cfma_conj(re[0], im[0], a.x, a.y, e);
    cfma_conj(re[0], im[0], a.z, a.w, o);
    cfma_conj(re[1], im[1], b.x, b.y, e);
    cfma_conj(re[1], im[1], b.z, b.w, o);
  }
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int RPT>  // float4 row-chunks per thread in the axpy: ld <= RPT * 512
__global__ void __launch_bounds__(kSweepThreads) fused_sweep_kernel(const __grid_constant__ Pack<SweepJob> jobs,
                                                                    const __grid_constant__ FusionArgs fa, double mu,
                                                                    double beta, int n_clusters, int range, int tile,
                                                                    int prefetch) {
  extern __shared__ double2 sweep_smem[];
  __shared__ int s_lo, s_hi, s_hi2;
  const int q = (int)cluster_ctarank();
  const int cl = blockIdx.x / fa.Q;
  const SweepJob& jb = jobs.j[q];
  const int64_t ld = jb.ld;
  const int64_t half = ld >> 1;
  double2* sv = sweep_smem;
  double2* coef = sweep_smem + ld;
  int* cidx = reinterpret_cast<int*>(coef + kSweepTile);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int r = tid; r < ld; r += kSweepThreads) sv[(r & 1) ? half + (r >> 1) : (r >> 1)] = jb.w[r];
  const int p0 = cl * range, p1 = min(fa.N, p0 + range);
  if (tid == 0) s_hi = lower_bound_dev(jb.J, jb.n_act, p0);
  __syncthreads();
  const int steps = (int)(ld >> 6);
  const int slice = (tile + fa.Q - 1) / fa.Q;
  double acc[RPT][4];
#pragma unroll
  for (int u = 0; u < RPT; ++u) acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0.0;
  double qn[5] = {0, 0, 0, 0, 0};
  for (int t0 = p0; t0 < p1; t0 += tile) {
    const int t1 = min(p1, t0 + tile);
    if (tid == 0) {
      int lo = s_hi, hi = lo;
      while (hi < jb.n_act && jb.J[hi] < t1) ++hi;
      int hi2 = hi;
      const int t2 = min(p1, t1 + tile);
      while (hi2 < jb.n_act && jb.J[hi2] < t2) ++hi2;
      s_lo = lo;
      s_hi = hi;
      s_hi2 = hi2;
    }
    __syncthreads();
    const int lo = s_lo, hi = s_hi;
    // stage the next tile's columns into L2 with TMA bulk prefetches so the
    // HBM stream keeps running through the cluster barriers below
    if (prefetch && tid < s_hi2 - hi)
      prefetch_l2_bulk(jb.A + (int64_t)jb.J[hi + tid] * ld, (unsigned)(ld * sizeof(float2)));
    // (a) adjoint dots + x-update for this sensor's active columns in the tile
    for (int i0 = lo + 2 * warp; i0 < hi; i0 += 2 * (kSweepThreads / 32)) {
      const int i1 = min(i0 + 1, hi - 1);
      double re[2], im[2];
      sweep_dot2(jb.A, ld, jb.J[i0], jb.J[i1], steps, sv, half, lane, re, im);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        re[c] = warp_sum(re[c]);
        im[c] = warp_sum(im[c]);
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int i = i0 + c;
        if (lane == c && i < hi) {
          const double2 r = jb.rhs[i];
          const double2 xh = make_double2(__ddiv_rn(__dsub_rn(r.x, __dmul_rn(mu, re[c])), beta),
                                          __ddiv_rn(__dsub_rn(r.y, __dmul_rn(mu, im[c])), beta));
          const int p = jb.J[i];
          const double2 old = jb.x_full[p];
          jb.ring_slot[p] = c_abs(c_sub(xh, old));
          jb.x_full[p] = xh;
          jb.x_hat[i] = xh;
        }
      }
    }
    cluster_sync_acqrel();
    // (b) fusion for this CTA's slice of the tile's pixels
    {
      const int j = t0 + q * slice + tid;
      if (tid < slice && j < t1 && j < t0 + (q + 1) * slice)
        fusion_pixel(fa, j, [&](int k) { return __ldcg(jobs.j[k].x_full + j); }, qn);
    }
    cluster_sync_acqrel();
    // (c) rhs_{k+1} = data + beta gap + beta x_hat - sigma (admm.hpp:114-119)
    for (int i = lo + tid; i < hi; i += kSweepThreads) {
      const int c = jb.J[i];
      const double2 d = jb.data[i], g = __ldcg(fa.gap + c), xh = jb.x_hat[i], sg = __ldcg(fa.sigma + c);
      double2 v;
      v.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
      v.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
      jb.rhs[i] = v;
      coef[i - lo] = v;
      cidx[i - lo] = c;
    }
    __syncthreads();
    // (d) v_{k+1} += A(:, J_i) rhs_i  -- the tile's columns are L2-hot
    const int cnt = hi - lo;
    int c = 0;
#pragma unroll 1
    for (; c + 2 <= cnt; c += 2) {
      float4 x0[RPT], x1[RPT];
      const float2* col0 = jb.A + (int64_t)cidx[c] * ld;
      const float2* col1 = jb.A + (int64_t)cidx[c + 1] * ld;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r = 2 * tid + 512 * u;
        x0[u] = r < ld ? __ldg(reinterpret_cast<const float4*>(col0 + r)) : make_float4(0, 0, 0, 0);
        x1[u] = r < ld ? __ldg(reinterpret_cast<const float4*>(col1 + r)) : make_float4(0, 0, 0, 0);
      }
      const double2 k0 = coef[c], k1 = coef[c + 1];
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        cfma(acc[u][0], acc[u][1], x0[u].x, x0[u].y, k0);
        cfma(acc[u][2], acc[u][3], x0[u].z, x0[u].w, k0);
        cfma(acc[u][0], acc[u][1], x1[u].x, x1[u].y, k1);
        cfma(acc[u][2], acc[u][3], x1[u].z, x1[u].w, k1);
      }
    }
    for (; c < cnt; ++c) {
      const float2* col0 = jb.A + (int64_t)cidx[c] * ld;
      const double2 k0 = coef[c];
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int64_t r = 2 * tid + 512 * u;
        if (r < ld) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(col0 + r));
          cfma(acc[u][0], acc[u][1], x.x, x.y, k0);
          cfma(acc[u][2], acc[u][3], x.z, x.w, k0);
        }
      }
    }
    __syncthreads();
  }
  // partial v_{k+1} of this CTA (rows owned by this thread)
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int64_t r = 2 * tid + 512 * u;
    if (r < ld) {
      double2* out = jb.part + (int64_t)cl * ld + r;
      out[0] = make_double2(acc[u][0], acc[u][1]);
      out[1] = make_double2(acc[u][2], acc[u][3]);
    }
  }
  fusion_finish(fa, qn);
}

}  // namespace radmm_dev

namespace radmm_dev {

// ---------------------------------------------------------------------------
// Fused sweep v2: asynchronous, warp-specialised, one cluster = Q CTAs (one
// per sensor) over a shared pixel range, one CTA per SM.  Roles per CTA:
//   dot warps    stream the active columns of each pixel tile from HBM and
//                run the adjoint x-update (u = A^H w, x = (rhs - mu u)/beta)
//   fusion warp  when all Q CTAs finished tile T (DSMEM mbarrier), runs
//                FusionCore::round on its slice of T and tells the peers
//   axpy warps   when the whole cluster fused tile T, form rhs_{k+1} and
//                accumulate v_{k+1} += A(:,J_i) rhs_i, re-reading the tile's
//                columns while they are still L2-resident; then free the
//                tile slot for the dot warps (bounded lag = L2 footprint)
// Tiles flow through a DEPTH-deep ring of mbarriers; no role waits for a
// cluster-wide barrier, so the HBM stream of the dot warps never drains.
// ---------------------------------------------------------------------------
constexpr int kS2Dot = 8;        // dot warps
constexpr int kS2Fuse = 4;       // fusion warps (tile T handled by warp T % kS2Fuse)
constexpr int kS2Axpy = 4;       // axpy warps
constexpr int kS2Threads = (kS2Dot + kS2Fuse + kS2Axpy) * 32;
constexpr int kS2Depth = 8;      // tiles in flight per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* b, unsigned cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(b)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

template <int RPT>  // float4 row chunks per axpy thread: ld <= RPT * 256
__global__ void __launch_bounds__(kS2Threads, 1) fused_sweep2_kernel(const __grid_constant__ Pack<SweepJob> jobs,
                                                                     const __grid_constant__ FusionArgs fa, double mu,
                                                                     double beta, int range, int tile) {
  extern __shared__ double2 s2_smem[];
  __shared__ uint64_t bar_dots[kS2Depth], bar_xhat[kS2Depth], bar_fused[kS2Depth], bar_free[kS2Depth];
  __shared__ double2 s_coef[64];
  __shared__ int s_col[64];
  const int Q = fa.Q;
  const int q = (int)cluster_ctarank();
  const int cl = blockIdx.x / Q;
  const SweepJob& jb = jobs.j[q];
  const int64_t ld = jb.ld;
  const int64_t half = ld >> 1;
  double2* sv = s2_smem;                                   // w_q, split by row parity
  int* tlo = reinterpret_cast<int*>(s2_smem + ld);         // tile -> first active index
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p0 = cl * range, p1 = min(fa.N, p0 + range);
  const int ntiles = p1 > p0 ? (p1 - p0 + tile - 1) / tile : 0;
  for (int r = tid; r < ld; r += kS2Threads) sv[(r & 1) ? half + (r >> 1) : (r >> 1)] = jb.w[r];
  for (int t = tid; t <= ntiles; t += kS2Threads) tlo[t] = lower_bound_dev(jb.J, jb.n_act, min(p1, p0 + t * tile));
  if (tid == 0) {
    for (int b = 0; b < kS2Depth; ++b) {
      mbar_init(&bar_dots[b], kS2Dot);
      mbar_init(&bar_xhat[b], Q);
      mbar_init(&bar_fused[b], Q);
      mbar_init(&bar_free[b], kS2Axpy);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster_sync_acqrel();  // peers' barriers are initialised before anyone arrives remotely
  double qn[5] = {0, 0, 0, 0, 0};
  if (warp < kS2Dot) {
    // ---------------- dot warps ----------------
    const int steps = (int)(ld >> 6);
    for (int T = 0; T < ntiles; ++T) {
      const int b = T % kS2Depth;
      if (T >= kS2Depth) mbar_wait_cluster(&bar_free[b], ((T / kS2Depth) - 1) & 1);
      const int lo = tlo[T], hi = tlo[T + 1];
      for (int i0 = lo + 2 * warp; i0 < hi; i0 += 2 * kS2Dot) {
        const int i1 = min(i0 + 1, hi - 1);
        double re[2], im[2];
        sweep_dot2(jb.A, ld, jb.J[i0], jb.J[i1], steps, sv, half, lane, re, im);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          re[c] = warp_sum(re[c]);
          im[c] = warp_sum(im[c]);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int i = i0 + c;
          if (lane == c && i < hi) {
            const double2 r = jb.rhs[i];
            const double2 xh = make_double2(__ddiv_rn(__dsub_rn(r.x, __dmul_rn(mu, re[c])), beta),
                                            __ddiv_rn(__dsub_rn(r.y, __dmul_rn(mu, im[c])), beta));
            const int p = jb.J[i];
            const double2 old = jb.x_full[p];
            jb.ring_slot[p] = c_abs(c_sub(xh, old));
            jb.x_full[p] = xh;
            jb.x_hat[i] = xh;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&bar_dots[b]);
    }
  } else if (warp < kS2Dot + kS2Fuse) {
    // ---------------- fusion warps ----------------
    const int slice = (tile + Q - 1) / Q;
    for (int T = warp - kS2Dot; T < ntiles; T += kS2Fuse) {
      const int b = T % kS2Depth;
      const unsigned par = (T / kS2Depth) & 1;
      mbar_wait_cluster(&bar_dots[b], par);  // this CTA's x-updates of tile T are written
      if (lane == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        for (int k = 0; k < Q; ++k) mbar_arrive_remote(&bar_xhat[b], (unsigned)k);
      }
      mbar_wait_cluster(&bar_xhat[b], par);  // every sensor's x-updates of tile T are written
      const int t0 = p0 + T * tile, t1 = min(p1, t0 + tile);
      for (int j = t0 + q * slice + lane; j < min(t1, t0 + (q + 1) * slice); j += 32)
        fusion_pixel(fa, j, [&](int k) { return __ldcg(jobs.j[k].x_full + j); }, qn);
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        for (int k = 0; k < Q; ++k) mbar_arrive_remote(&bar_fused[b], (unsigned)k);
      }
    }
  } else {
    // ---------------- axpy warps ----------------
    const int at = tid - (kS2Dot + kS2Fuse) * 32;  // 0 .. 32*kS2Axpy-1
    double acc[RPT][4];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0.0;
    for (int T = 0; T < ntiles; ++T) {
      const int b = T % kS2Depth;
      mbar_wait_cluster(&bar_fused[b], (T / kS2Depth) & 1);
      const int lo = tlo[T], hi = tlo[T + 1];
      // rhs_{k+1} = data + beta gap + beta x_hat - sigma (admm.hpp:114-119), one column per thread
      for (int i = lo + at; i < hi; i += 32 * kS2Axpy) {
        const int c = jb.J[i];
        const double2 d = jb.data[i], g = __ldcg(fa.gap + c), xh = __ldcg(jb.x_hat + i), sg = __ldcg(fa.sigma + c);
        double2 v;
        v.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
        v.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
        jb.rhs[i] = v;
        s_coef[i - lo] = v;
        s_col[i - lo] = c;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kS2Axpy) : "memory");
      const int cnt = hi - lo;
      int t = 0;
      for (; t + 2 <= cnt; t += 2) {
        const float2* c0 = jb.A + (int64_t)s_col[t] * ld;
        const float2* c1 = jb.A + (int64_t)s_col[t + 1] * ld;
        float4 x0[RPT], x1[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t r = 2 * (at + 32 * kS2Axpy * u);
          x0[u] = r < ld ? __ldg(reinterpret_cast<const float4*>(c0 + r)) : make_float4(0, 0, 0, 0);
          x1[u] = r < ld ? __ldg(reinterpret_cast<const float4*>(c1 + r)) : make_float4(0, 0, 0, 0);
        }
        const double2 v0 = s_coef[t], v1 = s_coef[t + 1];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          cfma(acc[u][0], acc[u][1], x0[u].x, x0[u].y, v0);
          cfma(acc[u][2], acc[u][3], x0[u].z, x0[u].w, v0);
          cfma(acc[u][0], acc[u][1], x1[u].x, x1[u].y, v1);
          cfma(acc[u][2], acc[u][3], x1[u].z, x1[u].w, v1);
        }
      }
      if (t < cnt) {
        const float2* c0 = jb.A + (int64_t)s_col[t] * ld;
        const double2 v0 = s_coef[t];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int64_t r = 2 * (at + 32 * kS2Axpy * u);
          if (r < ld) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(c0 + r));
            cfma(acc[u][0], acc[u][1], x.x, x.y, v0);
            cfma(acc[u][2], acc[u][3], x.z, x.w, v0);
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kS2Axpy) : "memory");  // s_coef reused next tile
      if (lane == 0) mbar_arrive_local(&bar_free[b]);
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int64_t r = 2 * (at + 32 * kS2Axpy * u);
      if (r < ld) {
        double2* out = jb.part + (int64_t)cl * ld + r;
        out[0] = make_double2(acc[u][0], acc[u][1]);
        out[1] = make_double2(acc[u][2], acc[u][3]);
      }
    }
  }
  __syncthreads();
  cluster_sync_acqrel();  // no CTA leaves while a peer may still arrive on its barriers
  fusion_finish(fa, qn);
}

}  // namespace radmm_dev

namespace radmm_dev {

// ---------------------------------------------------------------------------
// Fused sweep v3: row-split cluster, TMA-fed shared-memory column ring.
//
// A cluster of kS3R CTAs owns a pixel range; CTA `rank` owns rows
// [rank*sl, (rank+1)*sl) of EVERY sensor's operator (sl = ld / kS3R).  Per
// pixel tile (kS3P pixels) one elected thread bulk-copies (TMA,
// cp.async.bulk) the row slices of the tile's active columns of all sensors
// into one of two shared-memory buffers.  Then:
//   dots     warp q computes the partial dots slice(A_q(:,j))^H w_q[slice]
//            for sensor q's columns of the tile (w slices live in smem)
//   exchange cluster barrier; every CTA sums the kS3R partial dots of each
//            column from its peers' shared memory (DSMEM, fixed rank order)
//            -> identical full dots in every CTA
//   x-update x = (rhs - mu u)/beta for the tile's columns (rank 0 writes)
//   fusion   FusionCore::round for the tile's pixels, computed redundantly
//            (identically) by every CTA from the local x values
//   forward  v_{k+1}[slice] += A(slice, j) rhs_{k+1,j}, from the same smem
// Each operator byte crosses HBM once per iteration; the TMA of tile t+1
// overlaps the work on tile t.
// ---------------------------------------------------------------------------
constexpr int kS3R = 8;          // CTAs per cluster (row split)
constexpr int kS3P = 4;          // pixels per tile
constexpr int kS3Q = 8;          // max sensors (one warp each in the dot phase)
constexpr int kS3Threads = 256;  // one slice row per thread (sl <= 256)
constexpr int kS3Cols = kS3P * kS3Q;

struct Sweep3Job {
  const float2* A;
  const int* J;
  int n_act;
  const double2* w;
  const double2* data;
  double2* rhs;
  double2* x_hat;
  double2* x_full;
  double* ring_slot;
  double2* part;  // [n_clusters][ld]
};

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ double2 dsmem_load2(const double2* local, unsigned rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  double x, y;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(ra) : "memory");
  return make_double2(x, y);
}

struct __align__(16) S3Tile {  // one tile, staged by the producer warp (per buffer)
  double2 rhs[kS3Cols];   // rhs_k of each column (column order, contiguous per sensor)
  double2 data[kS3Cols];  // data term of each column
  double2 xg[kS3P];       // x_G before this round
  double2 sg[kS3P];       // sigma before this round
  double2 xf[kS3Q][kS3P]; // x_q before this round (frozen values, ring baseline)
  int n;                  // columns in the tile
  int q[kS3Cols];         // sensor of column c
  int i[kS3Cols];         // active index within J_q
  int pix[kS3Cols];       // pixel
  int qstart[kS3Q + 1];   // columns of sensor q: [qstart[q], qstart[q+1])
  int pq[kS3P][kS3Q];     // column of (pixel p, sensor q), -1 if frozen
};

__global__ void __launch_bounds__(kS3Threads, 1) fused_sweep3_kernel(const __grid_constant__ Pack<Sweep3Job> jobs,
                                                                     const __grid_constant__ FusionArgs fa, double mu,
                                                                     double beta, int64_t ld, int range) {
  extern __shared__ __align__(128) unsigned char s3_raw[];
  __shared__ __align__(8) uint64_t full_bar[2];
  __shared__ S3Tile tiles[2];
  __shared__ double2 pdot[2][kS3Cols];  // this CTA's partial dots (read by peers)
  __shared__ double2 xloc[kS3Cols];     // x-update of the tile's columns
  __shared__ double2 coef[kS3Cols];     // rhs_{k+1} of the tile's columns
  __shared__ double2 gap_s[kS3P], sig_s[kS3P];
  const int Q = fa.Q;
  const unsigned rank = cluster_ctarank();
  const int cl = blockIdx.x / kS3R;
  const int sl = (int)(ld / kS3R);  // slice rows (<= 256)
  const int64_t row0 = (int64_t)rank * sl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p0 = cl * range, p1 = min(fa.N, p0 + range);
  const int ntiles = p1 > p0 ? (p1 - p0 + kS3P - 1) / kS3P : 0;
  float2* buf0 = reinterpret_cast<float2*>(s3_raw);                                          // [2][kS3Cols][sl]
  double2* wsl = reinterpret_cast<double2*>(s3_raw + 2ull * kS3Cols * sl * sizeof(float2));  // [Q][sl]
  int* tab = reinterpret_cast<int*>(wsl + (size_t)Q * sl);                                   // [Q][ntiles+1]
  for (int e = tid; e < Q * sl; e += kS3Threads) {
    const int q = e / sl, r = e % sl;
    wsl[e] = jobs.j[q].w[row0 + r];
  }
  for (int e = tid; e < Q * (ntiles + 1); e += kS3Threads) {
    const int q = e / (ntiles + 1), t = e % (ntiles + 1);
    tab[e] = lower_bound_dev(jobs.j[q].J, jobs.j[q].n_act, min(p1, p0 + t * kS3P));
  }
  if (tid == 0) {
    mbar_init(&full_bar[0], 1);
    mbar_init(&full_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned slice_bytes = (unsigned)(sl * sizeof(float2));
  // producer warp: describe tile t and bulk-copy (TMA) its column slices and
  // every per-tile input into buffer b; completion on full_bar[b]
  auto issue = [&](int t, int b) {
    S3Tile& T = tiles[b];
    const int t0 = p0 + t * kS3P, np = min(p1, t0 + kS3P) - t0;
    if (lane == 0) {
      int n = 0;
      for (int q = 0; q < kS3Q; ++q) {
        T.qstart[q] = n;
        if (q < Q) n += tab[q * (ntiles + 1) + t + 1] - tab[q * (ntiles + 1) + t];
      }
      T.qstart[kS3Q] = n;
      T.n = n;
      unsigned bytes = (unsigned)n * (slice_bytes + 2u * sizeof(double2)) + 2u * np * sizeof(double2) +
                       (unsigned)Q * np * sizeof(double2);
      mbar_arrive_expect_tx(&full_bar[b], bytes);
    }
    reinterpret_cast<int*>(T.pq)[lane] = -1;  // kS3P * kS3Q == 32
    __syncwarp();
    const int n = T.n;
    float2* dst = buf0 + (size_t)b * kS3Cols * sl;
    if (lane < n) {
      int q = 0;
      while (T.qstart[q + 1] <= lane) ++q;
      const int i = tab[q * (ntiles + 1) + t] + (lane - T.qstart[q]);
      const int pix = jobs.j[q].J[i];
      T.q[lane] = q;
      T.i[lane] = i;
      T.pix[lane] = pix;
      T.pq[pix - t0][q] = lane;
      tma_bulk_g2s(dst + (size_t)lane * sl, jobs.j[q].A + (int64_t)pix * ld + row0, slice_bytes, &full_bar[b]);
    }
    if (lane < Q) {
      const int q = lane;
      const int c0 = T.qstart[q], cnt = T.qstart[q + 1] - c0;
      const int i0 = tab[q * (ntiles + 1) + t];
      if (cnt > 0) {
        tma_bulk_g2s(&T.rhs[c0], jobs.j[q].rhs + i0, (unsigned)cnt * sizeof(double2), &full_bar[b]);
        tma_bulk_g2s(&T.data[c0], jobs.j[q].data + i0, (unsigned)cnt * sizeof(double2), &full_bar[b]);
      }
      tma_bulk_g2s(&T.xf[q][0], jobs.j[q].x_full + t0, (unsigned)np * sizeof(double2), &full_bar[b]);
    } else if (lane == kS3Q) {
      tma_bulk_g2s(&T.xg[0], fa.xg + t0, (unsigned)np * sizeof(double2), &full_bar[b]);
    } else if (lane == kS3Q + 1) {
      tma_bulk_g2s(&T.sg[0], fa.sigma + t0, (unsigned)np * sizeof(double2), &full_bar[b]);
    }
  };
  if (warp == 0) {
    if (ntiles > 0) issue(0, 0);
    __syncwarp();
    if (ntiles > 1) issue(1, 1);
  }
  cluster_sync_acqrel();  // peers' pdot buffers exist
  double acc[kS3Q][2];
#pragma unroll
  for (int q = 0; q < kS3Q; ++q) acc[q][0] = acc[q][1] = 0.0;
  double qn[5] = {0, 0, 0, 0, 0};
  for (int t = 0; t < ntiles; ++t) {
    const int b = t & 1;
    mbar_wait_cluster(&full_bar[b], (t >> 1) & 1);
    const S3Tile& T = tiles[b];
    const float2* sb = buf0 + (size_t)b * kS3Cols * sl;
    const int t0 = p0 + t * kS3P, np = min(p1, t0 + kS3P) - t0;
    // ---- partial dots: warp q <-> sensor q, up to kS3P columns per warp ----
    if (warp < Q) {
      const int c0 = T.qstart[warp], c1 = T.qstart[warp + 1];
      if (c0 < c1) {
        double re[kS3P], im[kS3P];
#pragma unroll
        for (int u = 0; u < kS3P; ++u) re[u] = im[u] = 0.0;
        const double2* wq = wsl + (size_t)warp * sl;
        for (int r = lane; r < sl; r += 32) {
          const double2 wv = wq[r];
#pragma unroll
          for (int u = 0; u < kS3P; ++u)
            if (c0 + u < c1) {
              const float2 a = sb[(size_t)(c0 + u) * sl + r];
              cfma_conj(re[u], im[u], a.x, a.y, wv);
            }
        }
#pragma unroll
        for (int u = 0; u < kS3P; ++u) {
          re[u] = warp_sum(re[u]);
          im[u] = warp_sum(im[u]);
        }
#pragma unroll
        for (int u = 0; u < kS3P; ++u)
          if (lane == u && c0 + u < c1) pdot[b][c0 + u] = make_double2(re[u], im[u]);
      }
    }
    cluster_sync_acqrel();
    // ---- full dots (fixed rank order) and the x-update ----
    if (tid < T.n) {
      double2 v[kS3R];
#pragma unroll
      for (int r = 0; r < kS3R; ++r) v[r] = dsmem_load2(&pdot[b][tid], (unsigned)r);
      double ur = 0.0, ui = 0.0;
#pragma unroll
      for (int r = 0; r < kS3R; ++r) {
        ur += v[r].x;
        ui += v[r].y;
      }
      const double2 rr = T.rhs[tid];
      const double2 xh = make_double2(__ddiv_rn(__dsub_rn(rr.x, __dmul_rn(mu, ur)), beta),
                                      __ddiv_rn(__dsub_rn(rr.y, __dmul_rn(mu, ui)), beta));
      xloc[tid] = xh;
      if (rank == 0) {
        const int q = T.q[tid], p = T.pix[tid];
        const Sweep3Job& jb = jobs.j[q];
        jb.ring_slot[p] = c_abs(c_sub(xh, T.xf[q][p - t0]));
        jb.x_full[p] = xh;
        jb.x_hat[T.i[tid]] = xh;
      }
    }
    __syncthreads();
    // ---- fusion for the tile's pixels (identical in every CTA) ----
    if (tid < np) {
      const int j = t0 + tid;
      double2 s = make_double2(0.0, 0.0);
      for (int k = 0; k < Q; ++k) {
        const int c = T.pq[tid][k];
        s = c_add(s, c >= 0 ? xloc[c] : T.xf[k][tid]);
      }
      s = make_double2(__ddiv_rn(s.x, (double)Q), __ddiv_rn(s.y, (double)Q));
      const double2 xgp = T.xg[tid];
      const double2 sg = T.sg[tid];
      const double2 v = make_double2(__dadd_rn(s.x, __ddiv_rn(sg.x, beta)), __dadd_rn(s.y, __ddiv_rn(sg.y, beta)));
      const double2 xg = soft_threshold1(v, fa.kappa);
      const double2 eta = c_sub(s, xg);
      const double2 dx = c_sub(xg, xgp);
      const double2 sn = make_double2(__dadd_rn(sg.x, __dmul_rn(beta, eta.x)), __dadd_rn(sg.y, __dmul_rn(beta, eta.y)));
      const double2 gp = c_sub(xg, s);
      gap_s[tid] = gp;
      sig_s[tid] = sn;
      if (rank == 0) {
        fa.sigma_pre[j] = sg;
        fa.s[j] = s;
        fa.xg[j] = xg;
        fa.sigma[j] = sn;
        fa.gap[j] = gp;
        qn[0] += c_norm2(eta);
        qn[1] += c_norm2(dx);
        qn[2] += c_norm2(s);
        qn[3] += c_norm2(xg);
        qn[4] += c_norm2(sn);
      }
    }
    __syncthreads();
    // ---- rhs_{k+1} = data + beta gap + beta x - sigma (admm.hpp:114-119) ----
    if (tid < T.n) {
      const int p = T.pix[tid] - t0;
      const double2 d = T.data[tid], g = gap_s[p], xh = xloc[tid], sg = sig_s[p];
      double2 v;
      v.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
      v.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
      coef[tid] = v;
      if (rank == 0) jobs.j[T.q[tid]].rhs[T.i[tid]] = v;
    }
    __syncthreads();
    // ---- forward accumulate from the same shared-memory slice ----
    if (tid < sl) {
#pragma unroll
      for (int q = 0; q < kS3Q; ++q) {
        if (q >= Q) break;
        for (int c = T.qstart[q]; c < T.qstart[q + 1]; ++c) {
          const float2 a = sb[(size_t)c * sl + tid];
          cfma(acc[q][0], acc[q][1], a.x, a.y, coef[c]);
        }
      }
    }
    __syncthreads();  // buffer b (and tiles[b]) free
    if (warp == 0 && t + 2 < ntiles) issue(t + 2, b);
  }
  if (tid < sl) {
#pragma unroll
    for (int q = 0; q < kS3Q; ++q) {
      if (q >= Q) break;
      jobs.j[q].part[(int64_t)cl * ld + row0 + tid] = make_double2(acc[q][0], acc[q][1]);
    }
  }
  cluster_sync_acqrel();  // peers may still read our pdot
  fusion_finish(fa, qn);
}

}  // namespace radmm_dev

namespace radmm_dev {

// ---------------------------------------------------------------------------
// Hermitian G-apply  w = G v  reading only the lower block triangle of G.
//
// G (dual capacitance inverse, complex128, column-major, ld) is split into
// 64 x 64 tiles; a work item is a strip of up to kHermStrip tiles
// (I0 .. I0+nt-1) of tile column J, I0 >= J.  Column j of the strip feeds
//   dot part: w[j] += sum_i conj(G[i, j]) v[i]   (i in the strip, incl. the
//             diagonal tile: G[j, i] = conj(G[i, j]))
//   ax part:  w[i] += sum_j G[i, j] v[j]         (tiles strictly below the
//             diagonal: their upper mirror is never read)
// Each item writes one dot partial (64 values, slot (J, g)) and one ax
// partial per off-diagonal tile (slot tri(I, J)); herm_reduce_kernel sums
// them in a fixed order, so the result is deterministic.  HBM bytes per
// apply: ~(n^2/2 + 32 n) * 16 instead of n^2 * 16.
// ---------------------------------------------------------------------------
constexpr int kHermTile = 64;
constexpr int kHermStrip = 4;

struct HermJob {
  const double2* G;
  int64_t ld;
  int n;             // matrix order (rows of the sensor)
  int nb;            // tiles per side
  int groups;        // strip groups per tile column: ceil(nb / kHermStrip)
  const double2* v;
  double2* w;
  double2* dotp;     // [nb][groups][64]
  double2* axp;      // [nb (nb - 1) / 2][64], slot I (I - 1) / 2 + J
};

// item word: q (16) | J (16) | I0 (16) | nt (16)
__host__ __device__ inline uint64_t herm_item(int q, int J, int I0, int nt) {
  return (uint64_t)q << 48 | (uint64_t)J << 32 | (uint64_t)I0 << 16 | (uint64_t)nt;
}

__global__ void __launch_bounds__(256) herm_gapply_kernel(const __grid_constant__ Pack<HermJob> P,
                                                         const uint64_t* __restrict__ items,
                                                         const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  const uint64_t it = items[blockIdx.x];
  const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF), I0 = (int)(it >> 16 & 0xFFFF), nt = (int)(it & 0xFFFF);
  const HermJob& jb = P.j[q];
  __shared__ double2 vJ[kHermTile];
  __shared__ double2 vI[kHermStrip * kHermTile];
  __shared__ double2 sax[2][8][kHermTile];  // double-buffered: one barrier per tile
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = jb.n;
  if (tid < kHermTile) {
    const int j = J * kHermTile + tid;
    vJ[tid] = j < n ? jb.v[j] : make_double2(0.0, 0.0);
  }
  for (int t = tid; t < nt * kHermTile; t += 256) {
    const int i = I0 * kHermTile + t;
    vI[t] = i < n ? jb.v[i] : make_double2(0.0, 0.0);
  }
  const int c0 = warp * 8;  // this warp's 8 columns of the tile column
  const double2* Gc = jb.G + (int64_t)(J * kHermTile + c0) * jb.ld;
  double2 g[8][2];
  auto load_tile = [&](int I) {
    const int ib = I * kHermTile;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib + lane + 32 * h, j = J * kHermTile + c0 + k;
        g[k][h] = (i < n && j < n) ? __ldg(Gc + (int64_t)k * jb.ld + i) : make_double2(0.0, 0.0);
      }
  };
  load_tile(I0);
  __syncthreads();
  double dr[8], di[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) dr[k] = di[k] = 0.0;
  int par = 0;
  for (int t = 0; t < nt; ++t) {
    const int I = I0 + t;
    double ar[2] = {0.0, 0.0}, ai[2] = {0.0, 0.0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double2 vi = vI[t * kHermTile + lane + 32 * h];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        // conj(g) * v_i
        dr[k] = fma(g[k][h].x, vi.x, dr[k]);
        dr[k] = fma(g[k][h].y, vi.y, dr[k]);
        di[k] = fma(g[k][h].x, vi.y, di[k]);
        di[k] = fma(-g[k][h].y, vi.x, di[k]);
        // g * v_j
        const double2 vj = vJ[c0 + k];
        ar[h] = fma(g[k][h].x, vj.x, ar[h]);
        ar[h] = fma(-g[k][h].y, vj.y, ar[h]);
        ai[h] = fma(g[k][h].x, vj.y, ai[h]);
        ai[h] = fma(g[k][h].y, vj.x, ai[h]);
      }
    }
    if (t + 1 < nt) load_tile(I + 1);  // in flight across the reduction below
    if (I != J) {  // strictly-lower tile: its mirror contributes to rows of block I
#pragma unroll
      for (int h = 0; h < 2; ++h) sax[par][warp][lane + 32 * h] = make_double2(ar[h], ai[h]);
      __syncthreads();
      if (tid < kHermTile) {
        double2 sum = sax[par][0][tid];
#pragma unroll
        for (int w8 = 1; w8 < 8; ++w8) {
          sum.x += sax[par][w8][tid].x;
          sum.y += sax[par][w8][tid].y;
        }
        jb.axp[((int64_t)I * (I - 1) / 2 + J) * kHermTile + tid] = sum;
      }
      par ^= 1;  // the other buffer's readers are past this barrier
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    dr[k] = warp_sum(dr[k]);
    di[k] = warp_sum(di[k]);
  }
  if (lane == 0) {
    const int gi = (I0 - J) / kHermStrip;
    double2* dp = jb.dotp + ((int64_t)J * jb.groups + gi) * kHermTile + c0;
#pragma unroll
    for (int k = 0; k < 8; ++k) dp[k] = make_double2(dr[k], di[k]);
  }
}

// w[b*64 + r] = sum_g dotp[b][g][r] + sum_{J < b} axp[tri(b, J)][r]  (fixed order)
// 256 threads per row block: slice s = tid / 64 sums the partials k = s, s+4, ...
// of the row's list (4 independent loads in flight), then the 4 slice sums are
// added in slice order -- deterministic.
__global__ void __launch_bounds__(256) herm_reduce_kernel(const __grid_constant__ Pack<HermJob> P,
                                                         const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;
  const HermJob& jb = P.j[blockIdx.y];
  const int b = blockIdx.x, r = threadIdx.x & 63, sl = threadIdx.x >> 6;
  __shared__ double2 part[4][kHermTile];
  if (b >= jb.nb) return;
  const int ng = (jb.nb - b + kHermStrip - 1) / kHermStrip;
  const int total = ng + b;  // dot partials, then ax partials J = 0 .. b-1
  const double2* dbase = jb.dotp + (int64_t)b * jb.groups * kHermTile + r;
  const double2* abase = jb.axp + (int64_t)b * (b - 1) / 2 * kHermTile + r;
  double2 s = make_double2(0.0, 0.0);
  for (int k0 = sl; k0 < total; k0 += 16) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + 4 * u;
      v[u] = k < total ? (k < ng ? dbase[(int64_t)k * kHermTile] : abase[(int64_t)(k - ng) * kHermTile])
                       : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s.x += v[u].x;
      s.y += v[u].y;
    }
  }
  part[sl][r] = s;
  __syncthreads();
  if (sl == 0) {
    const int row = b * kHermTile + r;
    double2 t = part[0][r];
#pragma unroll
    for (int u = 1; u < 4; ++u) {
      t.x += part[u][r].x;
      t.y += part[u][r].y;
    }
    if (row < jb.n) jb.w[row] = t;
  }
}

// TMA-staged variant: persistent CTAs (one per SM) walk the item list
// round-robin; warp 8 streams each 64 x 64 tile (64 column segments of
// <= 1 KB) into a kHermStages-deep shared ring with cp.async.bulk, and the
// eight compute warps consume it exactly like herm_gapply_kernel.
constexpr int kHermStages = 3;
constexpr int kHermTileBytes = kHermTile * kHermTile * 16;
constexpr size_t kHermTmaSmem = (size_t)kHermStages * kHermTileBytes + 2 * 8 * kHermTile * 16 + 2 * kHermStages * 8;

__device__ __forceinline__ void mbar_wait_cta_acq(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "HW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra HW_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__global__ void __launch_bounds__(288, 1) herm_gapply_tma_kernel(const __grid_constant__ Pack<HermJob> P,
                                                                const uint64_t* __restrict__ items, int n_items,
                                                                const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;
  extern __shared__ __align__(128) uint8_t hsm[];
  double2* ring = reinterpret_cast<double2*>(hsm);
  double2(*sax)[8][kHermTile] = reinterpret_cast<double2(*)[8][kHermTile]>(hsm + (size_t)kHermStages * kHermTileBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(hsm + (size_t)kHermStages * kHermTileBytes + 2 * 8 * kHermTile * 16);
  uint64_t* empty = full + kHermStages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kHermStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {
    // producer: the same tile sequence the consumers walk
    int slot = 0;
    unsigned phase = 0;
    int seq = 0;
    for (int it_i = blockIdx.x; it_i < n_items; it_i += gridDim.x) {
      const uint64_t it = items[it_i];
      const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF), I0 = (int)(it >> 16 & 0xFFFF),
                nt = (int)(it & 0xFFFF);
      const HermJob& jb = P.j[q];
      const int cols = min(kHermTile, jb.n - J * kHermTile);
      for (int t = 0; t < nt; ++t, ++seq) {
        const int I = I0 + t;
        const int rows = min(kHermTile, jb.n - I * kHermTile);
        if (seq >= kHermStages) mbar_wait_cta_acq(&empty[slot], phase ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&full[slot], (unsigned)(cols * rows * 16));
        __syncwarp();
        double2* dst = ring + (size_t)slot * kHermTile * kHermTile;
        const double2* src = jb.G + (int64_t)(J * kHermTile) * jb.ld + I * kHermTile;
        for (int c = lane; c < cols; c += 32)
          tma_bulk_g2s(dst + c * kHermTile, src + (int64_t)c * jb.ld, (unsigned)(rows * 16), &full[slot]);
        if (++slot == kHermStages) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  // consumers (warps 0..7)
  int slot = 0;
  unsigned phase = 0;
  int par = 0;
  const int c0 = warp * 8;
  for (int it_i = blockIdx.x; it_i < n_items; it_i += gridDim.x) {
    const uint64_t it = items[it_i];
    const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF), I0 = (int)(it >> 16 & 0xFFFF), nt = (int)(it & 0xFFFF);
    const HermJob& jb = P.j[q];
    const int n = jb.n;
    double2 vj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int j = J * kHermTile + c0 + k;
      vj[k] = j < n ? jb.v[j] : make_double2(0.0, 0.0);
    }
    double dr[8], di[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dr[k] = di[k] = 0.0;
    for (int t = 0; t < nt; ++t) {
      const int I = I0 + t;
      const int ib = I * kHermTile;
      double2 vi[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib + lane + 32 * h;
        vi[h] = i < n ? jb.v[i] : make_double2(0.0, 0.0);
      }
      mbar_wait_cta_acq(&full[slot], phase);
      const double2* tile = ring + (size_t)slot * kHermTile * kHermTile;
      double ar[2] = {0.0, 0.0}, ai[2] = {0.0, 0.0};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = J * kHermTile + c0 + k;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = ib + lane + 32 * h;
          const double2 g = (i < n && j < n) ? tile[(c0 + k) * kHermTile + lane + 32 * h] : make_double2(0.0, 0.0);
          dr[k] = fma(g.x, vi[h].x, dr[k]);
          dr[k] = fma(g.y, vi[h].y, dr[k]);
          di[k] = fma(g.x, vi[h].y, di[k]);
          di[k] = fma(-g.y, vi[h].x, di[k]);
          ar[h] = fma(g.x, vj[k].x, ar[h]);
          ar[h] = fma(-g.y, vj[k].y, ar[h]);
          ai[h] = fma(g.x, vj[k].y, ai[h]);
          ai[h] = fma(g.y, vj[k].x, ai[h]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&empty[slot]);
      if (++slot == kHermStages) {
        slot = 0;
        phase ^= 1;
      }
      if (I != J) {
#pragma unroll
        for (int h = 0; h < 2; ++h) sax[par][warp][lane + 32 * h] = make_double2(ar[h], ai[h]);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (tid < kHermTile) {
          double2 s = sax[par][0][tid];
#pragma unroll
          for (int w8 = 1; w8 < 8; ++w8) {
            s.x += sax[par][w8][tid].x;
            s.y += sax[par][w8][tid].y;
          }
          jb.axp[((int64_t)I * (I - 1) / 2 + J) * kHermTile + tid] = s;
        }
        par ^= 1;  // the other buffer is free: its readers passed this barrier
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dr[k] = warp_sum(dr[k]);
      di[k] = warp_sum(di[k]);
    }
    if (lane == 0) {
      const int g = (I0 - J) / kHermStrip;
      double2* dp = jb.dotp + ((int64_t)J * jb.groups + g) * kHermTile + c0;
#pragma unroll
      for (int k = 0; k < 8; ++k) dp[k] = make_double2(dr[k], di[k]);
    }
  }
}

// Hermitian projection of a factor in place: G <- (G + G^H) / 2 (the nearest
// Hermitian matrix; never increases the Frobenius error of an inverse).
// One 32 x 32 tile pair (I > J) or diagonal tile per CTA, staged through
// shared memory so both halves are read and written coalesced.
__global__ void __launch_bounds__(256) herm_symmetrize_kernel(double2* __restrict__ G, int64_t ld, int n) {
  __shared__ double2 a[32][33], b[32][33];
  int t = blockIdx.x, I = 0;
  while (t > I) { t -= I + 1; ++I; }
  const int J = t;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int i = I * 32 + tx, j = J * 32 + r;          // tile (I, J): column j, row i
    a[r][tx] = (i < n && j < n) ? G[i + (int64_t)j * ld] : make_double2(0.0, 0.0);
    const int i2 = J * 32 + tx, j2 = I * 32 + r;        // tile (J, I)
    b[r][tx] = (i2 < n && j2 < n) ? G[i2 + (int64_t)j2 * ld] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 m[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = ty + 8 * u;
    // element (row I*32+tx, col J*32+r) pairs with (row J*32+r, col I*32+tx) = b[tx][r]
    const double2 x = a[r][tx], y = b[tx][r];
    m[u] = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
    if (I * 32 + tx == J * 32 + r) m[u].y = 0.0;
  }
  __syncthreads();  // everyone has read a and b
#pragma unroll
  for (int u = 0; u < 4; ++u) a[ty + 8 * u][tx] = m[u];
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = I * 32 + tx, j = J * 32 + r;  // tile (I, J), coalesced over tx
    if (i < n && j < n) G[i + (int64_t)j * ld] = a[r][tx];
    const int i2 = J * 32 + tx, j2 = I * 32 + r;  // tile (J, I) = conj transpose
    const double2 v = a[tx][r];
    if (I != J && i2 < n && j2 < n) G[i2 + (int64_t)j2 * ld] = make_double2(v.x, -v.y);
  }
}

// Row-segmented adjoint (KM too large for one shared vector per CTA): the
// segment kernels stored partial dots part[s * stride + i]; sum them in
// segment order and apply the x-update epilogue (admm.hpp:114-122).
struct XFinJob {
  ColDotJob a;
  const double2* part;
  int nseg;
  int64_t stride;
};

__global__ void __launch_bounds__(256) xdual_finish_kernel(const __grid_constant__ Pack<XFinJob> P, double mu,
                                                          double beta, const int* __restrict__ go) {
  if (go && __ldg(go) == 0) return;
  const XFinJob& jb = P.j[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= jb.a.n_out) return;
  double re = 0.0, im = 0.0;
  for (int sg = 0; sg < jb.nseg; ++sg) {
    const double2 v = jb.part[(int64_t)sg * jb.stride + i];
    re += v.x;
    im += v.y;
  }
  coldot_epilogue<EPI_XDUAL>(jb.a, i, re, im, mu, beta);
}

// back_projection (forward_model.hpp:203-220): |sum_q A_q^H y_q| for every
// pixel, summing the per-sensor adjoint images in global sensor order.
__global__ void bp_sum_kernel(const double2* const* __restrict__ imgs, int Q, int N, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int q = 0; q < Q; ++q) acc = c_add(acc, imgs[q][j]);
  out[j] = c_abs(acc);
}

// ---------------------------------------------------------------------------
// Frame-batched contractions (BASELINE config 5).  F <= 16 frames that share
// a sensor's operator and full active set turn the three per-iteration
// matvecs into GEMMs with F right-hand sides, so A_q is streamed ONCE for all
// frames and the work runs on the fp64 tensor cores (DMMA m8n8k4):
//   FWD  V_f = A_q RHS_f        (M = rows,   K = pixels; split-K partials)
//   GAP  W_f = G_q V_f          (M = rows,   K = rows;   split-K partials)
//   ADJ  X_f = (RHS_f - mu A_q^H W_f) / beta, + history / scatter epilogue
//        (M = pixels, K = rows)
// CTA tile 128 x 16 (frames), BK = 8, 8 warps x (16 rows x 16 frames).
// ---------------------------------------------------------------------------
constexpr int kFB = 16;            // max frames per batch
constexpr int kFbBM = 128, kFbPA = 132, kFbPB = 20;
enum { FB_FWD = 0, FB_GAP = 1, FB_ADJ = 2 };

struct FrameBatchJob {
  const void* A;        // float2 operator (FWD/ADJ) or double2 factor (GAP)
  int64_t lda;
  int m, k;             // GEMM M and K
  int nf;               // frames in this batch
  const double2* B[kFB];  // per-frame right-hand side (length k)
  double2* part;        // FWD/GAP: partials [split][kFB][ldp]
  int64_t ldp;
  // ADJ epilogue, per frame
  const double2* rhs[kFB];
  double2* x_hat[kFB];
  double2* x_full[kFB];
  double* ring[kFB];
};

constexpr int kFbBK = 16;  // K per shared stage (4 DMMA k-steps per barrier)
constexpr size_t kFbSmem = (size_t)2 * 2 * kFbBK * (kFbPA + kFbPB) * sizeof(double);

template <int MODE>
__global__ void __launch_bounds__(256, 2) frame_batch_kernel(const FrameBatchJob* __restrict__ jobs, int nsplit,
                                                            double mu, double beta) {
  constexpr int BK = kFbBK, LA = kFbBM * BK / 256;
  const FrameBatchJob& jb = jobs[blockIdx.z];
  const int m0 = blockIdx.x * kFbBM;
  if (m0 >= jb.m) return;
  const int split = blockIdx.y;
  const int nk_all = (jb.k + BK - 1) / BK;
  const int per = (nk_all + nsplit - 1) / nsplit;
  const int t0 = split * per, t1 = min(nk_all, t0 + per);
  extern __shared__ double fsm[];
  double(*As)[2][BK][kFbPA] = reinterpret_cast<double(*)[2][BK][kFbPA]>(fsm);
  double(*Bs)[2][BK][kFbPB] = reinterpret_cast<double(*)[2][BK][kFbPB]>(fsm + 2 * 2 * BK * kFbPA);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp * 16, fr = lane >> 2, fc = lane & 3;
  const int nb = jb.nf > 8 ? 2 : 1;  // 8-frame DMMA column blocks actually used
  double cr[2][2][2], ci[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
  double2 pa[LA], pb = make_double2(0.0, 0.0);
  auto a_pos = [&](int e, int& ii, int& kk) {
    if (MODE == FB_ADJ) { kk = e & (BK - 1); ii = e / BK; } else { ii = e & (kFbBM - 1); kk = e / kFbBM; }
  };
  auto fetch = [&](int kk0) {
#pragma unroll
    for (int t = 0; t < LA; ++t) {
      int ii, kk;
      a_pos(tid + t * 256, ii, kk);
      const int gi = m0 + ii, gk = kk0 + kk;
      double2 v = make_double2(0.0, 0.0);
      if (gi < jb.m && gk < jb.k) {
        if (MODE == FB_GAP) {
          v = reinterpret_cast<const double2*>(jb.A)[gi + (int64_t)gk * jb.lda];
        } else if (MODE == FB_FWD) {
          const float2 x = reinterpret_cast<const float2*>(jb.A)[gi + (int64_t)gk * jb.lda];
          v = make_double2((double)x.x, (double)x.y);
        } else {  // conj(A[gk, gi])
          const float2 x = reinterpret_cast<const float2*>(jb.A)[gk + (int64_t)gi * jb.lda];
          v = make_double2((double)x.x, -(double)x.y);
        }
      }
      pa[t] = v;
    }
    {  // B: BK x 16 frames, one element per thread
      const int kk = tid & (BK - 1), f = tid / BK, gk = kk0 + kk;
      pb = (f < jb.nf && gk < jb.k) ? jb.B[f][gk] : make_double2(0.0, 0.0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int t = 0; t < LA; ++t) {
      int ii, kk;
      a_pos(tid + t * 256, ii, kk);
      As[buf][0][kk][ii] = pa[t].x;
      As[buf][1][kk][ii] = pa[t].y;
    }
    const int kk = tid & (BK - 1), f = tid / BK;
    Bs[buf][0][kk][f] = pb.x;
    Bs[buf][1][kk][f] = pb.y;
  };
  if (t0 < t1) {
    fetch(t0 * BK);
    stash(0);
  }
  __syncthreads();
  for (int t = t0; t < t1; ++t) {
    const int cur = (t - t0) & 1;
    if (t + 1 < t1) fetch((t + 1) * BK);  // a whole stage ahead of its use
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[2], ai[2], nai[2], br[2], bi[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        ar[a] = As[cur][0][k4 + fc][wm + 8 * a + fr];
        ai[a] = As[cur][1][k4 + fc][wm + 8 * a + fr];
        nai[a] = -ai[a];
      }
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        br[b] = Bs[cur][0][k4 + fc][8 * b + fr];
        bi[b] = Bs[cur][1][k4 + fc][8 * b + fr];
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          if (b < nb) {
            dmma884(cr[a][b], ar[a], br[b]);
            dmma884(cr[a][b], nai[a], bi[b]);
            dmma884(ci[a][b], ar[a], bi[b]);
            dmma884(ci[a][b], ai[a], br[b]);
          }
        }
    }
    if (t + 1 < t1) stash(cur ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = m0 + wm + 8 * a + fr, f = 8 * b + 2 * fc + v;
        if (i >= jb.m || f >= jb.nf) continue;
        if (MODE != FB_ADJ) {
          jb.part[((int64_t)split * kFB + f) * jb.ldp + i] = make_double2(cr[a][b][v], ci[a][b][v]);
        } else {
          // x = (rhs - mu A^H w) / beta  (Woodbury form of solver_core.hpp:47-51), admm.hpp:120-123
          const double2 r = jb.rhs[f][i];
          const double2 xh = make_double2(__ddiv_rn(__dsub_rn(r.x, __dmul_rn(mu, cr[a][b][v])), beta),
                                          __ddiv_rn(__dsub_rn(r.y, __dmul_rn(mu, ci[a][b][v])), beta));
          const double2 old = jb.x_full[f][i];
          jb.ring[f][i] = c_abs(c_sub(xh, old));
          jb.x_full[f][i] = xh;
          jb.x_hat[f][i] = xh;
        }
      }
}

// Operator passes (FWD, ADJ) of the frame batch as a kFbStages-deep cp.async
// pipeline: raw complex64 operator tiles and complex128 frame vectors go
// global -> shared without registers (zero-filled outside the matrix), and
// are converted to fp64 (conjugated for ADJ) when the DMMA fragments are
// loaded.  FWD tiles are k-major ([kk][row], 128 contiguous complex64 per
// kk); ADJ tiles are pixel-major ([pixel][kk], each pixel's 16 rows are one
// 128-B run), so every 16-B chunk lands contiguously.  Pitches keep the
// fragment loads of each half warp on distinct banks.
constexpr int kFbStages = 4;
constexpr int kFbPF = 132;  // FWD: float2 per kk row (128 + 4)
constexpr int kFbPX = 20;   // ADJ: float2 per pixel row (16 + 4)
constexpr int kFbPV = 20;   // frame vectors: double2 per frame row (16 + 4)
constexpr size_t kFbStageA = (size_t)kFbBK * kFbPF * 8 > (size_t)kFbBM * kFbPX * 8 ? (size_t)kFbBK * kFbPF * 8
                                                                                     : (size_t)kFbBM * kFbPX * 8;
constexpr size_t kFbStageB = (size_t)kFB * kFbPV * 16;
constexpr size_t kFb2Smem = kFbStages * (kFbStageA + kFbStageB) + kFB * 8;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(256, 2) frame_batch2_kernel(const FrameBatchJob* __restrict__ jobs, int nsplit,
                                                             double mu, double beta) {
  constexpr int BK = kFbBK, S = kFbStages;
  const FrameBatchJob& jb = jobs[blockIdx.z];
  const int m0 = blockIdx.x * kFbBM;
  if (m0 >= jb.m) return;
  const int split = blockIdx.y;
  const int nk_all = (jb.k + BK - 1) / BK;
  const int per = (nk_all + nsplit - 1) / nsplit;
  const int t0 = split * per, t1 = min(nk_all, t0 + per);
  const int nt = max(0, t1 - t0);
  extern __shared__ __align__(16) uint8_t fsm2[];
  uint8_t* sA = fsm2;
  uint8_t* sB = fsm2 + S * kFbStageA;
  const double2** Bp = reinterpret_cast<const double2**>(fsm2 + S * (kFbStageA + kFbStageB));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kFB) Bp[tid] = tid < jb.nf ? jb.B[tid] : nullptr;
  __syncthreads();
  const int wm = warp * 16, fr = lane >> 2, fc = lane & 3;
  const int nb = jb.nf > 8 ? 2 : 1;
  const int m = jb.m, kdim = jb.k, nf = jb.nf;
  const int64_t lda = jb.lda;
  const float2* A = reinterpret_cast<const float2*>(jb.A);
  auto issue = [&](int t, int slot) {  // stage t (absolute) -> shared slot
    const int k0 = t * BK;
    float2* a = reinterpret_cast<float2*>(sA + slot * kFbStageA);
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // 1024 16-B chunks of A
      const int c = tid + 256 * u;
      if (MODE == FB_FWD) {  // chunk: rows 2*(c & 63) .. +1 of column kk = c >> 6
        const int kk = c >> 6, ii = 2 * (c & 63);
        const int gi = m0 + ii, gk = k0 + kk;
        // rows [m, lda) are the operator's zeroed padding: readable, and zero
        const bool ok = gi < lda && gk < kdim;
        cp_async16(a + kk * kFbPF + ii, ok ? A + gi + (int64_t)gk * lda : A, ok);
      } else {  // ADJ chunk: rows 2*(c & 7) .. +1 of pixel ii = c >> 3
        const int ii = c >> 3, kk = 2 * (c & 7);
        const int gi = m0 + ii, gk = k0 + kk;
        const bool ok = gi < m && gk < kdim;
        cp_async16(a + ii * kFbPX + kk, ok ? A + gk + (int64_t)gi * lda : A, ok);
      }
    }
    {  // B: 16 frames x 16 k (double2), one chunk per thread
      double2* b = reinterpret_cast<double2*>(sB + slot * kFbStageB);
      const int f = tid >> 4, kk = tid & 15, gk = k0 + kk;
      const bool ok = f < nf && gk < kdim;
      cp_async16(b + f * kFbPV + kk, ok ? Bp[f] + gk : reinterpret_cast<const double2*>(A), ok);
    }
  };
  // 3M (Karatsuba) complex products: P1 = sum Ar Br, P2 = sum Ai Bi,
  // P3 = sum (Ar + Ai)(Br + Bi); Re = P1 - P2, Im = P3 - P1 - P2 (3 DMMAs per
  // complex 8x8x4 block instead of 4)
  double p1[2][2][2], p2[2][2][2], p3[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) p1[a][b][v] = p2[a][b][v] = p3[a][b][v] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < S - 1; ++s0) {
    if (s0 < nt) issue(t0 + s0, s0);
    cp_async_commit();
  }
  for (int t = 0; t < nt; ++t) {
    cp_async_wait<S - 2>();
    __syncthreads();  // stage t landed for everyone; slot (t-1) % S is free
    if (t + S - 1 < nt) issue(t0 + t + S - 1, (t + S - 1) % S);
    cp_async_commit();
    const int slot = t % S;
    const float2* a = reinterpret_cast<const float2*>(sA + slot * kFbStageA);
    const double2* b = reinterpret_cast<const double2*>(sB + slot * kFbStageB);
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[2], ai[2], as[2], br[2], bi[2], bs[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int row = wm + 8 * q + fr, kk = k4 + fc;
        const float2 x = MODE == FB_FWD ? a[kk * kFbPF + row] : a[row * kFbPX + kk];
        ar[q] = (double)x.x;
        ai[q] = MODE == FB_FWD ? (double)x.y : -(double)x.y;
        as[q] = ar[q] + ai[q];
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 y = b[(8 * q + fr) * kFbPV + k4 + fc];
        br[q] = y.x;
        bi[q] = y.y;
        bs[q] = y.x + y.y;
      }
#pragma unroll
      for (int qa = 0; qa < 2; ++qa)
#pragma unroll
        for (int qb = 0; qb < 2; ++qb)
          if (qb < nb) {
            dmma884(p1[qa][qb], ar[qa], br[qb]);
            dmma884(p2[qa][qb], ai[qa], bi[qb]);
            dmma884(p3[qa][qb], as[qa], bs[qb]);
          }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int qa = 0; qa < 2; ++qa)
#pragma unroll
    for (int qb = 0; qb < 2; ++qb)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = m0 + wm + 8 * qa + fr, f = 8 * qb + 2 * fc + v;
        if (i >= m || f >= nf) continue;
        const double cre = p1[qa][qb][v] - p2[qa][qb][v];
        const double cim = p3[qa][qb][v] - p1[qa][qb][v] - p2[qa][qb][v];
        if (MODE == FB_FWD) {
          jb.part[((int64_t)split * kFB + f) * jb.ldp + i] = make_double2(cre, cim);
        } else {
          const double2 r = jb.rhs[f][i];
          const double2 xh = make_double2(__ddiv_rn(__dsub_rn(r.x, __dmul_rn(mu, cre)), beta),
                                          __ddiv_rn(__dsub_rn(r.y, __dmul_rn(mu, cim)), beta));
          const double2 old = jb.x_full[f][i];
          jb.ring[f][i] = c_abs(c_sub(xh, old));
          jb.x_full[f][i] = xh;
          jb.x_hat[f][i] = xh;
        }
      }
}

// Dual capacitance C = beta I + mu A_J A_J^H (the Woodbury system of
// solver_core.hpp:39-40) on the fp64 tensor cores: 4-stage cp.async pipeline
// of the complex64 columns A(:, J_k) (both operands come from the same
// columns: rows i of the tile and rows j of its mirror), DMMA m8n8k4 f64.
// Lower 128 x 64 tiles only; the upper triangle is written as the exact
// conjugate mirror and the diagonal is exactly real, as the SIMT path does.
// The active-column indices of stage t+S-1 are fetched into registers one
// iteration ahead so the gathered addresses never stall the pipeline.
struct GramJob {
  const float2* A;
  int64_t lda;
  const int* J;  // active columns (n entries)
  int n;         // K
  int m;         // rows (matrix order)
  double2* C;
  int64_t ldc;
};
constexpr int kGrBM = 128, kGrBN = 64, kGrPA = 132, kGrPB = 68;
constexpr size_t kGrStage = (size_t)kFbBK * (kGrPA + kGrPB) * 8;
constexpr size_t kGramSmem = kFbStages * kGrStage;

__global__ void __launch_bounds__(256, 1) gram_dmma_kernel(const GramJob* __restrict__ jobs, double mu, double beta) {
  constexpr int BK = kFbBK, S = kFbStages;
  const GramJob& jb = jobs[blockIdx.z];
  const int m0 = blockIdx.y * kGrBM, n0 = blockIdx.x * kGrBN;
  const int m = jb.m;
  if (m0 >= m || n0 >= m || m0 + kGrBM <= n0) return;  // outside, or strictly upper
  extern __shared__ __align__(16) uint8_t gsm2[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32, fr = lane >> 2, fc = lane & 3;
  const int64_t lda = jb.lda;
  const float2* A = jb.A;
  const int* J = jb.J;
  const int nk = (jb.n + BK - 1) / BK;
  // chunk c of the A tile: rows 2*(c & 63) of column kk = c >> 6 (4 per thread);
  // B tile: rows 2*(c & 31) of column kk = c >> 5 (2 per thread)
  int ja[4], jbn[2];
  auto load_j = [&](int t) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int gk = t * BK + ((tid + 256 * u) >> 6);
      ja[u] = gk < jb.n ? (J ? __ldg(J + gk) : gk) : -1;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int gk = t * BK + ((tid + 256 * u) >> 5);
      jbn[u] = gk < jb.n ? (J ? __ldg(J + gk) : gk) : -1;
    }
  };
  auto issue = [&](int slot) {
    float2* a = reinterpret_cast<float2*>(gsm2 + slot * kGrStage);
    float2* b = a + BK * kGrPA;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = tid + 256 * u, kk = c >> 6, ii = 2 * (c & 63);
      const int gi = m0 + ii;
      const bool ok = ja[u] >= 0 && gi < lda;
      cp_async16(a + kk * kGrPA + ii, ok ? A + gi + (int64_t)ja[u] * lda : A, ok);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = tid + 256 * u, kk = c >> 5, jj = 2 * (c & 31);
      const int gj = n0 + jj;
      const bool ok = jbn[u] >= 0 && gj < lda;
      cp_async16(b + kk * kGrPB + jj, ok ? A + gj + (int64_t)jbn[u] * lda : A, ok);
    }
  };
  // 3M complex products (see frame_batch2_kernel): P1 = sum ar br, P2 = sum ai bi,
  // P3 = sum (ar + ai)(br + bi); Re = P1 - P2, Im = P3 - P1 - P2
  double p1[4][4][2], p2[4][4][2], p3[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) p1[a][b][v] = p2[a][b][v] = p3[a][b][v] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < S - 1; ++s0) {
    if (s0 < nk) {
      load_j(s0);
      issue(s0);
    }
    cp_async_commit();
  }
  if (S - 1 < nk) load_j(S - 1);
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<S - 2>();
    __syncthreads();
    if (t + S - 1 < nk) {
      issue((t + S - 1) % S);                   // indices fetched last iteration
      if (t + S < nk) load_j(t + S);            // in flight during this stage's math
    }
    cp_async_commit();
    const float2* a = reinterpret_cast<const float2*>(gsm2 + (t % S) * kGrStage);
    const float2* b = a + BK * kGrPA;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double ar[4], ai[4], as[4], br[4], bi[4], bs[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 x = a[(k4 + fc) * kGrPA + wm + 8 * q + fr];
        ar[q] = (double)x.x;
        ai[q] = (double)x.y;
        as[q] = ar[q] + ai[q];
        const float2 y = b[(k4 + fc) * kGrPB + wn + 8 * q + fr];  // B = conj(A(j, k))
        br[q] = (double)y.x;
        bi[q] = -(double)y.y;
        bs[q] = br[q] + bi[q];
      }
#pragma unroll
      for (int qa = 0; qa < 4; ++qa)
#pragma unroll
        for (int qb = 0; qb < 4; ++qb) {
          dmma884(p1[qa][qb], ar[qa], br[qb]);
          dmma884(p2[qa][qb], ai[qa], bi[qb]);
          dmma884(p3[qa][qb], as[qa], bs[qb]);
        }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int qa = 0; qa < 4; ++qa)
#pragma unroll
    for (int qb = 0; qb < 4; ++qb)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int i = m0 + wm + 8 * qa + fr, j = n0 + wn + 8 * qb + 2 * fc + v;
        if (i >= m || j >= m || i < j) continue;
        const double cre = p1[qa][qb][v] - p2[qa][qb][v];
        const double cim = p3[qa][qb][v] - p1[qa][qb][v] - p2[qa][qb][v];
        double2 o = make_double2(mu * cre, mu * cim);
        if (i == j) {
          o.x += beta;
          o.y = 0.0;  // exact real diagonal of a Hermitian matrix
        }
        jb.C[i + (int64_t)j * jb.ldc] = o;
        if (i != j) jb.C[j + (int64_t)i * jb.ldc] = make_double2(o.x, -o.y);
      }
}

// out_f[i] = sum_s part[s][f][i] (fixed split order) for every frame of a job
struct FrameReduceJob {
  const double2* part;
  int64_t ldp;
  int m, nf, nsplit;
  double2* out[kFB];
};

__global__ void frame_reduce_kernel(const FrameReduceJob* __restrict__ jobs) {
  const FrameReduceJob& jb = jobs[blockIdx.z];
  const int i = blockIdx.x * blockDim.x + threadIdx.x, f = blockIdx.y;
  if (i >= jb.m || f >= jb.nf) return;
  double2 s = make_double2(0.0, 0.0);
  for (int sp = 0; sp < jb.nsplit; ++sp) {
    const double2 v = jb.part[((int64_t)sp * kFB + f) * jb.ldp + i];
    s.x += v.x;
    s.y += v.y;
  }
  jb.out[f][i] = s;
}

// rhs_f[j] = data_f[j] + beta gap_f[j] + beta x_hat_f[j] - sigma_f[j] for the
// full active set (admm.hpp:114-119), every (sensor, frame) of the batch.
struct FrameRhsJob {
  int n;
  const double2* data;
  const double2* x_hat;
  const double2* gap;
  const double2* sigma;
  double2* rhs;
};

__global__ void frame_rhs_kernel(const FrameRhsJob* __restrict__ jobs, double beta) {
  const FrameRhsJob& jb = jobs[blockIdx.y];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= jb.n) return;
  const double2 d = jb.data[j], g = jb.gap[j], x = jb.x_hat[j], sg = jb.sigma[j];
  jb.rhs[j] = make_double2(__dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, x.x)), sg.x),
                           __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, x.y)), sg.y));
}

// ---------------------------------------------------------------------------
// Fused single-pass sweep v4 (RADMM_FUSED=4): every operator column is read
// ONCE per iteration.  Cooperative persistent grid: CTA (c, q) owns sensor q's
// 4-pixel tiles of pixel chunk c (the Q CTAs of a chunk run concurrently).
// Shared memory: w_q (the capacitance-inverse apply, KM complex128) and a
// 3-slot ring of A tiles (4 columns x KM complex64, bulk-copied).  Step b:
//   dots(b): x_q = (rhs_q - mu A_q^H w_q) / beta for the tile, + the x-update
//            epilogue (history, scatter) -- admm.hpp:114-123;
//   publish: the Q-th sensor to finish tile b (global arrival counter) runs
//            FusionCore::round for its 4 pixels (admm.hpp:236-258), writes the
//            tile's norm partials and releases the tile flag;
//   fwd(b-1): once tile b-1's flag is up, rhs_{k+1} = data + beta gap +
//            beta x_hat - sigma (admm.hpp:114-119) and v += A(:, tile) rhs from
//            the tile still in shared memory (register accumulators);
//   refill:  tile b+2 into tile b-1's slot.
// The last CTA reduces the tile norm partials in tile order (deterministic)
// and evaluates the stopping rule.  Requires the full active set (J = id).
// ---------------------------------------------------------------------------
constexpr int kS4P = 4;          // pixels per tile
constexpr int kS4Slots = 3;
constexpr int kS4Threads = 256;

struct Sweep4Job {
  const float2* A;
  const double2* w;
  const double2* data;
  double2* rhs;
  double2* x_hat;
  double2* x_full;
  double* ring_slot;
  double2* part;  // [chunk][ld]
};

struct Sweep4Ctl {
  unsigned* tile_cnt;    // arrivals per tile (monotonic)
  unsigned* tile_flag;   // = seq when the tile's fusion is done
  double* tile_norms;    // 5 per tile
  unsigned* done;        // CTAs finished (reset by the last one)
  unsigned seq;
  int tiles_per_chunk;
  double2* xg_out;       // v5: new x_G / sigma (the inputs fa.xg / fa.sigma stay untouched)
  double2* sigma_out;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kS4Threads, 1) fused_sweep4_kernel(const __grid_constant__ Pack<Sweep4Job> P,
                                                                     const __grid_constant__ FusionArgs fa,
                                                                     const __grid_constant__ Sweep4Ctl ctl,
                                                                     double mu, double beta, int64_t ld) {
  if (fa.go && __ldg(fa.go) == 0) return;  // cancelled speculative iteration
  extern __shared__ __align__(128) uint8_t s4[];
  const int q = blockIdx.y, chunk = blockIdx.x;
  const Sweep4Job& jb = P.j[q];
  const int Q = fa.Q, N = fa.N;
  double2* sw = reinterpret_cast<double2*>(s4);                             // ld
  float2* ring = reinterpret_cast<float2*>(s4 + (size_t)ld * sizeof(double2));  // slots x P x ld
  uint64_t* full = reinterpret_cast<uint64_t*>(s4 + (size_t)ld * 16 + (size_t)kS4Slots * kS4P * ld * 8);
  __shared__ double dots[kS4P][2][2];
  __shared__ double2 rhs4[kS4P];
  __shared__ double qn[kS4P][5];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = (N + kS4P - 1) / kS4P;
  const int t0 = chunk * ctl.tiles_per_chunk, t1 = min(ntiles, t0 + ctl.tiles_per_chunk);
  const unsigned tile_bytes = (unsigned)(kS4P * ld * sizeof(float2));
  if (tid == 0) {
    for (int i = 0; i < kS4Slots; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = tid; r < ld; r += kS4Threads) sw[r] = jb.w[r];
  __syncthreads();
  auto issue = [&](int b) {  // tile b -> its slot (thread 0)
    const int slot = (b - t0) % kS4Slots;
    mbar_arrive_expect_tx(&full[slot], tile_bytes);
    for (int p = 0; p < kS4P; ++p)
      tma_bulk_g2s(ring + ((size_t)slot * kS4P + p) * ld, jb.A + (int64_t)(b * kS4P + p) * ld,
                   (unsigned)(ld * sizeof(float2)), &full[slot]);
  };
  if (tid == 0)
    for (int b = t0; b < min(t1, t0 + kS4Slots - 1); ++b) issue(b);
  double2 vacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) vacc[i] = make_double2(0.0, 0.0);
  const int rows_per_half = (int)(ld / 2);
  auto forward_tile = [&](int b) {  // v += A(:, tile b) rhs_{k+1}(tile b), once the tile's fusion is done
    if (tid == 0)
      while (ld_acquire_u32(ctl.tile_flag + b) != ctl.seq) {
      }
    __syncwarp();
    __syncthreads();
    if (tid < kS4P) {
      const int j = b * kS4P + tid;
      double2 r = make_double2(0.0, 0.0);
      if (j < N) {
        // gap / sigma were just written by another CTA: read through L2 (L1 is not coherent)
        const double2 d = jb.data[j], g = __ldcg(fa.gap + j), xh = jb.x_hat[j], sg = __ldcg(fa.sigma + j);
        r.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
        r.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
        jb.rhs[j] = r;
      }
      rhs4[tid] = r;
    }
    __syncthreads();
    const int slot = (b - t0) % kS4Slots;
#pragma unroll
    for (int p = 0; p < kS4P; ++p) {
      const float2* col = ring + ((size_t)slot * kS4P + p) * ld;
      const double2 r = rhs4[p];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = tid + kS4Threads * i;
        if (row < ld) {
          const float2 a = col[row];
          vacc[i].x = fma((double)a.x, r.x, fma(-(double)a.y, r.y, vacc[i].x));
          vacc[i].y = fma((double)a.x, r.y, fma((double)a.y, r.x, vacc[i].y));
        }
      }
    }
    __syncthreads();  // the slot is free again
  };
  for (int b = t0; b < t1; ++b) {
    const int slot = (b - t0) % kS4Slots;
    const unsigned par = (unsigned)(((b - t0) / kS4Slots) & 1);
    mbar_wait_cta_acq(&full[slot], par);
    {  // dots: warp (pixel p = warp & 3, row half h = warp >> 2)
      const int p = warp & 3, h = warp >> 2;
      const float2* col = ring + ((size_t)slot * kS4P + p) * ld + (size_t)h * rows_per_half;
      const double2* wv = sw + (size_t)h * rows_per_half;
      double re = 0.0, im = 0.0;
      for (int r = lane; r < rows_per_half; r += 32) {
        const float2 a = col[r];
        const double2 v = wv[r];
        cfma_conj(re, im, (double)a.x, (double)a.y, v);
      }
      re = warp_sum(re);
      im = warp_sum(im);
      if (lane == 0) {
        dots[p][h][0] = re;
        dots[p][h][1] = im;
      }
    }
    __syncthreads();
    if (tid < kS4P) {  // x-update epilogue (admm.hpp:120-123) for pixel j = b*4 + tid
      const int j = b * kS4P + tid;
      if (j < N) {
        const double re = dots[tid][0][0] + dots[tid][1][0], im = dots[tid][0][1] + dots[tid][1][1];
        const double2 r = jb.rhs[j];
        const double2 xh = make_double2(__ddiv_rn(__dsub_rn(r.x, __dmul_rn(mu, re)), beta),
                                        __ddiv_rn(__dsub_rn(r.y, __dmul_rn(mu, im)), beta));
        const double2 old = jb.x_full[j];
        jb.ring_slot[j] = c_abs(c_sub(xh, old));
        jb.x_full[j] = xh;
        jb.x_hat[j] = xh;
      }
      __threadfence();
    }
    __syncthreads();
    {  // publish; the Q-th arrival runs the tile's fusion round
      __shared__ bool last;
      if (tid == 0) last = (atomicAdd(ctl.tile_cnt + b, 1u) % (unsigned)Q) == (unsigned)(Q - 1);
      __syncthreads();
      if (last) {
        __threadfence();
        if (tid < kS4P) {
          double qv[5] = {0, 0, 0, 0, 0};
          const int j = b * kS4P + tid;
          if (j < N)
            // other CTAs' x_q: through L2 (L1 may hold a stale line from a neighbouring tile)
            fusion_pixel(fa, j, [&](int k) { return __ldcg(fa.contrib[k] + j); }, qv);
          for (int t = 0; t < 5; ++t) qn[tid][t] = qv[t];
        }
        __syncthreads();
        if (tid < 5) {
          double a = 0.0;
          for (int p = 0; p < kS4P; ++p) a += qn[p][tid];  // fixed pixel order
          ctl.tile_norms[(size_t)b * 5 + tid] = a;
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release_u32(ctl.tile_flag + b, ctl.seq);
      }
    }
    if (b > t0) forward_tile(b - 1);
    if (tid == 0 && b + kS4Slots - 1 < t1) issue(b + kS4Slots - 1);
  }
  if (t1 > t0) forward_tile(t1 - 1);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = tid + kS4Threads * i;
    if (row < ld) jb.part[(size_t)chunk * ld + row] = vacc[i];
  }
  // grid-wide: the last CTA reduces the tile norms in tile order and
  // evaluates the stopping rule (admm.hpp:244-256)
  __threadfence();
  __shared__ bool lastcta;
  __syncthreads();
  if (tid == 0) lastcta = atomicAdd(ctl.done, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!lastcta) return;
  __threadfence();
  __shared__ double red5[5][kS4Threads / 32];
  double acc[5] = {0, 0, 0, 0, 0};
  // each thread sums a contiguous block of tiles (in order), then blocks in order
  const int per = (ntiles + kS4Threads - 1) / kS4Threads;
  const int b0 = tid * per, b1 = min(ntiles, b0 + per);
  for (int b = b0; b < b1; ++b)
    for (int t = 0; t < 5; ++t) acc[t] += ((volatile const double*)ctl.tile_norms)[(size_t)b * 5 + t];
  double* blocksum = reinterpret_cast<double*>(ring);  // the tile ring is free now: 5 x threads
  for (int t = 0; t < 5; ++t) blocksum[t * kS4Threads + tid] = acc[t];
  __syncthreads();
  if (tid < 5) {
    double a = 0.0;
    for (int i = 0; i < kS4Threads; ++i) a += blocksum[tid * kS4Threads + i];
    red5[tid][0] = a;
  }
  __syncthreads();
  if (tid == 0) {
    FusionScalars f;
    for (int t = 0; t < 5; ++t) f.sq[t] = red5[t][0];
    f.pri_res = sqrt(f.sq[0]);
    f.dual_res = fa.beta * sqrt(f.sq[1]);
    f.eps_pri = fa.root_n_eps_abs + fa.eps_rel * fmax(sqrt(f.sq[2]), sqrt(f.sq[3]));
    f.eps_dual = fa.root_n_eps_abs + fa.eps_rel * sqrt(f.sq[4]);
    f.trigger = f.pri_res <= f.eps_pri;
    f.converged = fa.has_prev && f.trigger && f.dual_res <= f.eps_dual;
    if (fa.go_next) *fa.go_next = !((fa.stop_on_converge && f.converged) || (fa.screen_next_possible && f.trigger));
    f.iteration = fa.iteration;
    f.pad = 0;
    *fa.out_dev = f;
    if (fa.out_host) {
      volatile FusionScalars* hp = fa.out_host;
      hp->pri_res = f.pri_res; hp->dual_res = f.dual_res; hp->eps_pri = f.eps_pri; hp->eps_dual = f.eps_dual;
      for (int t = 0; t < 5; ++t) hp->sq[t] = f.sq[t];
      hp->trigger = f.trigger; hp->converged = f.converged;
      __threadfence_system();
      hp->iteration = f.iteration;
    }
    *ctl.done = 0u;
  }
}

// ---------------------------------------------------------------------------
// Fused single-pass sweep v5 (RADMM_FUSED=5): v4's data flow with the
// cross-SM latency chain taken off the streaming path (warp specialisation):
//   warp 0       producer: bulk-copies tile b into a 3-slot ring;
//   warps 1-8    dots + x-update epilogue for tile b, free the slot at once,
//                then publish (red.release on the tile's arrival counter);
//   warp 9       (sensor-0 CTA of each chunk) fusion: waits for all Q
//                arrivals of tile b, runs FusionCore::round for its 4 pixels,
//                writes the tile's norm partials, releases the tile flag;
//   warps 10-17  forward: wait for the flag of tile b, form rhs_{k+1} and add
//                A(:, tile) rhs into register accumulators, re-reading the
//                tile's columns from L2.
// The dot warps stay at most kS5Lag tiles ahead of the forward warps, which
// bounds the L2 footprint of the re-read (~kS5Lag x 64 KB per CTA).
// ---------------------------------------------------------------------------
constexpr int kS5Slots = 3;
constexpr int kS5Lag = 3;
constexpr int kS5DotWarps = 4;   // one per pixel of the tile, all rows
constexpr int kS5FwdWarps = 16;  // 4 rows per thread (KM <= 2048)
constexpr int kS5Threads = (1 + kS5DotWarps + kS5FwdWarps) * 32;
constexpr int kS5FwdRows = 4;

__global__ void __launch_bounds__(kS5Threads, 1) fused_sweep5_kernel(const __grid_constant__ Pack<Sweep4Job> P,
                                                                     const __grid_constant__ FusionArgs fa,
                                                                     const __grid_constant__ Sweep4Ctl ctl,
                                                                     double mu, double beta, int64_t ld) {
  if (fa.go && __ldg(fa.go) == 0) return;
  extern __shared__ __align__(128) uint8_t s5[];
  const int q = blockIdx.y, chunk = blockIdx.x;
  const Sweep4Job& jb = P.j[q];
  const int Q = fa.Q, N = fa.N;
  double2* sw = reinterpret_cast<double2*>(s5);
  float2* ring = reinterpret_cast<float2*>(s5 + (size_t)ld * sizeof(double2));
  uint64_t* full = reinterpret_cast<uint64_t*>(s5 + (size_t)ld * 16 + (size_t)kS5Slots * kS4P * ld * 8);
  uint64_t* empty = full + kS5Slots;
  __shared__ double2 rhs4[2][kS4P];
  __shared__ volatile int fwd_done;  // last tile whose forward finished (t0 - 1 initially)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntiles = N / kS4P;
  const int t0 = chunk * ctl.tiles_per_chunk, t1 = min(ntiles, t0 + ctl.tiles_per_chunk);
  const unsigned tile_bytes = (unsigned)(kS4P * ld * sizeof(float2));
  // arrivals per tile after this launch: one per (sensor, tile)
  const unsigned target = ctl.seq * (unsigned)Q;
  if (tid == 0) {
    for (int i = 0; i < kS5Slots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kS5DotWarps);
    }
    fwd_done = t0 - 1;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int r = tid; r < ld; r += kS5Threads) sw[r] = jb.w[r];
  __syncthreads();
  if (warp == 0) {
    // ---- producer --------------------------------------------------------
    if (lane == 0) {
      for (int b = t0; b < t1; ++b) {
        const int u = b - t0, slot = u % kS5Slots;
        if (u >= kS5Slots) mbar_wait_cta_acq(&empty[slot], (unsigned)(((u / kS5Slots) - 1) & 1));
        mbar_arrive_expect_tx(&full[slot], tile_bytes);
        for (int p = 0; p < kS4P; ++p)
          tma_bulk_g2s(ring + ((size_t)slot * kS4P + p) * ld, jb.A + (int64_t)(b * kS4P + p) * ld,
                       (unsigned)(ld * sizeof(float2)), &full[slot]);
      }
    }
    __syncwarp();
  } else if (warp <= kS5DotWarps) {
    // ---- dots + x-update + publish (warp = pixel of the tile) ---------------
    const int p = warp - 1;
    for (int b = t0; b < t1; ++b) {
      const int u = b - t0, slot = u % kS5Slots;
      while (b - fwd_done > kS5Lag) __nanosleep(64);  // bound the L2 re-read distance
      const int j = b * kS4P + p;
      double2 r_in = make_double2(0.0, 0.0), old = make_double2(0.0, 0.0);
      if (lane == 0) {  // epilogue inputs, fetched before the tile lands
        r_in = jb.rhs[j];
        old = jb.x_full[j];
      }
      mbar_wait_cta_acq(&full[slot], (unsigned)((u / kS5Slots) & 1));
      const float2* col = ring + ((size_t)slot * kS4P + p) * ld;
      double re = 0.0, im = 0.0;
      for (int r = lane; r < ld; r += 32) {
        const float2 a = col[r];
        cfma_conj(re, im, (double)a.x, (double)a.y, sw[r]);
      }
      re = warp_sum(re);
      im = warp_sum(im);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_local(&empty[slot]);  // slot consumed
        const double2 xh = make_double2(__ddiv_rn(__dsub_rn(r_in.x, __dmul_rn(mu, re)), beta),
                                        __ddiv_rn(__dsub_rn(r_in.y, __dmul_rn(mu, im)), beta));
        jb.ring_slot[j] = c_abs(c_sub(xh, old));
        jb.x_full[j] = xh;
        jb.x_hat[j] = xh;
      }
      // one arrival per (sensor, tile) once all 4 pixels are written: each
      // writer fences, the dot warps meet, and warp 1 publishes (release)
      if (lane == 0) __threadfence();
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"n"(kS5DotWarps * 32) : "memory");
      if (p == 0 && lane == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctl.tile_cnt + b) : "memory");
      __syncwarp();
    }
  } else {
    // ---- forward: v += A(:, tile) rhs_{k+1}; next tile's columns prefetched --
    const int ft = tid - (kS5DotWarps + 1) * 32;  // 0 .. 16 * 32 - 1
    constexpr int FT = kS5FwdWarps * 32;
    double2 vacc[kS5FwdRows];
#pragma unroll
    for (int i = 0; i < kS5FwdRows; ++i) vacc[i] = make_double2(0.0, 0.0);
    float2 a[kS4P][kS5FwdRows];
    auto load = [&](int b) {  // A does not depend on the fusion: fetched ahead of the flag
#pragma unroll
      for (int pp = 0; pp < kS4P; ++pp)
#pragma unroll
        for (int i = 0; i < kS5FwdRows; ++i) {
          const int row = ft + FT * i;
          a[pp][i] = row < ld ? __ldcg(jb.A + (int64_t)(b * kS4P + pp) * ld + row) : make_float2(0.f, 0.f);
        }
    };
    if (t0 < t1) load(t0);
    for (int b = t0; b < t1; ++b) {
      const int par = (b - t0) & 1;
      if (ft == 0)  // all Q sensors have published tile b
        while (ld_acquire_u32(ctl.tile_cnt + b) < target) {
        }
      __syncwarp();
      asm volatile("bar.sync 2, %0;" ::"n"(FT) : "memory");
      if (ft < kS4P) {
        // FusionCore::round for pixel j (admm.hpp:236-258), computed identically
        // in every sensor's CTA from the previous round's x_G / sigma (never
        // overwritten in this launch); sensor 0's CTA stores the new state.
        const int j = b * kS4P + ft;
        double2 sm = make_double2(0.0, 0.0);
        for (int k = 0; k < Q; ++k) sm = c_add(sm, __ldcg(fa.contrib[k] + j));  // fixed sensor order
        sm = make_double2(__ddiv_rn(sm.x, (double)Q), __ddiv_rn(sm.y, (double)Q));
        const double2 xgp = fa.xg[j];
        const double2 sg = fa.sigma[j];
        const double2 vv = make_double2(__dadd_rn(sm.x, __ddiv_rn(sg.x, fa.beta)), __dadd_rn(sm.y, __ddiv_rn(sg.y, fa.beta)));
        const double2 xg = soft_threshold1(vv, fa.kappa);
        const double2 eta = c_sub(sm, xg);
        const double2 dx = c_sub(xg, xgp);
        const double2 sn = make_double2(__dadd_rn(sg.x, __dmul_rn(fa.beta, eta.x)), __dadd_rn(sg.y, __dmul_rn(fa.beta, eta.y)));
        const double2 gp = c_sub(xg, sm);
        if (q == 0) {
          fa.sigma_pre[j] = sg;
          fa.s[j] = sm;
          ctl.xg_out[j] = xg;
          ctl.sigma_out[j] = sn;
          fa.gap[j] = gp;
          double qv[5] = {c_norm2(eta), c_norm2(dx), c_norm2(sm), c_norm2(xg), c_norm2(sn)};
#pragma unroll
          for (int t = 0; t < 5; ++t) {  // fixed pixel order: (p0 + p1) + (p2 + p3)
            double a2 = qv[t] + __shfl_down_sync(0xFu, qv[t], 1);
            a2 = a2 + __shfl_down_sync(0xFu, a2, 2);
            if (ft == 0) ctl.tile_norms[(size_t)b * 5 + t] = a2;
          }
        }
        // rhs_{k+1} = data + beta gap + beta x_hat - sigma (admm.hpp:114-119)
        const double2 d = jb.data[j], xh = __ldcg(jb.x_hat + j);
        double2 r;
        r.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, gp.x)), __dmul_rn(beta, xh.x)), sn.x);
        r.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, gp.y)), __dmul_rn(beta, xh.y)), sn.y);
        jb.rhs[j] = r;
        rhs4[par][ft] = r;
      }
      __syncwarp();
      asm volatile("bar.sync 2, %0;" ::"n"(FT) : "memory");
#pragma unroll
      for (int pp = 0; pp < kS4P; ++pp) {
        const double2 r = rhs4[par][pp];
#pragma unroll
        for (int i = 0; i < kS5FwdRows; ++i) {
          vacc[i].x = fma((double)a[pp][i].x, r.x, fma(-(double)a[pp][i].y, r.y, vacc[i].x));
          vacc[i].y = fma((double)a[pp][i].x, r.y, fma((double)a[pp][i].y, r.x, vacc[i].y));
        }
      }
      if (b + 1 < t1) load(b + 1);  // in flight during the next flag wait
      if (ft == 0) fwd_done = b;
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < kS5FwdRows; ++i) {
      const int row = ft + FT * i;
      if (row < ld) jb.part[(size_t)chunk * ld + row] = vacc[i];
    }
  }
  // ---- grid-wide: stopping rule by the last CTA ------------------------------
  __syncthreads();
  __threadfence();
  __shared__ bool lastcta;
  if (tid == 0) lastcta = atomicAdd(ctl.done, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!lastcta) return;
  __threadfence();
  double acc[5] = {0, 0, 0, 0, 0};
  const int per = (ntiles + kS5Threads - 1) / kS5Threads;
  const int b0 = tid * per, b1 = min(ntiles, b0 + per);
  for (int b = b0; b < b1; ++b)
    for (int t = 0; t < 5; ++t) acc[t] += ((volatile const double*)ctl.tile_norms)[(size_t)b * 5 + t];
  double* blocksum = reinterpret_cast<double*>(ring);
  for (int t = 0; t < 5; ++t) blocksum[t * kS5Threads + tid] = acc[t];
  __syncthreads();
  if (tid == 0) {
    FusionScalars f;
    for (int t = 0; t < 5; ++t) {
      double a = 0.0;
      for (int i = 0; i < kS5Threads; ++i) a += blocksum[t * kS5Threads + i];
      f.sq[t] = a;
    }
    f.pri_res = sqrt(f.sq[0]);
    f.dual_res = fa.beta * sqrt(f.sq[1]);
    f.eps_pri = fa.root_n_eps_abs + fa.eps_rel * fmax(sqrt(f.sq[2]), sqrt(f.sq[3]));
    f.eps_dual = fa.root_n_eps_abs + fa.eps_rel * sqrt(f.sq[4]);
    f.trigger = f.pri_res <= f.eps_pri;
    f.converged = fa.has_prev && f.trigger && f.dual_res <= f.eps_dual;
    if (fa.go_next) *fa.go_next = !((fa.stop_on_converge && f.converged) || (fa.screen_next_possible && f.trigger));
    f.iteration = fa.iteration;
    f.pad = 0;
    *fa.out_dev = f;
    if (fa.out_host) {
      volatile FusionScalars* hp = fa.out_host;
      hp->pri_res = f.pri_res; hp->dual_res = f.dual_res; hp->eps_pri = f.eps_pri; hp->eps_dual = f.eps_dual;
      for (int t = 0; t < 5; ++t) hp->sq[t] = f.sq[t];
      hp->trigger = f.trigger; hp->converged = f.converged;
      __threadfence_system();
      hp->iteration = f.iteration;
    }
    *ctl.done = 0u;
  }
}

}  // namespace radmm_dev
