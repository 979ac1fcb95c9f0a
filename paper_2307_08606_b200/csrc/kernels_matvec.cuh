// kernels_matvec.cuh: shared helpers, job packs, column-dot and forward matvecs, fusion round, screening
// Part of kernels.cuh (see that file's header); included in order from there.
#pragma once

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
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }
// a * b + c
__device__ __forceinline__ double2 c_fma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
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
  pdl_enter();
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

// Software-pipelined column dot for complex64 operators (the adjoint pass):
// the same math and summation order as coldot_kernel<float2, EPI, true, 2>,
// but a warp streams its columns as one continuous sequence -- the loads of
// the next column pair are issued before the current pair's shuffle
// reduction and epilogue, and the epilogue's inputs (rhs, pixel, old x) are
// fetched at the start of the pair -- so no load bubble opens at column
// boundaries.  Needs a multiple of four 64-row steps (KM % 256 == 0).
template <int EPI, int THREADS, int MINB, int CPW = 2>
__global__ void __launch_bounds__(THREADS, MINB) coldot_pipe_kernel(const __grid_constant__ Pack<ColDotJob> jobs, double mu,
                                                              double beta, const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  extern __shared__ double2 sv[];
  constexpr int kWarps = THREADS / 32;
  const ColDotJob& jb = jobs.j[blockIdx.y];
  const int n_out = jb.n_out;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const int i_begin = (int)(gw * n_out / nw);
  const int i_end = (int)((gw + 1) * n_out / nw);
  if ((int)((int64_t)blockIdx.x * kWarps * n_out / nw) >= n_out) return;  // whole CTA idle
  const int64_t ld = jb.ld;
  const int64_t vld = jb.vld ? jb.vld : ld;
  const int64_t half = vld >> 1;
  for (int r = threadIdx.x; r < vld; r += blockDim.x)
    sv[ColLoad<float2, CPW>::slot(r, half)] = (r < jb.len) ? jb.vec[r] : make_double2(0.0, 0.0);
  __syncthreads();
  if (i_begin >= i_end) return;
  const int lane = threadIdx.x & 31;
  const int steps = (int)((jb.len + 63) / 64);  // multiple of 4 (host-checked)
  const float2* base = reinterpret_cast<const float2*>(jb.M);
  const double2* ve = sv + lane;
  const double2* vo = sv + half + lane;
  auto colptr = [&](int i) -> const float4* {
    const int ic = min(i, i_end - 1);
    const int col = jb.cols ? __ldg(jb.cols + ic) : ic;
    return reinterpret_cast<const float4*>(base + (int64_t)col * ld) + lane;
  };
  const float4* p[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) p[c] = colptr(i_begin + c);
  // ping-pong register buffers (no register moves of in-flight loads):
  // buffer A holds steps s, s+1 while B loads s+2, s+3, and vice versa; the
  // step count is a multiple of 4, so A holds the next pair's first steps
  // when a pair ends.
  float4 a0[CPW], a1[CPW], b0[CPW], b1[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    a0[c] = __ldg(p[c]);
    a1[c] = __ldg(p[c] + 32);
  }
  for (int i0 = i_begin; i0 < i_end; i0 += CPW) {
    const int i1 = i0 + CPW;
    const float4* pn[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) pn[c] = colptr(i1 + c);
    // epilogue inputs of this pair (lane c finishes column i0 + c)
    double2 e_rhs = make_double2(0.0, 0.0), e_old = make_double2(0.0, 0.0);
    int e_pix = 0;
    if (EPI == EPI_XDUAL && lane < CPW && i0 + lane < i_end) {
      e_rhs = jb.rhs[i0 + lane];
      e_pix = jb.pix[i0 + lane];
      e_old = jb.x_full[e_pix];
    }
    double re[CPW], im[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) re[c] = im[c] = 0.0;
    const bool more = i1 < i_end;
#pragma unroll 1
    for (int s = 0; s < steps; s += 4) {
#pragma unroll
      for (int c = 0; c < CPW; ++c) {  // B <- steps s+2, s+3 (always inside this pair)
        b0[c] = __ldg(p[c] + (s + 2) * 32);
        b1[c] = __ldg(p[c] + (s + 3) * 32);
      }
      {
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
      if (s + 4 < steps) {  // A <- steps s+4, s+5, or the next pair's first two
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          a0[c] = __ldg(p[c] + (s + 4) * 32);
          a1[c] = __ldg(p[c] + (s + 5) * 32);
        }
      } else if (more) {
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          a0[c] = __ldg(pn[c]);
          a1[c] = __ldg(pn[c] + 32);
        }
      }
      {
        const double2 e0 = ve[(s + 2) * 32], o0 = vo[(s + 2) * 32];
        const double2 e1 = ve[(s + 3) * 32], o1 = vo[(s + 3) * 32];
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          cfma_conj(re[c], im[c], b0[c].x, b0[c].y, e0);
          cfma_conj(re[c], im[c], b0[c].z, b0[c].w, o0);
          cfma_conj(re[c], im[c], b1[c].x, b1[c].y, e1);
          cfma_conj(re[c], im[c], b1[c].z, b1[c].w, o1);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      re[c] = warp_sum(re[c]);
      im[c] = warp_sum(im[c]);
    }
#pragma unroll
    for (int c = 0; c < CPW; ++c)
      if (lane == c && i0 + c < i_end) {
        if (EPI == EPI_XDUAL) {
          const double2 xh = make_double2(__ddiv_rn(__dsub_rn(e_rhs.x, __dmul_rn(mu, re[c])), beta),
                                          __ddiv_rn(__dsub_rn(e_rhs.y, __dmul_rn(mu, im[c])), beta));
          jb.ring_slot[e_pix] = c_abs(c_sub(xh, e_old));  // admm.hpp:143
          jb.x_full[e_pix] = xh;                          // admm.hpp:121-122
          jb.x_hat[i0 + c] = xh;                          // admm.hpp:120
        } else {
          coldot_epilogue<EPI>(jb, i0 + c, re[c], im[c], mu, beta);
        }
      }
#pragma unroll
    for (int c = 0; c < CPW; ++c) p[c] = pn[c];
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

// 256 threads (512-row tiles) up to KM = 4096; 512 threads (1024-row tiles) on
// taller operators (config 3: 6.0 -> 6.4 TB/s; config 2 prefers 256)
constexpr int kFwdThreads = 256;
constexpr int kFwdTile = 2 * kFwdThreads;
constexpr int kFwdTallRows = 4096;
__host__ __device__ constexpr int fwd_threads_for(int64_t ld) { return ld > kFwdTallRows ? 512 : 256; }

template <int MODE, int THREADS>
__global__ void __launch_bounds__(THREADS) fwd_kernel(const __grid_constant__ Pack<FwdJob> jobs,
                                                          const double2* __restrict__ gap,
                                                          const double2* __restrict__ sigma, double beta,
                                                          const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  extern __shared__ unsigned char smem_raw[];
  const FwdJob& jb = jobs.j[blockIdx.z];
  // row tiles fastest: the CTAs that run together cover every row tile of the
  // same column chunk, so each column is streamed whole (DRAM page / TLB locality)
  const int chunk = blockIdx.y;
  if (chunk >= jb.n_chunks) return;
  const int64_t row0 = (int64_t)blockIdx.x * (2 * THREADS);
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
      if (blockIdx.x == 0) jb.rhs_out[i] = v;
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
  pdl_enter();
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
  pdl_enter();
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
  // device-guarded screening: set when the next round screens (trigger staged,
  // not stopping); the screening kernels enqueued behind this round read it
  int* screen_go;
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
  // fixed sensor order (admm.hpp:239); the pixel's previous x_G and sigma and
  // up to eight sensor values are loaded together, then summed in order
  const double2 xgp = a.xg[j];
  const double2 sg = a.sigma[j];
  double2 s = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < a.Q; k0 += 8) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = k0 + u < a.Q ? contrib(k0 + u) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < a.Q) s = c_add(s, v[u]);
  }
  s = make_double2(__ddiv_rn(s.x, (double)a.Q), __ddiv_rn(s.y, (double)a.Q));
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
    if (a.screen_go)
      *a.screen_go = a.screen_next_possible && f.trigger && !(a.stop_on_converge && f.converged);
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
  pdl_enter();
  if (a.go && __ldg(a.go) == 0) return;  // cancelled speculative iteration
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double q[5] = {0, 0, 0, 0, 0};
  if (j < a.N) fusion_pixel(a, j, [&](int k) { return a.contrib[k][j]; }, q);
  fusion_finish(a, q);
}

// One fusion round per frame of a multi-frame batch (blockIdx.y = frame);
// each frame reduces over its own row of blocks with its own counter.
__global__ void __launch_bounds__(kFusionThreads) fusion_frames_kernel(const __grid_constant__ Pack<FusionArgs> P) {
  pdl_enter();
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

// Screening kernels run unconditionally (go, sgo == nullptr) or behind a
// fusion round, guarded by its go flag and the screen flag it wrote.
__device__ __forceinline__ bool screen_off(const int* go, const int* sgo) {
  return (go && __ldg(go) == 0) || (sgo && __ldg(sgo) == 0);
}

__global__ void __launch_bounds__(kScanBlock) screen_flags_kernel(const __grid_constant__ Pack<ScreenJob> jobs, int W, double tol,
                                                                const int* __restrict__ go, const int* __restrict__ sgo) {
  pdl_enter();
  if (screen_off(go, sgo)) return;
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

// One block: warp q scans sensor q's block counts; the kept counts go to the
// mapped host array (the host reads them after the round's event, no copy).
// If no active set changes (nothing removed; a would-be-empty set stalls and
// stays), the already-enqueued next round may run: *go_next = 1.
__global__ void __launch_bounds__(256) screen_scan_kernel(const __grid_constant__ Pack<ScreenJob> jobs, int nq,
                                                          const int* __restrict__ go, const int* __restrict__ sgo,
                                                          int* totals_host, int* go_next) {
  pdl_enter();
  if (screen_off(go, sgo)) return;
  __shared__ int changed;
  if (threadIdx.x == 0) changed = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < nq; q += 8) {
    if (lane != 0) continue;
    const ScreenJob& jb = jobs.j[q];
    const int nb = (jb.n + kScanBlock - 1) / kScanBlock;
    int s = 0;
    for (int b = 0; b < nb; ++b) {
      jb.block_offsets[b] = s;
      s += jb.block_counts[b];
    }
    jb.totals[0] = s;
    if (totals_host) ((volatile int*)totals_host)[q] = s;
    if (s != jb.n && s != 0) atomicOr(&changed, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (go_next && !changed) *go_next = 1;
  }
}

__global__ void __launch_bounds__(kScanBlock) screen_scatter_kernel(const __grid_constant__ Pack<ScreenJob> jobs,
                                                                  const int* __restrict__ go, const int* __restrict__ sgo) {
  pdl_enter();
  if (screen_off(go, sgo)) return;
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

// The same screening in ONE launch: sensor q is one cluster of kScreenCluster
// CTAs (blockIdx.y = q); each CTA owns a contiguous range of `per` rounds of
// kScanBlock entries, keeps its flags in a register mask, scans its
// (round, warp) kept counts in shared memory and reads the other CTAs' kept
// totals through distributed shared memory for its output offset.  The last
// sensor to finish (arrival ticket) sets *go_next when no set changed.  Same
// outputs, same order as screen_flags / screen_scan / screen_scatter.
constexpr int kScreenCluster = 8;
constexpr int kScreenMaxE = 8;  // rounds per CTA: n <= 8 * 1024 * 8 = 65536

__device__ __forceinline__ int dsmem_ld_i32(const int* p, unsigned cta) {
  uint32_t ra;
  int v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(cta));
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
  return v;
}

__global__ void __cluster_dims__(kScreenCluster, 1, 1) __launch_bounds__(kScanBlock)
    screen_fused_kernel(const __grid_constant__ Pack<ScreenJob> jobs, int nq, int W, double tol,
                        const int* __restrict__ go, const int* __restrict__ sgo, int* totals_host, int* go_next,
                        unsigned* sync /* [0] arrival ticket, [1] changed; zero between launches */) {
  pdl_enter();
  if (screen_off(go, sgo)) return;
  const ScreenJob& jb = jobs.j[blockIdx.y];
  const unsigned rank = cluster_ctarank();
  const int n = jb.n;
  const int per = (n + kScreenCluster * kScanBlock - 1) / (kScreenCluster * kScanBlock);
  const int base = (int)rank * per * kScanBlock;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int cnt[kScreenMaxE * 32];  // kept count per (round, warp) -> exclusive offset in the CTA
  __shared__ int wsum[32];
  __shared__ int blk_total, blk_off, sensor_total;

  int pix[kScreenMaxE];
#pragma unroll
  for (int r = 0; r < kScreenMaxE; ++r) {
    const int i = base + r * kScanBlock + threadIdx.x;
    pix[r] = (r < per && i < n) ? __ldg(jb.J + i) : -1;
  }
  double z[kScreenMaxE];
#pragma unroll
  for (int r = 0; r < kScreenMaxE; ++r) {
    z[r] = 0.0;
    if (pix[r] >= 0)
      for (int t = 0; t < W; ++t) {
        const int slot = (jb.first_slot + t) % W;
        z[r] += __ldg(jb.ring + (int64_t)slot * jb.ring_stride + pix[r]);
      }
  }
  unsigned kmask = 0;
#pragma unroll
  for (int r = 0; r < kScreenMaxE; ++r) {
    if (r >= per) break;
    const bool k = pix[r] >= 0 && z[r] / (double)W >= tol;
    if (k) kmask |= 1u << r;
    const unsigned b = __ballot_sync(0xffffffffu, k);
    if (lane == 0) cnt[r * 32 + warp] = __popc(b);
  }
  __syncthreads();
  // exclusive scan of the per*32 counts, round-major (= index order)
  const int nv = per * 32;
  const int v = (int)threadIdx.x < nv ? cnt[threadIdx.x] : 0;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int w = wsum[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    wsum[lane] = wi - w;
    if (lane == 31) blk_total = wi;
  }
  __syncthreads();
  if ((int)threadIdx.x < nv) cnt[threadIdx.x] = inc - v + wsum[warp];
  cluster_sync_acqrel();  // every CTA's blk_total is written
  if (threadIdx.x == 0) {
    int off = 0, tot = 0;
    for (unsigned r = 0; r < (unsigned)kScreenCluster; ++r) {
      const int t = dsmem_ld_i32(&blk_total, r);
      if (r < rank) off += t;
      tot += t;
    }
    blk_off = off;
    sensor_total = tot;
  }
  cluster_sync_acqrel();  // no CTA leaves while its blk_total may still be read
  const int off = blk_off;
#pragma unroll
  for (int r = 0; r < kScreenMaxE; ++r) {
    if (r >= per) break;
    const bool k = (kmask >> r) & 1u;
    const unsigned b = __ballot_sync(0xffffffffu, k);
    if (pix[r] < 0) continue;
    const int i = base + r * kScanBlock + threadIdx.x;
    const int kept_before = off + cnt[r * 32 + warp] + __popc(b & ((1u << lane) - 1u));
    if (k) {
      jb.Jnew[kept_before] = pix[r];
      jb.keep_pos[kept_before] = i;
      jb.x_hat_new[kept_before] = jb.x_hat[i];  // x_full[J_new] (admm.hpp:153-156)
      jb.data_new[kept_before] = jb.data[i];
    } else {
      const int rpos = i - kept_before;
      jb.rem_pix[rpos] = pix[r];
      jb.rem_pos[rpos] = i;
    }
  }
  if (rank == 0 && threadIdx.x == 0) {
    const int s = sensor_total;
    jb.totals[0] = s;
    if (totals_host) ((volatile int*)totals_host)[blockIdx.y] = s;
    if (s != n && s != 0) atomicOr(sync + 1, 1u);
    __threadfence_system();
    if (atomicAdd(sync, 1u) == (unsigned)nq - 1) {
      const unsigned changed = atomicExch(sync + 1, 0u);
      atomicExch(sync, 0u);
      if (go_next && !changed) *go_next = 1;
    }
  }
}

}  // namespace radmm_dev
