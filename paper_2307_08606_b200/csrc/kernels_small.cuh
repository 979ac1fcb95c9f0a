// kernels_small.cuh: one persistent cooperative launch per ASADMM iteration
// for problems whose operators, factors and state sit in L2 (BASELINE config
// 1: 4 x 256 x 1024, 18.9 MB).  Part of kernels.cuh.
//
// At these sizes every phase is a few microseconds of work and the ~16
// separate launches of the general path cost more than the work itself
// (config 1: 95.7 us per iteration).  Here the whole local update + fusion
// round of SensorCore::local_update / FusionCore::round (admm.hpp:111-126,
// 236-258) runs in one grid of resident CTAs, separated by grid-wide
// barriers (cooperative launch):
//   rhs -> forward partials -> v -> u = G v [-> lazy terms] [-> refinement:
//   rho = v - C w (+ mu A_D A_D^H w), dw = G rho (+ lazy), w += dw]
//   -> x-update (adjoint / primal Hinv) + scatter + ring -> fusion round.
// Work is split over (sensor, row block / column chunk / column) items with
// fixed per-item summation orders, so the result is deterministic run to
// run.  Screening stays in its own (guarded) launch behind it.
#pragma once
#include <cooperative_groups.h>

namespace radmm_dev {

constexpr int kSmallThreads = 256;
constexpr int kSmallMaxRows = 1024;  // rows staged in shared memory (dual sensors)
constexpr int kSmallChunk = 64;      // forward columns per item

struct SmallJob {
  int primal;                 // 1: x = Hinv rhs (G is Hinv, n_act x n_act)
  const float2* A;
  int64_t ld;
  int rows, n_act;
  const int* J;
  const double2* data;
  double2* x_hat;
  double2* rhs;
  double2* x_full;
  double* ring_slot;
  double2* v;
  double2* w;
  double2* rho;
  double2* dw;
  double2* part;              // [nchunk][ld] forward partials
  int nchunk;
  const double2* bz;          // lagged data term: v += beta z (nullptr: none)
  const double2* G;           // full column-major (ldg)
  int64_t ldg;
  const double2* Cp;          // packed capacitance (refinement) or nullptr
  int d;                      // lazy columns
  const int* pix;
  const double2* P;           // ld x d
  const double2* Sinv;        // d x d (lds)
  int64_t lds;
  double2* t;                 // 3 x kLazyMax scratch: A_D^H u, A_D^H w, A_D^H dw
};

struct SmallArgs {
  Pack<SmallJob> jobs;        // only the first Q entries are read
  int Q;
  int any_lazy, any_refine, any_dual;
  double mu, beta;
  const int* go;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// element (r, k) of a Hermitian matrix stored as packed lower tiles
__device__ __forceinline__ double2 packed_at(const double2* Cp, int r, int k) {
  const int I = r >> 6, K = k >> 6;
  if (I >= K) return Cp[herm_packed_tile(I, K) + (r & 63) + (k & 63) * kHermTile];
  const double2 v = Cp[herm_packed_tile(K, I) + (k & 63) + (r & 63) * kHermTile];
  return make_double2(v.x, -v.y);
}

// out[r] = (base ? base[r] : 0) + M vec over the rows of sensor jobs, one
// thread per row, vec staged in shared memory; packed: Hermitian packed tiles.
// Items are (sensor, block of kSmallThreads rows), grid-strided.
__device__ __forceinline__ void small_matvec(const SmallArgs& a, int which, double2* svec) {
  // which: 0 u = G v (w), 1 rho = v - C w, 2 dw = G rho
  int items = 0;
  for (int q = 0; q < a.Q; ++q)
    if (!a.jobs.j[q].primal) items += (a.jobs.j[q].rows + kSmallThreads - 1) / kSmallThreads;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int q = 0, rest = it;
    for (; q < a.Q; ++q) {
      const SmallJob& jb = a.jobs.j[q];
      if (jb.primal) continue;
      const int nb = (jb.rows + kSmallThreads - 1) / kSmallThreads;
      if (rest < nb) break;
      rest -= nb;
    }
    const SmallJob& jb = a.jobs.j[q];
    if (which == 1 && !jb.Cp) continue;
    const double2* src = which == 0 ? jb.v : which == 1 ? jb.w : jb.rho;
    __syncthreads();
    for (int k = threadIdx.x; k < jb.rows; k += blockDim.x) {
      double2 x = src[k];
      if (which == 2 && jb.d > 0) {  // rho += mu A_D (A_D^H w), the lazy part of the residual
        double re = 0.0, im = 0.0;
        for (int j = 0; j < jb.d; ++j) {
          const float2 av = jb.A[k + (int64_t)jb.pix[j] * jb.ld];
          const double2 t = jb.t[kLazyMax + j];
          re = fma((double)av.x, t.x, re);
          re = fma(-(double)av.y, t.y, re);
          im = fma((double)av.x, t.y, im);
          im = fma((double)av.y, t.x, im);
        }
        x.x += a.mu * re;
        x.y += a.mu * im;
      }
      svec[k] = x;
    }
    __syncthreads();
    const int r = rest * kSmallThreads + threadIdx.x;
    if (r >= jb.rows) continue;
    double re = 0.0, im = 0.0;
    if (which == 1) {
      for (int k = 0; k < jb.rows; ++k) {
        const double2 m = packed_at(jb.Cp, r, k), x = svec[k];
        re = fma(m.x, x.x, re);
        re = fma(-m.y, x.y, re);
        im = fma(m.x, x.y, im);
        im = fma(m.y, x.x, im);
      }
      const double2 vv = jb.v[r];
      jb.rho[r] = make_double2(vv.x - re, vv.y - im);
    } else {
      const double2* Gc = jb.G + r;
      for (int k = 0; k < jb.rows; ++k) {
        const double2 m = Gc[(int64_t)k * jb.ldg], x = svec[k];
        re = fma(m.x, x.x, re);
        re = fma(-m.y, x.y, re);
        im = fma(m.x, x.y, im);
        im = fma(m.y, x.x, im);
      }
      (which == 0 ? jb.w : jb.dw)[r] = make_double2(re, im);
    }
  }
}

// t[slot][j] = A_D^H vec (one warp per (sensor, lazy column))
__device__ __forceinline__ void small_lazy_dots(const SmallArgs& a, int slot) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int items = 0;
  for (int q = 0; q < a.Q; ++q) items += a.jobs.j[q].primal ? 0 : a.jobs.j[q].d;
  for (int it = warp; it < items; it += nwarps) {
    int q = 0, rest = it;
    for (; q < a.Q; ++q) {
      const int d = a.jobs.j[q].primal ? 0 : a.jobs.j[q].d;
      if (rest < d) break;
      rest -= d;
    }
    const SmallJob& jb = a.jobs.j[q];
    const double2* vec = slot == 0 ? jb.w : slot == 1 ? jb.w : jb.dw;
    const float2* col = jb.A + (int64_t)jb.pix[rest] * jb.ld;
    double re = 0.0, im = 0.0;
    for (int r = lane; r < jb.rows; r += 32) {
      const float2 av = col[r];
      const double2 x = vec[r];
      re = fma((double)av.x, x.x, re);
      re = fma((double)av.y, x.y, re);
      im = fma((double)av.x, x.y, im);
      im = fma(-(double)av.y, x.x, im);
    }
    re = warp_sum(re);
    im = warp_sum(im);
    if (lane == 0) jb.t[slot * kLazyMax + rest] = make_double2(re, im);
  }
}

// out[r] += P (mu Sinv t[slot]) for the lazy sensors; s = mu Sinv t staged per item
__device__ __forceinline__ void small_lazy_axpy(const SmallArgs& a, int slot, bool on_dw, double2* ss) {
  int items = 0;
  for (int q = 0; q < a.Q; ++q)
    if (!a.jobs.j[q].primal && a.jobs.j[q].d > 0) items += (a.jobs.j[q].rows + kSmallThreads - 1) / kSmallThreads;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int q = 0, rest = it;
    for (; q < a.Q; ++q) {
      const SmallJob& jb = a.jobs.j[q];
      if (jb.primal || jb.d == 0) continue;
      const int nb = (jb.rows + kSmallThreads - 1) / kSmallThreads;
      if (rest < nb) break;
      rest -= nb;
    }
    const SmallJob& jb = a.jobs.j[q];
    __syncthreads();
    if (threadIdx.x < jb.d) {  // s_j = mu sum_k Sinv[j, k] t_k (fixed order)
      const int j = threadIdx.x;
      double re = 0.0, im = 0.0;
      for (int k = 0; k < jb.d; ++k) {
        const double2 m = jb.Sinv[j + (int64_t)k * jb.lds], x = jb.t[slot * kLazyMax + k];
        re = fma(m.x, x.x, re);
        re = fma(-m.y, x.y, re);
        im = fma(m.x, x.y, im);
        im = fma(m.y, x.x, im);
      }
      ss[j] = make_double2(a.mu * re, a.mu * im);
    }
    __syncthreads();
    const int r = rest * kSmallThreads + threadIdx.x;
    if (r >= jb.rows) continue;
    double re = 0.0, im = 0.0;
    for (int k = 0; k < jb.d; ++k) {
      const double2 p = jb.P[r + (int64_t)k * jb.ld], x = ss[k];
      re = fma(p.x, x.x, re);
      re = fma(-p.y, x.y, re);
      im = fma(p.x, x.y, im);
      im = fma(p.y, x.x, im);
    }
    double2* out = on_dw ? jb.dw : jb.w;
    const double2 u = out[r];
    out[r] = make_double2(u.x + re, u.y + im);
  }
}

__global__ void __launch_bounds__(kSmallThreads) small_iter_kernel(const __grid_constant__ SmallArgs a,
                                                                   FusionArgs f) {
  namespace cg = cooperative_groups;
  if (a.go && __ldg(a.go) == 0) return;  // cancelled speculative iteration (uniform over the grid)
  cg::grid_group grid = cg::this_grid();
  __shared__ double2 svec[kSmallMaxRows];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gsize = gridDim.x * blockDim.x;
  const double beta = a.beta, mu = a.mu;
  // 1. rhs = data + beta gap[J] + beta x_hat - sigma[J] (admm.hpp:114-119)
  {
    for (int q = 0; q < a.Q; ++q) {
      const SmallJob& jb = a.jobs.j[q];
      for (int i = gtid; i < jb.n_act; i += gsize) {
        const int c = jb.J[i];
        const double2 d = jb.data[i], g = f.gap[c], xh = jb.x_hat[i], sg = f.sigma[c];
        double2 v;
        v.x = __dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, xh.x)), sg.x);
        v.y = __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, xh.y)), sg.y);
        jb.rhs[i] = v;
      }
    }
  }
  grid.sync();
  if (a.any_dual) {
    // 2. forward partials: item = (sensor, chunk of kSmallChunk columns)
    int items = 0;
    for (int q = 0; q < a.Q; ++q) items += a.jobs.j[q].primal ? 0 : a.jobs.j[q].nchunk;
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
      int q = 0, rest = it;
      for (; q < a.Q; ++q) {
        const int nc = a.jobs.j[q].primal ? 0 : a.jobs.j[q].nchunk;
        if (rest < nc) break;
        rest -= nc;
      }
      const SmallJob& jb = a.jobs.j[q];
      const int i0 = rest * kSmallChunk, i1 = min(jb.n_act, i0 + kSmallChunk);
      for (int r = threadIdx.x; r < jb.rows; r += blockDim.x) {
        double re = 0.0, im = 0.0;
        for (int i = i0; i < i1; ++i) {
          const float2 av = jb.A[r + (int64_t)jb.J[i] * jb.ld];
          const double2 x = jb.rhs[i];
          re = fma((double)av.x, x.x, re);
          re = fma(-(double)av.y, x.y, re);
          im = fma((double)av.x, x.y, im);
          im = fma((double)av.y, x.x, im);
        }
        jb.part[(int64_t)rest * jb.ld + r] = make_double2(re, im);
      }
    }
    grid.sync();
    // 3. v = beta z + sum of the partials (chunk order)
    for (int q = 0; q < a.Q; ++q) {
      const SmallJob& jb = a.jobs.j[q];
      if (jb.primal) continue;
      for (int r = gtid; r < jb.rows; r += gsize) {
        double2 s = jb.bz ? jb.bz[r] : make_double2(0.0, 0.0);
        for (int cch = 0; cch < jb.nchunk; ++cch) {
          const double2 p = jb.part[(int64_t)cch * jb.ld + r];
          s.x += p.x;
          s.y += p.y;
        }
        jb.v[r] = s;
      }
    }
    grid.sync();
    // 4. u = G v, then the lazy terms: w = u + mu P Sinv (A_D^H u)
    small_matvec(a, 0, svec);
    grid.sync();
    if (a.any_lazy) {
      small_lazy_dots(a, 0);
      grid.sync();
      small_lazy_axpy(a, 0, false, svec);
      grid.sync();
    }
    if (a.any_refine) {
      // 5. refinement: rho = v - C w (+ mu A_D A_D^H w, folded into the next stage's staging)
      if (a.any_lazy) small_lazy_dots(a, 1);
      small_matvec(a, 1, svec);
      grid.sync();
      small_matvec(a, 2, svec);  // dw = G rho (rho staged with its lazy part)
      grid.sync();
      if (a.any_lazy) {
        small_lazy_dots(a, 2);
        grid.sync();
        small_lazy_axpy(a, 2, true, svec);
        grid.sync();
      }
      for (int q = 0; q < a.Q; ++q) {
        const SmallJob& jb = a.jobs.j[q];
        if (jb.primal || !jb.Cp) continue;
        for (int r = gtid; r < jb.rows; r += gsize) {
          const double2 x = jb.w[r], y = jb.dw[r];
          jb.w[r] = make_double2(x.x + y.x, x.y + y.y);
        }
      }
      grid.sync();
    }
  }
  // 6. x-update: dual x = (rhs - mu A_J^H w)/beta (warp per column), primal
  //    x = Hinv rhs (thread per row); scatter into x_full and the screening ring
  {
    const int warp = gtid >> 5, lane = threadIdx.x & 31, nwarps = gsize >> 5;
    int items = 0;
    for (int q = 0; q < a.Q; ++q) items += a.jobs.j[q].primal ? 0 : a.jobs.j[q].n_act;
    for (int it = warp; it < items; it += nwarps) {
      int q = 0, rest = it;
      for (; q < a.Q; ++q) {
        const int n = a.jobs.j[q].primal ? 0 : a.jobs.j[q].n_act;
        if (rest < n) break;
        rest -= n;
      }
      const SmallJob& jb = a.jobs.j[q];
      const int p = jb.J[rest];
      const float2* col = jb.A + (int64_t)p * jb.ld;
      double re = 0.0, im = 0.0;
      for (int r = lane; r < jb.rows; r += 32) {
        const float2 av = col[r];
        const double2 x = jb.w[r];
        re = fma((double)av.x, x.x, re);
        re = fma((double)av.y, x.y, re);
        im = fma((double)av.x, x.y, im);
        im = fma(-(double)av.y, x.x, im);
      }
      re = warp_sum(re);
      im = warp_sum(im);
      if (lane == 0) {
        const double2 rr = jb.rhs[rest];
        const double2 xh = make_double2(__ddiv_rn(__dsub_rn(rr.x, __dmul_rn(mu, re)), beta),
                                        __ddiv_rn(__dsub_rn(rr.y, __dmul_rn(mu, im)), beta));
        const double2 old = jb.x_full[p];
        jb.ring_slot[p] = c_abs(c_sub(xh, old));
        jb.x_full[p] = xh;
        jb.x_hat[rest] = xh;
      }
    }
    for (int q = 0; q < a.Q; ++q) {
      const SmallJob& jb = a.jobs.j[q];
      if (!jb.primal) continue;
      for (int i = gtid; i < jb.n_act; i += gsize) {
        double re = 0.0, im = 0.0;
        for (int k = 0; k < jb.n_act; ++k) {
          const double2 m = jb.G[i + (int64_t)k * jb.ldg], x = jb.rhs[k];
          re = fma(m.x, x.x, re);
          re = fma(-m.y, x.y, re);
          im = fma(m.x, x.y, im);
          im = fma(m.y, x.x, im);
        }
        const double2 xh = make_double2(re, im);
        const int p = jb.J[i];
        const double2 old = jb.x_full[p];
        jb.ring_slot[p] = c_abs(c_sub(xh, old));
        jb.x_full[p] = xh;
        jb.x_hat[i] = xh;
      }
    }
  }
  grid.sync();
  // 7. FusionCore::round over all pixels (fusion_pixel / fusion_finish of the
  //    general path: the same per-pixel arithmetic and deterministic reduction)
  double qn[5] = {0, 0, 0, 0, 0};
  for (int j = gtid; j < f.N; j += gsize) fusion_pixel(f, j, [&](int k) { return f.contrib[k][j]; }, qn);
  fusion_finish(f, qn, gridDim.x, blockIdx.x);
}

}  // namespace radmm_dev
