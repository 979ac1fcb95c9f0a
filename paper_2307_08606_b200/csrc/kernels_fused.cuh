// kernels_fused.cuh: experimental single-pass sweeps v1-v5 (RADMM_FUSED)
// Part of kernels.cuh (see that file's header); included in order from there.
#pragma once

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
  pdl_enter();
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



template <int RPT>  // float4 row chunks per axpy thread: ld <= RPT * 256
__global__ void __launch_bounds__(kS2Threads, 1) fused_sweep2_kernel(const __grid_constant__ Pack<SweepJob> jobs,
                                                                     const __grid_constant__ FusionArgs fa, double mu,
                                                                     double beta, int range, int tile) {
  pdl_enter();
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
  pdl_enter();
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


__global__ void __launch_bounds__(kS4Threads, 1) fused_sweep4_kernel(const __grid_constant__ Pack<Sweep4Job> P,
                                                                     const __grid_constant__ FusionArgs fa,
                                                                     const __grid_constant__ Sweep4Ctl ctl,
                                                                     double mu, double beta, int64_t ld) {
  pdl_enter();
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
  pdl_enter();
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
