// kernels_batched.cuh: Hermitian G-apply and projection, back-projection, frame-batched DMMA contractions, tensor-core Gram
// Part of kernels.cuh (see that file's header); included in order from there.
#pragma once

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
  const double2* v;  // right-hand side 0 (nullptr: the job sits this launch out)
  double2* w;
  const double2* v1; // right-hand side 1 (NR >= 2 launches; nullptr: none)
  double2* w1;
  const double2* v2; // right-hand sides 2, 3 (NR = 4 launches: an event's 2-3 removed columns
  double2* w2;       // ride the iteration's own pass over G; nullptr: none)
  const double2* v3;
  double2* w3;
  double2* dotp;     // [NR][nb][groups][64], column stride dstride
  double2* axp;      // [NR][nb (nb - 1) / 2][64], slot I (I - 1) / 2 + J, column stride astride
  int64_t dstride, astride;
  int packed;          // G is a packed lower-tile array (cap_pack_kernel), not column-major ld
  const float2* G32;   // packed complex64 copy of G read instead of G (refinement's correction pass)
  const double2* base; // right-hand side 0 output: w = base + sgn * (G v) (nullptr: w = G v)
  double sgn;
};

// Packed lower-tile storage of a Hermitian matrix (the dual capacitance C,
// kept next to its explicit inverse for the KM-space refinement): tile (I, J),
// I >= J, at tile slot I (I + 1) / 2 + J, 64 x 64 column-major (ld 64),
// zero-padded past n.  Only the lower triangle is stored.
__host__ __device__ inline int64_t herm_packed_tile(int I, int J) {
  return ((int64_t)I * (I + 1) / 2 + J) * (int64_t)(kHermTile * kHermTile);
}

// item word: q (16) | J (16) | I0 (16) | nt (16)
__host__ __device__ inline uint64_t herm_item(int q, int J, int I0, int nt) {
  return (uint64_t)q << 48 | (uint64_t)J << 32 | (uint64_t)I0 << 16 | (uint64_t)nt;
}

#if RADMM_EXPERIMENTAL  // one CTA per item (superseded by the persistent kernel below)
// NR right-hand sides per pass of G: NR = 1 is the iteration's w = G v; NR = 2
// also forms a lazy-downdate column P[:, u] = G a_u from the same tile reads
// (see lazy_* below).  A missing second column (v1 == nullptr) is zero.
template <int NR>
__global__ void __launch_bounds__(256) herm_gapply_kernel(const __grid_constant__ Pack<HermJob> P,
                                                         const uint64_t* __restrict__ items,
                                                         const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  const uint64_t it = items[blockIdx.x];
  const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF), I0 = (int)(it >> 16 & 0xFFFF), nt = (int)(it & 0xFFFF);
  const HermJob& jb = P.j[q];
  if (!jb.v) return;
  __shared__ double2 vJ[NR][kHermTile];
  __shared__ double2 vI[NR][kHermStrip * kHermTile];
  __shared__ double2 sax[2][NR][8][kHermTile];  // double-buffered: one barrier per tile
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = jb.n;
  const double2* vs[2] = {jb.v, jb.v1};
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    const double2* vc = vs[c];
    if (tid < kHermTile) {
      const int j = J * kHermTile + tid;
      vJ[c][tid] = (vc && j < n) ? vc[j] : make_double2(0.0, 0.0);
    }
    for (int t = tid; t < nt * kHermTile; t += 256) {
      const int i = I0 * kHermTile + t;
      vI[c][t] = (vc && i < n) ? vc[i] : make_double2(0.0, 0.0);
    }
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
  double dr[NR][8], di[NR][8];
#pragma unroll
  for (int c = 0; c < NR; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) dr[c][k] = di[c][k] = 0.0;
  int par = 0;
  for (int t = 0; t < nt; ++t) {
    const int I = I0 + t;
    double ar[NR][2], ai[NR][2];
#pragma unroll
    for (int c = 0; c < NR; ++c) ar[c][0] = ar[c][1] = ai[c][0] = ai[c][1] = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        const double2 vi = vI[c][t * kHermTile + lane + 32 * h];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // conj(g) * v_i
          dr[c][k] = fma(g[k][h].x, vi.x, dr[c][k]);
          dr[c][k] = fma(g[k][h].y, vi.y, dr[c][k]);
          di[c][k] = fma(g[k][h].x, vi.y, di[c][k]);
          di[c][k] = fma(-g[k][h].y, vi.x, di[c][k]);
          // g * v_j
          const double2 vj = vJ[c][c0 + k];
          ar[c][h] = fma(g[k][h].x, vj.x, ar[c][h]);
          ar[c][h] = fma(-g[k][h].y, vj.y, ar[c][h]);
          ai[c][h] = fma(g[k][h].x, vj.y, ai[c][h]);
          ai[c][h] = fma(g[k][h].y, vj.x, ai[c][h]);
        }
      }
    }
    if (t + 1 < nt) load_tile(I + 1);  // in flight across the reduction below
    if (I != J) {  // strictly-lower tile: its mirror contributes to rows of block I
#pragma unroll
      for (int c = 0; c < NR; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) sax[par][c][warp][lane + 32 * h] = make_double2(ar[c][h], ai[c][h]);
      __syncthreads();
      if (tid < NR * kHermTile) {
        const int c = tid / kHermTile, r = tid % kHermTile;
        double2 sum = sax[par][c][0][r];
#pragma unroll
        for (int w8 = 1; w8 < 8; ++w8) {
          sum.x += sax[par][c][w8][r].x;
          sum.y += sax[par][c][w8][r].y;
        }
        jb.axp[c * jb.astride + ((int64_t)I * (I - 1) / 2 + J) * kHermTile + r] = sum;
      }
      par ^= 1;  // the other buffer's readers are past this barrier
    }
  }
#pragma unroll
  for (int c = 0; c < NR; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dr[c][k] = warp_sum(dr[c][k]);
      di[c][k] = warp_sum(di[c][k]);
    }
  if (lane == 0) {
    const int gi = (I0 - J) / kHermStrip;
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      double2* dp = jb.dotp + c * jb.dstride + ((int64_t)J * jb.groups + gi) * kHermTile + c0;
#pragma unroll
      for (int k = 0; k < 8; ++k) dp[k] = make_double2(dr[c][k], di[c][k]);
    }
  }
}

#endif

constexpr size_t herm_persist_smem(int nr) {
  return (size_t)(2 * nr * kHermTile + 2 * nr * kHermStrip * kHermTile + kHermStrip * nr * 8 * kHermTile) * 16;
}

// Persistent variant: a fixed grid (resident CTAs) walks the item list
// round-robin; while the last tile of one item is reduced, the first tile of
// the CTA's next item and that item's vector slices are already loading
// (registers and a second shared buffer), so items cost no start-up latency.
// Per-item arithmetic and partial slots are exactly herm_gapply_kernel's.
template <int NR>
__global__ void __launch_bounds__(256, NR <= 2 ? 2 : 1) herm_gapply_persist_kernel(const __grid_constant__ Pack<HermJob> P,
                                                                    const uint64_t* __restrict__ items, int n_items,
                                                                    const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration
  extern __shared__ __align__(16) double2 hps[];  // herm_persist_smem(NR) bytes
  double2(*vJ)[NR][kHermTile] = reinterpret_cast<double2(*)[NR][kHermTile]>(hps);
  double2(*vI)[NR][kHermStrip * kHermTile] =
      reinterpret_cast<double2(*)[NR][kHermStrip * kHermTile]>(hps + 2 * NR * kHermTile);
  // per-warp axpy partials of every tile of the strip: summed once at the end
  // of the item (one barrier per item instead of one per tile)
  double2(*sax)[NR][8][kHermTile] =
      reinterpret_cast<double2(*)[NR][8][kHermTile]>(hps + 2 * NR * kHermTile + 2 * NR * kHermStrip * kHermTile);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = warp * 8;
  // next active item at or after index i (inactive jobs have v == nullptr)
  auto next_item = [&](int i) {
    for (; i < n_items; i += gridDim.x) {
      const uint64_t it = __ldg(items + i);
      if (P.j[(int)(it >> 48)].v) return i;
    }
    return n_items;
  };
  auto load_vec = [&](int buf, uint64_t it) {
    const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF), I0 = (int)(it >> 16 & 0xFFFF), nt = (int)(it & 0xFFFF);
    const HermJob& jb = P.j[q];
    const double2* vs[4] = {jb.v, jb.v1, jb.v2, jb.v3};
#pragma unroll
    for (int c = 0; c < NR; ++c) {
      const double2* vc = vs[c];
      if (tid < kHermTile) {
        const int j = J * kHermTile + tid;
        vJ[buf][c][tid] = (vc && j < jb.n) ? vc[j] : make_double2(0.0, 0.0);
      }
      for (int t = tid; t < nt * kHermTile; t += 256) {
        const int i = I0 * kHermTile + t;
        vI[buf][c][t] = (vc && i < jb.n) ? vc[i] : make_double2(0.0, 0.0);
      }
    }
  };
  double2 g[8][2];
  auto load_tile = [&](uint64_t it, int I) {
    const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF);
    const HermJob& jb = P.j[q];
    const int ib = I * kHermTile;
    if (jb.packed) {  // tile-contiguous: 64 KB per tile (32 KB in complex64), zero-padded
      if (jb.G32) {
        const float2* Gt = jb.G32 + herm_packed_tile(I, J) + (int64_t)c0 * kHermTile;
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 x = __ldg(Gt + k * kHermTile + lane + 32 * h);
            g[k][h] = make_double2(x.x, x.y);
          }
        return;
      }
      const double2* Gt = jb.G + herm_packed_tile(I, J) + (int64_t)c0 * kHermTile;
#pragma unroll
      for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) g[k][h] = __ldg(Gt + k * kHermTile + lane + 32 * h);
      return;
    }
    const double2* Gc = jb.G + (int64_t)(J * kHermTile + c0) * jb.ld;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = ib + lane + 32 * h, j = J * kHermTile + c0 + k;
        g[k][h] = (i < jb.n && j < jb.n) ? __ldg(Gc + (int64_t)k * jb.ld + i) : make_double2(0.0, 0.0);
      }
  };
  int cur = next_item(blockIdx.x);
  if (cur >= n_items) return;
  uint64_t it = __ldg(items + cur);
  int buf = 0;
  load_vec(buf, it);
  load_tile(it, (int)(it >> 16 & 0xFFFF));
  while (true) {
    const int q = (int)(it >> 48), J = (int)(it >> 32 & 0xFFFF), I0 = (int)(it >> 16 & 0xFFFF), nt = (int)(it & 0xFFFF);
    const HermJob& jb = P.j[q];
    // right-hand sides beyond the first are optional per job (absent: skipped)
    const bool has[4] = {true, NR > 1 && jb.v1 != nullptr, NR > 2 && jb.v2 != nullptr, NR > 3 && jb.v3 != nullptr};
    const int nxt = next_item(cur + gridDim.x);
    const uint64_t it_n = nxt < n_items ? __ldg(items + nxt) : 0;
    __syncthreads();  // vectors of `buf` visible; the other buffer's readers are done
    if (nxt < n_items) load_vec(buf ^ 1, it_n);
    double dr[NR][8], di[NR][8];
#pragma unroll
    for (int c = 0; c < NR; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) dr[c][k] = di[c][k] = 0.0;
    for (int t = 0; t < nt; ++t) {
      const int I = I0 + t;
      double ar[NR][2], ai[NR][2];
#pragma unroll
      for (int c = 0; c < NR; ++c) ar[c][0] = ar[c][1] = ai[c][0] = ai[c][1] = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int c = 0; c < NR; ++c) {
          if (!has[c]) continue;
          const double2 vi = vI[buf][c][t * kHermTile + lane + 32 * h];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            dr[c][k] = fma(g[k][h].x, vi.x, dr[c][k]);
            dr[c][k] = fma(g[k][h].y, vi.y, dr[c][k]);
            di[c][k] = fma(g[k][h].x, vi.y, di[c][k]);
            di[c][k] = fma(-g[k][h].y, vi.x, di[c][k]);
            const double2 vj = vJ[buf][c][c0 + k];
            ar[c][h] = fma(g[k][h].x, vj.x, ar[c][h]);
            ar[c][h] = fma(-g[k][h].y, vj.y, ar[c][h]);
            ai[c][h] = fma(g[k][h].x, vj.y, ai[c][h]);
            ai[c][h] = fma(g[k][h].y, vj.x, ai[c][h]);
          }
        }
      }
      if (t + 1 < nt) load_tile(it, I + 1);                       // in flight across the work below
      else if (nxt < n_items) load_tile(it_n, (int)(it_n >> 16 & 0xFFFF));  // the next item's first tile
      if (I != J) {
#pragma unroll
        for (int c = 0; c < NR; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h) sax[t][c][warp][lane + 32 * h] = make_double2(ar[c][h], ai[c][h]);
      }
    }
    __syncthreads();  // every warp's axpy partials of the strip are in shared memory
    {
      for (int e = tid; e < nt * NR * kHermTile; e += 256) {
        const int t = e / (NR * kHermTile), c = (e / kHermTile) % NR, r = e % kHermTile;
        const int I = I0 + t;
        if (I == J || !has[c]) continue;
        double2 sum = sax[t][c][0][r];
#pragma unroll
        for (int w8 = 1; w8 < 8; ++w8) {
          sum.x += sax[t][c][w8][r].x;
          sum.y += sax[t][c][w8][r].y;
        }
        jb.axp[c * jb.astride + ((int64_t)I * (I - 1) / 2 + J) * kHermTile + r] = sum;
      }
    }
#pragma unroll
    for (int c = 0; c < NR; ++c)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        dr[c][k] = warp_sum(dr[c][k]);
        di[c][k] = warp_sum(di[c][k]);
      }
    if (lane == 0) {
      const int gi = (I0 - J) / kHermStrip;
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        if (!has[c]) continue;
        double2* dp = jb.dotp + c * jb.dstride + ((int64_t)J * jb.groups + gi) * kHermTile + c0;
#pragma unroll
        for (int k = 0; k < 8; ++k) dp[k] = make_double2(dr[c][k], di[c][k]);
      }
    }
    if (nxt >= n_items) break;
    cur = nxt;
    it = it_n;
    buf ^= 1;
  }
}

// w[b*64 + r] = sum_g dotp[b][g][r] + sum_{J < b} axp[tri(b, J)][r]  (fixed order)
// 256 threads per row block: slice s = tid / 64 sums the partials k = s, s+4, ...
// of the row's list (4 independent loads in flight), then the 4 slice sums are
// added in slice order -- deterministic.  blockIdx.z = right-hand side.
constexpr int kHermRedSlices = 8;  // 512 threads: 8 slices x 64 rows, 4 loads in flight each

__global__ void __launch_bounds__(kHermRedSlices * kHermTile) herm_reduce_kernel(const __grid_constant__ Pack<HermJob> P,
                                                                                const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;
  const HermJob& jb = P.j[blockIdx.y];
  const int c = blockIdx.z;
  double2* const out = c == 0 ? jb.w : c == 1 ? jb.w1 : c == 2 ? jb.w2 : jb.w3;
  const double2* const vin = c == 0 ? jb.v : c == 1 ? jb.v1 : c == 2 ? jb.v2 : jb.v3;
  if (!jb.v || !out || !vin) return;
  const int b = blockIdx.x, r = threadIdx.x & 63, sl = threadIdx.x >> 6;
  __shared__ double2 part[kHermRedSlices][kHermTile];
  if (b >= jb.nb) return;
  const int ng = (jb.nb - b + kHermStrip - 1) / kHermStrip;
  const int total = ng + b;  // dot partials, then ax partials J = 0 .. b-1
  const double2* dbase = jb.dotp + c * jb.dstride + (int64_t)b * jb.groups * kHermTile + r;
  const double2* abase = jb.axp + c * jb.astride + (int64_t)b * (b - 1) / 2 * kHermTile + r;
  double2 s = make_double2(0.0, 0.0);
  for (int k0 = sl; k0 < total; k0 += 4 * kHermRedSlices) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + kHermRedSlices * u;
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
    for (int u = 1; u < kHermRedSlices; ++u) {
      t.x += part[u][r].x;
      t.y += part[u][r].y;
    }
    if (row < jb.n) {
      if (c == 0 && jb.base) {  // refinement: residual v - C w, or correction w + G rho
        const double2 b = jb.base[row];
        t = make_double2(b.x + jb.sgn * t.x, b.y + jb.sgn * t.y);
      }
      out[row] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Lazy Woodbury downdates (dual form).  After columns D (pixels pix[0..d)) are
// eliminated, the capacitance becomes C_D = C - mu A_D A_D^H; with the factor
// G = C^{-1} of the base set kept unchanged,
//   C_D^{-1} v = u + mu P Sinv (A_D^H u),   u = G v,  P = G A_D,
//   Sinv = (I - mu A_D^H P)^{-1}  (d x d),
// so an elimination event appends columns to P (one pass of G, shared with
// the iteration's own G-apply) instead of rewriting G.
//   lazy_dot_kernel:   t = A_D^H u            grid (d, jobs)
//   lazy_axpy_kernel:  w = u + mu P (Sinv t)  grid (row blocks, jobs)
// ---------------------------------------------------------------------------
constexpr int kLazyMax = 64;  // accumulated columns before they are folded into G

struct LazyJob {
  const float2* A;      // operator (complex64, column-major, ld)
  int64_t ld;
  int rows;
  const int* pix;       // D: eliminated pixels (operator columns)
  int d;
  const double2* P;     // ld x d
  const double2* Sinv;  // d x d, leading dimension lds
  int64_t lds;
  double2* w;           // in: u = G v; out: C_D^{-1} v
  double2* t;           // d (scratch): t = A_D^H u, then s = mu Sinv t in t + kLazyMax
  unsigned* cnt;        // arrival counter of the job's dot blocks (zero between launches)
  int ident;            // refinement residual: s = mu t (no Sinv), then dst += A_D s
  double2* dst;         //   (lazy_resid_axpy_kernel; w is only read)
  double2* sum_into;    // correction pass: sum_into += w + mu P s instead of w += mu P s (w untouched);
                        //   folds the refinement's final w = w1 + dw into the lazy term of dw
};

// s = mu Sinv t for one job by one block: four threads per row of Sinv,
// fixed-order shuffle combine (deterministic)
__device__ __forceinline__ void lazy_s(const LazyJob& jb, double mu, const double2* t, double2* s) {
  const int j = threadIdx.x >> 2, sub = threadIdx.x & 3;
  double re = 0.0, im = 0.0;
  if (j < jb.d)
    for (int k = sub; k < jb.d; k += 4) {
      const double2 m = jb.Sinv[j + (int64_t)k * jb.lds], x = t[k];
      re = fma(m.x, x.x, re);
      re = fma(-m.y, x.y, re);
      im = fma(m.x, x.y, im);
      im = fma(m.y, x.x, im);
    }
  re += __shfl_xor_sync(0xffffffffu, re, 1);
  im += __shfl_xor_sync(0xffffffffu, im, 1);
  re += __shfl_xor_sync(0xffffffffu, re, 2);
  im += __shfl_xor_sync(0xffffffffu, im, 2);
  if (sub == 0 && j < jb.d) s[j] = make_double2(mu * re, mu * im);
}

// t = A_D^H u (one block per column); the job's last block to finish also
// forms s = mu Sinv t (lazy_s), so lazy_axpy_kernel only streams P.
__global__ void __launch_bounds__(256) lazy_dot_kernel(const __grid_constant__ Pack<LazyJob> P, double mu,
                                                       const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;
  const LazyJob& jb = P.j[blockIdx.y];
  const int j = blockIdx.x;
  if (j >= jb.d) return;
  const float2* a = jb.A + (int64_t)jb.pix[j] * jb.ld;
  double re = 0.0, im = 0.0;
#pragma unroll 4
  for (int i = threadIdx.x; i < jb.rows; i += 256) {
    const float2 x = a[i];
    const double2 u = jb.w[i];
    // conj(a) * u
    re = fma((double)x.x, u.x, re);
    re = fma((double)x.y, u.y, re);
    im = fma((double)x.x, u.y, im);
    im = fma(-(double)x.y, u.x, im);
  }
  __shared__ double sr[8], si[8];
  re = warp_sum(re);
  im = warp_sum(im);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sr[warp] = re; si[warp] = im; }
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    double a0 = sr[0], b0 = si[0];
    for (int k = 1; k < 8; ++k) { a0 += sr[k]; b0 += si[k]; }
    jb.t[j] = make_double2(a0, b0);
    __threadfence();
    last = atomicAdd(jb.cnt, 1u) == (unsigned)jb.d - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double2 ts[kLazyMax];
  if (threadIdx.x < jb.d) {
    const volatile double* tv = reinterpret_cast<volatile double*>(jb.t) + 2 * threadIdx.x;
    ts[threadIdx.x] = make_double2(tv[0], tv[1]);
  }
  __syncthreads();
  if (jb.ident) {
    if (threadIdx.x < jb.d) jb.t[kLazyMax + threadIdx.x] = make_double2(mu * ts[threadIdx.x].x, mu * ts[threadIdx.x].y);
  } else {
    lazy_s(jb, mu, ts, jb.t + kLazyMax);
  }
  if (threadIdx.x == 0) *jb.cnt = 0u;
}

__global__ void __launch_bounds__(256) lazy_axpy_kernel(const __grid_constant__ Pack<LazyJob> P, double mu,
                                                        const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;
  const LazyJob& jb = P.j[blockIdx.y];
  if (jb.d <= 0 || (int64_t)blockIdx.x * 256 >= jb.rows) return;
  __shared__ double2 sv[kLazyMax];  // s = mu Sinv t, formed by lazy_dot_kernel's last block
  if (threadIdx.x < jb.d) sv[threadIdx.x] = jb.t[kLazyMax + threadIdx.x];
  __syncthreads();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= jb.rows) return;
  double re = 0.0, im = 0.0;
  int k = 0;
  for (; k + 8 <= jb.d; k += 8) {  // eight independent loads in flight, summed in order
    double2 p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = jb.P[i + (int64_t)(k + u) * jb.ld];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 x = sv[k + u];
      re = fma(p[u].x, x.x, re);
      re = fma(-p[u].y, x.y, re);
      im = fma(p[u].x, x.y, im);
      im = fma(p[u].y, x.x, im);
    }
  }
  for (; k < jb.d; ++k) {
    const double2 p = jb.P[i + (int64_t)k * jb.ld], x = sv[k];
    re = fma(p.x, x.x, re);
    re = fma(-p.y, x.y, re);
    im = fma(p.x, x.y, im);
    im = fma(p.y, x.x, im);
  }
  const double2 u = jb.w[i];
  if (jb.sum_into) {
    const double2 a = jb.sum_into[i];
    jb.sum_into[i] = make_double2(a.x + (u.x + re), a.y + (u.y + im));
  } else {
    jb.w[i] = make_double2(u.x + re, u.y + im);
  }
}

// The lazy term in ONE launch for short operators (up to kLazyFusedRows rows,
// where the two launches are pure latency: config 1 98 -> 88 us per iteration): a
// cluster of kLazyCluster CTAs per sensor.  Each warp dots one eliminated
// column with the vector (t = A_D^H u), the CTAs read each other's dots
// through distributed shared memory, every CTA forms s = mu Sinv t (or mu t)
// for itself, and then applies its share of the rows (w += P s, or
// dst += A_D s for the refinement residual).  Replaces lazy_dot_kernel +
// lazy_axpy_kernel / lazy_resid_axpy_kernel: one dependent launch instead of
// two in every post-trigger iteration (three lazy terms per refined solve).
constexpr int kLazyCluster = 8;
constexpr int kLazyFusedRows = 1024;  // above this the dots want more than 8 CTAs per sensor (C2 geometry: 2 launches are faster)

__device__ __forceinline__ double2 dsmem_ld_double2(const double2* p, unsigned cta) {
  uint32_t ra;
  double2 v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(cta));
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}

__global__ void __cluster_dims__(kLazyCluster, 1, 1) __launch_bounds__(256)
    lazy_fused_kernel(const __grid_constant__ Pack<LazyJob> P, double mu, const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;  // cancelled speculative iteration (the whole cluster)
  const LazyJob& jb = P.j[blockIdx.y];
  const int d = jb.d;
  if (d <= 0) return;
  const unsigned rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ __align__(16) double2 t_loc[8];  // dots of columns rank * 8 + warp
  __shared__ double2 t_all[kLazyMax];
  __shared__ double2 sv[kLazyMax];
  __shared__ int px[kLazyMax];
  {
    const int j = (int)rank * 8 + warp;
    double re = 0.0, im = 0.0;
    if (j < d) {
      const float2* a = jb.A + (int64_t)jb.pix[j] * jb.ld;
#pragma unroll 4
      for (int i = lane; i < jb.rows; i += 32) {
        const float2 x = a[i];
        const double2 u = jb.w[i];
        // conj(a) * u
        re = fma((double)x.x, u.x, re);
        re = fma((double)x.y, u.y, re);
        im = fma((double)x.x, u.y, im);
        im = fma(-(double)x.y, u.x, im);
      }
      re = warp_sum(re);
      im = warp_sum(im);
    }
    if (lane == 0) t_loc[warp] = make_double2(re, im);
  }
  cluster_sync_acqrel();  // every CTA's dots are written
  if ((int)threadIdx.x < d) {
    t_all[threadIdx.x] = dsmem_ld_double2(&t_loc[threadIdx.x & 7], threadIdx.x >> 3);
    px[threadIdx.x] = jb.pix[threadIdx.x];
  }
  __syncthreads();
  cluster_sync_acqrel();  // no CTA leaves while its dots may still be read
  if (jb.ident) {
    if ((int)threadIdx.x < d) sv[threadIdx.x] = make_double2(mu * t_all[threadIdx.x].x, mu * t_all[threadIdx.x].y);
  } else {
    lazy_s(jb, mu, t_all, sv);
  }
  __syncthreads();
  // this CTA's rows
  const int per = ((jb.rows + kLazyCluster - 1) / kLazyCluster + 31) & ~31;
  const int i_end = min(jb.rows, ((int)rank + 1) * per);
  for (int i = (int)rank * per + threadIdx.x; i < i_end; i += 256) {
    double re = 0.0, im = 0.0;
    if (jb.ident) {
      for (int k = 0; k < d; ++k) {
        const float2 a = jb.A[i + (int64_t)px[k] * jb.ld];
        const double2 x = sv[k];
        re = fma((double)a.x, x.x, re);
        re = fma(-(double)a.y, x.y, re);
        im = fma((double)a.x, x.y, im);
        im = fma((double)a.y, x.x, im);
      }
      const double2 u = jb.dst[i];
      jb.dst[i] = make_double2(u.x + re, u.y + im);
    } else {
      int k = 0;
      for (; k + 8 <= d; k += 8) {  // eight independent loads in flight, summed in order
        double2 p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) p[u] = jb.P[i + (int64_t)(k + u) * jb.ld];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 x = sv[k + u];
          re = fma(p[u].x, x.x, re);
          re = fma(-p[u].y, x.y, re);
          im = fma(p[u].x, x.y, im);
          im = fma(p[u].y, x.x, im);
        }
      }
      for (; k < d; ++k) {
        const double2 p = jb.P[i + (int64_t)k * jb.ld], x = sv[k];
        re = fma(p.x, x.x, re);
        re = fma(-p.y, x.y, re);
        im = fma(p.x, x.y, im);
        im = fma(p.y, x.x, im);
      }
      const double2 u = jb.w[i];
      if (jb.sum_into) {
        const double2 a = jb.sum_into[i];
        jb.sum_into[i] = make_double2(a.x + (u.x + re), a.y + (u.y + im));
      } else {
        jb.w[i] = make_double2(u.x + re, u.y + im);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// KM-space iterative refinement of the dual solve.  The explicit inverse G
// (Gauss-Jordan) applies C^{-1} with an error ~eps cond(C) |G| in every
// direction; the Woodbury x-update r - mu A^H w cancels in the operator's
// dominant directions and amplifies it by mu sigma^2 / beta (C2: 5.7e-6 per
// solve).  One step of fixed-precision refinement with the exact capacitance
//   rho = v - C_D w1,   w = w1 + C_D^{-1} rho,
//   C_D = C - mu A_D A_D^H  (C: packed lower tiles, kept next to G),
// makes the solve backward stable -- the accuracy of the reference's Cholesky
// (solver_core.hpp:41-51; DESIGN.md section 3 has the measurements).
// The C w1 product is the Hermitian apply over the packed tiles
// (herm_gapply_persist_kernel, packed = 1) with the reduce writing v - C w1;
// the kernels below add the lazy term and maintain C.
// ---------------------------------------------------------------------------

// dst += A_D s,  s = mu A_D^H w1 from lazy_dot_kernel (ident = 1)
__global__ void __launch_bounds__(256) lazy_resid_axpy_kernel(const __grid_constant__ Pack<LazyJob> P,
                                                              const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;
  const LazyJob& jb = P.j[blockIdx.y];
  if (jb.d <= 0 || (int64_t)blockIdx.x * 256 >= jb.rows) return;
  __shared__ double2 sv[kLazyMax];
  __shared__ int px[kLazyMax];
  if (threadIdx.x < jb.d) {
    sv[threadIdx.x] = jb.t[kLazyMax + threadIdx.x];
    px[threadIdx.x] = jb.pix[threadIdx.x];
  }
  __syncthreads();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= jb.rows) return;
  double re = 0.0, im = 0.0;
  for (int k = 0; k < jb.d; ++k) {
    const float2 a = jb.A[i + (int64_t)px[k] * jb.ld];
    const double2 x = sv[k];
    re = fma((double)a.x, x.x, re);
    re = fma(-(double)a.y, x.y, re);
    im = fma((double)a.x, x.y, im);
    im = fma((double)a.y, x.x, im);
  }
  const double2 u = jb.dst[i];
  jb.dst[i] = make_double2(u.x + re, u.y + im);
}

// C (column-major, ldc, Hermitian: lower tiles valid) -> packed lower tiles
__global__ void __launch_bounds__(256) cap_pack_kernel(const double2* __restrict__ C, int64_t ldc, int n,
                                                       double2* __restrict__ Cp) {
  pdl_enter();
  int t = blockIdx.x, I = 0;
  while (t > I) { t -= I + 1; ++I; }
  const int J = t;
  double2* dst = Cp + herm_packed_tile(I, J);
  for (int e = threadIdx.x; e < kHermTile * kHermTile; e += 256) {
    const int r = e & 63, cc = e >> 6, i = I * kHermTile + r, j = J * kHermTile + cc;
    dst[e] = (i < n && j < n) ? C[i + (int64_t)j * ldc] : make_double2(0.0, 0.0);
  }
}

// Packed C <- C - mu A_R A_R^H over the lower tiles (columns R = pix[0..r) of
// the complex64 operator): the capacitance of the smaller active set after a
// fold or eager downdate.  One CTA per (tile, job); 64-column chunks of R in
// shared memory (16 at a time), fp64 products of the promoted entries, fixed order.
struct CapJob {
  double2* Cp;
  const float2* A;
  int64_t ld;
  int n;
  const int* pix;
  int r;
};

__global__ void __launch_bounds__(256) cap_update_kernel(const __grid_constant__ Pack<CapJob> P, double mu) {
  pdl_enter();
  const CapJob& jb = P.j[blockIdx.y];
  const int nb = (jb.n + kHermTile - 1) / kHermTile;
  if ((int64_t)blockIdx.x >= (int64_t)nb * (nb + 1) / 2 || jb.r <= 0) return;
  int t = blockIdx.x, I = 0;
  while (t > I) { t -= I + 1; ++I; }
  const int J = t;
  constexpr int kCh = 16;  // columns of R per shared stage
  __shared__ double2 ai[kCh][kHermTile + 1], aj[kCh][kHermTile + 1];
  const int tr = threadIdx.x & 63, tc = threadIdx.x >> 6;  // row, column phase (4)
  double accr[16], acci[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) accr[u] = acci[u] = 0.0;
  for (int k0 = 0; k0 < jb.r; k0 += kCh) {
    const int kn = min(kCh, jb.r - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kCh * kHermTile; e += 256) {
      const int k = e >> 6, rr = e & 63;
      double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
      if (k < kn) {
        const int64_t col = (int64_t)jb.pix[k0 + k] * jb.ld;
        const int i = I * kHermTile + rr, j = J * kHermTile + rr;
        if (i < jb.n) { const float2 a = jb.A[col + i]; x = make_double2(a.x, a.y); }
        if (j < jb.n) { const float2 a = jb.A[col + j]; y = make_double2(a.x, a.y); }
      }
      ai[k][rr] = x;
      aj[k][rr] = y;
    }
    __syncthreads();
    for (int k = 0; k < kn; ++k) {
      const double2 x = ai[k][tr];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double2 y = aj[k][tc + 4 * u];
        // x * conj(y)
        accr[u] = fma(x.x, y.x, accr[u]);
        accr[u] = fma(x.y, y.y, accr[u]);
        acci[u] = fma(x.y, y.x, acci[u]);
        acci[u] = fma(-x.x, y.y, acci[u]);
      }
    }
  }
  double2* dst = jb.Cp + herm_packed_tile(I, J);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int cc = tc + 4 * u, i = I * kHermTile + tr, j = J * kHermTile + cc;
    if (i >= jb.n || j >= jb.n || (I == J && i < j)) continue;  // diagonal tiles: lower half + exact mirror
    double2 v = dst[tr + cc * kHermTile];
    v.x -= mu * accr[u];
    v.y -= mu * acci[u];
    if (i == j) v.y = 0.0;  // the diagonal of a Hermitian matrix stays real
    dst[tr + cc * kHermTile] = v;
    if (I == J && i > j) dst[cc + tr * kHermTile] = make_double2(v.x, -v.y);
  }
}

// Packed lower tiles of a Hermitian G <- G + alpha X Y^H (X, Y: ld x d,
// complex128): the lazy fold / eager downdate of a packed dual factor
// (G + mu (P Sinv) P^H).  One CTA per (tile, job), fixed order.
struct PackedUpdJob {
  double2* Gp;
  const double2* X;
  const double2* Y;
  int64_t ld;
  int n, d;
};

__global__ void __launch_bounds__(256) herm_packed_update_kernel(const __grid_constant__ Pack<PackedUpdJob> P,
                                                                 double alpha) {
  pdl_enter();
  const PackedUpdJob& jb = P.j[blockIdx.y];
  const int nb = (jb.n + kHermTile - 1) / kHermTile;
  if ((int64_t)blockIdx.x >= (int64_t)nb * (nb + 1) / 2 || jb.d <= 0) return;
  int t = blockIdx.x, I = 0;
  while (t > I) { t -= I + 1; ++I; }
  const int J = t;
  constexpr int kCh = 16;
  __shared__ double2 xi[kCh][kHermTile + 1], yj[kCh][kHermTile + 1];
  const int tr = threadIdx.x & 63, tc = threadIdx.x >> 6;
  double accr[16], acci[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) accr[u] = acci[u] = 0.0;
  for (int k0 = 0; k0 < jb.d; k0 += kCh) {
    const int kn = min(kCh, jb.d - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kCh * kHermTile; e += 256) {
      const int k = e >> 6, rr = e & 63;
      const int i = I * kHermTile + rr, j = J * kHermTile + rr;
      xi[k][rr] = (k < kn && i < jb.n) ? jb.X[i + (int64_t)(k0 + k) * jb.ld] : make_double2(0.0, 0.0);
      yj[k][rr] = (k < kn && j < jb.n) ? jb.Y[j + (int64_t)(k0 + k) * jb.ld] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int k = 0; k < kn; ++k) {
      const double2 x = xi[k][tr];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double2 y = yj[k][tc + 4 * u];
        accr[u] = fma(x.x, y.x, accr[u]);
        accr[u] = fma(x.y, y.y, accr[u]);
        acci[u] = fma(x.y, y.x, acci[u]);
        acci[u] = fma(-x.x, y.y, acci[u]);
      }
    }
  }
  double2* dst = jb.Gp + herm_packed_tile(I, J);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int cc = tc + 4 * u, i = I * kHermTile + tr, j = J * kHermTile + cc;
    if (i >= jb.n || j >= jb.n || (I == J && i < j)) continue;  // diagonal tiles: lower half + exact mirror
    double2 v = dst[tr + cc * kHermTile];
    v.x += alpha * accr[u];
    v.y += alpha * acci[u];
    if (i == j) v.y = 0.0;
    dst[tr + cc * kHermTile] = v;
    if (I == J && i > j) dst[cc + tr * kHermTile] = make_double2(v.x, -v.y);
  }
}

// w[i] += dw[i] for the listed vectors (refinement correction after the lazy
// terms were applied to dw)
struct VaddJob {
  double2* w;
  const double2* dw;
  int n;
};
__global__ void __launch_bounds__(256) vadd_kernel(const __grid_constant__ Pack<VaddJob> P, const int* __restrict__ go) {
  pdl_enter();
  if (go && __ldg(go) == 0) return;
  const VaddJob& jb = P.j[blockIdx.y];
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= jb.n) return;
  const double2 a = jb.w[i], b = jb.dw[i];
  jb.w[i] = make_double2(a.x + b.x, a.y + b.y);
}

// Bordered update of Sinv when r <= kBorderMax columns join D (d0 -> d0 + r):
//   S' = [[S11, S12], [S12^H, S22]],  S12 = -mu A_old^H P_new,
//   S22 = I - mu A_new^H P_new,  S11^{-1} = Sinv (known)
//   W = Sinv S12,  Z = S22 - S12^H W (Schur complement, HPD),  X = W Z^{-1}
//   S'^{-1} = [[Sinv + X W^H, -X], [-X^H, Z^{-1}]]
// lazy_border_dots_kernel forms B = A_D^H P_new (grid (d0 + r, jobs)), then
// lazy_border_inv_kernel (one CTA per job) does the O(d^2 r) rest; a
// non-positive pivot of Z sets *fail (the reference's "Cholesky failed").
constexpr int kBorderMax = 16;

struct BorderJob {
  const float2* A;
  int64_t ld;
  int rows;
  const int* pix;      // D (d0 + r pixels)
  int d0, r;
  const double2* P;    // ld x (d0 + r)
  double2* B;          // (d0 + r) x kBorderMax scratch: B[j][u] = a_j^H P[:, d0 + u]
  double2* Sinv;       // kLazyMax x kLazyMax (column-major)
  int* fail;
};

__global__ void __launch_bounds__(256) lazy_border_dots_kernel(const __grid_constant__ Pack<BorderJob> P) {
  pdl_enter();
  const BorderJob& jb = P.j[blockIdx.y];
  const int j = blockIdx.x;
  if (j >= jb.d0 + jb.r) return;
  const float2* a = jb.A + (int64_t)jb.pix[j] * jb.ld;
  double re[kBorderMax], im[kBorderMax];
#pragma unroll
  for (int u = 0; u < kBorderMax; ++u) re[u] = im[u] = 0.0;
  for (int i = threadIdx.x; i < jb.rows; i += 256) {
    const float2 x = a[i];
    const double xr = x.x, xi = x.y;
#pragma unroll
    for (int u = 0; u < kBorderMax; ++u) {
      if (u >= jb.r) break;
      const double2 p = jb.P[(int64_t)(jb.d0 + u) * jb.ld + i];
      re[u] = fma(xr, p.x, re[u]);
      re[u] = fma(xi, p.y, re[u]);
      im[u] = fma(xr, p.y, im[u]);
      im[u] = fma(-xi, p.x, im[u]);
    }
  }
  __shared__ double sr[8][kBorderMax], si[8][kBorderMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < kBorderMax; ++u) {
    if (u >= jb.r) break;
    const double a0 = warp_sum(re[u]), b0 = warp_sum(im[u]);
    if (lane == 0) { sr[warp][u] = a0; si[warp][u] = b0; }
  }
  __syncthreads();
  if (threadIdx.x < jb.r) {
    const int u = threadIdx.x;
    double a0 = sr[0][u], b0 = si[0][u];
    for (int w = 1; w < 8; ++w) { a0 += sr[w][u]; b0 += si[w][u]; }
    jb.B[(int64_t)j * kBorderMax + u] = make_double2(a0, b0);
  }
}

constexpr size_t kBorderSmem = (size_t)(kLazyMax * kLazyMax + 3 * kLazyMax * kBorderMax + kBorderMax * kBorderMax) * 16;

__global__ void __launch_bounds__(256) lazy_border_inv_kernel(const __grid_constant__ Pack<BorderJob> P, double mu) {
  pdl_enter();
  const BorderJob& jb = P.j[blockIdx.x];
  extern __shared__ __align__(16) double2 bsm[];
  double2* S = bsm;                                   // Sinv_old  d0 x d0 (ld kLazyMax)
  double2* S12 = S + kLazyMax * kLazyMax;             // d0 x r   (ld kLazyMax)
  double2* W = S12 + kLazyMax * kBorderMax;           // d0 x r
  double2* X = W + kLazyMax * kBorderMax;             // d0 x r
  double2* Z = X + kLazyMax * kBorderMax;             // r x r    (ld kBorderMax)
  __shared__ int bad;
  const int d0 = jb.d0, r = jb.r, tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < d0 * d0; e += 256) {
    const int i = e % d0, k = e / d0;
    S[i + k * kLazyMax] = jb.Sinv[i + (int64_t)k * kLazyMax];
  }
  for (int e = tid; e < d0 * r; e += 256) {
    const int i = e % d0, u = e / d0;
    const double2 b = jb.B[(int64_t)i * kBorderMax + u];
    S12[i + u * kLazyMax] = make_double2(-mu * b.x, -mu * b.y);
  }
  for (int e = tid; e < r * r; e += 256) {
    const int v = e % r, u = e / r;
    const double2 b = jb.B[(int64_t)(d0 + v) * kBorderMax + u];
    Z[v + u * kBorderMax] = make_double2((v == u ? 1.0 : 0.0) - mu * b.x, -mu * b.y);
  }
  __syncthreads();
  // W = Sinv_old S12
  for (int e = tid; e < d0 * r; e += 256) {
    const int i = e % d0, u = e / d0;
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < d0; ++k) acc = c_fma(S[i + k * kLazyMax], S12[k + u * kLazyMax], acc);
    W[i + u * kLazyMax] = acc;
  }
  __syncthreads();
  // Z -= S12^H W
  for (int e = tid; e < r * r; e += 256) {
    const int v = e % r, u = e / r;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < d0; ++i) acc = c_fma(c_conj(S12[i + v * kLazyMax]), W[i + u * kLazyMax], acc);
    Z[v + u * kBorderMax] = c_sub(Z[v + u * kBorderMax], acc);
  }
  __syncthreads();
  // Z <- Z^{-1}: Gauss-Jordan without pivoting (Z is HPD)
  for (int k = 0; k < r; ++k) {
    const double2 pk = Z[k + k * kBorderMax];
    if (!(pk.x > 0.0)) {
      if (tid == 0) bad = 1;
    }
    __syncthreads();
    if (bad) break;
    const double2 inv = make_double2(1.0 / pk.x, 0.0);  // HPD: real positive pivot
    // row k of the rest / column k: standard in-place GJ step
    const int i = tid % kBorderMax, j = tid / kBorderMax;  // 256 threads cover 16 x 16
    double2 v = make_double2(0.0, 0.0);
    if (i < r && j < r) {
      const double2 zik = Z[i + k * kBorderMax], zkj = Z[k + j * kBorderMax], zij = Z[i + j * kBorderMax];
      if (i == k && j == k) v = inv;
      else if (i == k) v = c_mul(zkj, inv);
      else if (j == k) v = c_mul(make_double2(-zik.x, -zik.y), inv);
      else v = c_sub(zij, c_mul(c_mul(zik, inv), zkj));
    }
    __syncthreads();
    if (i < r && j < r) Z[i + j * kBorderMax] = v;
    __syncthreads();
  }
  if (tid == 0) *jb.fail = bad;
  if (bad) return;
  // X = W Zinv
  for (int e = tid; e < d0 * r; e += 256) {
    const int i = e % d0, u = e / d0;
    double2 acc = make_double2(0.0, 0.0);
    for (int v = 0; v < r; ++v) acc = c_fma(W[i + v * kLazyMax], Z[v + u * kBorderMax], acc);
    X[i + u * kLazyMax] = acc;
  }
  __syncthreads();
  // S'^{-1}
  for (int e = tid; e < d0 * d0; e += 256) {
    const int i = e % d0, k = e / d0;
    double2 acc = S[i + k * kLazyMax];
    for (int u = 0; u < r; ++u) acc = c_fma(X[i + u * kLazyMax], c_conj(W[k + u * kLazyMax]), acc);
    jb.Sinv[i + (int64_t)k * kLazyMax] = acc;
  }
  for (int e = tid; e < d0 * r; e += 256) {
    const int i = e % d0, u = e / d0;
    const double2 x = X[i + u * kLazyMax];
    jb.Sinv[i + (int64_t)(d0 + u) * kLazyMax] = make_double2(-x.x, -x.y);
    jb.Sinv[(d0 + u) + (int64_t)i * kLazyMax] = make_double2(-x.x, x.y);
  }
  for (int e = tid; e < r * r; e += 256) {
    const int v = e % r, u = e / r;
    jb.Sinv[(d0 + v) + (int64_t)(d0 + u) * kLazyMax] = Z[v + u * kBorderMax];
  }
}

#if RADMM_EXPERIMENTAL  // TMA-ring variant (RADMM_HERM=2), measured slower
// TMA-staged variant: persistent CTAs (one per SM) walk the item list
// round-robin; warp 8 streams each 64 x 64 tile (64 column segments of
// <= 1 KB) into a kHermStages-deep shared ring with cp.async.bulk, and the
// eight compute warps consume it exactly like herm_gapply_kernel.
constexpr int kHermStages = 3;
constexpr int kHermTileBytes = kHermTile * kHermTile * 16;
constexpr size_t kHermTmaSmem = (size_t)kHermStages * kHermTileBytes + 2 * 8 * kHermTile * 16 + 2 * kHermStages * 8;


__global__ void __launch_bounds__(288, 1) herm_gapply_tma_kernel(const __grid_constant__ Pack<HermJob> P,
                                                                const uint64_t* __restrict__ items, int n_items,
                                                                const int* __restrict__ go) {
  pdl_enter();
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
#endif

// Hermitian projection of a factor in place: G <- (G + G^H) / 2 (the nearest
// Hermitian matrix; never increases the Frobenius error of an inverse).
// One 32 x 32 tile pair (I > J) or diagonal tile per CTA, staged through
// shared memory so both halves are read and written coalesced.
__global__ void __launch_bounds__(256) herm_symmetrize_kernel(double2* __restrict__ G, int64_t ld, int n) {
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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


template <int MODE>
__global__ void __launch_bounds__(256, 2) frame_batch2_kernel(const FrameBatchJob* __restrict__ jobs, int nsplit,
                                                             double mu, double beta) {
  pdl_enter();
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

__device__ __forceinline__ void gram_dmma_body(const GramJob& jb, double mu, double beta) {
  constexpr int BK = kFbBK, S = kFbStages;
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

__global__ void __launch_bounds__(256, 1) gram_dmma_kernel(const GramJob* __restrict__ jobs, double mu, double beta) {
  pdl_enter();
  gram_dmma_body(jobs[blockIdx.z], mu, beta);
}

// one job passed by value (no job-table upload on the issuing stream)
__global__ void __launch_bounds__(256, 1) gram_dmma1_kernel(const __grid_constant__ GramJob job, double mu, double beta) {
  pdl_enter();
  gram_dmma_body(job, mu, beta);
}

// C <- beta I + mu C for a raw Gram (eager_gram): the same roundings as
// gram_dmma_kernel applying mu, beta itself (mu * c, then + beta on the
// diagonal, imaginary diagonal exactly 0).
__global__ void gram_scale_kernel(double2* __restrict__ C, int64_t ldc, int n, double mu, double beta) {
  pdl_enter();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * n) return;
  const int i = (int)(e % n), j = (int)(e / n);
  double2* p = C + i + (int64_t)j * ldc;
  const double2 v = *p;
  double2 o = make_double2(mu * v.x, mu * v.y);
  if (i == j) {
    o.x += beta;
    o.y = 0.0;
  }
  *p = o;
}

// out_f[i] = sum_s part[s][f][i] (fixed split order) for every frame of a job
struct FrameReduceJob {
  const double2* part;
  int64_t ldp;
  int m, nf, nsplit;
  double2* out[kFB];
  const double2* base[kFB];  // refinement: out = base + sgn * sum (nullptr: out = sum)
  double sgn;
};

__global__ void frame_reduce_kernel(const FrameReduceJob* __restrict__ jobs) {
  pdl_enter();
  const FrameReduceJob& jb = jobs[blockIdx.z];
  const int i = blockIdx.x * blockDim.x + threadIdx.x, f = blockIdx.y;
  if (i >= jb.m || f >= jb.nf) return;
  double2 s = make_double2(0.0, 0.0);
  for (int sp = 0; sp < jb.nsplit; ++sp) {
    const double2 v = jb.part[((int64_t)sp * kFB + f) * jb.ldp + i];
    s.x += v.x;
    s.y += v.y;
  }
  if (jb.base[f]) {
    const double2 b = jb.base[f][i];
    s = make_double2(b.x + jb.sgn * s.x, b.y + jb.sgn * s.y);
  }
  jb.out[f][i] = s;
}

// packed complex128 tiles -> packed complex64 tiles (the refinement's
// correction pass only needs modest relative accuracy: its input is the small
// residual)
__global__ void __launch_bounds__(256) pack_to_c64_kernel(const double2* __restrict__ Gp, float2* __restrict__ G32,
                                                          int64_t n) {
  pdl_enter();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = Gp[i];
    G32[i] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
  }
}

// packed lower tiles -> full Hermitian matrix (column-major, ld), for the
// frame-batched refinement pass R = V - C W on the fp64 tensor cores
__global__ void __launch_bounds__(256) cap_unpack_kernel(const double2* __restrict__ Cp, int n,
                                                         double2* __restrict__ C, int64_t ldc) {
  pdl_enter();
  int t = blockIdx.x, I = 0;
  while (t > I) { t -= I + 1; ++I; }
  const int J = t;
  const double2* src = Cp + herm_packed_tile(I, J);
  for (int e = threadIdx.x; e < kHermTile * kHermTile; e += 256) {
    const int r = e & 63, cc = e >> 6, i = I * kHermTile + r, j = J * kHermTile + cc;
    if (i >= n || j >= n) continue;
    const double2 v = src[e];
    if (I == J) {
      if (i >= j) {
        C[i + (int64_t)j * ldc] = v;
        C[j + (int64_t)i * ldc] = make_double2(v.x, -v.y);
      }
    } else {
      C[i + (int64_t)j * ldc] = v;
      C[j + (int64_t)i * ldc] = make_double2(v.x, -v.y);
    }
  }
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
  pdl_enter();
  const FrameRhsJob& jb = jobs[blockIdx.y];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= jb.n) return;
  const double2 d = jb.data[j], g = jb.gap[j], x = jb.x_hat[j], sg = jb.sigma[j];
  jb.rhs[j] = make_double2(__dsub_rn(__dadd_rn(__dadd_rn(d.x, __dmul_rn(beta, g.x)), __dmul_rn(beta, x.x)), sg.x),
                           __dsub_rn(__dadd_rn(__dadd_rn(d.y, __dmul_rn(beta, g.y)), __dmul_rn(beta, x.y)), sg.y));
}

}  // namespace radmm_dev
