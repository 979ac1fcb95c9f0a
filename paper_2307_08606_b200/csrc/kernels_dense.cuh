// kernels_dense.cuh: fp64 complex GEMMs (SIMT and DMMA), Gauss-Jordan inverse, small utility kernels
// Part of kernels.cuh (see that file's header); included in order from there.
#pragma once

namespace radmm_dev {

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
  pdl_enter();
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
  pdl_enter();
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


template <int EPI>
__global__ void __launch_bounds__(256, 1) gemm_dmma_kernel(const __grid_constant__ Pack<GemmJob> jobs) {
  pdl_enter();
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
  // Epilogue, one 8-row block (a) at a time: its 8 C / R' inputs are loaded
  // first (independent loads in flight together), then combined and stored.
  // Interleaving each read with the previous element's store would serialise
  // them (the compiler cannot move a load above a possibly aliasing store):
  // 32 dependent round trips per thread on the read-modify-write updates.
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = m0 + wm + 8 * a + fr;
    double2 cin[4][2];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = n0 + wn + 8 * b + 2 * fc + v;
        cin[b][v] = make_double2(0.0, 0.0);
        if (i >= jb.m || j >= jb.n) continue;
        if (EPI == GEPI_PLAIN) {
          if (jb.beta0 != 0.0 && !(jb.herm && i < j)) cin[b][v] = jb.c[i + (int64_t)j * jb.ldc];
        } else if (i >= jb.k0 && i < jb.k0 + jb.kb) {
          cin[b][v] = reinterpret_cast<const double2*>(jb.b.p)[(i - jb.k0) + (int64_t)j * jb.b.ld];
        } else if (!(j >= jb.k0 && j < jb.k0 + jb.kb)) {
          cin[b][v] = jb.c[i + (int64_t)j * jb.ldc];
        }
      }
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = n0 + wn + 8 * b + 2 * fc + v;
        if (i >= jb.m || j >= jb.n) continue;
        double2* cp = jb.c + i + (int64_t)j * jb.ldc;
        const double accr = p1[a][b][v] - p2[a][b][v], acci = p3[a][b][v] - p1[a][b][v] - p2[a][b][v];
        const double2 c0 = cin[b][v];
        if (EPI == GEPI_PLAIN) {
          if (jb.herm && i < j) continue;
          double2 o = make_double2(jb.alpha * accr, jb.alpha * acci);
          if (jb.beta0 != 0.0) {
            o.x += jb.beta0 * c0.x;
            o.y += jb.beta0 * c0.y;
          }
          if (i == j) {
            o.x += jb.diag_add;
            if (jb.herm) o.y = 0.0;
          }
          *cp = o;
          if (jb.herm && i != j) jb.c[j + (int64_t)i * jb.ldc] = make_double2(o.x, -o.y);
        } else if (i >= jb.k0 && i < jb.k0 + jb.kb) {
          //   i in K:      M[i,j] = R'[i-k0, j]
          *cp = c0;
        } else {
          //   i not in K:  M[i,j] = (j in K ? 0 : M[i,j]) - (F R')[i,j]
          *cp = make_double2(c0.x - accr, c0.y - acci);
        }
      }
  }
}

// Gauss-Jordan rank-kb update (kb <= 64), the dominant cost of the explicit
// inverse: M[i,j] = (j in K ? 0 : M[i,j]) - sum_k F[i,k] R'[k,j] for i not in
// K, M[i,j] = R'[i-k0, j] for i in K.  The whole K extent of both operands
// fits in shared memory (F tile 128 x 64, R' tile 64 x 64, complex128, pitches
// = 2 (mod 8) so a quarter warp's 16-B fragment loads hit distinct banks), so
// one cp.async batch fills it and the 16 k4-steps of 3M DMMAs run without a
// barrier.  Same k order and DMMA sequence as gemm_dmma_kernel<GEPI_GJ>:
// bitwise-identical results.
constexpr int kGjuBM = 128, kGjuBN = 64, kGjuPF = 130, kGjuPR = 66;
constexpr size_t kGjuSmem = (size_t)64 * (kGjuPF + kGjuPR) * sizeof(double2);

struct GjUpdJob {
  double2* M;
  int64_t ldm;
  int n;
  const double2* F;  // n x kb, leading dimension ldf
  int64_t ldf;
  const double2* R;  // kb x n, leading dimension 64
  int k0, kb;
};

// HERM: the Hermitian sweep (gj_invert, herm = true): F = T = M[:, K] P,
// R[k, j] = conj(M[j, K][k]); only tiles that touch the lower triangle
// (n0 < m0 + 128) are updated, M[i, j] -= (T R)[i, j] everywhere in them; the
// pivot rows / columns are rewritten afterwards by gj_hfix_kernel.
template <bool HERM>
__global__ void __launch_bounds__(256, 1) gj_update_kernel(const __grid_constant__ Pack<GjUpdJob> P) {
  pdl_enter();
  const GjUpdJob& jb = P.j[blockIdx.z];
  const int m0 = blockIdx.y * kGjuBM, n0 = blockIdx.x * kGjuBN, n = jb.n, kb = jb.kb;
  if (m0 >= n || n0 >= n) return;
  if (HERM && n0 >= m0 + kGjuBM) return;  // strictly upper tile: never read
  extern __shared__ __align__(16) double2 gju[];
  double2* Fs = gju;                   // [k][kGjuPF]
  double2* Rs = gju + 64 * kGjuPF;     // [k][kGjuPR]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 64 * kGjuBM; e += 256) {  // F tile: 128 rows x 64 k (column-major source)
    const int i = e % kGjuBM, k = e / kGjuBM;
    const bool ok = m0 + i < n && k < kb;
    cp_async16(Fs + k * kGjuPF + i, ok ? jb.F + (m0 + i) + (int64_t)k * jb.ldf : jb.F, ok);
  }
  for (int e = tid; e < 64 * kGjuBN; e += 256) {  // R' tile: 64 k x 64 columns
    const int k = e % 64, j = e / 64;
    const bool ok = n0 + j < n && k < kb;
    cp_async16(Rs + k * kGjuPR + j, ok ? jb.R + k + (int64_t)(n0 + j) * 64 : jb.R, ok);
  }
  cp_async_commit();
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32, fr = lane >> 2, fc = lane & 3;
  double p1[4][4][2], p2[4][4][2], p3[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) p1[a][b][v] = p2[a][b][v] = p3[a][b][v] = 0.0;
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll 1
  for (int k4 = 0; k4 < 64; k4 += 4) {
    double ar[4], ai[4], as[4], br[4], bi[4], bs[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double2 x = Fs[(k4 + fc) * kGjuPF + wm + 8 * a + fr];
      ar[a] = x.x;
      ai[a] = x.y;
      as[a] = ar[a] + ai[a];
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const double2 y = Rs[(k4 + fc) * kGjuPR + wn + 8 * b + fr];
      br[b] = y.x;
      bi[b] = y.y;
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
  // epilogue (gemm_dmma_kernel<GEPI_GJ>), one 8-row block at a time, inputs first
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = m0 + wm + 8 * a + fr;
    const bool iK = !HERM && i >= jb.k0 && i < jb.k0 + kb;
    double2 cin[4][2];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = n0 + wn + 8 * b + 2 * fc + v;
        cin[b][v] = make_double2(0.0, 0.0);
        if (i >= n || j >= n) continue;
        if (iK) cin[b][v] = jb.R[(i - jb.k0) + (int64_t)j * 64];
        else if (HERM || !(j >= jb.k0 && j < jb.k0 + kb)) cin[b][v] = jb.M[i + (int64_t)j * jb.ldm];
      }
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int j = n0 + wn + 8 * b + 2 * fc + v;
        if (i >= n || j >= n) continue;
        double2* cp = jb.M + i + (int64_t)j * jb.ldm;
        if (iK) {
          *cp = cin[b][v];
        } else {
          const double accr = p1[a][b][v] - p2[a][b][v], acci = p3[a][b][v] - p1[a][b][v] - p2[a][b][v];
          *cp = make_double2(cin[b][v].x - accr, cin[b][v].y - acci);
        }
      }
  }
}

// C = alpha * sum_s ws[job*nsplit + s] + beta0 * C (+ diag), fixed split order.
__global__ void gemm_split_reduce(const __grid_constant__ Pack<GemmJob> jobs, int nsplit,
                                  const double2* __restrict__ ws, int64_t ws_stride) {
  pdl_enter();
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
  double2* M;      // the matrix being swept (read by the pivot / panel kernels, rewritten by gj_hfix_kernel)
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
  int herm;       // Hermitian sweep: the pivot block and its inverse are made exactly Hermitian
};

__global__ void __launch_bounds__(1024) gj_diag_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  pdl_enter();
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
  // Hermitian sweep: the row panel is taken as the conjugate transpose of the
  // column panel M[:, K] P, which is only consistent if P is exactly
  // Hermitian -- an unsymmetric rounding-level defect of P compounds from
  // block to block (measured on config 2's capacitance, cond 2e5: |G C - I|
  // 4.7e3 without this, 2e-7 with it; the general sweep: 1.3e-6).
  auto hermitize = [&]() {
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
      const int r = e % kb, c = e / kb;
      if (r < c) continue;
      const double2 a = S[r][c], b = S[c][r];
      const double2 m = r == c ? make_double2(a.x, 0.0) : make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      S[r][c] = m;
      S[c][r] = make_double2(m.x, -m.y);
    }
    __syncthreads();
  };
  if (jb.herm) hermitize();
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
  if (jb.herm) hermitize();
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int r = e % kb, c = e / kb;
    jb.P[r + (int64_t)c * jb.ldp] = S[r][c];
  }
}

// F = M[:, K] (pivot column panel), grid-stride over n*kb per job.
__global__ void gj_panel_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  pdl_enter();
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
  pdl_enter();
  const DiagJob& jb = jobs.j[blockIdx.x];
  if (jb.k0 >= jb.n) return;
  for (int e = threadIdx.x; e < jb.kb * jb.kb; e += blockDim.x) {
    const int r = e % jb.kb, c = e / jb.kb;
    jb.R[r + (int64_t)(jb.k0 + c) * jb.ldr] = jb.P[r + (int64_t)c * jb.ldp];
  }
}

// ---- Hermitian sweep (blocked symmetric Gauss-Jordan for HPD matrices) -------
// Sweeping pivot block K of a Hermitian M:  M_KK <- -inv(M_KK) = -P,
// M_iK <- M_iK P,  M_ij <- M_ij - M_iK P M_Kj; every intermediate matrix is
// Hermitian, so only the lower triangle is kept and updated (half the DMMA
// work and half the memory traffic of the general sweep), and after the last
// block M = -inv(M0).
//
// F[i, c] = M[i, k0 + c] read from the lower triangle (rows above the pivot
// block come from the conjugate of the pivot rows), and R[c, i] = conj(F[i, c])
// (the update's right operand).
__global__ void gj_hpanel_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  pdl_enter();
  const DiagJob& jb = jobs.j[blockIdx.y];
  if (jb.k0 >= jb.n) return;
  const int kb = jb.kb, k0 = jb.k0;
  // rows at / below the pivot block: column segments of M (row index fastest)
  const int64_t low = (int64_t)(jb.n - k0) * kb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < low; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = k0 + (int)(e % (jb.n - k0)), c = (int)(e / (jb.n - k0));
    const double2 v = jb.M[i + (int64_t)(k0 + c) * jb.ld];
    jb.F[i + (int64_t)c * jb.ldf] = v;
    jb.R[c + (int64_t)i * jb.ldr] = make_double2(v.x, -v.y);
  }
  // rows above: conj of the pivot rows (pivot-row index fastest: contiguous in M)
  const int64_t up = (int64_t)k0 * kb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < up; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % kb), i = (int)(e / kb);
    const double2 v = jb.M[(k0 + c) + (int64_t)i * jb.ld];
    jb.F[i + (int64_t)c * jb.ldf] = make_double2(v.x, -v.y);
    jb.R[c + (int64_t)i * jb.ldr] = v;
  }
}

// After the update: M[i, K] = T[i, :] below the pivot block, M[K, i] = T[i, :]^H
// left of it, M_KK = -P.  T = F P (n x kb, ld = ldf) travels in jb.F.
__global__ void gj_hfix_kernel(const __grid_constant__ Pack<DiagJob> jobs) {
  pdl_enter();
  const DiagJob& jb = jobs.j[blockIdx.y];
  if (jb.k0 >= jb.n) return;
  const int kb = jb.kb, k0 = jb.k0;
  const int64_t low = (int64_t)(jb.n - k0) * kb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < low; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = k0 + (int)(e % (jb.n - k0)), c = (int)(e / (jb.n - k0));
    double2 v;
    if (i < k0 + kb) {
      const double2 p = jb.P[(i - k0) + (int64_t)c * jb.ldp];
      v = make_double2(-p.x, -p.y);
    } else {
      v = jb.F[i + (int64_t)c * jb.ldf];
    }
    jb.M[i + (int64_t)(k0 + c) * jb.ld] = v;
  }
  const int64_t up = (int64_t)k0 * kb;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < up; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % kb), i = (int)(e / kb);
    const double2 v = jb.F[i + (int64_t)c * jb.ldf];
    jb.M[(k0 + c) + (int64_t)i * jb.ld] = make_double2(v.x, -v.y);
  }
}

// M <- -M on the lower triangle, mirrored conjugate to the upper one, real
// diagonal: the inverse, exactly Hermitian.  One 32 x 32 tile (I >= J) per CTA.
__global__ void __launch_bounds__(256) gj_hfinish_kernel(double2* __restrict__ G, int64_t ld, int n) {
  pdl_enter();
  __shared__ double2 a[32][33];
  int t = blockIdx.x, I = 0;
  while (t > I) { t -= I + 1; ++I; }
  const int J = t;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int i = I * 32 + tx, j = J * 32 + r;  // tile (I, J): column j, row i
    double2 v = (i < n && j < n) ? G[i + (int64_t)j * ld] : make_double2(0.0, 0.0);
    if (I == J && i < j) {  // upper half of a diagonal tile: from its mirror, below
      v = (i < n && j < n) ? G[j + (int64_t)i * ld] : make_double2(0.0, 0.0);
      v.y = -v.y;
    }
    v = make_double2(-v.x, -v.y);
    if (i == j) v.y = 0.0;
    a[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = I * 32 + tx, j = J * 32 + r;
    if (i < n && j < n) G[i + (int64_t)j * ld] = a[r][tx];
    const int i2 = J * 32 + tx, j2 = I * 32 + r;  // tile (J, I) = conj transpose
    const double2 v = a[tx][r];
    if (I != J && i2 < n && j2 < n) G[i2 + (int64_t)j2 * ld] = make_double2(v.x, -v.y);
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
  pdl_enter();
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
  pdl_enter();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)rows * cols) return;
  const int r = (int)(e % rows);
  const int64_t c = e / rows;
  const double2 v = src[r + c * lds];
  dst[r + c * ldd] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
}

__global__ void soft_threshold_kernel(const double2* __restrict__ v, int64_t n, double kappa, double2* __restrict__ out) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = soft_threshold1(v[i], kappa);
}

__global__ void abs_kernel(const double2* __restrict__ v, int n, double* __restrict__ out) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = c_abs(v[i]);
}

// out = beta * (a - b): the accumulated frozen echo z = y_eff_s - y_eff,
// scaled, that is folded into v when the stored data term lags (see
// local_updates in radmm_b200.cu).
__global__ void scaled_diff_kernel(double2* __restrict__ out, const double2* __restrict__ a,
                                   const double2* __restrict__ b, double beta, int64_t n) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = make_double2(beta * (a[i].x - b[i].x), beta * (a[i].y - b[i].y));
}

// Rb[:, t] = A[:, rem_pix[t]] promoted to complex128 (zero-padded to ld).
__global__ void gather_cols_c128_kernel(const float2* __restrict__ A, int64_t ld, const int* __restrict__ pix,
                                        int r, double2* __restrict__ out) {
  pdl_enter();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ld * r) return;
  const int t = (int)(e / ld);
  const int64_t row = e % ld;
  const float2 v = A[row + (int64_t)pix[t] * ld];
  out[e] = make_double2((double)v.x, (double)v.y);
}

// Per-sensor bookkeeping of one elimination event, all sensors in one launch
// (blockIdx.y = sensor); every part is optional (null pointer = skip):
//   log_dst[t] = lz_pix_dst[t] = rem_pix[t]            (removal log, lazy D list)
//   lz_R[:, t] = A[:, rem_pix[t]] as complex128         (columns for P = G A_D)
//   bz = beta (y_eff_s - y_eff)                         (lagged data term)
struct EventJob {
  const int* rem_pix;
  int r;
  int* log_dst;
  int* lz_pix_dst;
  const float2* A;
  int64_t ld;
  double2* lz_R;
  double2* bz;
  const double2* y_eff_s;
  const double2* y_eff;
  double beta;
};

__global__ void event_prep_kernel(const __grid_constant__ Pack<EventJob> P) {
  pdl_enter();
  const EventJob& jb = P.j[blockIdx.y];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t t = t0; t < jb.r; t += stride) {
    const int p = jb.rem_pix[t];
    if (jb.log_dst) jb.log_dst[t] = p;
    if (jb.lz_pix_dst) jb.lz_pix_dst[t] = p;
  }
  if (jb.lz_R)
    for (int64_t e = t0; e < jb.ld * jb.r; e += stride) {
      const int u = (int)(e / jb.ld);
      const int64_t row = e % jb.ld;
      const float2 v = jb.A[row + (int64_t)jb.rem_pix[u] * jb.ld];
      jb.lz_R[e] = make_double2((double)v.x, (double)v.y);
    }
  if (jb.bz)
    for (int64_t i = t0; i < jb.ld; i += stride)
      jb.bz[i] = make_double2(jb.beta * (jb.y_eff_s[i].x - jb.y_eff[i].x), jb.beta * (jb.y_eff_s[i].y - jb.y_eff[i].y));
}

__global__ void iota_kernel(int* __restrict__ J, int n) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) J[i] = i;
}

// Gather x_full[J] -> x_hat (and zero a vector) etc.
__global__ void gather_kernel(const double2* __restrict__ src, const int* __restrict__ idx, int n, double2* __restrict__ dst) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// Portable (cos 2 pi t, sin 2 pi t), t in [0, 1): the exact operation sequence of
// scenario.sincos_turns -- octant reduction, Taylor polynomials on [0, pi/4] in
// Horner form, every op a separately rounded fp64 op (no FMA contraction) -- so
// the device operator is bitwise the host one (tests/test_gpu_parity.py).
__device__ __forceinline__ void sincos_turns(double t, double* c_out, double* s_out) {
  const double t8 = __dmul_rn(t, 8.0);
  const double o = floor(t8);
  const double f = __dsub_rn(t8, o);
  const int oi = (int)o;
  const double h = (oi & 1) ? __dsub_rn(1.0, f) : f;
  const double x = __dmul_rn(h, 0.7853981633974483);
  const double x2 = __dmul_rn(x, x);
  double p = 2.8114572543455206e-15;
  p = __dadd_rn(-7.647163731819816e-13, __dmul_rn(x2, p));
  p = __dadd_rn(1.6059043836821613e-10, __dmul_rn(x2, p));
  p = __dadd_rn(-2.505210838544172e-08, __dmul_rn(x2, p));
  p = __dadd_rn(2.7557319223985893e-06, __dmul_rn(x2, p));
  p = __dadd_rn(-0.0001984126984126984, __dmul_rn(x2, p));
  p = __dadd_rn(0.008333333333333333, __dmul_rn(x2, p));
  p = __dadd_rn(-0.16666666666666666, __dmul_rn(x2, p));
  const double sx = __dadd_rn(x, __dmul_rn(__dmul_rn(x, x2), p));
  double r = -1.5619206968586225e-16;
  r = __dadd_rn(4.779477332387385e-14, __dmul_rn(x2, r));
  r = __dadd_rn(-1.1470745597729725e-11, __dmul_rn(x2, r));
  r = __dadd_rn(2.08767569878681e-09, __dmul_rn(x2, r));
  r = __dadd_rn(-2.755731922398589e-07, __dmul_rn(x2, r));
  r = __dadd_rn(2.48015873015873e-05, __dmul_rn(x2, r));
  r = __dadd_rn(-0.001388888888888889, __dmul_rn(x2, r));
  r = __dadd_rn(0.041666666666666664, __dmul_rn(x2, r));
  r = __dadd_rn(-0.5, __dmul_rn(x2, r));
  const double cx = __dadd_rn(1.0, __dmul_rn(x2, r));
  const bool sw = ((oi + 1) >> 1) & 1;
  const double sa = sw ? cx : sx, ca = sw ? sx : cx;
  *s_out = (oi >= 4) ? -sa : sa;
  *c_out = (oi >= 2 && oi <= 5) ? -ca : ca;
}

// BASELINE dechirped-LFM operator generator: scenario.baseline_operator
// operation by operation (no FMA contraction), phases in turns; bitwise equal
// to the host generator.
__global__ void dechirp_kernel(float2* __restrict__ A, int64_t ld, int M, int K, int N,
                               const double* __restrict__ pix, const double* __restrict__ tx,
                               const double* __restrict__ rx, const double* __restrict__ turns,
                               double alpha, double fc, double t_step, double c_light) {
  pdl_enter();
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
  double t = __dadd_rn(cyc, turns[n]);
  t = __dsub_rn(t, floor(t));
  double s, c;
  sincos_turns(t, &c, &s);
  A[r + (int64_t)n * ld] = make_float2(__double2float_rn(c), __double2float_rn(s));
}

// The reference's own operator on the device: EchoKernel::entry
// (forward_model.hpp:64-71) assembled densely like ForwardOperator::dense
// (:91-114), row r = m K + k.  The delay and phase are the reference's
// expression evaluated operation by operation (no FMA contraction, the same
// order as scenario.echo_operator):
//   tau   = (|tx - p_n| + |rx_m - p_n|) / c
//   t     = k / fs - tau;  zero outside [0, T]
//   phase = ((-2 pi) fc) tau + ((pi alpha) t) t
// then std::polar(1, phase) -> CUDA's fp64 sincos (full range reduction),
// stored as complex64.  Entries equal the host generator's to within one
// fp32 rounding (tests/test_gpu_parity.py::test_device_echo_operator_*).
__global__ void echo_kernel(float2* __restrict__ A, int64_t ld, int M, int K, int N,
                            const double* __restrict__ pix, const double* __restrict__ tx,
                            const double* __restrict__ rx, double fc, double fs, double alpha, double T,
                            double c_light, double pi) {
  pdl_enter();
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
  const double t = __dsub_rn(__ddiv_rn((double)k, fs), tau);
  float2 out = make_float2(0.f, 0.f);
  if (!(t < 0.0 || t > T)) {
    const double carrier = __dmul_rn(__dmul_rn(-2.0 * pi, fc), tau);
    const double chirp = __dmul_rn(__dmul_rn(__dmul_rn(pi, alpha), t), t);
    double s, c;
    sincos(__dadd_rn(carrier, chirp), &s, &c);
    out = make_float2(__double2float_rn(c), __double2float_rn(s));
  }
  A[r + (int64_t)n * ld] = out;
}

}  // namespace radmm_dev
