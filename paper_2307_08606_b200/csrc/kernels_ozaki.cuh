// kernels_ozaki.cuh: int8 GEMM tile on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, int32 accumulators in tensor memory), the building
// block of the Ozaki-sliced capacitance Gram.
//
//   D[128 x 128] (int32, TMEM) += A[128 x K] . B[128 x K]^T   (int8, both K-major)
//
// Operands stream through a kOzStages-deep shared ring with cp.async; each
// 128-row x 128-byte stage is stored in the canonical K-major SWIZZLE_128B
// layout (8-row x 128-byte atoms, 16-byte chunk c of row r at c ^ (r & 7)), so
// one smem descriptor per stage serves four K = 32 MMAs by advancing its
// start address 32 bytes at a time.  One thread issues the MMAs; each stage's
// MMAs commit to that stage's mbarrier, which releases the slot for the next
// copy.  Exact: int8 x int8 products, int32 sums (|sum| < 2^31 for
// K < 2^17 with operands in [-127, 127]).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace radmm_oz {

// Programmatic dependent launch (see radmm_dev::pdl_enter in kernels_async.cuh):
// wait for the predecessor grid, then let the successor launch.
__device__ __forceinline__ void oz_pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int kOzBM = 128, kOzBN = 128, kOzBK = 128, kOzStages = 4;
constexpr int kOzStageBytes = (kOzBM + kOzBN) * kOzBK;  // 32 KB
constexpr size_t kOzSmem = (size_t)kOzStages * kOzStageBytes + 1024 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void oz_cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void oz_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void oz_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void oz_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void oz_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// SWIZZLE_128B K-major smem descriptor (cute UMMA::SmemDescriptor layout):
// start >> 4 in [0,14), LBO (ignored for swizzled K-major) = 1, SBO = 1024 B
// between 8-row groups, version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// kind::i8 instruction descriptor: D = S32, A = B = signed int8, both
// K-major, N = 128, M = 128.
constexpr uint32_t kOzIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kOzBN >> 3) << 17) |
                              ((uint32_t)(kOzBM >> 4) << 24);

struct TcI8Tile {
  uint8_t* ring;       // 1024-aligned: kOzStages x (A 16 KB | B 16 KB)
  uint64_t* bar;       // kOzStages stage-release barriers
  uint32_t tmem;       // accumulator base (column 0 of lane 0)
  uint32_t ncols;
  uint32_t uses;       // stages issued so far (ring position / barrier phases)

  // n_acc accumulators of 128 columns each (TMEM allocation: power of two)
  __device__ void init(uint8_t* smem_raw, int n_acc) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    ring = base;
    bar = reinterpret_cast<uint64_t*>(base + (size_t)kOzStages * kOzStageBytes);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + kOzStages);
    ncols = n_acc <= 1 ? 128u : n_acc <= 2 ? 256u : 512u;
    uses = 0;
    if (threadIdx.x == 0) {
      for (int s = 0; s < kOzStages; ++s) oz_mbar_init(&bar[s], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if ((threadIdx.x >> 5) == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                   "r"(ncols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tmem = *slot;
  }

  // stage copy: 8 threads per 128-byte row (coalesced), 16 rows per pass
  __device__ void load(int s, const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int kb) {
    const int t = threadIdx.x, c = t & 7;
    const uint32_t a_s = smem_u32(ring + (size_t)s * kOzStageBytes), b_s = a_s + kOzBM * kOzBK;
#pragma unroll
    for (int p = 0; p < kOzBM / 16; ++p) {
      const int r = (t >> 3) + 16 * p;
      const uint32_t off = r * kOzBK + ((c ^ (r & 7)) << 4);
      oz_cp16(a_s + off, A + (int64_t)r * lda + (int64_t)kb * kOzBK + c * 16);
      oz_cp16(b_s + off, B + (int64_t)r * ldb + (int64_t)kb * kOzBK + c * 16);
    }
  }

  // D[acc] (+)= A B^T over K (a multiple of kOzBK); `accumulate` false starts
  // the accumulator at zero.  Blocks all 128 threads of the CTA.
  __device__ void run(const int8_t* A, int64_t lda, const int8_t* B, int64_t ldb, int K, int acc, bool accumulate) {
    const int nk = K / kOzBK;
#pragma unroll
    for (int p = 0; p < kOzStages - 1; ++p) {
      if (p < nk) {
        const uint32_t u = uses + p;
        if (u >= kOzStages) oz_mbar_wait(&bar[u % kOzStages], ((u / kOzStages) - 1) & 1);
        load(u % kOzStages, A, lda, B, ldb, p);
      }
      oz_commit();
    }
    for (int kb = 0; kb < nk; ++kb) {
      const int ld_kb = kb + kOzStages - 1;
      if (ld_kb < nk) {
        const uint32_t u = uses + ld_kb;
        if (u >= kOzStages) oz_mbar_wait(&bar[u % kOzStages], ((u / kOzStages) - 1) & 1);
        load(u % kOzStages, A, lda, B, ldb, ld_kb);
      }
      oz_commit();
      oz_wait<kOzStages - 1>();  // this thread's copies of stage kb landed
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t u = uses + kb;
        const uint32_t a_s = smem_u32(ring + (size_t)(u % kOzStages) * kOzStageBytes), b_s = a_s + kOzBM * kOzBK;
#pragma unroll
        for (int k = 0; k < kOzBK / 32; ++k) {
          const uint64_t ad = oz_desc(a_s + 32 * k), bd = oz_desc(b_s + 32 * k);
          const uint32_t en = (accumulate || kb > 0 || k > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(
                  tmem + (uint32_t)acc * 128u),
              "l"(ad), "l"(bd), "r"(kOzIdesc), "r"(en), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
              : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar[u % kOzStages]))
                     : "memory");
      }
    }
    uses += nk;
  }

  // wait for every issued MMA (the last stage's barrier covers all earlier ones)
  __device__ void wait_all() {
    if (uses > 0) {
      const uint32_t u = uses - 1;
      oz_mbar_wait(&bar[u % kOzStages], (u / kOzStages) & 1);
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }

  // 32 consecutive accumulator columns of the warp's 32 rows (lanes 32w..32w+31)
  __device__ void load32(int acc, int warp, int col0, uint32_t (&v)[32]) {
    const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)acc * 128u + (uint32_t)col0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  }

  __device__ void finish() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
  }
};

// ---------------------------------------------------------------------------
// Ozaki-sliced capacitance Gram  C = A_J A_J^H  (complex64 A, exact-to-fp64
// level products on the int8 tensor cores).
//
// Row r of A_J is scaled by 2^-e_r (e_r: exponent of the row's largest
// |re|, |im|, so |v| < 1) and split into kOzSlices int8 slices,
//   v = sum_{s=1..S} d_s 2^{-7s},  d_s in [-127, 127]  (truncation: exact
//   residuals, |v - sum| < 2^{-7S}),
// stored K-major with the real and imaginary parts side by side:
//   P_s = [Re d_s | Im d_s],  Q_s = [Im d_s | -Re d_s]   (rows x 2N bytes),
// so that for each slice pair (s1, s2)
//   Re(A A^H) part = P_s1 P_s2^T,  Im part = Q_s1 P_s2^T   (int32, exact).
// Pairs with s1 + s2 <= kOzSlices + 3 are kept: every complex64 entry whose
// |re|, |im| lies within 2^-25 of its row maximum is represented exactly by
// its 7 slices (24-bit mantissa), and the dropped pairs are below 2^-56
// relative per product -- so C matches an fp64 Gram to ~1e-16 relative, which
// the KM-space refinement of the dual solve needs (its residual uses this C;
// a 6-slice / s1 + s2 <= 7 Gram left ~2^-42 and cost three decades of solve
// accuracy).  oz_combine_kernel sums the pairs in a
// fixed order in fp64, scales by 2^{e_i + e_j} and writes the lower tiles
// with an exact conjugate mirror, like gram_dmma_kernel.
// ---------------------------------------------------------------------------
constexpr int kOzSlices = 7;
constexpr int kOzMaxSum = kOzSlices + 3;
constexpr int oz_pair_count() {
  int n = 0;
  for (int t = 2; t <= kOzMaxSum; ++t)
    for (int s1 = 1; s1 <= kOzSlices; ++s1)
      if (t - s1 >= 1 && t - s1 <= kOzSlices) ++n;
  return n;
}
constexpr int kOzPairs = oz_pair_count();  // 39

__host__ __device__ inline void oz_pair(int p, int& s1, int& s2) {
  // pairs ordered by t = s1 + s2 (largest contributions first), then s1
  for (int t = 2; t <= kOzMaxSum; ++t)
    for (int a = 1; a <= kOzSlices; ++a) {
      const int b = t - a;
      if (b < 1 || b > kOzSlices) continue;
      if (p-- == 0) {
        s1 = a;
        s2 = b;
        return;
      }
    }
  s1 = s2 = 1;
}

// row maxima of |re|, |im| over the listed columns (float bits: order-preserving
// for non-negative floats, so atomicMax on the bits is exact)
__global__ void oz_rowmax_kernel(const float2* __restrict__ A, int64_t ld, int rows, const int* __restrict__ J, int n,
                                 unsigned* __restrict__ rowmax) {
  oz_pdl_enter();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int per = (n + gridDim.y - 1) / gridDim.y;
  const int c0 = blockIdx.y * per, c1 = min(n, c0 + per);
  float m = 0.f;
  for (int c = c0; c < c1; ++c) {
    const float2 a = A[r + (int64_t)(J ? J[c] : c) * ld];
    m = fmaxf(m, fmaxf(fabsf(a.x), fabsf(a.y)));
  }
  atomicMax(rowmax + r, __float_as_uint(m));
}

// slices of a 32-column x 64-row block, transposed through shared memory so
// both the column-major read and the K-major writes are coalesced
__global__ void __launch_bounds__(256) oz_slice_kernel(const float2* __restrict__ A, int64_t ld, int rows,
                                                      const int* __restrict__ J, int n, int npad,
                                                      const unsigned* __restrict__ rowmax, int8_t* __restrict__ P,
                                                      int8_t* __restrict__ Q, int64_t slice_stride, int col0) {
  // columns col0 .. col0 + n of the list (a pixel chunk of the chunked Gram;
  // col0 = 0, n = all for the one-pass Gram) land in slice columns 0 .. n
  oz_pdl_enter();
  __shared__ int8_t sre[kOzSlices][64][33], sim[kOzSlices][64][33];
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 32;
  const int tr = threadIdx.x & 63, tq = threadIdx.x >> 6;  // row in tile, column phase
  const int r = r0 + tr;
  int e = 0;
  if (r < rows) {
    const float m = __uint_as_float(rowmax[r]);
    e = m > 0.f ? ilogbf(m) + 1 : 0;
  }
  for (int cc = tq; cc < 32; cc += 4) {
    const int c = c0 + cc;
    double vr = 0.0, vi = 0.0;
    if (r < rows && c < n) {
      const float2 a = A[r + (int64_t)(J ? J[col0 + c] : col0 + c) * ld];
      vr = ldexp((double)a.x, -e);
      vi = ldexp((double)a.y, -e);
    }
#pragma unroll
    for (int sl = 0; sl < kOzSlices; ++sl) {
      const double dr = trunc(vr * 128.0), di = trunc(vi * 128.0);  // exact: |v| < 1
      sre[sl][tr][cc] = (int8_t)dr;
      sim[sl][tr][cc] = (int8_t)di;
      vr = vr * 128.0 - dr;  // exact remainder, |.| < 1
      vi = vi * 128.0 - di;
    }
  }
  __syncthreads();
  // write: row rr, 32 consecutive columns per slice (re half, im half); rows
  // are npad long per half (zero columns beyond n stay as memset)
  for (int e2 = threadIdx.x; e2 < 64 * 32; e2 += 256) {
    const int rr = e2 >> 5, cc = e2 & 31, row = r0 + rr, c = c0 + cc;
    if (row >= rows || c >= n) continue;
#pragma unroll
    for (int sl = 0; sl < kOzSlices; ++sl) {
      int8_t* Pr = P + sl * slice_stride + (int64_t)row * 2 * npad;
      int8_t* Qr = Q + sl * slice_stride + (int64_t)row * 2 * npad;
      const int8_t re = sre[sl][rr][cc], im = sim[sl][rr][cc];
      Pr[c] = re;
      Pr[npad + c] = im;
      if (Q) {  // the chunked Gram needs no negated copy
        Qr[c] = im;
        Qr[npad + c] = (int8_t)(-re);
      }
    }
  }
}

// One CTA per (lower 128 x 128 tile, slice pair): Re and Im int32 blocks of
// the pair to R[tile][pair][part][128][128] (rows 128 apart in the tile).
__global__ void __launch_bounds__(128, 1) oz_gram_pairs_kernel(const int8_t* __restrict__ P,
                                                              const int8_t* __restrict__ Q, int64_t slice_stride,
                                                              int rows, int kdim, int32_t* __restrict__ R) {
  oz_pdl_enter();
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  int tile = blockIdx.x, I = 0;
  while (tile > I) {
    tile -= I + 1;
    ++I;
  }
  const int Jt = tile, pair = blockIdx.y;
  int s1, s2;
  oz_pair(pair, s1, s2);
  const int64_t ldk = kdim;  // bytes per slice row
  const int m0 = I * kOzBM, n0 = Jt * kOzBN;
  TcI8Tile t;
  t.init(oz_smem, 2);
  const int8_t* Pa = P + (s1 - 1) * slice_stride + (int64_t)m0 * ldk;
  const int8_t* Qa = Q + (s1 - 1) * slice_stride + (int64_t)m0 * ldk;
  const int8_t* Pb = P + (s2 - 1) * slice_stride + (int64_t)n0 * ldk;
  t.run(Pa, ldk, Pb, ldk, kdim, 0, false);
  t.run(Qa, ldk, Pb, ldk, kdim, 1, false);
  t.wait_all();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* out = R + ((int64_t)blockIdx.x * kOzPairs + pair) * 2 * kOzBM * kOzBN;
  for (int part = 0; part < 2; ++part)
    for (int c0 = 0; c0 < kOzBN; c0 += 32) {
      uint32_t v[32];
      t.load32(part, warp, c0, v);
      int4* dst = reinterpret_cast<int4*>(out + (int64_t)part * kOzBM * kOzBN + (int64_t)(32 * warp + lane) * kOzBN + c0);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2], (int)v[4 * q + 3]);
    }
  t.finish();
}

// TMA + warp-specialised variant of oz_gram_pairs_kernel (default): the
// slices are read by cp.async.bulk.tensor through SWIZZLE_128B tensor maps
// (the hardware writes the canonical layout the descriptors expect), one
// elected thread of warp 0 produces, one of warp 1 issues the MMAs, and each
// stage carries both A operands (P_s1 and Q_s1 rows of tile I) with one
// shared B (P_s2 rows of tile J): Re and Im accumulate together.
constexpr int kOzTStages = 4;
constexpr int kOzTStageBytes = 3 * kOzBM * kOzBK;  // A_P | A_Q | B, 16 KB each
constexpr size_t kOzTSmem = (size_t)kOzTStages * kOzTStageBytes + 1024 + 256;

__device__ __forceinline__ void oz_tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) oz_gram_pairs_tma_kernel(const __grid_constant__ CUtensorMap tP,
                                                                  const __grid_constant__ CUtensorMap tQ,
                                                                  int rows_pad, int kdim, int32_t* __restrict__ R) {
  oz_pdl_enter();
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)kOzTStages * kOzTStageBytes);
  uint64_t* empty = full + kOzTStages;
  uint64_t* done = empty + kOzTStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  int tile = blockIdx.x, I = 0;
  while (tile > I) {
    tile -= I + 1;
    ++I;
  }
  const int Jt = tile, pair = blockIdx.y;
  int s1, s2;
  oz_pair(pair, s1, s2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kOzTStages; ++st) {
      oz_mbar_init(&full[st], 1);
      oz_mbar_init(&empty[st], 1);
    }
    oz_mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int nk = kdim / kOzBK;
  const int ya = (s1 - 1) * rows_pad + I * kOzBM, yb = (s2 - 1) * rows_pad + Jt * kOzBN;
  if (warp == 0 && lane == 0) {  // producer
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % kOzTStages;
      if (kb >= kOzTStages) oz_mbar_wait(&empty[st], ((kb / kOzTStages) - 1) & 1);
      const uint32_t sa = smem_u32(base + (size_t)st * kOzTStageBytes), fb = smem_u32(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(kOzTStageBytes)
                   : "memory");
      oz_tma_2d(sa, &tP, kb * kOzBK, ya, fb);
      oz_tma_2d(sa + kOzBM * kOzBK, &tQ, kb * kOzBK, ya, fb);
      oz_tma_2d(sa + 2 * kOzBM * kOzBK, &tP, kb * kOzBK, yb, fb);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % kOzTStages;
      oz_mbar_wait(&full[st], (kb / kOzTStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = smem_u32(base + (size_t)st * kOzTStageBytes);
#pragma unroll
      for (int k = 0; k < kOzBK / 32; ++k) {
        const uint32_t en = (kb > 0 || k > 0) ? 1u : 0u;
        const uint64_t bd = oz_desc(sa + 2 * kOzBM * kOzBK + 32 * k);
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const uint64_t ad = oz_desc(sa + part * kOzBM * kOzBK + 32 * k);
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(
                  tmem + (uint32_t)part * 128u),
              "l"(ad), "l"(bd), "r"(kOzIdesc), "r"(en), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
              : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&empty[st]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(done))
                 : "memory");
  }
  oz_mbar_wait(done, 0);
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  int32_t* out = R + ((int64_t)blockIdx.x * kOzPairs + pair) * 2 * kOzBM * kOzBN;
  for (int part = 0; part < 2; ++part)
    for (int c0 = 0; c0 < kOzBN; c0 += 32) {
      uint32_t v[32];
      const uint32_t addr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)part * 128u + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      int4* dst =
          reinterpret_cast<int4*>(out + (int64_t)part * kOzBM * kOzBN + (int64_t)(32 * warp + lane) * kOzBN + c0);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = make_int4((int)v[4 * q], (int)v[4 * q + 1], (int)v[4 * q + 2], (int)v[4 * q + 3]);
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

// C[i, j] (i >= j, lower tiles) = mu 2^{e_i + e_j} sum_pairs 2^{-7(s1+s2)} (R_re + i R_im)
// (+ beta on the diagonal, exact real), mirrored conjugate to C[j, i].
__global__ void oz_combine_kernel(const int32_t* __restrict__ R, const unsigned* __restrict__ rowmax, int rows,
                                  double2* __restrict__ C, int64_t ldc, double mu, double beta) {
  oz_pdl_enter();
  const int tile = blockIdx.y;
  int t = tile, I = 0;
  while (t > I) {
    t -= I + 1;
    ++I;
  }
  const int Jt = t;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // element in the 128 x 128 tile
  if (e >= kOzBM * kOzBN) return;
  const int ii = e / kOzBN, jj = e % kOzBN, i = I * kOzBM + ii, j = Jt * kOzBN + jj;
  if (i >= rows || j >= rows || i < j) return;
  const int32_t* base = R + (int64_t)tile * kOzPairs * 2 * kOzBM * kOzBN + e;
  double re = 0.0, im = 0.0;
  for (int p = 0; p < kOzPairs; ++p) {
    int s1, s2;
    oz_pair(p, s1, s2);
    const double sc = ldexp(1.0, -7 * (s1 + s2));
    re += sc * (double)base[(int64_t)p * 2 * kOzBM * kOzBN];
    im += sc * (double)base[(int64_t)p * 2 * kOzBM * kOzBN + kOzBM * kOzBN];
  }
  const float mi = __uint_as_float(rowmax[i]), mj = __uint_as_float(rowmax[j]);
  const int ei = mi > 0.f ? ilogbf(mi) + 1 : 0, ej = mj > 0.f ? ilogbf(mj) + 1 : 0;
  re = ldexp(re, ei + ej);
  im = ldexp(im, ei + ej);
  double2 o = make_double2(mu * re, mu * im);
  if (i == j) {
    o.x += beta;
    o.y = 0.0;
  }
  C[i + (int64_t)j * ldc] = o;
  if (i != j) C[j + (int64_t)i * ldc] = make_double2(o.x, -o.y);
}

// ---------------------------------------------------------------------------
// Chunked Gram for problems whose one-pass scratch (all slices + one int32
// block per tile and pair: config 3, 26 GB per sensor) does not fit next to
// the resident operators, and whose one-pass pair kernel is bound by the
// L2 -> SM operand feed (48 KB per 4.2 M MACs; measured 47% tensor pipe at
// config-3 shapes).  The pixels are processed kOzChunk at a time: a chunk is
// sliced into a small scratch holding only P_s = [Re d_s | Im d_s]
// (7 x rows x 2*kOzChunk bytes), and oz_gram_chunk_kernel -- ONE CTA per lower
// 128 x 128 tile -- walks all 39 slice pairs of the chunk.  A stage carries
// the Re and Im halves of both operands (4 x 16 KB) and feeds FOUR real
// products,
//   Re += Re_a Re_b^T + Im_a Im_b^T,  X += Im_a Re_b^T,  Y += Re_a Im_b^T,
//   Im = X - Y  (in the epilogue: no negated slices are stored),
// i.e. 64 KB per 8.4 M MACs.  Pairs with the same t = s1 + s2 carry the same
// weight 2^-7t, so they accumulate in the same TMEM accumulators (exact: at
// most 7 pairs x 2*kOzChunk x 127^2 < 2^31); after each of the 9 weight
// groups the four epilogue warps add the group's int32 blocks, scaled, to
// fp64 accumulators in C (chunk-major, then t ascending: a fixed order).
// oz_gram_finish_kernel then scales by mu 2^{e_i+e_j}, adds beta and mirrors,
// like oz_combine_kernel.
// ---------------------------------------------------------------------------
constexpr int kOzChunk = 8192;  // pixels per chunk: 7 * 2 * 8192 * 127^2 = 1.85e9 < 2^31
constexpr int kOzGroups = kOzMaxSum - 1;  // t = 2 .. kOzMaxSum
constexpr int kOzCThreads = 192;  // warps 0-3: epilogue (TMEM lanes 32w..), warp 4: TMA producer, warp 5: MMA issuer
constexpr int kOzCStages = 3;
constexpr int kOzBand = 12;  // tile rows per band of the launch order
constexpr int kOzCStageBytes = 4 * kOzBM * kOzBK;  // Re_a | Im_a | Re_b | Im_b, 16 KB each
constexpr size_t kOzCSmem = (size_t)kOzCStages * kOzCStageBytes + 1024 + 256;

__device__ __forceinline__ void oz_mma_i8(uint32_t d, uint64_t ad, uint64_t bd, uint32_t en) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
      "l"(ad), "l"(bd), "r"(kOzIdesc), "r"(en), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

__device__ __forceinline__ void oz_tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

// tP: 2-D int8 map over the chunk's P slices, [kOzSlices * rows_pad] rows x
// (2 * half) bytes; half = chunk columns (a multiple of kOzBK): Re at byte
// columns [0, half), Im at [half, 2 half).
__global__ void __launch_bounds__(kOzCThreads, 1) oz_gram_chunk_kernel(const __grid_constant__ CUtensorMap tP,
                                                                      int rows_pad, int half, int rows,
                                                                      double2* __restrict__ C, int64_t ldc) {
  oz_pdl_enter();
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)kOzCStages * kOzCStageBytes);
  uint64_t* empty = full + kOzCStages;
  uint64_t* accfull = empty + kOzCStages;  // a weight group's MMAs are complete
  uint64_t* accfree = accfull + 1;         // the epilogue has drained the accumulators
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accfree + 1);
  // Tile order: bands of kOzBand tile rows, column by column inside a band, so
  // the ~148 CTAs resident together cover a ~12 x 12 block of tiles and share
  // 12 + 12 row blocks of slices through L2 (row-major order: 3 + 40).
  int I, Jt;
  {
    const int T = rows_pad / kOzBM;
    int idx = blockIdx.x, r0 = 0, h = min(kOzBand, T);
    for (;;) {  // band [r0, r0 + h): sum_{I in band} (I + 1) tiles
      const int cnt = h * r0 + h * (h + 1) / 2;
      if (idx < cnt) break;
      idx -= cnt;
      r0 += h;
      h = min(kOzBand, T - r0);
    }
    const int full = (r0 + 1) * h;  // columns 0 .. r0: every row of the band
    if (idx < full) {
      Jt = idx / h;
      I = r0 + idx % h;
    } else {  // columns r0 + 1 ..: rows Jt .. r0 + h - 1
      idx -= full;
      int col = 1;
      while (idx >= h - col) {
        idx -= h - col;
        ++col;
      }
      Jt = r0 + col;
      I = Jt + idx;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kOzCStages; ++st) {
      oz_mbar_init(&full[st], 1);
      oz_mbar_init(&empty[st], 1);
    }
    oz_mbar_init(accfull, 1);
    oz_mbar_init(accfree, 4);  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const int nk = half / kOzBK;
  if (warp == 4 && lane == 0) {  // producer: every (group, pair, k block) in order
    uint32_t it = 0;
    for (int t = 2; t <= kOzMaxSum; ++t)
      for (int s1 = 1; s1 <= kOzSlices; ++s1) {
        const int s2 = t - s1;
        if (s2 < 1 || s2 > kOzSlices) continue;
        const int ya = (s1 - 1) * rows_pad + I * kOzBM, yb = (s2 - 1) * rows_pad + Jt * kOzBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t st = it % kOzCStages;
          if (it >= (uint32_t)kOzCStages) oz_mbar_wait(&empty[st], ((it / kOzCStages) - 1) & 1);
          const uint32_t sa = smem_u32(base + (size_t)st * kOzCStageBytes), fb = smem_u32(&full[st]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(kOzCStageBytes)
                       : "memory");
          oz_tma_2d(sa, &tP, kb * kOzBK, ya, fb);
          oz_tma_2d(sa + kOzBM * kOzBK, &tP, half + kb * kOzBK, ya, fb);
          oz_tma_2d(sa + 2 * kOzBM * kOzBK, &tP, kb * kOzBK, yb, fb);
          oz_tma_2d(sa + 3 * kOzBM * kOzBK, &tP, half + kb * kOzBK, yb, fb);
        }
      }
  } else if (warp == 5 && lane == 0) {  // MMA issuer
    uint32_t it = 0;
    int g = 0;
    for (int t = 2; t <= kOzMaxSum; ++t, ++g) {
      if (g >= 1) {  // the epilogue has read the previous group
        oz_mbar_wait(accfree, (g - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      bool fresh = true;  // the group's first MMAs overwrite the accumulators
      for (int s1 = 1; s1 <= kOzSlices; ++s1) {
        const int s2 = t - s1;
        if (s2 < 1 || s2 > kOzSlices) continue;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t st = it % kOzCStages;
          oz_mbar_wait(&full[st], (it / kOzCStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(base + (size_t)st * kOzCStageBytes);
#pragma unroll
          for (int k = 0; k < kOzBK / 32; ++k) {
            const uint32_t first = (fresh && k == 0) ? 0u : 1u;
            const uint64_t re_a = oz_desc(sa + 32 * k), im_a = oz_desc(sa + kOzBM * kOzBK + 32 * k);
            const uint64_t re_b = oz_desc(sa + 2 * kOzBM * kOzBK + 32 * k), im_b = oz_desc(sa + 3 * kOzBM * kOzBK + 32 * k);
            oz_mma_i8(tmem, re_a, re_b, first);         // Re += Re_a Re_b^T
            oz_mma_i8(tmem, im_a, im_b, 1u);            // Re += Im_a Im_b^T
            oz_mma_i8(tmem + 128u, im_a, re_b, first);  // X  += Im_a Re_b^T
            oz_mma_i8(tmem + 256u, re_a, im_b, first);  // Y  += Re_a Im_b^T
          }
          fresh = false;
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(accfull))
                   : "memory");
    }
  } else if (warp < 4) {  // epilogue: row i of the tile per thread
    const int i = I * kOzBM + 32 * warp + lane;
    for (int g = 0; g < kOzGroups; ++g) {
      oz_mbar_wait(accfull, g & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const double sc = __longlong_as_double((long long)(1023 - 7 * (g + 2)) << 52);  // 2^-7t
      for (int c0 = 0; c0 < kOzBN; c0 += 16) {
        uint32_t vr[16], vx[16], vy[16];
        const uint32_t ar = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
        oz_tmem_ld16(ar, vr);
        oz_tmem_ld16(ar + 128u, vx);
        oz_tmem_ld16(ar + 256u, vy);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // a warp's 32 rows are consecutive in a column of C: 512-byte accesses
        double2 acc[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = Jt * kOzBN + c0 + jj;
          acc[jj] = (i < rows && j < rows) ? C[i + (int64_t)j * ldc] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = Jt * kOzBN + c0 + jj;
          if (i < rows && j < rows)  // |X - Y| < 2^31: the difference is exact in int64, then in fp64
            C[i + (int64_t)j * ldc] =
                make_double2(fma(sc, (double)(int)vr[jj], acc[jj].x),
                             fma(sc, (double)((long long)(int)vx[jj] - (long long)(int)vy[jj]), acc[jj].y));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(accfree)) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// C[i, j] (i >= j) <- mu 2^{e_i + e_j} acc[i, j] (+ beta on the diagonal, exact
// real), mirrored conjugate to C[j, i]; acc is what oz_gram_chunk_kernel left.
__global__ void oz_gram_finish_kernel(const unsigned* __restrict__ rowmax, int rows, double2* __restrict__ C,
                                      int64_t ldc, double mu, double beta) {
  oz_pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= rows || j >= rows || i < j) return;
  const float mi = __uint_as_float(rowmax[i]), mj = __uint_as_float(rowmax[j]);
  const int ei = mi > 0.f ? ilogbf(mi) + 1 : 0, ej = mj > 0.f ? ilogbf(mj) + 1 : 0;
  const double2 a = C[i + (int64_t)j * ldc];
  double2 o = make_double2(mu * ldexp(a.x, ei + ej), mu * ldexp(a.y, ei + ej));
  if (i == j) {
    o.x += beta;
    o.y = 0.0;
  }
  C[i + (int64_t)j * ldc] = o;
  if (i != j) C[j + (int64_t)i * ldc] = make_double2(o.x, -o.y);
}

}  // namespace radmm_oz
