// Standalone check of the hand-written tcgen05 int8 GEMM building block used by
// the Ozaki-sliced Gram (kernels_ozaki.cuh): C (int32) = A B^T with A (M x K)
// and B (N x K) int8, both K-major, against a CPU reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_i8_gemm_test tools/tc_i8_gemm_test.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2307_08606_b200/csrc/kernels_ozaki.cuh"

using namespace radmm_oz;

__global__ void __launch_bounds__(128, 1) test_gemm_kernel(const int8_t* A, const int8_t* B, int K, int64_t lda,
                                                           int64_t ldb, int32_t* C, int64_t ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TcI8Tile t;
  t.init(smem_raw, 1);
  const int m0 = blockIdx.y * kOzBM, n0 = blockIdx.x * kOzBN;
  t.run(A + (int64_t)m0 * lda, lda, B + (int64_t)n0 * ldb, ldb, K, 0, /*accumulate=*/false);
  t.wait_all();
  // epilogue: warp w owns rows 32w..32w+31 (TMEM lanes), 32 columns per load
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < kOzBN; c0 += 32) {
    uint32_t v[32];
    t.load32(0, warp, c0, v);
    for (int j = 0; j < 32; ++j) C[(int64_t)(m0 + 32 * warp + lane) * ldc + n0 + c0 + j] = (int32_t)v[j];
  }
  t.finish();
}

int main() {
  const int M = 256, N = 256, K = 1024;
  std::vector<int8_t> a((size_t)M * K), b((size_t)N * K);
  srand(1);
  for (auto& x : a) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : b) x = (int8_t)(rand() % 255 - 127);
  int8_t *da, *db;
  int32_t* dc;
  cudaMalloc(&da, a.size());
  cudaMalloc(&db, b.size());
  cudaMalloc(&dc, sizeof(int32_t) * M * N);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
  cudaMemset(dc, 0, sizeof(int32_t) * M * N);
  cudaFuncSetAttribute(test_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOzSmem);
  test_gemm_kernel<<<dim3(N / kOzBN, M / kOzBM), 128, kOzSmem>>>(da, db, K, K, K, dc, N);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<int32_t> c((size_t)M * N);
  cudaMemcpy(c.data(), dc, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int32_t r = 0;
      for (int k = 0; k < K; ++k) r += (int32_t)a[(size_t)i * K + k] * (int32_t)b[(size_t)j * K + k];
      if (r != c[(size_t)i * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): gpu %d ref %d\n", i, j, c[(size_t)i * N + j], r);
        ++bad;
      }
    }
  printf("mismatches: %ld of %d\n", bad, M * N);
  return bad ? 1 : 0;
}
