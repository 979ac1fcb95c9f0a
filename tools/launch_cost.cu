// Host cost of one kernel launch vs the size of its __grid_constant__ parameter
// block and the PDL attribute (tools/launch_cost.cu; nvcc -arch=sm_100a).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct P { char b[B]; };
template <int B> __global__ void k(const __grid_constant__ P<B> p) { if (threadIdx.x == 1000) printf("%d", p.b[0]); }
template <int B> double run(cudaStream_t s, bool pdl, int n) {
  P<B> p{};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k<B>, p);
  cudaStreamSynchronize(s);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&cfg, k<B>, p);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::steady_clock::now();
  printf("param %6d B pdl %d: host %.2f us/launch, total %.2f us/launch\n", B, pdl,
         std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
         std::chrono::duration<double, std::micro>(t2 - t0).count() / n);
  return 0;
}
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<256>(s, pdl, 2000); run<2048>(s, pdl, 2000); run<4096>(s, pdl, 2000);
    run<8192>(s, pdl, 2000); run<16384>(s, pdl, 2000);
  }
}
