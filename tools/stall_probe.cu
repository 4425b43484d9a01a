// Platform stall probe (profiling helper): back-to-back launches of a fixed-work kernel on
// all SMs (one CTA per SM, ~600 us of FMA work), each recording its own %globaltimer span;
// reports the distribution. Outliers here are not the megakernel's.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void work(int iters, unsigned long long* span, float* sink) {
  __shared__ unsigned long long t0;
  if (threadIdx.x == 0) t0 = gt();
  __syncthreads();
  float a = threadIdx.x, b = 1.0001f;
  for (int i = 0; i < iters; ++i) a = a * b + 0.5f;
  if (a == 12345.f) sink[0] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(&span[0], t0);
    atomicMax(&span[1], gt());
  }
}
int main() {
  const int n = 20000;
  unsigned long long* spans;
  cudaMalloc(&spans, sizeof(unsigned long long) * 2 * n);
  std::vector<unsigned long long> init(2 * n);
  for (int i = 0; i < n; ++i) { init[2 * i] = ~0ull; init[2 * i + 1] = 0; }
  cudaMemcpy(spans, init.data(), sizeof(unsigned long long) * 2 * n, cudaMemcpyHostToDevice);
  float* sink;
  cudaMalloc(&sink, 4);
  for (int i = 0; i < n; ++i) work<<<148, 256>>>(150000, spans + 2 * i, sink);
  cudaDeviceSynchronize();
  cudaMemcpy(init.data(), spans, sizeof(unsigned long long) * 2 * n, cudaMemcpyDeviceToHost);
  std::vector<double> us(n);
  for (int i = 0; i < n; ++i) us[i] = (init[2 * i + 1] - init[2 * i]) / 1e3;
  std::vector<double> s = us;
  std::sort(s.begin(), s.end());
  int big = 0;
  for (double v : us) big += v > 1.5 * s[n / 2];
  printf("fixed-work kernel: p50 %.1f us, p99 %.1f, p99.99 %.1f, max %.1f; %d of %d > 1.5 x p50\n",
         s[n / 2], s[(int)(n * 0.99)], s[(int)(n * 0.9999)], s[n - 1], big, n);
  return 0;
}
