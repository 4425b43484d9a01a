// store bandwidth vs warps per SM (coalesced 16B stores, each warp writes 32 x 512 B rows)
#include <cuda_runtime.h>
#include <cstdio>
__global__ void st(uint4* out, int per_warp_kb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  uint4* base = out + wid * per_warp_kb * 64;  // per_warp_kb KB per warp
  for (int i = 0; i < per_warp_kb * 64; i += 32) base[i + lane] = make_uint4(i, lane, 1, 2);
}
__global__ void ld(const uint4* in, uint4* sink, int per_warp_kb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  const uint4* base = in + wid * per_warp_kb * 64;
  uint4 acc = make_uint4(0,0,0,0);
  for (int i = 0; i < per_warp_kb * 64; i += 32) { uint4 v = __ldcg(base + i + lane); acc.x ^= v.x; acc.y ^= v.y; }
  if (acc.x == 12345) sink[0] = acc;
}
int main() {
  const size_t total = 32ull << 20;  // 32 MB
  uint4* out; cudaMalloc(&out, total); uint4* sink; cudaMalloc(&sink, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int warps : {4, 8, 16, 32}) {
    const int nw = 148 * warps;
    const int kb = (int)(total / 1024 / nw);
    for (int mode = 0; mode < 2; ++mode) {
      float best = 1e9;
      for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a);
        if (mode == 0) st<<<148, warps * 32>>>(out, kb); else ld<<<148, warps * 32>>>(out, sink, kb);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (r > 2 && ms < best) best = ms;
      }
      printf("%s warps/SM %2d: %.2f us for %.1f MB -> %.0f GB/s\n", mode ? "load " : "store", warps, best * 1e3,
             148.0 * warps * kb / 1024.0, 148.0 * warps * kb * 1024 / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
