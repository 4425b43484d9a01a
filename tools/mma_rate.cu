// tcgen05.mma throughput probe (profiling helper, not product).
// One CTA per SM; one thread issues MMAs of M=128 x N x K=16 (bf16 -> fp32)
// from smem operands that were zero-filled first. Variants:
//   0: n_kb k-blocks of 4 MMAs, ONE commit at the end (pure issue/execute rate)
//   1: a commit after every k-block, no waits
//   2: a commit after every k-block, wait for the commit of k-block i-8 (ring of 8)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

__global__ void __launch_bounds__(128, 1) probe(int n_kb, int bn, int variant, int swz,
                                                long long* cycles, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const uint32_t sb = smem_u32(base);
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[9];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_bf16_f32(128, bn);
    uint32_t par = 0;
    const long long t0 = clock64();
    for (int i = 0; i < n_kb; ++i) {
      const int s = i & 7;
      const uint32_t a = sb + (s & 3) * 40960;
      uint64_t ad, bd;
      if (swz == 128) {
        ad = sw128_kmajor_desc(a);
        bd = sw128_kmajor_desc(a + 16384);
      } else {
        ad = (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (4ull << 61);
        bd = ad + (16384 >> 4);
      }
      if (variant == 2 && i >= 8) {
        mbar_wait(smem_u32(&bars[s]), (par >> s) & 1);
        par ^= 1u << s;
      }
      const int step = swz == 128 ? 2 : 2;
      for (int k = 0; k < 4; ++k)
        for (int j = 0; j < nacc; ++j)
          mma_bf16(tmem + j * bn, ad + step * k + j * 512, bd + step * k, idesc, (i | k) != 0);
      if (variant >= 1) mma_commit(smem_u32(&bars[s]));
    }
    mma_commit(smem_u32(&bars[8]));
    mbar_wait(smem_u32(&bars[8]), 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  for (int swz : {128})
    for (int grid : {148})
      for (int variant : {0, 2})
        for (int nacc : {1, 2, 4})
        for (int bn : {64, 128, 256}) {
          if (nacc * bn > 512) continue;
          const int n = 2048;
          probe<<<grid, 128, 170 * 1024>>>(8, bn, variant, swz, d, nacc);  // warm
          probe<<<grid, 128, 170 * 1024>>>(n, bn, variant, swz, d, nacc);
          long long c = 0;
          cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          const double flop = 2.0 * 128 * bn * 64 * nacc;
          printf("nacc %d swz %3d grid %3d variant %d N=%3d: %7.1f cycles per k-block (%5.0f flop/clk/SM, ideal %4.0f cyc)\n",
                 nacc, swz, grid, variant, bn, (double)c / n, flop / ((double)c / n), flop / 8192);
          fflush(stdout);
        }
  return 0;
}
