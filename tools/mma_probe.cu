// tcgen05.mma issue/throughput probe (profiling helper, not product): one CTA
// per SM issues K-blocks of M=128 x N x K=64 (4 x K=16 instructions) from
// resident smem operands into one TMEM accumulator, committing each K-block to
// an mbarrier like the megakernel's ring, and reports cycles per K-block.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

__global__ void __launch_bounds__(128, 1) probe(int n_kb, int bn, int wait_each, int nacc, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const uint32_t sb = smem_u32(base);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[9];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(smem_u32(&bars[i]), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 256);
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
      const uint32_t a = sb + (s & 3) * 49152;
      const uint64_t ad = sw128_kmajor_desc(a), bd = sw128_kmajor_desc(a + 16384);
      if (wait_each && i >= 8) {  // like the ring: reuse slot s only after its last commit
        mbar_wait(smem_u32(&bars[s]), (par >> s) & 1);
        par ^= 1u << s;
      }
      // nacc independent accumulators (TMEM column blocks of bn) share the k-block
      for (int k = 0; k < 4; ++k)
        for (int j = 0; j < nacc; ++j)
          mma_bf16(tmem + j * bn, ad + 2 * k + j * 1024, bd + 2 * k, idesc, (i | k) != 0);
      mma_commit(smem_u32(&bars[s]));
    }
    // drain: one more commit tracks completion of every MMA issued so far
    mma_commit(smem_u32(&bars[8]));
    mbar_wait(smem_u32(&bars[8]), 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int bn : {64, 128, 256})
    for (int nacc : {1, 2, 4})
      for (int we : {1}) {
        if (bn * nacc > 256) continue;
        const int grid = 148;
        const int n = 512;
        probe<<<grid, 128, 200 * 1024>>>(n, bn, we, nacc, d);
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        const double flop = 2.0 * 128 * bn * 64 * nacc;
        printf("N=%3d x %d accumulators wait_each=%d: %.1f cycles per k-block (%.0f flop/clk/SM)\n",
               bn, nacc, we, (double)c / n, flop / ((double)c / n));
        fflush(stdout);
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
