// tcgen05.mma issue-rate probe (profiling helper, not product): a whole warp
// enters the issue loop, one elected lane issues; descriptors are warp-uniform
// and the inner block is fully unrolled, so the SASS is UTCHMMA back to back.
// Template parameters fix N and the number of independent accumulators.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

template <int BN, int NACC, int SAME_A, int EXTRA>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const uint32_t sb = smem_u32(base);
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bars[3];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bars[0]), 1);
    mbar_init(smem_u32(&bars[1]), 1);
    mbar_init(smem_u32(&bars[2]), 1);
    mbar_arrive(smem_u32(&bars[1]));  // phase 0 of bars[1] complete
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
    const uint64_t ad = sw128_kmajor_desc(sb);
    const uint64_t bd = sw128_kmajor_desc(sb + 65536);
    const long long t0 = clock64();
    int slot = 0;
    for (int i = 0; i < iters; ++i) {
      if (EXTRA & 2) mbar_wait(smem_u32(&bars[1]), 0);
      if (EXTRA & 4) tc_fence_after();
      uint64_t a2 = ad, b2 = bd;
      if (EXTRA & 8) {
        a2 = sw128_kmajor_desc(sb + slot * 24576);
        b2 = sw128_kmajor_desc(sb + slot * 24576 + 16384);
        if (++slot == 4) slot = 0;
      }
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < NACC; ++j)
            mma_bf16(tmem + j * BN, a2 + 2 * k + (SAME_A ? 0 : j * 1024), b2 + 2 * k, idesc, 1);
        if (EXTRA & 1) mma_commit(smem_u32(&bars[2]));
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(smem_u32(&bars[0]));
    __syncwarp();
    mbar_wait(smem_u32(&bars[0]), 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int BN, int NACC, int SAME_A, int EXTRA = 0>
void run(long long* d) {
  auto k = probe<BN, NACC, SAME_A, EXTRA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
  const int iters = 1024;
  k<<<148, 128, 170 * 1024>>>(8, d);
  k<<<148, 128, 170 * 1024>>>(iters, d);
  long long c = 0;
  if (cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    printf("error\n");
    exit(1);
  }
  const double mmas = 4.0 * NACC;
  printf("extra %2d N=%3d nacc=%d sameA=%d: %6.1f cycles per MMA (ideal %5.1f), %5.0f flop/clk/SM\n", EXTRA, BN, NACC,
         SAME_A, (double)c / iters / mmas, 2.0 * 128 * BN * 16 / 8192,
         2.0 * 128 * BN * 16 * mmas / ((double)c / iters));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 1, 0, 0>(d);
  run<64, 1, 0, 1>(d);
  run<64, 1, 0, 2>(d);
  run<64, 1, 0, 4>(d);
  run<64, 1, 0, 8>(d);
  run<64, 1, 0, 15>(d);
  run<128, 1, 0, 15>(d);
  run<256, 1, 0, 15>(d);
  return 0;
}
