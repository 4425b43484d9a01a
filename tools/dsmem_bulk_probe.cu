// Sanitizer probe (profiling helper, not product): is compute-sanitizer memcheck's
// "Invalid __shared__ write ... not located in remote CTA" on epi_csplit's DSMEM bulk copies
// a real out-of-bounds write or a tool limitation? A 2-CTA cluster with the megakernel's
// dynamic shared-memory size; each rank bulk-copies 4 KB (cp.async.bulk.shared::cluster,
// destination + mbarrier from mapa) into the peer at the offsets epi_csplit uses, waits on
// the transaction count, then checks every byte it received. Pass = data correct; run it
// under `compute-sanitizer --tool memcheck` to see whether the tool flags the same copy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/dsmem_bulk_probe tools/dsmem_bulk_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

constexpr uint32_t kBlk = 4096;

__global__ void __cluster_dims__(2, 1, 1) probe(uint32_t dst_off, uint32_t src_off, int* bad) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int t = threadIdx.x;
  for (uint32_t i = t; i < kBlk / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(smem + src_off)[i] = (rank << 24) | i;
    reinterpret_cast<uint32_t*>(smem + dst_off)[i] = 0xdeadbeefu;
  }
  if (t == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  __syncthreads();
  cluster_sync();  // both barriers initialised, both destinations cleared
  if (t == 0) {
    mbar_arrive_expect_tx(smem_u32(&bar), kBlk);
    bulk_s2cluster(mapa_shared(smem_u32(smem + dst_off), peer), smem_u32(smem + src_off), kBlk,
                   mapa_shared(smem_u32(&bar), peer));
  }
  mbar_wait(smem_u32(&bar), 0);
  int nbad = 0;
  for (uint32_t i = t; i < kBlk / 4; i += blockDim.x)
    nbad += reinterpret_cast<uint32_t*>(smem + dst_off)[i] != ((peer << 24) | i);
  atomicAdd(bad, nbad);
  cluster_sync();  // the peer's copy out of this CTA has completed before it exits
}

int main() {
  int* bad;
  cudaMalloc(&bad, sizeof(int));
  // (dst, src) offsets: small smem, and the megakernel's ~220 KB with the receive block at
  // 0x26800 (the address memcheck reports)
  struct Case { uint32_t smem, dst, src; } cases[] = {{16384, 0, 8192},
                                                      {220 * 1024, 0x26800, 0x26800 + 0x8000}};
  int fails = 0;
  for (const Case& c : cases) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    cudaMemset(bad, 0, sizeof(int));
    probe<<<2, 128, c.smem>>>(c.dst, c.src, bad);
    int h = -1;
    cudaError_t e = cudaMemcpy(&h, bad, sizeof(int), cudaMemcpyDeviceToHost);
    printf("smem %u dst 0x%x src 0x%x: %s, %d wrong words\n", c.smem, c.dst, c.src,
           cudaGetErrorString(e), h);
    fails += e != cudaSuccess || h != 0;
  }
  printf(fails ? "FAIL\n" : "PASS\n");
  return fails != 0;
}
