// TMA load throughput probe (profiling helper, not product): every CTA streams
// k-blocks of an A tile (128 rows x 128 B, 2D or 4D NHWC box, optionally with
// element stride 2) and a B tile (64 rows x 128 B) through an N-slot smem ring
// into a consumer thread that only waits on the full barriers (no MMA).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma2(uint32_t dst, const void* tm, uint32_t bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(dst), "l"(tm), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tma4(uint32_t dst, const void* tm, uint32_t bar, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               ::"r"(dst), "l"(tm), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}

struct Maps {
  CUtensorMap a2, a4, a4s, b;
};

__global__ void __launch_bounds__(64) probe(const __grid_constant__ Maps mp, const Maps* mg, int mode,
                                             int slots, int kbs, int a_rows, int do_mma) {
  __shared__ uint32_t tslot;
  if (threadIdx.x >= 32) cw::tmem_alloc(smem_u32(&tslot), 128);
  const Maps& m = mg ? *mg : mp;
  if (mg && threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mg->a2) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mg->a4) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mg->b) : "memory");
  }
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const uint32_t sb = smem_u32(base);
  const uint32_t slot_bytes = 24 * 1024;
  const uint32_t full = sb + slots * slot_bytes, empty = full + 8 * 16;
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cw::tc_fence_before();
  __syncthreads();
  cw::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t tx = a_rows * 128 + 64 * 128;
  if (threadIdx.x == 0) {
    uint32_t par = 0;
    for (int k = 0; k < kbs; ++k) {
      const int s = k % slots;
      wait(empty + 8 * s, ((par >> s) & 1) ^ 1);
      par ^= 1u << s;
      expect(full + 8 * s, tx);
      const uint32_t dst = sb + s * slot_bytes;
      const int kk = k % 16;
      tma2(dst + 16384, &m.b, full + 8 * s, kk * 64, (blockIdx.x % 8) * 64);
      if (mode == 0) tma2(dst, &m.a2, full + 8 * s, kk * 64, (blockIdx.x % 64) * 128);
      else if (mode == 1) tma4(dst, &m.a4, full + 8 * s, kk * 64 % 256, 0, (blockIdx.x % 7) * 4, blockIdx.x % 16);
      else tma4(dst, &m.a4s, full + 8 * s, kk * 64 % 256, 0, (blockIdx.x % 7) * 8, blockIdx.x % 16);
    }
  } else if (threadIdx.x == 32) {
    uint32_t par = 0;
    for (int k = 0; k < kbs; ++k) {
      const int s = k % slots;
      wait(full + 8 * s, (par >> s) & 1);
      par ^= 1u << s;
      if (do_mma) {
        cw::tc_fence_after();
        const uint32_t a = sb + s * slot_bytes;
        const uint64_t ad = cw::sw128_kmajor_desc(a), bd = cw::sw128_kmajor_desc(a + 16384);
        for (int kk = 0; kk < 4; ++kk)
          cw::mma_bf16(tmem, ad + 2 * kk, bd + 2 * kk, cw::idesc_bf16_f32(128, 64), (k | kk) != 0);
        cw::mma_commit(empty + 8 * s);
      } else {
        arrive(empty + 8 * s);
      }
    }
  }
  if (do_mma && threadIdx.x == 32) {
    // wait for the last commits
    uint32_t par = 0;
    for (int k = 0; k < kbs; ++k) par ^= 1u << (k % slots);
    for (int s = 0; s < slots; ++s) wait(empty + 8 * s, ((par >> s) & 1) ^ 1);
  }
  cw::tc_fence_before();
  __syncthreads();
  if (threadIdx.x >= 32) { cw::tc_fence_after(); cw::tmem_dealloc(tmem, 128); }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  // activations: NHWC [16][28][28][256] bf16 (6.4 MB) and [16][56][56][256] for the strided map
  void *act, *act2, *w;
  cudaMalloc(&act, 1024 * 12544 * 2);
  cudaMalloc(&act2, 16 * 56 * 56 * 256 * 2);
  cudaMalloc(&w, 1024 * 1024 * 2);
  cudaMemset(act, 0, 1024 * 12544 * 2);
  cudaMemset(act2, 0, 16 * 56 * 56 * 256 * 2);
  cudaMemset(w, 0, 1024 * 1024 * 2);
  Maps m;
  cuuint32_t e1[4] = {1, 1, 1, 1}, e2[4] = {1, 2, 2, 1};
  {
    cuuint64_t d[2] = {1024, 16 * 784};
    cuuint64_t s[1] = {1024 * 2};
    cuuint32_t b[2] = {64, 128};
    enc(&m.a2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, d, s, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t d[4] = {256, 28, 28, 16};
    cuuint64_t s[3] = {256 * 2, 28 * 256 * 2, 28 * 28 * 256 * 2};
    cuuint32_t b[4] = {64, 28, 4, 1};
    enc(&m.a4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, act, d, s, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t d[4] = {256, 56, 56, 16};
    cuuint64_t s[3] = {256 * 2, 56 * 256 * 2, 56 * 56 * 256 * 2};
    cuuint32_t b[4] = {64, 56, 8, 1};
    enc(&m.a4s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, act2, d, s, b, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t d[2] = {1024, 1024};
    cuuint64_t s[1] = {1024 * 2};
    cuuint32_t b[2] = {64, 64};
    enc(&m.b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, d, s, b, e1, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, ev1;
  cudaEventCreate(&e0);
  cudaEventCreate(&ev1);
  Maps* mg;
  cudaMalloc(&mg, sizeof(Maps));
  cudaMemcpy(mg, &m, sizeof(Maps), cudaMemcpyHostToDevice);
  const char* names[3] = {"2D 128 rows     ", "4D 28x4 px      ", "4D 28x4 stride 2"};
  for (int do_mma = 0; do_mma < 2; ++do_mma)
  for (int glob = 0; glob < 1; ++glob)
  for (int mode = 0; mode < 3; ++mode)
    for (int grid : {148})
      for (int slots : {8}) {
        const int kbs = 512, a_rows = mode == 0 ? 128 : 112;
        float best = 1e9;
        for (int rep = 0; rep < 8; ++rep) {
          cudaEventRecord(e0);
          probe<<<grid, 64, 220 * 1024>>>(m, glob ? mg : nullptr, mode, slots, kbs, a_rows, do_mma);
          cudaEventRecord(ev1);
          cudaEventSynchronize(ev1);
          float ms;
          cudaEventElapsedTime(&ms, e0, ev1);
          if (rep > 1 && ms < best) best = ms;
        }
        const double bytes = (double)kbs * (a_rows * 128 + 64 * 128);
        printf("%s %s grid %3d slots %d: %.3f us per k-block, %.1f GB/s per SM\n",
               do_mma ? "tma+mma" : "tma    ", names[mode], grid,
               slots, best * 1e3 / kbs, bytes / (best * 1e-3) / 1e9);
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
