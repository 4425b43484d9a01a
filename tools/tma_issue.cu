// TMA issue-cost probe (profiling helper, not product): one warp issues n 2D tensor-map
// loads of a 64 x 128 bf16 box (16 KB) into a 4-slot ring (full/empty mbarriers, a second
// warp consumes by waiting on full and arriving on empty), measuring cycles per TMA.
//   variant 0: coordinates from per-thread registers, whole warp + elect per TMA
//   variant 1: coordinates from per-thread registers, one elect block issues 2 TMAs per slot
//   variant 2: coordinates in uniform registers (loop counter only), elect per slot
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap tm,
                                               const __grid_constant__ CUtensorMap tm4, int n, int variant,
                                               const int* coords, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const uint32_t sb = smem_u32(base);
  __shared__ __align__(8) uint64_t full[4], empty[4];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int c_base = coords[blockIdx.x & 7];  // per-thread register (not provably uniform)
  if (warp == 0) {
    uint32_t par = 0;
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const int s = i & 3;
      if (i >= 4) {
        mbar_wait(smem_u32(&empty[s]), ((par >> s) & 1) ^ 1);
      }
      par ^= 1u << s;
      const uint32_t dst = sb + s * 32768, fb = smem_u32(&full[s]);
      if (variant == 0) {
        if (elect_one()) mbar_arrive_expect_tx(fb, 32768);
        __syncwarp();
        if (elect_one()) tma_load_2d(dst, &tm, fb, ((c_base + i) & 7) * 64, 0);
        __syncwarp();
        if (elect_one()) tma_load_2d(dst + 16384, &tm, fb, ((c_base + 2 * i) & 7) * 64, 128);
        __syncwarp();
      } else if (variant == 1) {
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, 32768);
          tma_load_2d(dst, &tm, fb, ((c_base + i) & 7) * 64, 0);
          tma_load_2d(dst + 16384, &tm, fb, ((c_base + 2 * i) & 7) * 64, 128);
        }
        __syncwarp();
      } else if (variant == 2) {
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, 32768);
          tma_load_2d(dst, &tm, fb, (i & 7) * 64, 0);
          tma_load_2d(dst + 16384, &tm, fb, (i & 7) * 64, 128);
        }
        __syncwarp();
      } else {
        // 4D NHWC boxes (64 ch x 14 w x 9 h x 1 n = 126 rows, 16128 B), 3x3 tap shifts
        const int tap = i % 9, q = tap % 3 - 1, r = tap / 3 - 1;
        const int img = (i / 9) & 15, h0 = ((i / 144) & 1) * 9 - 1;
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, 2 * 16128);
          tma_load_4d(dst, &tm4, fb, 0, q, h0 + r + 1, img);
          tma_load_4d(dst + 16384, &tm4, fb, 64 * (variant - 3), q, h0 + r + 1, (img + 1) & 15);
        }
        __syncwarp();
      }
    }
    const long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
  } else {
    uint32_t par = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i & 3;
      mbar_wait(smem_u32(&full[s]), (par >> s) & 1);
      par ^= 1u << s;
      if (elect_one()) mbar_arrive(smem_u32(&empty[s]));
      __syncwarp();
    }
  }
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
  void* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 0, 64 << 20);
  CUtensorMap tm;
  cuuint64_t dims[2] = {4096, 4096};
  cuuint64_t strides[1] = {4096 * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap tm4;
  {
    cuuint64_t d4[4] = {256, 14, 14, 16};
    cuuint64_t s4[3] = {256 * 2, 14 * 256 * 2, 14 * 14 * 256 * 2};
    cuuint32_t b4[4] = {64, 14, 9, 1};
    cuuint32_t e4[4] = {1, 1, 1, 1};
    enc(&tm4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int* coords;
  cudaMalloc(&coords, 64);
  cudaMemset(coords, 0, 64);
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  for (int grid : {1, 148})
    for (int v : {0, 1, 2, 3, 4}) {
      const int n = 2048;
      probe<<<grid, 64, 140 * 1024>>>(tm, tm4, 16, v, coords, d);
      probe<<<grid, 64, 140 * 1024>>>(tm, tm4, n, v, coords, d);
      long long c = 0;
      if (cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
        printf("error\n");
        return 1;
      }
      printf("grid %3d variant %d: %.1f cycles per slot (2 TMAs, 32 KB) -> %.1f B/clk\n", grid, v,
             (double)c / n, 32768.0 / ((double)c / n));
    }
  return 0;
}
