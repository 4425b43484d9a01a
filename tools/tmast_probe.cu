// Store-path throughput probe (profiling helper, not product). Every CTA (one per SM)
// writes 16 KB chunks (128 rows x 64 bf16 columns of a [rows][256] bf16 tensor, the
// megakernel's epilogue chunk) into an L2-resident 29 MB tensor, many times over:
//   mode 0: TMA stores (128-byte swizzle box) issued by `issuers` threads in different warps,
//           each with its own staging buffers (cp.async.bulk.wait_group.read before reuse)
//   mode 1: st.global.v4 by 8 warps, coalesced (each warp instruction: 4 rows x 128 B)
//   mode 2: st.global.v4 by 8 warps, row per thread (the accumulator layout: a warp
//           instruction touches 32 rows x 16 B)
//   mode 3: per-warp TMA stores: each of the 8 warps' lane 0 stores its own 32 rows x 32
//           columns (a 2 KB box, 64-byte swizzle) of every chunk, no CTA barrier
// Also reports the issuing thread's cycles per store instruction + commit (issue cost).
// Reports bytes per clock per SM and the aggregate bandwidth.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

__global__ void __launch_bounds__(256) probe(const __grid_constant__ CUtensorMap tm,
                                              const __grid_constant__ CUtensorMap tm32, uint4* out,
                                              int mode, int issuers, int reps, int tiles,
                                              unsigned long long* cyc, unsigned long long* icyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (cw::smem_u32(smem) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  const long long t0 = clock64();
  const int chunks = tiles * 4;
  long long issue = 0;
  int nissue = 0;
  if (mode == 0) {
    if (lane == 0 && warp < issuers) {
      int n = 0;
      for (int r = 0; r < reps; ++r)
        for (int i = warp; i < chunks; i += issuers, ++n) {
          const int nb = issuers == 1 ? 4 : 12 / issuers;
          const uint32_t src = base + (warp * nb + n % nb) * 16384u;
          const int row = (blockIdx.x * tiles + i / 4) * 128, col = (i % 4) * 64;
          cw::bulk_wait_read_n(nb - 1);
          const long long q0 = clock64();
          cw::tma_store_2d(&tm, src, col, row);
          cw::bulk_commit();
          issue += clock64() - q0;
          ++nissue;
        }
      cw::bulk_wait_all();
    }
  } else if (mode == 3) {
    // warp w: rows 32 (w & 3) .. +31, columns 32 (w >> 2) .. +31 of each 64-column chunk
    if (lane == 0) {
      int n = 0;
      for (int r = 0; r < reps; ++r)
        for (int i = 0; i < chunks; ++i, ++n) {
          const uint32_t src = base + (uint32_t)(warp * 6 + n % 6) * 2048u;
          const int row = (blockIdx.x * tiles + i / 4) * 128 + 32 * (warp & 3);
          const int col = (i % 4) * 64 + 32 * (warp >> 2);
          cw::bulk_wait_read_n(5);
          const long long q0 = clock64();
          cw::tma_store_2d(&tm32, src, col, row);
          cw::bulk_commit();
          issue += clock64() - q0;
          ++nissue;
        }
      cw::bulk_wait_all();
    }
    __syncwarp();
  } else {
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    for (int r = 0; r < reps; ++r)
      for (int i = 0; i < chunks; ++i) {
        // chunk i: rows (blockIdx.x * tiles + i / 4) * 128 .. +127, 128-byte column block i % 4
        uint4* rowbase = out + (size_t)(blockIdx.x * tiles + i / 4) * 128 * 32 + (i % 4) * 8;
        if (mode == 1) {
          // warp w: rows 16w .. 16w+15; lane: row 16w + 4j + lane / 8, 16-byte piece lane % 8
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int rr = 16 * warp + 4 * j + (lane >> 3);
            rowbase[rr * 32 + (lane & 7)] = v;
          }
        } else {
          // thread: row (warp & 3) * 32 + lane, pieces 4 (warp >> 2) .. +3
          const int rr = (warp & 3) * 32 + lane;
#pragma unroll
          for (int j = 0; j < 4; ++j) rowbase[rr * 32 + 4 * (warp >> 2) + j] = v;
        }
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  if (threadIdx.x == 0) icyc[blockIdx.x] = nissue ? issue / nissue : 0;
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
  const int tiles = 3;
  const long long rows = 148LL * 128 * tiles;  // 29 MB
  void* buf;
  cudaMalloc(&buf, rows * 512);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  unsigned long long* icyc;
  cudaMalloc(&icyc, 148 * 8);
  CUtensorMap tm, tm32;
  cuuint64_t d[2] = {256, (cuuint64_t)rows};
  cuuint64_t s[1] = {512};
  cuuint32_t b[2] = {64, 128}, e[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint32_t b32[2] = {32, 32};
  enc(&tm32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d, s, b32, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  const int reps = 20;
  struct Case { int mode, issuers; const char* name; } cases[] = {
      {0, 1, "TMA store, 1 issuer   "}, {0, 2, "TMA store, 2 issuers  "},
      {0, 3, "TMA store, 3 issuers  "}, {0, 6, "TMA store, 6 issuers  "},
      {3, 8, "TMA store, per warp   "},
      {1, 0, "st.global coalesced   "}, {2, 0, "st.global row/thread  "}};
  for (const Case& c : cases) {
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      probe<<<148, 256, 12 * 16384 + 1024>>>(tm, tm32, (uint4*)buf, c.mode, c.issuers, reps, tiles,
                                             cyc, icyc);
      cudaEventRecord(z);
      cudaEventSynchronize(z);
      float ms;
      cudaEventElapsedTime(&ms, a, z);
      if (ms < best) best = ms;
    }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long hi[148];
    cudaMemcpy(hi, icyc, sizeof(hi), cudaMemcpyDeviceToHost);
    double mc = 0, mi = 0;
    for (int i = 0; i < 148; ++i) mc += (double)h[i] / 148, mi += (double)hi[i] / 148;
    const double per_sm = (double)reps * tiles * 4 * 16384;
    printf("%s %7.1f us  %6.0f GB/s  %5.1f B/clk/SM  (%5.0f cycles per 16 KB chunk, issue %4.0f "
           "cycles per store)\n", c.name, best * 1e3, 148 * per_sm / (best * 1e-3) / 1e9,
           per_sm / mc, mc / (reps * tiles * 4), mi);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
