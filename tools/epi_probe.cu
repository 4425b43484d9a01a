// Epilogue store-path probe (profiling helper, not product): 148 CTAs x 4 warps
// write 128 x 256 bf16 tiles (64 KB) to a 25 MB NHWC-like buffer, 3 tiles per
// CTA, through (a) row-per-thread 16-byte stores, (b) a warp-staged coalesced
// pattern; optionally with a release-add + bar per tile, and optionally with a
// 5th warp spinning on ld.acquire.gpu (the megakernel's dependency poll).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(160) probe(uint4* out, uint32_t* flag, uint32_t* ctr, int tiles,
                                              int poll, int release,
                                              const __grid_constant__ CUtensorMap tm) {
  __shared__ __align__(1024) uint4 stage[4][2][32 * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4) {
    if (lane == 0 && poll) {
      // spin until the other warps are done (flag set by thread 0 at the end)
      volatile uint32_t* f = flag + blockIdx.x;
      while (true) {
        uint32_t v = poll == 1 ? ld_acquire(ctr + 4096) : ld_relaxed(ctr + 4096);
        if (*f) break;
        (void)v;
      }
    }
    return;
  }
  const int row = warp * 32 + lane;
  for (int t = 0; t < tiles; ++t) {
    const long long tile = (long long)blockIdx.x * tiles + t;
    uint4* base = out + tile * 128 * 32;  // 128 rows x 512 B
    for (int c = 0; c < 4; ++c) {         // 64-column chunks
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = make_uint4(row, c, k, t);
      if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) base[row * 32 + c * 8 + k] = v[k];
      } else if (MODE == 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) stage[warp][0][lane * 8 + (k ^ (lane & 7))] = v[k];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = i * 4 + (lane >> 3), ch = lane & 7;
          base[(warp * 32 + r) * 32 + c * 8 + ch] = stage[warp][0][r * 8 + (ch ^ (r & 7))];
        }
        __syncwarp();
      } else {
        const int b = c & 1;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) stage[warp][b][lane * 8 + (k ^ (lane & 7))] = v[k];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const uint32_t src = (uint32_t)__cvta_generic_to_shared(&stage[warp][b][0]);
          const int x = c * 64, y = (int)(tile * 128 + warp * 32);
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
              "r"(src), "r"(x), "r"(y)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (MODE == 2 && lane == 0) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (release) {
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + blockIdx.x) : "memory");
    }
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (threadIdx.x == 0) {
    __threadfence();
    *(volatile uint32_t*)(flag + blockIdx.x) = 1;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                            CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                            CUtensorMapFloatOOBfill);

int main() {
  const int G = 148, tiles = 3;
  uint4* out;
  uint32_t *flag, *ctr;
  cudaMalloc(&out, (size_t)G * tiles * 128 * 512);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {256, (cuuint64_t)G * tiles * 128};
  cuuint64_t strides[1] = {512};
  cuuint32_t box[2] = {64, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  cudaMalloc(&flag, G * 4);
  cudaMalloc(&ctr, 8192 * 4);
  cudaMemset(ctr, 0, 8192 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int poll = 0; poll < 3; ++poll)
      for (int rel = 0; rel < 2; ++rel) {
        float best = 1e9;
        for (int rep = 0; rep < 20; ++rep) {
          cudaMemset(flag, 0, G * 4);
          cudaEventRecord(e0);
          if (mode == 0) probe<0><<<G, 160>>>(out, flag, ctr, tiles, poll, rel, tm);
          else if (mode == 1) probe<1><<<G, 160>>>(out, flag, ctr, tiles, poll, rel, tm);
          else probe<2><<<G, 160>>>(out, flag, ctr, tiles, poll, rel, tm);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep > 2 && ms < best) best = ms;
        }
        printf("%s poll=%s release=%d: %.2f us for %d x 64 KB tiles per SM (%.0f GB/s total)\n",
               mode == 2 ? "tma    " : (mode ? "staged " : "per-row"), poll == 0 ? "none   " : (poll == 1 ? "acquire" : "relaxed"),
               rel, best * 1e3, tiles, G * tiles * 65536.0 / (best * 1e-3) / 1e9);
      }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
