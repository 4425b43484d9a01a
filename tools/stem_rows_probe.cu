// TMA probe for the stem's staged input rows (profiling helper, not product): the 4D map
// (8 elements, wp/2, hp, n) over padded NHWC4 bf16 rows, box (8, wp/2, rows, 1), no swizzle;
// one CTA loads the rows of a few (row0, image) origins and checks the bytes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap tm, int row0, int img, int bytes,
                      uint16_t* out, int* ok) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(smem_u32(&bar), (uint32_t)bytes);
    tma_load_4d(smem_u32(sm), &tm, smem_u32(&bar), 0, 0, row0, img);
    const long long t0 = clock64();
    bool done = false;
    while (!done && clock64() - t0 < 200000000ll) {
      uint32_t r;
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(r) : "r"(smem_u32(&bar)) : "memory");
      done = r != 0;
    }
    *ok = done;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  const int n = 2, hp = 230, wp = 234, rows = 11;
  std::vector<uint16_t> h((size_t)n * hp * wp * 4);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 16);
  void* d;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  const uint64_t row = (uint64_t)wp * 8;
  cuuint64_t dims[4] = {8, (cuuint64_t)wp / 2, (cuuint64_t)hp, (cuuint64_t)n};
  cuuint64_t strides[3] = {16, row, hp * row};
  cuuint32_t box[4] = {8, (cuuint32_t)wp / 2, (cuuint32_t)rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  const int bytes = rows * (int)row;
  uint16_t* dout;
  int* dok;
  cudaMalloc(&dout, bytes);
  cudaMalloc(&dok, 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int row0 : {-2, 0, 50, 219}) {
    for (int img : {0, 1}) {
      cudaMemset(dok, 0, 4);
      probe<<<1, 128, 32 * 1024>>>(tm, row0, img, bytes, dout, dok);
      cudaError_t e = cudaDeviceSynchronize();
      int ok = 0;
      cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
      std::vector<uint16_t> o(bytes / 2);
      cudaMemcpy(o.data(), dout, bytes, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int rr = 0; rr < rows; ++rr)
        for (int i = 0; i < wp * 4; ++i) {
          const int gr = row0 + rr;
          const uint16_t want = (gr < 0 || gr >= hp) ? 0 : h[(((size_t)img * hp + gr) * wp) * 4 + i];
          if (o[(size_t)rr * wp * 4 + i] != want) ++bad;
        }
      printf("row0 %4d img %d: completed %d, mismatches %d [%s]\n", row0, img, ok, bad,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
