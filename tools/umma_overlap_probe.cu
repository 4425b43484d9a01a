// Correctness probe (profiling helper, not product): can a tcgen05.mma A operand be an
// implicit im2col view of ONE staged NHWC4 input row — rows 16 bytes apart, 64 bytes long
// (overlapping), described by a SWIZZLE_NONE K-major descriptor with LBO = 16 B (K-adjacent
// core matrices) and SBO = 128 B (8-row groups)? That is the 7x7/s2 stem's A operand
// (conv column j reads input pixels 2j .. 2j+7 of 4 channels). One CTA: D[128][64] =
// A_view[128][32] x B[64][32]^T (two K=16 MMAs), compared with the CPU product.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

#include "../paper_2006_02464_b200/csrc/ptx.cuh"

using namespace cw;

__device__ __forceinline__ uint64_t desc_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);  // layout type 0 = no swizzle
}

__global__ void probe(const __nv_bfloat16* row, const __nv_bfloat16* bmat, float* out, int swap, int aoff) {
  __shared__ __align__(1024) uint8_t sa[8192];
  __shared__ __align__(1024) uint8_t sbm[4096];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // A: the staged row, 2 px per 16 B; 300 px x 4 ch = 2400 B (+ slack)
  for (int i = t; i < 8192 / 2; i += blockDim.x) reinterpret_cast<__nv_bfloat16*>(sa)[i] = __float2bfloat16(0.f);
  __syncthreads();
  for (int i = t; i < 1200; i += blockDim.x) reinterpret_cast<__nv_bfloat16*>(sa + aoff)[i] = row[i];
  // B: [64 n][32 k] as no-swizzle K-major core matrices: (n/8)*512 + (k/8)*128 + (n%8)*16 + (k%8)*2
  for (int i = t; i < 64 * 32; i += blockDim.x) {
    const int n = i / 32, k = i % 32;
    const int off = (n / 8) * 512 + (k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sbm + off) = bmat[i];
  }
  if (t == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(smem_u32(&tslot), 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (t == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 64);
    const uint32_t a0 = smem_u32(sa) + aoff, b0 = smem_u32(sbm);
    const uint32_t alb = swap ? 128 : 16, asb = swap ? 16 : 128;
    for (int k = 0; k < 2; ++k) {  // K = 16 per MMA: A +32 B, B +2 core matrices (256 B)
      const uint64_t ad = desc_none(a0 + 32 * k, alb, asb);
      const uint64_t bd = desc_none(b0 + 256 * k, 128, 512);
      mma_bf16(tmem, ad, bd, idesc, k != 0);
    }
    mma_commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  uint32_t v[16];
  for (int c = 0; c < 64; c += 16) {
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[(warp * 32 + lane) * 64 + c + i] = __uint_as_float(v[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

int main() {
  std::vector<__nv_bfloat16> row(1200), b(64 * 32);
  std::vector<float> rf(1200), bf(64 * 32);
  for (int i = 0; i < 1200; ++i) { rf[i] = (float)((i * 37 % 17) - 8) / 8.f; row[i] = __float2bfloat16(rf[i]); rf[i] = __bfloat162float(row[i]); }
  for (int i = 0; i < 64 * 32; ++i) { bf[i] = (float)((i * 13 % 11) - 5) / 4.f; b[i] = __float2bfloat16(bf[i]); bf[i] = __bfloat162float(b[i]); }
  __nv_bfloat16 *drow, *db;
  float* dout;
  cudaMalloc(&drow, 2400);
  cudaMalloc(&db, 4096);
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(drow, row.data(), 2400, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), 4096, cudaMemcpyHostToDevice);
  for (int aoff : {0, 16, 32, 48, 80, 1888, 3760}) {
    const int swap = 0;
    cudaMemset(dout, 0, 128 * 64 * 4);
    probe<<<1, 128>>>(drow, db, dout, swap, aoff);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(128 * 64);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int j = 0; j < 128; ++j)
      for (int n = 0; n < 64; ++n) {
        double s = 0;
        for (int k = 0; k < 32; ++k) {
          const int idx = 8 * j + k;  // element offset of A(j, k) in the staged row
          s += (idx < 1200 ? rf[idx] : 0.0) * bf[n * 32 + k];
        }
        maxerr = fmax(maxerr, fabs(s - out[j * 64 + n]));
      }
    printf("A start offset %4d B: max abs err %.3g  [%s]\n", aoff, maxerr, cudaGetErrorString(e));
  }
  return 0;
}
