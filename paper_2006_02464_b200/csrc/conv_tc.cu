// Implicit-GEMM convolution on the 5th-generation tensor cores (sm_100a).
//
//   D[M, Cout] = A[M, K] * W[Cout, K]^T   with  M = output pixels (N*OH*OW),
//                                              K = KH*KW*Cin (tap-major, channel-minor)
//   out = relu?( D + bias[Cout] (+ residual) )  -> bf16 NHWC
//
// Replaces the emulated Exec wait of the reference worker
// (pkg/src/sloserve/worker.py:273-277: `dur = exec_duration[b]; call_at(now+dur)`)
// with the real batched CNN forward; this kernel carries every convolution
// of the ResNet family (1x1, 3x3, strided, downsample, and conv1 after the
// input-stage im2col).
//
// One CTA computes one 128 x BN output tile; 6 warps:
//   warp 0      TMA producer: per 64-wide k-block, A tile (128 rows x 128 B) and
//               W tile (BN rows x 128 B), both 128B-swizzled, into a STAGES ring.
//               mode 0: A via a 2D tensor map over a [M][K] matrix.
//               mode 1: A via a 4D NHWC tensor map; k-block -> (tap r,s; 64 channels)
//               and the box origin is shifted by the tap. Padding is TMA
//               out-of-bounds zero fill; stride is the TMA element stride.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN,
//               K=16 per instruction, fp32 accumulators in TMEM).
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 16 columns, + bias, + residual,
//               ReLU, bf16 pack, 32-byte stores of NHWC rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "cw_device.h"
#include "ptx.cuh"

namespace cw {

constexpr int kConvThreads = 192;
constexpr uint32_t kATileBytes = 128 * 128;

template <int BN, int STAGES>
struct ConvSmem {
  static constexpr uint32_t kBBytes = BN * 128;
  static constexpr uint32_t kStageBytes = kATileBytes + kBBytes;
  static constexpr uint32_t kBarOff = STAGES * kStageBytes;
  static constexpr uint32_t kBiasOff = kBarOff + 256;
  static constexpr uint32_t kTotal = kBiasOff + BN * 4 + 1024;  // + alignment slack
  static_assert((2 * STAGES + 2) * 8 <= 256, "barrier area");
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kConvThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const ConvArgs args) {
  using L = ConvSmem<BN, STAGES>;
  const ActionBlock* ab = args.ab;
  if (ab->skip) return;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + L::kBarOff;             // STAGES x 8 B
  const uint32_t bar_empty = bar_full + STAGES * 8;         // STAGES x 8 B
  const uint32_t bar_tfull = bar_empty + STAGES * 8;        // 8 B
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kBarOff + (2 * STAGES + 1) * 8);
  float* sbias = reinterpret_cast<float*>(smem + L::kBiasOff);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint8_t* hdr = ab->hdr;
  const CUtensorMap* tmap_b = reinterpret_cast<const CUtensorMap*>(hdr + args.layer * kTmapBytes);
  const float* bias = reinterpret_cast<const float* const*>(hdr + kHdrBiasOff)[args.layer];
  const int n0 = blockIdx.y * BN;

  // Output-tile origin.
  int m0 = 0, ow0 = 0, oh0 = 0, img0 = 0;
  if (args.mode == 0) {
    m0 = blockIdx.x * 128;
  } else {
    const int t = blockIdx.x;
    const int tw = t % args.tiles_w;
    const int th = (t / args.tiles_w) % args.tiles_h;
    const int tn = t / (args.tiles_w * args.tiles_h);
    ow0 = tw * args.box_w;
    oh0 = th * args.box_h;
    img0 = tn * args.box_n;
  }

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    mbar_init(bar_tfull, 1);
    fence_mbar_init();
    tmap_acquire(tmap_b);
    tmap_prefetch(&tmap_a);
    tmap_prefetch(tmap_b);
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), BN);
  if (warp >= 2) {
    for (int i = threadIdx.x - 64; i < BN; i += 128) sbias[i] = bias[n0 + i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int num_kb = args.num_kb;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      const uint32_t a_rows = args.mode == 0 ? 128u : (uint32_t)(args.box_w * args.box_h * args.box_n);
      const uint32_t tx_bytes = a_rows * 128u + L::kBBytes;
      const int wb = ow0 * args.stride - args.pad;
      const int hb = oh0 * args.stride - args.pad;
      int s = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(bar_empty + 8 * s, phase ^ 1);
        const uint32_t a_dst = sbase + s * L::kStageBytes;
        const uint32_t b_dst = a_dst + kATileBytes;
        const uint32_t full = bar_full + 8 * s;
        mbar_arrive_expect_tx(full, tx_bytes);
        if (args.mode == 0) {
          tma_load_2d(a_dst, &tmap_a, full, kb * 64, m0);
        } else {
          const int tap = kb / args.cin_kb;
          const int c0 = (kb - tap * args.cin_kb) * 64;
          const int r = tap / args.kw;
          const int q = tap - r * args.kw;
          tma_load_4d(a_dst, &tmap_a, full, c0, wb + q, hb + r, img0);
        }
#pragma unroll
        for (int j = 0; j < BN / 64; ++j)
          tma_load_2d(b_dst + j * 8192, tmap_b, full, kb * 64, n0 + 64 * j);
        if (++s == STAGES) { s = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN);
      int s = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(bar_full + 8 * s, phase);
        tc_fence_after();
        const uint32_t a_addr = sbase + s * L::kStageBytes;
        const uint64_t adesc = sw128_kmajor_desc(a_addr);
        const uint64_t bdesc = sw128_kmajor_desc(a_addr + kATileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // +32 bytes along K inside the 128-byte swizzled row = +2 in desc units.
          mma_bf16(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
        }
        mma_commit(bar_empty + 8 * s);
        if (++s == STAGES) { s = 0; phase ^= 1; }
      }
      mma_commit(bar_tfull);
    }
  } else {
    // ---------------- epilogue (warps 2..5; TMEM lane quarter = warp % 4)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    bool valid;
    long long m;
    if (args.mode == 0) {
      m = (long long)m0 + row;
      valid = m < args.m_total;
    } else {
      const int rows = args.box_w * args.box_h * args.box_n;
      const int wi = row % args.box_w;
      const int t = row / args.box_w;
      const int hi = t % args.box_h;
      const int ni = t / args.box_h;
      const int ow = ow0 + wi, oh = oh0 + hi, n = img0 + ni;
      valid = row < rows && ow < args.ow && oh < args.oh && n < args.nimg;
      m = ((long long)n * args.oh + oh) * args.ow + ow;
    }
    __nv_bfloat16* out_row = reinterpret_cast<__nv_bfloat16*>(args.out) + m * args.n_out + n0;
    const __nv_bfloat16* res_row =
        args.residual ? reinterpret_cast<const __nv_bfloat16*>(args.residual) + m * args.n_out + n0
                      : nullptr;
    mbar_wait(bar_tfull, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t v[16];
      tmem_ld16(taddr + c, v);
      tmem_ld_wait();
      if (valid) {
        float f[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + sbias[c + i];
        if (res_row) {
          const uint4* rp = reinterpret_cast<const uint4*>(res_row + c);
          uint4 r0 = rp[0], r1 = rp[1];
          const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&r0);
          const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&r1);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 a = __bfloat1622float2(h0[i]);
            float2 b = __bfloat1622float2(h1[i]);
            f[2 * i] += a.x;
            f[2 * i + 1] += a.y;
            f[8 + 2 * i] += b.x;
            f[8 + 2 * i + 1] += b.y;
          }
        }
        if (args.relu) {
#pragma unroll
          for (int i = 0; i < 16; ++i) f[i] = fmaxf(f[i], 0.0f);
        }
        uint4 o0, o1;
        o0.x = pack_bf16x2(f[0], f[1]);
        o0.y = pack_bf16x2(f[2], f[3]);
        o0.z = pack_bf16x2(f[4], f[5]);
        o0.w = pack_bf16x2(f[6], f[7]);
        o1.x = pack_bf16x2(f[8], f[9]);
        o1.y = pack_bf16x2(f[10], f[11]);
        o1.z = pack_bf16x2(f[12], f[13]);
        o1.w = pack_bf16x2(f[14], f[15]);
        uint4* op = reinterpret_cast<uint4*>(out_row + c);
        op[0] = o0;
        op[1] = o1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, BN);
  }
}

// ------------------------------------------------------------------ host side

template <int BN, int STAGES>
static cudaError_t configure_bn() {
  return cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              ConvSmem<BN, STAGES>::kTotal);
}

template <int BN, int STAGES>
static cudaError_t launch_bn(const CUtensorMap& tmap_a, const ConvArgs& a, int m_tiles,
                             cudaStream_t st) {
  dim3 grid(m_tiles, a.n_out / BN);
  conv_tc_kernel<BN, STAGES><<<grid, kConvThreads, ConvSmem<BN, STAGES>::kTotal, st>>>(tmap_a, a);
  return cudaGetLastError();
}

// Must run once per device before the first launch (and before graph capture).
cudaError_t configure_conv_tc() {
  cudaError_t e;
  if ((e = configure_bn<64, 6>()) != cudaSuccess) return e;
  if ((e = configure_bn<128, 5>()) != cudaSuccess) return e;
  return configure_bn<256, 4>();
}

cudaError_t launch_conv_tc(const CUtensorMap& tmap_a, const ConvArgs& a, int bn, int m_tiles,
                           cudaStream_t st) {
  switch (bn) {
    case 64: return launch_bn<64, 6>(tmap_a, a, m_tiles, st);
    case 128: return launch_bn<128, 5>(tmap_a, a, m_tiles, st);
    case 256: return launch_bn<256, 4>(tmap_a, a, m_tiles, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace cw
