// Memory-bound INFER kernels (vectorised SIMT) and the executor's device-side
// window gate / timestamps.
//
//   gate_kernel       K8: per-INFER window gate. Pulls the next descriptor from
//                     the host ring (mapped pinned memory), spins on %globaltimer
//                     until `earliest`, rejects if past `latest` (the reference's
//                     `now > action.latest` test, pkg/src/sloserve/worker.py:230),
//                     stamps Exec start, publishes the ActionBlock for the graph.
//   exec_done_kernel  stamps Exec end (device_duration = t_end - t_start,
//                     worker.py:292-299 `_exec_done`).
//   stem_im2col       K1: fp32 NCHW request inputs (IOCache slots) -> bf16
//                     im2col rows for the 7x7/s2 stem convolution.
//   maxpool3x3s2      K3: 3x3 stride-2 pad-1 max pool, bf16 NHWC, 16-byte vectors.
//   avgpool           K7a: global average pool -> fp32 [b][C].
//   fc_kernel         K7b: logits = pooled . W^T + bias, one warp per class,
//                     written straight into each request's IOCache output slot.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "cw_device.h"
#include "ptx.cuh"

namespace cw {

__global__ void gate_kernel(ActionBlock* ab, const ActionDesc* ring, uint32_t ring_mask,
                            uint64_t* ctr, ExecRecord* recs) {
  __shared__ uint64_t words[sizeof(ActionDesc) / 8];
  __shared__ uint64_t idx_s;
  if (threadIdx.x == 0) {
    uint64_t i = *ctr;
    *ctr = i + 1;
    idx_s = i;
  }
  __syncthreads();
  const uint64_t i = idx_s;
  // Parallel fetch of the descriptor over PCIe (one 8-byte word per thread).
  const volatile uint64_t* src =
      reinterpret_cast<const volatile uint64_t*>(&ring[i & ring_mask]);
  for (int w = threadIdx.x; w < (int)(sizeof(ActionDesc) / 8); w += blockDim.x) words[w] = src[w];
  __syncthreads();
  if (threadIdx.x == 0) {
    const ActionDesc* d = reinterpret_cast<const ActionDesc*>(words);
    ab->hdr = d->hdr;
    for (int k = 0; k < kMaxBatch; ++k) {
      ab->in[k] = d->in[k];
      ab->out[k] = d->out[k];
    }
    ab->batch = d->batch;
    ab->seq = i;
    uint64_t t = globaltimer();
    while (t < d->earliest_gt) t = globaltimer();
    const int rej = t > d->latest_gt;
    ab->skip = rej;
    ExecRecord* r = &recs[i & ring_mask];
    r->t_start = t;
    r->rejected = rej;
    __threadfence_system();
    r->seq_started = i + 1;
    __threadfence();
  }
}

__global__ void exec_done_kernel(const ActionBlock* ab, uint32_t ring_mask, ExecRecord* recs) {
  griddep_wait();
  const uint64_t i = ab->seq;
  ExecRecord* r = &recs[i & ring_mask];
  r->t_end = globaltimer();
  __threadfence_system();
  r->seq_done = i + 1;
}

__global__ void out_done_kernel(ExecRecord* rec, uint64_t seq) {
  rec->t_out = globaltimer();
  __threadfence_system();
  rec->seq_out = seq;
}

// Publishes %globaltimer continuously (bounded by max_ns) for host clock calibration.
__global__ void clock_pub_kernel(volatile uint64_t* slot, uint64_t max_ns) {
  const uint64_t t0 = globaltimer();
  uint64_t t = t0;
  while (t - t0 < max_ns) {
    slot[0] = t;
    __threadfence_system();
    t = globaltimer();
  }
  slot[1] = 1;
}

// Stamp kernel for the LOAD copy stream: slot[0] = time, then slot[1] = tag.
__global__ void stamp_kernel(volatile uint64_t* slot, uint64_t tag) {
  slot[0] = globaltimer();
  __threadfence_system();
  slot[1] = tag;
}

// K = (r*7 + s)*3 + c for r,s < 7, c < 3 (147 values), zero-padded to kpad.
__global__ void stem_im2col_kernel(const ActionBlock* ab, __nv_bfloat16* __restrict__ a, int batch,
                                   int H, int W, int OH, int OW, int kpad) {
  griddep_wait();
  griddep_trigger();
  if (ab->skip) return;
  const int chunks = kpad / 8;
  const long long total = (long long)batch * OH * OW * chunks;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t % chunks);
    const long long p = t / chunks;
    const int ow = (int)(p % OW);
    const int oh = (int)((p / OW) % OH);
    const int n = (int)(p / ((long long)OW * OH));
    const float* img = ab->in[n];
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int k = j * 8 + e;
      float x = 0.0f;
      if (k < 147) {
        const int r = k / 21;
        const int s = (k % 21) / 3;
        const int c = k % 3;
        const int ih = oh * 2 - 3 + r;
        const int iw = ow * 2 - 3 + s;
        if (ih >= 0 && ih < H && iw >= 0 && iw < W) x = __ldg(img + ((long long)c * H + ih) * W + iw);
      }
      v[e] = x;
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    reinterpret_cast<uint4*>(a)[t] = o;
  }
}

__global__ void maxpool3x3s2_kernel(const ActionBlock* ab, const __nv_bfloat16* __restrict__ in,
                                    __nv_bfloat16* __restrict__ out, int batch, int H, int W, int C,
                                    int OH, int OW) {
  griddep_wait();
  griddep_trigger();
  if (ab->skip) return;
  const int chunks = C / 8;
  const long long total = (long long)batch * OH * OW * chunks;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t % chunks);
    const long long p = t / chunks;
    const int ow = (int)(p % OW);
    const int oh = (int)((p / OW) % OH);
    const int n = (int)(p / ((long long)OW * OH));
    float m[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) m[e] = -INFINITY;
    for (int r = 0; r < 3; ++r) {
      const int ih = oh * 2 - 1 + r;
      if (ih < 0 || ih >= H) continue;
      for (int s = 0; s < 3; ++s) {
        const int iw = ow * 2 - 1 + s;
        if (iw < 0 || iw >= W) continue;
        uint4 u = *reinterpret_cast<const uint4*>(in + (((long long)n * H + ih) * W + iw) * C + j * 8);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h[e]);
          m[2 * e] = fmaxf(m[2 * e], f.x);
          m[2 * e + 1] = fmaxf(m[2 * e + 1], f.y);
        }
      }
    }
    uint4 o;
    o.x = pack_bf16x2(m[0], m[1]);
    o.y = pack_bf16x2(m[2], m[3]);
    o.z = pack_bf16x2(m[4], m[5]);
    o.w = pack_bf16x2(m[6], m[7]);
    reinterpret_cast<uint4*>(out)[t] = o;
  }
}

__global__ void avgpool_kernel(const ActionBlock* ab, const __nv_bfloat16* __restrict__ in,
                               float* __restrict__ pooled, int batch, int HW, int C) {
  griddep_wait();
  griddep_trigger();
  if (ab->skip) return;
  const int chunks = C / 8;
  const int total = batch * chunks;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int j = t % chunks;
  const int n = t / chunks;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const __nv_bfloat16* base = in + (long long)n * HW * C + j * 8;
  for (int p = 0; p < HW; ++p) {
    uint4 u = *reinterpret_cast<const uint4*>(base + (long long)p * C);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      acc[2 * e] += f.x;
      acc[2 * e + 1] += f.y;
    }
  }
  const float inv = 1.0f / (float)HW;
  float4* o = reinterpret_cast<float4*>(pooled + (long long)n * C + j * 8);
  o[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
  o[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
}

// logits[n][j] = pooled[n] . W[j] + bias[j]. One CTA per 8 classes (one warp
// each); the pooled features of the whole batch are staged in shared memory
// once per CTA, the class's weight row lives in registers. C % 256 == 0, C <= 2048.
__global__ void fc_kernel(const ActionBlock* ab, const float* __restrict__ pooled, int layer,
                          int batch, int C, int classes) {
  extern __shared__ float sp[];  // [batch][C]
  griddep_wait();
  griddep_trigger();
  if (ab->skip) return;
  for (int i = threadIdx.x * 4; i < batch * C; i += blockDim.x * 4)
    *reinterpret_cast<float4*>(sp + i) = __ldcg(reinterpret_cast<const float4*>(pooled + i));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= classes) return;
  const uint8_t* hdr = ab->hdr;
  const __nv_bfloat16* w =
      reinterpret_cast<const __nv_bfloat16* const*>(hdr + kHdrWeightOff)[layer] + (long long)j * C;
  const float* bias = reinterpret_cast<const float* const*>(hdr + kHdrBiasOff)[layer];
  const int chunks = C / 256;  // 16-byte weight chunks per lane
  float wf[64];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (i < chunks) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(w + (i * 32 + lane) * 8));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        wf[i * 8 + 2 * e] = f.x;
        wf[i * 8 + 2 * e + 1] = f.y;
      }
    }
  }
  const float b = __ldg(bias + j);
  for (int n = 0; n < batch; ++n) {
    const float* pn = sp + n * C;
    float acc = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < chunks) {
        const float4 p0 = *reinterpret_cast<const float4*>(pn + (i * 32 + lane) * 8);
        const float4 p1 = *reinterpret_cast<const float4*>(pn + (i * 32 + lane) * 8 + 4);
        acc += wf[i * 8 + 0] * p0.x + wf[i * 8 + 1] * p0.y + wf[i * 8 + 2] * p0.z +
               wf[i * 8 + 3] * p0.w + wf[i * 8 + 4] * p1.x + wf[i * 8 + 5] * p1.y +
               wf[i * 8 + 6] * p1.z + wf[i * 8 + 7] * p1.w;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ab->out[n][j] = acc + b;
  }
}

// ------------------------------------------------------------------ launchers

static int grid_for(long long total, int threads) {
  long long g = (total + threads - 1) / threads;
  const long long cap = 148LL * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

void launch_gate(ActionBlock* ab, const ActionDesc* ring, uint32_t mask, uint64_t* ctr,
                 ExecRecord* recs, cudaStream_t st) {
  gate_kernel<<<1, 64, 0, st>>>(ab, ring, mask, ctr, recs);
}
cudaError_t configure_simt() {
  return cudaFuncSetAttribute(fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kMaxBatch * 2048 * 4);
}

template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

void launch_exec_done(const ActionBlock* ab, uint32_t mask, ExecRecord* recs, cudaStream_t st) {
  launch_pdl(exec_done_kernel, dim3(1), dim3(1), 0, st, ab, mask, recs);
}
void launch_out_done(ExecRecord* rec, uint64_t seq, cudaStream_t st) {
  out_done_kernel<<<1, 1, 0, st>>>(rec, seq);
}
void launch_stamp(volatile uint64_t* slot, uint64_t tag, cudaStream_t st) {
  stamp_kernel<<<1, 1, 0, st>>>(slot, tag);
}
void launch_clock_pub(volatile uint64_t* slot, uint64_t max_ns, cudaStream_t st) {
  clock_pub_kernel<<<1, 1, 0, st>>>(slot, max_ns);
}
void launch_stem_im2col(const ActionBlock* ab, void* a, int batch, int H, int W, int OH, int OW,
                        int kpad, cudaStream_t st) {
  long long total = (long long)batch * OH * OW * (kpad / 8);
  launch_pdl(stem_im2col_kernel, dim3(grid_for(total, 256)), dim3(256), 0, st, ab,
             reinterpret_cast<__nv_bfloat16*>(a), batch, H, W, OH, OW, kpad);
}
void launch_maxpool(const ActionBlock* ab, const void* in, void* out, int batch, int H, int W,
                    int C, int OH, int OW, cudaStream_t st) {
  long long total = (long long)batch * OH * OW * (C / 8);
  launch_pdl(maxpool3x3s2_kernel, dim3(grid_for(total, 256)), dim3(256), 0, st, ab,
             reinterpret_cast<const __nv_bfloat16*>(in), reinterpret_cast<__nv_bfloat16*>(out),
             batch, H, W, C, OH, OW);
}
void launch_avgpool(const ActionBlock* ab, const void* in, float* pooled, int batch, int HW, int C,
                    cudaStream_t st) {
  int total = batch * (C / 8);
  launch_pdl(avgpool_kernel, dim3((total + 127) / 128), dim3(128), 0, st, ab,
             reinterpret_cast<const __nv_bfloat16*>(in), pooled, batch, HW, C);
}
void launch_fc(const ActionBlock* ab, const float* pooled, int layer, int batch, int C, int classes,
               cudaStream_t st) {
  launch_pdl(fc_kernel, dim3((classes + 7) / 8), dim3(256), (size_t)batch * C * 4, st, ab, pooled,
             layer, batch, C, classes);
}

}  // namespace cw
