// The INFER megakernel: the whole batched CNN forward of one Exec in ONE
// persistent launch (replaces the emulated Exec wait of the reference worker,
// pkg/src/sloserve/worker.py:273-277 `dur = exec_duration[b]; call_at(now+dur)`).
//
// Grid = one CTA per SM (148 on B200), 384 threads (3 warpgroups), ~227 KB of
// shared memory. Every CTA walks the plan (mk.h) layer by layer; the tasks of a
// layer are dealt round-robin (rotated per layer) over the CTAs. Warp roles:
//
//   warpgroup 0 (setmaxnreg 120)
//     warp 0   TMA producer. For each of the CTA's conv tasks, per k-block: the
//              weight tile (B, K-major, from the model's paged weights through
//              the per-model tensor map in the model header) and the activation
//              tile (A): mode 0 a [M][K] matrix box, mode 1 a tap-shifted NHWC
//              box (implicit GEMM; padding = TMA out-of-bounds zero fill,
//              stride = TMA element stride), mode 2 the stem's 11 padded input
//              rows of one pooled row (one box per task, read by the MMAs as an
//              implicit im2col with overlapping no-swizzle rows), mode 3 the
//              3x3/s1 row box shared by the three horizontal taps; a fused
//              projection shortcut adds a second K segment (its own A map and
//              weights). Weight tiles of a layer's first task are issued BEFORE
//              waiting for the layer's inputs.
//     warp 1   tcgen05.mma issuer (one elected thread): M=128, N=bn, K=16 steps,
//              fp32 accumulators in TMEM, two 256-column accumulators so the
//              epilogue of task i overlaps the MMAs of task i+1.
//     warps 2-3 the DenseNet BN+ReLU A-tile prologue and the optional softmax
//              tail; idle otherwise.
//   warpgroups 1-2 (setmaxnreg 192): eight epilogue warps, two per TMEM lane
//              quarter (group g = columns [32g, 32g+32) of every 64-column
//              chunk): tcgen05.ld -> + bias (folded BatchNorm), + residual,
//              ReLU -> bf16 into a 128-byte-swizzled staging buffer -> TMA
//              store (branch-free per residual / ReLU variant); or fp32 split-K
//              partials, the cluster split-K reduction through distributed shared
//              memory, the stem's 3x3/s2 max pool, or the fused global average
//              pool. The same warps run the SIMT layers (input conversion, max
//              pool, avg pool, BN pool, im2col, split-K reduce, FC + logits).
//
// Layer completion: after a layer's stores, one epilogue thread per CTA adds its
// task count to counter[L]; consumers spin with relaxed loads, then one acquire
// load (plus an async-proxy fence before TMA reads). Waits time out (trap) rather
// than hang the GPU if the plan were ever inconsistent.
//
// Memory-model note (hardware assumption, see red_after_bulk_add): layers whose every
// global write is a TMA / bulk store publish with a RELAXED add after
// cp.async.bulk.wait_group 0 + fence.proxy.async; build with -DCW_STRICT_RELEASE to
// publish every layer with red.release instead (tests/test_gpu_strict_release.py).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "cw_device.h"
#include "mk.h"
#include "ptx.cuh"

namespace cw {

__constant__ MkLayer c_plan[kMkMaxPlanLayers];  // the running INFER's plan (see mk.h)

// residual chunks land this many chunks ahead of their use (<= kMkOutBufs - 1)
#ifndef CW_RES_DIST
#define CW_RES_DIST 3
#endif
constexpr int kResDist = CW_RES_DIST;
#ifndef CW_TIMEOUT_NS
#define CW_TIMEOUT_NS 2000000000ull  // 2 s: far above any INFER (sanitizer builds: raised)
#endif
constexpr uint64_t kMkTimeoutNs = CW_TIMEOUT_NS;

// L2 residency policies: the weights stream (every INFER may run another model copy: evict
// first), a layer's outputs are the next layer's inputs (evict last: keep the activation
// working set in the 126 MB L2 instead of writing it back), a residual is read for the
// last time (evict first). CW_NO_L2_HINTS: every access at normal priority.
#ifdef CW_NO_L2_HINTS
constexpr uint64_t kHintW = 0x1000000000000000ull, kHintOut = 0x1000000000000000ull,
                   kHintRes = 0x1000000000000000ull;
#else
constexpr uint64_t kHintW = kL2EvictFirst, kHintOut = kL2EvictLast, kHintRes = kL2EvictFirst;
#endif

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Completion count of a layer whose every global write was a TMA store issued by THIS
// thread and already waited for with cp.async.bulk.wait_group 0 (writes performed at
// their L2 home) + fence.proxy.async: the consumers only read those bytes after seeing
// the count (TMA loads served by L2, or generic loads behind their acquire load, which
// invalidates L1). red.release would add a MEMBAR.ALL.GPU that waits for every memory
// operation in flight on the SM (the producer's prefetch of the next layer): ~0.65 us
// per layer boundary (b=1 324 -> 280 us, b=16 568 -> 533 us). Layers with generic
// stores (SIMT layers, the fused average pool) keep red_release_add.
//
// HARDWARE ASSUMPTION (outside the PTX memory model): a relaxed RMW gives no
// happens-before edge, so this relies on bulk-async writes that wait_group 0 reported
// complete being visible at L2 to any later reader of the count, which holds on sm_100
// (every consumer reads through TMA / L2 or behind its own acquire load; thousands of
// alternating-input INFERs reproduce bit for bit, tools/handoff_stress.py). Builds with
// -DCW_STRICT_RELEASE use red.release.gpu here (one MEMBAR per layer boundary, slower).
__device__ __forceinline__ void red_after_bulk_add(uint32_t* p, uint32_t v) {
#ifdef CW_STRICT_RELEASE
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __noinline__ void mk_timeout(int where) {
  printf("cw megakernel: wait timeout (site %d, block %d, thread %d)\n", where, blockIdx.x,
         threadIdx.x);
  __trap();
}

// Phase wait with a suspend-time hint: a waiting thread sleeps in hardware
// until the phase completes (or the hint expires) instead of spinning, so the
// four epilogue warps waiting on an accumulator do not steal issue slots from
// the producer / MMA threads that share their SM sub-partitions.
template <uint32_t kHintNs>
__device__ __forceinline__ bool mbar_try_wait_hint(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "n"(kHintNs)
      : "memory");
  return ok != 0;
}

// ptxas turns the hint into a NANOSLEEP between checks, i.e. the wake-up
// granularity of a waiting warp.
#ifndef CW_HINT_EPI
#define CW_HINT_EPI 512
#endif
constexpr uint32_t kEpiWaitNs = CW_HINT_EPI;

__device__ __forceinline__ bool mbar_try_wait_nohint(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

template <uint32_t kHintNs>
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  if constexpr (kHintNs == 0) return mbar_try_wait_nohint(bar, parity);
  else return mbar_try_wait_hint<kHintNs>(bar, parity);
}

#ifndef CW_HINT_EMPTY
#define CW_HINT_EMPTY 256
#endif
#ifndef CW_HINT_FULL
#define CW_HINT_FULL 32
#endif
#ifndef CW_HINT_TEMPTY
#define CW_HINT_TEMPTY 512
#endif

template <uint32_t kHintNs = 64>
__device__ __forceinline__ void mbar_wait_to(uint32_t bar, uint32_t parity, int site) {
  if (mbar_try<kHintNs>(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try<kHintNs>(bar, parity)) {
    if (globaltimer() - t0 > kMkTimeoutNs) mk_timeout(site);
  }
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spin with relaxed loads (an acquire load invalidates the SM's L1 every time:
// CCTL.IVALL; the timer is read every 64 polls), then ONE acquire load once the count
// is reached. Not fence.acq_rel.gpu: its MEMBAR.ALL.GPU also waits for the warp's
// in-flight bulk copies (the producer's weight prefetch), ~0.5 us per layer boundary
// (b=16 595 -> 568 us, b=1 356 -> 324 us). The counter only grows, so the acquire load
// reads a value of the release sequence of every contributing red.release.
__device__ __noinline__ void mk_dep_timeout(int site, int layer, int dep, uint32_t have,
                                            uint32_t want) {
  printf("cw megakernel: dependency timeout (site %d, block %d, layer %d waits for layer %d: "
         "count %u of %u)\n", site, blockIdx.x, layer, dep, have, want);
  __trap();
}

__device__ __forceinline__ void wait_count(const uint32_t* c, uint32_t target, int site,
                                           int layer = -1, int dep = -1) {
  if ((int32_t)(ld_relaxed_u32(c) - target) < 0) {
    const uint64_t t0 = globaltimer();
    uint32_t it = 0;
    while ((int32_t)(ld_relaxed_u32(c) - target) < 0) {
      // (twice the in-layer timeout: a layer that hangs reports its own wait site first)
      if ((++it & 63) == 0 && globaltimer() - t0 > 2 * kMkTimeoutNs)
        mk_dep_timeout(site, layer, dep, ld_relaxed_u32(c), target);
    }
  }
  (void)ld_acquire_u32(c);
}

// Wait until every dependency layer of `d` has completed in this generation.
// (reads the dependency list from the smem plan: a register copy of the layer
// indexed dynamically would be demoted to local memory)
__device__ __forceinline__ void wait_deps(const MkLayer* sl, int L, const uint32_t* counters,
                                          uint32_t gen1, int site) {
  const int nd = sl[L].ndeps;
  for (int i = 0; i < nd; ++i) {
    const int p = sl[L].deps[i];
    wait_count(counters + p, gen1 * (uint32_t)sl[p].tasks, site, L, p);
  }
}

// UMMA shared-memory descriptor, K-major, 64-byte swizzle (rows of 32 bf16,
// 8-row atoms 512 B apart).
__device__ __forceinline__ uint64_t sw64_kmajor_desc(uint32_t smem_addr) {
  return (uint64_t)((smem_addr & 0x3FFFFu) >> 4) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) |
         (4ull << 61);
}

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows x 16 B, rows
// 16 B apart; lbo = byte distance of K-adjacent core matrices, sbo = of M-adjacent ones. Rows
// may overlap (lbo 16): the stem's implicit im2col (tools/umma_overlap_probe.cu checks it).
__device__ __forceinline__ uint64_t desc_none(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((smem_addr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ int first_task(const MkLayer& d, int cta, int G) {
  int t = cta - d.rot % G;
  return t < 0 ? t + G : t;
}

// K range of split z: [kb0, kb1), balanced over units of one k-block (mode 3: one kernel row
// of one channel block = 3 k-blocks); the planner keeps every split non-empty.
__device__ __forceinline__ void split_range(const MkLayer& d, int z, int& kb0, int& kb1) {
  const int u = d.mode == 3 ? 3 : 1;
  const int units = d.num_kb / u;
  kb0 = units * z / d.splits * u;
  kb1 = units * (z + 1) / d.splits * u;
}

// Rows of the A tile (output pixels) for one task.
__device__ __forceinline__ uint32_t a_rows(const MkLayer& d) {
  return d.mode == 0 ? 128u : (uint32_t)(d.box_w * d.box_h * d.box_n);
}

struct TileOrigin {
  int m0, ow0, oh0, img0, n0;
};

__device__ __forceinline__ TileOrigin tile_origin(const MkLayer& d, int tile) {
  TileOrigin o;
  const int mt = tile / d.n_tiles;
  o.n0 = (tile - mt * d.n_tiles) * d.bn;
  o.m0 = 0;
  o.ow0 = o.oh0 = o.img0 = 0;
  if (d.mode == 0) {
    o.m0 = mt * 128;
  } else {
    const int tw = mt % d.tiles_w;
    const int th = (mt / d.tiles_w) % d.tiles_h;
    const int tn = mt / (d.tiles_w * d.tiles_h);
    if (d.pool_pw) {  // fused stem max pool: tile = pooled row th, pooled columns from tw*pool_pw
      o.ow0 = 2 * tw * d.pool_pw - 1;
      o.oh0 = 2 * th - 1;
    } else {
      o.ow0 = tw * d.box_w;
      o.oh0 = th * d.box_h;
    }
    o.img0 = tn * d.box_n;
  }
  return o;
}

// Output row index (NHWC pixel) of accumulator row `row` in a tile; false if padding.
__device__ __forceinline__ bool row_pixel(const MkLayer& d, const TileOrigin& o, int row,
                                          long long* m) {
  if (d.mode == 0) {
    *m = (long long)o.m0 + row;
    return *m < d.m_total;
  }
  const int rows = d.box_w * d.box_h * d.box_n;
  const int wi = row % d.box_w;
  const int t = row / d.box_w;
  const int hi = t % d.box_h;
  const int ni = t / d.box_h;
  const int ow = o.ow0 + wi, oh = o.oh0 + hi, n = o.img0 + ni;
  *m = ((long long)n * d.oh + oh) * d.ow + ow;
  return row < rows && ow >= 0 && oh >= 0 && ow < d.ow && oh < d.oh && n < d.nimg;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}

// ------------------------------------------------------------------ SIMT layers
// All run on the kMkEpiThreads epilogue threads of every CTA (et = 0..255, G CTAs).

// fp32 [C=3][H][W] per request -> bf16 [n][H][W + 2*pad][4] (pixel data at column + pad).
// The CTA's image rows (a contiguous range of (n, h)) come in by bulk copies (plane-major,
// up to 64 KB per phase into the epilogue staging buffers): generic loads would be capped by
// the few KB of L1 the megakernel leaves; the conversion then reads shared memory only.
__device__ __forceinline__ void simt_input(const MkLayer& d, const ActionBlock* ab, int cta, int G,
                                        int et, float* stage, uint32_t stage_addr,
                                        uint32_t stage_bytes, uint32_t bar, uint32_t& phase) {
  const int W = d.W, H = d.H, W4 = W / 4, Wp = W + 2 * kMkPadW;
  const int rows_total = d.batch * H;
  const int R = (rows_total + G - 1) / G;
  const int r0 = cta * R, r1 = min(rows_total, r0 + R);
  const int P = (int)(stage_bytes / (3u * W * 4u));  // rows per phase
  const long long plane = (long long)H * W;
  uint2* out = reinterpret_cast<uint2*>(d.out);
  for (int pr = r0; pr < r1; pr += P) {
    const int pe = min(r1, pr + P), nr = pe - pr;
    if (et == 0) {
      mbar_arrive_expect_tx(bar, (uint32_t)(3 * nr * W * 4));
      for (int a = pr; a < pe;) {
        const int n = a / H, h = a - n * H;
        const int b = min(pe, (n + 1) * H);  // rows of this image in the phase
        for (int p = 0; p < 3; ++p)
          bulk_g2s(stage_addr + (uint32_t)((p * P + (a - pr)) * W * 4),
                   ab->in[n] + p * plane + (long long)h * W, (uint32_t)((b - a) * W * 4), bar);
        a = b;
      }
    }
    mbar_wait_to<64>(bar, phase & 1, 12);
    ++phase;
    for (int it = et; it < nr * W4; it += kMkEpiThreads) {
      const int i = it / W4, w4 = it - i * W4;
      const int a = pr + i, n = a / H, h = a - n * H;
      const float4 r = *reinterpret_cast<const float4*>(stage + (0 * P + i) * W + w4 * 4);
      const float4 g = *reinterpret_cast<const float4*>(stage + (1 * P + i) * W + w4 * 4);
      const float4 b = *reinterpret_cast<const float4*>(stage + (2 * P + i) * W + w4 * 4);
      uint2* o = out + ((long long)n * (H + 2 * kMkPadH) + h + kMkPadH) * Wp + kMkPadW + w4 * 4;
      uint4 p0, p1;
      p0.x = pack_bf16x2(r.x, g.x);
      p0.y = pack_bf16x2(b.x, 0.0f);
      p0.z = pack_bf16x2(r.y, g.y);
      p0.w = pack_bf16x2(b.y, 0.0f);
      p1.x = pack_bf16x2(r.z, g.z);
      p1.y = pack_bf16x2(b.z, 0.0f);
      p1.z = pack_bf16x2(r.w, g.w);
      p1.w = pack_bf16x2(b.w, 0.0f);
      reinterpret_cast<uint4*>(o)[0] = p0;
      reinterpret_cast<uint4*>(o)[1] = p1;
    }
    named_bar(1, kMkEpiThreads);  // the stage is read before the next phase overwrites it
  }
}

// 3x3 max pool, stride / padding from the plan (padding = -inf: skipped), input channel
// stride in_ctot, output at the layer's channel slice of a buffer of stride out_ctot. One
// thread per (output pixel, 8-channel chunk); the maxima on packed bf16 pairs (exact: the
// max of bf16 values is one of them, as it was through fp32).
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&a),
                             *reinterpret_cast<const __nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
// Issue the 9 window loads of item t (padding taps read a clamped in-bounds pixel and are
// masked to -inf afterwards: no branches between the loads).
__device__ __forceinline__ void maxpool_loads(const MkLayer& d, const __nv_bfloat16* in, int t,
                                              int chunks, uint4 (&v)[9], uint32_t& valid,
                                              long long& out_off) {
  const int H = d.H, W = d.W, OW = d.OW, OH = d.OH;
  const long long ct = d.in_ctot;
  const int p = t / chunks;
  const int j = t - p * chunks;
  const int q = p / OW;
  const int ow = p - q * OW;
  const int n = q / OH;
  const int oh = q - n * OH;
  const int ih0 = oh * d.stride - d.pad, iw0 = ow * d.stride - d.pad;
  const __nv_bfloat16* base = in + ((long long)n * H * W) * ct + j * 8;
  valid = 0;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int ih = ih0 + r, iw = iw0 + s;
      const bool ok = ih >= 0 && ih < H && iw >= 0 && iw < W;
      valid |= (ok ? 1u : 0u) << (r * 3 + s);
      const int ihc = min(max(ih, 0), H - 1), iwc = min(max(iw, 0), W - 1);
      v[r * 3 + s] = __ldcg(reinterpret_cast<const uint4*>(base + ((long long)ihc * W + iwc) * ct));
    }
  }
  out_off = (long long)p * d.out_ctot + j * 8;
}
__device__ __forceinline__ uint4 maxpool_reduce(const uint4 (&v)[9], uint32_t valid) {
  uint4 m = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);  // -inf
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    if (!((valid >> i) & 1u)) continue;
    m.x = bmax2(m.x, v[i].x);
    m.y = bmax2(m.y, v[i].y);
    m.z = bmax2(m.z, v[i].z);
    m.w = bmax2(m.w, v[i].w);
  }
  return m;
}
__device__ __forceinline__ void simt_maxpool(const MkLayer& d, int cta, int G, int et) {
  const __nv_bfloat16* in = reinterpret_cast<const __nv_bfloat16*>(d.in);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(d.out);
  const int chunks = d.C / 8;
  const int total = d.batch * d.OH * d.OW * chunks;
  for (int t = cta * kMkEpiThreads + et; t < total; t += G * kMkEpiThreads) {
    uint4 v[9];
    uint32_t valid;
    long long o;
    maxpool_loads(d, in, t, chunks, v, valid, o);
    *reinterpret_cast<uint4*>(out + o) = maxpool_reduce(v, valid);
  }
}

// Per-channel BatchNorm + ReLU of an input (DenseNet pre-activation): the header's
// scale[cpad] / shift[cpad] table of layer `pre`, 8 channels from c.
struct BnRelu8 {
  float s[8], h[8];
  __device__ __forceinline__ void load(const float* tab, int cpad, int c) {
    const float4 s0 = __ldg(reinterpret_cast<const float4*>(tab + c));
    const float4 s1 = __ldg(reinterpret_cast<const float4*>(tab + c + 4));
    const float4 h0 = __ldg(reinterpret_cast<const float4*>(tab + cpad + c));
    const float4 h1 = __ldg(reinterpret_cast<const float4*>(tab + cpad + c + 4));
    s[0] = s0.x; s[1] = s0.y; s[2] = s0.z; s[3] = s0.w;
    s[4] = s1.x; s[5] = s1.y; s[6] = s1.z; s[7] = s1.w;
    h[0] = h0.x; h[1] = h0.y; h[2] = h0.z; h[3] = h0.w;
    h[4] = h1.x; h[5] = h1.y; h[6] = h1.z; h[7] = h1.w;
  }
  __device__ __forceinline__ void apply(float* f) const {
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = fmaxf(fmaf(f[e], s[e], h[e]), 0.0f);
  }
};

__device__ __forceinline__ const float* pre_table(const uint8_t* hdr, int layer) {
  return reinterpret_cast<const float* const*>(hdr + kHdrPreOff)[layer];
}

// Global average pool -> fp32 [b][C]; with an input BatchNorm (DenseNet's norm5 + ReLU)
// applied to every pixel first.
__device__ __forceinline__ void simt_avgpool(const MkLayer& d, const uint8_t* hdr, int cta, int G,
                                             int et) {
  const __nv_bfloat16* in = reinterpret_cast<const __nv_bfloat16*>(d.in);
  const int chunks = d.C / 8;
  const int total = d.batch * chunks;
  const int HW = d.H * d.W;
  const int cpad = (d.C + 63) / 64 * 64;
  const float* tab = d.pre_layer >= 0 ? pre_table(hdr, d.pre_layer) : nullptr;
  float* pooled = reinterpret_cast<float*>(d.out);
  for (int t = cta * kMkEpiThreads + et; t < total; t += G * kMkEpiThreads) {
    const int j = t % chunks;
    const int n = t / chunks;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, f[8];
    const __nv_bfloat16* base = in + (long long)n * HW * d.in_ctot + j * 8;
    if (tab) {  // (BN + ReLU per pixel: the scale / shift loads hit L1)
      for (int p = 0; p < HW; ++p) {
        bf16x8_to_f32(__ldcg(reinterpret_cast<const uint4*>(base + (long long)p * d.in_ctot)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          acc[e] += fmaxf(fmaf(f[e], __ldg(tab + j * 8 + e), __ldg(tab + cpad + j * 8 + e)), 0.0f);
      }
    } else {
      for (int p = 0; p < HW; ++p) {
        bf16x8_to_f32(__ldcg(reinterpret_cast<const uint4*>(base + (long long)p * d.in_ctot)), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += f[e];
      }
    }
    const float inv = 1.0f / (float)HW;
    float4* o = reinterpret_cast<float4*>(pooled + (long long)n * d.C + j * 8);
    o[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    o[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
  }
}

// DenseNet transition prefix: BatchNorm + ReLU, then the 2x2 / stride-2 average pool, into
// a bf16 buffer the transition's 1x1 conv reads (pool before conv: both linear).
__device__ __forceinline__ void simt_bnpool(const MkLayer& d, const uint8_t* hdr, int cta, int G,
                                            int et) {
  const __nv_bfloat16* in = reinterpret_cast<const __nv_bfloat16*>(d.in);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(d.out);
  const int chunks = d.C / 8;
  const int total = d.batch * d.OH * d.OW * chunks;
  const int cpad = (d.C + 63) / 64 * 64;
  const float* tab = pre_table(hdr, d.pre_layer);
  for (int t = cta * kMkEpiThreads + et; t < total; t += G * kMkEpiThreads) {
    const int j = t % chunks;
    const int p = t / chunks;
    const int ow = p % d.OW;
    const int oh = (p / d.OW) % d.OH;
    const int n = p / (d.OW * d.OH);
    BnRelu8 bn;
    bn.load(tab, cpad, j * 8);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, f[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ih = 2 * oh + (q >> 1), iw = 2 * ow + (q & 1);
      bf16x8_to_f32(__ldcg(reinterpret_cast<const uint4*>(
                        in + (((long long)n * d.H + ih) * d.W + iw) * d.in_ctot + j * 8)), f);
      bn.apply(f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += f[e];
    }
    uint4 o;
    o.x = pack_bf16x2(0.25f * acc[0], 0.25f * acc[1]);
    o.y = pack_bf16x2(0.25f * acc[2], 0.25f * acc[3]);
    o.z = pack_bf16x2(0.25f * acc[4], 0.25f * acc[5]);
    o.w = pack_bf16x2(0.25f * acc[6], 0.25f * acc[7]);
    *reinterpret_cast<uint4*>(out + (long long)p * d.out_ctot + j * 8) = o;
  }
}

// First conv of a net whose input is not NHWC4-friendly (Inception-v3: 3 channels at
// 299x299, 3x3/s2 valid): patches of the fp32 NCHW request images -> bf16 [M][64] rows
// (k = (r*KW + s)*C + c, zero past KH*KW*C), the A operand of a 1x1-shaped GEMM. One
// thread per output pixel: consecutive threads read stride-2 columns of the same rows.
// The layer is load-latency bound (8 warps per SM): 3x3 kernels over 3 channels (the only
// user) issue all 27 loads of a pixel at once, (c, r, s) of every k resolved at compile
// time; other shapes take the generic loop (two pixels per round spill the epilogue warps'
// registers: measured slower).
// 3x3 x 3-channel patch of output pixel m: its 27 loads issued together (k >= 27 zero).
__device__ __forceinline__ void im2col_33_loads(const MkLayer& d, const ActionBlock* ab, int m,
                                                float (&f)[32]) {
  const int OW = d.OW, OH = d.OH, H = d.H, W = d.W;
  const long long plane = (long long)H * W;
  const int t = m / OW;
  const int ow = m - t * OW;
  const int n = t / OH;
  const int oh = t - n * OH;
  const int ih0 = oh * d.stride - d.pad, iw0 = ow * d.stride - d.pad;
  const float* img = ab->in[n];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int c = k % 3, r = (k / 3) / 3, s = (k / 3) % 3;
    const int ih = ih0 + r, iw = iw0 + s;
    f[k] = (k < 27 && ih >= 0 && ih < H && iw >= 0 && iw < W)
               ? __ldg(img + c * plane + (long long)ih * W + iw) : 0.0f;
  }
}
__device__ __forceinline__ void im2col_33_store(uint4* o, const float (&f)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    o[q] = make_uint4(pack_bf16x2(f[8 * q], f[8 * q + 1]), pack_bf16x2(f[8 * q + 2], f[8 * q + 3]),
                      pack_bf16x2(f[8 * q + 4], f[8 * q + 5]), pack_bf16x2(f[8 * q + 6], f[8 * q + 7]));
#pragma unroll
  for (int q = 4; q < 8; ++q) o[q] = make_uint4(0u, 0u, 0u, 0u);
}
__device__ __forceinline__ void simt_im2col(const MkLayer& d, const ActionBlock* ab, int cta,
                                            int G, int et) {
  uint4* out = reinterpret_cast<uint4*>(d.out);
  const int K = d.kw, C = d.C, st = d.stride, pd = d.pad, OW = d.OW, OH = d.OH, H = d.H, W = d.W;
  const int total = d.batch * OH * OW;
  const int step = G * kMkEpiThreads;
  if (K == 3 && C == 3) {
    for (int m = cta * kMkEpiThreads + et; m < total; m += step) {
      float f[32];
      im2col_33_loads(d, ab, m, f);
      im2col_33_store(out + (long long)m * 8, f);
    }
    return;
  }
  const long long plane = (long long)H * W;
  const int kkc = K * K * C;
  for (int m = cta * kMkEpiThreads + et; m < total; m += step) {
    const int t = m / OW;
    const int ow = m - t * OW;
    const int n = t / OH;
    const int oh = t - n * OH;
    const int ih0 = oh * st - pd, iw0 = ow * st - pd;
    const float* img = ab->in[n];
    uint4* o = out + (long long)m * 8;
    for (int q = 0; q < 8; ++q) {
      float f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = 8 * q + e;
        const int c = k % C, rs = k / C, s = rs % K, r = rs / K;
        const int ih = ih0 + r, iw = iw0 + s;
        f[e] = (k < kkc && ih >= 0 && ih < H && iw >= 0 && iw < W)
                   ? __ldg(img + c * plane + (long long)ih * W + iw) : 0.0f;
      }
      o[q] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                        pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
    }
  }
}

// logits[n][j] = pooled[n] . W[j] + bias[j]. Each CTA takes blocks of <= 8 classes. The
// pooled features [batch][C] fp32 (into the idle ring) and the block's weight rows (into the
// staging buffers) arrive by bulk copies; the 128 threads are (image n) x (128 / pow2(batch)
// K parts, interleaved 8-element chunks): a thread reads its part of pooled[n] once per block
// and accumulates all the block's classes from it, then the K parts reduce (shuffles, and
// shared memory when an image spans several warps). C % 64 == 0, batch <= 16.
// Warp reduce-scatter of V per-lane partial sums (V = 8 or 16, a power of two <= 32):
// log2(V) halving exchanges (offsets 16, 8, ...) then full exchanges, so every value is
// summed over the 32 lanes with V - 1 + 5 - log2(V) shuffles instead of 5 V. Lane l ends
// with value index fc_rs_index<V>(l).
template <int V>
__device__ __forceinline__ float fc_reduce_scatter(float (&v)[V], int lane) {
  int o = 16;
#pragma unroll
  for (int h = V / 2; h >= 1; h /= 2, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  float r = v[0];
  for (; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}
template <int V>
__device__ __forceinline__ int fc_rs_index(int lane) {
  int idx = 0, o = 16;
  for (int h = V / 2; h >= 1; h /= 2, o >>= 1) idx += (lane & o) ? h : 0;
  return idx;
}

// Partial dot products of NI images x 8 classes over this thread's interleaved 8-element K
// chunks (consecutive threads read consecutive 16-byte words of the staged rows).
template <int NI>
__device__ __forceinline__ void fc_mac(const float* const (&pn)[NI], const __nv_bfloat16* sw, int C,
                                       int k0, int kstep, float (&acc)[NI * 8]) {
#pragma unroll
  for (int i = 0; i < NI * 8; ++i) acc[i] = 0.0f;
#pragma unroll 2
  for (int k = k0; k < C; k += kstep) {
    uint4 wv[8];  // all 8 rows' words first (rows >= nj hold stale data: sums discarded)
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) wv[jj] = *reinterpret_cast<const uint4*>(sw + jj * C + k);
#pragma unroll
    for (int ii = 0; ii < NI; ++ii) {
      const float4 p0 = *reinterpret_cast<const float4*>(pn[ii] + k);
      const float4 p1 = *reinterpret_cast<const float4*>(pn[ii] + k + 4);
      const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const uint32_t u = e2 == 0 ? wv[jj].x : e2 == 1 ? wv[jj].y : e2 == 2 ? wv[jj].z : wv[jj].w;
          float& a = acc[ii * 8 + jj];
          a = fmaf(__uint_as_float(u << 16), pv[2 * e2], a);
          a = fmaf(__uint_as_float(u & 0xFFFF0000u), pv[2 * e2 + 1], a);
        }
      }
    }
  }
}

// Fully connected layer over the pooled features (fp32 [batch][C]) with bf16 weights
// [classes][C]: CTA g takes classes 8g..8g+7; the pooled block and the weight rows are
// bulk-copied into shared memory. Batch <= 8: an image per group of 256/nbp threads, each
// thread 8 classes x its K chunks, warp reduce-scatter, then the image's warps through
// shared memory. Batch 9..16: a warp per image pair (images w and w+8), 2 x 8 sums per
// thread: half the shared-memory weight reads per FMA.
// The CTA's first weight block does not depend on the previous layers: requested (with the
// transaction bytes of the pooled block too) before the dependency wait.
__device__ __forceinline__ void simt_fc_prefetch(const MkLayer& d, const uint8_t* hdr, int cta,
                                                 uint32_t sw_addr, uint32_t bar) {
  if (cta >= (d.classes + 7) / 8) return;
  const __nv_bfloat16* wbase =
      reinterpret_cast<const __nv_bfloat16* const*>(hdr + kHdrWeightOff)[d.wlayer];
  const int j0 = cta * 8, nj = min(8, d.classes - j0);
  const uint32_t wbytes = (uint32_t)(nj * d.C * 2);
  mbar_arrive_expect_tx(bar, wbytes + (uint32_t)(d.batch * d.C * 4));
  bulk_g2s(sw_addr, wbase + (size_t)j0 * d.C, wbytes, bar);
}
__device__ __forceinline__ void simt_fc(const MkLayer& d, const ActionBlock* ab, const uint8_t* hdr,
                                     int cta, int G, int et, float* sp, uint32_t sp_addr,
                                     const __nv_bfloat16* sw, uint32_t sw_addr, float* sred,
                                     uint32_t bar, uint32_t& phase) {
  const int C = d.C;
  int nbp = 1;
  while (nbp < d.batch) nbp <<= 1;
  const int lane = et & 31, warp = et >> 5;
  const __nv_bfloat16* wbase =
      reinterpret_cast<const __nv_bfloat16* const*>(hdr + kHdrWeightOff)[d.wlayer];
  const float* bias = reinterpret_cast<const float* const*>(hdr + kHdrBiasOff)[d.wlayer];
  const int ngroups = (d.classes + 7) / 8;
  bool pooled_in = false;
  for (int g = cta; g < ngroups; g += G) {
    const int j0 = g * 8;
    const int nj = min(8, d.classes - j0);
    if (et == 0) {
      fence_proxy_async();  // pooled was written by generic stores of other CTAs
      const uint32_t wbytes = (uint32_t)(nj * C * 2);
      const uint32_t pbytes = pooled_in ? 0u : (uint32_t)(d.batch * C * 4);
      if (pooled_in) {
        mbar_arrive_expect_tx(bar, wbytes);
        bulk_g2s(sw_addr, wbase + (size_t)j0 * C, wbytes, bar);
      } else {  // first block: its weights were requested by simt_fc_prefetch
        bulk_g2s(sp_addr, d.in, pbytes, bar);
      }
    }
    pooled_in = true;
#ifdef CW_KB_TRACE
    const long long tf0 = clock64();
#endif
    mbar_wait_to<64>(bar, phase & 1, 10);
    ++phase;
#ifdef CW_KB_TRACE
    const long long tf1 = clock64();
#endif
    if (nbp > 8) {
      // warp w: images w and w + 8 (the second may not exist: its sums are discarded)
      const int n1 = warp + 8 < d.batch ? warp + 8 : warp;
      const float* const pn[2] = {sp + warp * C, sp + n1 * C};
      float acc[16];
      fc_mac<2>(pn, sw, C, lane * 8, 256, acc);
      const float v = fc_reduce_scatter<16>(acc, lane);
      const int idx = fc_rs_index<16>(lane), jj = idx & 7, n = warp + (idx >> 3) * 8;
      if ((lane & 1) == 0 && jj < nj && n < d.batch && warp < d.batch)
        ab->out[n][j0 + jj] = v + __ldg(bias + j0 + jj);
    } else {
      const int parts = kMkEpiThreads / nbp, n = et / parts, part = et % parts;
      const float* const pn[1] = {sp + (n < d.batch ? n : 0) * C};
      float acc[8];
      fc_mac<1>(pn, sw, C, part * 8, parts * 8, acc);
      const float v = fc_reduce_scatter<8>(acc, lane);
      const int jj = fc_rs_index<8>(lane);
      if (parts == 32) {
        if ((lane & 3) == 0 && jj < nj && n < d.batch)
          ab->out[n][j0 + jj] = v + __ldg(bias + j0 + jj);
      } else {  // an image spans parts / 32 warps: finish through shared memory
        if ((lane & 3) == 0) sred[warp * 8 + jj] = v;
        named_bar(1, kMkEpiThreads);
        const int wpi = parts >> 5, ni = et >> 3, cj = et & 7;
        if (ni < d.batch && cj < nj) {
          float s = __ldg(bias + j0 + cj);
          for (int w = ni * wpi; w < (ni + 1) * wpi; ++w) s += sred[w * 8 + cj];
          ab->out[ni][j0 + cj] = s;
        }
      }
    }
#ifdef CW_KB_TRACE
    if (et == 0 && (cta == 0 || cta == 100))
      printf("fc cta %d: copy wait %lld, compute %lld cycles\n", cta, tf1 - tf0, clock64() - tf1);
#endif
    named_bar(1, kMkEpiThreads);  // weights (and sred) read before the next block's copy
  }
}

// Optional softmax tail (the last plan layer), run by warps 2-3 so the epilogue warps' code
// (and register allocation) is untouched: once the FC layer completed, request n's logits
// in its IOCache output slot -> probabilities in place. One CTA per request; 64 threads,
// max and sum of exp by warp shuffles and two shared-memory words per warp.
__device__ __noinline__ void softmax_tail(const MkLayer* sl, int nl, int cta, int G,
                                          const ActionBlock* ab, uint32_t* counters,
                                          uint32_t gen1, float* sred, int t64) {
  const MkLayer& d = sl[nl - 1];
  if (first_task(d, cta, G) >= d.tasks) return;
  if (t64 == 0) wait_deps(sl, nl - 1, counters, gen1, 14);
  named_bar(3, 64);
  const int lane = t64 & 31, w = t64 >> 5;
  int done = 0;
  for (int n = first_task(d, cta, G); n < d.tasks; n += G, ++done) {
    float* x = ab->out[n];
    float m = -INFINITY;
    for (int j = t64; j < d.classes; j += 64) m = fmaxf(m, __ldcg(x + j));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) sred[w] = m;
    named_bar(3, 64);
    m = fmaxf(sred[0], sred[1]);
    float s = 0.0f;
    for (int j = t64; j < d.classes; j += 64) s += __expf(__ldcg(x + j) - m);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sred[2 + w] = s;
    named_bar(3, 64);
    const float inv = 1.0f / (sred[2] + sred[3]);
    for (int j = t64; j < d.classes; j += 64) x[j] = __expf(__ldcg(x + j) - m) * inv;
    named_bar(3, 64);  // sred reused by the next request
  }
  // the probabilities are read by nothing in this grid (mk_done / Output copies follow it)
  if (t64 == 0) red_after_bulk_add(counters + nl - 1, (uint32_t)done);
}

// Split-K reduction of one task: rows [part*red_rows, +red_rows) of one tile.
// Split-K reduction of one task: rows [part*red_rows, +red_rows) of one tile. The S partial
// row blocks (contiguous in [tile][split][128][bn]) arrive by bulk copies into the staging
// buffers; the sum + bias (+ residual) (+ ReLU) goes out as bf16.
__device__ __forceinline__ void simt_reduce(const MkLayer& d, const uint8_t* hdr, int task, int et,
                                            const float* stage, uint32_t stage_addr, uint32_t bar,
                                            uint32_t& phase, uint8_t* sout, uint32_t sout_addr) {
  const int R = d.red_parts;
  const int tile = task / R;
  const int r0 = (task - tile * R) * d.red_rows;
  const TileOrigin o = tile_origin(d, tile);
  const float* bias = reinterpret_cast<const float* const*>(hdr + kHdrBiasOff)[d.wlayer] + o.n0;
  const int c4n = d.bn / 4;
  const int S = d.splits;
  const int rr = min(d.red_rows, 128 - r0);
  const uint32_t blk = (uint32_t)(rr * d.bn * 4);
  if (et == 0) {
    fence_proxy_async();  // the partials were written by other CTAs
    mbar_arrive_expect_tx(bar, blk * (uint32_t)S);
    const float* part = d.partial + ((size_t)tile * S * 128 + r0) * d.bn;
    for (int z = 0; z < S; ++z)
      bulk_g2s(stage_addr + z * blk, part + (size_t)z * 128 * d.bn, blk, bar);
  }
  mbar_wait_to<64>(bar, phase & 1, 15);
  ++phase;
  for (int idx = et; idx < rr * c4n; idx += kMkEpiThreads) {
    const int i = idx / c4n;
    const int c = (idx - i * c4n) * 4;
    long long m;
    if (!row_pixel(d, o, r0 + i, &m)) continue;
    float4 acc = __ldg(reinterpret_cast<const float4*>(bias + c));
    const float* src = stage + i * d.bn + c;
    for (int z = 0; z < S; ++z) {
      const float4 p = *reinterpret_cast<const float4*>(src + z * (blk / 4));
      acc.x += p.x;
      acc.y += p.y;
      acc.z += p.z;
      acc.w += p.w;
    }
    const size_t oidx = (size_t)m * d.n_out + o.n0 + c;
    if (d.res) {
      const uint2 r = __ldcg(reinterpret_cast<const uint2*>(
          reinterpret_cast<const __nv_bfloat16*>(d.res) + oidx));
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
      acc.x += a.x;
      acc.y += a.y;
      acc.z += b.x;
      acc.w += b.y;
    }
    uint2 ov;
    if (d.relu) {
      ov.x = pack_bf16x2_relu(acc.x, acc.y);
      ov.y = pack_bf16x2_relu(acc.z, acc.w);
    } else {
      ov.x = pack_bf16x2(acc.x, acc.y);
      ov.y = pack_bf16x2(acc.z, acc.w);
    }
    *reinterpret_cast<uint2*>(sout + (i * d.bn + c) * 2) = ov;
  }
  // the bf16 rows leave by 1D bulk copies (one per output pixel row), so the layer's
  // completion count needs no MEMBAR (red_after_bulk_add)
  fence_proxy_async_smem();
  named_bar(1, kMkEpiThreads);
  bool issued = false;
  const int ncols = min(d.bn, d.n_valid - o.n0);  // padded N-tile columns are not stored
  for (int i = et; i < rr && ncols > 0; i += kMkEpiThreads) {
    long long m;
    if (!row_pixel(d, o, r0 + i, &m)) continue;
    bulk_s2g(reinterpret_cast<__nv_bfloat16*>(d.out) + (size_t)m * d.out_ctot + o.n0,
             sout_addr + (uint32_t)(i * d.bn * 2), (uint32_t)(ncols * 2));
    issued = true;
  }
  if (issued) {
    bulk_commit();
    bulk_wait_all();
    fence_proxy_async();
  }
  named_bar(1, kMkEpiThreads);  // the stages are read before the next task's copies
}

__device__ __forceinline__ void mbar_wait_cluster_to(uint32_t bar, uint32_t parity, int site) {
  if (mbar_try_wait_cluster(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait_cluster(bar, parity))
    if (globaltimer() - t0 > kMkTimeoutNs) mk_timeout(site);
}

// Cluster split-K epilogue (d.csplit): split z of a tile runs on cluster rank z (planner:
// tasks = tiles x C, rotation a multiple of C, bn = 64). Rank z stages its fp32 partial tile
// [128][64] in the upper half of its staging buffers (16-byte chunks XOR-swizzled by row),
// then ONE bulk DSMEM copy per other rank j moves row block j (rows [j*rpc, (j+1)*rpc),
// rpc = 128/C) into slot z of rank j's receive buffer (the lower half; block z itself stays in
// this rank's staging half and is read there); each rank then sums the C partial
// blocks of its own rows + bias (+ residual) (+ ReLU) -> bf16 rows -> bulk stores. Per task
// (the ranks of a cluster run the same task sequence): bar_crdy completes once all C ranks'
// buffers are free (each rank arrives on every rank's), bar_crx once this rank's C blocks
// have landed (transaction bytes of the copies). A rank's staging half is rewritten only
// after the next bar_crdy (every receiver has consumed the previous copies); after the
// layer's last task, bar_cdone (csplit_drain) covers the copies still in flight.
template <int C>
__device__ __noinline__ void epi_csplit(const MkLayer& d, const TileOrigin& o, int z,
                                        uint32_t taddr, int row, int grp, int et, uint32_t obase,
                                        uint8_t* obufs, uint32_t bar_acc, uint32_t acc_par,
                                        uint32_t bar_crdy, uint32_t bar_crx, uint32_t cpar,
                                        const float* bias) {
  constexpr int bn = 64, c4n = bn / 4;
  constexpr uint32_t kTile = 128u * bn * 4u;  // one fp32 partial tile
  constexpr int rpc = 128 / C;
  constexpr uint32_t blk = (uint32_t)rpc * bn * 4u;
#ifdef CW_CSPLIT_TRACE
  long long ts[9];
  ts[0] = clock64();
#define CW_CST(i_) ts[i_] = clock64()
#else
#define CW_CST(i_) do {} while (0)
#endif
  // this rank's staging buffers are free: its earlier TMA stores have read them
  if (et == 0) bulk_wait_read<0>();
  named_bar(1, kMkEpiThreads);
  // (relaxed signals: this rank's reads of its receive buffer are complete, their values were
  // consumed before the barrier; the copies into it are ordered by the transaction count)
  if (et == 0) mbar_arrive_expect_tx(bar_crx, kTile - blk);
  if ((et & 31) == 0)
    for (int j = et >> 5; j < C; j += kMkEpiThreads / 32)
      mbar_arrive_remote(mapa_shared(bar_crdy, (uint32_t)j));
  CW_CST(1);
  // this thread's output element groups of the reduction (rpc x 16 float4: 8 / C per
  // thread, C in {2, 4, 8}), their bias and residual loaded while the partials are in flight
  const int r0 = z * rpc;
  constexpr int ni = 8 / C;
  int li[ni], c4[ni];
  long long m[ni];
  bool mine[ni];
  float4 acc[ni];
  uint2 rres[ni];
#pragma unroll
  for (int k = 0; k < ni; ++k) {
    const int idx = et + k * kMkEpiThreads;
    li[k] = idx / c4n;
    c4[k] = idx - li[k] * c4n;
    m[k] = 0;
    mine[k] = li[k] < rpc && row_pixel(d, o, r0 + li[k], &m[k]) &&
              o.n0 + c4[k] * 4 < d.n_valid;
    acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    rres[k] = make_uint2(0u, 0u);
    if (mine[k]) {
      acc[k] = __ldg(reinterpret_cast<const float4*>(bias) + c4[k]);
      if (d.res)
        rres[k] = __ldcg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(d.res) +
                                                        (size_t)m[k] * d.n_out + o.n0 + c4[k] * 4));
    }
  }
  mbar_wait_to<kEpiWaitNs>(bar_acc, acc_par, 8);
  tc_fence_after();
  CW_CST(2);
  mbar_wait_cluster_to(bar_crdy, cpar, 16);
  CW_CST(3);
  {
    uint32_t v[32];
    tmem_ld16(taddr + 32 * grp, *reinterpret_cast<uint32_t(*)[16]>(v));
    tmem_ld16(taddr + 32 * grp + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
    tmem_ld_wait();
    uint8_t* stage = obufs + kTile + (uint32_t)row * (bn * 4);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int ch = 8 * grp + kk;  // logical 16-byte chunk of the row
      *reinterpret_cast<uint4*>(stage + ((ch ^ (row & 7)) << 4)) =
          make_uint4(v[4 * kk], v[4 * kk + 1], v[4 * kk + 2], v[4 * kk + 3]);
    }
  }
  fence_proxy_async_smem();  // generic stores -> the bulk copies' async-proxy reads
  named_bar(1, kMkEpiThreads);
  if ((et & 31) == 0)  // (one issuing lane per warp: the copies leave in parallel)
    for (uint32_t j = (uint32_t)(et >> 5); j < (uint32_t)C; j += kMkEpiThreads / 32)
      if (j != (uint32_t)z)  // (this rank's own block is read from its staging half)
        bulk_s2cluster(mapa_shared(obase + (uint32_t)z * blk, j), obase + kTile + j * blk, blk,
                       mapa_shared(bar_crx, j));
  CW_CST(4);
  mbar_wait_cluster_to(bar_crx, cpar, 17);
  CW_CST(5);
  const float4* src = reinterpret_cast<const float4*>(obufs);
#pragma unroll
  for (int k = 0; k < ni; ++k) {
    if (!mine[k]) continue;
    float4 a4 = acc[k];
    const int pc = c4[k] ^ (li[k] & 7);  // (row & 7 == li & 7: rpc is a multiple of 8)
    for (int s = 0; s < C; ++s) {
      // (summed in rank order 0..C-1: every rank's rows see the same association)
      const float4 p = s == z ? src[(C * rpc + r0 + li[k]) * c4n + pc] : src[(s * rpc + li[k]) * c4n + pc];
      a4.x += p.x;
      a4.y += p.y;
      a4.z += p.z;
      a4.w += p.w;
    }
    if (d.res) {
      const float2 ra = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rres[k].x));
      const float2 rb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rres[k].y));
      a4.x += ra.x;
      a4.y += ra.y;
      a4.z += rb.x;
      a4.w += rb.y;
    }
    uint2 ov;
    if (d.relu) {
      ov.x = pack_bf16x2_relu(a4.x, a4.y);
      ov.y = pack_bf16x2_relu(a4.z, a4.w);
    } else {
      ov.x = pack_bf16x2(a4.x, a4.y);
      ov.y = pack_bf16x2(a4.z, a4.w);
    }
    // generic stores (16 threads cover a row's 128 bytes): a per-row bulk copy costs ~500
    // issue cycles; the layer publishes with red.release instead (epi_csplit's caller)
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(d.out) + (size_t)m[k] * d.out_ctot +
                              o.n0 + c4[k] * 4) = ov;
  }
  CW_CST(6);
  CW_CST(7);
#ifdef CW_CSPLIT_TRACE
  if (et == 0 && blockIdx.x < 8)
    printf("csplit cta %d z %d n0 %d: bar %lld acc %lld crdy %lld send %lld crx %lld red %lld "
           "rbar %lld st %lld\n",
           blockIdx.x, z, o.n0, ts[1] - ts[0], ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3],
           ts[5] - ts[4], ts[6] - ts[5], ts[7] - ts[6], clock64() - ts[7]);
#endif
#undef CW_CST
}

// After a cluster split-K layer's last task: every rank has received all its partial blocks
// (so every copy this rank sent has landed) before the staging buffers are reused.
__device__ __noinline__ void csplit_drain(int C, int et, uint32_t bar_cdone, uint32_t par) {
  if ((et & 31) == 0)
    for (int j = et >> 5; j < C; j += kMkEpiThreads / 32)
      mbar_arrive_remote(mapa_shared(bar_cdone, (uint32_t)j));
  mbar_wait_cluster_to(bar_cdone, par, 18);
}

// Stem conv with the 3x3/s2/p1 max pool fused: the tile's conv pixels
// (3 conv rows x 2*pool_pw+1 columns) -> bias, ReLU, bf16 into the CTA staging
// buffer, then each pooled pixel = max over its valid 3x3 window (identical to
// pooling the bf16 conv output; padding = -inf = skipped).
// One epilogue thread's share of one 64-column chunk of the TMA epilogue: its row's 32
// accumulator columns `v` (in registers) + folded-BN bias (+ the residual chunk that landed in
// the staging buffer) (+ ReLU) -> bf16, rewritten in place (128-byte swizzle). Branch-free
// per (residual, ReLU) variant with every shared-memory load issued before the math (the
// generic version's branches and its bias loads ordered behind stores measured ~550 cycles
// per chunk, the whole epilogue warp's latency chain).
template <bool RES, bool RELU>
__device__ __forceinline__ void epi_chunk32(const uint32_t (&v)[32], const float* bias32,
                                            uint8_t* buf, int row, int grp) {
  const float4* bp = reinterpret_cast<const float4*>(__builtin_assume_aligned(bias32, 16));
  float4 bq[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) bq[i] = bp[i];
  uint4 rv[4];
  if constexpr (RES) {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      rv[kk] = *reinterpret_cast<const uint4*>(buf + row * 128 + (((4 * grp + kk) ^ (row & 7)) << 4));
  }
  uint32_t w[16];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const float bb[8] = {bq[2 * kk].x, bq[2 * kk].y, bq[2 * kk].z, bq[2 * kk].w,
                         bq[2 * kk + 1].x, bq[2 * kk + 1].y, bq[2 * kk + 1].z, bq[2 * kk + 1].w};
    float f[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[8 * kk + e]);
#pragma unroll
    for (int e = 0; e < 8; e += 2) fadd2(f[e], f[e + 1], bb[e], bb[e + 1]);
    if constexpr (RES) {
      float rf[8];
      bf16x8_to_f32(rv[kk], rf);
#pragma unroll
      for (int e = 0; e < 8; e += 2) fadd2(f[e], f[e + 1], rf[e], rf[e + 1]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      w[4 * kk + e] = RELU ? pack_bf16x2_relu(f[2 * e], f[2 * e + 1]) : pack_bf16x2(f[2 * e], f[2 * e + 1]);
  }
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    *reinterpret_cast<uint4*>(buf + row * 128 + (((4 * grp + kk) ^ (row & 7)) << 4)) =
        make_uint4(w[4 * kk], w[4 * kk + 1], w[4 * kk + 2], w[4 * kk + 3]);
}

__device__ __forceinline__ void epi_stem_pool(const MkLayer* dp, const TileOrigin o, uint32_t taddr,
                                           const float* bias, uint8_t* pb, uint8_t* ps,
                                           uint32_t ps_addr, const CUtensorMap* tmo, int row,
                                           int grp, int et) {
  const MkLayer& d = *dp;
  // 1) vertical max: this thread's conv column (accumulator row) over the task's 3 conv rows
  // (accumulators 64 columns apart), ReLU folded in (maxima start at 0: post-ReLU values are
  // >= 0 and a conv row outside the image contributes nothing), its group's 32 channels
  float mx[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) mx[k] = 0.0f;
  const float4* bp = reinterpret_cast<const float4*>(__builtin_assume_aligned(bias + 32 * grp, 16));
  float4 bq[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) bq[i] = bp[i];
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    const int cr = o.oh0 + c;
    if (cr < 0 || cr >= d.oh) continue;  // (uniform over the CTA)
    uint32_t v[32];
    tmem_ld16(taddr + 64 * c + 32 * grp, *reinterpret_cast<uint32_t(*)[16]>(v));
    tmem_ld16(taddr + 64 * c + 32 * grp + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      mx[4 * i] = fmaxf(mx[4 * i], __uint_as_float(v[4 * i]) + bq[i].x);
      mx[4 * i + 1] = fmaxf(mx[4 * i + 1], __uint_as_float(v[4 * i + 1]) + bq[i].y);
      mx[4 * i + 2] = fmaxf(mx[4 * i + 2], __uint_as_float(v[4 * i + 2]) + bq[i].z);
      mx[4 * i + 3] = fmaxf(mx[4 * i + 3], __uint_as_float(v[4 * i + 3]) + bq[i].w);
    }
  }
  // staged as bf16 [conv column][64 channels] (128-byte swizzle); rows >= out_w are junk the
  // pooling never reads
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    *reinterpret_cast<uint4*>(pb + row * 128 + (((4 * grp + kk) ^ (row & 7)) << 4)) =
        make_uint4(pack_bf16x2(mx[8 * kk], mx[8 * kk + 1]), pack_bf16x2(mx[8 * kk + 2], mx[8 * kk + 3]),
                   pack_bf16x2(mx[8 * kk + 4], mx[8 * kk + 5]), pack_bf16x2(mx[8 * kk + 6], mx[8 * kk + 7]));
  if (et == 0) bulk_wait_read<0>();  // the previous task's store has read the pooled stage
  named_bar(1, kMkEpiThreads);
  // 2) horizontal max over conv columns 2pw-1 .. 2pw+1 (the column left of 0 and right of the
  // image contribute 0): the staged values are non-negative bf16, whose bit patterns order like
  // their values: an unsigned 16-bit SIMD max per word is exact
  const int ow = d.ow, npix = d.pool_pw * 8;
  for (int it = et; it < npix; it += kMkEpiThreads) {
    const int j = it >> 3, k = it & 7;
    uint32_t m4[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int dc = -1; dc <= 1; ++dc) {
      const int cc = 2 * j + dc;
      if (cc < 0 || cc >= ow) continue;
      const uint4 q = *reinterpret_cast<const uint4*>(pb + cc * 128 + ((k ^ (cc & 7)) << 4));
      m4[0] = __vmaxu2(m4[0], q.x & 0x7FFF7FFFu);  // (a -0 from fmaxf orders as +0)
      m4[1] = __vmaxu2(m4[1], q.y & 0x7FFF7FFFu);
      m4[2] = __vmaxu2(m4[2], q.z & 0x7FFF7FFFu);
      m4[3] = __vmaxu2(m4[3], q.w & 0x7FFF7FFFu);
    }
    *reinterpret_cast<uint4*>(ps + j * 128 + ((k ^ (j & 7)) << 4)) = make_uint4(m4[0], m4[1], m4[2], m4[3]);
  }
  fence_proxy_async_smem();
  named_bar(1, kMkEpiThreads);
  if (et == 0) {
    tma_store_4d(tmo, ps_addr, 0, 0, (o.oh0 + 1) / 2, o.img0);
    bulk_commit();
  }
}
// Warps 2-3: the input BatchNorm + ReLU prologue of DenseNet's pre-activation 1x1 convs:
// relu(x * scale[c] + shift[c]) applied to the A tile of every k-block in place in shared
// memory, between its TMA landing and its MMAs. The producer completes such a layer's
// fills on bar_fpre (not bar_full) and the MMA waits on bar_xf, so these warps only see the
// phases of BN layers: they can neither run ahead of a fill (parity aliasing) nor fall two
// phases behind one (the slot is refilled only after the MMA, i.e. after them). Thread t
// owns physical 16-byte chunk t & 7 of rows (t >> 3) + 8i: under the 128-byte swizzle (chunk
// j of row r at j ^ (r & 7)) that is ONE logical chunk, i.e. the same 8 channels, for all
// its rows, so the k-block's scale/shift of those channels stay in registers.
#ifndef CW_PRE_UNROLL
#define CW_PRE_UNROLL 4
#endif
constexpr int kPreUnroll = CW_PRE_UNROLL;
__device__ __noinline__ void bn_prologue(const MkLayer* sl, int nl, int cta, int G,
                                         const uint8_t* hdr, uint8_t* smem, uint32_t bar_fpre,
                                         uint32_t bar_xf, int t64) {
  uint32_t par = 0;  // bit s: parity of the BN-layer fills of slot s seen so far
  const int rg = t64 >> 3, pc = t64 & 7, lc = pc ^ rg;
  for (int L = 0; L < nl; ++L) {
    if (sl[L].kind != MK_CONV || sl[L].pre_layer < 0) continue;
    const MkLayer& d = sl[L];
    const int ns = d.slots;
    const uint32_t sb = (uint32_t)d.slot_bytes;
    const float* ptab = reinterpret_cast<const float* const*>(hdr + kHdrPreOff)[d.pre_layer];
    const int cpad = d.num_kb * 64;
    int slot = 0;
    for (int t = first_task(d, cta, G); t < d.tasks; t += G) {
      int kb0, kb1;
      split_range(d, t % d.splits, kb0, kb1);
      const int n = kb1 - kb0;  // kpack = 1: a k-block per slot
      // this thread's 8 channels' scale / shift, one k-block ahead (an L2 round trip per
      // k-block otherwise sits between the tile landing and its rewrite)
      float4 s0, s1, h0, h1;
      auto load_tab = [&](int kb) {
        const int c0 = kb * 64 + lc * 8;
        s0 = __ldg(reinterpret_cast<const float4*>(ptab + c0));
        s1 = __ldg(reinterpret_cast<const float4*>(ptab + c0 + 4));
        h0 = __ldg(reinterpret_cast<const float4*>(ptab + cpad + c0));
        h1 = __ldg(reinterpret_cast<const float4*>(ptab + cpad + c0 + 4));
      };
      if (n > 0) load_tab(kb0);
      for (int i = 0; i < n; ++i) {
        const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const float sh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
        if (i + 1 < n) load_tab(kb0 + i + 1);
        mbar_wait_to<64>(bar_fpre + 8 * slot, (par >> slot) & 1, 13);
        par ^= 1u << slot;
        uint8_t* tile = smem + slot * sb;
#ifdef CW_PRE_NOOP  // experiments: the hand-off without the rewrite (wrong logits; timing only)
        if (sb != 0u) { fence_proxy_async_smem(); mbar_arrive(bar_xf + 8 * slot); if (++slot == ns) slot = 0; continue; }
#endif
#ifndef CW_PRE_F32
        // relu(x * scale + shift) as one packed bf16 fma per channel pair (HFMA2.BF16 with
        // fused ReLU, one rounding): the k-block's scale / shift rounded to bf16 once. The fp32
        // FFMA2 + unpack / repack form (-DCW_PRE_F32) is ~3x the instructions and measured
        // DenseNet-121 b=16 1062 vs 893 us, b=1 700 vs 601; logit margin 0.0063 vs 0.0060
        // (bound 0.02).
        uint32_t s2[4], h2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          s2[e] = pack_bf16x2(sc[2 * e], sc[2 * e + 1]);
          h2[e] = pack_bf16x2(sh[2 * e], sh[2 * e + 1]);
        }
        // all 16 of this thread's chunk loads issued before its first store (the compiler
        // cannot prove the in-place rows disjoint; 4-deep software order measured 16-18 us slower)
        uint4 v[16];
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) v[i2] = *reinterpret_cast<const uint4*>(tile + (rg + 8 * i2) * 128 + pc * 16);
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          asm("fma.rn.relu.bf16x2 %0, %0, %1, %2;" : "+r"(v[i2].x) : "r"(s2[0]), "r"(h2[0]));
          asm("fma.rn.relu.bf16x2 %0, %0, %1, %2;" : "+r"(v[i2].y) : "r"(s2[1]), "r"(h2[1]));
          asm("fma.rn.relu.bf16x2 %0, %0, %1, %2;" : "+r"(v[i2].z) : "r"(s2[2]), "r"(h2[2]));
          asm("fma.rn.relu.bf16x2 %0, %0, %1, %2;" : "+r"(v[i2].w) : "r"(s2[3]), "r"(h2[3]));
          *reinterpret_cast<uint4*>(tile + (rg + 8 * i2) * 128 + pc * 16) = v[i2];
        }
#else
#pragma unroll kPreUnroll
        for (int r = rg; r < 128; r += 8) {
          uint4* q = reinterpret_cast<uint4*>(tile + r * 128 + pc * 16);
          float f[8];
          bf16x8_to_f32(*q, f);
#pragma unroll
          for (int e = 0; e < 8; e += 2) ffma2(f[e], f[e + 1], sc[e], sc[e + 1], sh[e], sh[e + 1]);
          uint4 o;
          o.x = pack_bf16x2_relu(f[0], f[1]);
          o.y = pack_bf16x2_relu(f[2], f[3]);
          o.z = pack_bf16x2_relu(f[4], f[5]);
          o.w = pack_bf16x2_relu(f[6], f[7]);
          *q = o;
        }
#endif
        fence_proxy_async_smem();  // generic-proxy writes -> the MMA's async-proxy reads
        mbar_arrive(bar_xf + 8 * slot);
        if (++slot == ns) slot = 0;
      }
    }
  }
}

// ------------------------------------------------------------------ the kernel

__global__ void __launch_bounds__(kMkThreads, 1) mk_infer_kernel(const __grid_constant__ MkArgs args) {
  const ActionBlock* ab = args.ab;
  // programmatic dependent launch: the CTAs become resident while the gate still runs; the
  // action block (and everything before it) is visible after the wait
  griddep_wait();
  if (ab->skip) return;  // window missed: the gate kernel already recorded the rejection
  uint64_t* clk_trace =
      args.trace ? args.trace + ((size_t)args.n_layers * gridDim.x + blockIdx.x) * 4 : nullptr;
  if (clk_trace && threadIdx.x == 0) {
    clk_trace[0] = globaltimer();
    clk_trace[1] = clock64();
  }
  if (threadIdx.x == 0) atomicMin(const_cast<unsigned long long*>(&ab->mk_t0), globaltimer());
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t ring_bytes = args.ring_bytes;
  // Layout after the ring: epilogue staging buffers (1024-aligned), barriers, tmem/gen slots,
  // bias [2][256] f32, then the plan's layer table.
  uint8_t* obufs = smem + ring_bytes;
  const uint32_t obase = sbase + ring_bytes;
  const uint32_t bar_full = obase + kMkOutBufs * kMkOutBufBytes;
  const uint32_t bar_empty = bar_full + 8 * kMkMaxSlots;
  const uint32_t bar_tfull = bar_empty + 8 * kMkMaxSlots;  // 2 x 8 B
  const uint32_t bar_tempty = bar_tfull + 2 * 8;          // 2 x 8 B
  const uint32_t bar_simt = bar_tempty + 2 * 8;           // SIMT-layer bulk copies
  const uint32_t bar_res = bar_simt + 8;                  // kMkOutBufs x 8 B: residual chunks
  const uint32_t bar_stemb = bar_res + 8 * kMkOutBufs;    // resident stem weights
  const uint32_t bar_xf = bar_stemb + 8;                  // kMkMaxSlots: A tile BN-transformed
  const uint32_t bar_fpre = bar_xf + 8 * kMkMaxSlots;     // kMkMaxSlots: fills of BN layers
  const uint32_t bar_crdy = bar_fpre + 8 * kMkMaxSlots;   // cluster split-K: all receivers ready
  const uint32_t bar_crx = bar_crdy + 8;                  // cluster split-K: partials landed
  const uint32_t bar_cdone = bar_crx + 8;                 // cluster split-K: layer's copies done
  uint8_t* bar_area = obufs + kMkOutBufs * kMkOutBufBytes;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_area + kMkBarBytes - 32);
  uint32_t* gen_slot = tmem_slot + 1;
  float* sbias = reinterpret_cast<float*>(bar_area + kMkBarBytes);
  float* sred = reinterpret_cast<float*>(obufs + kMkOutBufBytes);  // 2 x [128][17] f32 (avg pool)
  uint4* sstage = reinterpret_cast<uint4*>(obufs + kMkScratch);    // stem pool / split-K staging
  const MkLayer* sl = c_plan;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
#ifdef CW_KB_TRACE
  __shared__ uint64_t kbt[4][64];  // debug: producer acquire / A issued, MMA full / committed
  __shared__ uint64_t ket[2][64];  // debug: epilogue events (clock, tag)
  int kbp = 0, kbm = 0, kbe = 0;
#ifndef CW_KB_LAYER
#define CW_KB_LAYER -1  // trace one plan layer only (-1: from the first)
#endif
#ifndef CW_KB_ET
#define CW_KB_ET 0  // the traced epilogue thread
#endif
#define CW_KET(tag_)                                                   \
  do {                                                                 \
    if (cta == 0 && et == CW_KB_ET && kbe < 64 && (CW_KB_LAYER < 0 || L == CW_KB_LAYER)) { \
      ket[0][kbe] = clock64();                                         \
      ket[1][kbe++] = (tag_);                                          \
    }                                                                  \
  } while (0)
#else
#define CW_KET(tag_) do {} while (0)
#endif
  const int G = gridDim.x;
  const int nl = args.n_layers;

  // ---- prologue: barriers, TMEM
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMkMaxSlots; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(bar_tfull + 8 * a, 1);
      mbar_init(bar_tempty + 8 * a, kMkEpiThreads / 32);
    }
    mbar_init(bar_simt, 1);
    for (int b = 0; b < kMkOutBufs; ++b) mbar_init(bar_res + 8 * b, 1);
    mbar_init(bar_stemb, 1);
    for (int sl = 0; sl < kMkMaxSlots; ++sl) {
      mbar_init(bar_xf + 8 * sl, 64);
      mbar_init(bar_fpre + 8 * sl, 1);
    }
    mbar_init(bar_crdy, (uint32_t)args.csize);  // one arrival per CTA of the cluster
    mbar_init(bar_crx, 1);                      // the local expect_tx; the data by bulk copies
    mbar_init(bar_cdone, (uint32_t)args.csize);
    fence_mbar_init();
    *gen_slot = *reinterpret_cast<const volatile uint32_t*>(args.gen);
  }
  if (warp == 1) tmem_alloc(smem_u32(tmem_slot), kMkTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (args.csize > 1) cluster_sync();  // every CTA's barriers initialised before remote arrivals
  const uint32_t tmem = *tmem_slot;
  const uint32_t gen1 = *gen_slot + 1u;
  const uint8_t* hdr = ab->hdr;
  uint32_t* counters = args.counters;

  if (warp < kMkEpiWarp0) {
  setmaxnreg_dec<kMkRegsCtl>();  // warpgroup 0: TMA producer(s) and the MMA issuer
  if (warp == 0 || (kMkProducers > 1 && warp == 2)) {
    const int pw = warp == 0 ? 0 : 1;  // producer index
    {
      // ======================= TMA producer (whole warp converged; one elected lane issues)
      // A ring slot holds `kpack` consecutive k-blocks (sub-slots of sub_bytes: A tile, then
      // B tile at b_off) behind one full/empty barrier pair. Slots restart at 0 every layer;
      // bit s of `par` = parity of the fills of slot s so far (fill n waits for consumption
      // n-1). A layer whose slot geometry differs from the previous one first drains the ring.
      uint32_t par = 0;
      int cur_slots = 0, cur_bytes = 0;
      for (int L = 0; L < nl; ++L) {
        if (sl[L].kind != MK_CONV) continue;
#ifndef CW_NO_WPREFETCH
        {
          // the NEXT conv's weights into L2 (they stream from HBM: every INFER may run another
          // model copy), a 1/G slice per CTA: its first B tiles then hit L2, not HBM latency
          int Ln = L;
          for (int ahead = 0; ahead < args.pf_depth; ++ahead) {
            ++Ln;
            while (Ln < nl && sl[Ln].kind != MK_CONV && sl[Ln].kind != MK_FC) ++Ln;
            if (Ln >= nl) break;
            if ((sl[Ln].kind == MK_FC || sl[Ln].mode != 2) && elect_one()) {
              const MkLayer& dn = sl[Ln];
              const uint8_t* const* wt = reinterpret_cast<const uint8_t* const*>(hdr + kHdrWeightOff);
              // (a fused shortcut: its weight layer is the second segment)
              for (int sg = 0; sg < (dn.kind == MK_CONV && dn.f_kb ? 2 : 1); ++sg) {
                const uint8_t* w = wt[sg ? dn.f_wlayer : dn.wlayer];
                const uint32_t kbs = dn.kind == MK_FC ? 0u : (uint32_t)(sg ? dn.f_kb : dn.num_kb - dn.f_kb);
                const uint32_t bytes = dn.kind == MK_FC ? (uint32_t)dn.classes * (uint32_t)dn.C * 2u
                                                        : (uint32_t)dn.n_out * kbs * (uint32_t)dn.kblk * 2u;
                const uint32_t per = ((bytes + G - 1) / G + 255u) & ~255u;
                const uint32_t off = (uint32_t)cta * per;
                if (off < bytes) bulk_prefetch_l2(w + off, min(per, bytes - off));
              }
            }
            __syncwarp();
          }
        }
#endif
        const MkLayer d = sl[L];  // registers: the asm memory clobbers would force re-loads
        int t = first_task(d, cta, G);
        if (t >= d.tasks) continue;
        const CUtensorMap* ta = args.tmaps + d.tmap;
        // B: one TMA per k-block when the N tile spans the wide map's box (min(256, Cout) rows)
        const bool wide = d.kblk == 64 && d.bn == min(256, d.n_out);
        const CUtensorMap* tb = reinterpret_cast<const CUtensorMap*>(
            hdr + (wide ? kHdrWideOff : 0) + d.wlayer * kTmapBytes);
        // a fused shortcut (k-blocks [seg1, num_kb)): its own A map and weight layer
        const int seg1 = d.num_kb - d.f_kb;
        const CUtensorMap* ta2 = args.tmaps + d.f_tmap;
        const CUtensorMap* tb2 = reinterpret_cast<const CUtensorMap*>(
            hdr + (wide ? kHdrWideOff : 0) + d.f_wlayer * kTmapBytes);
        if (elect_one()) {
          tmap_acquire(tb);
          tmap_prefetch(ta);
          tmap_prefetch(tb);
          if (d.f_kb) {
            tmap_acquire(tb2);
            tmap_prefetch(ta2);
            tmap_prefetch(tb2);
          }
        }
        __syncwarp();
        const int ns = d.slots;
        const uint32_t sb = (uint32_t)d.slot_bytes;
        if (ns != cur_slots || d.slot_bytes != cur_bytes) {
          for (int s = 0; s < cur_slots; ++s)
            if (s % kMkProducers == pw) mbar_wait_to(bar_empty + 8 * s, ((par >> s) & 1) ^ 1, 1);
          // a new slot may overlap an old slot of the other producer: both drain first
          if (kMkProducers > 1) named_bar(2, 32 * kMkProducers);
          cur_slots = ns;
          cur_bytes = d.slot_bytes;
        }
        if (d.mode == 2) {
          // stem: weights once per layer (resident in the staging buffers), then per task ONE
          // box = the kMkStemRows padded input rows of the task's 3 conv rows
          if (elect_one()) {
            mbar_arrive_expect_tx(bar_stemb, 7u * 64u * 64u);
            for (int r = 0; r < 7; ++r)
              tma_load_2d(obase + kMkStemB + r * 4096u, tb, bar_stemb, r * 32, 0);
          }
          __syncwarp();
          wait_deps(sl, L, counters, gen1, 2);
          fence_proxy_async();
          if (args.trace && lane == 0 && pw == 0)
            args.trace[((size_t)L * G + cta) * 4 + 1] = globaltimer();
          int slot = 0;
          for (; t < d.tasks; t += G) {
            const TileOrigin o = tile_origin(d, t);
            if (slot % kMkProducers == pw) {
              mbar_wait_to<CW_HINT_EMPTY>(bar_empty + 8 * slot, ((par >> slot) & 1) ^ 1, 3);
              par ^= 1u << slot;
              if (elect_one()) {
                // padded rows 2*oh0 .. 2*oh0 + 10: conv rows oh0 .. oh0 + 2, kernel rows 0 .. 6
                mbar_arrive_expect_tx(bar_full + 8 * slot, (uint32_t)(kMkStemRows * d.sub_bytes));
                tma_load_4d(sbase + slot * sb, ta, bar_full + 8 * slot, 0, 0, 2 * o.oh0, o.img0);
              }
              __syncwarp();
            }
            if (++slot == ns) slot = 0;
          }
          continue;
        }
        if (d.mode == 3) {
          // 3x3 / stride 1: a slot = (kernel row r, channel block): ONE A box (columns -1 ..
          // box_w - 2 of the input rows, OOB zero fill = padding) + the B tiles of taps q = 0..2
          const uint32_t a3 = a_rows(d) * 128u, b3 = (uint32_t)d.bn * 128u;
          const uint32_t tx3 = a3 + 3u * b3;
          const uint32_t b_off = (uint32_t)d.b_off, b_box = 64u * 128u;
          const int nbox = wide ? 1 : d.bn / 64;
          int slot = 0;
          bool waited = false;
          for (; t < d.tasks; t += G) {
            const int tile = t / d.splits;
            const int z = t - tile * d.splits;
            const TileOrigin o = tile_origin(d, tile);
            int kb0, kb1;
            split_range(d, z, kb0, kb1);
            const int g0 = kb0 / 3, ng = (kb1 - kb0) / 3;
            auto load_b = [&](int g, int s) {
              const int r = g / d.cin_kb, cb = g - r * d.cin_kb;
              if (elect_one())
                for (int q = 0; q < 3; ++q)
                  for (int j = 0; j < nbox; ++j)
                    tma_load_2d_hint(sbase + s * sb + b_off + q * b3 + j * b_box, tb,
                                     bar_full + 8 * s, ((r * 3 + q) * d.cin_kb + cb) * 64,
                                     o.n0 + 64 * j, kHintW);
              __syncwarp();
            };
            const int chan0 = d.grouped ? o.n0 : 0;  // grouped: the tile's own channel block
            auto load_a = [&](int g, int s) {
              const int r = g / d.cin_kb, cb = g - r * d.cin_kb;
              if (elect_one())
                tma_load_4d(sbase + s * sb, ta, bar_full + 8 * s, chan0 + cb * 64, o.ow0 - 1,
                            o.oh0 + r - 1, o.img0);
              __syncwarp();
            };
            auto acquire = [&](int s) {
              mbar_wait_to<CW_HINT_EMPTY>(bar_empty + 8 * s, ((par >> s) & 1) ^ 1, 3);
              par ^= 1u << s;
              if (elect_one()) mbar_arrive_expect_tx(bar_full + 8 * s, tx3);
              __syncwarp();
            };
            int c = 0;
            if (!waited) {  // weights first (no dependency), then the inputs
              const int pre = ng < ns ? ng : ns;
              int s = slot;
              for (int k = 0; k < pre; ++k) {
                if (s % kMkProducers == pw) {
                  acquire(s);
                  load_b(g0 + k, s);
                }
                if (++s == ns) s = 0;
              }
              wait_deps(sl, L, counters, gen1, 2);
              fence_proxy_async();
              waited = true;
              if (args.trace && lane == 0 && pw == 0)
                args.trace[((size_t)L * G + cta) * 4 + 1] = globaltimer();
              for (; c < pre; ++c) {
                if (slot % kMkProducers == pw) load_a(g0 + c, slot);
                if (++slot == ns) slot = 0;
              }
            }
            for (; c < ng; ++c) {
              if (slot % kMkProducers == pw) {
                acquire(slot);
                load_b(g0 + c, slot);
                load_a(g0 + c, slot);
              }
              if (++slot == ns) slot = 0;
            }
          }
          continue;
        }
        const uint32_t a_bytes = a_rows(d) * (uint32_t)d.kblk * 2u;
#ifdef CW_EXPERIMENTS
        const bool no_a = args.flags & 2, no_b = args.flags & 4;
#else
        constexpr bool no_a = false, no_b = false;
#endif
        const uint32_t tx1 = (no_a ? 0u : a_bytes) + (no_b ? 0u : (uint32_t)d.bn * (uint32_t)d.kblk * 2u);
        const uint32_t b_box = 64u * (uint32_t)d.kblk * 2u;
        const int nbox = wide ? 1 : d.bn / 64;
        const int cin = d.cin_kb * 64;
        const int mode = d.mode, kw = d.kw, kblk = d.kblk, kpack = d.kpack;
        // a BN-prologue layer's fills complete on bar_fpre (warps 2-3 transform, then bar_xf)
        const uint32_t fullb = d.pre_layer >= 0 ? bar_fpre : bar_full;
        const uint32_t b_off = (uint32_t)d.b_off, sub = (uint32_t)d.sub_bytes;
        int slot = 0;
        bool waited = false;
        for (; t < d.tasks; t += G) {
          const int tile = t / d.splits;
          const int z = t - tile * d.splits;
          const TileOrigin o = tile_origin(d, tile);
          int kb0, kb1;
          split_range(d, z, kb0, kb1);
          const int wb = o.ow0 * d.stride - d.pad_w;
          const int hb = o.oh0 * d.stride - d.pad;
          const int wb2 = o.ow0 * d.f_stride, hb2 = o.oh0 * d.f_stride;  // fused shortcut (1x1)
          const int chan0 = d.grouped ? o.n0 : 0;  // grouped: the tile's own channel block
          // A coordinates walk k-blocks in order: (channel block, tap column q, tap row r)
          int a_kb = kb0, a_c0 = 0, a_q = 0, a_r = 0;
          if (d.mode == 1) {
            const int tap = kb0 / d.cin_kb;
            a_c0 = (kb0 - tap * d.cin_kb) * 64;
            a_r = tap / d.kw;
            a_q = tap - a_r * d.kw;
          }
          const int n = kb1 - kb0;
          const int nslots = (n + kpack - 1) / kpack;
#define CW_ACQUIRE(s_, m_)                                                          \
  do {                                                                              \
    mbar_wait_to<CW_HINT_EMPTY>(bar_empty + 8 * (s_), ((par >> (s_)) & 1) ^ 1, 3);  \
    par ^= 1u << (s_);                                                              \
    if (elect_one()) mbar_arrive_expect_tx(fullb + 8 * (s_), tx1 * (uint32_t)(m_));    \
    __syncwarp();                                                                   \
  } while (0)
#define CW_LOAD_B(kb_, dst0_, s_)                                                   \
  do {                                                                              \
    const uint32_t dst_ = (dst0_) + b_off;                                          \
    const bool s2_ = (kb_) >= seg1;                                                 \
    const int kx_ = ((kb_) - (s2_ ? seg1 : 0)) * kblk;                              \
    if (elect_one())                                                                \
      for (int j = 0; j < (no_b ? 0 : nbox); ++j)                                   \
        tma_load_2d_hint(dst_ + j * b_box, s2_ ? tb2 : tb, fullb + 8 * (s_), kx_,   \
                         o.n0 + 64 * j, kHintW);                                    \
    __syncwarp();                                                                   \
  } while (0)
#define CW_ADV_A()                                                                      \
  do {                                                                                 \
    if (mode == 1) {                                                                   \
      a_c0 += 64;                                                                      \
      if (a_c0 == cin) {                                                               \
        a_c0 = 0;                                                                      \
        if (++a_q == kw) {                                                             \
          a_q = 0;                                                                     \
          ++a_r;                                                                       \
        }                                                                              \
      }                                                                                \
    }                                                                                  \
    ++a_kb;                                                                            \
  } while (0)
#define CW_LOAD_A(dst_, s_)                                                            \
  do {                                                                                 \
    const uint32_t fb_ = fullb + 8 * (s_);                                             \
    if (elect_one()) {                                                                 \
      if (no_a) {                                                                      \
      } else if (a_kb >= seg1) {                                                       \
        if (mode == 0) tma_load_2d(dst_, ta2, fb_, (a_kb - seg1) * 64, o.m0);          \
        else tma_load_4d(dst_, ta2, fb_, (a_kb - seg1) * 64, wb2, hb2, o.img0);        \
      } else if (mode == 0) {                                                          \
        tma_load_2d(dst_, ta, fb_, a_kb * 64, o.m0);                                   \
      } else if (mode == 1) {                                                          \
        tma_load_4d(dst_, ta, fb_, chan0 + a_c0, wb + a_q, hb + a_r, o.img0);          \
      } else {                                                                         \
        tma_load_4d(dst_, ta, fb_, 0, o.ow0, hb + a_kb, o.img0);                       \
      }                                                                                \
    }                                                                                  \
    __syncwarp();                                                                      \
    CW_ADV_A();                                                                        \
  } while (0)
#define CW_MINE(s_) ((s_) % kMkProducers == pw)
          int c = 0;  // slots of this task done
          if (!waited) {
            // weights first (independent of the previous layers), then the inputs
            const int pre = nslots < ns ? nslots : ns;
            int s = slot;
            for (int k = 0; k < pre; ++k) {
              if (CW_MINE(s)) {
                const int m = min(kpack, n - k * kpack);
                CW_ACQUIRE(s, m);
                for (int j = 0; j < m; ++j) CW_LOAD_B(kb0 + k * kpack + j, sbase + s * sb + j * sub, s);
              }
              if (++s == ns) s = 0;
            }
            wait_deps(sl, L, counters, gen1, 2);
            fence_proxy_async();
            waited = true;
            if (args.trace && lane == 0 && pw == 0)
              args.trace[((size_t)L * G + cta) * 4 + 1] = globaltimer();
            for (; c < pre; ++c) {
              const int m = min(kpack, n - c * kpack);
              if (CW_MINE(slot)) {
                for (int j = 0; j < m; ++j) CW_LOAD_A(sbase + slot * sb + j * sub, slot);
              } else {
                for (int j = 0; j < m; ++j) CW_ADV_A();
              }
              if (++slot == ns) slot = 0;
            }
          }
          for (; c < nslots; ++c) {
            const int m = min(kpack, n - c * kpack);
            if (CW_MINE(slot)) {
              CW_ACQUIRE(slot, m);
#ifdef CW_KB_TRACE
              if (cta == 0 && kbp < 64 && lane == 0 && pw == 0) kbt[0][kbp] = clock64();
#endif
              for (int j = 0; j < m; ++j) {
                const uint32_t dst = sbase + slot * sb + j * sub;
                CW_LOAD_B(kb0 + c * kpack + j, dst, slot);
                CW_LOAD_A(dst, slot);
              }
#ifdef CW_KB_TRACE
              if (cta == 0 && kbp < 64 && lane == 0 && pw == 0) kbt[1][kbp] = clock64();
              if (pw == 0) ++kbp;
#endif
            } else {
              for (int j = 0; j < m; ++j) CW_ADV_A();
            }
            if (++slot == ns) slot = 0;
          }
#undef CW_ACQUIRE
#undef CW_LOAD_B
#undef CW_LOAD_A
#undef CW_ADV_A
#undef CW_MINE
        }
      }
    }
  } else if ((warp == 2 || warp == 3) && (args.pre_bn || args.softmax)) {
    if (args.pre_bn) bn_prologue(sl, nl, cta, G, hdr, smem, bar_fpre, bar_xf, threadIdx.x - 64);
    if (args.softmax)
      softmax_tail(sl, nl, cta, G, ab, counters, gen1,
                   reinterpret_cast<float*>(bar_area + kMkBarBytes - 64), threadIdx.x - 64);

  } else if (warp == 1) {
    {
      // ======================= MMA issuer (whole warp converged; one elected lane issues)
      uint32_t par = 0;  // bit s: parity of the consumptions of slot s so far
      uint32_t xpar = 0;  // bit s: parity of the BN-transformed consumptions of slot s
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int L = 0; L < nl; ++L) {
        if (sl[L].kind != MK_CONV) continue;
        const MkLayer d = sl[L];
        const uint32_t idesc = idesc_bf16_f32(128, d.bn);
        const bool sw64 = d.kblk == 32;
        const int ns = d.slots, kpack = d.kpack;
        const uint32_t sb = (uint32_t)d.slot_bytes;
        // descriptor of slot 0 / sub-slot 0, and the 16-byte-unit strides of slots / sub-slots
        const uint64_t adesc0 = sw64 ? sw64_kmajor_desc(sbase) : sw128_kmajor_desc(sbase);
        const uint64_t bdesc0 = adesc0 + ((uint32_t)d.b_off >> 4);
        const uint32_t sdesc = sb >> 4, subdesc = (uint32_t)d.sub_bytes >> 4;
        int slot = 0;
        bool first = true;
        if (d.mode == 2) {
          // stem: per task 3 conv rows (accumulators 64 columns apart) x 7 kernel rows x 2 K=16
          // steps; A row j (conv column j) = the 64 bytes at 16j of staged row 2c + r: a
          // no-swizzle K-major view with overlapping rows (LBO 16 B, SBO 128 B); B resident
          // (4 KB of 64-byte-swizzled weights per kernel row)
          const uint64_t bst = sw64_kmajor_desc(obase + kMkStemB);
          const uint32_t pitch = (uint32_t)d.sub_bytes;
          if (first_task(d, cta, G) >= d.tasks) continue;  // (no weights were loaded here)
          mbar_wait_to<CW_HINT_FULL>(bar_stemb, 0, 5);
          for (int t = first_task(d, cta, G); t < d.tasks; t += G) {
            mbar_wait_to<CW_HINT_TEMPTY>(bar_tempty + 8 * acc, acc_phase ^ 1, 4);
            tc_fence_after();
            const uint32_t dtm = tmem + acc * 256;
            mbar_wait_to<CW_HINT_FULL>(bar_full + 8 * slot, (par >> slot) & 1, 5);
            par ^= 1u << slot;
            if (first) {
              if (lane == 0 && args.trace) args.trace[((size_t)L * G + cta) * 4 + 3] = globaltimer();
              first = false;
            }
            tc_fence_after();
            const uint32_t sa = sbase + slot * sb;
            if (elect_one()) {
#pragma unroll 1
              for (int c = 0; c < 3; ++c) {
#pragma unroll
                for (int r = 0; r < 7; ++r) {
                  const uint32_t ra = sa + (uint32_t)(2 * c + r) * pitch;
                  mma_bf16(dtm + 64 * c, desc_none(ra, 16, 128), bst + r * (4096 >> 4), idesc, r != 0);
                  mma_bf16(dtm + 64 * c, desc_none(ra + 32, 16, 128), bst + r * (4096 >> 4) + 2, idesc, 1);
                }
              }
              mma_commit(bar_empty + 8 * slot);
              mma_commit(bar_tfull + 8 * acc);
            }
            __syncwarp();
            if (++slot == ns) slot = 0;
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          }
          continue;
        }
        if (d.mode == 3) {
          // per slot: taps q = 0..2 of one (kernel row, channel block): the A operand is the
          // shared box read from row q (start + q x 128 B: the 128-byte swizzle follows the
          // absolute address bits, so an unaligned start needs no base-offset field)
          const uint32_t b3 = (uint32_t)d.bn * 128u;
          for (int t = first_task(d, cta, G); t < d.tasks; t += G) {
            int kb0, kb1;
            split_range(d, t % d.splits, kb0, kb1);
            const int ng = (kb1 - kb0) / 3;
            mbar_wait_to<CW_HINT_TEMPTY>(bar_tempty + 8 * acc, acc_phase ^ 1, 4);
            tc_fence_after();
            const uint32_t dtm = tmem + acc * 256;
            for (int i = 0; i < ng; ++i) {
              mbar_wait_to<CW_HINT_FULL>(bar_full + 8 * slot, (par >> slot) & 1, 5);
              par ^= 1u << slot;
              if (first) {
                if (lane == 0 && args.trace) args.trace[((size_t)L * G + cta) * 4 + 3] = globaltimer();
                first = false;
              }
              tc_fence_after();
              const uint32_t sa = sbase + slot * sb;
              if (elect_one()) {
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                  const uint64_t ad = sw128_kmajor_desc(sa + q * 128u);  // swizzle from address bits
                  const uint64_t bd = sw128_kmajor_desc(sa + d.b_off + q * b3);
                  mma_bf16(dtm, ad, bd, idesc, (i | q) != 0);
#pragma unroll
                  for (int k = 1; k < 4; ++k) mma_bf16(dtm, ad + 2 * k, bd + 2 * k, idesc, 1);
                }
                mma_commit(bar_empty + 8 * slot);
              }
              __syncwarp();
              if (++slot == ns) slot = 0;
            }
            if (elect_one()) mma_commit(bar_tfull + 8 * acc);
            __syncwarp();
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          }
          continue;
        }
        // a layer with an input BatchNorm consumes each A tile after warps 2-3 transformed
        // it in place: it waits on bar_xf (own phase bits xpar), and the fill of bar_full
        // it skipped still advances par
        const bool pre = d.pre_layer >= 0;
        const uint32_t bar_in = pre ? bar_xf : bar_full;
        for (int t = first_task(d, cta, G); t < d.tasks; t += G) {
          int kb0, kb1;
          split_range(d, t % d.splits, kb0, kb1);
          const int n = kb1 - kb0;
          mbar_wait_to<CW_HINT_TEMPTY>(bar_tempty + 8 * acc, acc_phase ^ 1, 4);
          tc_fence_after();
          const uint32_t dtm = tmem + acc * 256;
          for (int i = 0; i < n; i += kpack) {
            mbar_wait_to<CW_HINT_FULL>(bar_in + 8 * slot, ((pre ? xpar : par) >> slot) & 1, 5);
#ifdef CW_KB_TRACE
            if (cta == 0 && kbm < 64 && lane == 0) kbt[2][kbm] = clock64();
#endif
            (pre ? xpar : par) ^= 1u << slot;  // (a BN layer's fills never touch bar_full)
            if (first) {
              if (lane == 0 && args.trace) args.trace[((size_t)L * G + cta) * 4 + 3] = globaltimer();
              first = false;
            }
            tc_fence_after();
            const uint64_t ad = adesc0 + slot * sdesc, bd = bdesc0 + slot * sdesc;
            const int m = min(kpack, n - i);
            if (elect_one()) {
#ifdef CW_EXPERIMENTS
              if (!(args.flags & 1))
#endif
              {
                if (!sw64) {
                  mma_bf16(dtm, ad, bd, idesc, i != 0);
#pragma unroll
                  for (int k = 1; k < 4; ++k) mma_bf16(dtm, ad + 2 * k, bd + 2 * k, idesc, 1);
                  if (m > 1) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                      mma_bf16(dtm, ad + subdesc + 2 * k, bd + subdesc + 2 * k, idesc, 1);
                  }
                } else {
                  mma_bf16(dtm, ad, bd, idesc, i != 0);
                  mma_bf16(dtm, ad + 2, bd + 2, idesc, 1);
                  if (m > 1) {
                    mma_bf16(dtm, ad + subdesc, bd + subdesc, idesc, 1);
                    mma_bf16(dtm, ad + subdesc + 2, bd + subdesc + 2, idesc, 1);
                  }
                }
              }
              mma_commit(bar_empty + 8 * slot);
            }
            __syncwarp();
#ifdef CW_KB_TRACE
            if (cta == 0 && kbm < 64 && lane == 0) kbt[3][kbm] = clock64();
            ++kbm;
#endif
            if (++slot == ns) slot = 0;
          }
          if (elect_one()) mma_commit(bar_tfull + 8 * acc);
          __syncwarp();
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  }
  } else {
    setmaxnreg_inc<kMkRegsEpi>();  // warpgroups 1-2: epilogue
    // ======================= epilogue + SIMT layers (warps 4..11)
    const int q = warp & 3;  // TMEM lane quarter
    const int grp = (warp - kMkEpiWarp0) >> 2;  // column half of every 64-column chunk
    const int row = q * 32 + lane;
    const int et = threadIdx.x - kMkEpiWarp0 * 32;
    uint32_t ocnt = 0;  // TMA-epilogue chunks staged so far (buffer ocnt % kMkOutBufs)
    uint32_t rpar = 0;  // bit b: phase parity of the next residual landing in buffer b
    uint32_t simt_phase = 0;  // completed phases of bar_simt (SIMT-layer bulk copies)
    uint32_t cpar = 0;        // phase parity of bar_crdy / bar_crx (cluster split-K tasks)
    uint32_t cdpar = 0;       // phase parity of bar_cdone (cluster split-K layers)
    // per-warp staging: 32 rows x 128 B, 16-byte chunks XOR-swizzled by row
    uint8_t* stg = reinterpret_cast<uint8_t*>(sstage) + (warp - kMkEpiWarp0) * 4096;
    auto stg_chunk = [stg](int r, int c) {
      return reinterpret_cast<uint4*>(stg + r * 128 + ((c ^ (r & 7)) << 4));
    };
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int L = 0; L < nl; ++L) {
      if (sl[L].kind == MK_CONV) {
        const MkLayer& d = sl[L];  // constant-bank plan
        int t = first_task(d, cta, G);
        if (t >= d.tasks) continue;
        const float* bias_all = reinterpret_cast<const float* const*>(hdr + kHdrBiasOff)[d.wlayer];
        if (d.splits == 1) {
          // the layer's whole folded-BN bias (weights: no dependency), once per layer: no
          // per-task global loads or barriers (the previous layer ended on a barrier)
          if (d.f_kb) {  // fused shortcut: the two folded-BN biases add up
            const float* bias_sc =
                reinterpret_cast<const float* const*>(hdr + kHdrBiasOff)[d.f_wlayer];
            for (int i = et; i < d.n_out; i += kMkEpiThreads)
              sbias[i] = __ldg(bias_all + i) + __ldg(bias_sc + i);
          } else {
            for (int i = et; i < d.n_out; i += kMkEpiThreads) sbias[i] = __ldg(bias_all + i);
          }
        }
        if (et == 0) wait_deps(sl, L, counters, gen1, 6);
        named_bar(1, kMkEpiThreads);
        bool first = true;
        int done = 0;
        for (; t < d.tasks; t += G, ++done) {
          const int tile = t / d.splits;
          const int z = t - tile * d.splits;
          const TileOrigin o = tile_origin(d, tile);
          const uint32_t taddr = tmem + acc * 256 + ((uint32_t)(q * 32) << 16);
          CW_KET(62);
          if (d.csplit) {
            const uint32_t bar_acc = bar_tfull + 8 * acc;
            if (args.csize == 8)
              epi_csplit<8>(d, o, z, taddr, row, grp, et, obase, obufs, bar_acc, acc_phase,
                            bar_crdy, bar_crx, cpar, bias_all + o.n0);
            else if (args.csize == 4)
              epi_csplit<4>(d, o, z, taddr, row, grp, et, obase, obufs, bar_acc, acc_phase,
                            bar_crdy, bar_crx, cpar, bias_all + o.n0);
            else
              epi_csplit<2>(d, o, z, taddr, row, grp, et, obase, obufs, bar_acc, acc_phase,
                            bar_crdy, bar_crx, cpar, bias_all + o.n0);
            cpar ^= 1u;
          } else if (d.splits > 1) {
            // fp32 partial tile: 32-column chunks through the staging buffers (same protocol
            // as the TMA epilogue), drained by TMA stores into [tile][split][128][bn]
            mbar_wait_to<kEpiWaitNs>(bar_tfull + 8 * acc, acc_phase, 7);
            tc_fence_after();
            const CUtensorMap* tmp = args.tmaps + d.tmap_out;
            const int prow = (tile * d.splits + z) * 128;
            for (int c = 0; c < d.bn; c += 32, ++ocnt) {
              const uint32_t b = ocnt % kMkOutBufs;
              uint8_t* buf = obufs + b * kMkOutBufBytes;
              uint32_t v[16];
              tmem_ld16(taddr + c + 16 * grp, v);
              tmem_ld_wait();
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const int k = 4 * grp + kk;
                *reinterpret_cast<uint4*>(buf + row * 128 + ((k ^ (row & 7)) << 4)) =
                    make_uint4(v[4 * kk], v[4 * kk + 1], v[4 * kk + 2], v[4 * kk + 3]);
              }
              fence_proxy_async_smem();
              if (et == 0) bulk_wait_read<kMkOutBufs - 2>();
              named_bar(1, kMkEpiThreads);
              if (et == 0) {
                tma_store_2d(tmp, obase + b * kMkOutBufBytes, c, prow);
                bulk_commit();
              }
            }
          } else {
            // folded-BN bias of this tile's columns (staged for the whole layer)
            const float* bias = sbias + o.n0;
            constexpr bool bias_fixed = true;
            if (d.pool_pw) {
              CW_KET(200);
              mbar_wait_to<kEpiWaitNs>(bar_tfull + 8 * acc, acc_phase, 8);
              CW_KET(201);
              tc_fence_after();
              named_bar(1, kMkEpiThreads);  // bias staged; the previous tile's pooling reads are done
              epi_stem_pool(sl + L, o, taddr, bias, reinterpret_cast<uint8_t*>(sstage),
                            obufs + kMkPoolStage, obase + kMkPoolStage, args.tmaps + d.tmap_out,
                            row, grp, et);
              CW_KET(202);
            } else if (d.pool_out) {
              // Last conv: + bias (+ residual), ReLU, then a deterministic in-CTA
              // global average pool (the tile holds whole images).
              // (this row's pixel: only the pooled epilogue addresses rows itself)
              long long m;
              const bool valid = row_pixel(d, o, row, &m);
              const __nv_bfloat16* res_row =
                  (d.res && valid) ? reinterpret_cast<const __nv_bfloat16*>(d.res) + m * d.n_out + o.n0
                                   : nullptr;
              mbar_wait_to<kEpiWaitNs>(bar_tfull + 8 * acc, acc_phase, 8);
              tc_fence_after();
              if (!bias_fixed) named_bar(1, kMkEpiThreads);  // bias staged
              // the two column groups take alternate 16-column steps, each with its own
              // [128][17] reduction scratch
              float* sr = sred + grp * (128 * 17);
              const int etl = et & 127;
              for (int c = 16 * grp; c < d.bn; c += 32) {
                uint32_t v[16];
                tmem_ld16(taddr + c, v);
                tmem_ld_wait();
                float f[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]) + bias[c + i];
                if (res_row) {
                  float rf[8];
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    bf16x8_to_f32(__ldcg(reinterpret_cast<const uint4*>(res_row + c) + h), rf);
#pragma unroll
                    for (int e = 0; e < 8; ++e) f[8 * h + e] += rf[e];
                  }
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  if (d.relu) f[i] = fmaxf(f[i], 0.0f);
                  sr[row * 17 + i] = valid ? f[i] : 0.0f;
                }
                named_bar(1, kMkEpiThreads);
                const int hw = d.oh * d.ow;
                if (etl < 16 * d.box_n) {
                  const int img = etl >> 4, col = etl & 15;
                  float s = 0.0f;
                  for (int r = img * hw; r < (img + 1) * hw; ++r) s += sr[r * 17 + col];
                  if (o.img0 + img < d.nimg)
                    d.pool_out[(size_t)(o.img0 + img) * d.n_out + o.n0 + c + col] = s * d.pool_scale;
                }
                named_bar(1, kMkEpiThreads);
              }
            } else {
              // TMA epilogue, 64-column chunks through the staging buffers (running chunk
              // counter ocnt, buffer ocnt % kMkOutBufs): the residual chunk lands by TMA
              // (issued kMkOutBufs-1 chunks ahead, the first ones before the accumulator
              // wait), each thread rewrites its row in place with bias + residual (+ ReLU) in
              // bf16, and one thread drains the chunk with a TMA store (partial tiles are
              // clipped by the tensor map bounds).
              const CUtensorMap* tmo = args.tmaps + d.tmap_out;
              const CUtensorMap* tmr = d.res ? args.tmaps + d.tmap_res : nullptr;
              const int nch = d.bn >> 6;
              const bool m2d = d.mode == 0, relu = d.relu != 0;
              auto issue_res = [&](uint32_t b, int c) {
                const uint32_t dst = obase + b * kMkOutBufBytes, bar = bar_res + 8 * b;
                mbar_arrive_expect_tx(bar, a_rows(d) * 128u);  // the box: tile rows x 64 cols
                if (m2d) tma_load_2d_hint(dst, tmr, bar, o.n0 + 64 * c, o.m0, kHintRes);
                else tma_load_4d_hint(dst, tmr, bar, o.n0 + 64 * c, o.ow0, o.oh0, o.img0, kHintRes);
              };
              if (tmr && et == 0) {
                for (int j = 0; j < nch && j < kResDist; ++j) {
                  bulk_wait_read_n(kMkOutBufs - 1 - j);  // the buffer's previous store has read it
                  issue_res((ocnt + j) % kMkOutBufs, j);
                }
              }
              CW_KET(100 + t / G);
              mbar_wait_to<kEpiWaitNs>(bar_tfull + 8 * acc, acc_phase, 8);
              tc_fence_after();
              CW_KET(1);
              if (first && et == 0 && args.trace)
                args.trace[((size_t)L * G + cta) * 4 + 2] = globaltimer();
              first = false;
              if (!bias_fixed) named_bar(1, kMkEpiThreads);  // bias staged
              for (int c = 0; c < nch; ++c, ++ocnt) {
                const uint32_t b = ocnt % kMkOutBufs;
                uint8_t* buf = obufs + b * kMkOutBufBytes;
                auto chunk = [buf, row](int k) {
                  return reinterpret_cast<uint4*>(buf + row * 128 + ((k ^ (row & 7)) << 4));
                };
                // this thread's row: its group's 32 columns of the chunk (groups 4 grp .. +3),
                // in flight while the residual chunk is awaited
                uint32_t v[32];
                tmem_ld16(taddr + 64 * c + 32 * grp, *reinterpret_cast<uint32_t(*)[16]>(v));
                tmem_ld16(taddr + 64 * c + 32 * grp + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
                if (tmr) {
                  mbar_wait_to<64>(bar_res + 8 * b, (rpar >> b) & 1, 11);
                  rpar ^= 1u << b;
                }
                CW_KET(10 + c);
                tmem_ld_wait();
                CW_KET(40 + c);
                // branch-free per (residual, ReLU) variant: every shared-memory load first
                const float* b32 = bias + 64 * c + 32 * grp;
                if (tmr) {
                  if (relu) epi_chunk32<true, true>(v, b32, buf, row, grp);
                  else epi_chunk32<true, false>(v, b32, buf, row, grp);
                } else {
                  if (relu) epi_chunk32<false, true>(v, b32, buf, row, grp);
                  else epi_chunk32<false, false>(v, b32, buf, row, grp);
                }
                CW_KET(50 + c);
                fence_proxy_async_smem();
                // before the barrier: the store that last used the NEXT chunk's buffer has read it
                CW_KET(20 + c);
                if (et == 0) bulk_wait_read<kMkOutBufs - 2>();
                named_bar(1, kMkEpiThreads);
                CW_KET(30 + c);
                if (et == 0) {
                  const uint32_t src = obase + b * kMkOutBufBytes;
                  if (m2d) tma_store_2d_hint(tmo, src, o.n0 + 64 * c, o.m0, kHintOut);
                  else tma_store_4d_hint(tmo, src, o.n0 + 64 * c, o.ow0, o.oh0, o.img0, kHintOut);
                  bulk_commit();
                  if (tmr && c + kResDist < nch) {
                    // buffer of chunk c + kResDist - kMkOutBufs is free
                    bulk_wait_read<kMkOutBufs - kResDist>();
                    issue_res((ocnt + kResDist) % kMkOutBufs, c + kResDist);
                  }
                }
              }
            }
          }
          // accumulator drained: hand it back to the MMA warp
          CW_KET(60);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_tempty + 8 * acc);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          CW_KET(61);
        }
        if (d.csplit) {  // (this CTA had tasks: the cluster's ranks all did)
          csplit_drain(args.csize, et, bar_cdone, cdpar);
          cdpar ^= 1u;
        }
        // one release per layer and CTA: all of its tasks' stores (the TMA stores complete,
        // the threads' own stores cumulative over the bar.sync)
        CW_KET(90);
        if ((et & 31) == 0) {  // (et 0: TMA stores; lane 0 of every warp: split-K row stores)
          bulk_wait_all();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        CW_KET(91);
        named_bar(1, kMkEpiThreads);
        if (et == 0) {
          if (d.pool_out || d.csplit) red_release_add(counters + L, (uint32_t)done);  // generic stores
          else red_after_bulk_add(counters + L, (uint32_t)done);
        }
        CW_KET(92);
      } else {
        // SIMT layer (every CTA takes part; MK_REDUCE: its own task list)
        const MkLayer& d = sl[L];
        if (d.kind == MK_SOFTMAX) continue;  // run by warps 2-3 (softmax_tail)
        if (d.kind == MK_REDUCE && first_task(d, cta, G) >= d.tasks) continue;
        if (d.kind == MK_FC && et == 0) simt_fc_prefetch(d, hdr, cta, obase, bar_simt);
        if (et == 0) wait_deps(sl, L, counters, gen1, 9);
        named_bar(1, kMkEpiThreads);
        if (args.trace && et == 0) args.trace[((size_t)L * G + cta) * 4 + 1] = globaltimer();
        int done = 1;
        switch (d.kind) {
          case MK_INPUT:
            // staged in the operand ring, idle until this layer completes (the stem's weights
            // go to the staging buffers; its A boxes wait for this layer): the CTA's image rows
            // arrive in one phase (ResNet-50 b=16: 25 rows, 67 KB) instead of three
            if (ring_bytes >= kMkOutBufs * kMkOutBufBytes - kMkInputStage)
              simt_input(d, ab, cta, G, et, reinterpret_cast<float*>(smem), sbase, ring_bytes,
                         bar_simt, simt_phase);
            else
              simt_input(d, ab, cta, G, et, reinterpret_cast<float*>(obufs + kMkInputStage),
                         obase + kMkInputStage, kMkOutBufs * kMkOutBufBytes - kMkInputStage,
                         bar_simt, simt_phase);
            break;
          case MK_MAXPOOL: simt_maxpool(d, cta, G, et); break;
          case MK_AVGPOOL: simt_avgpool(d, hdr, cta, G, et); break;
          case MK_BNPOOL: simt_bnpool(d, hdr, cta, G, et); break;
          case MK_IM2COL: simt_im2col(d, ab, cta, G, et); break;
          case MK_FC:
            simt_fc(d, ab, hdr, cta, G, et, reinterpret_cast<float*>(smem), sbase,
                    reinterpret_cast<const __nv_bfloat16*>(obufs), obase,
                    reinterpret_cast<float*>(obufs + 3 * kMkOutBufBytes), bar_simt, simt_phase);
            break;

          case MK_REDUCE: {
            done = 0;
            for (int t = first_task(d, cta, G); t < d.tasks; t += G, ++done)
              simt_reduce(d, hdr, t, et, reinterpret_cast<const float*>(obufs), obase, bar_simt,
                          simt_phase, reinterpret_cast<uint8_t*>(sbias), smem_u32(sbias));
            break;
          }
          default: break;
        }
        if (args.trace && et == 0) args.trace[((size_t)L * G + cta) * 4 + 2] = globaltimer();
        named_bar(1, kMkEpiThreads);
        if (et == 0) {
          // reduce rows left by bulk copies; the last layer's outputs (FC logits or the
          // softmax) are read by nothing in this grid (mk_done and the output copies are
          // ordered after its completion); an FC followed by a softmax releases its stores
          if (d.kind == MK_REDUCE || (d.kind == MK_FC && !args.softmax))
            red_after_bulk_add(counters + L, (uint32_t)done);
          else red_release_add(counters + L, (uint32_t)done);  // generic stores
        }
      }
      if (args.trace && et == 0) args.trace[((size_t)L * G + cta) * 4] = globaltimer();
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef CW_KB_TRACE
  if (cta == 0 && threadIdx.x == kMkEpiWarp0 * 32 + CW_KB_ET) {
    for (int i = 0; i < kbe; ++i)
      printf("ep %2d tag %3d t %6lld\n", i, (int)ket[1][i], (long long)(ket[0][i] - ket[0][0]));
  }
  if (cta == 0 && threadIdx.x == 0) {
    for (int i = 0; i < 40; ++i)
      printf("kb %2d acq %6lld issued %6lld full %6lld committed %6lld\n", i,
             (long long)(kbt[0][i] - kbt[0][0]), (long long)(kbt[1][i] - kbt[0][0]),
             (long long)(kbt[2][i] - kbt[0][0]), (long long)(kbt[3][i] - kbt[0][0]));
  }
#endif
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, kMkTmemCols);
  }
  // (every remote access to this CTA's shared memory is awaited by this CTA itself; the
  // cluster barrier only keeps the exits ordered behind the cluster's last DSMEM traffic)
  if (args.csize > 1) cluster_sync();
  if (clk_trace && threadIdx.x == 0) {
    clk_trace[3] = clock64();
    clk_trace[2] = globaltimer();
  }
  if (threadIdx.x == 0) atomicMax(const_cast<unsigned long long*>(&ab->mk_t1), globaltimer());
  griddep_trigger();
}

// Bumps the plan generation after a completed (non-skipped) INFER and stamps Exec end.
__global__ void mk_done_kernel(const ActionBlock* ab, uint32_t ring_mask, ExecRecord* recs,
                               uint32_t* gen, volatile uint64_t* done) {
  griddep_wait();  // the megakernel has completed
  const uint64_t i = ab->seq;
  if (!ab->skip) *gen += 1u;
  ExecRecord* r = &recs[i & ring_mask];
  const uint64_t t_end = globaltimer();
  r->t_start = ab->t_start;
  r->rejected = ab->rejected;
  r->t_mk0 = ab->mk_t0;
  r->t_mk1 = ab->mk_t1;
  r->t_end = t_end;
  r->seq_started = i + 1;
  __threadfence_system();
  r->seq_done = i + 1;
  *done = i + 1;  // monotonic: INFERs of a device run in order on one Exec stream
}

// ------------------------------------------------------------------ host side

cudaError_t configure_mk() {
  cudaError_t e = cudaFuncSetAttribute(mk_infer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kMkSmemCap);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(mk_infer_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

// CTAs of the persistent grid for clusters of `csize` (all co-resident: CTAs wait on each
// other): the number of clusters of that size the GPU can hold at once, times csize.
int mk_cluster_ctas(int csize, uint32_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize * 256);
  cfg.blockDim = dim3(kMkThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, mk_infer_kernel, &cfg) != cudaSuccess) return 0;
  return n * csize;
}

uint32_t mk_smem_bytes(uint32_t ring_bytes, int n_layers) {
  (void)n_layers;  // the plan is in the constant bank
  return 1024 + ring_bytes + kMkOutBufs * kMkOutBufBytes + kMkBarBytes + kMkMaxCout * 4;
}

int mk_blocks_per_sm(uint32_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mk_infer_kernel, kMkThreads, smem) !=
      cudaSuccess)
    return 0;
  return n;
}

cudaError_t copy_plan(const MkLayer* d_layers, int n, cudaStream_t st) {
  if (n > kMkMaxPlanLayers) return cudaErrorInvalidValue;
  void* dst = nullptr;
  cudaError_t e = cudaGetSymbolAddress(&dst, c_plan);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(dst, d_layers, sizeof(MkLayer) * n, cudaMemcpyDeviceToDevice, st);
}

// Launch with programmatic stream serialization (PDL): the kernel may start before its
// predecessor in the stream completes; it synchronises with griddepcontrol.wait.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, uint32_t smem,
                              cudaStream_t st, int csize, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (csize > 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = csize;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

cudaError_t launch_mk(const MkArgs& a, int grid, uint32_t smem, cudaStream_t st) {
  return launch_pdl(mk_infer_kernel, dim3(grid), dim3(kMkThreads), smem, st, a.csize, a);
}

void launch_mk_done(const ActionBlock* ab, uint32_t mask, ExecRecord* recs, uint32_t* gen,
                    volatile uint64_t* done, cudaStream_t st) {
  launch_pdl(mk_done_kernel, dim3(1), dim3(1), 0, st, 1, ab, mask, recs, gen, done);
}

}  // namespace cw
