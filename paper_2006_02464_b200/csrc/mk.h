// The INFER megakernel's plan format (host planner <-> device kernel).
//
// One persistent kernel per INFER runs the whole network: grid = one CTA per
// SM, each CTA walks the plan's layers in order and executes the tasks of each
// layer that the static round-robin assigns to it. Layers synchronise through
// per-layer completion counters in global memory (release/acquire at gpu
// scope) instead of kernel boundaries, so there is no per-layer launch,
// prologue, TMEM allocation or tensor-map fetch on the critical path, and the
// kernel sequence of an (arch, batch) plan is fixed (one
// precompiled kernel sequence per batch size).
//
// Counters never reset: a plan's generation g (bumped by mk_done after every
// non-skipped INFER) makes layer L complete when counter[L] == (g+1)*tasks[L]
// (mod 2^32, compared wrap-safely).
#pragma once
#include <cuda.h>
#include <cstdint>

#include "cw_device.h"

namespace cw {

enum MkKind : int32_t {
  MK_CONV = 1,     // tcgen05 implicit-GEMM conv tile(s)
  MK_INPUT = 2,    // fp32 NCHW request images -> bf16 NHWC4 (left/right padded rows)
  MK_MAXPOOL = 3,  // 3x3 / stride 2 / pad 1
  MK_AVGPOOL = 4,  // global average pool -> fp32 [b][C]
  MK_FC = 5,       // logits = pooled . W^T + bias -> request output slots
  MK_REDUCE = 6,   // split-K: sum fp32 partial tiles + bias (+ residual) (+ ReLU) -> bf16
  MK_IM2COL = 7,   // fp32 NCHW request images -> bf16 [M][64] patches (first conv, C=3)
  MK_BNPOOL = 8,   // BatchNorm + ReLU + 2x2/s2 average pool (DenseNet transition)
  MK_SOFTMAX = 9,  // logits -> probabilities in the request output slots (optional tail)
};

constexpr int kMkMaxDeps = 6;
#ifndef CW_PRODUCERS
#define CW_PRODUCERS 1
#endif
// TMA producer warps: warp 0 (and warp 2): producer p fills the ring slots s with s % P == p, so
// the issue path of P k-blocks runs in parallel (one warp's path is ~570 cycles per k-block).
constexpr int kMkProducers = CW_PRODUCERS;
// Warpgroup 0: warp 0 (+2) TMA, warp 1 MMA (registers lowered to kMkRegsCtl). Warpgroups 1-2:
// eight epilogue / SIMT warps (registers raised to kMkRegsEpi), two per TMEM lane quarter:
// epilogue group g = (warp - 4) / 4 takes columns [32g, 32g + 32) of every 64-column chunk.
constexpr int kMkThreads = 384;
constexpr int kMkEpiWarp0 = 4;
constexpr int kMkEpiThreads = 256;
constexpr int kMkRegsCtl = 120;
constexpr int kMkRegsEpi = 192;
static_assert(kMkRegsCtl * 128 + kMkRegsEpi * 256 <= 65536, "register file");
constexpr uint32_t kMkATile = 128 * 128;   // A tile: 128 rows x 128 B
// MK_INPUT: zero pixels left (and right) of every row. 4: conv column j of the 7x7/s2 stem
// reads padded pixels 2j .. 2j+7 (input columns 2j-4 .. 2j+3: the weights' K slot 0 is the
// zero tap), i.e. the 64 bytes at byte 16j of the row: 16-byte aligned rows of the stem's
// implicit-im2col A operand (see the stem in mk_infer.cu)
constexpr int kMkPadW = 4;
constexpr int kMkPadH = 3;                 // MK_INPUT: zero rows above and below every image
// stem (mode 2): one task = one pooled output row = 3 conv rows x the full conv width; its A
// operand is the kMkStemRows padded input rows those conv rows read, staged once (one TMA box),
// each MMA reading conv column j's 8 pixels x 4 channels at byte 16j of a staged row
// (overlapping rows of a no-swizzle K-major descriptor: LBO 16 B, SBO 128 B)
constexpr int kMkStemRows = 11;
// staging-buffer map: resident stem weights [0, 28 KB) (written by the producer while the
// input conversion still runs), input-conversion stage [32 KB, 64 KB), stem-pool / split-K
// scratch at 32 KB, avg-pool scratch at 16 KB
constexpr uint32_t kMkStemB = 0;
constexpr uint32_t kMkInputStage = 32768;
constexpr uint32_t kMkScratch = 32768;
constexpr uint32_t kMkPoolStage = 49152;  // stem: pooled pixels of one tile (TMA-store source)
constexpr uint32_t kMkTmemCols = 512;      // two accumulators of up to 256 columns
constexpr int kMkMaxSlots = 16;            // smem ring slots (per-layer slot size)
constexpr uint32_t kMkBarBytes = 1024;
constexpr int kMkMaxCout = 2048;  // shared-memory bias of one layer (fp32)
// Epilogue staging: kMkOutBufs buffers of one 128-row x 64-column bf16 chunk (16 KB, 128-byte
// swizzle): a chunk's residual lands there by TMA, the epilogue rewrites it in place with the
// output, and a TMA store drains it. Also the stem-pool / split-K / avg-pool scratch.
#ifndef CW_OUT_BUFS
#define CW_OUT_BUFS 4
#endif
constexpr int kMkOutBufs = CW_OUT_BUFS;
constexpr uint32_t kMkOutBufBytes = 16384;
static_assert(kMkOutBufs >= 4, "the staging-buffer map (kMkStemB, kMkInputStage) needs 64 KB");
#ifdef CW_KB_TRACE
constexpr uint32_t kMkSmemCap = 224 * 1024;  // debug builds keep a static trace array
#else
constexpr uint32_t kMkSmemCap = 227 * 1024;  // dynamic shared memory per CTA
#endif      // full/empty[16], tfull/tempty[2], tmem + gen slots

struct MkLayer {
  int32_t kind, tasks, rot, ndeps;
  int32_t deps[kMkMaxDeps];
  // ---- MK_CONV / MK_REDUCE geometry
  int32_t mode;  // 0: A = [M][K] matrix; 1: A = NHWC tensor (tap-shifted boxes); 2: stem windows
  int32_t bn, m_tiles, n_tiles, splits, kb_per_split, num_kb, cin_kb, kw, stride, pad;
  int32_t box_w, box_h, box_n, tiles_w, tiles_h, m_total, nimg, oh, ow;
  int32_t relu, wlayer, n_out, tmap, red_rows, kblk;  // kblk: K elements per k-block (64 or 32)
  int32_t slots, slot_bytes, b_off;  // smem ring geometry of this layer (B tile at b_off in a sub-slot)
  int32_t kpack, sub_bytes;  // k-blocks per ring slot (sub-slots of sub_bytes) behind one barrier
  int32_t tmap_out, tmap_res;  // TMA store / residual-load maps (64-column boxes), -1 if unused
  // stem with fused 3x3/s2/p1 max pool: pooled columns per tile (0 = no fusion);
  // a tile covers conv rows 2ph-1..2ph+1 and conv columns 2pw0-1..2pw0+2*pool_pw-1
  int32_t pool_pw, pool_oh;
  float pool_scale;
  // ---- SIMT layers
  int32_t H, W, C, OH, OW, classes, batch, red_parts;
  // ---- zoo generalisation
  int32_t pad_w;      // conv: horizontal padding (pad = vertical)
  int32_t in_ctot;    // SIMT: channel stride of the input buffer
  int32_t out_ctot;   // SIMT / split-K reduce: channel stride of the output buffer
  int32_t out_coff;   // ... and the first channel written (conv TMA stores: folded into the map)
  int32_t n_valid;    // channels actually stored (cout; n_out is cout padded to the N tile)
  int32_t grouped;    // conv: K walks the tile's own 64-channel block only (ResNeXt groups)
  int32_t pre_layer;  // BatchNorm + ReLU of the input (conv A tile / pool), header entry; -1
  // conv: split-K across the CTAs of one thread-block cluster (splits == cluster size, split z
  // on cluster rank z): the partial tiles are reduced through distributed shared memory in the
  // epilogue (no fp32 partials in global memory, no reduce layer)
  int32_t csplit;
  // conv: a second K segment accumulated into the same tile (a bottleneck's projection
  // shortcut fused into its conv3: K = [conv3's input | the block input], the shortcut's
  // 1x1 / stride f_stride conv read through its own A map f_tmap and weight layer f_wlayer);
  // k-blocks [num_kb - f_kb, num_kb) belong to it; f_kb == 0: no second segment
  int32_t f_tmap, f_wlayer, f_kb, f_stride;
  void* out;              // bf16 NHWC output (conv / reduce / pools), NHWC4 (input)
  const void* res;        // bf16 residual, same shape as out, or null
  float* partial;         // split-K fp32 partials [tile][split][128][bn]
  float* pool_out;        // fused global average pool [b][n_out] fp32, or null
  const void* in;         // SIMT input
};

static_assert(sizeof(MkLayer) % 16 == 0, "MkLayer is copied in 16-byte units");
// The plan's layer table lives in a __constant__ bank (mk_infer.cu), refreshed by a
// device-to-device memcpy node at the head of every INFER graph: uniform (ULDC) operand
// reads for the producer / MMA loops and no shared memory, whatever the depth of the net.
constexpr int kMkMaxPlanLayers = 210;
static_assert(kMkMaxPlanLayers * sizeof(MkLayer) <= 64000, "constant bank (64 KB)");

struct MkArgs {
  const MkLayer* layers;
  const CUtensorMap* tmaps;  // A-operand tensor maps (64-byte aligned, device memory)
  int32_t n_layers;
  uint32_t ring_bytes;       // smem ring (slots of the per-layer size)
  const ActionBlock* ab;
  uint32_t* counters;        // [n_layers]
  const uint32_t* gen;
  // optional [n_layers][gridDim.x][4] %globaltimer: 0 layer done (epilogue), 1 inputs
  // ready (producer), 2 first accumulator ready (epilogue), 3 first tile landed (MMA)
  uint64_t* trace;
  uint32_t flags;            // experiments only (CW_MK_FLAGS): 1 no MMA, 2 no A loads, 4 no B loads
  int32_t pf_depth;          // weight layers L2-prefetched ahead of the running conv
  int32_t pre_bn;            // 1: some conv applies a BN+ReLU prologue (warps 2-3 run it)
  int32_t softmax;           // 1: the last layer is a softmax tail (warps 2-3 run it)
  int32_t csize;             // thread-block cluster size of the launch (1: no clusters)
};

}  // namespace cw
