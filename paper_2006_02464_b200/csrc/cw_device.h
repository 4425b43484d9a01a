// Device-side data structures shared by the INFER kernels and the host runtime.
//
// Layout in HBM:
//   * Model header: the first kHeaderBytes of a resident model's page 0. It is
//     written by the LOAD copy (built on the host at LOAD time because it holds
//     absolute addresses of the model's pages): two CUtensorMaps per layer for
//     the weight matrix ([Cout][KH*KW*Cin] bf16, K-major; 64-row boxes and
//     min(256, Cout)-row boxes), then a table of per-layer bias pointers (fp32,
//     folded BatchNorm shift) and raw weight pointers.
//   * ActionBlock: one per engine in device memory, rewritten by the gate
//     kernel at the start of every INFER from the host descriptor ring. Every
//     kernel of the per-(arch, batch) CUDA graph reads its dynamic inputs
//     (model header, IOCache input/output slots, skip flag) from here, so one
//     graph serves every copy of an arch.
#pragma once
#include <cstdint>

namespace cw {

constexpr int kMaxLayers = 192;        // header entries: DenseNet-169 has 173, ResNet-152 156
constexpr int kMaxBatch = 16;
constexpr uint32_t kTmapBytes = 128;
// weight tensor maps: box 64 rows x 64 K at [0, ...), box min(256, Cout) rows at kHdrWideOff
constexpr uint32_t kHdrWideOff = kMaxLayers * kTmapBytes;
constexpr uint32_t kHdrBiasOff = 2 * kMaxLayers * kTmapBytes;       // const float* [kMaxLayers]
constexpr uint32_t kHdrWeightOff = kHdrBiasOff + kMaxLayers * 8;   // const void*  [kMaxLayers]
// input BatchNorm (DenseNet pre-activation): const float* [kMaxLayers] -> scale[cin_pad],
// shift[cin_pad]
constexpr uint32_t kHdrPreOff = kHdrWeightOff + kMaxLayers * 8;
constexpr uint32_t kHeaderBytes = 65536;                             // reserved at blob start
static_assert(kHdrPreOff + kMaxLayers * 8 <= kHeaderBytes, "model header overflow");

struct ActionBlock {
  const uint8_t* hdr;          // model header (page 0 of the model)
  const float* in[kMaxBatch];  // per-request input image, fp32 NCHW 3xHxW (IOCache slot)
  float* out[kMaxBatch];       // per-request logits destination (IOCache slot)
  int32_t skip;                // 1: window missed, every kernel returns immediately
  int32_t batch;
  uint64_t seq;
  unsigned long long mk_t0;    // megakernel: earliest CTA start / latest CTA end (%globaltimer)
  unsigned long long mk_t1;
  uint64_t t_start;            // gate: Exec start (%globaltimer); copied to the host record by
  int32_t rejected;            // mk_done, off the gate -> megakernel critical path
  int32_t pad_;
};

// Host -> device descriptor ring entry (mapped pinned memory).
struct ActionDesc {
  uint64_t seq;
  uint64_t earliest_gt;        // %globaltimer domain
  uint64_t latest_gt;
  const uint8_t* hdr;
  const float* in[kMaxBatch];
  float* out[kMaxBatch];
  int32_t batch;
  int32_t pad_;
};

// Device -> host completion record (mapped pinned memory).
struct alignas(64) ExecRecord {
  volatile uint64_t seq_started;   // == seq once the gate ran
  volatile uint64_t t_start;       // %globaltimer at Exec start
  volatile uint64_t seq_done;      // == seq once the last Exec kernel ran
  volatile uint64_t t_end;         // %globaltimer at Exec end
  volatile int32_t rejected;       // gate found now > latest
  volatile int32_t pad_;
  volatile uint64_t seq_out;       // == seq once the Output copy completed
  volatile uint64_t t_out;
  volatile uint64_t t_mk0;         // megakernel span inside [t_start, t_end] (diagnostics)
  volatile uint64_t t_mk1;
};

}  // namespace cw
