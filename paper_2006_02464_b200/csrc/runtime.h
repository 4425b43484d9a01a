// Per-GPU device runtime of the B200 Clockwork worker.
//
// Owns every byte of device memory the worker uses, all allocated once at
// open ("Workspace / IOCache / PageCache"):
//   * PageCache pool: pages_total x page_bytes of HBM. Model weights are copied
//     into non-contiguous pages; no allocator call on the LOAD/INFER path.
//   * IOCache: fixed per-request slots (fp32 input image + fp32 logits).
//   * Workspace: per-arch activation buffers sized for the largest batch.
// and three streams: Exec (INFER graph), Load (weights H2D, PAPER.md:1633
// "dedicated CUDA streams"), IO (request input H2D / logits D2H).
//
// One CUDA graph per (arch, batch size) is instantiated at start; the graph
// reads its per-action parameters from the device ActionBlock, which the
// gate kernel fills from the host descriptor ring.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <map>
#include <string>
#include <vector>
#include "cw_device.h"
#include "mk.h"

namespace cw {

// Mirrors struct cw_op in include/cw.h.
struct CwOp {
  int32_t kind;  // OpKind
  int32_t layer;
  int32_t in_buf, out_buf, res_buf;
  int32_t cin, cout, kh, kw, stride, pad, relu;
  int32_t in_h, in_w, out_h, out_w;
  int32_t kpad;
  int32_t pad_w, in_ctot, out_ctot, out_coff, cout_pad, flags, pre_layer;
};
enum OpKind { OP_STEM = 0, OP_CONV = 1, OP_MAXPOOL = 2, OP_AVGPOOL = 3, OP_FC = 4,
              OP_IM2COL = 5, OP_BNPOOL = 6, OP_SOFTMAX = 7 };
enum OpFlags { OPF_GROUPED64 = 1, OPF_PRE_BN = 2 };

// Mirrors struct cw_tensor_loc: where one layer's tensors sit in a blob (-1 = absent).
struct CwTensorLoc {
  int64_t w_off;  // bf16 [rows][k] at this blob byte offset
  int64_t b_off;  // fp32 [rows]
  int32_t rows;
  int32_t k;
  int64_t s_off;  // fp32 [2][cin_pad]: BatchNorm scale / shift applied to the layer's input
};

// One (arch, batch) INFER plan: the megakernel's layer table (mk.h) in device
// memory, its A-operand tensor maps, completion counters and generation, and
// the captured graph gate -> megakernel -> done.
struct Plan {
  int batch = 0;
  std::vector<MkLayer> layers;
  std::vector<int> layer_op;  // arch op index of each layer
  std::vector<CUtensorMap> tmaps;
  MkLayer* d_layers = nullptr;
  CUtensorMap* d_tmaps = nullptr;
  uint32_t* d_counters = nullptr;
  uint32_t* d_gen = nullptr;
  uint64_t* d_trace = nullptr;
  float* d_partial = nullptr;
  uint32_t ring_bytes = 0, smem = 0;
  int grid = 0;
  int csize = 1;  // thread-block cluster size of the megakernel launch (cluster split-K)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // the same INFER without the plan-table copy into the constant bank: launched when the
  // previous INFER on this device ran this very plan (its table is still there)
  cudaGraph_t graph_nocopy = nullptr;
  cudaGraphExec_t exec_nocopy = nullptr;
  uint64_t uid = 0;  // process-unique plan id (what the device's constant bank holds)
  int launches = 0;  // kernels per INFER (gate + megakernel + done)
};

struct Arch {
  int id = -1;
  std::vector<CwOp> ops;
  int n_layers = 0;
  int in_c = 3, in_h = 224, in_w = 224, classes = 1000;
  std::vector<void*> bufs;
  std::vector<size_t> buf_bytes;
  std::map<int, Plan> plans;
  double flops_per_image = 0;
  float* in_pool = nullptr;  // pinned synthetic request inputs of this arch (image r % n)
  int in_pool_n = 0;
  int64_t in_pool_bytes = 0;
};

struct Blob {
  int id = -1;
  int arch = -1;
  uint8_t* host = nullptr;  // pinned
  size_t bytes = 0;
  int npages = 0;
  std::vector<CwTensorLoc> locs;
};

// Completion record for LOAD copies (mapped pinned memory).
struct alignas(64) LoadRecord {
  volatile uint64_t t_start, tag_start;
  volatile uint64_t t_end, tag_end;
};
// Completion record for Input copies.
struct alignas(32) StampRecord {
  volatile uint64_t t, tag;
};

class Runtime {
 public:
  static constexpr uint32_t kRing = 1024;

  Runtime() = default;
  ~Runtime();
  // Returns "" on success, else an error message.
  std::string open(int device, int64_t pages_total, int64_t page_bytes, int64_t io_slots,
                   int64_t in_bytes_max, int64_t out_bytes_max, int input_pool);
  std::string register_arch(int id, const CwOp* ops, int n_ops, int n_layers, int in_c, int in_h,
                            int in_w, int classes, const int* batches, int n_batches);
  std::string register_blob(int id, int arch, const void* data, size_t bytes,
                            const CwTensorLoc* locs, int n_locs);
  std::string build_plans();  // allocate workspace + capture graphs

  int device() const { return device_; }
  int64_t pages_total() const { return pages_total_; }
  int64_t page_bytes() const { return page_bytes_; }
  uint8_t* page_ptr(int32_t p) const { return pool_ + (int64_t)p * page_bytes_; }
  int blob_pages(int blob) const;
  int arch_of_blob(int blob) const;

  // ---- LOAD: copy blob `blob` into physical pages (async on the Load stream).
  // Page-reuse fence: when fence_seq >= 0 (the last INFER that read one of these pages)
  // and that INFER has not completed, the copy first waits for it on the device.
  // The record slot is returned; completion when rec->tag_end == tag.
  // peer: copy the weights from `peer`'s resident pages of the same
  // blob (cudaMemcpyPeerAsync) instead of from pinned host memory; the header (absolute
  // addresses of THESE pages) still comes from the host. `waits`: events of earlier peer
  // copies that read these pages as their source (they must finish before the overwrite);
  // `done`: recorded on the Load stream after the copies.
  std::string load_async(int blob, const int32_t* pages, int npages, int64_t fence_seq,
                         uint64_t tag, LoadRecord** rec, const Runtime* peer = nullptr,
                         const int32_t* peer_pages = nullptr,
                         const std::vector<cudaEvent_t>* waits = nullptr,
                         cudaEvent_t done = nullptr);

  // ---- Input stage: copy request inputs into IOCache slots (async, IO stream).
  // Completion when rec->tag == tag.
  std::string input_async(int arch, const int32_t* slots, const uint64_t* request_ids, int batch,
                          uint64_t tag, StampRecord** rec);
  // Device-resident variant for tests/bench: copy from a host buffer of `batch` images.
  std::string input_from_host(int arch, const int32_t* slots, const float* host, int batch);

  // ---- Exec: dispatch the (arch, batch) graph for a resident model whose
  // header sits at page `hdr_page`. Returns the exec sequence number; the
  // ExecRecord ring entry seq & (kRing-1) completes when seq_done == seq+1.
  // input_seq >= 0: the Exec stream first waits for that Input copy.
  std::string exec_async(int arch, int batch, int32_t hdr_page, const int32_t* slots,
                         uint64_t earliest_gt, uint64_t latest_gt, int64_t input_seq,
                         uint64_t* seq_out);
  int64_t last_input_seq() const { return last_input_seq_; }
  ExecRecord* exec_record(uint64_t seq) { return &exec_recs_[seq & (kRing - 1)]; }
  uint64_t exec_issued() const { return exec_seq_; }
  // INFERs completed on the device (monotonic, written by mk_done): exec seq s is done
  // iff exec_completed() > s, whatever the ring slot of s holds by now
  uint64_t exec_completed() const { return *exec_done_; }

  // ---- Output stage: after exec `seq`, copy logits of the slots to pinned host
  // memory (out_ring entry seq) and stamp completion into the ExecRecord.
  std::string output_async(int arch, uint64_t seq, const int32_t* slots, int batch);
  const float* output_host(uint64_t seq) const {
    return out_host_ + (seq & (kRing - 1)) * (size_t)kMaxBatch * out_floats_max_;
  }

  // One INFER of the (arch, batch) plan with the megakernel's per-layer trace
  // read back: for every plan layer, the time (ms) from Exec start until its
  // last task finished on any SM, and the layer kind (profiling / roofline).
  std::string profile_layers(int arch, int batch, int32_t hdr_page, std::vector<float>* end_ms,
                             std::vector<int>* kinds);
  const Plan* plan(int arch, int batch) const;
  // Raw trace of the last profile_layers run ([layers][grid][4], see MkArgs::trace).
  const std::vector<uint64_t>& last_trace() const { return last_trace_; }
  uint64_t last_trace_t0() const { return last_trace_t0_; }

  // Blocking helpers (tests, bench).
  std::string sync_all();
  int64_t clock_offset() const { return gt_offset_; }  // globaltimer - CLOCK_REALTIME
  std::string calibrate_clock();
  // A fresh globaltimer - CLOCK_REALTIME measurement (diagnostics: drift since open).
  std::string measure_clock_offset(int64_t* offset);
  // Quick re-calibration (call while no INFER runs, so the stamp kernel finds an SM): the
  // globaltimer drifts against CLOCK_REALTIME by tens of ppm (measured ~1.7 ms / min), far
  // too much for the controller's 1 ms window slack. One stamp kernel per attempt, accepted
  // if its host round trip is short; *step = the offset change applied (0 if none).
  bool resync_clock(int64_t* step);
  const Arch* arch(int id) const;
  cudaStream_t exec_stream() const { return s_exec_; }
  float* slot_in(int32_t s) const { return reinterpret_cast<float*>(io_ + (int64_t)s * slot_bytes_); }
  float* slot_out(int32_t s) const {
    return reinterpret_cast<float*>(io_ + (int64_t)s * slot_bytes_ + in_bytes_max_);
  }
  int64_t io_slots() const { return io_slots_; }
  int64_t output_stride_floats() const { return out_floats_max_; }
  // Fill an arch's input pool with `n` images of `bytes` each (pinned copy).
  std::string set_input_pool(int arch, const float* data, int n, int64_t bytes);

 private:
  std::string build_plan(Arch& a, int batch, bool allow_split = true);
  std::string capture(Arch& a, Plan& p);
  int num_sms_ = 148;
  std::vector<uint64_t> last_trace_;
  uint64_t last_trace_t0_ = 0;

  int device_ = -1;
  int64_t pages_total_ = 0, page_bytes_ = 0;
  uint8_t* pool_ = nullptr;
  uint8_t* io_ = nullptr;
  int64_t io_slots_ = 0, slot_bytes_ = 0, in_bytes_max_ = 0, out_bytes_max_ = 0;
  int64_t out_floats_max_ = 0;
  cudaStream_t s_exec_ = nullptr, s_load_ = nullptr, s_io_ = nullptr, s_cap_ = nullptr,
               s_out_ = nullptr;
  ActionBlock* ab_ = nullptr;   // device
  uint64_t* ctr_ = nullptr;     // device
  ActionDesc* ring_ = nullptr;  // mapped host
  ExecRecord* exec_recs_ = nullptr;  // mapped host
  volatile uint64_t* exec_done_ = nullptr;  // mapped host: INFERs completed (mk_done)
  volatile uint64_t* sync_slot_ = nullptr;  // mapped host: resync stamp (time, tag)
  uint64_t sync_tag_ = 0;
  LoadRecord* load_recs_ = nullptr;  // mapped host
  StampRecord* in_recs_ = nullptr;   // mapped host
  float* out_host_ = nullptr;        // pinned host, kRing x kMaxBatch x out_floats
  uint8_t* hdr_stage_ = nullptr;     // pinned host, kRing/16 headers
  uint64_t exec_seq_ = 0;
  uint64_t load_seq_ = 0;
  uint64_t in_seq_ = 0;
  int64_t last_input_seq_ = -1;
  std::vector<cudaEvent_t> exec_events_;  // recorded after each exec, ring
  std::vector<cudaEvent_t> in_events_;    // recorded after each input copy, ring
  std::map<int, Arch> archs_;
  std::map<int, Blob> blobs_;
  int64_t gt_offset_ = 0;
  bool plans_built_ = false;
};

}  // namespace cw
