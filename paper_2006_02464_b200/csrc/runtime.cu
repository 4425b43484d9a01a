#include "runtime.h"

#include <algorithm>
#include <climits>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <mutex>
#include <thread>
#include <vector>

#include "experiments.h"
#include "kernels.h"
#include "tmap.h"

namespace cw {

#define CW_TRY(expr)                                                                  \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return std::string(#expr) + ": " + cudaGetErrorString(_e);                      \
  } while (0)

// One Exec stream per device for every Runtime of the process: the megakernel's plan
// lives in a process-wide __constant__ bank (copied by the head node of each INFER
// graph) and its persistent grid assumes it owns the SMs, so INFERs of two runtimes on
// one device must never overlap. Sharing the stream serialises them.
namespace {
std::mutex g_exec_mu;
std::map<int, std::pair<cudaStream_t, int>> g_exec_streams;  // device -> (stream, users)
// device -> uid of the plan whose table the last INFER launched on it copied into the
// constant bank (launches are serialised on the device's Exec stream, in this order)
std::map<int, uint64_t> g_bank_plan;
std::atomic<uint64_t> g_plan_uid{1};

cudaError_t acquire_exec_stream(int device, cudaStream_t* out) {
  std::lock_guard<std::mutex> lk(g_exec_mu);
  auto it = g_exec_streams.find(device);
  if (it != g_exec_streams.end()) {
    ++it->second.second;
    *out = it->second.first;
    return cudaSuccess;
  }
  cudaError_t e = cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
  if (e == cudaSuccess) g_exec_streams[device] = {*out, 1};
  return e;
}

void release_exec_stream(int device) {
  std::lock_guard<std::mutex> lk(g_exec_mu);
  auto it = g_exec_streams.find(device);
  if (it == g_exec_streams.end()) return;
  if (--it->second.second == 0) {
    cudaStreamDestroy(it->second.first);
    g_exec_streams.erase(it);
  }
}
}  // namespace

static int64_t realtime_ns() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

Runtime::~Runtime() {
  if (device_ < 0) return;
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  for (auto& [id, a] : archs_) {
    for (auto& [b, p] : a.plans) {
      if (p.exec) cudaGraphExecDestroy(p.exec);
      if (p.graph) cudaGraphDestroy(p.graph);
      if (p.exec_nocopy) cudaGraphExecDestroy(p.exec_nocopy);
      if (p.graph_nocopy) cudaGraphDestroy(p.graph_nocopy);
      cudaFree(p.d_layers);
      cudaFree(p.d_tmaps);
      cudaFree(p.d_counters);
      cudaFree(p.d_gen);
      cudaFree(p.d_trace);
      cudaFree(p.d_partial);
    }
    for (void* b : a.bufs) cudaFree(b);
    if (a.in_pool) cudaFreeHost(a.in_pool);
  }
  for (auto& [id, bl] : blobs_) cudaFreeHost(bl.host);
  for (auto e : exec_events_) cudaEventDestroy(e);
  for (auto e : in_events_) cudaEventDestroy(e);
  cudaFree(pool_);
  cudaFree(io_);
  cudaFree(ab_);
  cudaFree(ctr_);
  cudaFreeHost(ring_);
  cudaFreeHost(exec_recs_);
  cudaFreeHost((void*)exec_done_);
  cudaFreeHost((void*)sync_slot_);
  cudaFreeHost(load_recs_);
  cudaFreeHost(in_recs_);
  cudaFreeHost(out_host_);
  cudaFreeHost(hdr_stage_);
  for (auto s : {s_load_, s_io_, s_cap_, s_out_})
    if (s) cudaStreamDestroy(s);
  if (s_exec_) release_exec_stream(device_);
}

std::string Runtime::open(int device, int64_t pages_total, int64_t page_bytes, int64_t io_slots,
                          int64_t in_bytes_max, int64_t out_bytes_max, int input_pool) {
  int n = 0;
  CW_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return "device index out of range";
  device_ = device;
  CW_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CW_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return std::string("sm_100a required, found ") + prop.name;
  if (!tmap_init()) return "cuTensorMapEncodeTiled unavailable";
  CW_TRY(configure_mk());
  num_sms_ = prop.multiProcessorCount;
  pages_total_ = pages_total;
  page_bytes_ = page_bytes;
  CW_TRY(cudaMalloc(&pool_, (size_t)(pages_total * page_bytes)));
  in_bytes_max_ = (in_bytes_max + 255) / 256 * 256;
  out_bytes_max_ = (out_bytes_max + 255) / 256 * 256;
  out_floats_max_ = out_bytes_max_ / 4;
  slot_bytes_ = in_bytes_max_ + out_bytes_max_;
  io_slots_ = io_slots;
  CW_TRY(cudaMalloc(&io_, (size_t)(io_slots * slot_bytes_)));
  for (cudaStream_t* s : {&s_load_, &s_io_, &s_cap_, &s_out_})
    CW_TRY(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
  CW_TRY(acquire_exec_stream(device, &s_exec_));
  CW_TRY(cudaMalloc(&ab_, sizeof(ActionBlock)));
  CW_TRY(cudaMemset(ab_, 0, sizeof(ActionBlock)));
  CW_TRY(cudaMalloc(&ctr_, sizeof(uint64_t)));
  CW_TRY(cudaMemset(ctr_, 0, sizeof(uint64_t)));
  CW_TRY(cudaHostAlloc(&ring_, sizeof(ActionDesc) * kRing, cudaHostAllocMapped));
  CW_TRY(cudaHostAlloc(&exec_recs_, sizeof(ExecRecord) * kRing, cudaHostAllocMapped));
  {
    void* p = nullptr;
    CW_TRY(cudaHostAlloc(&p, 64, cudaHostAllocMapped));
    exec_done_ = static_cast<volatile uint64_t*>(p);
    *exec_done_ = 0;
    CW_TRY(cudaHostAlloc(&p, 64, cudaHostAllocMapped));
    sync_slot_ = static_cast<volatile uint64_t*>(p);
    sync_slot_[0] = sync_slot_[1] = 0;
  }
  CW_TRY(cudaHostAlloc(&load_recs_, sizeof(LoadRecord) * kRing, cudaHostAllocMapped));
  CW_TRY(cudaHostAlloc(&in_recs_, sizeof(StampRecord) * kRing, cudaHostAllocMapped));
  memset((void*)ring_, 0, sizeof(ActionDesc) * kRing);
  memset((void*)exec_recs_, 0, sizeof(ExecRecord) * kRing);
  memset((void*)load_recs_, 0, sizeof(LoadRecord) * kRing);
  memset((void*)in_recs_, 0, sizeof(StampRecord) * kRing);
  CW_TRY(cudaHostAlloc(&out_host_, (size_t)kRing * kMaxBatch * out_bytes_max_, cudaHostAllocDefault));
  CW_TRY(cudaHostAlloc(&hdr_stage_, (size_t)16 * kHeaderBytes, cudaHostAllocDefault));
  exec_events_.resize(kRing);
  in_events_.resize(kRing);
  for (auto& e : exec_events_) CW_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : in_events_) CW_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  (void)input_pool;
  return calibrate_clock();
}

std::string Runtime::set_input_pool(int arch, const float* data, int n, int64_t bytes) {
  CW_TRY(cudaSetDevice(device_));
  auto it = archs_.find(arch);
  if (it == archs_.end()) return "unknown arch";
  Arch& a = it->second;
  if (bytes != (int64_t)a.in_c * a.in_h * a.in_w * 4) return "input pool image size != arch input";
  if (a.in_pool) CW_TRY(cudaFreeHost(a.in_pool));
  a.in_pool = nullptr;
  if (bytes > in_bytes_max_) return "input image larger than IOCache slot";
  CW_TRY(cudaHostAlloc(&a.in_pool, (size_t)n * bytes, cudaHostAllocDefault));
  memcpy(a.in_pool, data, (size_t)n * bytes);
  a.in_pool_n = n;
  a.in_pool_bytes = bytes;
  return "";
}

std::string Runtime::calibrate_clock() {
  int64_t off = 0;
  std::string err = measure_clock_offset(&off);
  if (err.empty()) gt_offset_ = off;
  return err;
}

bool Runtime::resync_clock(int64_t* step) {
  *step = 0;
  if (cudaSetDevice(device_) != cudaSuccess) return false;
  int64_t best_rtt = INT64_MAX, best = 0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    const uint64_t tag = ++sync_tag_;
    const int64_t t0 = realtime_ns();
    launch_stamp(sync_slot_, tag, s_cap_);
    int64_t t1 = realtime_ns();
    while (sync_slot_[1] != tag && t1 - t0 < 2000000) t1 = realtime_ns();
    if (sync_slot_[1] != tag) {
      cudaStreamSynchronize(s_cap_);  // an SM was busy: give up for now
      return false;
    }
    // the stamp is written ~1.5 us (one PCIe posted write + the host poll) before t1
    if (t1 - t0 < best_rtt) {
      best_rtt = t1 - t0;
      best = (int64_t)sync_slot_[0] - (t1 - 1500);
    }
  }
  if (best_rtt > 40000) return false;
  *step = best - gt_offset_;
  gt_offset_ = best;
  return true;
}

std::string Runtime::measure_clock_offset(int64_t* offset) {
  CW_TRY(cudaSetDevice(device_));
  uint64_t* slot = nullptr;
  CW_TRY(cudaHostAlloc(&slot, 64, cudaHostAllocMapped));
  volatile uint64_t* vs = slot;
  vs[0] = 0;
  vs[1] = 0;
  launch_clock_pub(vs, 20ull * 1000 * 1000, s_cap_);
  CW_TRY(cudaGetLastError());
  const int64_t deadline = realtime_ns() + 2000000000LL;
  while (vs[0] == 0 && realtime_ns() < deadline) {
  }
  std::vector<int64_t> est;
  for (int i = 0; i < 2000 && vs[1] == 0; ++i) {
    const int64_t t0 = realtime_ns();
    const uint64_t g = vs[0];
    const int64_t t1 = realtime_ns();
    if (t1 - t0 < 2000) est.push_back((int64_t)g - (t0 + t1) / 2 + 300);
  }
  CW_TRY(cudaStreamSynchronize(s_cap_));
  if (est.empty()) {
    // The publisher did not run concurrently with this thread (e.g. kernels serialised under
    // a profiler): a coarse offset from one stamp (error ~ the synchronise latency).
    vs[2] = 0;
    launch_stamp(vs + 2, 1, s_cap_);
    CW_TRY(cudaStreamSynchronize(s_cap_));
    if (vs[2] != 0) est.push_back((int64_t)vs[2] - realtime_ns());
  }
  cudaFreeHost(slot);
  if (est.empty()) return "clock calibration failed";
  std::nth_element(est.begin(), est.begin() + est.size() / 2, est.end());
  *offset = est[est.size() / 2];
  return "";
}

const Arch* Runtime::arch(int id) const {
  auto it = archs_.find(id);
  return it == archs_.end() ? nullptr : &it->second;
}

int Runtime::blob_pages(int blob) const {
  auto it = blobs_.find(blob);
  return it == blobs_.end() ? -1 : it->second.npages;
}
int Runtime::arch_of_blob(int blob) const {
  auto it = blobs_.find(blob);
  return it == blobs_.end() ? -1 : it->second.arch;
}

std::string Runtime::register_arch(int id, const CwOp* ops, int n_ops, int n_layers, int in_c,
                                   int in_h, int in_w, int classes, const int* batches,
                                   int n_batches) {
  if (plans_built_) return "register_arch after build_plans";
  if (n_layers > kMaxLayers) return "too many layers";
  Arch a;
  a.id = id;
  a.ops.assign(ops, ops + n_ops);
  a.n_layers = n_layers;
  a.in_c = in_c;
  a.in_h = in_h;
  a.in_w = in_w;
  a.classes = classes;
  if ((int64_t)in_c * in_h * in_w * 4 > in_bytes_max_) return "input larger than IOCache slot";
  if ((int64_t)classes * 4 > out_bytes_max_) return "output larger than IOCache slot";
  int max_b = 1;
  for (int i = 0; i < n_batches; ++i) {
    if (batches[i] < 1 || batches[i] > kMaxBatch) return "batch size out of range";
    max_b = std::max(max_b, batches[i]);
    a.plans[batches[i]].batch = batches[i];
  }
  // Workspace buffer sizes at the largest batch (a concat buffer is sized by its channel
  // stride, whichever op writes or reads it).
  auto grow = [&](int buf, size_t bytes) {
    if (buf < 0) return;
    if ((size_t)buf >= a.buf_bytes.size()) a.buf_bytes.resize(buf + 1, 0);
    a.buf_bytes[buf] = std::max(a.buf_bytes[buf], bytes);
  };
  for (CwOp& op : a.ops) {
    if (op.in_ctot <= 0) op.in_ctot = op.cin;
    if (op.out_ctot <= 0) op.out_ctot = op.cout;
    if (op.pad_w < 0) op.pad_w = op.pad;
    if (op.kind == OP_CONV && op.cout_pad <= 0) op.cout_pad = (op.cout + 63) / 64 * 64;
    if (op.kind == OP_CONV || op.kind == OP_MAXPOOL || op.kind == OP_AVGPOOL ||
        op.kind == OP_BNPOOL)
      grow(op.in_buf, (size_t)max_b * op.in_h * op.in_w * op.in_ctot * 2);
    if (op.kind == OP_FC) grow(op.in_buf, (size_t)max_b * op.cin * 4);
    if (op.out_buf < 0) continue;
    size_t bytes = 0;
    switch (op.kind) {
      case OP_STEM:  // NHWC4 rows with kMkPadW zero pixels on both sides, kMkPadH zero rows
        bytes = (size_t)max_b * (op.in_h + 2 * kMkPadH) * (op.in_w + 2 * kMkPadW) * 4 * 2;
        break;
      case OP_IM2COL: bytes = (size_t)max_b * op.out_h * op.out_w * 64 * 2; break;
      case OP_CONV:
      case OP_MAXPOOL:
      case OP_BNPOOL: bytes = (size_t)max_b * op.out_h * op.out_w * op.out_ctot * 2; break;
      case OP_AVGPOOL: bytes = (size_t)max_b * op.cin * 4; break;
      default: break;
    }
    grow(op.out_buf, bytes);
    if (op.kind == OP_CONV)
      a.flops_per_image += 2.0 * op.out_h * op.out_w * op.cout * (double)op.kpad;
    if (op.kind == OP_CONV && (op.cout_pad % 64 != 0 || (op.kpad % 64 != 0 && op.kpad != 224)))
      return "conv shape not 64-aligned";
    if ((op.kind == OP_CONV || op.kind == OP_MAXPOOL) &&
        (op.out_ctot % 8 || op.out_coff % 8 || op.in_ctot % 8 != 0) && op.kpad != 224)
      return "channel strides / offsets must be multiples of 8 (16-byte TMA alignment)";
  }
  archs_[id] = std::move(a);
  return "";
}

std::string Runtime::register_blob(int id, int arch, const void* data, size_t bytes,
                                   const CwTensorLoc* locs, int n_locs) {
  CW_TRY(cudaSetDevice(device_));
  Blob b;
  b.id = id;
  b.arch = arch;
  b.bytes = bytes;
  b.npages = (int)((bytes + page_bytes_ - 1) / page_bytes_);
  b.locs.assign(locs, locs + n_locs);
  if (n_locs > kMaxLayers) return "more layers than the model header holds";
  for (const auto& l : b.locs) {
    if (l.s_off >= 0 && (l.s_off % 16 || l.s_off < (int64_t)kHeaderBytes ||
                         l.s_off >= (int64_t)bytes))
      return "bad input-BatchNorm offset";
    if (l.rows <= 0) continue;  // a BatchNorm-only entry
    const int64_t wend = l.w_off + (int64_t)l.rows * l.k * 2;
    if (l.w_off / page_bytes_ != (wend - 1) / page_bytes_) return "weight tensor straddles a page";
    if (l.w_off % 256 || l.b_off % 16) return "unaligned tensor offset";
    if (l.w_off < (int64_t)kHeaderBytes || wend > (int64_t)bytes) return "tensor outside blob";
  }
  CW_TRY(cudaHostAlloc(&b.host, bytes, cudaHostAllocDefault));
  memcpy(b.host, data, bytes);
  blobs_[id] = std::move(b);
  return "";
}

// ---------------------------------------------------------------- planning

static void box_dims(int nimg, int oh, int ow, int* bw, int* bh, int* bn) {
  int w = std::min(ow, 128);
  int h = std::max(1, std::min(oh, 128 / w));
  h = (oh + (oh + h - 1) / h - 1) / ((oh + h - 1) / h);  // balance rows across tiles
  int n = std::max(1, std::min(nimg, 128 / (w * h)));
  n = (nimg + (nimg + n - 1) / n - 1) / ((nimg + n - 1) / n);
  *bw = w;
  *bh = h;
  *bn = n;
}

// Mode-1 tiles (any box shape works there): when the box_dims shape leaves more than 30 % of
// the 128 accumulator rows idle (a wide row split 128 + remainder: Inception-v3's 147 / 73 /
// 71-wide stages keep 57 % busy), the w x h x n box that covers the output with the fewest
// idle rows (ties: the wider box): 21 x 6 at 147 wide and batch 1 (96 %), 4 x 2 x 16 images
// at batch 16 (99 %). Inception-v3 b=16 1356 -> 1207 us, logits unchanged to the bit.
// ResNet's 56 / 28 / 14 / 7 maps (>= 77 % busy) keep box_dims: denser (narrow) boxes there
// measured 2-7 us slower.
static void box_dims_dense(int nimg, int oh, int ow, int* bw, int* bh, int* bn) {
  box_dims(nimg, oh, ow, bw, bh, bn);
  auto util = [&](int w, int h, int n) {
    const double tiles = (double)((ow + w - 1) / w) * ((oh + h - 1) / h) * ((nimg + n - 1) / n);
    return (double)ow * oh * nimg / (tiles * 128.0);
  };
  const double base = util(*bw, *bh, *bn);
  static const double thresh = exp_env("CW_DENSE_BELOW") ? atof(exp_env("CW_DENSE_BELOW")) : 0.7;
  if (base >= thresh) return;
  double best = -1.0;
  int bw2 = *bw, bh2 = *bh, bn2 = *bn;
  for (int w = 1; w <= std::min(ow, 128); ++w)
    for (int h = 1; h <= std::min(oh, 128 / w); ++h) {
      int n = std::max(1, std::min(nimg, 128 / (w * h)));
      n = (nimg + (nimg + n - 1) / n - 1) / ((nimg + n - 1) / n);
      const double u = util(w, h, n);
      if (u > best + 1e-9 || (u > best - 1e-9 && w > bw2)) {  // (ties: the wider box)
        best = u;
        bw2 = w;
        bh2 = h;
        bn2 = n;
      }
    }
  if (best >= base + 0.02) {
    *bw = bw2;
    *bh = bh2;
    *bn = bn2;
  }
}

// Tile width and split-K choice for one conv at one batch size, for G SMs, from
// a cost model with constants measured on B200 (tools/mma_probe.cu,
// tools/tma_probe.cu, tools/epi_probe.cu):
//   * a 64-deep k-block of tcgen05.mma (4 x K=16) costs ~0.27 us at ANY N <= 256
//     (per-instruction cost), so FLOP efficiency grows with the N tile;
//   * the single producer thread spends ~0.08 us per TMA it issues;
//   * TMA feeds one SM at ~140 GB/s;
//   * the 4-warp epilogue drains ~20 GB/s per SM (bf16 tile rows, ~3 TB/s chip)
//     plus ~0.8 us of fixed latency per tile (bias / residual loads, barriers);
//   * a split-K reduce layer costs ~3 us plus its partial-tile traffic.
// Epilogue of task i overlaps the MMAs of task i+1 (two TMEM accumulators).
// Cluster plans (csize > 1): a split conv uses exactly csize splits, one per CTA of a
// cluster, reduced through distributed shared memory in the epilogue (~2.5 us, no reduce layer,
// no partials in global memory); bn = 64 (received partials + the staged own tile = 64 KB).
static void plan_conv(MkLayer& d, int cout, int G, bool allow_split, bool grouped, int csize) {
  // a split layer adds a reduce layer and one more whole-GPU dependency (~6 us in the
  // network, measured with tools/sweep_bn.sh + op_profile; CW_SPLIT_US overrides)
  static const double split_us = exp_env("CW_SPLIT_US") ? atof(exp_env("CW_SPLIT_US")) : 6.0;
  static const double csplit_us = exp_env("CW_CSPLIT_US") ? atof(exp_env("CW_CSPLIT_US")) : 2.5;
  const int units = d.num_kb / (d.mode == 3 ? 3 : 1);
  static const int kBn[3] = {256, 128, 64};
  const double rows = d.mode == 0 ? 128.0 : (double)(d.box_w * d.box_h * d.box_n);
  const double a_bytes = rows * d.kblk * 2;
  double best = 1e30;
  int best_bn = 64, best_s = 1;
  for (int i = 0; i < 3; ++i) {
    const int bn = kBn[i];
    if (cout % bn) continue;
    if ((d.mode == 2 || grouped) && bn != 64) continue;  // grouped: one 64-channel block per tile
    const int tiles = d.m_tiles * (cout / bn);
    const int n_tma = 1 + ((bn == std::min(256, cout) && d.kblk == 64) ? 1 : bn / 64);
    // (an input-BatchNorm layer: warps 2-3 rewrite every A k-block in shared memory before
    // its MMAs, ~1.25 us per k-block measured on DenseNet-121's 1x1 convs)
    static const double pre_us = exp_env("CW_PRE_KB_US") ? atof(exp_env("CW_PRE_KB_US")) : 1.25;
    const double t_kb = std::max({d.pre_layer >= 0 ? pre_us : 0.30, 0.08 * n_tma + 0.1,
                                  (a_bytes + bn * d.kblk * 2.0) / 140e3});
    for (int s = 1; s <= 32; ++s) {
      int per;
      if (csize > 1) {
        // cluster plans: no split, or exactly csize non-empty splits
        // (one wave at most: the ranks of a cluster wait for each other at every task)
        if (s > 1 && (s != csize || !allow_split || bn != 64 || units < s || d.num_kb / s < 1 ||
                      tiles * s > G))
          continue;
        per = (units + s - 1) / s * (d.mode == 3 ? 3 : 1);
      } else {
        if (s > 1 && (!allow_split || d.num_kb / s < 2)) break;
        per = (d.num_kb + s - 1) / s;
        if (d.mode == 3) per = (per + 2) / 3 * 3;  // whole (kernel row, channel block) groups
        const int splits = (d.num_kb + per - 1) / per;
        if (splits != s) continue;
      }
      const int tasks = tiles * s;
      const int waves = (tasks + G - 1) / G;
      const double t_main = per * t_kb;
      const double t_epi = rows * bn * (s > 1 ? 4.0 : 2.0) / 20e3 + 0.8;  // + per-task fixed cost
      double t = waves * std::max(t_main, t_epi) + std::min(t_main, t_epi) + 1.5;
      if (s > 1 && csize > 1) t += csplit_us;
      else if (s > 1) t += split_us + (double)tiles * 128 * bn * (4.0 * s + 2.0) / (G * 40e3);
      if (t < best - 1e-9) {
        best = t;
        best_bn = bn;
        best_s = s;
      }
    }
  }
  // experiment overrides (profiling only): CW_BN_CAP, CW_FORCE_BN, CW_FORCE_SPLIT
  if (const char* e = exp_env("CW_BN_CAP")) {
    const int cap = atoi(e);
    if (cap >= 64 && best_bn > cap && cout % cap == 0 && best_s == 1) best_bn = cap;
  }
  if (const char* e = exp_env("CW_FORCE_BN")) {
    const int bn = atoi(e);
    if (bn > 0 && cout % bn == 0 && ((d.mode != 2 && !grouped) || bn == 64)) best_bn = bn;
  }
  if (const char* e = exp_env("CW_FORCE_SPLIT")) {
    const int sp = atoi(e);
    if (sp > 0 && allow_split && d.num_kb / sp >= 1 && (csize <= 1 || sp == 1 || sp == csize))
      best_s = sp;
  }
  d.csplit = csize > 1 && best_s > 1;
  d.bn = best_bn;
  d.n_tiles = cout / best_bn;
  d.splits = best_s;
  d.kb_per_split = (d.num_kb + best_s - 1) / best_s;
  if (d.mode == 3) d.kb_per_split = (d.kb_per_split + 2) / 3 * 3;
  d.tasks = d.m_tiles * d.n_tiles * best_s;
}

namespace {
// One buffer access of a layer: channels [c0, c1) of workspace buffer `buf` (concats are
// disjoint channel slices of one buffer: their writers do not order each other).
struct Access {
  int buf;
  int c0 = 0, c1 = 1 << 30;
};

// Buffer / channel-range hazard tracking -> per-layer dependency lists (RAW, WAR, WAW),
// transitively reduced.
struct DepTracker {
  struct Use {
    int layer, c0, c1;
  };
  std::map<int, std::vector<Use>> writers, readers;
  std::vector<std::vector<char>> reach;  // reach[L][p]: L (transitively) waits for p

  static bool overlap(const Use& u, const Access& a) { return u.c0 < a.c1 && a.c0 < u.c1; }

  std::string add(MkLayer& d, int L, const std::vector<Access>& reads,
                  const std::vector<Access>& writes) {
    std::vector<int> deps;
    for (const Access& a : reads)
      for (const Use& w : writers[a.buf])
        if (overlap(w, a)) deps.push_back(w.layer);
    for (const Access& a : writes) {
      for (const Use& w : writers[a.buf])
        if (overlap(w, a)) deps.push_back(w.layer);
      for (const Use& r : readers[a.buf])
        if (overlap(r, a)) deps.push_back(r.layer);
    }
    std::sort(deps.begin(), deps.end());
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    deps.erase(std::remove(deps.begin(), deps.end(), L), deps.end());
    reach.emplace_back(L + 1, 0);
    std::vector<int> kept;
    for (int p : deps) {
      bool implied = false;
      for (int o : deps)
        if (o > p && reach[o][p]) implied = true;
      if (!implied) kept.push_back(p);
    }
    for (int p : deps) {
      reach[L][p] = 1;
      for (int x = 0; x < p; ++x)
        if (reach[p][x]) reach[L][x] = 1;
    }
    if ((int)kept.size() > kMkMaxDeps) return "too many layer dependencies";
    d.ndeps = (int)kept.size();
    for (size_t i = 0; i < kept.size(); ++i) d.deps[i] = kept[i];
    for (const Access& a : reads) readers[a.buf].push_back({L, a.c0, a.c1});
    for (const Access& a : writes) {
      // uses inside the new write's range are ordered before it: later accesses that
      // overlap them overlap it too, and wait for it (transitively for them)
      auto covered = [&](const Use& u) { return u.c0 >= a.c0 && u.c1 <= a.c1; };
      auto& ws = writers[a.buf];
      ws.erase(std::remove_if(ws.begin(), ws.end(), covered), ws.end());
      auto& rs = readers[a.buf];
      rs.erase(std::remove_if(rs.begin(), rs.end(), covered), rs.end());
      ws.push_back({L, a.c0, a.c1});
    }
    return "";
  }
};
constexpr int kBufPartial = 1000;  // pseudo-buffer: the split-K partial workspace
constexpr int kBufLogits = 1001;   // pseudo-buffer: the request output slots (FC -> softmax)
}  // namespace

std::string Runtime::build_plan(Arch& a, int batch, bool allow_split) {
  Plan& p = a.plans[batch];
  p.batch = batch;
  p.layers.clear();
  p.layer_op.clear();
  p.tmaps.clear();
  // Cluster split-K (csize > 1) for small batches, whose layers have far fewer output tiles
  // than SMs: the persistent grid then holds as many whole clusters as the GPU co-schedules
  // (B200: 120 CTAs in clusters of 8, 132 in clusters of 4, all 148 in pairs). Measured
  // (ResNet-50 Exec p50 without -> with, tools/ab_quick.py): b=1 275 -> 248 us (8), b=2 305 ->
  // 279 (4), b=4 346 -> 309 (4), b=8 422 -> 400 (2), b=16 551 -> 524 (2).
  // Nets with input-BatchNorm layers (DenseNet: long-K 1x1 bottlenecks whose k-blocks cost
  // ~4x an MMA's) gain from one size larger: DenseNet-121 b=4 777 -> 744 us, b=8 951 -> 843;
  // DenseNet-169 b=2 1093 -> 1029, b=4 1139 -> 1057, b=8 1451 -> 1209.
  bool has_pre_bn = false;
  for (const CwOp& op : a.ops) has_pre_bn |= (op.flags & OPF_PRE_BN) != 0;
  int csize = has_pre_bn ? (batch <= 4 ? 8 : batch <= 8 ? 4 : 2)
                         : (batch == 1 ? 8 : batch <= 4 ? 4 : 2);
  if (const char* e = exp_env("CW_CSIZE")) csize = atoi(e);
  if (csize != 1 && csize != 2 && csize != 4 && csize != 8) return "cluster size must be 1, 2, 4 or 8";
  int G = num_sms_;
  if (csize > 1) {
    const uint32_t fixed0 = mk_smem_bytes(0, 0);
    const int ctas = mk_cluster_ctas(csize, mk_smem_bytes((kMkSmemCap - fixed0) / 1024 * 1024, 0));
    if (ctas >= 2 * csize) G = std::min(ctas, num_sms_) / csize * csize;
    else csize = 1;
  }
  p.csize = csize;
  DepTracker deps;
  size_t partial_need = 0;
  int rot = 0;
  std::map<int, int> producer_kind;  // buffer -> op kind that last wrote it
  bool fc_seen = false;
  auto push = [&](MkLayer& d, int oi, const std::vector<Access>& rd,
                  const std::vector<Access>& wr) -> std::string {
    const int L = (int)p.layers.size();
    if (L >= kMkMaxPlanLayers) return "plan has too many layers";
    std::string err = deps.add(d, L, rd, wr);
    if (!err.empty()) return err;
    if (d.csplit) rot = (rot + csize - 1) / csize * csize % G;  // split z on cluster rank z
    d.rot = rot;
    rot = (rot + d.tasks) % G;
    p.layers.push_back(d);
    p.layer_op.push_back(oi);
    return "";
  };
  // A bottleneck's projection shortcut (1x1 / stride s conv, no ReLU, no residual) whose output
  // is read only as the residual of the NEXT op, a 1x1 / stride 1 conv of the same output shape,
  // runs inside that conv as a second K segment: one layer, no shortcut tensor in memory, no
  // residual read, one rounding (the kernel sequence is ours to choose).
  auto fusable_shortcut = [&](size_t i) -> bool {
    if (i + 1 >= a.ops.size()) return false;
    const CwOp& s = a.ops[i];
    const CwOp& c = a.ops[i + 1];
    if (s.kind != OP_CONV || c.kind != OP_CONV) return false;
    if (s.relu || s.res_buf >= 0 || s.flags || c.flags || s.kh != 1 || s.kw != 1 || s.pad ||
        s.pad_w || (s.stride != 1 && s.stride != 2))
      return false;
    if (c.kh != 1 || c.kw != 1 || c.stride != 1 || c.pad || c.pad_w || c.res_buf != s.out_buf)
      return false;
    if (c.cout != s.cout || c.cout_pad != s.cout_pad || c.out_h != s.out_h || c.out_w != s.out_w ||
        s.out_ctot != s.cout || s.out_coff || c.out_ctot != c.cout || c.out_coff)
      return false;
    if (s.kpad % 64 || c.kpad % 64 || s.cin % 64 || c.cin % 64) return false;
    if (c.in_buf == s.out_buf) return false;
    // small batches: a deep shortcut (stages 3-4: 8-16 k-blocks) ran on SMs the 3x3 conv before
    // it leaves idle; serialised into conv3 it costs more than the layer it saves (ResNet-50
    // b=1: stage 1 -2.4 us, stage 2 -1.8, stage 3 +2.0, stage 4 +4.3; b=16: -8.5 .. -0.5)
    if (batch < 8 && s.kpad / 64 > 4) return false;
    // the shortcut tensor must be dead after the conv: no later read before a rewrite
    for (size_t j = i + 2; j < a.ops.size(); ++j) {
      const CwOp& o = a.ops[j];
      if (o.in_buf == s.out_buf || o.res_buf == s.out_buf) return false;
      if (o.out_buf == s.out_buf) break;
    }
    return true;
  };
  const bool fuse_shortcuts = exp_env("CW_NO_FUSE_SC") == nullptr;  // (experiments: A/B)
  int shortcut = -1;  // op index of the shortcut fused into the next conv
  for (size_t oi = 0; oi < a.ops.size(); ++oi) {
    const CwOp& op = a.ops[oi];
    if (fc_seen && op.kind != OP_SOFTMAX) return "the FC op must be the last op (or a softmax)";
    if (fuse_shortcuts && fusable_shortcut(oi)) {
      shortcut = (int)oi;
      continue;
    }
    const CwOp* sc = (shortcut >= 0 && (size_t)shortcut + 1 == oi) ? &a.ops[shortcut] : nullptr;
    MkLayer d;
    memset(&d, 0, sizeof(d));
    d.pre_layer = -1;
    d.batch = batch;
    void* in = op.in_buf >= 0 ? a.bufs[op.in_buf] : nullptr;
    void* out = op.out_buf >= 0 ? a.bufs[op.out_buf] : nullptr;
    std::string err;
    switch (op.kind) {
      case OP_STEM: {
        d.kind = MK_INPUT;
        d.tasks = G;
        d.H = op.in_h;
        d.W = op.in_w;
        d.out = out;
        if (op.in_w % 4) return "input width must be a multiple of 4";
        err = push(d, (int)oi, {}, {Access{op.out_buf}});
        break;
      }
      case OP_CONV: {
        const int cout_p = op.cout_pad;
        if (cout_p > kMkMaxCout) return "conv Cout exceeds kMkMaxCout (shared-memory bias)";
        const bool grouped = op.flags & OPF_GROUPED64;
        const bool pre_bn = op.flags & OPF_PRE_BN;
        d.kind = MK_CONV;
        d.wlayer = op.layer;
        d.n_out = cout_p;
        d.n_valid = op.cout;
        d.relu = op.relu;
        d.nimg = batch;
        d.oh = op.out_h;
        d.ow = op.out_w;
        d.kw = op.kw;
        d.stride = op.stride;
        d.pad = op.pad;
        d.pad_w = op.pad_w;
        d.grouped = grouped;
        d.pre_layer = pre_bn ? op.pre_layer : -1;
        d.out_ctot = op.out_ctot;
        d.out_coff = op.out_coff;
        d.res = (op.res_buf >= 0 && !sc) ? a.bufs[op.res_buf] : nullptr;
        if (d.res && (op.out_ctot != op.cout || op.out_coff)) return "residual into a concat slice";
        // the layer's channel slice of its output buffer: every store of the layer (TMA maps,
        // split-K reduce rows) addresses it from here with the buffer's channel stride
        void* out_slice = out ? static_cast<uint8_t*>(out) + (size_t)op.out_coff * 2 : nullptr;
        d.out = out_slice;
        const CwOp* nxt = oi + 1 < a.ops.size() ? &a.ops[oi + 1] : nullptr;
        const bool from_stem = producer_kind.count(op.in_buf) && producer_kind[op.in_buf] == OP_STEM;
        bool fuse_pool = nxt && nxt->kind == OP_AVGPOOL && nxt->in_buf == op.out_buf &&
                         op.out_h * op.out_w <= 128 && !from_stem && !(nxt->flags & OPF_PRE_BN) &&
                         op.out_ctot == op.cout && op.out_coff == 0 && op.cout == cout_p;
        if (pre_bn && (op.kh != 1 || op.kw != 1 || op.stride != 1 || op.pad || op.pad_w))
          return "an input BatchNorm prologue needs a 1x1/s1 conv";
        if (grouped && op.cin != op.cout) return "grouped conv with cin != cout";
        CUtensorMap tm;
        if (from_stem) {
          // 7x7 / stride 2 stem over the NHWC4 rows: k-block = kernel row (32 = 8 px x 4 ch)
          if (op.kh != 7 || op.kw != 7 || op.stride != 2 || op.pad != 3 || op.kpad != 224)
            return "unsupported stem geometry";
          d.mode = 2;
          d.kblk = 32;
          d.num_kb = 7;
          const bool fuse_max = nxt && nxt->kind == OP_MAXPOOL && nxt->in_buf == op.out_buf;
          if (!fuse_max || nxt->out_h * 2 != op.out_h || nxt->pad != 1 || nxt->stride != 2)
            return "the stem conv must be followed by a 3x3/s2/p1 max pool";
          if (cout_p != 64 || op.cout != 64) return "the stem conv must have 64 channels";
          // one task per pooled row: conv rows 2ph-1 .. 2ph+1 over the full width (one
          // accumulator of op.out_w <= 128 rows each), A = the kMkStemRows padded input rows
          // they read, staged whole (weights resident in the staging buffers)
          if (op.out_w > 128 || nxt->out_w > 256) return "stem wider than 128 conv columns";
          d.pool_pw = nxt->out_w;
          d.OH = nxt->out_h;
          d.OW = nxt->out_w;
          d.box_w = op.out_w;
          d.box_h = 3;
          d.box_n = 1;
          d.tiles_w = 1;
          d.tiles_h = d.OH;
          d.m_tiles = d.tiles_h * batch;
          d.out = static_cast<uint8_t*>(a.bufs[nxt->out_buf]) + (size_t)nxt->out_coff * 2;
          d.out_ctot = nxt->out_ctot;
          const int wp = op.in_w + 2 * kMkPadW;
          d.sub_bytes = wp * 8;  // staged row pitch
          if (2 * (op.out_w - 1) + 8 > wp) return "stem rows too narrow for the windows";
          if (!make_tmap_stem_rows(&tm, in, batch, op.in_h + 2 * kMkPadH, wp, kMkStemRows))
            return "tensor map (stem) failed";
        } else if (!fuse_pool && op.kh == 1 && op.kw == 1 && op.stride == 1 && op.pad == 0 &&
                   op.pad_w == 0 && !(sc && sc->stride != 1)) {
          // 1x1: A = the [M][cin] matrix of the input buffer (row stride in_ctot; channels
          // >= cin are out of bounds: zero-filled)
          d.mode = 0;
          d.kblk = 64;
          d.num_kb = op.kpad / 64;
          d.m_total = batch * op.out_h * op.out_w;
          d.m_tiles = (d.m_total + 127) / 128;
          if (!make_tmap_2d(&tm, in, (uint64_t)op.cin, (uint64_t)d.m_total, 128,
                            (uint64_t)op.in_ctot))
            return "tensor map (2d) failed";
        } else if (!fuse_pool && !pre_bn && op.kh == 3 && op.kw == 3 && op.stride == 1 &&
                   op.pad == 1 && op.pad_w == 1 && op.out_w + 2 <= 128 &&
                   exp_env("CW_NO_MODE3") == nullptr) {
          // 3x3 / stride 1: tiles of full rows widened by the 2 padding columns, so the three
          // horizontal taps of a kernel row are ONE TMA box read at row shifts 0, 1, 2 (the
          // two extra columns per row are junk outputs, clipped by the store map)
          d.mode = 3;
          d.kblk = 64;
          d.num_kb = op.kpad / 64;
          d.cin_kb = grouped ? 1 : (op.cin + 63) / 64;
          if (d.num_kb != 9 * d.cin_kb) return "mode-3 conv K layout";
          box_dims(batch, op.out_h, op.out_w + 2, &d.box_w, &d.box_h, &d.box_n);
          d.tiles_w = 1;
          d.tiles_h = (op.out_h + d.box_h - 1) / d.box_h;
          d.m_tiles = d.tiles_h * ((batch + d.box_n - 1) / d.box_n);
          if (!make_tmap_nhwc(&tm, in, batch, op.in_h, op.in_w, op.cin, d.box_w, d.box_h,
                              d.box_n, 1, op.in_ctot))
            return "tensor map (nhwc, mode 3) failed";
        } else {
          if (pre_bn) return "input BatchNorm prologue on a tap-shifted conv";
          d.mode = 1;
          d.kblk = 64;
          d.num_kb = op.kpad / 64;
          d.cin_kb = grouped ? 1 : (op.cin + 63) / 64;
          if (d.num_kb != op.kh * op.kw * d.cin_kb) return "mode-1 conv K layout";
          if (fuse_pool) {
            d.box_w = op.out_w;
            d.box_h = op.out_h;
            d.box_n = std::max(1, std::min(batch, 128 / (op.out_w * op.out_h)));
          } else if (exp_env("CW_NO_DENSE_BOX") == nullptr) {
            box_dims_dense(batch, op.out_h, op.out_w, &d.box_w, &d.box_h, &d.box_n);
          } else {
            box_dims(batch, op.out_h, op.out_w, &d.box_w, &d.box_h, &d.box_n);
          }
          d.tiles_w = (op.out_w + d.box_w - 1) / d.box_w;
          d.tiles_h = (op.out_h + d.box_h - 1) / d.box_h;
          d.m_tiles = d.tiles_w * d.tiles_h * ((batch + d.box_n - 1) / d.box_n);
          if (!make_tmap_nhwc(&tm, in, batch, op.in_h, op.in_w, op.cin, d.box_w, d.box_h, d.box_n,
                              op.stride, op.in_ctot))
            return "tensor map (nhwc) failed";
        }
        CUtensorMap tm2;
        if (sc) {
          // the shortcut's K segment: its input through a map with the SAME row tiling (mode 0:
          // [M][cin] rows of the block input; mode 1: the box over the strided input pixels)
          void* sin = a.bufs[sc->in_buf];
          const bool ok = d.mode == 0
                              ? make_tmap_2d(&tm2, sin, (uint64_t)sc->cin, (uint64_t)d.m_total, 128,
                                             (uint64_t)sc->in_ctot)
                              : make_tmap_nhwc(&tm2, sin, batch, sc->in_h, sc->in_w, sc->cin,
                                               d.box_w, d.box_h, d.box_n, sc->stride, sc->in_ctot);
          if (!ok) return "tensor map (fused shortcut) failed";
          if (d.mode != 0 && d.mode != 1) return "fused shortcut on an unsupported conv mode";
          d.f_kb = sc->kpad / 64;
          d.f_wlayer = sc->layer;
          d.f_stride = sc->stride;
          d.num_kb += d.f_kb;
        }
        // (the fused pool runs in the epilogue of whole-image tiles: no split-K there; nor in a
        // layer with a fused shortcut, whose bias is the sum of two layers')
        plan_conv(d, cout_p, G, allow_split && !fuse_pool && !d.pool_pw && !sc, grouped, csize);
        d.tmap = (int)p.tmaps.size();
        p.tmaps.push_back(tm);
        if (sc) {
          d.f_tmap = (int)p.tmaps.size();
          p.tmaps.push_back(tm2);
        }
        d.tmap_out = d.tmap_res = -1;
        if (d.pool_pw) {  // stem: pooled output tiles of pool_pw pixels
          CUtensorMap mo;
          if (!make_tmap_nhwc(&mo, d.out, batch, d.OH, d.OW, op.cout, d.pool_pw, 1, 1, 1,
                              d.out_ctot))
            return "tensor map (stem output) failed";
          d.tmap_out = (int)p.tmaps.size();
          p.tmaps.push_back(mo);
        } else if (!fuse_pool && d.splits == 1) {
          // TMA-store epilogue: 64-column boxes over the output (and residual) tiles; the
          // map ends at the layer's real channels (padded N-tile columns are clipped)
          auto out_map = [&](CUtensorMap* m, const void* base, int ctot) {
            return d.mode == 0 ? make_tmap_2d(m, base, (uint64_t)op.cout, (uint64_t)d.m_total, 128,
                                              (uint64_t)ctot)
                               : make_tmap_nhwc(m, base, batch, op.out_h, op.out_w, op.cout,
                                                d.box_w, d.box_h, d.box_n, 1, ctot);
          };
          CUtensorMap mo;
          if (!out_map(&mo, out_slice, op.out_ctot)) return "tensor map (output) failed";
          d.tmap_out = (int)p.tmaps.size();
          p.tmaps.push_back(mo);
          if (d.res) {
            CUtensorMap mr;
            if (!out_map(&mr, d.res, op.cout)) return "tensor map (residual) failed";
            d.tmap_res = (int)p.tmaps.size();
            p.tmaps.push_back(mr);
          }
        }
        const Access out_acc{op.out_buf, op.out_coff, op.out_coff + op.cout};
        std::vector<Access> rd = {Access{op.in_buf, 0, op.cin}}, wr;
        if (sc) rd.push_back(Access{sc->in_buf, 0, sc->cin});
        if (d.pool_pw) {
          wr.push_back(Access{nxt->out_buf, nxt->out_coff, nxt->out_coff + nxt->cout});
          ++oi;  // the max pool op is done in this layer's epilogue
        } else if (fuse_pool) {
          d.pool_out = reinterpret_cast<float*>(a.bufs[nxt->out_buf]);
          d.pool_scale = 1.0f / (float)(op.out_h * op.out_w);
          d.out = nullptr;
          wr.push_back(Access{nxt->out_buf});
          ++oi;  // the avgpool op is done in this layer's epilogue
        } else if (d.splits == 1 || d.csplit) {
          wr.push_back(out_acc);
        }
        if (d.splits > 1 && !d.csplit) {
          wr.push_back(Access{kBufPartial});
          const size_t tiles = (size_t)d.m_tiles * d.n_tiles;
          partial_need = std::max(partial_need, tiles * d.splits * 128 * d.bn * 4);
          MkLayer r = d;
          d.out = nullptr;
          d.res = nullptr;
          err = push(d, (int)oi, rd, wr);
          if (!err.empty()) return err;
          // the reduce: one task per (tile, row group), ~G tasks in all
          r.kind = MK_REDUCE;
          const int rows = d.mode == 0 ? 128 : d.box_w * d.box_h * d.box_n;
          int parts = 1;
          while (parts * 2 <= rows && (size_t)tiles * parts * 2 <= (size_t)G) parts *= 2;
          // a task's S partial row blocks are bulk-copied into the 64 KB staging buffers
          while (parts < rows && (size_t)d.splits * ((rows + parts - 1) / parts) * d.bn * 4 >
                                     (size_t)kMkOutBufs * kMkOutBufBytes)
            parts *= 2;
          // and its bf16 output rows are staged in the bias area for the bulk stores
          while (parts < rows && (size_t)((rows + parts - 1) / parts) * d.bn * 2 >
                                     (size_t)kMkMaxCout * 4)
            parts *= 2;
          if ((size_t)d.splits * ((rows + parts - 1) / parts) * d.bn * 4 >
                  (size_t)kMkOutBufs * kMkOutBufBytes ||
              (size_t)((rows + parts - 1) / parts) * d.bn * 2 > (size_t)kMkMaxCout * 4)
            return "split-K reduce rows exceed the staging buffers";
          r.red_rows = (rows + parts - 1) / parts;
          r.red_parts = (rows + r.red_rows - 1) / r.red_rows;
          r.tasks = (int)tiles * r.red_parts;
          std::vector<Access> rrd = {Access{kBufPartial}};
          if (op.res_buf >= 0) rrd.push_back(Access{op.res_buf});
          err = push(r, (int)oi, rrd, {out_acc});
        } else {
          if (op.res_buf >= 0 && !sc) rd.push_back(Access{op.res_buf});
          err = push(d, (int)oi, rd, wr);
        }
        break;
      }
      case OP_MAXPOOL: {
        d.kind = MK_MAXPOOL;
        d.tasks = G;
        d.in = in;
        d.out = static_cast<uint8_t*>(out) + (size_t)op.out_coff * 2;
        d.H = op.in_h;
        d.W = op.in_w;
        d.C = op.cin;
        d.OH = op.out_h;
        d.OW = op.out_w;
        d.kw = op.kh;
        d.stride = op.stride;
        d.pad = op.pad;
        d.in_ctot = op.in_ctot;
        d.out_ctot = op.out_ctot;
        if (op.cin % 8) return "maxpool C must be a multiple of 8";
        if (op.kh != 3 || op.kw != 3) return "max pool window must be 3x3";
        err = push(d, (int)oi, {Access{op.in_buf, 0, op.cin}},
                   {Access{op.out_buf, op.out_coff, op.out_coff + op.cin}});
        break;
      }
      case OP_AVGPOOL: {
        d.kind = MK_AVGPOOL;
        d.tasks = G;
        d.in = in;
        d.out = out;
        d.H = op.in_h;
        d.W = op.in_w;
        d.C = op.cin;
        d.in_ctot = op.in_ctot;
        d.pre_layer = (op.flags & OPF_PRE_BN) ? op.pre_layer : -1;
        if (op.cin % 8 || op.in_ctot % 8) return "avgpool C must be a multiple of 8";
        err = push(d, (int)oi, {Access{op.in_buf, 0, op.cin}}, {Access{op.out_buf}});
        break;
      }
      case OP_BNPOOL: {
        d.kind = MK_BNPOOL;
        d.tasks = G;
        d.in = in;
        d.out = out;
        d.H = op.in_h;
        d.W = op.in_w;
        d.C = op.cin;
        d.OH = op.out_h;
        d.OW = op.out_w;
        d.in_ctot = op.in_ctot;
        d.out_ctot = op.out_ctot;
        d.pre_layer = op.pre_layer;
        if (op.cin % 8 || op.pre_layer < 0) return "BN pool: C % 8 and an input BatchNorm";
        err = push(d, (int)oi, {Access{op.in_buf, 0, op.cin}}, {Access{op.out_buf}});
        break;
      }
      case OP_IM2COL: {
        d.kind = MK_IM2COL;
        d.tasks = G;
        d.out = out;
        d.H = op.in_h;
        d.W = op.in_w;
        d.C = op.cin;
        d.OH = op.out_h;
        d.OW = op.out_w;
        d.kw = op.kw;
        d.stride = op.stride;
        d.pad = op.pad;
        if (op.kh != op.kw || op.kh * op.kw * op.cin > 64) return "im2col patch > 64 values";
        err = push(d, (int)oi, {}, {Access{op.out_buf}});
        break;
      }
      case OP_SOFTMAX: {
        if (!fc_seen) return "softmax must follow the FC op";
        d.kind = MK_SOFTMAX;
        d.tasks = batch;  // one CTA per request
        d.classes = op.cout;
        if (op.cout % 4) return "softmax classes must be a multiple of 4";
        err = push(d, (int)oi, {Access{kBufLogits}}, {Access{kBufLogits}});
        break;
      }
      case OP_FC: {
        d.kind = MK_FC;
        d.tasks = G;
        d.in = in;
        d.wlayer = op.layer;
        d.C = op.cin;
        d.classes = op.cout;
        if (op.cin % 64) return "fc input features must be a multiple of 64";
        if (batch > 16) return "fc batch must be <= 16";
        fc_seen = true;
        err = push(d, (int)oi, {Access{op.in_buf}}, {Access{kBufLogits}});
        break;
      }
      default:
        return "unknown op kind";
    }
    if (!err.empty()) return err;
    if (op.out_buf >= 0) producer_kind[op.out_buf] = op.kind;
  }
  // ---- shared memory: the ring takes what the plan table and scratch leave; each
  // conv layer cuts it into as many slots (A tile + B tile, 1 KB aligned) as fit.
  const int nl = (int)p.layers.size();
  const uint32_t cap = kMkSmemCap;
  const uint32_t fixed = mk_smem_bytes(0, nl);
  if (fixed + 64 * 1024 > cap) return "plan too large for shared memory";
  p.ring_bytes = (cap - fixed) / 1024 * 1024;
  p.smem = mk_smem_bytes(p.ring_bytes, nl);
  int kpack_env = 0, min_slots = 2 * kMkProducers;  // experiment overrides (profiling only)
  if (const char* e = exp_env("CW_KPACK")) kpack_env = atoi(e);
  if (const char* e = exp_env("CW_KPACK_MINSLOTS")) min_slots = atoi(e);
  for (auto& d : p.layers) {
    if (d.kind != MK_CONV) continue;
    if (d.mode == 2) {  // stem: one slot = the task's staged input rows (weights resident);
      // + 256 B: the junk accumulator rows (conv columns >= out_w) read past the last row
      d.kpack = 1;
      d.b_off = 0;
      d.slot_bytes = (int)((kMkStemRows * d.sub_bytes + 256 + 1023) / 1024 * 1024);
      d.slots = std::min<int>(kMkMaxSlots, p.ring_bytes / d.slot_bytes);
      d.slots -= d.slots % kMkProducers;
      if (d.slots < 2) return "ring too small for the stem";
      continue;
    }
    if (d.mode == 3) {  // one slot = the shared A box (+2 rows read by the shifts) + 3 B tiles
      const uint32_t rows = (uint32_t)(d.box_w * d.box_h * d.box_n);
      d.kpack = 3;
      d.b_off = (int)((std::max(rows, 128u) * 128u + 256u + 1023u) / 1024u * 1024u);
      d.sub_bytes = d.bn * 128;
      d.slot_bytes = (int)((d.b_off + 3u * d.bn * 128u + 1023u) / 1024u * 1024u);
      d.slots = std::min<int>(kMkMaxSlots, p.ring_bytes / d.slot_bytes);
      d.slots -= d.slots % kMkProducers;
      if (d.slots < 2) return "ring too small for a mode-3 conv tile";
      continue;
    }
    const uint32_t rows = d.mode == 0 ? 128u : (uint32_t)(d.box_w * d.box_h * d.box_n);
    const uint32_t a_bytes = rows * d.kblk * 2;
    d.b_off = (int)((a_bytes + 1023) / 1024 * 1024);
    d.sub_bytes = (int)((d.b_off + (uint32_t)d.bn * d.kblk * 2 + 1023) / 1024 * 1024);
    // k-blocks per slot: 2 halves the per-k-block barrier / issue work of the producer and
    // MMA warps when the ring still holds >= 2 slots per producer
    int kpack = 2;
    if (kpack_env > 0) kpack = std::min(kpack_env, 2);  // the MMA loop issues <= 2 per slot
    if ((int)(p.ring_bytes / (kpack * d.sub_bytes)) < min_slots) kpack = 1;
    if (d.pre_layer >= 0) kpack = 1;  // the BN prologue transforms one A tile per slot
    d.kpack = kpack;
    d.slot_bytes = kpack * d.sub_bytes;
    d.slots = std::min<int>(kMkMaxSlots, p.ring_bytes / d.slot_bytes);
    d.slots -= d.slots % kMkProducers;  // producer p owns the slots s % P == p
    if (d.slots < 2) return "ring too small for a conv tile";
  }
  if (fc_seen) {
    const MkLayer& f = p.layers.back().kind == MK_FC ? p.layers.back() : p.layers[p.layers.size() - 2];
    if ((size_t)batch * f.C * 4 > p.ring_bytes) return "fc: pooled features exceed the ring";
    if ((size_t)8 * f.C * 2 > (size_t)kMkOutBufs * kMkOutBufBytes) return "fc: weight block exceeds staging";
  }
  if (mk_blocks_per_sm(p.smem) < 1) return "megakernel does not fit on an SM";
  p.grid = G;
  // ---- device copies
  if (partial_need) {
    CW_TRY(cudaMalloc(&p.d_partial, partial_need));
    for (auto& d : p.layers) {
      if (d.kind == MK_CONV && d.splits > 1 && !d.csplit) {
        // the split conv TMA-stores fp32 partial chunks: [tiles * S * 128][bn], 32-column boxes
        d.partial = p.d_partial;
        CUtensorMap mp;
        const uint64_t rows = (uint64_t)d.m_tiles * d.n_tiles * d.splits * 128;
        if (!make_tmap_2d_f32(&mp, p.d_partial, (uint64_t)d.bn, rows, 128))
          return "tensor map (split-K partials) failed";
        d.tmap_out = (int)p.tmaps.size();
        p.tmaps.push_back(mp);
      } else if (d.kind == MK_REDUCE) {
        d.partial = p.d_partial;
      }
    }
  }
  CW_TRY(cudaMalloc(&p.d_layers, sizeof(MkLayer) * nl));
  CW_TRY(cudaMemcpy(p.d_layers, p.layers.data(), sizeof(MkLayer) * nl, cudaMemcpyHostToDevice));
  CW_TRY(cudaMalloc(&p.d_tmaps, sizeof(CUtensorMap) * std::max<size_t>(1, p.tmaps.size())));
  if (!p.tmaps.empty())
    CW_TRY(cudaMemcpy(p.d_tmaps, p.tmaps.data(), sizeof(CUtensorMap) * p.tmaps.size(),
                      cudaMemcpyHostToDevice));
  CW_TRY(cudaMalloc(&p.d_counters, sizeof(uint32_t) * nl));
  CW_TRY(cudaMemset(p.d_counters, 0, sizeof(uint32_t) * nl));
  CW_TRY(cudaMalloc(&p.d_gen, sizeof(uint32_t)));
  CW_TRY(cudaMemset(p.d_gen, 0, sizeof(uint32_t)));
  CW_TRY(cudaMalloc(&p.d_trace, sizeof(uint64_t) * (nl + 1) * G * 4));
  CW_TRY(cudaMemset(p.d_trace, 0, sizeof(uint64_t) * (nl + 1) * G * 4));
  // pageable-source copies and legacy-stream memsets vs the non-blocking Exec stream
  CW_TRY(cudaStreamSynchronize(0));
  return "";
}

std::string Runtime::capture(Arch& a, Plan& p) {
  (void)a;
  MkArgs args{};
  args.layers = p.d_layers;
  args.tmaps = p.d_tmaps;
  args.n_layers = (int)p.layers.size();
  args.ring_bytes = p.ring_bytes;
  args.ab = ab_;
  args.counters = p.d_counters;
  args.gen = p.d_gen;
  args.trace = p.d_trace;
  if (const char* e = exp_env("CW_MK_FLAGS")) args.flags = (uint32_t)atoi(e);  // experiments only
  // two weight layers ahead at b=1 (short layers: 277 -> 272 us), one at larger batches
  // (two: b=2 +2.5 us, b=16 +3 us)
  args.pf_depth = p.batch == 1 ? 2 : 1;
  args.pre_bn = 0;
  for (const auto& d : p.layers)
    if (d.kind == MK_CONV && d.pre_layer >= 0) args.pre_bn = 1;
  args.softmax = p.layers.back().kind == MK_SOFTMAX;
  args.csize = p.csize;
  for (int copy = 1; copy >= 0; --copy) {
    CW_TRY(cudaStreamBeginCapture(s_cap_, cudaStreamCaptureModeThreadLocal));
    cudaError_t ce = copy ? copy_plan(p.d_layers, (int)p.layers.size(), s_cap_) : cudaSuccess;
    launch_gate(ab_, ring_, kRing - 1, ctr_, exec_recs_, s_cap_);
    cudaError_t le = launch_mk(args, p.grid, p.smem, s_cap_);
    launch_mk_done(ab_, kRing - 1, exec_recs_, p.d_gen, exec_done_, s_cap_);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s_cap_, &g);
    CW_TRY(ce);
    CW_TRY(le);
    CW_TRY(e);
    (copy ? p.graph : p.graph_nocopy) = g;
    CW_TRY(cudaGraphInstantiate(copy ? &p.exec : &p.exec_nocopy, g, 0));
  }
  p.uid = g_plan_uid.fetch_add(1);
  p.launches = 3;
  return "";
}

const Plan* Runtime::plan(int arch, int batch) const {
  auto it = archs_.find(arch);
  if (it == archs_.end()) return nullptr;
  auto pit = it->second.plans.find(batch);
  return pit == it->second.plans.end() ? nullptr : &pit->second;
}

std::string Runtime::build_plans() {
  CW_TRY(cudaSetDevice(device_));
  for (auto& [id, a] : archs_) {
    a.bufs.assign(a.buf_bytes.size(), nullptr);
    for (size_t i = 0; i < a.buf_bytes.size(); ++i) {
      if (!a.buf_bytes[i]) continue;
      CW_TRY(cudaMalloc(&a.bufs[i], a.buf_bytes[i]));
      CW_TRY(cudaMemset(a.bufs[i], 0, a.buf_bytes[i]));  // NHWC4 row padding stays zero
    }
    for (auto& [b, p] : a.plans) {
      std::string err = build_plan(a, b);
      // a deep net whose split-K reduce layers overflow the plan table: no split-K
      if (err == "plan has too many layers") err = build_plan(a, b, false);
      if (!err.empty()) return err;
      err = capture(a, p);
      if (!err.empty()) return err;
    }
  }
  plans_built_ = true;
  return "";
}

// ---------------------------------------------------------------- actions

std::string Runtime::load_async(int blob, const int32_t* pages, int npages, int64_t fence_seq,
                                uint64_t tag, LoadRecord** rec_out, const Runtime* peer,
                                const int32_t* peer_pages,
                                const std::vector<cudaEvent_t>* waits, cudaEvent_t done) {
  CW_TRY(cudaSetDevice(device_));
  auto it = blobs_.find(blob);
  if (it == blobs_.end()) return "unknown blob";
  const Blob& b = it->second;
  if (npages < b.npages) return "not enough pages for blob";
  for (int i = 0; i < b.npages; ++i)
    if (pages[i] < 0 || pages[i] >= pages_total_) return "page index out of range";
  const uint64_t ls = load_seq_++;
  LoadRecord* rec = &load_recs_[ls & (kRing - 1)];
  // Header: per-layer weight tensor maps + bias/weight pointer tables, with the
  // absolute addresses of this load's pages.
  uint8_t* hdr = hdr_stage_ + (ls & 15) * (size_t)kHeaderBytes;
  memset(hdr, 0, kHeaderBytes);
  auto addr = [&](int64_t off) -> uint8_t* {
    return page_ptr(pages[off / page_bytes_]) + off % page_bytes_;
  };
  const float** bias_tab = reinterpret_cast<const float**>(hdr + kHdrBiasOff);
  const void** w_tab = reinterpret_cast<const void**>(hdr + kHdrWeightOff);
  const float** pre_tab = reinterpret_cast<const float**>(hdr + kHdrPreOff);
  for (size_t l = 0; l < b.locs.size(); ++l) {
    const CwTensorLoc& t = b.locs[l];
    if (t.s_off >= 0) pre_tab[l] = reinterpret_cast<const float*>(addr(t.s_off));
    if (t.rows <= 0) continue;
    uint8_t* w = addr(t.w_off);
    CUtensorMap* tm = reinterpret_cast<CUtensorMap*>(hdr + l * kTmapBytes);
    CUtensorMap* tw = reinterpret_cast<CUtensorMap*>(hdr + kHdrWideOff + l * kTmapBytes);
    if (t.k % 64 == 0 && !make_tmap_2d(tm, w, t.k, t.rows, 64)) return "weight tensor map failed";
    if (t.k % 64 == 0 && !make_tmap_2d(tw, w, t.k, t.rows, std::min(256, t.rows)))
      return "weight tensor map (wide) failed";
    if (t.k % 64 == 32 && !make_tmap_2d_sw64(tm, w, t.k, t.rows, 64))
      return "weight tensor map (64B swizzle) failed";
    bias_tab[l] = reinterpret_cast<const float*>(addr(t.b_off));
    w_tab[l] = w;
  }
  if (fence_seq >= 0 && exec_completed() <= (uint64_t)fence_seq) {
    // Still in flight. INFERs complete in order on the Exec stream, so when the fence's
    // event slot was re-recorded by a newer INFER (> kRing later) the newest event covers it.
    const uint64_t s = exec_seq_ - (uint64_t)fence_seq <= kRing ? (uint64_t)fence_seq : exec_seq_ - 1;
    CW_TRY(cudaStreamWaitEvent(s_load_, exec_events_[s & (kRing - 1)], 0));
  }
  if (waits)
    for (cudaEvent_t e : *waits) CW_TRY(cudaStreamWaitEvent(s_load_, e, 0));
  if (peer && peer->page_bytes_ != page_bytes_) return "peer load: page sizes differ";
  launch_stamp(&rec->t_start, tag, s_load_);
  for (int i = 0; i < b.npages; ++i) {
    const size_t off = (size_t)i * page_bytes_;
    const size_t skip = i == 0 ? kHeaderBytes : 0;
    const size_t n = std::min((size_t)page_bytes_, b.bytes - off);
    if (peer)  // the same bytes, resident on the peer GPU (its header differs: skipped)
      CW_TRY(cudaMemcpyPeerAsync(page_ptr(pages[i]) + skip, device_,
                                 peer->page_ptr(peer_pages[i]) + skip, peer->device_, n - skip,
                                 s_load_));
    else
      CW_TRY(cudaMemcpyAsync(page_ptr(pages[i]) + skip, b.host + off + skip, n - skip,
                             cudaMemcpyHostToDevice, s_load_));
  }
  CW_TRY(cudaMemcpyAsync(page_ptr(pages[0]), hdr, kHeaderBytes, cudaMemcpyHostToDevice, s_load_));
  launch_stamp(&rec->t_end, tag, s_load_);
  if (done) CW_TRY(cudaEventRecord(done, s_load_));
  CW_TRY(cudaGetLastError());
  *rec_out = rec;
  return "";
}

std::string Runtime::input_async(int arch, const int32_t* slots, const uint64_t* request_ids,
                                 int batch, uint64_t tag, StampRecord** rec_out) {
  CW_TRY(cudaSetDevice(device_));
  const Arch* a = this->arch(arch);
  if (!a) return "unknown arch";
  const int64_t bytes = (int64_t)a->in_c * a->in_h * a->in_w * 4;
  if (!a->in_pool || a->in_pool_bytes != bytes) return "input pool not set for this arch";
  for (int j = 0; j < batch; ++j) {
    const float* src = a->in_pool + (request_ids[j] % a->in_pool_n) * (bytes / 4);
    CW_TRY(cudaMemcpyAsync(slot_in(slots[j]), src, bytes, cudaMemcpyHostToDevice, s_io_));
  }
  const uint64_t s = in_seq_++;
  CW_TRY(cudaEventRecord(in_events_[s & (kRing - 1)], s_io_));
  StampRecord* rec = &in_recs_[s & (kRing - 1)];
  launch_stamp(&rec->t, tag, s_io_);
  CW_TRY(cudaGetLastError());
  last_input_seq_ = (int64_t)s;
  if (rec_out) *rec_out = rec;
  return "";
}

std::string Runtime::input_from_host(int arch, const int32_t* slots, const float* host, int batch) {
  CW_TRY(cudaSetDevice(device_));
  const Arch* a = this->arch(arch);
  if (!a) return "unknown arch";
  const int64_t bytes = (int64_t)a->in_c * a->in_h * a->in_w * 4;
  for (int j = 0; j < batch; ++j)
    CW_TRY(cudaMemcpy(slot_in(slots[j]), host + j * (bytes / 4), bytes, cudaMemcpyHostToDevice));
  // a pageable-memory cudaMemcpy may return before its DMA lands, and the Exec stream is
  // non-blocking (no implicit ordering with the legacy stream)
  CW_TRY(cudaStreamSynchronize(0));
  return "";
}

std::string Runtime::exec_async(int arch, int batch, int32_t hdr_page, const int32_t* slots,
                                uint64_t earliest_gt, uint64_t latest_gt, int64_t input_seq,
                                uint64_t* seq_out) {
  auto it = archs_.find(arch);
  if (it == archs_.end()) return "unknown arch";
  auto pit = it->second.plans.find(batch);
  if (pit == it->second.plans.end() || !pit->second.exec) return "no plan for batch size";
  const uint64_t seq = exec_seq_;
  ActionDesc& d = ring_[seq & (kRing - 1)];
  d.seq = seq;
  d.earliest_gt = earliest_gt;
  d.latest_gt = latest_gt;
  d.hdr = page_ptr(hdr_page);
  for (int j = 0; j < kMaxBatch; ++j) {
    d.in[j] = j < batch ? slot_in(slots[j]) : nullptr;
    d.out[j] = j < batch ? slot_out(slots[j]) : nullptr;
  }
  d.batch = batch;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  if (input_seq >= 0) CW_TRY(cudaStreamWaitEvent(s_exec_, in_events_[input_seq & (kRing - 1)], 0));
  {
    // the plan-table copy only when the device's constant bank holds another plan
    std::lock_guard<std::mutex> lk(g_exec_mu);
    uint64_t& bank = g_bank_plan[device_];
    const Plan& p = pit->second;
    CW_TRY(cudaGraphLaunch(bank == p.uid ? p.exec_nocopy : p.exec, s_exec_));
    bank = p.uid;
  }
  exec_seq_ = seq + 1;  // the gate consumed ring entry seq: host and device stay aligned
  CW_TRY(cudaEventRecord(exec_events_[seq & (kRing - 1)], s_exec_));
  *seq_out = seq;
  return "";
}

std::string Runtime::output_async(int arch, uint64_t seq, const int32_t* slots, int batch) {
  const Arch* a = this->arch(arch);
  if (!a) return "unknown arch";
  CW_TRY(cudaStreamWaitEvent(s_out_, exec_events_[seq & (kRing - 1)], 0));
  float* dst = out_host_ + (seq & (kRing - 1)) * (size_t)kMaxBatch * out_floats_max_;
  for (int j = 0; j < batch; ++j)
    CW_TRY(cudaMemcpyAsync(dst + j * out_floats_max_, slot_out(slots[j]), a->classes * 4,
                           cudaMemcpyDeviceToHost, s_out_));
  launch_out_done(exec_record(seq), seq + 1, s_out_);
  CW_TRY(cudaGetLastError());
  return "";
}

std::string Runtime::profile_layers(int arch, int batch, int32_t hdr_page, std::vector<float>* end_ms,
                                    std::vector<int>* kinds) {
  CW_TRY(cudaSetDevice(device_));
  const Plan* pp = plan(arch, batch);
  if (!pp || !pp->exec) return "no plan for batch size";
  const Plan& p = *pp;
  const int nl = (int)p.layers.size();
  CW_TRY(cudaMemsetAsync(p.d_trace, 0, sizeof(uint64_t) * (nl + 1) * p.grid * 4, s_exec_));
  int32_t slots[kMaxBatch];
  for (int j = 0; j < kMaxBatch; ++j) slots[j] = j;
  uint64_t seq = 0;
  std::string err = exec_async(arch, batch, hdr_page, slots, 0, ~0ull, -1, &seq);
  if (!err.empty()) return err;
  CW_TRY(cudaStreamSynchronize(s_exec_));
  std::vector<uint64_t>& tr = last_trace_;
  tr.assign((size_t)(nl + 1) * p.grid * 4, 0);
  CW_TRY(cudaMemcpy(tr.data(), p.d_trace, tr.size() * 8, cudaMemcpyDeviceToHost));
  const uint64_t t0 = exec_record(seq)->t_start;
  last_trace_t0_ = t0;
  end_ms->assign(nl, 0.0f);
  kinds->assign(nl, 0);
  for (int L = 0; L < nl; ++L) {
    uint64_t mx = 0;
    for (int c = 0; c < p.grid; ++c) mx = std::max(mx, tr[((size_t)L * p.grid + c) * 4]);
    (*end_ms)[L] = mx > t0 ? (float)((mx - t0) * 1e-6) : 0.0f;
    (*kinds)[L] = p.layers[L].kind;
  }
  return "";
}

std::string Runtime::sync_all() {
  CW_TRY(cudaSetDevice(device_));
  CW_TRY(cudaDeviceSynchronize());
  return "";
}

}  // namespace cw
