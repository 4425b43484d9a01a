#include "runtime.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <thread>
#include <vector>

#include "kernels.h"
#include "tmap.h"

namespace cw {

#define CW_TRY(expr)                                                                  \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return std::string(#expr) + ": " + cudaGetErrorString(_e);                      \
  } while (0)

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
    }
    for (void* b : a.bufs) cudaFree(b);
    cudaFree(a.partial);
    cudaFree(a.counters);
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
  cudaFreeHost(load_recs_);
  cudaFreeHost(in_recs_);
  cudaFreeHost(out_host_);
  cudaFreeHost(hdr_stage_);
  cudaFreeHost(in_pool_);
  for (auto s : {s_exec_, s_load_, s_io_, s_cap_, s_out_})
    if (s) cudaStreamDestroy(s);
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
  CW_TRY(configure_conv_tc());
  CW_TRY(configure_simt());
  pdl_ = getenv("CW_NO_PDL") == nullptr;
  pages_total_ = pages_total;
  page_bytes_ = page_bytes;
  CW_TRY(cudaMalloc(&pool_, (size_t)(pages_total * page_bytes)));
  in_bytes_max_ = (in_bytes_max + 255) / 256 * 256;
  out_bytes_max_ = (out_bytes_max + 255) / 256 * 256;
  out_floats_max_ = out_bytes_max_ / 4;
  slot_bytes_ = in_bytes_max_ + out_bytes_max_;
  io_slots_ = io_slots;
  CW_TRY(cudaMalloc(&io_, (size_t)(io_slots * slot_bytes_)));
  for (cudaStream_t* s : {&s_exec_, &s_load_, &s_io_, &s_cap_, &s_out_})
    CW_TRY(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
  CW_TRY(cudaMalloc(&ab_, sizeof(ActionBlock)));
  CW_TRY(cudaMemset(ab_, 0, sizeof(ActionBlock)));
  CW_TRY(cudaMalloc(&ctr_, sizeof(uint64_t)));
  CW_TRY(cudaMemset(ctr_, 0, sizeof(uint64_t)));
  CW_TRY(cudaHostAlloc(&ring_, sizeof(ActionDesc) * kRing, cudaHostAllocMapped));
  CW_TRY(cudaHostAlloc(&exec_recs_, sizeof(ExecRecord) * kRing, cudaHostAllocMapped));
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

std::string Runtime::set_input_pool(const float* data, int n, int64_t bytes) {
  CW_TRY(cudaSetDevice(device_));
  if (in_pool_) CW_TRY(cudaFreeHost(in_pool_));
  in_pool_ = nullptr;
  if (bytes > in_bytes_max_) return "input image larger than IOCache slot";
  CW_TRY(cudaHostAlloc(&in_pool_, (size_t)n * bytes, cudaHostAllocDefault));
  memcpy(in_pool_, data, (size_t)n * bytes);
  in_pool_n_ = n;
  in_pool_bytes_ = bytes;
  return "";
}

std::string Runtime::calibrate_clock() {
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
  cudaFreeHost(slot);
  if (est.empty()) return "clock calibration failed";
  std::nth_element(est.begin(), est.begin() + est.size() / 2, est.end());
  gt_offset_ = est[est.size() / 2];
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
  // Workspace buffer sizes at the largest batch.
  auto grow = [&](int buf, size_t bytes) {
    if (buf < 0) return;
    if ((size_t)buf >= a.buf_bytes.size()) a.buf_bytes.resize(buf + 1, 0);
    a.buf_bytes[buf] = std::max(a.buf_bytes[buf], bytes);
  };
  for (const CwOp& op : a.ops) {
    if (op.kind == OP_CONV || op.kind == OP_MAXPOOL || op.kind == OP_AVGPOOL)
      grow(op.in_buf, (size_t)max_b * op.in_h * op.in_w * op.cin * 2);
    if (op.kind == OP_FC) grow(op.in_buf, (size_t)max_b * op.cin * 4);
    if (op.out_buf < 0) continue;
    size_t bytes = 0;
    switch (op.kind) {
      case OP_STEM: bytes = (size_t)max_b * op.out_h * op.out_w * op.kpad * 2; break;
      case OP_CONV: bytes = (size_t)max_b * op.out_h * op.out_w * op.cout * 2; break;
      case OP_MAXPOOL: bytes = (size_t)max_b * op.out_h * op.out_w * op.cin * 2; break;
      case OP_AVGPOOL: bytes = (size_t)max_b * op.cin * 4; break;
      default: break;
    }
    grow(op.out_buf, bytes);
    if (op.kind == OP_CONV)
      a.flops_per_image += 2.0 * op.out_h * op.out_w * op.cout * (double)op.kpad;
    if (op.kind == OP_CONV && (op.cout % 64 != 0 || op.kpad % 64 != 0)) return "conv shape not 64-aligned";
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
  for (const auto& l : b.locs) {
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

// Tile / pipeline / split-K choice for one conv at one batch size. B200: 148 SMs,
// two 107 KB CTAs per SM when a layer has more than one wave of tiles, else one
// CTA per SM with a deep (up to 8-stage) pipeline; split K until the grid covers
// the SMs, keeping >= 4 k-blocks per slice.
static void plan_conv(ConvArgs& c, int cout, int m_tiles, int* bn_out) {
  int bn = (cout % 128 == 0) ? 128 : 64;
  if (bn == 128 && m_tiles * (cout / 128) < 148) bn = 64;
  const int tiles = m_tiles * (cout / bn);
  int splits = 1;
  if (tiles < 148) {
    splits = std::max(1, std::min(2 * 148 / tiles, c.num_kb / 4));
    const int per = (c.num_kb + splits - 1) / splits;
    splits = (c.num_kb + per - 1) / per;
  }
  c.splits = splits;
  c.kb_per_split = (c.num_kb + splits - 1) / splits;
  const int ctas = tiles * splits;
  const int stage_kb = bn == 64 ? 24 : (bn == 128 ? 32 : 48);
  int stages = ctas > 148 ? (bn == 64 ? 4 : 3) : 192 / stage_kb;
  stages = std::max(1, std::min(stages, c.kb_per_split));
  c.stages = stages;
  *bn_out = bn;
}

std::string Runtime::build_plan(Arch& a, int batch) {
  Plan& p = a.plans[batch];
  p.batch = batch;
  p.ops.clear();
  for (size_t oi = 0; oi < a.ops.size(); ++oi) {
    const CwOp& op = a.ops[oi];
    PlanOp po;
    po.kind = op.kind;
    po.batch = batch;
    po.layer = op.layer;
    po.in_h = op.in_h;
    po.in_w = op.in_w;
    po.out_h = op.out_h;
    po.out_w = op.out_w;
    po.kpad = op.kpad;
    po.c = op.cin;
    po.classes = op.cout;
    po.in = op.in_buf >= 0 ? a.bufs[op.in_buf] : nullptr;
    po.out = op.out_buf >= 0 ? a.bufs[op.out_buf] : nullptr;
    if (op.kind == OP_AVGPOOL && !p.ops.empty() && p.ops.back().kind == OP_CONV &&
        p.ops.back().args.pool_out != nullptr) {
      po.kind = -1;  // fused into the previous conv's epilogue
    }
    if (op.kind == OP_CONV) {
      ConvArgs& c = po.args;
      c.layer = op.layer;
      c.n_out = op.cout;
      c.num_kb = op.kpad / 64;
      c.relu = op.relu;
      c.out = po.out;
      c.residual = op.res_buf >= 0 ? a.bufs[op.res_buf] : nullptr;
      c.ab = ab_;
      c.nimg = batch;
      c.oh = op.out_h;
      c.ow = op.out_w;
      c.kw = op.kw;
      c.stride = op.stride;
      c.pad = op.pad;
      // Fuse a following global average pool when one tile can hold whole images.
      const CwOp* nxt = oi + 1 < a.ops.size() ? &a.ops[oi + 1] : nullptr;
      const bool fuse_pool = nxt && nxt->kind == OP_AVGPOOL && nxt->in_buf == op.out_buf &&
                             op.out_h * op.out_w <= 128 && op.cin % 64 == 0;
      if (!fuse_pool && op.kh == 1 && op.kw == 1 && op.stride == 1 && op.pad == 0) {
        c.mode = 0;
        c.m_total = batch * op.out_h * op.out_w;
        po.m_tiles = (c.m_total + 127) / 128;
        if (!make_tmap_2d(&po.tmap, po.in, (uint64_t)op.kpad, (uint64_t)c.m_total, 128))
          return "tensor map (2d) failed";
      } else {
        if (op.cin % 64) return "conv Cin must be a multiple of 64";
        c.mode = 1;
        c.cin_kb = op.cin / 64;
        if (fuse_pool) {
          c.box_w = op.out_w;
          c.box_h = op.out_h;
          c.box_n = std::max(1, std::min(batch, 128 / (op.out_w * op.out_h)));
          c.pool_out = reinterpret_cast<float*>(a.bufs[nxt->out_buf]);
          c.pool_scale = 1.0f / (float)(op.out_h * op.out_w);
          c.out = nullptr;
        } else {
          box_dims(batch, op.out_h, op.out_w, &c.box_w, &c.box_h, &c.box_n);
        }
        c.tiles_w = (op.out_w + c.box_w - 1) / c.box_w;
        c.tiles_h = (op.out_h + c.box_h - 1) / c.box_h;
        const int tiles_n = (batch + c.box_n - 1) / c.box_n;
        po.m_tiles = c.tiles_w * c.tiles_h * tiles_n;
        if (!make_tmap_nhwc(&po.tmap, po.in, batch, op.in_h, op.in_w, op.cin, c.box_w, c.box_h,
                            c.box_n, op.stride))
          return "tensor map (nhwc) failed";
      }
      plan_conv(c, op.cout, po.m_tiles, &po.bn);
      const int tiles = po.m_tiles * (op.cout / po.bn);
      if (c.splits > 1) {
        if (tiles > kCounterStride) return "too many split-K tiles";
        const size_t need = (size_t)tiles * c.splits * 128 * po.bn * 4;
        if (need > a.partial_bytes) return "split-K workspace too small";
        c.partial = a.partial;
        c.counters = a.counters + oi * kCounterStride;
      }
    }
    p.ops.push_back(po);
  }
  return "";
}

std::string Runtime::launch_ops(const Plan& p, cudaStream_t st) {
  for (const PlanOp& po : p.ops) {
    switch (po.kind) {
      case OP_STEM:
        launch_stem_im2col(ab_, po.out, po.batch, po.in_h, po.in_w, po.out_h, po.out_w, po.kpad, st);
        break;
      case OP_CONV:
        CW_TRY(launch_conv_tc(po.tmap, po.args, po.bn, po.m_tiles, st, pdl_));
        break;
      case -1:
        break;
      case OP_MAXPOOL:
        launch_maxpool(ab_, po.in, po.out, po.batch, po.in_h, po.in_w, po.c, po.out_h, po.out_w, st);
        break;
      case OP_AVGPOOL:
        launch_avgpool(ab_, po.in, reinterpret_cast<float*>(po.out), po.batch, po.in_h * po.in_w,
                       po.c, st);
        break;
      case OP_FC:
        launch_fc(ab_, reinterpret_cast<const float*>(po.in), po.layer, po.batch, po.c, po.classes,
                  st);
        break;
      default:
        return "unknown op kind";
    }
    CW_TRY(cudaGetLastError());
  }
  return "";
}

std::string Runtime::capture(Arch& a, Plan& p) {
  (void)a;
  CW_TRY(cudaStreamBeginCapture(s_cap_, cudaStreamCaptureModeThreadLocal));
  launch_gate(ab_, ring_, kRing - 1, ctr_, exec_recs_, s_cap_);
  std::string err = launch_ops(p, s_cap_);
  launch_exec_done(ab_, kRing - 1, exec_recs_, s_cap_);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(s_cap_, &g);
  if (!err.empty()) return err;
  CW_TRY(e);
  p.graph = g;
  CW_TRY(cudaGraphInstantiate(&p.exec, g, 0));
  p.launches = 2;
  for (const PlanOp& po : p.ops) p.launches += po.kind >= 0 ? 1 : 0;
  return "";
}

std::string Runtime::build_plans() {
  CW_TRY(cudaSetDevice(device_));
  for (auto& [id, a] : archs_) {
    a.bufs.assign(a.buf_bytes.size(), nullptr);
    for (size_t i = 0; i < a.buf_bytes.size(); ++i)
      if (a.buf_bytes[i]) CW_TRY(cudaMalloc(&a.bufs[i], a.buf_bytes[i]));
    // Split-K: at most 2*148 CTAs per split conv, 128 x 128 fp32 partial each.
    a.partial_bytes = (size_t)2 * 148 * 128 * 128 * 4 * 2;
    CW_TRY(cudaMalloc(&a.partial, a.partial_bytes));
    CW_TRY(cudaMalloc(&a.counters, a.ops.size() * kCounterStride * sizeof(int)));
    CW_TRY(cudaMemset(a.counters, 0, a.ops.size() * kCounterStride * sizeof(int)));
    for (auto& [b, p] : a.plans) {
      std::string err = build_plan(a, b);
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
                                uint64_t tag, LoadRecord** rec_out) {
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
  for (size_t l = 0; l < b.locs.size(); ++l) {
    const CwTensorLoc& t = b.locs[l];
    if (t.rows <= 0) continue;
    uint8_t* w = addr(t.w_off);
    if (t.k % 64 == 0 &&
        !make_tmap_2d(reinterpret_cast<CUtensorMap*>(hdr + l * kTmapBytes), w, t.k, t.rows, 64))
      return "weight tensor map failed";
    bias_tab[l] = reinterpret_cast<const float*>(addr(t.b_off));
    w_tab[l] = w;
  }
  if (fence_seq >= 0) CW_TRY(cudaStreamWaitEvent(s_load_, exec_events_[fence_seq & (kRing - 1)], 0));
  launch_stamp(&rec->t_start, tag, s_load_);
  for (int i = 0; i < b.npages; ++i) {
    const size_t off = (size_t)i * page_bytes_;
    const size_t skip = i == 0 ? kHeaderBytes : 0;
    const size_t n = std::min((size_t)page_bytes_, b.bytes - off);
    CW_TRY(cudaMemcpyAsync(page_ptr(pages[i]) + skip, b.host + off + skip, n - skip,
                           cudaMemcpyHostToDevice, s_load_));
  }
  CW_TRY(cudaMemcpyAsync(page_ptr(pages[0]), hdr, kHeaderBytes, cudaMemcpyHostToDevice, s_load_));
  launch_stamp(&rec->t_end, tag, s_load_);
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
  if (!in_pool_ || in_pool_bytes_ != bytes) return "input pool not set for this input shape";
  for (int j = 0; j < batch; ++j) {
    const float* src = in_pool_ + (request_ids[j] % in_pool_n_) * (bytes / 4);
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
  CW_TRY(cudaGraphLaunch(pit->second.exec, s_exec_));
  CW_TRY(cudaEventRecord(exec_events_[seq & (kRing - 1)], s_exec_));
  exec_seq_ = seq + 1;
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

std::string Runtime::profile_ops(int arch, int batch, int32_t hdr_page, std::vector<float>* ms,
                                 std::vector<int>* kinds) {
  CW_TRY(cudaSetDevice(device_));
  auto it = archs_.find(arch);
  if (it == archs_.end()) return "unknown arch";
  auto pit = it->second.plans.find(batch);
  if (pit == it->second.plans.end()) return "no plan for batch size";
  const Plan& p = pit->second;
  const uint64_t seq = exec_seq_;
  ActionDesc& d = ring_[seq & (kRing - 1)];
  d.seq = seq;
  d.earliest_gt = 0;
  d.latest_gt = ~0ull;
  d.hdr = page_ptr(hdr_page);
  for (int j = 0; j < kMaxBatch; ++j) {
    d.in[j] = j < batch ? slot_in(j) : nullptr;
    d.out[j] = j < batch ? slot_out(j) : nullptr;
  }
  d.batch = batch;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  std::vector<cudaEvent_t> ev(p.ops.size() + 1);
  for (auto& e : ev) CW_TRY(cudaEventCreate(&e));
  launch_gate(ab_, ring_, kRing - 1, ctr_, exec_recs_, s_exec_);
  CW_TRY(cudaEventRecord(ev[0], s_exec_));
  for (size_t i = 0; i < p.ops.size(); ++i) {
    Plan one;
    one.ops.push_back(p.ops[i]);
    std::string err = launch_ops(one, s_exec_);
    if (!err.empty()) return err;
    CW_TRY(cudaEventRecord(ev[i + 1], s_exec_));
  }
  launch_exec_done(ab_, kRing - 1, exec_recs_, s_exec_);
  exec_seq_ = seq + 1;
  CW_TRY(cudaStreamSynchronize(s_exec_));
  ms->resize(p.ops.size());
  kinds->resize(p.ops.size());
  for (size_t i = 0; i < p.ops.size(); ++i) {
    CW_TRY(cudaEventElapsedTime(&(*ms)[i], ev[i], ev[i + 1]));
    (*kinds)[i] = p.ops[i].kind;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return "";
}

std::string Runtime::sync_all() {
  CW_TRY(cudaSetDevice(device_));
  CW_TRY(cudaDeviceSynchronize());
  return "";
}

}  // namespace cw
