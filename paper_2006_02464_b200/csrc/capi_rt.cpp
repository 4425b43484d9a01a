// extern "C" surface of the device runtime (include/cw.h, cw_rt_*).
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstring>
#include <ctime>
#include <string>
#include <vector>

#include "../../include/cw.h"
#include "capi_util.h"
#include "experiments.h"
#include "runtime.h"

using cw::Runtime;

static_assert(sizeof(cw_op) == sizeof(cw::CwOp), "cw_op layout");
static_assert(sizeof(cw_tensor_loc) == sizeof(cw::CwTensorLoc), "cw_tensor_loc layout");

namespace cw {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace cw

extern "C" {

const char* cw_last_error(void) { return cw::g_err.c_str(); }

int cw_abi_version(void) { return CW_ABI_VERSION; }

int cw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

cw_runtime* cw_rt_open(int device, int64_t pages_total, int64_t page_bytes, int64_t io_slots,
                       int64_t in_bytes_max, int64_t out_bytes_max) {
  auto* h = new cw_runtime();
  std::string err = h->rt.open(device, pages_total, page_bytes, io_slots, in_bytes_max,
                               out_bytes_max, 0);
  if (!err.empty()) {
    cw::set_error(err);
    delete h;
    return nullptr;
  }
  return h;
}

void cw_rt_close(cw_runtime* rt) {
  if (rt && rt->owned) delete rt;
}

int cw_rt_register_arch(cw_runtime* rt, int arch_id, const cw_op* ops, int n_ops, int n_layers,
                        int in_c, int in_h, int in_w, int classes, const int32_t* batches,
                        int n_batches) {
  std::vector<int> b(batches, batches + n_batches);
  return cw::check(rt->rt.register_arch(arch_id, reinterpret_cast<const cw::CwOp*>(ops), n_ops,
                                        n_layers, in_c, in_h, in_w, classes, b.data(), n_batches));
}

int cw_rt_register_blob(cw_runtime* rt, int blob_id, int arch_id, const void* data, int64_t bytes,
                        const cw_tensor_loc* locs, int n_locs) {
  return cw::check(rt->rt.register_blob(blob_id, arch_id, data, (size_t)bytes,
                                        reinterpret_cast<const cw::CwTensorLoc*>(locs), n_locs));
}

int cw_rt_build(cw_runtime* rt) { return cw::check(rt->rt.build_plans()); }

int cw_rt_set_input_pool(cw_runtime* rt, int arch_id, const float* images, int n,
                         int64_t bytes) {
  return cw::check(rt->rt.set_input_pool(arch_id, images, n, bytes));
}

int64_t cw_rt_clock_offset(cw_runtime* rt) { return rt->rt.clock_offset(); }

int cw_rt_plan_info(cw_runtime* rt, int arch_id, int batch, int32_t* launches,
                    double* flops_per_image) {
  const cw::Arch* a = rt->rt.arch(arch_id);
  if (!a) return cw::fail("unknown arch");
  auto it = a->plans.find(batch);
  if (it == a->plans.end()) return cw::fail("no plan for batch");
  if (launches) *launches = it->second.launches;
  if (flops_per_image) *flops_per_image = a->flops_per_image;
  return 0;
}

int cw_rt_load_sync(cw_runtime* rt, int blob_id, const int32_t* pages, int npages,
                    int64_t* copy_ns) {
  cw::LoadRecord* rec = nullptr;
  static uint64_t tag = 1ull << 40;
  const uint64_t my = ++tag;
  std::string err = rt->rt.load_async(blob_id, pages, npages, -1, my, &rec);
  if (!err.empty()) return cw::fail(err);
  err = rt->rt.sync_all();
  if (!err.empty()) return cw::fail(err);
  if (rec->tag_end != my) return cw::fail("load record not written");
  if (copy_ns) *copy_ns = (int64_t)(rec->t_end - rec->t_start);
  return 0;
}

int cw_rt_infer_sync(cw_runtime* rt, int arch_id, int batch, int32_t hdr_page,
                     const float* host_in, float* host_out, int64_t* exec_ns) {
  Runtime& r = rt->rt;
  const cw::Arch* a = r.arch(arch_id);
  if (!a) return cw::fail("unknown arch");
  if (batch < 1 || batch > cw::kMaxBatch || batch > r.io_slots()) return cw::fail("bad batch");
  std::vector<int32_t> slots(batch);
  for (int j = 0; j < batch; ++j) slots[j] = j;
  std::string err = r.input_from_host(arch_id, slots.data(), host_in, batch);
  if (!err.empty()) return cw::fail(err);
  uint64_t seq = 0;
  err = r.exec_async(arch_id, batch, hdr_page, slots.data(), 0, ~0ull, -1, &seq);
  if (!err.empty()) return cw::fail(err);
  err = r.sync_all();
  if (!err.empty()) return cw::fail(err);
  cw::ExecRecord* rec = r.exec_record(seq);
  if (rec->seq_done != seq + 1) return cw::fail("exec record not written");
  if (exec_ns) *exec_ns = (int64_t)(rec->t_end - rec->t_start);
  for (int j = 0; j < batch; ++j) {
    if (cudaMemcpy(host_out + (size_t)j * a->classes, r.slot_out(slots[j]), a->classes * 4,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return cw::fail("logits copy failed");
  }
  return 0;
}

int cw_rt_exec_many(cw_runtime* rt, int arch_id, int batch, const int32_t* hdr_pages, int n,
                    int64_t* exec_ns, int64_t* wall_ns) {
  Runtime& r = rt->rt;
  if (batch < 1 || batch > cw::kMaxBatch || batch > r.io_slots()) return cw::fail("bad batch");
  std::vector<int32_t> slots(batch);
  for (int j = 0; j < batch; ++j) slots[j] = j;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<uint64_t> seqs(n);
  // The exec records live in a ring of kRing entries: harvest each INFER's record once it is
  // done and before its slot is reused (at most kRing / 2 INFERs in flight).
  int harvested = 0;
  const int part = cw::exp_env("CW_EXEC_PART") ? atoi(cw::exp_env("CW_EXEC_PART")) : 0;
  auto harvest = [&](int upto) {
    for (; harvested < upto; ++harvested) {
      cw::ExecRecord* rec = r.exec_record(seqs[harvested]);
      while (rec->seq_done != seqs[harvested] + 1) {
      }
      if (exec_ns) {  // CW_EXEC_PART (diagnostics): 1 = megakernel span, 2 = gate -> megakernel
        exec_ns[harvested] = part == 1   ? (int64_t)(rec->t_mk1 - rec->t_mk0)
                             : part == 2 ? (int64_t)(rec->t_mk0 - rec->t_start)
                                         : (int64_t)(rec->t_end - rec->t_start);
      }
    }
  };
  cudaEventRecord(e0, r.exec_stream());
  for (int i = 0; i < n; ++i) {
    if (i >= Runtime::kRing / 2) harvest(i - Runtime::kRing / 2 + 1);
    std::string err = r.exec_async(arch_id, batch, hdr_pages[i], slots.data(), 0, ~0ull, -1, &seqs[i]);
    if (!err.empty()) return cw::fail(err);
  }
  cudaEventRecord(e1, r.exec_stream());
  if (cudaEventSynchronize(e1) != cudaSuccess) return cw::fail("exec_many sync failed");
  harvest(n);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (wall_ns) *wall_ns = (int64_t)(ms * 1e6);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 0;
}

int cw_rt_exec_closed(cw_runtime* rt, int arch_id, int batch, const int32_t* hdr_pages, int n,
                      int64_t* exec_ns, int64_t* host_ns) {
  Runtime& r = rt->rt;
  if (batch < 1 || batch > cw::kMaxBatch || batch > r.io_slots()) return cw::fail("bad batch");
  std::vector<int32_t> slots(batch);
  for (int j = 0; j < batch; ++j) slots[j] = j;
  auto mono = [] {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
  };
  for (int i = 0; i < n; ++i) {
    uint64_t seq = 0;
    const int64_t t0 = mono();
    std::string err = r.exec_async(arch_id, batch, hdr_pages[i], slots.data(), 0, ~0ull, -1, &seq);
    if (!err.empty()) return cw::fail(err);
    cw::ExecRecord* rec = r.exec_record(seq);
    while (rec->seq_done != seq + 1) {
    }
    const int64_t t1 = mono();
    if (host_ns) host_ns[i] = t1 - t0;
    if (exec_ns) exec_ns[i] = (int64_t)(rec->t_end - rec->t_start);
  }
  return 0;
}

int cw_rt_buffer_io(cw_runtime* rt, int arch_id, int buf, void* host, int64_t bytes,
                    int to_device) {
  const cw::Arch* a = rt->rt.arch(arch_id);
  if (!a || buf < 0 || (size_t)buf >= a->bufs.size() || !a->bufs[buf]) return cw::fail("bad buffer");
  if ((size_t)bytes > a->buf_bytes[buf]) return cw::fail("buffer too small");
  cudaError_t e = to_device ? cudaMemcpy(a->bufs[buf], host, bytes, cudaMemcpyHostToDevice)
                            : cudaMemcpy(host, a->bufs[buf], bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && to_device) e = cudaStreamSynchronize(0);  // DMA landed (pageable)
  return e == cudaSuccess ? 0 : cw::fail(cudaGetErrorString(e));
}

int cw_rt_exec_window(cw_runtime* rt, int arch_id, int batch, int32_t hdr_page, int64_t earliest_gt,
                      int64_t latest_gt, int32_t* rejected, int64_t* t_start_gt,
                      int64_t* t_end_gt) {
  Runtime& r = rt->rt;
  std::vector<int32_t> slots(batch);
  for (int j = 0; j < batch; ++j) slots[j] = j;
  uint64_t seq = 0;
  std::string err = r.exec_async(arch_id, batch, hdr_page, slots.data(), (uint64_t)earliest_gt,
                                 (uint64_t)latest_gt, -1, &seq);
  if (!err.empty()) return cw::fail(err);
  err = r.sync_all();
  if (!err.empty()) return cw::fail(err);
  cw::ExecRecord* rec = r.exec_record(seq);
  if (rejected) *rejected = rec->rejected;
  if (t_start_gt) *t_start_gt = (int64_t)rec->t_start;
  if (t_end_gt) *t_end_gt = (int64_t)rec->t_end;
  return 1;
}

int cw_rt_profile_layers(cw_runtime* rt, int arch_id, int batch, int32_t hdr_page, float* end_ms,
                         int32_t* kinds, int max_layers) {
  std::vector<float> ms;
  std::vector<int> k;
  std::string err = rt->rt.profile_layers(arch_id, batch, hdr_page, &ms, &k);
  if (!err.empty()) return cw::fail(err);
  const int n = (int)ms.size();
  for (int i = 0; i < n && i < max_layers; ++i) {
    end_ms[i] = ms[i];
    kinds[i] = k[i];
  }
  return n;
}

int64_t cw_rt_last_trace(cw_runtime* rt, uint64_t* out, int64_t max_words) {
  const auto& tr = rt->rt.last_trace();
  const int64_t n = (int64_t)tr.size();
  for (int64_t i = 0; i < n && i < max_words; ++i) out[i] = tr[i];
  return n;
}

int cw_rt_plan_layers(cw_runtime* rt, int arch_id, int batch, int32_t* out8, int max_layers) {
  const cw::Plan* p = rt->rt.plan(arch_id, batch);
  if (!p) return cw::fail("no plan for batch");
  const int n = (int)p->layers.size();
  for (int i = 0; i < n && i < max_layers; ++i) {
    const cw::MkLayer& d = p->layers[i];
    int32_t* o = out8 + 8 * i;
    o[0] = d.kind;
    o[1] = d.kind == cw::MK_CONV ? d.mode : -1;
    o[2] = d.bn;
    o[3] = d.tasks;
    o[4] = d.splits;
    o[5] = d.num_kb;
    o[6] = p->layer_op[i];
    o[7] = (d.pool_out != nullptr ? 1 : 0) | (d.csplit ? 2 : 0);
  }
  return n;
}

int cw_rt_plan_launch(cw_runtime* rt, int arch_id, int batch, int32_t* grid, int32_t* csize) {
  const cw::Plan* p = rt->rt.plan(arch_id, batch);
  if (!p) return cw::fail("no plan for batch");
  *grid = p->grid;
  *csize = p->csize;
  return 0;
}

}  // extern "C"

