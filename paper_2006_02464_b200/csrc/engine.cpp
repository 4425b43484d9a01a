#include "engine.h"

#include <algorithm>
#include <climits>
#include <chrono>
#include <cstring>
#include <ctime>

#include <pthread.h>
#include <sched.h>

namespace cw {

static int64_t realtime_ns() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

Engine::~Engine() { close(); }

std::string Engine::open(const cw_engine_config& cfg) {
  cfg_ = cfg;
  if (cfg.gpu_count < 1) return "gpu_count < 1";
  if (cfg.pages_per_gpu <= 0) return "pages_per_gpu <= 0";
  if (cfg.mode != 0 && cfg.mode != 1) return "mode must be 0 (sim) or 1 (cuda)";
  models_.assign(cfg.models, cfg.models + cfg.n_models);
  for (const auto& m : models_)
    if (m.n_batches < 1 || m.n_batches > 8) return "model with invalid batch table";
  gpus_.resize(cfg.gpu_count);
  for (int g = 0; g < cfg.gpu_count; ++g) {
    GpuState& gs = gpus_[g];
    gs.pages.total = gs.pages.free = cfg.pages_per_gpu;
    gs.io.capacity = cfg.io_capacity;
    if (cfg.mode == 1) {
      const int dev = cfg.devices ? cfg.devices[g] : g;
      gs.rt = new cw_runtime();
      gs.rt->owned = false;
      std::string err = gs.rt->rt.open(dev, cfg.pages_per_gpu, cfg.page_bytes, cfg.io_slots,
                                       cfg.in_bytes_max, cfg.out_bytes_max, 0);
      if (!err.empty()) return "gpu " + std::to_string(g) + ": " + err;
      gs.free_pages.resize(cfg.pages_per_gpu);
      // LIFO free list handing out low page ids first.
      for (int64_t p = 0; p < cfg.pages_per_gpu; ++p)
        gs.free_pages[p] = (int32_t)(cfg.pages_per_gpu - 1 - p);
      gs.page_fence.assign(cfg.pages_per_gpu, -1);
      gs.page_peer.assign(cfg.pages_per_gpu, {});
      gs.free_slots.resize(cfg.io_slots);
      for (int64_t s = 0; s < cfg.io_slots; ++s) gs.free_slots[s] = (int32_t)(cfg.io_slots - 1 - s);
    }
  }
  if (cfg.mode == 1 && cfg.peer_load && cfg.gpu_count > 1) {
    // peer LOAD: every GPU of the worker may read every other's pages
    for (int g = 0; g < cfg.gpu_count; ++g)
      for (int h = 0; h < cfg.gpu_count; ++h) {
        const int dg = gpus_[g].rt->rt.device(), dh = gpus_[h].rt->rt.device();
        if (dg == dh) continue;
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, dg, dh) != cudaSuccess || !ok)
          return "peer_load: device " + std::to_string(dg) + " cannot access " + std::to_string(dh);
        cudaSetDevice(dg);
        const cudaError_t e = cudaDeviceEnablePeerAccess(dh, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return std::string("peer_load: ") + cudaGetErrorString(e);
        cudaGetLastError();  // (clear "already enabled")
      }
  }
  return "";
}

std::string Engine::start() {
  if (started_) return "already started";
  if (cfg_.mode == 1) {
    for (int g = 0; g < (int)gpus_.size(); ++g) {
      Runtime& rt = gpus_[g].rt->rt;
      for (size_t m = 0; m < models_.size(); ++m) {
        const auto& mi = models_[m];
        if (mi.blob_id < 0) return "model " + std::to_string(m) + " has no weights blob";
        const int bp = rt.blob_pages(mi.blob_id);
        if (bp < 0) return "model " + std::to_string(m) + ": blob not registered";
        if (bp > mi.pages_needed)
          return "model " + std::to_string(m) + ": blob needs " + std::to_string(bp) +
                 " pages but the catalog accounts " + std::to_string(mi.pages_needed);
      }
      std::string err = rt.build_plans();
      if (!err.empty()) return "gpu " + std::to_string(g) + ": " + err;
    }
    stop_ = false;
    thread_ = std::thread([this] { run_loop(); });
    // executor threads pinned to a core, at real-time priority when allowed
    if (cfg_.executor_cpu >= 0) {
      cpu_set_t set;
      CPU_ZERO(&set);
      CPU_SET(cfg_.executor_cpu, &set);
      if (pthread_setaffinity_np(thread_.native_handle(), sizeof(set), &set) == 0)
        exec_cpu_ = cfg_.executor_cpu;
    }
    if (cfg_.executor_rt_prio > 0) {
      sched_param sp{};
      sp.sched_priority = cfg_.executor_rt_prio;
      if (pthread_setschedparam(thread_.native_handle(), SCHED_FIFO, &sp) == 0) exec_rt_ = 1;
    }
  }
  started_ = true;
  return "";
}

void Engine::close() {
  if (thread_.joinable()) {
    stop_ = true;
    thread_.join();
  }
  for (auto& g : gpus_) {
    if (g.rt) {
      delete g.rt;
      g.rt = nullptr;
    }
  }
  for (auto* a : owned_) delete a;
  owned_.clear();
  gpus_.clear();
}

int64_t Engine::now() const {
  if (cfg_.mode == 0) return sim_now_;
  return realtime_ns() - cfg_.epoch_ns;
}

int64_t Engine::gt_to_epoch(int g, uint64_t gt) const {
  return (int64_t)gt - gpus_[g].rt->rt.clock_offset() - cfg_.epoch_ns;
}
uint64_t Engine::epoch_to_gt(int g, int64_t t) const {
  if (t >= kNever / 2) return ~0ull;
  const int64_t v = t + cfg_.epoch_ns + gpus_[g].rt->rt.clock_offset();
  return v < 0 ? 0 : (uint64_t)v;
}

void Engine::call_at(int64_t t, Event ev) {
  // SimLoop.call_at clamps to now (timebase.py:70-74); seq breaks ties FIFO.
  const int64_t n = now();
  ev.t = t < n ? n : t;
  ev.seq = ++ev_seq_;
  timers_.push(ev);
  if (cfg_.mode == 0 && ev.type != EV_DELIVER) sim_new_.emplace_back(ev.t, ev.seq);
}

// ------------------------------------------------------------------ API

int Engine::submit(const cw_action& a, int64_t at) {
  if (failed_) return fail("engine failed after a device error; see the first error");
  if (cfg_.mode == 0) {
    std::lock_guard<std::mutex> lk(state_mu_);
    auto* copy = new cw_action(a);
    Event ev{};
    ev.type = EV_DELIVER;
    ev.a = copy;
    call_at(at, ev);
    return 0;
  }
  {
    std::lock_guard<std::mutex> lk(in_mu_);
    inbox_.push_back(a);
  }
  return 0;
}

int Engine::poll(cw_result* out, int max, int64_t timeout_us) {
  std::unique_lock<std::mutex> lk(out_mu_);
  if (outbox_.empty() && timeout_us > 0 && !failed_)
    out_cv_.wait_for(lk, std::chrono::microseconds(timeout_us),
                     [&] { return !outbox_.empty() || failed_; });
  if (outbox_.empty() && failed_) return -1;
  int n = 0;
  while (n < max && !outbox_.empty()) {
    out[n++] = outbox_.front();
    outbox_.pop_front();
  }
  return n;
}

int Engine::sim_deliver(const cw_action& a, int64_t now) {
  if (cfg_.mode != 0) return -1;
  std::lock_guard<std::mutex> lk(state_mu_);  // (state readers: pages(), io_in_use())
  sim_now_ = std::max(sim_now_, now);
  on_action(new cw_action(a));
  return 0;
}

int Engine::stats(int g, int64_t* out, int max) {
  if (g < 0 || g >= (int)gpus_.size()) return -1;
  std::lock_guard<std::mutex> lk(state_mu_);
  const ExecStats& s = gpus_[g].stats;
  const int64_t v[] = {s.dispatched, s.host_late, s.host_eff_late, s.gate_late, s.done,
                       s.dispatch_delay_sum, s.dispatch_delay_max, s.gate_late_sum,
                       s.gate_late_max, s.start_slack_min, s.busy_gap_sum, s.busy_gap_max,
                       s.busy_gaps, s.launch_lat_sum, s.launch_lat_max, s.observe_lat_sum,
                       s.observe_lat_max, s.clock_resyncs, s.clock_step_max};
  const int n = (int)(sizeof(v) / sizeof(v[0]));
  for (int i = 0; i < n && i < max; ++i) out[i] = v[i];
  return n;
}

int Engine::sim_run_to(int64_t t, uint64_t seq) {
  if (cfg_.mode != 0) return -1;
  std::lock_guard<std::mutex> lk(state_mu_);
  int n = 0;
  while (!timers_.empty()) {
    const Event& top = timers_.top();
    if (top.t > t || (top.t == t && top.seq > seq)) break;
    Event ev = top;
    timers_.pop();
    sim_now_ = std::max(sim_now_, ev.t);
    ++n;
    switch (ev.type) {
      case EV_DELIVER: on_action(ev.a); break;
      case EV_WAKE: wake(ev.gpu, ev.infer_exec); break;
      case EV_LOAD_DONE: load_done(ev.gpu, ev.a, ev.started, sim_now_, ev.dur); break;
      case EV_EXEC_DONE: exec_done(ev.gpu, ev.a, ev.started, ev.dur); break;
      case EV_OUTPUT_DONE: output_done(ev.gpu, ev.a, ev.started, sim_now_, ev.dur); break;
    }
  }
  return n;
}

int Engine::sim_take_new(int64_t* times, uint64_t* seqs, int max) {
  std::lock_guard<std::mutex> lk(state_mu_);
  int n = 0;
  while (n < max && !sim_new_.empty()) {
    times[n] = sim_new_.front().first;
    seqs[n] = sim_new_.front().second;
    sim_new_.pop_front();
    ++n;
  }
  return n;
}

int Engine::sim_run(int64_t until) {
  if (cfg_.mode != 0) return -1;
  std::lock_guard<std::mutex> lk(state_mu_);
  // SimLoop.run_until (timebase.py:79-89).
  int n = 0;
  while (!timers_.empty()) {
    Event ev = timers_.top();
    if (ev.t > until) break;
    timers_.pop();
    sim_now_ = ev.t;
    ++n;
    switch (ev.type) {
      case EV_DELIVER: on_action(ev.a); break;
      case EV_WAKE: wake(ev.gpu, ev.infer_exec); break;
      case EV_LOAD_DONE: load_done(ev.gpu, ev.a, ev.started, sim_now_, ev.dur); break;
      case EV_EXEC_DONE: exec_done(ev.gpu, ev.a, ev.started, ev.dur); break;
      case EV_OUTPUT_DONE: output_done(ev.gpu, ev.a, ev.started, sim_now_, ev.dur); break;
    }
  }
  sim_now_ = std::max(sim_now_, until);
  return n;
}

int Engine::pages(int g, int64_t* free, int32_t* models, int32_t* counts, int max, int32_t* n) {
  if (g < 0 || g >= (int)gpus_.size()) return -1;
  std::lock_guard<std::mutex> lk(state_mu_);
  const PageCache& pc = gpus_[g].pages;
  if (free) *free = pc.free;
  std::vector<std::pair<uint32_t, int64_t>> v(pc.resident.begin(), pc.resident.end());
  std::sort(v.begin(), v.end());
  int k = 0;
  for (auto& [m, p] : v) {
    if (k < max) {
      if (models) models[k] = (int32_t)m;
      if (counts) counts[k] = (int32_t)p;
    }
    ++k;
  }
  if (n) *n = k;
  return 0;
}

int64_t Engine::io_in_use(int g) {
  if (g < 0 || g >= (int)gpus_.size()) return -1;
  std::lock_guard<std::mutex> lk(state_mu_);
  return gpus_[g].io.in_use;
}

int Engine::output(int g, int64_t ref, float* dst, int batch, int classes) {
  if (cfg_.mode != 1 || g < 0 || g >= (int)gpus_.size() || ref < 0) return -1;
  Runtime& rt = gpus_[g].rt->rt;
  if ((uint64_t)ref + Runtime::kRing <= rt.exec_issued()) return -1;  // overwritten
  const float* src = rt.output_host((uint64_t)ref);
  const int64_t stride = (int64_t)(rt.output_stride_floats());
  for (int j = 0; j < batch; ++j) memcpy(dst + (int64_t)j * classes, src + j * stride, classes * 4);
  return 0;
}

// ------------------------------------------------------------------ state machine

// worker.py:198-219
void Engine::on_action(cw_action* a) {
  owned_.insert(a);
  const int64_t now = this->now();
  if (a->model_id >= models_.size() || a->gpu_index < 0 || a->gpu_index >= (int)gpus_.size()) {
    finish(a, MALFORMED_ACTION, now, now, 0);
    return;
  }
  GpuState& gpu = gpus_[a->gpu_index];
  if (a->kind == INFER) {
    const cw_model_info& p = model(a->model_id);
    bool ok = false;
    for (int i = 0; i < p.n_batches; ++i) ok |= p.batch_sizes[i] == a->batch_size;
    if (!ok) {
      finish(a, MALFORMED_ACTION, now, now, 0);
      return;
    }
    // Input stage starts immediately on receipt.
    bool acquired = gpu.io.try_acquire(io_bytes(a));
    if (acquired && !device_input(a->gpu_index, a)) {  // physical IOCache slots exhausted
      gpu.io.release(io_bytes(a));
      acquired = false;
    }
    if (acquired)
      input_started(a->gpu_index, a, now);
    else
      gpu.io_waiting.push_back(a);
    gpu.infer_exec.push(a);
    try_start(a->gpu_index, true);
  } else if (a->kind == LOAD || a->kind == UNLOAD) {
    gpu.load_exec.push(a);
    try_start(a->gpu_index, false);
  } else {
    finish(a, MALFORMED_ACTION, now, now, 0);
  }
}

void Engine::input_started(int g, cw_action* a, int64_t now) {
  (void)g;
  input_done_[a->action_id] = now + (int64_t)a->batch_size * model(a->model_id).input_transfer_ns;
}

// worker.py:223-278
void Engine::try_start(int g, bool infer) {
  GpuState& gpu = gpus_[g];
  Executor& ex = infer ? gpu.infer_exec : gpu.load_exec;
  if (ex.busy) return;
  const int64_t now = this->now();
  while (!ex.pending.empty()) {
    const PendingEntry top = ex.pending.top();
    cw_action* a = top.a;
    if (now > a->latest) {
      ex.pending.pop();
      if (a->kind == INFER) ++gpu.stats.host_late;
      reject(g, a, now);
      continue;
    }
    int64_t eff = top.earliest;
    if (a->kind == INFER) {
      auto it = input_done_.find(a->action_id);
      eff = std::max(eff, it == input_done_.end() ? kNever : it->second);
    }
    if (eff > a->latest) {
      // Window will certainly be missed (e.g. IOCache-blocked input).
      if (eff < kNever) {
        ex.pending.pop();
        if (a->kind == INFER) ++gpu.stats.host_eff_late;
        reject(g, a, now);
        continue;
      }
      return;
    }
    if (eff > now) {
      if (ex.next_wake > eff) {
        ex.next_wake = eff;
        Event ev{};
        ev.type = EV_WAKE;
        ev.gpu = g;
        ev.infer_exec = infer;
        call_at(eff, ev);
      }
      return;
    }
    ex.pending.pop();
    if (a->kind == UNLOAD) {
      if (gpu.pages.is_resident(a->model_id) && cfg_.mode == 1) device_unload(g, a->model_id);
      gpu.pages.release(a->model_id);
      finish(a, SUCCESS, now, now, 0);
      continue;
    }
    if (a->kind == LOAD) {
      if (gpu.pages.is_resident(a->model_id)) {
        gpu.pages.touch(a->model_id, now);
        finish(a, SUCCESS, now, now, 0);
        continue;
      }
      const int64_t pages = model(a->model_id).pages_needed;
      if (!gpu.pages.reserve(a->model_id, pages)) {
        finish(a, OUT_OF_PAGES, now, now, 0);
        continue;
      }
      ex.busy = true;
      if (cfg_.mode == 0) {
        const int64_t dur = model(a->model_id).weights_transfer_ns;
        Event ev{};
        ev.type = EV_LOAD_DONE;
        ev.gpu = g;
        ev.a = a;
        ev.started = now;
        ev.dur = dur;
        call_at(now + dur, ev);
      } else {
        device_load(g, a, now);
      }
      return;
    }
    // INFER
    if (!gpu.pages.is_resident(a->model_id)) {
      release_io(g, a);
      finish(a, MODEL_NOT_LOADED, now, now, 0);
      continue;
    }
    ex.busy = true;
    gpu.pages.touch(a->model_id, now);
    if (cfg_.mode == 0) {
      const cw_model_info& p = model(a->model_id);
      int64_t dur = 0;
      for (int i = 0; i < p.n_batches; ++i)
        if (p.batch_sizes[i] == a->batch_size) dur = p.exec_ns[i];
      Event ev{};
      ev.type = EV_EXEC_DONE;
      ev.gpu = g;
      ev.a = a;
      ev.started = now;
      ev.dur = dur;
      call_at(now + dur, ev);
    } else {
      device_exec(g, a, now);
    }
    return;
  }
}

// worker.py:280-282
void Engine::wake(int g, bool infer) {
  (infer ? gpus_[g].infer_exec : gpus_[g].load_exec).next_wake = kNever;
  try_start(g, infer);
}

// worker.py:284-290
void Engine::load_done(int g, cw_action* a, int64_t started, int64_t end, int64_t dur) {
  GpuState& gpu = gpus_[g];
  gpu.pages.commit(a->model_id, end);
  gpu.load_exec.busy = false;
  finish(a, SUCCESS, started, end, dur);
  try_start(g, false);
}

// worker.py:292-299
void Engine::exec_done(int g, cw_action* a, int64_t started, int64_t dur) {
  GpuState& gpu = gpus_[g];
  const int64_t now = this->now();
  gpu.infer_exec.busy = false;
  if (cfg_.mode == 0) {
    const int64_t out_t = (int64_t)a->batch_size * model(a->model_id).output_transfer_ns;
    Event ev{};
    ev.type = EV_OUTPUT_DONE;
    ev.gpu = g;
    ev.a = a;
    ev.started = started;
    ev.dur = dur;
    call_at(now + out_t, ev);
  }
  try_start(g, true);
}

// worker.py:301-305
void Engine::output_done(int g, cw_action* a, int64_t started, int64_t end, int64_t dur) {
  int64_t ref = -1;
  if (cfg_.mode == 1) {
    for (auto& e : gpus_[g].execs)
      if (e.a == a) ref = (int64_t)e.seq;
  }
  release_io(g, a);
  drain_io_waiting(g);
  finish(a, SUCCESS, started, end, dur, ref);
}

// worker.py:313-322
void Engine::release_io(int g, cw_action* a) {
  GpuState& gpu = gpus_[g];
  auto it = input_done_.find(a->action_id);
  if (it != input_done_.end()) {
    input_done_.erase(it);
    gpu.io.release(io_bytes(a));
    if (cfg_.mode == 1) device_release_slots(g, a);
  } else {
    auto w = std::find(gpu.io_waiting.begin(), gpu.io_waiting.end(), a);
    if (w != gpu.io_waiting.end()) gpu.io_waiting.erase(w);
  }
}

// worker.py:324-338
void Engine::drain_io_waiting(int g) {
  GpuState& gpu = gpus_[g];
  const int64_t now = this->now();
  bool started = false;
  while (!gpu.io_waiting.empty()) {
    cw_action* head = gpu.io_waiting.front();
    if (!gpu.io.try_acquire(io_bytes(head))) break;
    if (!device_input(g, head)) {
      gpu.io.release(io_bytes(head));
      break;
    }
    gpu.io_waiting.pop_front();
    input_started(g, head, now);
    started = true;
  }
  if (started) try_start(g, true);
}

// worker.py:340-343
void Engine::reject(int g, cw_action* a, int64_t now) {
  if (a->kind == INFER) release_io(g, a);
  finish(a, REJECTED_TOO_LATE, now, now, 0);
}

// worker.py:345-351
void Engine::finish(cw_action* a, int status, int64_t start, int64_t end, int64_t dur,
                    int64_t output_ref) {
  cw_result r{};
  r.action_id = a->action_id;
  r.status = status;
  r.kind = a->kind;
  r.start = start;
  r.end = end;
  r.device_duration = dur;
  r.output_ref = output_ref;
  r.pages_free = (a->gpu_index >= 0 && a->gpu_index < (int)gpus_.size())
                     ? gpus_[a->gpu_index].pages.free
                     : -1;
  {
    std::lock_guard<std::mutex> lk(out_mu_);
    outbox_.push_back(r);
  }
  out_cv_.notify_one();
  // The action is referenced by no executor or queue any more.
  owned_.erase(a);
  delete a;
}

// ------------------------------------------------------------------ cuda device hooks

bool Engine::device_input(int g, cw_action* a) {
  if (cfg_.mode == 0) return true;
  GpuState& gpu = gpus_[g];
  if ((int)gpu.free_slots.size() < a->batch_size) return false;  // physical IOCache full
  std::vector<int32_t> slots(a->batch_size);
  for (int j = 0; j < a->batch_size; ++j) {
    slots[j] = gpu.free_slots.back();
    gpu.free_slots.pop_back();
  }
  const int arch = models_[a->model_id].arch_id;
  std::string err = gpu.rt->rt.input_async(arch, slots.data(), a->request_ids, a->batch_size, 0,
                                           nullptr);
  gpu.action_input_seq[a->action_id] = gpu.rt->rt.last_input_seq();
  gpu.action_slots[a->action_id] = std::move(slots);
  if (!err.empty()) {
    fail_device("input: " + err);
    return false;
  }
  return true;
}

void Engine::fail_device(const std::string& what) {
  set_error("engine failed (device error, no further actions run): " + what);
  {
    std::lock_guard<std::mutex> lk(out_mu_);
    failed_ = true;
  }
  out_cv_.notify_all();
}

void Engine::device_release_slots(int g, cw_action* a) {
  GpuState& gpu = gpus_[g];
  auto it = gpu.action_slots.find(a->action_id);
  if (it == gpu.action_slots.end()) return;
  for (int32_t s : it->second) gpu.free_slots.push_back(s);
  gpu.action_slots.erase(it);
  gpu.action_input_seq.erase(a->action_id);
}

void Engine::device_load(int g, cw_action* a, int64_t now) {
  GpuState& gpu = gpus_[g];
  const cw_model_info& mi = models_[a->model_id];
  Runtime& rt = gpu.rt->rt;
  const int n = rt.blob_pages(mi.blob_id);
  std::vector<int32_t> pages(n);
  int64_t fence = -1;
  for (int i = 0; i < n; ++i) {
    pages[i] = gpu.free_pages.back();
    gpu.free_pages.pop_back();
    fence = std::max(fence, gpu.page_fence[pages[i]]);
  }
  // Page-reuse fence: a copy must not overwrite pages an in-flight Exec still reads
  // (Runtime::load_async waits on the device only if that Exec has not completed), nor pages
  // a peer LOAD of another GPU is still reading.
  const uint64_t tag = ++load_tag_;
  LoadRecord* rec = nullptr;
  std::vector<cudaEvent_t> waits;
  std::vector<std::shared_ptr<CUevent_st>> keep;  // (alive until the waits are enqueued)
  for (int32_t p : pages) {
    for (auto& e : gpu.page_peer[p]) {
      waits.push_back(e.get());
      keep.push_back(e);
    }
    gpu.page_peer[p].clear();
  }
  // Peer source: another GPU of this worker with the model resident
  // and its own LOAD of it complete.
  int src = -1;
  if (cfg_.peer_load)
    for (int h = 0; h < (int)gpus_.size() && src < 0; ++h) {
      if (h == g || !gpus_[h].model_pages.count(a->model_id)) continue;
      bool loading = false;
      for (const InflightLoad& l : gpus_[h].loads) loading |= l.a->model_id == a->model_id;
      if (!loading) src = h;
    }
  std::shared_ptr<CUevent_st> done;
  if (src >= 0) {
    cudaSetDevice(rt.device());
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      fail_device("load: peer event");
      return;
    }
    done.reset(e, [](CUevent_st* x) { cudaEventDestroy(x); });
  }
  std::string err =
      src < 0 ? rt.load_async(mi.blob_id, pages.data(), n, fence, tag, &rec, nullptr, nullptr,
                              &waits)
              : rt.load_async(mi.blob_id, pages.data(), n, fence, tag, &rec, &gpus_[src].rt->rt,
                              gpus_[src].model_pages[a->model_id].data(), &waits, done.get());
  if (src >= 0)  // the source pages stay readable until this copy completed
    for (int32_t p : gpus_[src].model_pages[a->model_id]) gpus_[src].page_peer[p].push_back(done);
  gpu.model_pages[a->model_id] = std::move(pages);
  if (!err.empty()) {
    fail_device("load: " + err);
    return;
  }
  gpu.loads.push_back({a, rec, tag, now});
}

void Engine::device_unload(int g, uint32_t model) {
  GpuState& gpu = gpus_[g];
  auto it = gpu.model_pages.find(model);
  if (it == gpu.model_pages.end()) return;
  auto le = gpu.model_last_exec.find(model);
  const int64_t fence = le == gpu.model_last_exec.end() ? -1 : le->second;
  for (int32_t p : it->second) {
    gpu.page_fence[p] = fence;
    gpu.free_pages.push_back(p);
  }
  gpu.model_pages.erase(it);
}

void Engine::device_exec(int g, cw_action* a, int64_t now) {
  GpuState& gpu = gpus_[g];
  const cw_model_info& mi = models_[a->model_id];
  Runtime& rt = gpu.rt->rt;
  const auto& slots = gpu.action_slots[a->action_id];
  const int64_t in_seq = gpu.action_input_seq.count(a->action_id)
                             ? gpu.action_input_seq[a->action_id]
                             : -1;
  uint64_t seq = 0;
  std::string err = rt.exec_async(mi.arch_id, a->batch_size, gpu.model_pages[a->model_id][0],
                                  slots.data(), epoch_to_gt(g, a->earliest),
                                  epoch_to_gt(g, a->latest), in_seq, &seq);
  if (!err.empty()) {
    fail_device("exec: " + err);
    return;
  }
  gpu.model_last_exec[a->model_id] = (int64_t)seq;
  ExecStats& st = gpu.stats;
  ++st.dispatched;
  int64_t ready = a->earliest;
  auto it = input_done_.find(a->action_id);
  if (it != input_done_.end()) ready = std::max(ready, it->second);
  InflightExec ie{a, seq, now, 0, false};
  ie.ready = ready;
  ie.dispatched = this->now();
  gpu.execs.push_back(ie);
  if (gpu.last_done_seen > ready) ready = gpu.last_done_seen;
  const int64_t delay = now - ready;
  if (delay > 0) {
    st.dispatch_delay_sum += delay;
    st.dispatch_delay_max = std::max(st.dispatch_delay_max, delay);
  }
}

bool Engine::poll_device() {
  bool progressed = false;
  for (int g = 0; g < (int)gpus_.size(); ++g) {
    GpuState& gpu = gpus_[g];
    Runtime& rt = gpu.rt->rt;
    for (size_t i = 0; i < gpu.loads.size();) {
      InflightLoad l = gpu.loads[i];
      if (l.rec->tag_end == l.tag) {
        gpu.loads.erase(gpu.loads.begin() + i);
        const int64_t end = gt_to_epoch(g, l.rec->t_end);
        const int64_t dur = (int64_t)(l.rec->t_end - l.rec->t_start);
        load_done(g, l.a, l.started, std::max(end, l.started), dur);
        progressed = true;
      } else {
        ++i;
      }
    }
    for (size_t i = 0; i < gpu.execs.size();) {
      InflightExec& e = gpu.execs[i];
      ExecRecord* rec = rt.exec_record(e.seq);
      if (!e.output && rec->seq_done == e.seq + 1) {
        cw_action* a = e.a;
        const int64_t t0 = gt_to_epoch(g, rec->t_start);
        ExecStats& st = gpu.stats;
        gpu.last_done_seen = now();
        if (gpu.last_exec_end >= 0 && e.ready <= gpu.last_exec_end) {
          const int64_t gap = t0 - gpu.last_exec_end;
          st.busy_gap_sum += gap;
          st.busy_gap_max = std::max(st.busy_gap_max, gap);
          ++st.busy_gaps;
        }
        const int64_t t_end = gt_to_epoch(g, rec->t_end);
        const int64_t ll = t0 - e.dispatched, ol = gpu.last_done_seen - t_end;
        st.launch_lat_sum += ll;
        st.launch_lat_max = std::max(st.launch_lat_max, ll);
        st.observe_lat_sum += ol;
        st.observe_lat_max = std::max(st.observe_lat_max, ol);
        gpu.last_exec_end = t_end;
        if (rec->rejected) {
          ++st.gate_late;
          const int64_t late = t0 - a->latest;
          st.gate_late_sum += late;
          st.gate_late_max = std::max(st.gate_late_max, late);
        } else {
          ++st.done;
          st.start_slack_min = std::min(st.start_slack_min, a->latest - t0);
        }
        if (rec->rejected) {
          gpu.execs.erase(gpu.execs.begin() + i);
          gpu.infer_exec.busy = false;
          reject(g, a, t0);
          try_start(g, true);
          progressed = true;
          continue;
        }
        e.output = true;
        e.started = t0;
        e.dur = (int64_t)(rec->t_end - rec->t_start);
        const int arch = models_[a->model_id].arch_id;
        std::string err = rt.output_async(arch, e.seq, gpu.action_slots[a->action_id].data(),
                                          a->batch_size);
        if (!err.empty()) {
          fail_device("output: " + err);
          return progressed;
        }
        const int64_t started = e.started, dur = e.dur;
        exec_done(g, a, started, dur);  // may append to execs
        progressed = true;
        ++i;
        continue;
      }
      if (e.output && rec->seq_out == e.seq + 1) {
        cw_action* a = e.a;
        const int64_t started = e.started, dur = e.dur;
        const int64_t end = std::max(gt_to_epoch(g, rec->t_out), started);
        output_done(g, a, started, end, dur);
        // output_done looked the entry up by pointer; remove it now.
        for (size_t k = 0; k < gpu.execs.size(); ++k)
          if (gpu.execs[k].a == a) {
            gpu.execs.erase(gpu.execs.begin() + k);
            break;
          }
        progressed = true;
        continue;
      }
      ++i;
    }
  }
  return progressed;
}

void Engine::run_loop() {
  std::vector<cw_action> batch;
  int idle = 0;
  while (!stop_ && !failed_) {
    bool progressed = false;
    {
      std::lock_guard<std::mutex> lk(in_mu_);
      batch.swap(inbox_);
    }
    std::unique_lock<std::mutex> state(state_mu_);
    for (const cw_action& a : batch) {
      on_action(new cw_action(a));
      progressed = true;
    }
    batch.clear();
    progressed |= poll_device();
    // keep the globaltimer <-> CLOCK_REALTIME offset current (drift: tens of ppm), between
    // INFERs so the stamp kernel finds an SM
    for (int g = 0; g < (int)gpus_.size(); ++g) {
      GpuState& gpu = gpus_[g];
      if (!gpu.execs.empty() && !gpu.execs.back().output) continue;
      const int64_t t = now();
      if (t < gpu.next_clock_sync) continue;
      int64_t step = 0;
      if (gpu.rt->rt.resync_clock(&step)) {
        ++gpu.stats.clock_resyncs;
        gpu.stats.clock_step_max = std::max(gpu.stats.clock_step_max, step < 0 ? -step : step);
        gpu.next_clock_sync = t + 100000000;  // 10 per second
      } else {
        gpu.next_clock_sync = t + 1000000;
      }
    }
    while (!timers_.empty() && timers_.top().t <= now()) {
      Event ev = timers_.top();
      timers_.pop();
      if (ev.type == EV_WAKE) wake(ev.gpu, ev.infer_exec);
      progressed = true;
    }
    if (progressed) {
      idle = 0;
      continue;
    }
    bool busy = false;
    for (auto& g : gpus_) busy |= !g.loads.empty() || !g.execs.empty();
    if (!busy && (timers_.empty() || timers_.top().t - now() > 200000) && ++idle > 1000) {
      state.unlock();
      std::this_thread::sleep_for(std::chrono::microseconds(50));
      state.lock();
    }
  }
}

}  // namespace cw
