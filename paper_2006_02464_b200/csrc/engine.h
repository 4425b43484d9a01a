// The worker's action executor: a restatement of the reference
// EmulatedWorker state machine (pkg/src/sloserve/worker.py) in C++, with a
// pluggable device.
//
//   sim  mode: virtual time; Load/Exec/Output take the profiled durations
//              (worker.py:263-266, 273-277, 296-298). Used to prove the page
//              accounting and status semantics bit-exact against the reference.
//   cuda mode: wall time (CLOCK_REALTIME - epoch, timebase.py:45-52); LOAD is a
//              real paged H2D copy, INFER a real CUDA-graph forward pass whose
//              window is re-checked on the device by the gate kernel; completions
//              are observed by polling mapped-memory records.
//
// The control flow (on_action, _try_start, _wake, _load_done, _exec_done,
// _output_done, _release_io, _drain_io_waiting, _reject, _finish) follows the
// reference function by function; each method cites the lines it restates.
#pragma once
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/cw.h"
#include "capi_util.h"

namespace cw {

constexpr int64_t kNever = 1LL << 62;  // worker.py:36
enum Kind { LOAD = 1, UNLOAD = 2, INFER = 3 };
enum Status { SUCCESS = 1, REJECTED_TOO_LATE = 2, OUT_OF_PAGES = 3, MODEL_NOT_LOADED = 4,
              MALFORMED_ACTION = 5 };

struct PageCache {  // worker.py:63-99
  int64_t total = 0, free = 0;
  std::unordered_map<uint32_t, int64_t> resident, in_transit, lru;
  bool is_resident(uint32_t m) const { return resident.count(m) != 0; }
  bool reserve(uint32_t m, int64_t pages) {
    if (pages > free) return false;
    free -= pages;
    in_transit[m] = pages;
    return true;
  }
  void commit(uint32_t m, int64_t now) {
    auto it = in_transit.find(m);
    resident[m] = it->second;
    in_transit.erase(it);
    lru[m] = now;
  }
  void touch(uint32_t m, int64_t now) { lru[m] = now; }
  int64_t release(uint32_t m) {
    int64_t pages = 0;
    auto it = resident.find(m);
    if (it != resident.end()) {
      pages = it->second;
      resident.erase(it);
    }
    free += pages;
    lru.erase(m);
    return pages;
  }
};

struct IOGauge {  // worker.py:102-117
  int64_t capacity = 0, in_use = 0;
  bool try_acquire(int64_t n) {
    if (in_use + n > capacity) return false;
    in_use += n;
    return true;
  }
  void release(int64_t n) { in_use -= n; }
};

struct PendingEntry {
  int64_t earliest;
  uint64_t seq;
  cw_action* a;
  bool operator>(const PendingEntry& o) const {
    return earliest != o.earliest ? earliest > o.earliest : seq > o.seq;
  }
};

struct Executor {  // worker.py:135-146
  std::priority_queue<PendingEntry, std::vector<PendingEntry>, std::greater<PendingEntry>> pending;
  bool busy = false;
  int64_t next_wake = kNever;
  uint64_t seq = 0;
  void push(cw_action* a) { pending.push({a->earliest, ++seq, a}); }
};

struct InflightLoad {
  cw_action* a;
  LoadRecord* rec;
  uint64_t tag;
  int64_t started;
};
struct InflightExec {
  cw_action* a;
  uint64_t seq;
  int64_t started;  // epoch ns (device Exec start)
  int64_t dur;
  bool output;      // false: waiting for Exec end; true: waiting for Output end
  int64_t ready = 0;     // max(earliest, input_done) when dispatched
  int64_t dispatched = 0;  // host time of the graph launch
};

// Executor diagnostics (cuda): where INFER windows are met or missed.
struct ExecStats {
  int64_t dispatched = 0;      // INFER graphs launched
  int64_t host_late = 0;       // rejected by try_start: now > latest (worker.py:230-233)
  int64_t host_eff_late = 0;   // rejected by try_start: eff > latest (worker.py:237-242)
  int64_t gate_late = 0;       // rejected by the device gate (Exec start > latest)
  int64_t done = 0;            // Exec completed on the device
  int64_t dispatch_delay_sum = 0, dispatch_delay_max = 0;  // host dispatch - max(eff, prev end)
  int64_t gate_late_sum = 0, gate_late_max = 0;            // device start - latest (rejects)
  int64_t start_slack_min = INT64_MAX;                      // latest - device start (ok)
  // back-to-back INFERs (the next one was eligible before the previous Exec ended):
  // device start - previous device end
  int64_t busy_gap_sum = 0, busy_gap_max = 0, busy_gaps = 0;
  int64_t launch_lat_sum = 0, launch_lat_max = 0;    // device start - host dispatch
  int64_t observe_lat_sum = 0, observe_lat_max = 0;  // host sees the end - device end
  int64_t clock_resyncs = 0, clock_step_max = 0;      // |offset change| per resync
};

struct GpuState {
  PageCache pages;
  IOGauge io;
  Executor load_exec, infer_exec;
  std::deque<cw_action*> io_waiting;  // worker.py:157
  // cuda device state
  cw_runtime* rt = nullptr;
  std::vector<int32_t> free_pages;
  std::vector<int64_t> page_fence;  // per physical page: last exec seq that read it, -1 none
  // per physical page: the events of the peer LOADs that copied FROM it to other GPUs since
  // it was last written (a LOAD into the page on this GPU waits for them)
  std::vector<std::vector<std::shared_ptr<CUevent_st>>> page_peer;
  std::unordered_map<uint32_t, std::vector<int32_t>> model_pages;
  std::unordered_map<uint32_t, int64_t> model_last_exec;
  std::vector<int32_t> free_slots;
  std::unordered_map<uint64_t, std::vector<int32_t>> action_slots;
  std::unordered_map<uint64_t, int64_t> action_input_seq;
  std::vector<InflightLoad> loads;
  std::vector<InflightExec> execs;
  ExecStats stats;
  int64_t last_exec_end = -1;  // epoch ns of the previous Exec end (device)
  int64_t last_done_seen = -1; // host time the engine saw it
  int64_t next_clock_sync = 0; // host time of the next globaltimer resync
};

enum EvType { EV_DELIVER, EV_WAKE, EV_LOAD_DONE, EV_EXEC_DONE, EV_OUTPUT_DONE };
struct Event {
  int64_t t;
  uint64_t seq;
  int type;
  int gpu;
  bool infer_exec;  // EV_WAKE: which executor
  cw_action* a;
  int64_t started, dur;
  bool operator>(const Event& o) const { return t != o.t ? t > o.t : seq > o.seq; }
};

class Engine {
 public:
  ~Engine();
  std::string open(const cw_engine_config& cfg);
  std::string start();
  void close();
  cw_runtime* runtime(int g) { return g >= 0 && g < (int)gpus_.size() ? gpus_[g].rt : nullptr; }
  int submit(const cw_action& a, int64_t at);
  int poll(cw_result* out, int max, int64_t timeout_us);
  int sim_run(int64_t until);
  int64_t now() const;
  int64_t next_event_time() {
    std::lock_guard<std::mutex> lk(state_mu_);
    return timers_.empty() ? -1 : timers_.top().t;
  }
  int pages(int g, int64_t* free, int32_t* models, int32_t* counts, int max, int32_t* n);
  int64_t io_in_use(int g);
  // A CUDA failure is fatal to the engine (never turned into a protocol status): the engine
  // stops executing, poll() returns -1 once the results issued before it are drained.
  bool failed() const { return failed_; }
  void executor_info(int32_t* cpu, int32_t* rt) const {
    *cpu = exec_cpu_;
    *rt = exec_rt_;
  }
  // sim: deliver an action now (at virtual time `now` >= every processed event), ahead of
  // engine events at the same time that the caller's loop has not run yet.
  int sim_deliver(const cw_action& a, int64_t now);
  // sim, driven by an external event loop: process events up to (t, seq) in (time, seq)
  // order, and hand out the (t, seq) of every event scheduled since the last call so the
  // caller schedules one loop callback per engine event, in the same order as the
  // reference's loop.call_at calls (worker.py:246, 265, 276, 296).
  int sim_run_to(int64_t t, uint64_t seq);
  int stats(int g, int64_t* out, int max);
  int sim_take_new(int64_t* times, uint64_t* seqs, int max);
  int output(int g, int64_t ref, float* dst, int batch, int classes);

 private:
  // --- reference state machine (worker.py)
  void on_action(cw_action* a);
  void try_start(int g, bool infer);
  void wake(int g, bool infer);
  void load_done(int g, cw_action* a, int64_t started, int64_t end, int64_t dur);
  void exec_done(int g, cw_action* a, int64_t started, int64_t dur);
  void output_done(int g, cw_action* a, int64_t started, int64_t end, int64_t dur);
  void release_io(int g, cw_action* a);
  void drain_io_waiting(int g);
  void reject(int g, cw_action* a, int64_t now);
  void finish(cw_action* a, int status, int64_t start, int64_t end, int64_t dur,
              int64_t output_ref = -1);
  void input_started(int g, cw_action* a, int64_t now);
  // --- device hooks (cuda)
  void fail_device(const std::string& what);
  bool device_input(int g, cw_action* a);
  void device_release_slots(int g, cw_action* a);
  void device_load(int g, cw_action* a, int64_t now);
  void device_unload(int g, uint32_t model);
  void device_exec(int g, cw_action* a, int64_t now);
  bool poll_device();
  void call_at(int64_t t, Event ev);
  void run_loop();
  int64_t gt_to_epoch(int g, uint64_t gt) const;
  uint64_t epoch_to_gt(int g, int64_t t) const;
  const cw_model_info& model(uint32_t m) const { return models_[m]; }
  int64_t io_bytes(const cw_action* a) const {
    const auto& p = model(a->model_id);
    return (int64_t)a->batch_size * (p.input_size + p.output_size);
  }

  cw_engine_config cfg_{};
  std::vector<cw_model_info> models_;
  std::vector<GpuState> gpus_;
  std::unordered_map<uint64_t, int64_t> input_done_;  // worker.py:177
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> timers_;
  uint64_t ev_seq_ = 0;
  int64_t sim_now_ = 0;
  std::deque<std::pair<int64_t, uint64_t>> sim_new_;  // scheduled, not yet handed out
  uint64_t load_tag_ = 0;
  std::unordered_set<cw_action*> owned_;  // live actions (freed at finish)

  // threading (cuda)
  std::mutex in_mu_;
  std::vector<cw_action> inbox_;
  std::mutex out_mu_;
  std::condition_variable out_cv_;
  std::deque<cw_result> outbox_;
  std::mutex state_mu_;
  std::thread thread_;
  volatile bool stop_ = false;
  volatile bool failed_ = false;
  int32_t exec_cpu_ = -1, exec_rt_ = 0;
  bool started_ = false;
};

}  // namespace cw
