// Native controller fast path: the reference's centralized
// proactive scheduler restated in C++ — admission, per-batch-size request queues,
// strategy heaps per Infer executor, speculative batch growth, demand statistics and
// load priorities, LRU eviction, result folding and the controller-side worker mirror.
//
// Decision-for-decision the same as /root/reference/pkg/src/sloserve/scheduler.py and
// controller_state.py (every function cites the one it restates), including the float
// arithmetic of the load statistics: CPython 3.12's sum() of floats is Neumaier-compensated
// (py_fsum below), and the file is compiled without FMA contraction. The Python shim
// (native_scheduler.py) feeds it the loop's events and replays its outputs — actions,
// responses, timer requests and action-sink records — in the order the reference emits
// them, so it drops in for sloserve.scheduler.Scheduler behind the unmodified harness.
// Thread-confined like the reference (scheduler.py:30).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <queue>
#include <set>
#include <unordered_map>
#include <utility>
#include <vector>


namespace cw {
namespace sched {

constexpr int64_t kInf = int64_t(1) << 62;                     // scheduler.py:48
enum : int { QUEUED = 0, DISPATCHED = 1, DONE = 2 };         // scheduler.py:44-46
enum : int { K_LOAD = 1, K_UNLOAD = 2, K_INFER = 3 };         // protocol.py:66-69
enum : int { R_SUCCESS = 1 };                                 // protocol.py:72-77
enum : int { S_OK = 1, S_DENIED = 2, S_TIMEOUT = 3 };         // protocol.py:80-83
// output event records (16 x int64) replayed by the shim in order
enum : int64_t { EV_ACTION = 1, EV_RESPONSE = 2, EV_TIMER = 3, EV_SINK = 4 };
enum : int64_t { T_DEADLINE = 1, T_WAKE = 2 };
constexpr int kRec = 16;

// CPython 3.12 builtin sum() over floats with an int start of 0: the first item is taken
// as is (0 + x), the rest are added with Neumaier compensation, the compensation added at
// the end when finite (Python/bltinmodule.c builtin_sum_impl).
static double py_fsum(const double* x, size_t n) {
  if (n == 0) return 0.0;
  double f = 0.0 + x[0], c = 0.0;
  for (size_t i = 1; i < n; ++i) {
    const double t = f + x[i];
    if (std::fabs(f) >= std::fabs(x[i])) c += (f - t) + x[i];
    else c += (x[i] - t) + f;
    f = t;
  }
  if (c != 0.0 && std::isfinite(c)) f += c;
  return f;
}

struct Config {  // scheduler.py:51-60
  int64_t work_horizon, capacity_horizon, lead_slack, tardy_slack, unload_tardy;
  int64_t estimator_window, default_slo;
  double load_eps;
};

struct Model {  // scheduler.py:80-109 (_ModelRuntime) + the profile constants it reads
  int id = 0;
  std::vector<int> sizes;
  std::vector<int64_t> seed_dur;
  int64_t unit = 0, input_transfer = 0, output_transfer = 0, weights_transfer = 0;
  int pages = 1;
  std::vector<std::deque<int>> queues;  // request slots
  std::vector<int> counts;
  int64_t seq = 0, last_load = 0, queued_requests = 0;
  int64_t output_margin(int64_t slo, int64_t tardy) const {
    int b_cap = sizes[0];
    for (size_t i = 0; i < sizes.size(); ++i)
      if (seed_dur[i] <= slo) b_cap = sizes[i];
    return (int64_t)b_cap * output_transfer + tardy;
  }
  int index_of(int b) const {
    for (size_t i = 0; i < sizes.size(); ++i)
      if (sizes[i] == b) return (int)i;
    return -1;
  }
};

struct Req {  // scheduler.py:63-77 (PendingRequest)
  uint64_t request_id = 0;
  int model = 0;
  int64_t arrival = 0, slo = 0, deadline = 0;
  int state = QUEUED;
  bool cold = false;
  uint32_t size_mask = 0;
  int served_batch = 0;
  int refs = 0;  // queue entries + armed deadline checks + outstanding actions + live
};

struct Estimator {  // controller_state.py:18-44 (DurationEstimator)
  int64_t seed = 0, est = 0;
  size_t maxlen = 10;
  std::vector<int64_t> w;
  void observe(int64_t d) {
    w.push_back(d);
    if (w.size() > maxlen) w.erase(w.begin());
    const size_t k = (size_t)std::ceil(0.99 * (double)w.size());
    if (k >= w.size()) {
      est = *std::max_element(w.begin(), w.end());
    } else {
      std::vector<int64_t> s = w;
      std::sort(s.begin(), s.end());
      est = s[k - 1];
    }
  }
};

struct Timeline {  // controller_state.py:47-72 (ExecutorTimeline)
  std::map<uint64_t, std::pair<int64_t, int64_t>> out;
  int64_t max_end = 0;
  void add(uint64_t id, int64_t s, int64_t e) {
    out[id] = {s, e};
    if (e > max_end) max_end = e;
  }
  void remove(uint64_t id) {
    auto it = out.find(id);
    if (it == out.end()) return;
    const int64_t e = it->second.second;
    out.erase(it);
    if (e >= max_end) {
      max_end = 0;
      for (auto& kv : out) max_end = std::max(max_end, kv.second.second);
    }
  }
  int64_t free_at(int64_t now) const { return max_end > now ? max_end : now; }
  int64_t outstanding(int64_t now) const { return free_at(now) - now; }
};

struct Gpu {  // controller_state.py:75-152 (GpuMirror)
  int64_t pages_total = 0, pages_free = 0;
  std::map<int, int64_t> resident, resident_from, lru;
  std::map<int, uint64_t> pending_load;
  std::map<int, int64_t> inflight;
  Timeline infer_tl, load_tl;
  bool resident_or_pending(int m) const { return resident.count(m) != 0; }
  bool confirmed(int m) const { return resident.count(m) && !pending_load.count(m); }
  int64_t residency_time(int m) const {
    auto it = resident_from.find(m);
    return it == resident_from.end() ? 0 : it->second;
  }
  void plan_load(int m, int64_t pages, int64_t end, uint64_t id) {
    pages_free -= pages;
    resident[m] = pages;
    resident_from[m] = end;
    pending_load[m] = id;
    lru[m] = end;
  }
  void rollback_load(int m) {
    auto it = resident.find(m);
    if (it != resident.end()) {
      pages_free += it->second;
      resident.erase(it);
    }
    resident_from.erase(m);
    pending_load.erase(m);
    lru.erase(m);
  }
  void plan_unload(int m) {
    auto it = resident.find(m);
    if (it != resident.end()) {
      pages_free += it->second;
      resident.erase(it);
    }
    resident_from.erase(m);
    lru.erase(m);
  }
  void touch(int m, int64_t t) {
    auto it = lru.find(m);
    if (it != lru.end()) it->second = t;
  }
  void bump_inflight(int m, int64_t d) {
    const int64_t n = inflight[m] + d;
    if (n) inflight[m] = n;
    else inflight.erase(m);
  }
  Timeline& tl(int kind) { return kind == K_INFER ? infer_tl : load_tl; }
};

typedef std::pair<int, int> GKey;  // (worker_id, gpu_index)

struct Outstanding {  // controller_state.py:168-190
  uint64_t action_id = 0;
  int worker = 0, gpu = 0, kind = 0, model = 0, batch = 0;
  std::vector<int> reqs;
  int64_t pstart = 0, pend = 0, pdur = 0, presult_end = 0;
};

struct Strategy {  // heap entry (latest, -batch, model_id, seq), scheduler.py:132
  int64_t latest, negb, model, seq;
  bool operator>(const Strategy& o) const {
    if (latest != o.latest) return latest > o.latest;
    if (negb != o.negb) return negb > o.negb;
    if (model != o.model) return model > o.model;
    return seq > o.seq;
  }
};
typedef std::priority_queue<Strategy, std::vector<Strategy>, std::greater<Strategy>> Heap;

class Scheduler {
 public:
  Config cfg;
  std::vector<Model> models;
  std::vector<Req> reqs;
  std::vector<int> free_slots;
  std::unordered_map<uint64_t, int> live;  // request id -> slot (live_requests)
  // workers in handshake order (dict insertion order), their gpu mirrors
  std::vector<int> worker_order;
  std::map<int, std::vector<Gpu>> workers;
  std::map<std::tuple<int, int, int>, Estimator> infer_est;
  std::map<GKey, Estimator> load_est;
  std::unordered_map<uint64_t, Outstanding> outstanding;
  std::map<GKey, Heap> strategies;
  std::map<int, std::set<GKey>> resident_gpus;
  std::map<int, std::map<GKey, double>> alloc;
  std::map<GKey, double> gpu_load;
  std::map<int, double> priority;
  std::set<int> demand_models;
  std::map<std::tuple<int, int, int>, int64_t> wakes;
  uint64_t next_action_id = 1;
  // output
  std::vector<int64_t> ev;
  std::vector<uint64_t> ids;

  // ---------------------------------------------------------------- outputs
  int64_t* rec(int64_t type) {
    ev.resize(ev.size() + kRec, 0);
    int64_t* r = &ev[ev.size() - kRec];
    r[0] = type;
    return r;
  }
  void call_at(int64_t t, int64_t kind, int64_t a, int64_t b = 0, int64_t c = 0) {
    int64_t* r = rec(EV_TIMER);
    r[1] = t;
    r[2] = kind;
    r[3] = a;
    r[4] = b;
    r[5] = c;
  }
  void send_action(int wid, uint64_t id, int kind, int model, int64_t earliest, int64_t latest,
                   const std::vector<int>* members, int gpu, int64_t expected) {
    int64_t* r = rec(EV_ACTION);
    r[1] = wid;
    r[2] = (int64_t)id;
    r[3] = kind;
    r[4] = model;
    r[5] = earliest;
    r[6] = latest;
    r[7] = gpu;
    r[8] = expected;
    r[9] = members ? (int64_t)members->size() : 0;
    r[10] = (int64_t)ids.size();
    if (members)
      for (int s : *members) ids.push_back(reqs[s].request_id);
  }
  void respond(int slot, int status, int64_t now, int batch, int64_t latency, bool has_lat) {
    // scheduler.py:627-636 (_respond)
    Req& pr = reqs[slot];
    if (!has_lat) latency = now - pr.arrival;
    pr.state = DONE;
    pr.served_batch = batch;
    auto it = live.find(pr.request_id);
    if (it != live.end() && it->second == slot) {
      live.erase(it);
      unref(slot);
    }
    int64_t* r = rec(EV_RESPONSE);
    r[1] = 1;
    r[2] = (int64_t)pr.request_id;
    r[3] = status;
    r[4] = latency;
    r[5] = pr.cold;
    r[6] = pr.model;
    r[7] = pr.arrival;
    r[8] = pr.slo;
    r[9] = pr.deadline;
    r[10] = pr.served_batch;
  }
  void unref(int slot) {
    Req& pr = reqs[slot];
    if (--pr.refs == 0) free_slots.push_back(slot);
  }
  int new_req() {
    if (!free_slots.empty()) {
      const int s = free_slots.back();
      free_slots.pop_back();
      reqs[s] = Req();
      return s;
    }
    reqs.emplace_back();
    return (int)reqs.size() - 1;
  }

  // ---------------------------------------------------------------- state (controller_state.py)
  Gpu& gpu(int wid, int g) { return workers[wid][(size_t)g]; }
  Estimator& iest(int wid, int m, int b) {
    auto key = std::make_tuple(wid, m, b);
    auto it = infer_est.find(key);
    if (it == infer_est.end()) {
      Estimator e;
      const Model& mr = models[(size_t)m];
      e.seed = e.est = mr.seed_dur[(size_t)mr.index_of(b)];
      e.maxlen = (size_t)cfg.estimator_window;
      it = infer_est.emplace(key, e).first;
    }
    return it->second;
  }
  Estimator& lest(int wid, int m) {
    GKey key(wid, m);
    auto it = load_est.find(key);
    if (it == load_est.end()) {
      Estimator e;
      e.seed = e.est = models[(size_t)m].weights_transfer;
      e.maxlen = (size_t)cfg.estimator_window;
      it = load_est.emplace(key, e).first;
    }
    return it->second;
  }
  int64_t predict_infer(int wid, int m, int b) { return iest(wid, m, b).est; }
  int64_t predict_load(int wid, int m) { return lest(wid, m).est; }
  static std::pair<int64_t, int64_t> predict_completion(const Timeline& tl, int64_t dur,
                                                        int64_t ea, int64_t now) {
    int64_t start = tl.free_at(now);
    if (ea > start) start = ea;
    return {start, start + dur};
  }
  static std::pair<int64_t, int64_t> window_for(int64_t pstart, int64_t now, int64_t lead,
                                                int64_t tardy) {
    int64_t e = pstart - lead;
    if (e < now) e = now;
    return {e, pstart + tardy};
  }
  void register_out(Outstanding&& o) {
    Gpu& g = gpu(o.worker, o.gpu);
    g.tl(o.kind).add(o.action_id, o.pstart, o.pend);
    g.bump_inflight(o.model, +1);
    for (int s : o.reqs) ++reqs[s].refs;
    outstanding[o.action_id] = std::move(o);
  }
  bool is_warm(int m) {
    for (int wid : worker_order)
      for (const Gpu& g : workers[wid])
        if (g.confirmed(m)) return true;
    return false;
  }

  // ---------------------------------------------------------------- topology
  void on_handshake(int wid, int gpu_count, int64_t pages) {  // scheduler.py:146-150
    if (!workers.count(wid)) worker_order.push_back(wid);
    std::vector<Gpu> gs((size_t)gpu_count);
    for (Gpu& g : gs) g.pages_total = g.pages_free = pages;
    workers[wid] = std::move(gs);
    for (int g = 0; g < gpu_count; ++g) {
      strategies[GKey(wid, g)] = Heap();
      gpu_load[GKey(wid, g)] = 0.0;
    }
  }

  // ---------------------------------------------------------------- admission
  void on_request(int64_t now, uint64_t rid, int64_t model, int64_t slo) {  // :155-168
    if (model < 0 || model >= (int64_t)models.size() || slo <= 0) {
      int64_t* r = rec(EV_RESPONSE);
      r[1] = 0;
      r[2] = (int64_t)rid;
      r[3] = S_DENIED;
      return;
    }
    Model& mr = models[(size_t)model];
    const int s = new_req();
    Req& pr = reqs[(size_t)s];
    pr.request_id = rid;
    pr.model = (int)model;
    pr.arrival = now;
    pr.slo = slo;
    pr.deadline = now + slo - mr.output_margin(slo, cfg.tardy_slack);
    pr.cold = !is_warm((int)model);
    pr.refs = 1;  // until the response (or the admission's end)
    if (pr.deadline <= now || best_completion(mr, now) > pr.deadline) {
      live[rid] = s;  // (respond pops it)
      respond(s, S_DENIED, now, 0, 0, false);
      return;
    }
    live[rid] = s;
    if (!admit(s, mr, now)) return;
    pump(now);
  }

  int64_t best_completion(Model& mr, int64_t now) {  // scheduler.py:170-191
    const int m = mr.id, b = mr.sizes[0];
    int64_t best = kInf;
    for (int wid : worker_order) {
      std::vector<Gpu>& gs = workers[wid];
      for (size_t g = 0; g < gs.size(); ++g) {
        Gpu& mi = gs[g];
        const int64_t dur = predict_infer(wid, m, b);
        int64_t ea = now + (int64_t)b * mr.input_transfer;
        if (mi.resident_or_pending(m)) {
          const int64_t rt = mi.residency_time(m);
          if (rt > ea) ea = rt;
        } else {
          const int64_t le = predict_completion(mi.load_tl, predict_load(wid, m), now, now).second;
          if (le > ea) ea = le;
        }
        const int64_t end = predict_completion(mi.infer_tl, dur, ea, now).second;
        if (end < best) best = end;
      }
    }
    return best;
  }

  bool admit(int s, Model& mr, int64_t now) {  // scheduler.py:193-214
    uint32_t mask = 0;
    const int64_t margin = cfg.tardy_slack;
    for (size_t i = 0; i < mr.sizes.size(); ++i) {
      if (now + mr.seed_dur[i] + margin <= reqs[(size_t)s].deadline) {
        mr.queues[i].push_back(s);
        ++reqs[(size_t)s].refs;
        mr.counts[i] += 1;
        mask |= 1u << i;
      }
    }
    if (!mask) {
      respond(s, S_DENIED, now, 0, 0, false);
      return false;
    }
    Req& pr = reqs[(size_t)s];
    pr.size_mask = mask;
    pr.state = QUEUED;
    set_queued(mr, mr.queued_requests + 1);
    update_load_stats(mr.id);
    ++reqs[(size_t)s].refs;
    call_at(reqs[(size_t)s].deadline - margin - mr.seed_dur[0] + 1, T_DEADLINE, s);
    refresh_strategies(mr.id, now);
    return true;
  }

  void deadline_check(int s, int64_t now) {  // scheduler.py:216-227
    Req& pr = reqs[(size_t)s];
    if (pr.state != QUEUED) {
      unref(s);
      return;
    }
    Model& mr = models[(size_t)pr.model];
    drop_all_queues(mr, s);
    respond(s, S_DENIED, now, 0, 0, false);
    set_queued(mr, mr.queued_requests - 1);
    update_load_stats(mr.id);
    refresh_strategies(mr.id, now);
    unref(s);
    pump(now);
  }

  // ---------------------------------------------------------------- batch queues
  void drop_all_queues(Model& mr, int s) {  // scheduler.py:232-240
    uint32_t mask = reqs[(size_t)s].size_mask;
    int i = 0;
    while (mask) {
      if (mask & 1) mr.counts[(size_t)i] -= 1;
      mask >>= 1;
      ++i;
    }
    reqs[(size_t)s].size_mask = 0;
  }
  void purge_expired(Model& mr, int s, int i, int64_t now) {  // scheduler.py:242-250
    Req& pr = reqs[(size_t)s];
    mr.counts[(size_t)i] -= 1;
    pr.size_mask &= ~(1u << i);
    if (pr.size_mask == 0 && pr.state == QUEUED) {
      respond(s, S_DENIED, now, 0, 0, false);
      set_queued(mr, mr.queued_requests - 1);
      update_load_stats(mr.id);
    }
  }
  // pops dead / expired prefix entries of queue i (shared by _peek_batch and _queue_head)
  int clean_head(Model& mr, int i, int64_t now) {
    std::deque<int>& q = mr.queues[(size_t)i];
    const uint32_t bit = 1u << i;
    const int64_t cutoff = now + mr.seed_dur[(size_t)i] + cfg.tardy_slack;
    while (!q.empty()) {
      const int s = q.front();
      Req& pr = reqs[(size_t)s];
      if (pr.state != QUEUED || !(pr.size_mask & bit)) {
        q.pop_front();
        unref(s);
        continue;
      }
      if (pr.deadline < cutoff) {
        q.pop_front();
        purge_expired(mr, s, i, now);
        unref(s);
        continue;
      }
      return s;
    }
    return -1;
  }
  // scheduler.py:252-283 (_peek_batch): first `need` live members, their min deadline
  bool peek_batch(Model& mr, int i, int need, int64_t now, std::vector<int>& members,
                  int64_t& min_deadline) {
    clean_head(mr, i, now);
    if (mr.counts[(size_t)i] < need) return false;
    members.clear();
    min_deadline = kInf;
    const uint32_t bit = 1u << i;
    const int64_t cutoff = now + mr.seed_dur[(size_t)i] + cfg.tardy_slack;
    for (int s : mr.queues[(size_t)i]) {
      const Req& pr = reqs[(size_t)s];
      if (pr.state != QUEUED || !(pr.size_mask & bit)) continue;
      if (pr.deadline < cutoff) continue;
      members.push_back(s);
      if (pr.deadline < min_deadline) min_deadline = pr.deadline;
      if ((int)members.size() == need) return true;
    }
    return false;
  }
  void take_batch(Model& mr, int i, const std::vector<int>& members, int64_t now) {  // :285-302
    std::deque<int>& q = mr.queues[(size_t)i];
    const uint32_t bit = 1u << i;
    size_t taken = 0;
    const size_t want = members.size();
    while (taken < want) {
      const int s = q.front();
      q.pop_front();
      if (s == members[taken]) {
        ++taken;
      } else if (reqs[(size_t)s].state == QUEUED && (reqs[(size_t)s].size_mask & bit)) {
        purge_expired(mr, s, i, now);
      }
      unref(s);
    }
    for (int s : members) {
      drop_all_queues(mr, s);
      reqs[(size_t)s].state = DISPATCHED;
    }
    set_queued(mr, mr.queued_requests - (int64_t)want);
  }
  void set_queued(Model& mr, int64_t n) {  // scheduler.py:304-309
    mr.queued_requests = n;
    if (n > 0) demand_models.insert(mr.id);
    else demand_models.erase(mr.id);
  }

  // ---------------------------------------------------------------- strategies
  void refresh_strategies(int m, int64_t now) {  // scheduler.py:314-329
    Model& mr = models[(size_t)m];
    mr.seq += 1;
    auto git = resident_gpus.find(m);
    if (git == resident_gpus.end() || git->second.empty() || mr.queued_requests == 0) return;
    const int64_t seq = mr.seq;
    const std::set<GKey> gpus = git->second;
    for (const GKey& k : gpus) {
      Heap& heap = strategies[k];
      for (size_t i = 0; i < mr.sizes.size(); ++i) {
        const int s = clean_head(mr, (int)i, now);
        if (s < 0) continue;
        const int64_t latest = reqs[(size_t)s].deadline - predict_infer(k.first, m, mr.sizes[i]);
        heap.push(Strategy{latest, -(int64_t)mr.sizes[i], m, seq});
      }
    }
  }

  // ---------------------------------------------------------------- Infer scheduling
  void fill_infer(int wid, int g, int64_t now) {  // scheduler.py:348-369
    Gpu& mi = gpu(wid, g);
    Heap& heap = strategies[GKey(wid, g)];
    while (mi.infer_tl.outstanding(now) < cfg.work_horizon) {
      bool dispatched = false;
      while (!heap.empty()) {
        const Strategy st = heap.top();
        heap.pop();
        Model& mr = models[(size_t)st.model];
        if (st.seq != mr.seq) continue;
        if (st.latest < now) continue;
        if (!mi.resident_or_pending((int)st.model)) continue;
        const int i = mr.index_of((int)-st.negb);
        if (try_dispatch(wid, g, mr, i, now)) {
          dispatched = true;
          break;
        }
      }
      if (!dispatched) break;
    }
  }
  std::pair<int64_t, int64_t> infer_earliest(Gpu& mi, Model& mr, int b, int64_t now) {
    // scheduler.py:420-430: (earliest allowed start, hard floor)
    int64_t ea = now + (int64_t)b * mr.input_transfer;
    int64_t floor = now;
    const int64_t rt = mi.residency_time(mr.id);
    if (mi.pending_load.count(mr.id)) floor = rt;
    if (rt > ea) ea = rt;
    return {ea, floor};
  }
  bool try_dispatch(int wid, int g, Model& mr, int i, int64_t now) {  // scheduler.py:371-418
    Gpu& mi = gpu(wid, g);
    const int m = mr.id;
    std::vector<int> members;
    int64_t min_deadline;
    if (!peek_batch(mr, i, mr.sizes[(size_t)i], now, members, min_deadline)) return false;
    int64_t dur = predict_infer(wid, m, mr.sizes[(size_t)i]);
    auto ef = infer_earliest(mi, mr, mr.sizes[(size_t)i], now);
    auto se = predict_completion(mi.infer_tl, dur, ef.first, now);
    int64_t start = se.first, end = se.second, floor = ef.second;
    if (end > min_deadline) return false;
    std::vector<int> bigger;
    int64_t bmin;
    for (size_t j = (size_t)i + 1; j < mr.sizes.size(); ++j) {
      if (!peek_batch(mr, (int)j, mr.sizes[j], now, bigger, bmin)) break;
      const int64_t dj = predict_infer(wid, m, mr.sizes[j]);
      auto efj = infer_earliest(mi, mr, mr.sizes[j], now);
      auto sej = predict_completion(mi.infer_tl, dj, efj.first, now);
      if (sej.second > bmin) break;
      i = (int)j;
      members = bigger;
      min_deadline = bmin;
      dur = dj;
      start = sej.first;
      end = sej.second;
      floor = efj.second;
    }
    take_batch(mr, i, members, now);
    update_load_stats(m);
    auto win = window_for(start, now, cfg.lead_slack, cfg.tardy_slack);
    int64_t earliest = win.first;
    if (earliest < floor) earliest = floor;
    const uint64_t id = next_action_id++;
    const int b = mr.sizes[(size_t)i];
    send_action(wid, id, K_INFER, m, earliest, win.second, &members, g, dur);
    Outstanding o;
    o.action_id = id;
    o.worker = wid;
    o.gpu = g;
    o.kind = K_INFER;
    o.model = m;
    o.reqs = members;
    o.pstart = start;
    o.pend = end;
    o.pdur = dur;
    o.batch = b;
    o.presult_end = end + (int64_t)b * mr.output_transfer;
    // (the reference registers before sending; the action record is already queued and the
    // registration emits nothing)
    register_out(std::move(o));
    mi.touch(m, now);
    arm_executor_wake(wid, g, K_INFER, now);
    refresh_strategies(m, now);
    return true;
  }

  // ---------------------------------------------------------------- load statistics
  void update_load_stats(int m) {  // scheduler.py:435-469
    Model& mr = models[(size_t)m];
    const double d = (double)(mr.queued_requests * mr.unit);
    auto old = alloc.find(m);
    if (old != alloc.end())
      for (auto& kv : old->second) gpu_load[kv.first] -= kv.second;
    auto git = resident_gpus.find(m);
    if (git == resident_gpus.end() || git->second.empty()) {
      alloc.erase(m);
      priority[m] = d;
      return;
    }
    const double eps = cfg.load_eps;
    if (d == 0.0) {
      alloc.erase(m);
      priority[m] = 0.0;
      return;
    }
    std::vector<GKey> gk(git->second.begin(), git->second.end());  // sorted(gpus)
    std::vector<double> w(gk.size()), sh(gk.size());
    for (size_t k = 0; k < gk.size(); ++k) w[k] = 1.0 / std::max(gpu_load[gk[k]], eps);
    const double total_w = py_fsum(w.data(), w.size());
    for (size_t k = 0; k < gk.size(); ++k) sh[k] = d * w[k] / total_w;
    sh.back() = d - py_fsum(sh.data(), sh.size() - 1);
    std::map<GKey, double> na;
    for (size_t k = 0; k < gk.size(); ++k) {
      na[gk[k]] = sh[k];
      gpu_load[gk[k]] += sh[k];
    }
    const double cap = (double)cfg.capacity_horizon;
    double served = 0.0;
    for (auto& kv : na) served += kv.second * cap / std::max(gpu_load[kv.first], eps);
    alloc[m] = std::move(na);
    priority[m] = d - served;
  }
  double load_priority(int m) {  // scheduler.py:471-476
    auto it = priority.find(m);
    if (it == priority.end()) {
      update_load_stats(m);
      return priority[m];
    }
    return it->second;
  }

  // ---------------------------------------------------------------- Load scheduling
  void fill_load(int wid, int g, int64_t now) {  // scheduler.py:481-502
    Gpu& mi = gpu(wid, g);
    std::set<int> skipped;
    while (mi.load_tl.outstanding(now) < cfg.work_horizon) {
      int best = -1;
      double bp = 0;
      int64_t bl = 0;
      for (int m : demand_models) {
        if (skipped.count(m) || mi.resident_or_pending(m)) continue;
        const double p = load_priority(m);
        if (p <= 0.0) continue;
        // key (p, -last_load, -m): higher wins
        const int64_t ll = -models[(size_t)m].last_load;
        if (best < 0 || p > bp || (p == bp && (ll > bl || (ll == bl && -m > -best)))) {
          best = m;
          bp = p;
          bl = ll;
        }
      }
      if (best < 0) return;
      if (!schedule_load(wid, g, best, now)) skipped.insert(best);
    }
  }
  bool load_would_help(Model& mr, int64_t load_end) {  // scheduler.py:538-544
    const int64_t cutoff = load_end + mr.seed_dur[0] + cfg.tardy_slack;
    for (int s : mr.queues[0]) {
      const Req& pr = reqs[(size_t)s];
      if (pr.state == QUEUED && (pr.size_mask & 1u) && pr.deadline >= cutoff) return true;
    }
    return false;
  }
  bool pick_victims(Gpu& mi, int64_t short_pages, std::vector<int>& out) {  // :546-562
    std::vector<std::pair<int64_t, int>> cand;
    for (auto& kv : mi.lru) {
      const int m = kv.first;
      if (mi.pending_load.count(m)) continue;
      auto inf = mi.inflight.find(m);
      if (inf != mi.inflight.end() && inf->second) continue;
      if (models[(size_t)m].queued_requests != 0) continue;
      cand.emplace_back(kv.second, m);
    }
    std::sort(cand.begin(), cand.end());
    out.clear();
    int64_t freed = 0;
    for (auto& c : cand) {
      out.push_back(c.second);
      auto r = mi.resident.find(c.second);
      freed += r == mi.resident.end() ? 0 : r->second;
      if (freed >= short_pages) return true;
    }
    return false;
  }
  bool schedule_load(int wid, int g, int m, int64_t now) {  // scheduler.py:504-536
    Gpu& mi = gpu(wid, g);
    Model& mr = models[(size_t)m];
    const int64_t load_dur = predict_load(wid, m);
    const int64_t le = predict_completion(mi.load_tl, load_dur, now, now).second;
    if (!load_would_help(mr, le)) return false;
    const int64_t pages = mr.pages;
    if (mi.pages_free < pages) {
      std::vector<int> victims;
      if (!pick_victims(mi, pages - mi.pages_free, victims)) return false;
      for (int v : victims) emit_unload(wid, g, v, now);
    }
    auto se = predict_completion(mi.load_tl, load_dur, now, now);
    auto win = window_for(se.first, now, cfg.lead_slack, cfg.tardy_slack);
    const uint64_t id = next_action_id++;
    send_action(wid, id, K_LOAD, m, win.first, win.second, nullptr, g, 0);
    mi.plan_load(m, pages, se.second, id);
    resident_gpus[m].insert(GKey(wid, g));
    Outstanding o;
    o.action_id = id;
    o.worker = wid;
    o.gpu = g;
    o.kind = K_LOAD;
    o.model = m;
    o.pstart = se.first;
    o.pend = se.second;
    o.pdur = load_dur;
    o.presult_end = se.second;
    register_out(std::move(o));
    mr.last_load = now;
    arm_executor_wake(wid, g, K_LOAD, now);
    update_load_stats(m);
    refresh_strategies(m, now);
    return true;
  }
  void emit_unload(int wid, int g, int m, int64_t now) {  // scheduler.py:564-580
    Gpu& mi = gpu(wid, g);
    const int64_t start = predict_completion(mi.load_tl, 0, now, now).first;
    const uint64_t id = next_action_id++;
    send_action(wid, id, K_UNLOAD, m, now, start + cfg.unload_tardy, nullptr, g, 0);
    mi.plan_unload(m);
    auto git = resident_gpus.find(m);
    if (git != resident_gpus.end()) git->second.erase(GKey(wid, g));
    Outstanding o;
    o.action_id = id;
    o.worker = wid;
    o.gpu = g;
    o.kind = K_UNLOAD;
    o.model = m;
    o.pstart = start;
    o.pend = start;
    o.presult_end = start;
    register_out(std::move(o));
    update_load_stats(m);
    refresh_strategies(m, now);
  }

  // ---------------------------------------------------------------- results
  void on_result(int64_t now, uint64_t aid, int status, int64_t rstart, int64_t rend,
                 int64_t ddur) {  // scheduler.py:585-607 + controller_state.py:264-285
    (void)rstart;
    auto it = outstanding.find(aid);
    if (it == outstanding.end()) return;
    Outstanding info = std::move(it->second);
    outstanding.erase(it);
    Gpu& mi = gpu(info.worker, info.gpu);
    mi.tl(info.kind).remove(aid);
    mi.bump_inflight(info.model, -1);
    if (info.kind == K_INFER) {
      if (status == R_SUCCESS) iest(info.worker, info.model, info.batch).observe(ddur);
    } else if (info.kind == K_LOAD) {
      if (status == R_SUCCESS) {
        mi.pending_load.erase(info.model);
        lest(info.worker, info.model).observe(ddur);
      } else {
        mi.rollback_load(info.model);
      }
    }
    int64_t* r = rec(EV_SINK);
    r[1] = (int64_t)info.action_id;
    r[2] = info.kind;
    r[3] = info.model;
    r[4] = info.worker;
    r[5] = info.gpu;
    r[6] = info.batch;
    r[7] = info.pstart;
    r[8] = info.pend;
    r[9] = info.pdur;
    r[10] = info.presult_end;
    if (info.kind == K_INFER) {
      if (status == R_SUCCESS) {
        for (int s : info.reqs) {
          const int64_t lat = rend - reqs[(size_t)s].arrival;
          respond(s, lat <= reqs[(size_t)s].slo ? S_OK : S_TIMEOUT, now, info.batch, lat, true);
        }
      } else {
        requeue_or_deny(info.reqs, now);
      }
    } else if (info.kind == K_LOAD && status != R_SUCCESS) {
      auto git = resident_gpus.find(info.model);
      if (git != resident_gpus.end()) git->second.erase(GKey(info.worker, info.gpu));
      update_load_stats(info.model);
      refresh_strategies(info.model, now);
    }
    for (int s : info.reqs) unref(s);
    pump(now);
  }
  void requeue_or_deny(const std::vector<int>& rs, int64_t now) {  // scheduler.py:609-625
    std::set<int> touched;  // (one model per action: the iteration order cannot matter)
    for (int s : rs) {
      Model& mr = models[(size_t)reqs[(size_t)s].model];
      reqs[(size_t)s].state = QUEUED;
      if (best_completion(mr, now) <= reqs[(size_t)s].deadline && readmit(s, mr, now)) {
        touched.insert(mr.id);
      } else {
        reqs[(size_t)s].state = DONE;
        respond(s, S_DENIED, now, 0, 0, false);
      }
    }
    for (int m : touched) {
      update_load_stats(m);
      refresh_strategies(m, now);
    }
  }
  bool readmit(int s, Model& mr, int64_t now) {  // scheduler.py:627-642 (_readmit)
    uint32_t mask = 0;
    const int64_t margin = cfg.tardy_slack;
    for (size_t i = 0; i < mr.sizes.size(); ++i) {
      if (now + mr.seed_dur[i] + margin <= reqs[(size_t)s].deadline) {
        mr.queues[i].push_back(s);
        ++reqs[(size_t)s].refs;
        mr.counts[i] += 1;
        mask |= 1u << i;
      }
    }
    if (!mask) return false;
    reqs[(size_t)s].size_mask = mask;
    reqs[(size_t)s].state = QUEUED;
    set_queued(mr, mr.queued_requests + 1);
    ++reqs[(size_t)s].refs;
    call_at(reqs[(size_t)s].deadline - margin - mr.seed_dur[0] + 1, T_DEADLINE, s);
    return true;
  }

  // ---------------------------------------------------------------- pumping
  void pump(int64_t now) {  // scheduler.py:646-652
    for (int wid : worker_order) {
      const size_t n = workers[wid].size();
      for (size_t g = 0; g < n; ++g) {
        if (gpu(wid, (int)g).infer_tl.outstanding(now) < cfg.work_horizon) fill_infer(wid, (int)g, now);
        if (gpu(wid, (int)g).load_tl.outstanding(now) < cfg.work_horizon) fill_load(wid, (int)g, now);
      }
    }
  }
  void arm_executor_wake(int wid, int g, int kind, int64_t now) {  // scheduler.py:654-669
    Timeline& tl = gpu(wid, g).tl(kind);
    const int64_t t = tl.free_at(now) - cfg.work_horizon + 1;
    if (t <= now) return;
    auto key = std::make_tuple(wid, g, kind);
    auto it = wakes.find(key);
    if (it != wakes.end() && it->second >= t) return;
    wakes[key] = t;
    call_at(t, T_WAKE, wid, g, kind);
  }
  void executor_wake(int wid, int g, int kind, int64_t now) {  // scheduler.py:671-678
    wakes.erase(std::make_tuple(wid, g, kind));
    if (kind == K_INFER) fill_infer(wid, g, now);
    else fill_load(wid, g, now);
  }
};

}  // namespace sched
}  // namespace cw

using cw::sched::Scheduler;

extern "C" {

// Model table: n models (ids 0..n-1, the catalog order); per model its batch sizes (flat,
// counts in n_sizes), exec durations (same layout), input / output / weights transfer ns and
// pages needed. cfg: work_horizon, capacity_horizon, lead_slack, tardy_slack, unload_tardy,
// estimator_window, default_slo (ns / counts), load_eps (ns, as double).
void* cw_sched_create(int32_t n, const int32_t* n_sizes, const int32_t* sizes,
                             const int64_t* exec_dur, const int64_t* input_transfer,
                             const int64_t* output_transfer, const int64_t* weights_transfer,
                             const int32_t* pages, const int64_t* cfg, double load_eps) {
  auto* s = new Scheduler();
  s->cfg = {cfg[0], cfg[1], cfg[2], cfg[3], cfg[4], cfg[5], cfg[6], load_eps};
  size_t off = 0;
  for (int m = 0; m < n; ++m) {
    cw::sched::Model mr;
    mr.id = m;
    for (int k = 0; k < n_sizes[m]; ++k) {
      mr.sizes.push_back(sizes[off + k]);
      mr.seed_dur.push_back(exec_dur[off + k]);
    }
    off += (size_t)n_sizes[m];
    mr.unit = mr.seed_dur[0];
    mr.input_transfer = input_transfer[m];
    mr.output_transfer = output_transfer[m];
    mr.weights_transfer = weights_transfer[m];
    mr.pages = pages[m];
    mr.queues.resize(mr.sizes.size());
    mr.counts.assign(mr.sizes.size(), 0);
    s->models.push_back(std::move(mr));
  }
  return s;
}

void cw_sched_destroy(void* h) { delete static_cast<Scheduler*>(h); }

static void cw_sched_begin(Scheduler* s) {
  s->ev.clear();
  s->ids.clear();
}

int cw_sched_handshake(void* h, int32_t worker_id, int32_t gpu_count, int64_t pages) {
  auto* s = static_cast<Scheduler*>(h);
  cw_sched_begin(s);
  s->on_handshake(worker_id, gpu_count, pages);
  return (int)(s->ev.size() / cw::sched::kRec);
}

int cw_sched_request(void* h, int64_t now, uint64_t request_id, int64_t model_id,
                            int64_t slo) {
  auto* s = static_cast<Scheduler*>(h);
  cw_sched_begin(s);
  s->on_request(now, request_id, model_id, slo);
  return (int)(s->ev.size() / cw::sched::kRec);
}

int cw_sched_result(void* h, int64_t now, uint64_t action_id, int32_t status,
                           int64_t start, int64_t end, int64_t device_duration) {
  auto* s = static_cast<Scheduler*>(h);
  cw_sched_begin(s);
  s->on_result(now, action_id, status, start, end, device_duration);
  return (int)(s->ev.size() / cw::sched::kRec);
}

// A timer the shim armed from an EV_TIMER record fired: kind T_DEADLINE (a = request slot)
// or T_WAKE (a, b, c = worker, gpu, action kind).
int cw_sched_timer(void* h, int64_t now, int32_t kind, int64_t a, int64_t b, int64_t c) {
  auto* s = static_cast<Scheduler*>(h);
  cw_sched_begin(s);
  if (kind == cw::sched::T_DEADLINE) s->deadline_check((int)a, now);
  else s->executor_wake((int)a, (int)b, (int)c, now);
  return (int)(s->ev.size() / cw::sched::kRec);
}

// The output of the last call: `n` records of 16 int64 and the request ids of the actions.
const int64_t* cw_sched_records(void* h) { return static_cast<Scheduler*>(h)->ev.data(); }
const uint64_t* cw_sched_ids(void* h, int64_t* n) {
  auto* s = static_cast<Scheduler*>(h);
  *n = (int64_t)s->ids.size();
  return s->ids.data();
}
int64_t cw_sched_live(void* h) { return (int64_t)static_cast<Scheduler*>(h)->live.size(); }
double cw_sched_fsum(const double* x, int64_t n) { return cw::sched::py_fsum(x, (size_t)n); }

}  // extern "C"
