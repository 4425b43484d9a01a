// Native controller connection: the wire codec and the serving loop of the worker process,
// so an action goes socket -> decode -> cw_engine_submit and a result goes cw_engine_poll ->
// encode -> socket without the Python interpreter (the Python
// recv/send path of run_worker_server is the jitter behind late rejections).
//
// Byte format: reference pkg/src/sloserve/protocol.py:1-32 (u32 LE payload length, u8 tag,
// fixed-width LE fields, no padding), restated field by field in wire.py of this package;
// the decode-time invariants follow protocol.py:86-164 (Action.__post_init__ :91-104,
// frame cap :41). Serving contract: reference harness.py:525-575 (handshake first, then
// Action frames in, ActionResult frames out; on EOF the in-flight results drain for up to
// 2 s, as in server.py).
#include <sys/socket.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/cw.h"
#include "capi_util.h"

namespace {

constexpr uint32_t kMaxFrame = 64u << 20;  // protocol.py:41

template <typename T>
T rd(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));  // little-endian host (x86-64 / aarch64)
  return v;
}
template <typename T>
uint8_t* wr(uint8_t* p, T v) {
  std::memcpy(p, &v, sizeof(T));
  return p + sizeof(T);
}

bool send_all(int fd, const uint8_t* p, size_t n) {
  while (n) {
    const ssize_t k = ::send(fd, p, n, MSG_NOSIGNAL);
    if (k < 0 && errno == EINTR) continue;
    if (k <= 0) return false;
    p += k;
    n -= (size_t)k;
  }
  return true;
}

// 1 = got n bytes, 0 = clean EOF before the first byte, -1 = error / EOF mid-read
int recv_all(int fd, uint8_t* p, size_t n) {
  size_t got = 0;
  while (got < n) {
    const ssize_t k = ::recv(fd, p + got, n - got, 0);
    if (k < 0 && errno == EINTR) continue;
    if (k == 0) return got == 0 ? 0 : -1;
    if (k < 0) return -1;
    got += (size_t)k;
  }
  return 1;
}

}  // namespace

extern "C" {

// Action payload (tag 2): u64 id, u8 kind, u32 model, u16 gpu, i64 earliest, i64 latest,
// u16 n, u64 x n request ids, [i64 expected_duration iff INFER].
int cw_wire_decode_action(const uint8_t* p, int64_t n, cw_action* out) {
  constexpr int64_t kHead = 1 + 8 + 1 + 4 + 2 + 8 + 8 + 2;
  if (n < 1) return CW_WIRE_TRUNCATED;
  if (p[0] != 2) return CW_WIRE_BAD_TAG;
  if (n < kHead) return CW_WIRE_TRUNCATED;
  std::memset(out, 0, sizeof(*out));
  out->action_id = rd<uint64_t>(p + 1);
  const int kind = p[9];
  out->model_id = rd<uint32_t>(p + 10);
  out->gpu_index = rd<uint16_t>(p + 14);
  out->earliest = rd<int64_t>(p + 16);
  out->latest = rd<int64_t>(p + 24);
  const int cnt = rd<uint16_t>(p + 32);
  if (kind < 1 || kind > 3) return CW_WIRE_INVALID;  // ActionKind (protocol.py:66-69)
  int64_t pos = kHead;
  if (pos + 8LL * cnt > n) return CW_WIRE_TRUNCATED;
  for (int i = 0; i < cnt; ++i)
    if (i < CW_MAX_BATCH) out->request_ids[i] = rd<uint64_t>(p + pos + 8 * i);
  pos += 8LL * cnt;
  if (kind == 3) {
    if (pos + 8 > n) return CW_WIRE_TRUNCATED;
    out->expected_duration = rd<int64_t>(p + pos);
    pos += 8;
  }
  if (pos != n) return CW_WIRE_INVALID;  // trailing bytes
  out->kind = kind;
  out->batch_size = cnt;
  // Action.__post_init__ (protocol.py:91-104)
  if (out->earliest > out->latest) return CW_WIRE_INVALID;
  if (kind == 3) {
    if (cnt == 0 || out->expected_duration < 0) return CW_WIRE_INVALID;
  } else if (cnt != 0) {
    return CW_WIRE_INVALID;
  }
  return 0;
}

// ActionResult frame: u32 len = 34, u8 3, u64 id, u8 status, i64 start, i64 end,
// i64 device_duration. Non-success carries device_duration 0 (protocol.py:126-130).
int cw_wire_encode_result(const cw_result* r, uint8_t* out) {
  if (r->status < 1 || r->status > 5) return CW_WIRE_INVALID;
  if (r->status == 1 ? r->end < r->start : r->device_duration != 0) return CW_WIRE_INVALID;
  uint8_t* p = wr<uint32_t>(out, CW_WIRE_RESULT_FRAME - 4);
  p = wr<uint8_t>(p, 3);
  p = wr<uint64_t>(p, r->action_id);
  p = wr<uint8_t>(p, (uint8_t)r->status);
  p = wr<int64_t>(p, r->start);
  p = wr<int64_t>(p, r->end);
  wr<int64_t>(p, r->device_duration);
  return CW_WIRE_RESULT_FRAME;
}

// WorkerHandshake frame: u32 len, u8 1, u32 worker_id, u32 gpu_count, u64 pages_total,
// u32 n, u32 x n model ids. Returns the frame length, or a negative error.
int64_t cw_wire_encode_handshake(uint32_t worker_id, uint32_t gpu_count, uint64_t pages_total,
                                 const uint32_t* ids, int32_t n, uint8_t* out, int64_t cap) {
  if (gpu_count < 1 || pages_total == 0 || n < 0) return CW_WIRE_INVALID;
  const int64_t len = 4 + 1 + 4 + 4 + 8 + 4 + 4LL * n;
  if (cap < len) return CW_WIRE_TRUNCATED;
  uint8_t* p = wr<uint32_t>(out, (uint32_t)(len - 4));
  p = wr<uint8_t>(p, 1);
  p = wr<uint32_t>(p, worker_id);
  p = wr<uint32_t>(p, gpu_count);
  p = wr<uint64_t>(p, pages_total);
  p = wr<uint32_t>(p, (uint32_t)n);
  for (int i = 0; i < n; ++i) p = wr<uint32_t>(p, ids[i]);
  return len;
}

int cw_net_serve(cw_engine* e, int fd, const uint8_t* handshake, int64_t hs_len,
                 int64_t epoch_ns, cw_net_record* recs, int64_t rec_cap, int64_t* n_recs,
                 int64_t* n_actions) {
  if (!e || fd < 0) return cw::fail("cw_net_serve: bad engine or socket");
  // A sim-mode engine (virtual clock, emulated durations) runs in wall time here: its event
  // loop is advanced to CLOCK_REALTIME - epoch by the writer thread, and every engine call
  // is serialised (the sim engine is single-threaded), as WallLoop does for server.py.
  const bool sim = cw_engine_sim_run(e, 0) >= 0;
  std::mutex sim_mu;
  auto wall = [epoch_ns] {
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec - epoch_ns;
  };
  if (!send_all(fd, handshake, (size_t)hs_len)) return cw::fail("cw_net_serve: handshake send");
  struct Info {
    int32_t kind, gpu, batch;
    uint32_t model;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::unordered_map<uint64_t, Info> inflight;  // action id -> telemetry fields
  int64_t pending = 0, actions = 0, nrec = 0;
  std::atomic<bool> reading{true}, sock_ok{true}, engine_failed{false};

  // writer: engine results -> ActionResult frames (one send per poll batch)
  std::thread writer([&] {
    std::vector<cw_result> res(64);
    std::vector<uint8_t> buf;
    for (;;) {
      int k;
      if (sim) {
        {
          std::lock_guard<std::mutex> g(sim_mu);
          cw_engine_sim_run(e, wall());
        }
        // (woken at once by results the reader's own sim_run produced)
        k = cw_engine_poll(e, res.data(), (int)res.size(), 50);
      } else {
        k = cw_engine_poll(e, res.data(), (int)res.size(), 20000);
      }
      if (k < 0) {  // a device error stopped the engine: drop the controller connection
        engine_failed = true;
        shutdown(fd, SHUT_RDWR);
        break;
      }
      if (k > 0) {
        buf.clear();
        for (int i = 0; i < k; ++i) {
          uint8_t frame[CW_WIRE_RESULT_FRAME];
          if (cw_wire_encode_result(&res[i], frame) > 0)
            buf.insert(buf.end(), frame, frame + CW_WIRE_RESULT_FRAME);
        }
        if (sock_ok && !buf.empty() && !send_all(fd, buf.data(), buf.size())) sock_ok = false;
        std::lock_guard<std::mutex> g(mu);
        for (int i = 0; i < k; ++i) {
          auto it = inflight.find(res[i].action_id);
          if (it != inflight.end()) {
            if (recs && nrec < rec_cap) {
              cw_net_record& r = recs[nrec++];
              r.action_id = res[i].action_id;
              r.kind = it->second.kind;
              r.model_id = it->second.model;
              r.gpu_index = it->second.gpu;
              r.batch_size = it->second.batch;
              r.status = res[i].status;
              r.pad_ = 0;
              r.start = res[i].start;
              r.end = res[i].end;
              r.device_duration = res[i].device_duration;
            }
            inflight.erase(it);
          }
          --pending;
        }
        cv.notify_all();
      }
      std::lock_guard<std::mutex> g(mu);
      if (!reading && (pending <= 0 || !sock_ok)) break;
    }
  });

  // reader: Action frames -> engine
  std::vector<uint8_t> payload;
  int rc = 0;
  for (;;) {
    uint8_t hdr[4];
    const int h = recv_all(fd, hdr, 4);
    if (h <= 0) break;  // EOF / reset: the controller went away
    const uint32_t len = rd<uint32_t>(hdr);
    if (len > kMaxFrame) break;
    payload.resize(len);
    if (len && recv_all(fd, payload.data(), len) != 1) break;
    cw_action a;
    if (cw_wire_decode_action(payload.data(), (int64_t)len, &a) != 0) break;  // wire error
    {
      std::lock_guard<std::mutex> g(mu);
      inflight[a.action_id] = Info{a.kind, a.gpu_index, a.batch_size, a.model_id};
      ++pending;
      ++actions;
    }
    int src;
    if (sim) {
      std::lock_guard<std::mutex> g(sim_mu);
      const int64_t t = wall();
      src = cw_engine_sim_deliver(e, &a, t);  // on_action at once, as the Python path does
      cw_engine_sim_run(e, t);
    } else {
      src = cw_engine_submit(e, &a, 0);
    }
    if (src != 0) {
      rc = -1;
      break;
    }
  }
  {
    // drain the in-flight results for up to 2 s (server.py / harness.py:567-575)
    std::unique_lock<std::mutex> g(mu);
    reading = false;
    cv.wait_for(g, std::chrono::seconds(2), [&] { return pending <= 0; });
    pending = 0;  // give up on the rest: the writer exits at its next poll
  }
  writer.join();
  if (n_recs) *n_recs = nrec;
  if (n_actions) *n_actions = actions;
  if (engine_failed) return -1;  // cw_last_error() holds the engine's device error
  return rc == 0 ? 0 : cw::fail("cw_net_serve: engine submit failed");
}

}  // extern "C"
