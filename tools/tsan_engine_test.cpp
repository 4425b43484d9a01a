// ThreadSanitizer run of the worker's host threads (SURVEY §5 "TSAN on the C++ executor"):
// the native serving loop (csrc/net.cpp: reader thread -> engine, writer thread polling
// results -> socket) driving the sim-mode engine in wall time, while a third thread reads
// the page / IOCache state through the C ABI. Built and run by tools/tsan.sh (host code
// compiled with -fsanitize=thread); prints "tsan engine test ok" when every action got
// its result.
#include <sys/socket.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <thread>
#include <vector>

#include "../include/cw.h"

static int64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

template <typename T>
static uint8_t* put(uint8_t* p, T v) {
  std::memcpy(p, &v, sizeof(T));
  return p + sizeof(T);
}

int main() {
  constexpr int kModels = 6, kActions = 3000;
  std::vector<cw_model_info> models(kModels);
  for (int m = 0; m < kModels; ++m) {
    cw_model_info& mi = models[m];
    std::memset(&mi, 0, sizeof(mi));
    mi.blob_id = -1;
    mi.pages_needed = 7;
    mi.n_batches = 3;
    const int bs[3] = {1, 2, 4};
    for (int i = 0; i < 3; ++i) {
      mi.batch_sizes[i] = bs[i];
      mi.exec_ns[i] = 20000 * (i + 1);
    }
    mi.weights_transfer_ns = 50000;
    mi.input_size = 602000;
    mi.output_size = 4000;
    mi.input_transfer_ns = 2000;
    mi.output_transfer_ns = 1000;
  }
  cw_engine_config cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.mode = 0;
  cfg.gpu_count = 2;
  cfg.n_models = kModels;
  cfg.pages_per_gpu = 20;
  cfg.page_bytes = 16 << 20;
  cfg.io_capacity = 512LL << 20;
  cfg.models = models.data();
  cfg.executor_cpu = -1;
  cw_engine* e = cw_engine_open(&cfg);
  if (!e || cw_engine_start(e) != 0) {
    std::printf("open failed: %s\n", cw_last_error());
    return 1;
  }
  int sv[2];
  if (socketpair(AF_UNIX, SOCK_STREAM, 0, sv) != 0) return 1;
  const int64_t epoch = now_ns();
  uint32_t ids[kModels];
  for (int m = 0; m < kModels; ++m) ids[m] = m;
  uint8_t hs[256];
  const int64_t hs_len = cw_wire_encode_handshake(0, 2, 20, ids, kModels, hs, sizeof(hs));
  std::vector<cw_net_record> recs(kActions + 16);
  int64_t n_recs = 0, n_act = 0;
  std::atomic<bool> done{false};
  std::thread server([&] {
    cw_net_serve(e, sv[0], hs, hs_len, epoch, recs.data(), (int64_t)recs.size(), &n_recs, &n_act);
  });
  std::thread observer([&] {  // concurrent state reads through the ABI
    int64_t free_pages = 0;
    int32_t n = 0, ms[kModels], ps[kModels];
    while (!done) {
      cw_engine_pages(e, 0, &free_pages, ms, ps, kModels, &n);
      (void)cw_engine_io_in_use(e, 1);
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  });
  // client: read the handshake, then send actions while reading results
  uint8_t buf[4096];
  if (recv(sv[1], buf, (size_t)hs_len, MSG_WAITALL) != hs_len) return 1;
  std::atomic<int> got{0};
  std::thread reader([&] {
    uint8_t frame[CW_WIRE_RESULT_FRAME];
    while (got < kActions) {
      const ssize_t k = recv(sv[1], frame, sizeof(frame), MSG_WAITALL);
      if (k != (ssize_t)sizeof(frame)) break;
      ++got;
    }
  });
  unsigned seed = 12345;
  auto rnd = [&] { return seed = seed * 1103515245u + 12345u, (seed >> 8); };
  for (int i = 0; i < kActions; ++i) {
    uint8_t* p = buf + 4;
    const int r = (int)(rnd() % 10);
    const int kind = r < 6 ? 3 : (r < 8 ? 1 : 2);
    const int64_t t = now_ns() - epoch;
    p = put<uint8_t>(p, 2);
    p = put<uint64_t>(p, (uint64_t)i + 1);
    p = put<uint8_t>(p, (uint8_t)kind);
    p = put<uint32_t>(p, rnd() % kModels);
    p = put<uint16_t>(p, (uint16_t)(rnd() % 2));
    p = put<int64_t>(p, t);
    p = put<int64_t>(p, t + 50000000);
    const int b = kind == 3 ? 1 << (rnd() % 3) : 0;
    p = put<uint16_t>(p, (uint16_t)b);
    for (int j = 0; j < b; ++j) p = put<uint64_t>(p, (uint64_t)(i * 16 + j));
    if (kind == 3) p = put<int64_t>(p, 0);
    put<uint32_t>(buf, (uint32_t)(p - buf - 4));
    if (send(sv[1], buf, (size_t)(p - buf), MSG_NOSIGNAL) <= 0) return 1;
    if (i % 64 == 0) std::this_thread::sleep_for(std::chrono::microseconds(300));
  }
  const int64_t deadline = now_ns() + 20000000000LL;
  while (got < kActions && now_ns() < deadline)
    std::this_thread::sleep_for(std::chrono::milliseconds(5));
  shutdown(sv[1], SHUT_WR);
  server.join();
  reader.join();
  done = true;
  observer.join();
  close(sv[0]);
  close(sv[1]);
  cw_engine_close(e);
  std::printf("results %d of %d, actions %lld, telemetry rows %lld\n", got.load(), kActions,
              (long long)n_act, (long long)n_recs);
  if (got.load() != kActions) return 1;
  std::printf("tsan engine test ok\n");
  return 0;
}
