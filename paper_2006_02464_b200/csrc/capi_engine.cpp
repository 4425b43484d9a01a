// extern "C" surface of the worker engine (include/cw.h, cw_engine_*).
#include "../../include/cw.h"
#include "capi_util.h"
#include "engine.h"

struct cw_engine {
  cw::Engine e;
};

extern "C" {

cw_engine* cw_engine_open(const cw_engine_config* cfg) {
  auto* h = new cw_engine();
  std::string err = h->e.open(*cfg);
  if (!err.empty()) {
    cw::set_error(err);
    delete h;
    return nullptr;
  }
  return h;
}

cw_runtime* cw_engine_runtime(cw_engine* e, int gpu_index) { return e->e.runtime(gpu_index); }

int cw_engine_start(cw_engine* e) { return cw::check(e->e.start()); }

void cw_engine_close(cw_engine* e) { delete e; }

int cw_engine_submit(cw_engine* e, const cw_action* a, int64_t at) {
  if (a->batch_size < 0) return cw::fail("negative batch size");
  return e->e.submit(*a, at);
}

int cw_engine_poll(cw_engine* e, cw_result* out, int max, int64_t timeout_us) {
  return e->e.poll(out, max, timeout_us);  // -1: the engine failed (cw_last_error says why)
}

int cw_engine_sim_run(cw_engine* e, int64_t until) { return e->e.sim_run(until); }

int cw_engine_sim_deliver(cw_engine* e, const cw_action* a, int64_t now) {
  if (a->batch_size < 0) return cw::fail("negative batch size");
  return e->e.sim_deliver(*a, now) == 0 ? 0 : cw::fail("sim_deliver: not a sim engine");
}

int cw_engine_sim_run_to(cw_engine* e, int64_t t, uint64_t seq) { return e->e.sim_run_to(t, seq); }

int cw_engine_sim_take_new(cw_engine* e, int64_t* times, uint64_t* seqs, int max) {
  return e->e.sim_take_new(times, seqs, max);
}

int cw_engine_failed(cw_engine* e) { return e->e.failed() ? 1 : 0; }

int cw_engine_stats(cw_engine* e, int gpu_index, int64_t* out, int max) {
  const int n = e->e.stats(gpu_index, out, max);
  return n < 0 ? cw::fail("bad gpu index") : n;
}

int cw_engine_clock_drift(cw_engine* e, int gpu_index, int64_t* drift_ns) {
  cw_runtime* rt = e->e.runtime(gpu_index);
  if (!rt) return cw::fail("no device runtime");
  int64_t off = 0;
  std::string err = rt->rt.measure_clock_offset(&off);
  if (!err.empty()) return cw::fail(err);
  *drift_ns = off - rt->rt.clock_offset();
  return 0;
}

int cw_engine_executor_info(cw_engine* e, int32_t* cpu, int32_t* rt) {
  e->e.executor_info(cpu, rt);
  return 0;
}

int64_t cw_engine_now(cw_engine* e) { return e->e.now(); }

int64_t cw_engine_next_time(cw_engine* e) { return e->e.next_event_time(); }

int cw_engine_pages(cw_engine* e, int gpu_index, int64_t* pages_free, int32_t* resident_models,
                    int32_t* resident_pages, int max_resident, int32_t* n_resident) {
  return e->e.pages(gpu_index, pages_free, resident_models, resident_pages, max_resident,
                    n_resident);
}

int64_t cw_engine_io_in_use(cw_engine* e, int gpu_index) { return e->e.io_in_use(gpu_index); }

int cw_engine_output(cw_engine* e, int gpu_index, int64_t output_ref, float* dst, int batch,
                     int classes) {
  return e->e.output(gpu_index, output_ref, dst, batch, classes) == 0 ? 0
                                                                       : cw::fail("output gone");
}

}  // extern "C"
