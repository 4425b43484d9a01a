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
  return e->e.poll(out, max, timeout_us);
}

int cw_engine_sim_run(cw_engine* e, int64_t until) { return e->e.sim_run(until); }

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
