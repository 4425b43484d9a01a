/* cw.h — C ABI of libcw, the B200-native Clockwork worker.
 *
 * Plain C types only (pointers, sizes, int64 nanoseconds); no torch types.
 * Every function returns 0 (or a non-NULL handle) on success and a negative
 * value (NULL) on failure; cw_last_error() then describes the failure.
 *
 * Reference interfaces each group replaces (paths under the reference repo):
 *
 *   cw_engine_*  The worker object driven by the controller:
 *                EmulatedWorker(...)               pkg/src/sloserve/worker.py:164-179
 *                EmulatedWorker.handshake()        worker.py:193-196
 *                EmulatedWorker.on_action(action)  worker.py:198-219
 *                send_result(ActionResult)         worker.py:345-351 (_finish)
 *                PageCache / IOCacheGauge          worker.py:63-117
 *                Executor window gate              worker.py:223-278
 *   cw_rt_*      The device work those actions stand for, which the reference
 *                only emulates: Exec (worker.py:273-277 waits exec_duration[b]),
 *                Load copy (worker.py:263-266 waits weights_transfer),
 *                Input/Output transfers (worker.py:210-214, 296-299).
 *
 * Status codes are ResultStatus (pkg/src/sloserve/protocol.py:72-77):
 *   1 SUCCESS, 2 REJECTED_TOO_LATE, 3 OUT_OF_PAGES, 4 MODEL_NOT_LOADED,
 *   5 MALFORMED_ACTION.  Action kinds (protocol.py:66-69): 1 LOAD, 2 UNLOAD, 3 INFER.
 */
#ifndef CW_H_
#define CW_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CW_ABI_VERSION 2
#define CW_MAX_BATCH 16

/* ------------------------------------------------------------------ common */
int cw_abi_version(void);
const char* cw_last_error(void);
int cw_device_count(void);

/* ------------------------------------------------------------------ model artifacts */

/* One op of an architecture's forward pass (built by the Python arch tables, arch.py).
 * Activations are NHWC bf16 workspace buffers; a conv reads channels [0, cin) of a buffer
 * whose channel stride is in_ctot and writes cout channels at channel offset out_coff of
 * a buffer of stride out_ctot (concats are convs writing disjoint slices of one buffer). */
typedef struct cw_op {
  int32_t kind; /* 0 input (NHWC4 rows), 1 conv (tensor core), 2 maxpool, 3 global avgpool,
                   4 fc, 5 im2col (fp32 images -> [M][64]), 6 BN+ReLU+2x2 avgpool,
                   7 softmax of the FC's logits (optional last op) */
  int32_t layer; /* index into the model header (conv / fc weights) */
  int32_t in_buf, out_buf, res_buf; /* workspace buffer ids, -1 = none */
  int32_t cin, cout, kh, kw, stride, pad, relu; /* pad: vertical padding */
  int32_t in_h, in_w, out_h, out_w;
  int32_t kpad;     /* stored K: kh*kw*round_up(cin, 64) (64 per tap for grouped convs) */
  int32_t pad_w;    /* horizontal padding */
  int32_t in_ctot;  /* channel stride of the input buffer */
  int32_t out_ctot; /* channel stride of the output buffer */
  int32_t out_coff; /* first output channel in that buffer */
  int32_t cout_pad; /* weight rows = MMA columns: cout rounded up to 64 */
  int32_t flags;    /* 1: grouped within 64-channel blocks, 2: BN+ReLU on the input (pre_layer) */
  int32_t pre_layer; /* header entry holding the input BatchNorm's scale/shift, -1 none */
} cw_op;

/* Where one layer's folded weights (bf16 [rows][k]), bias (fp32 [rows]) and input
 * BatchNorm scale/shift (fp32 [2][cin_pad], DenseNet pre-activation) sit in a blob;
 * -1 = absent. */
typedef struct cw_tensor_loc {
  int64_t w_off;
  int64_t b_off;
  int32_t rows;
  int32_t k;
  int64_t s_off;
} cw_tensor_loc;

/* ------------------------------------------------------------------ device runtime */
typedef struct cw_runtime cw_runtime;

cw_runtime* cw_rt_open(int device, int64_t pages_total, int64_t page_bytes, int64_t io_slots,
                       int64_t in_bytes_max, int64_t out_bytes_max);
void cw_rt_close(cw_runtime* rt);
int cw_rt_register_arch(cw_runtime* rt, int arch_id, const cw_op* ops, int n_ops, int n_layers,
                        int in_c, int in_h, int in_w, int classes, const int32_t* batches,
                        int n_batches);
int cw_rt_register_blob(cw_runtime* rt, int blob_id, int arch_id, const void* data, int64_t bytes,
                        const cw_tensor_loc* locs, int n_locs);
int cw_rt_build(cw_runtime* rt);
/* The synthetic request inputs of one arch (request id r -> image r % n). */
int cw_rt_set_input_pool(cw_runtime* rt, int arch_id, const float* images, int n,
                         int64_t bytes_per_image);
int64_t cw_rt_clock_offset(cw_runtime* rt); /* %globaltimer - CLOCK_REALTIME, ns */
int cw_rt_plan_info(cw_runtime* rt, int arch_id, int batch, int32_t* launches,
                    double* flops_per_image);

/* Blocking LOAD of a blob into the given physical pages; *copy_ns = device copy time. */
int cw_rt_load_sync(cw_runtime* rt, int blob_id, const int32_t* pages, int npages,
                    int64_t* copy_ns);
/* Blocking INFER of `batch` fp32 inputs (host) through IOCache slots 0..batch-1:
 * H2D input, the (arch, batch) graph, D2H logits. *exec_ns = device Exec time. */
int cw_rt_infer_sync(cw_runtime* rt, int arch_id, int batch, int32_t hdr_page,
                     const float* host_in, float* host_out, int64_t* exec_ns);
/* Device-resident Exec only (inputs already in slots 0..batch-1): launches n graphs
 * back to back, model i's header at hdr_pages[i]; per-launch Exec times (device
 * %globaltimer) into exec_ns[i]; *wall_ns = CUDA-event time of all n on the Exec stream. */
int cw_rt_exec_many(cw_runtime* rt, int arch_id, int batch, const int32_t* hdr_pages, int n,
                    int64_t* exec_ns, int64_t* wall_ns);
/* Closed loop (one INFER in flight): per INFER i, exec_ns[i] = device Exec time and
 * host_ns[i] = host-observed span (CLOCK_MONOTONIC from before the graph launch until the
 * host sees the completion record). */
int cw_rt_exec_closed(cw_runtime* rt, int arch_id, int batch, const int32_t* hdr_pages, int n,
                      int64_t* exec_ns, int64_t* host_ns);
/* One INFER with the megakernel's per-layer trace read back: end_ms[i] = time from
 * Exec start until plan layer i finished on its last SM; kinds[i] = layer kind
 * (1 conv, 2 input, 3 maxpool, 4 avgpool, 5 fc, 6 split-K reduce). Returns the layer count. */
int cw_rt_profile_layers(cw_runtime* rt, int arch_id, int batch, int32_t hdr_page, float* end_ms,
                         int32_t* kinds, int max_layers);
/* Raw trace of the last cw_rt_profile_layers run: [layers + 1][SMs][4] %globaltimer
 * values (0 = not reached): layer done, inputs ready (TMA producer), first accumulator
 * ready (epilogue), first tile landed (MMA); the extra last row holds per SM
 * (globaltimer, clock64) at kernel start and (globaltimer, clock64) at kernel end.
 * Returns the word count. */
int64_t cw_rt_last_trace(cw_runtime* rt, uint64_t* out, int64_t max_words);
/* Megakernel plan: 8 ints per layer (kind, conv mode, N tile, tasks, split-K,
 * k-blocks, arch op index, flags: 1 fused avgpool, 2 cluster split-K); returns the
 * layer count. */
int cw_rt_plan_layers(cw_runtime* rt, int arch_id, int batch, int32_t* out8, int max_layers);
/* Megakernel launch shape of a plan: persistent grid (CTAs) and thread-block cluster size
 * (1: no clusters; > 1: split-K layers reduce through distributed shared memory). */
int cw_rt_plan_launch(cw_runtime* rt, int arch_id, int batch, int32_t* grid, int32_t* csize);
/* Copy to/from a workspace activation buffer (parity tests of single layers). */
int cw_rt_buffer_io(cw_runtime* rt, int arch_id, int buf, void* host, int64_t bytes,
                    int to_device);
/* Exec with the window gate only (tests): returns 1 if the gate ran, and the record. */
int cw_rt_exec_window(cw_runtime* rt, int arch_id, int batch, int32_t hdr_page, int64_t earliest_gt,
                      int64_t latest_gt, int32_t* rejected, int64_t* t_start_gt, int64_t* t_end_gt);

/* ------------------------------------------------------------------ worker engine */

/* Per catalog model (ModelCatalog entry, pkg/src/sloserve/profiles.py:50-143). */
typedef struct cw_model_info {
  int32_t blob_id;  /* weights blob / arch (replicas share one blob), -1 = none (sim only) */
  int32_t arch_id;
  int32_t pages_needed; /* ceil(weights_size / page_bytes), profiles.py:109-111 */
  int32_t n_batches;
  int32_t batch_sizes[8];
  int64_t exec_ns[8];          /* profiled exec_duration[b] (sim device) */
  int64_t weights_transfer_ns; /* profiled LOAD copy time (sim device) */
  int64_t input_size, output_size;        /* bytes per request (IOCache gauge) */
  int64_t input_transfer_ns, output_transfer_ns; /* per request */
} cw_model_info;

typedef struct cw_engine_config {
  int32_t mode; /* 0 = sim (virtual clock, emulated durations), 1 = cuda */
  int32_t worker_id;
  int32_t gpu_count;
  int32_t n_models;
  int64_t pages_per_gpu;
  int64_t page_bytes;
  int64_t io_capacity; /* IOCache gauge bytes */
  int64_t epoch_ns;    /* cuda: CLOCK_REALTIME epoch shared with the controller */
  const int32_t* devices; /* cuda: device index per gpu_index */
  const cw_model_info* models;
  int64_t io_slots;        /* cuda: physical IOCache slots per GPU */
  int64_t in_bytes_max, out_bytes_max;
  /* cuda: the executor thread is pinned to this CPU (-1: not pinned) and, when
   * executor_rt_prio > 0, run SCHED_FIFO at that priority if the process may
   * ("executor threads ... pinned, real-time priority"). */
  int32_t executor_cpu;
  int32_t executor_rt_prio;
  /* cuda, gpu_count > 1: 1 = a LOAD of a model that another GPU of
   * this worker holds resident copies the weights from that GPU's pages over NVLink
   * (cudaMemcpyPeerAsync) instead of from pinned host memory (worker.py:263-266 copies
   * host -> device). Off by default: it couples the two GPUs' copy engines and HBM, against
   * the "no implicit side effects" rule. */
  int32_t peer_load;
} cw_engine_config;

typedef struct cw_action {
  uint64_t action_id;
  int32_t kind;
  uint32_t model_id;
  int32_t gpu_index;
  int32_t batch_size;
  int64_t earliest;
  int64_t latest;
  int64_t expected_duration;
  uint64_t request_ids[CW_MAX_BATCH];
} cw_action;

typedef struct cw_result {
  uint64_t action_id;
  int32_t status;
  int32_t kind;
  int64_t start;
  int64_t end;
  int64_t device_duration;
  int64_t output_ref; /* cuda INFER: handle for cw_engine_output, else -1 */
  int64_t pages_free; /* PageCache.pages_free of the action's GPU when the result was emitted */
} cw_result;

typedef struct cw_engine cw_engine;

cw_engine* cw_engine_open(const cw_engine_config* cfg);
/* cuda mode: the runtime of gpu_index (register archs/blobs on it, then cw_engine_start). */
cw_runtime* cw_engine_runtime(cw_engine* e, int gpu_index);
int cw_engine_start(cw_engine* e);
void cw_engine_close(cw_engine* e);
/* Thread-safe. cuda: processed by the engine thread; sim: delivered at virtual time `at`. */
int cw_engine_submit(cw_engine* e, const cw_action* a, int64_t at);
/* Blocks up to timeout_us for >= 1 result; returns the number written (<= max), or -1 once
 * the engine has failed (a CUDA error is fatal to the engine: it is never reported as a
 * protocol status) and every result issued before the failure has been returned. */
int cw_engine_poll(cw_engine* e, cw_result* out, int max, int64_t timeout_us);
/* 1 if a device error stopped the engine (cw_last_error() holds the first error). */
int cw_engine_failed(cw_engine* e);
/* cuda: INFER executor counters of one GPU (19 int64, see ExecStats in csrc/engine.h and
 * Engine.STAT_NAMES in worker.py); returns the count written. */
int cw_engine_stats(cw_engine* e, int gpu_index, int64_t* out, int max);
/* cuda: globaltimer-vs-CLOCK_REALTIME offset measured now minus the one calibrated at open. */
int cw_engine_clock_drift(cw_engine* e, int gpu_index, int64_t* drift_ns);
/* cuda: how the executor thread runs: *cpu = pinned CPU or -1, *rt = 1 if SCHED_FIFO. */
int cw_engine_executor_info(cw_engine* e, int32_t* cpu, int32_t* rt);
/* sim: run the virtual-time event loop until no event is left at or before `until`. */
int cw_engine_sim_run(cw_engine* e, int64_t until);
int64_t cw_engine_now(cw_engine* e);
/* sim: virtual time of the next pending event, -1 if none. */
int64_t cw_engine_next_time(cw_engine* e);
/* sim, driven by the caller's event loop (the reference SimLoop, timebase.py:55-99):
 *   cw_engine_sim_deliver   on_action at virtual time `now` (worker.py:198-219), at once;
 *   cw_engine_sim_take_new  (time, seq) of every engine event scheduled since the last call:
 *                           the caller schedules one loop callback per event, mirroring the
 *                           reference's loop.call_at (worker.py:246, 265, 276, 296);
 *   cw_engine_sim_run_to    that callback: run engine events up to (time, seq). */
int cw_engine_sim_deliver(cw_engine* e, const cw_action* a, int64_t now);
int cw_engine_sim_take_new(cw_engine* e, int64_t* times, uint64_t* seqs, int max);
int cw_engine_sim_run_to(cw_engine* e, int64_t t, uint64_t seq);
/* Page accounting of one GPU (PageCache, worker.py:63-99). resident: (model, pages) pairs. */
int cw_engine_pages(cw_engine* e, int gpu_index, int64_t* pages_free, int32_t* resident_models,
                    int32_t* resident_pages, int max_resident, int32_t* n_resident);
int64_t cw_engine_io_in_use(cw_engine* e, int gpu_index);
/* Copy the logits of a finished INFER (cw_result.output_ref) to host memory. */
int cw_engine_output(cw_engine* e, int gpu_index, int64_t output_ref, float* dst, int batch,
                     int classes);

/* ------------------------------------------------------------------ cw_wire_* / cw_net_*
 * The controller connection in native code. Replaces, per action,
 * the Python path run_worker_server -> protocol.recv/decode -> on_action and
 * _finish -> send_result -> protocol.send:
 *   cw_wire_decode_action     protocol.py:177-229 (decode, tag 2) + Action invariants :91-104
 *   cw_wire_encode_result     protocol.py:146-152 (ActionResult encode) + invariants :126-130
 *   cw_wire_encode_handshake  protocol.py:133-139 (WorkerHandshake encode)
 *   cw_net_serve              harness.py:525-575 (run_worker_server's accept-side loop)
 * Decode errors (negative): */
#define CW_WIRE_TRUNCATED (-1) /* protocol.py:53-55 TruncatedFrame */
#define CW_WIRE_BAD_TAG (-2)   /* protocol.py:57-59 UnknownMessageType */
#define CW_WIRE_INVALID (-3)   /* protocol.py:61-63 InvalidMessage */
#define CW_WIRE_RESULT_FRAME 38 /* 4-byte length prefix + 34-byte ActionResult payload */

int cw_wire_decode_action(const uint8_t* payload, int64_t n, cw_action* out);
int cw_wire_encode_result(const cw_result* r, uint8_t* out /* CW_WIRE_RESULT_FRAME bytes */);
int64_t cw_wire_encode_handshake(uint32_t worker_id, uint32_t gpu_count, uint64_t pages_total,
                                 const uint32_t* ids, int32_t n, uint8_t* out, int64_t cap);

/* One telemetry row per finished action (server.py TELEMETRY_HEADER). */
typedef struct cw_net_record {
  uint64_t action_id;
  int32_t kind;
  uint32_t model_id;
  int32_t gpu_index;
  int32_t batch_size;
  int32_t status;
  int32_t pad_;
  int64_t start, end, device_duration;
} cw_net_record;

/* Serve one connected controller socket on a started engine: send the handshake
 * frame, then read Action frames into cw_engine_submit on this thread while a native
 * writer thread turns cw_engine_poll results into ActionResult frames. Returns 0 when the
 * controller closes the connection (or sends a malformed frame), after the in-flight
 * results drained for up to 2 s. Telemetry rows go to recs (up to rec_cap). Blocking.
 * A sim-mode engine is run in wall time (virtual clock = CLOCK_REALTIME - epoch_ns). */
int cw_net_serve(cw_engine* e, int fd, const uint8_t* handshake_frame, int64_t hs_len,
                 int64_t epoch_ns, cw_net_record* recs, int64_t rec_cap, int64_t* n_recs,
                 int64_t* n_actions);

/* ------------------------------------------------------------------ cw_sched_*
 * The controller fast path: the reference's Scheduler +
 * ControllerState decision logic in native code, driven event by event by a thin shim that
 * replaces sloserve.scheduler.Scheduler behind the unmodified harness
 * (paper_2006_02464_b200/native_scheduler.py). Entry point -> reference method it replaces:
 *   cw_sched_create     Scheduler.__init__ (scheduler.py:118-140), _ModelRuntime (:80-109)
 *   cw_sched_handshake  Scheduler.on_handshake (scheduler.py:146-150)
 *   cw_sched_request    Scheduler.on_request (scheduler.py:155-168) and what it pumps
 *   cw_sched_result     Scheduler.on_result (scheduler.py:585-607), ControllerState.record_result
 *                       (controller_state.py:264-285)
 *   cw_sched_timer      Scheduler._deadline_check (scheduler.py:216-227) / _executor_wake (:671-678)
 * Every call returns the number of output records (16 x int64 each, cw_sched_records) the
 * shim replays in order: 1 action (send_action), 2 response (send_response), 3 timer
 * (loop.call_at back into cw_sched_timer), 4 action-sink row. Action request ids are in
 * cw_sched_ids. cfg[7]: work_horizon, capacity_horizon, lead_slack, tardy_slack,
 * unload_tardy, estimator_window, default_slo (SchedulerConfig, scheduler.py:51-60). */
typedef struct cw_sched cw_sched;
cw_sched* cw_sched_create(int32_t n_models, const int32_t* n_sizes, const int32_t* sizes,
                          const int64_t* exec_dur, const int64_t* input_transfer,
                          const int64_t* output_transfer, const int64_t* weights_transfer,
                          const int32_t* pages_needed, const int64_t* cfg, double load_eps);
void cw_sched_destroy(cw_sched* s);
int cw_sched_handshake(cw_sched* s, int32_t worker_id, int32_t gpu_count, int64_t pages_total);
int cw_sched_request(cw_sched* s, int64_t now, uint64_t request_id, int64_t model_id, int64_t slo);
int cw_sched_result(cw_sched* s, int64_t now, uint64_t action_id, int32_t status, int64_t start,
                    int64_t end, int64_t device_duration);
int cw_sched_timer(cw_sched* s, int64_t now, int32_t kind, int64_t a, int64_t b, int64_t c);
const int64_t* cw_sched_records(cw_sched* s);
const uint64_t* cw_sched_ids(cw_sched* s, int64_t* n);
int64_t cw_sched_live(cw_sched* s);
/* CPython 3.12 sum() of floats (Neumaier), as the load statistics use it (for tests). */
double cw_sched_fsum(const double* x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* CW_H_ */
