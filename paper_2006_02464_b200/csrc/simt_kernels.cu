// The executor's device-side window gate and timestamp kernels.
//
//   gate_kernel       K8: per-INFER window gate. Pulls the next descriptor from
//                     the host ring (mapped pinned memory), spins on %globaltimer
//                     until `earliest`, rejects if past `latest` (the reference's
//                     `now > action.latest` test, pkg/src/sloserve/worker.py:230),
//                     stamps Exec start, publishes the ActionBlock for the graph.
//   (Exec end is stamped by mk_done_kernel in mk_infer.cu: device_duration =
//   t_end - t_start, worker.py:292-299 `_exec_done`.)
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdint>
#include "cw_device.h"
#include "ptx.cuh"

namespace cw {

__global__ void gate_kernel(ActionBlock* ab, const ActionDesc* ring, uint32_t ring_mask,
                            uint64_t* ctr, ExecRecord* recs) {
  __shared__ uint64_t words[sizeof(ActionDesc) / 8];
  __shared__ uint64_t idx_s;
  if (threadIdx.x == 0) {
    uint64_t i = *ctr;
    *ctr = i + 1;
    idx_s = i;
  }
  __syncthreads();
  const uint64_t i = idx_s;
  // Parallel fetch of the descriptor over PCIe (one 8-byte word per thread).
  const volatile uint64_t* src =
      reinterpret_cast<const volatile uint64_t*>(&ring[i & ring_mask]);
  for (int w = threadIdx.x; w < (int)(sizeof(ActionDesc) / 8); w += blockDim.x) words[w] = src[w];
  __syncthreads();
  if (threadIdx.x == 0) {
    const ActionDesc* d = reinterpret_cast<const ActionDesc*>(words);
    ab->hdr = d->hdr;
    for (int k = 0; k < kMaxBatch; ++k) {
      ab->in[k] = d->in[k];
      ab->out[k] = d->out[k];
    }
    ab->batch = d->batch;
    ab->seq = i;
    ab->mk_t0 = ~0ull;
    ab->mk_t1 = 0ull;
    uint64_t t = globaltimer();
    while (t < d->earliest_gt) t = globaltimer();
    const int rej = t > d->latest_gt;
    ab->skip = rej;
    ab->t_start = t;   // the host record is written by mk_done (no PCIe fence on this path)
    ab->rejected = rej;
    (void)recs;
  }
  __syncthreads();
  griddep_trigger();  // the megakernel (PDL) may proceed past its griddepcontrol.wait
}

__global__ void out_done_kernel(ExecRecord* rec, uint64_t seq) {
  rec->t_out = globaltimer();
  __threadfence_system();
  rec->seq_out = seq;
}

// Publishes %globaltimer continuously (bounded by max_ns) for host clock calibration.
__global__ void clock_pub_kernel(volatile uint64_t* slot, uint64_t max_ns) {
  const uint64_t t0 = globaltimer();
  uint64_t t = t0;
  while (t - t0 < max_ns) {
    slot[0] = t;
    __threadfence_system();
    t = globaltimer();
  }
  slot[1] = 1;
}

// Stamp kernel for the LOAD copy stream: slot[0] = time, then slot[1] = tag.
__global__ void stamp_kernel(volatile uint64_t* slot, uint64_t tag) {
  slot[0] = globaltimer();
  __threadfence_system();
  slot[1] = tag;
}

// ------------------------------------------------------------------ launchers

void launch_gate(ActionBlock* ab, const ActionDesc* ring, uint32_t mask, uint64_t* ctr,
                 ExecRecord* recs, cudaStream_t st) {
  gate_kernel<<<1, 64, 0, st>>>(ab, ring, mask, ctr, recs);
}
void launch_out_done(ExecRecord* rec, uint64_t seq, cudaStream_t st) {
  out_done_kernel<<<1, 1, 0, st>>>(rec, seq);
}
void launch_stamp(volatile uint64_t* slot, uint64_t tag, cudaStream_t st) {
  stamp_kernel<<<1, 1, 0, st>>>(slot, tag);
}
void launch_clock_pub(volatile uint64_t* slot, uint64_t max_ns, cudaStream_t st) {
  clock_pub_kernel<<<1, 1, 0, st>>>(slot, max_ns);
}
}  // namespace cw
