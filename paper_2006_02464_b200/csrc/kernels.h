// Host launchers for the device kernels (mk_infer.cu, simt_kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "cw_device.h"
#include "mk.h"

namespace cw {

cudaError_t configure_mk();
uint32_t mk_smem_bytes(uint32_t ring_bytes, int n_layers);
int mk_blocks_per_sm(uint32_t smem);
int mk_cluster_ctas(int csize, uint32_t smem);
cudaError_t copy_plan(const MkLayer* d_layers, int n, cudaStream_t st);  // -> constant bank
cudaError_t launch_mk(const MkArgs& a, int grid, uint32_t smem, cudaStream_t st);
void launch_mk_done(const ActionBlock* ab, uint32_t mask, ExecRecord* recs, uint32_t* gen,
                    volatile uint64_t* done, cudaStream_t st);

void launch_gate(ActionBlock* ab, const ActionDesc* ring, uint32_t mask, uint64_t* ctr,
                 ExecRecord* recs, cudaStream_t st);
void launch_out_done(ExecRecord* rec, uint64_t seq, cudaStream_t st);
void launch_stamp(volatile uint64_t* slot, uint64_t tag, cudaStream_t st);
void launch_clock_pub(volatile uint64_t* slot, uint64_t max_ns, cudaStream_t st);

}  // namespace cw
