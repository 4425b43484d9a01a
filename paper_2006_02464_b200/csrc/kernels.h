// Host launchers for the device kernels (conv_tc.cu, simt_kernels.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "cw_device.h"

namespace cw {

cudaError_t configure_conv_tc();
cudaError_t configure_simt();
uint32_t conv_smem_bytes(int bn, int stages);
cudaError_t launch_conv_tc(const CUtensorMap& tmap_a, const ConvArgs& a, int bn, int m_tiles,
                           cudaStream_t st, bool pdl);

void launch_gate(ActionBlock* ab, const ActionDesc* ring, uint32_t mask, uint64_t* ctr,
                 ExecRecord* recs, cudaStream_t st);
void launch_exec_done(const ActionBlock* ab, uint32_t mask, ExecRecord* recs, cudaStream_t st);
void launch_out_done(ExecRecord* rec, uint64_t seq, cudaStream_t st);
void launch_stamp(volatile uint64_t* slot, uint64_t tag, cudaStream_t st);
void launch_clock_pub(volatile uint64_t* slot, uint64_t max_ns, cudaStream_t st);
void launch_stem_im2col(const ActionBlock* ab, void* a, int batch, int H, int W, int OH, int OW,
                        int kpad, cudaStream_t st);
void launch_maxpool(const ActionBlock* ab, const void* in, void* out, int batch, int H, int W,
                    int C, int OH, int OW, cudaStream_t st);
void launch_avgpool(const ActionBlock* ab, const void* in, float* pooled, int batch, int HW, int C,
                    cudaStream_t st);
void launch_fc(const ActionBlock* ab, const float* pooled, int layer, int batch, int C, int classes,
               cudaStream_t st);

}  // namespace cw
