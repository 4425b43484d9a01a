// Launch-overhead probe: chains of small kernels in a CUDA graph, with and
// without programmatic dependent launch. Profiling helper (not product).
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k_plain(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1; }
__global__ void k_pdl(int* p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
__global__ void k_pdl_chain(int** pp) {
  // three dependent loads before the wait (emulates header/bias pointer chasing)
  int* a = pp[0];
  int* b = reinterpret_cast<int**>(a)[0] ? reinterpret_cast<int*>(a) : a;
  volatile int x = b[1];
  (void)x;
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(b + 2, 1);
}

template <typename K, typename... A>
void launch(K k, int grid, int block, cudaStream_t s, bool pdl, A... a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, a...);
}

int main() {
  int* d;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  int** pp;
  cudaMalloc(&pp, 64);
  cudaMemcpy(pp, &d, 8, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int N = 50;
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid : {1, 148, 592}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < N; ++i) {
        if (mode == 0) launch(k_plain, grid, 128, s, false, d);
        if (mode == 1) launch(k_pdl, grid, 128, s, i > 0, d);
        if (mode == 2) launch(k_pdl_chain, grid, 128, s, i > 0, pp);
        if (mode == 3) launch(k_plain, grid, 128, s, false, d);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      const int R = 50;
      for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* names[] = {"graph plain", "graph pdl", "graph pdl+loads", "graph plain(again)"};
      printf("%-20s grid %4d: %.2f us per kernel\n", names[mode], grid, ms * 1000 / (R * N));
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
