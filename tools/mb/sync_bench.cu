// microbenchmark: grid-wide barrier cost (cooperative launch) vs a chain of
// dependent tiny kernels replayed from a CUDA graph with programmatic dependent launch
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void k_coop(double *buf, int n, int steps) {
  cg::grid_group g = cg::this_grid();
  for (int s = 0; s < steps; ++s) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      buf[i] = buf[(i + 1) % n] * 0.5 + 1.0;
    g.sync();
  }
}
__global__ void k_step(double *buf, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    buf[i] = buf[(i + 1) % n] * 0.5 + 1.0;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

int main() {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int n = 16384, steps = 1000;
  double *buf; cudaMalloc(&buf, sizeof(double) * n); cudaMemset(buf, 0, sizeof(double) * n);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    int grid = nsm * bpsm;
    int nn = n, ss = steps;
    void *args[] = {&buf, &nn, &ss};
    cudaLaunchCooperativeKernel((void *)k_coop, grid, 256, args, 0, st);
    cudaEventRecord(a, st);
    cudaLaunchCooperativeKernel((void *)k_coop, grid, 256, args, 0, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cooperative grid %d x 256: %.3f us per step (grid.sync + tiny step) err=%s\n", grid, ms * 1e3 / steps,
           cudaGetErrorString(cudaGetLastError()));
  }
  // graph of `steps` dependent kernels with PDL
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    int grid = nsm * bpsm;
    cudaGraph_t gr; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int s = 0; s < 200; ++s) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_step, buf, n);
    }
    cudaStreamEndCapture(st, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(a, st);
    for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("graph+PDL grid %d x 256: %.3f us per kernel err=%s\n", grid, ms * 1e3 / 1000, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
