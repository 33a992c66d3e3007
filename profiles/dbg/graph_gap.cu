// Per-kernel cost of a chain of dependent small kernels replayed from a CUDA
// graph on B200, with and without programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(float* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0001f + 1.f;
}
__global__ void k_pdl(float* p, int n) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0001f + 1.f;
}

int main() {
  const int n = 148 * 256, chain = 50;
  float* p;
  cudaMalloc(&p, n * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int mode = 0; mode < 2; ++mode) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < chain; ++i) {
      if (mode == 0) {
        k_plain<<<148, 256, 0, s>>>(p, n);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = 148; cfg.blockDim = 256; cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_pdl, p, n);
      }
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.2f us per kernel in a %d-kernel graph\n", mode ? "PDL" : "plain", 1000.f * ms / (20 * chain), chain);
  }
  return 0;
}
