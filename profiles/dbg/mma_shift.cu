// Microbenchmark: cost of changing the A (or B) descriptor start between back-to-back
// tcgen05.mma kind::tf32 (M=128, K=8, one accumulator, no commits): every MMA at the same
// start, k8 steps only, or a start that moves by `shift` bytes every G MMAs.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "../../paper_1810_02272_b200/csrc/cudadnn/ptx.cuh"
using namespace cdnn;

__device__ uint64_t mkdesc(uint32_t a) {
  uint64_t d = 0;
  d |= uint64_t((a >> 4) & 0x3FFF); d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32; d |= uint64_t(1) << 46; d |= uint64_t(2) << 61;
  return d;
}

// which: 0 = shift A, 1 = shift B; kstep: 1 = walk the 4 k8 offsets within a group
__global__ void bench(int n, int total, int G, int shift, int which, int kstep, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(s)[i] = 0.f;
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t a = ptx::smem_u32(s), b = ptx::smem_u32(s) + 100 * 1024;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < total; ++i) {
      const int g = i / G;
      const uint32_t sh = uint32_t((g & 7) * shift);
      const uint32_t k = kstep ? uint32_t((i % G) & 3) * 32u : 0u;
      const uint64_t da = mkdesc(a + k + (which == 0 ? sh : 0)), db = mkdesc(b + k + (which == 1 ? sh : 0));
      ptx::mma_tf32_elect(tm, da, db, idesc, 1u);
    }
    __syncwarp();
    if (tid == 0) { ptx::mma_commit(&bar); ptx::mbar_wait(&bar, 0); }
    __syncwarp();
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && tid == 0) *out = t1 - t0;
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 256); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 220 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int total = 8192;
  struct Case { int G, shift, which, kstep; const char* what; };
  const Case cases[] = {
      {1, 0, 0, 0, "same A, same B every MMA"},
      {4, 0, 0, 1, "k8 walk only (4 starts)"},
      {1, 128, 0, 0, "A +128 B (1 row) every MMA"},
      {4, 128, 0, 1, "A +1 row every 4 MMAs, k8 walk"},
      {8, 128, 0, 1, "A +1 row every 8 MMAs, k8 walk"},
      {1, 1024, 0, 0, "A +1024 B (8 rows) every MMA"},
      {4, 1024, 0, 1, "A +8 rows every 4 MMAs, k8 walk"},
      {1, 4096, 0, 0, "A +4 KB every MMA"},
      {1, 128, 1, 0, "B +1 row every MMA"},
      {1, 1024, 1, 0, "B +8 rows every MMA"},
  };
  for (int n : {48, 128}) {
    for (const Case& c : cases) {
      bench<<<148, 128, smem>>>(n, total, c.G, c.shift, c.which, c.kstep, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long cyc;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      printf("N=%3d %-36s: %6.1f cyc/mma\n", n, c.what, double(cyc) / total);
    }
  }
  return 0;
}
