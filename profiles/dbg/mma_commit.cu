// Microbenchmark: does tcgen05.commit (one per tap in the conv kernels) or waiting on the
// ring's mbarriers stall back-to-back tcgen05.mma kind::tf32 into one accumulator?
// One CTA per SM, M = 128, K = 8; G MMAs per "tap" group; after each group a commit to
// bar[g % S]; mode 1 also waits, before group g, for the commit of group g - S (ring flow
// control done by the issuing thread itself).  Prints cycles per MMA.
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

__global__ void bench(int n, int groups, int G, int S, int mode, int fence, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[16];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(s)[i] = 0.f;
  if (tid == 0) { for (int i = 0; i < 16; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t a = ptx::smem_u32(s), b = ptx::smem_u32(s) + 48 * 1024;
    const unsigned long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (mode == 1 && g >= S) ptx::mbar_wait(&bar[g % S], uint32_t((g / S) - 1) & 1u);
      if (fence) ptx::tc_fence_after();
      for (int i = 0; i < G; ++i) {
        const uint64_t da = mkdesc(a + (i & 3) * 32 + (g & 7) * 128), db = mkdesc(b + (i & 3) * 32);
        ptx::mma_tf32_elect(tm, da, db, idesc, 1u);
      }
      if (mode >= 0) ptx::mma_commit_elect(&bar[g % S]);
    }
    __syncwarp();
    if (tid == 0) {
      // drain: commit everything to a fresh barrier... reuse bar[15] (not used when S <= 15)
      ptx::mma_commit(&bar[15]);
      ptx::mbar_wait(&bar[15], 0);
    }
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
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int total = 8192;
  for (int n : {48, 128}) {
    for (int G : {1, 4, 8, 12}) {
      for (int mode : {-1, 0, 1}) for (int fence : {1, 0}) {
        const int S = 8;
        bench<<<148, 128, smem>>>(n, total / G, G, S, mode, fence, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("N=%3d G=%2d fence=%d mode=%2d (%s): %6.1f cyc/mma\n", n, G, fence, mode,
               mode < 0 ? "no commit" : mode == 0 ? "commit/group" : "commit+ring wait S=8", double(c) / total);
      }
    }
  }
  return 0;
}
