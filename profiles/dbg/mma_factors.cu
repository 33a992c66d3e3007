// Microbenchmark: which factor of the tap-conv issue pattern slows tcgen05.mma
// (kind::tf32, M=128, N=64, K=8, A/B K-major SW128).  One CTA per SM, 400 MMAs.
// flags: 1 = move A start by a tap row shift every 4 MMAs, 2 = move B start every
// 4 MMAs, 4 = tcgen05.commit every 4 MMAs, 8 = alternate two A buffers (hi/lo)
// every MMA, 16 = N=32 instead of 64.  Prints cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include "../../paper_1810_02272_b200/csrc/cudadnn/ptx.cuh"
using namespace cdnn;

__device__ uint64_t d128(uint32_t a) {
  uint64_t d = 0;
  d |= uint64_t((a >> 4) & 0x3FFF); d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32; d |= uint64_t(1) << 46; d |= uint64_t(2) << 61;
  return d;
}

__device__ __forceinline__ void mma_el(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_el(uint64_t* bar) {
  asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
               ::"r"(ptx::smem_u32(bar)) : "memory");
}
__global__ void bench(int flags, int n_mma, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[16];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<float*>(s)[i] = (flags & 32) ? 0.f : __uint_as_float(((i * 2654435761u) & 0x007FE000u) | 0x3F000000u);
  if (tid == 0) { for (int i = 0; i < 16; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 128);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if ((flags & 128) ? warp == 0 : tid == 0) {
    const int n = (flags & 16) ? 32 : 64;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t A = ptx::smem_u32(s), AL = A + 216 * 128, B = A + 2 * 216 * 128;
    const uint64_t dA = d128(A), dAl = d128(AL);
    unsigned ncommit = 0;
    const unsigned long long t0 = clock64();
    if (flags & 64) {  // precomputed descriptors, 4 MMAs per unrolled step, tap offsets from a table
      for (int i = 0; i < n_mma; i += 4) {
        const uint64_t sh = (flags & 1) ? uint64_t(((i >> 2) & 7) * 21) * 8u : 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) ptx::mma_tf32(tm, dA + sh + uint64_t(j) * 2u, d128(B) + uint64_t(j) * 2u, idesc, 1u);
      }
    } else
    for (int i = 0; i < n_mma; ++i) {
      const int tap = (i >> 2) % 25;
      const uint64_t shift = (flags & 1) ? uint64_t((tap / 5) * 20 + tap % 5) * 8u : 0;
      const uint64_t dB = (flags & 2) ? d128(B + (tap % 8) * 8192) : d128(B);
      const uint64_t a = ((flags & 8) && (i & 1)) ? dAl : dA;
      if (flags & 128) mma_el(tm, a + shift + uint64_t(i & 3) * 2u, dB + uint64_t(i & 3) * 2u, idesc, 1u);
      else ptx::mma_tf32(tm, a + shift + uint64_t(i & 3) * 2u, dB + uint64_t(i & 3) * 2u, idesc, 1u);
      if ((flags & 4) && (i & 3) == 3) { if (flags & 128) commit_el(&bar[ncommit & 7]); else ptx::mma_commit(&bar[ncommit & 7]); ++ncommit; }
    }
    if (flags & 128) commit_el(&bar[15]); else ptx::mma_commit(&bar[15]);
    ptx::mbar_wait(&bar[15], 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 128); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int smem = 170 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int f : {0, 7, 15, 128, 135, 143, 151}) {
    for (int n_mma : {400, 1600}) {
      bench<<<148, 128, smem>>>(f, n_mma, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("f%d err %s\n", f, cudaGetErrorString(e)); return 1; }
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("flags %2d (shift %d Bmove %d commit %d hilo %d N%d) n=%d: %.1f cycles/MMA (zero %d, simple %d)\n", f, f & 1, (f >> 1) & 1,
             (f >> 2) & 1, (f >> 3) & 1, (f & 16) ? 32 : 64, n_mma, double(h) / n_mma, (f >> 5) & 1, (f >> 6) & 1);
    }
  }
  return 0;
}
