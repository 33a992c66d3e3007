// Microbenchmark: back-to-back tcgen05.mma kind::tf32 (and kind::f16) from
// shared memory, one CTA per SM, M=128 (or 64), N in {32..256}, K=8 (tf32) /
// 16 (f16) per instruction.  Prints cycles per MMA and FMA/clk/SM.
// Also tests whether a shifted (non-1024-aligned) A start slows the MMA.
// Usage: mma_rate (no args)
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

template <int KIND>  // 0 tf32, 1 f16
__global__ void bench(int n, int m, int iters, int shift_rows, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(s)[i] = 0.f;
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (tid == 0) {
    uint32_t idesc;
    if (KIND == 0) idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
    else idesc = (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);  // f16 in, f32 acc
    const uint32_t a = ptx::smem_u32(s) + shift_rows * 128, b = ptx::smem_u32(s) + 48 * 1024;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = mkdesc(a + (i & 3) * 32), db = mkdesc(b + (i & 3) * 32);
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(1) : "memory");
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(1) : "memory");
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
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
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int m : {128, 64})
      for (int n : {32, 64, 128, 256})
        for (int sh : {0, 3}) {
          if (kind == 0) bench<0><<<148, 128, smem>>>(n, m, iters, sh, d);
          else bench<1><<<148, 128, smem>>>(n, m, iters, sh, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          unsigned long long c;
          cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
          const double cyc = double(c) / iters;
          const int k = kind == 0 ? 8 : 16;
          printf("%s M=%3d N=%3d shift=%d: %6.1f cyc/mma  %7.0f FMA/clk/SM\n", kind == 0 ? "tf32" : "f16 ", m, n, sh,
                 cyc, double(m) * n * k / cyc);
        }
  return 0;
}
