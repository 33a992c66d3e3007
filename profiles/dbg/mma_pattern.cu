// Microbenchmark of the tap-conv MMA issue pattern in isolation (B200):
// per "tap": 4 k8 steps x {A_hi x [B_hi|B_lo] (N=64), A_lo x B_hi (N=32)} on a
// row-shifted A start, then tcgen05.commit to an mbarrier -- 25 taps per tile.
// Variants: 0 = pattern as in conv_tap, 1 = no per-tap commit, 2 = fixed A (no shift),
// 3 = only N=32 MMAs (3 per k8, no concatenation), 4 = separate accumulators per shape,
// 5 = uniform N=64 pair into one accumulator, 6 = uniform N=64 pair into two, 7 = one N=64 per k8.  Prints cycles per MMA.
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

__global__ void bench(int variant, int tiles, unsigned long long* out, int fill) {
  extern __shared__ uint8_t raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[16];
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(s)[i] = fill ? __uint_as_float(((i * 2654435761u) & 0x007FE000u) | 0x3F000000u) * ((i & 1) ? -1.f : 1.f) : 0.f;
  if (tid == 0) { for (int i = 0; i < 16; ++i) ptx::mbar_init(&bar[i], 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&slot, 128);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = slot;
  if (tid == 0) {
    const uint32_t idesc32 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(32 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t idesc64 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(64 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t A = ptx::smem_u32(s), AL = A + 216 * 128, B = A + 2 * 216 * 128;
    const uint64_t dA = d128(A), dAl = d128(AL);
    unsigned nmma = 0, ncommit = 0;
    const unsigned long long t0 = clock64();
    for (int t = 0; t < tiles; ++t)
      for (int tap = 0; tap < 25; ++tap) {
        const int r = tap / 5, sft = tap % 5;
        const uint64_t shift = variant == 2 ? 0 : uint64_t(r * 20 + sft) * 8u;
        const uint64_t dB = d128(B + (tap % 8) * 8192);
        const uint64_t dBl = dB + (4096 >> 4);
        for (int j = 0; j < 4; ++j) {
          const uint64_t kj = uint64_t(j) * 2u;
          if (variant == 4) {  // separate accumulators for the two shapes
            ptx::mma_tf32(tm, dA + shift + kj, dB + kj, idesc64, 1u);
            ptx::mma_tf32(tm + 64, dAl + shift + kj, dB + kj, idesc32, 1u);
            nmma += 2;
          } else if (variant == 5) {  // uniform N=64 shape, same accumulator (A_lo x [B_hi|B_lo])
            ptx::mma_tf32(tm, dA + shift + kj, dB + kj, idesc64, 1u);
            ptx::mma_tf32(tm, dAl + shift + kj, dB + kj, idesc64, 1u);
            nmma += 2;
          } else if (variant == 6) {  // uniform N=64, two accumulators
            ptx::mma_tf32(tm, dA + shift + kj, dB + kj, idesc64, 1u);
            ptx::mma_tf32(tm + 64, dAl + shift + kj, dB + kj, idesc64, 1u);
            nmma += 2;
          } else if (variant == 7) {  // only A_hi x [B_hi|B_lo]: one N=64 MMA per k8
            ptx::mma_tf32(tm, dA + shift + kj, dB + kj, idesc64, 1u);
            nmma += 1;
          } else if (variant == 3) {
            ptx::mma_tf32(tm, dAl + shift + kj, dB + kj, idesc32, 1u);
            ptx::mma_tf32(tm, dA + shift + kj, dBl + kj, idesc32, 1u);
            ptx::mma_tf32(tm, dA + shift + kj, dB + kj, idesc32, 1u);
            nmma += 3;
          } else {
            ptx::mma_tf32(tm, dA + shift + kj, dB + kj, idesc64, 1u);
            ptx::mma_tf32(tm, dAl + shift + kj, dB + kj, idesc32, 1u);
            nmma += 2;
          }
        }
        if (variant != 1) { ptx::mma_commit(&bar[ncommit & 15]); ++ncommit; }
      }
    ptx::mma_commit(&bar[15]);
    // wait for everything: the last commit's phase
    ptx::mbar_wait(&bar[15], 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = nmma; }
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 128); }
}

int main(int argc, char** argv) {
  const int fill = argc > 1 ? atoi(argv[1]) : 0;
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int smem = 170 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int v = 0; v < 8; ++v) {
    bench<<<148, 128, smem>>>(v, 4, d, fill);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("v%d err %s\n", v, cudaGetErrorString(e)); return 1; }
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("variant %d: %llu MMAs, %.1f cycles/MMA, %.1f us per 25-tap tile\n", v, h[1], double(h[0]) / h[1],
           double(h[0]) / 4 / 1.9e3);
  }
  return 0;
}
