// Debug probe: K-major SW128 A operand whose descriptor start is shifted by
// `t` 128-byte rows (t not a multiple of 8) inside a 1024B-aligned buffer
// written with the address-based 128B swizzle.  Checks whether UMMA needs the
// matrix-base-offset field (bits 49-51) for such starts, with K advance kk
// (0..3 = +32B steps) on top.  Usage: umma_rowshift <t> <boff 0|1> <kk>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include "../../paper_1810_02272_b200/csrc/cudadnn/ptx.cuh"
using namespace cdnn;

constexpr int ROWS = 256;

__device__ uint64_t mkdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t boff) {
  uint64_t d = 0;
  d |= uint64_t((a >> 4) & 0x3FFF); d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32; d |= uint64_t(1) << 46; d |= uint64_t(boff & 7) << 49;
  d |= uint64_t(layout & 7) << 61;
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int t, int boff, int kk) {
  extern __shared__ uint8_t raw[];
  uint8_t* pa = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* pb = pa + ROWS * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // A: ROWS x 32 fp32, K-major rows of 128B, address-based swizzle
  for (int i = tid; i < ROWS * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    const uint32_t off = r * 128 + ((((k / 4) ^ (r & 7)) & 7) << 4) + (k % 4) * 4;
    *reinterpret_cast<float*>(pa + off) = A[i];
  }
  // B: 32 x 32 fp32 K-major SW128
  for (int i = tid; i < 32 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    const uint32_t off = r * 128 + ((((k / 4) ^ (r & 7)) & 7) << 4) + (k % 4) * 4;
    *reinterpret_cast<float*>(pb + off) = B[i];
  }
  if (tid == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&tslot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tslot;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(32 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t sa = ptx::smem_u32(pa) + t * 128 + kk * 32;
    const uint64_t da = mkdesc(sa, 16, 1024, 2, boff ? ((sa >> 7) & 7) : 0);
    const uint64_t db = mkdesc(ptx::smem_u32(pb) + kk * 32, 16, 1024, 2, 0);
    ptx::mma_tf32(tm, da, db, idesc, 0u);
    ptx::mma_commit(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t r[16];
  for (int c = 0; c < 32; c += 16) {
    ptx::tmem_ld16(tm + (uint32_t(warp * 32) << 16) + c, r);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 32 + c + j] = __uint_as_float(r[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 32); }
}

int main(int argc, char** argv) {
  const int t = atoi(argv[1]), boff = atoi(argv[2]), kk = atoi(argv[3]);
  static float hA[ROWS * 32], hB[32 * 32], hD[128 * 32];
  for (int i = 0; i < ROWS * 32; ++i) hA[i] = float((i * 7) % 13) - 6.f;
  for (int i = 0; i < 32 * 32; ++i) hB[i] = float((i * 5) % 11) - 5.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  const int smem = 1024 + ROWS * 128 + 32 * 128;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, dD, t, boff, kk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("t %d boff %d kk %d: %s\n", t, boff, kk, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += double(hA[(t + m) * 32 + kk * 8 + k]) * hB[n * 32 + kk * 8 + k];
      maxerr = fmax(maxerr, fabs(s - hD[m * 32 + n]));
    }
  printf("t %3d boff %d kk %d: max err %g\n", t, boff, kk, maxerr);
  return 0;
}
