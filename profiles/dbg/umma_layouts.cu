// Debug probe: one tcgen05.mma (kind::tf32, M=128, N=32, K=8) with A in
// {K-major SW128, MN-major SW128/SW64/SW32} and B in {K-major SW128, SW32}.
// Usage: umma_layouts <a_mode 0..3> <b_mode 0..1>; prints max error.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include "../../paper_1810_02272_b200/csrc/cudadnn/ptx.cuh"
using namespace cdnn;

__device__ uint64_t mkdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((a >> 4) & 0x3FFF); d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32; d |= uint64_t(1) << 46; d |= uint64_t(layout & 7) << 61;
  return d;
}
// byte offset of 16B chunk `c` in row `r` for swizzle span `span` bytes (128/64/32)
__device__ uint32_t swz(uint32_t r, uint32_t c, uint32_t span) {
  // Swizzle<B,4,3>: XOR byte-offset bits [4,4+B) with bits [7,7+B)
  const uint32_t mask = span / 16 - 1;
  const uint32_t o = r * span + c * 16;
  return o ^ (((o >> 7) & mask) << 4);
}

__global__ void probe(const float* A, const float* B, float* D, int amode, int bmode) {
  __shared__ __align__(1024) float sa[128 * 32];
  __shared__ __align__(1024) float sb[32 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  uint8_t* pa = reinterpret_cast<uint8_t*>(sa);
  uint8_t* pb = reinterpret_cast<uint8_t*>(sb);
  // fill A (128 x 8) : A[m][k]
  for (int m = t; m < 128; m += blockDim.x)
    for (int k = 0; k < 8; ++k) {
      const float v = A[m * 8 + k];
      uint32_t off;
      if (amode == 0) {  // K-major SW128: row = m (128B), chunk = k/4
        off = (m / 8) * 1024 + swz(m % 8, k / 4, 128) + (k % 4) * 4;
      } else {  // MN-major, span bytes per row, row = k, MN atoms of span/4 elements
        const uint32_t span = amode == 1 ? 128 : amode == 2 ? 64 : 32;
        const uint32_t epr = span / 4;            // elements per row
        const uint32_t atom = m / epr, mi = m % epr;
        off = atom * (8 * span) + swz(k, mi / 4, span) + (mi % 4) * 4;
      }
      *reinterpret_cast<float*>(pa + off) = v;
    }
  // fill B (32 x 8): B[n][k], K-major
  for (int n = t; n < 32; n += blockDim.x)
    for (int k = 0; k < 8; ++k) {
      const float v = B[n * 8 + k];
      uint32_t off;
      if (bmode == 0) off = (n / 8) * 1024 + swz(n % 8, k / 4, 128) + (k % 4) * 4;   // rows of 128B (k 0..7 used)
      else off = (n / 8) * 256 + swz(n % 8, k / 4, 32) + (k % 4) * 4;               // rows of 32B
      *reinterpret_cast<float*>(pb + off) = v;
    }
  if (t == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&tslot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm = tslot;
  if (t == 0) {
    uint64_t da, db;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(32 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    if (amode == 0) da = mkdesc(ptx::smem_u32(pa), 16, 1024, 2);
    else {
      const uint32_t span = amode == 1 ? 128 : amode == 2 ? 64 : 32;
      da = mkdesc(ptx::smem_u32(pa), 8 * span, 8 * span, amode == 1 ? 2 : amode == 2 ? 4 : 6);
      idesc |= 1u << 15;
    }
    db = bmode == 0 ? mkdesc(ptx::smem_u32(pb), 16, 1024, 2) : mkdesc(ptx::smem_u32(pb), 16, 256, 6);
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
  const int am = atoi(argv[1]), bm = atoi(argv[2]);
  float hA[128 * 8], hB[32 * 8], hD[128 * 32];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = float((i * 7) % 13) - 6.f;
  for (int i = 0; i < 32 * 8; ++i) hB[i] = float((i * 5) % 11) - 5.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD, am, bm);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("amode %d bmode %d: %s\n", am, bm, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += double(hA[m * 8 + k]) * hB[n * 8 + k];
      maxerr = fmax(maxerr, fabs(s - hD[m * 32 + n]));
    }
  printf("amode %d bmode %d: max err %g\n", am, bm, maxerr);
  return 0;
}
