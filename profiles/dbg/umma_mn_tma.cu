// Debug probe: MN-major tf32 A loaded by TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
// one tcgen05.mma (M=128, N=32, K=8) with descriptor layout type / LBO / SBO from argv.
// Usage: umma_mn_tma <tma_swizzle 0..6> <layout 0..7> <lbo> <sbo>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1810_02272_b200/csrc/cudadnn/ptx.cuh"
using namespace cdnn;

__device__ uint64_t mkdesc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((a >> 4) & 0x3FFF); d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32; d |= uint64_t(1) << 46; d |= uint64_t(layout & 7) << 61;
  return d;
}
__device__ uint32_t swz128(uint32_t r, uint32_t c) { const uint32_t o = r * 128 + c * 16; return o ^ (((o >> 7) & 7) << 4); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, const float* B, float* D, uint32_t layout, uint32_t lbo, uint32_t sbo) {
  __shared__ __align__(1024) float sa[128 * 8];
  __shared__ __align__(1024) float sb[32 * 32];
  __shared__ uint64_t bar, tbar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  uint8_t* pb = reinterpret_cast<uint8_t*>(sb);
  for (int n = t; n < 32; n += blockDim.x)
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float*>(pb + (n / 8) * 1024 + swz128(n % 8, k / 4) + (k % 4) * 4) = B[n * 8 + k];
  if (t == 0) { ptx::mbar_init(&bar, 1); ptx::mbar_init(&tbar, 1); ptx::fence_mbar_init(); }
  if (warp == 0) ptx::tmem_alloc(&tslot, 32);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tm_addr = tslot;
  if (t == 0) {
    ptx::mbar_arrive_expect_tx(&tbar, 128 * 8 * 4);
    for (int a = 0; a < 4; ++a) ptx::tma_load_2d(reinterpret_cast<uint8_t*>(sa) + a * 1024, &tm, &tbar, a * 32, 0);
    ptx::mbar_wait(&tbar, 0);
    ptx::tc_fence_after();
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (uint32_t(32 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t da = mkdesc(ptx::smem_u32(sa), lbo, sbo, layout);
    const uint64_t db = mkdesc(ptx::smem_u32(sb), 16, 1024, 2);
    ptx::mma_tf32(tm_addr, da, db, idesc, 0u);
    ptx::mma_commit(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  uint32_t r[16];
  for (int c = 0; c < 32; c += 16) {
    ptx::tmem_ld16(tm_addr + (uint32_t(warp * 32) << 16) + c, r);
    ptx::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 32 + c + j] = __uint_as_float(r[j]);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm_addr, 32); }
}

int main(int argc, char** argv) {
  const int sw = atoi(argv[1]); const uint32_t layout = atoi(argv[2]), lbo = atoi(argv[3]), sbo = atoi(argv[4]);
  static float hAg[8 * 128], hB[32 * 8], hD[128 * 32];   // A stored MN-major: Ag[k][m]
  for (int k = 0; k < 8; ++k) for (int m = 0; m < 128; ++m) hAg[k * 128 + m] = float((m * 7 + k * 3) % 13) - 6.f;
  for (int i = 0; i < 32 * 8; ++i) hB[i] = float((i * 5) % 11) - 5.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hAg); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hAg, sizeof hAg, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm; memset(&tm, 0, sizeof tm);
  cuuint64_t dims[2] = {128, 8}, str[1] = {128 * 4}; cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (CUtensorMapSwizzle)sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
  probe<<<1, 128>>>(tm, dB, dD, layout, lbo, sbo);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("sw %d layout %u lbo %u sbo %u: %s\n", sw, layout, lbo, sbo, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) {
    double s = 0; for (int k = 0; k < 8; ++k) s += double(hAg[k * 128 + m]) * hB[n * 8 + k];
    maxerr = fmax(maxerr, fabs(s - hD[m * 32 + n]));
  }
  printf("sw %d layout %u lbo %u sbo %u: max err %g\n", sw, layout, lbo, sbo, maxerr);
  return 0;
}
