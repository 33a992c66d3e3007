// Debug probe: 4D TMA load {W,H,C,N} box {32,1,8,1} with a given swizzle and start coords.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../../paper_1810_02272_b200/csrc/cudadnn/ptx.cuh"
using namespace cdnn;
__global__ void probe(const __grid_constant__ CUtensorMap tm, float* out, int x0, int y0, int use4d) {
  __shared__ __align__(1024) float s[32 * 8];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1); ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bar, 32 * 8 * 4);
    if (use4d)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                   :: "r"(ptx::smem_u32(s)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(ptx::smem_u32(&bar)), "r"(x0), "r"(y0), "r"(0), "r"(0) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   :: "r"(ptx::smem_u32(s)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(ptx::smem_u32(&bar)), "r"(x0), "r"(y0), "r"(0) : "memory");
    ptx::mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = s[i];
}
int main(int argc, char** argv) {
  const int sw = atoi(argv[1]), x0 = atoi(argv[2]), y0 = atoi(argv[3]), rank = atoi(argv[4]);
  const int W = 32, H = 4, C = 8;
  static float h[W * H * C], o[256];
  for (int i = 0; i < W * H * C; ++i) h[i] = float(i);
  float *d, *dout; cudaMalloc(&d, sizeof h); cudaMalloc(&dout, sizeof o);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm; memset(&tm, 0, sizeof tm);
  cuuint64_t dims[4] = {W, H, C, 1}, str[3] = {W * 4, W * H * 4, W * H * C * 4};
  cuuint32_t box[4] = {32, 1, 8, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (CUtensorMapSwizzle)sw, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
  probe<<<1, 32>>>(tm, dout, x0, y0, rank == 4);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("sw %d x0 %d y0 %d rank %d: %s\n", sw, x0, y0, rank, cudaGetErrorString(e)); return 1; }
  cudaMemcpy(o, dout, sizeof o, cudaMemcpyDeviceToHost);
  printf("sw %d x0 %d y0 %d rank %d: ok first %g %g %g %g row1 %g\n", sw, x0, y0, rank, o[0], o[1], o[2], o[3], o[32]);
  return 0;
}
