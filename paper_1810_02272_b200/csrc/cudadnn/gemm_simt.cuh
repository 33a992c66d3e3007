// gemm_simt.cuh — SIMT implicit-GEMM engine for the FP64 (`real = double`)
// build: the same operand views and epilogues as the tensor-core engine, on
// DFMA.  64x64 output tile per 256-thread CTA, 4x4 register micro-tile,
// 16-deep k slabs double-buffered through shared memory.  Lanes walk m, so
// the host maps the output's contiguous index to m (coalesced stores).
#pragma once

#include <cstdint>

#include "operands.cuh"

namespace cdnn {
namespace simt {

constexpr int TBM = 64, TBN = 64, TBK = 16, kThreads = 256;

template <typename T, class V, int ROWS>
__device__ __forceinline__ void load_slab(const V& v, T (*s)[ROWS + 1], int row0, int k0, int t) {
  // ROWS x TBK elements, 256 threads -> ROWS*TBK/256 each
  constexpr int PER = ROWS * TBK / kThreads;
  if (v.m_contig()) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = t + i * kThreads;
      const int r = e % ROWS, k = e / ROWS;
      s[k][r] = v.at(v.row(row0 + r), k0 + k);
    }
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int e = t + i * kThreads;
      const int r = e / TBK, k = e % TBK;
      s[k][r] = v.at(v.row(row0 + r), k0 + k);
    }
  }
}

template <typename T, class VA, class VB, class EPI>
__global__ void __launch_bounds__(kThreads)
    simt_gemm_kernel(const VA va, const VB vb, const EPI epi, int M, int N, int K, int kt_per_split) {
  __shared__ T As[2][TBK][TBM + 1];
  __shared__ T Bs[2][TBK][TBN + 1];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const int m0 = blockIdx.x * TBM, n0 = blockIdx.y * TBN;
  const int split = blockIdx.z;
  const int kt_total = (K + TBK - 1) / TBK;
  const int kt_begin = split * kt_per_split;
  const int kt_end = min(kt_total, kt_begin + kt_per_split);

  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

  int buf = 0;
  if (kt_begin < kt_end) {
    load_slab<T, VA, TBM>(va, As[0], m0, kt_begin * TBK, t);
    load_slab<T, VB, TBN>(vb, Bs[0], n0, kt_begin * TBK, t);
  }
  __syncthreads();
  for (int kt = kt_begin; kt < kt_end; ++kt) {
    if (kt + 1 < kt_end) {
      load_slab<T, VA, TBM>(va, As[buf ^ 1], m0, (kt + 1) * TBK, t);
      load_slab<T, VB, TBN>(vb, Bs[buf ^ 1], n0, (kt + 1) * TBK, t);
    }
#pragma unroll
    for (int k = 0; k < TBK; ++k) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][k][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][k][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + tx + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + ty + 16 * j;
      if (n < N) epi.store(m, n, acc[i][j], split);
    }
  }
}

// ---- small GEMMs in one launch (no split-K partials, no reduce kernel) ----------------
// The CIFAR / LeNet / PG InnerProducts have few outputs: a tiled split-K GEMM then
// needs a second (reduce) launch, which costs more than the arithmetic.
//  * dot_warp_kernel:   one warp per output (m, n); lanes stride k, fixed xor-shuffle
//                       tree (deterministic) -- few outputs, long K;
//  * dot_thread_kernel: one thread per output, sequential k -- short K.
// Output index o = n*M + m (lanes walk m: coalesced epilogue stores).
template <typename T, class VA, class VB, class EPI>
__global__ void __launch_bounds__(256) dot_warp_kernel(const VA va, const VB vb, const EPI epi, int M, int N, int K) {
  const int64_t o = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (o >= int64_t(M) * N) return;  // warp-uniform
  const int m = int(o % M), n = int(o / M);
  const auto ra = va.row(m);
  const auto rb = vb.row(n);
  T s = T(0);
#pragma unroll 8  // loads of eight k-steps in flight; the summation order is unchanged
  for (int k = lane; k < K; k += 32) s += va.at(ra, k) * vb.at(rb, k);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) epi.store(m, n, s, 0);
}

// One block (8 warps) per output (m, n) for very few outputs with long K (the PG-MLP /
// LeNet / CIFAR dW at batch 1024 rows): threads stride k, a fixed xor tree per warp, the
// eight warp sums added in warp order by thread 0 (deterministic).
template <typename T, class VA, class VB, class EPI>
__global__ void __launch_bounds__(256) dot_block_kernel(const VA va, const VB vb, const EPI epi, int M, int N, int K) {
  __shared__ T part[8];
  const int o = blockIdx.x;
  const int m = o % M, n = o / M;
  const auto ra = va.row(m);
  const auto rb = vb.row(n);
  T s = T(0);
#pragma unroll 4
  for (int k = threadIdx.x; k < K; k += 256) s += va.at(ra, k) * vb.at(rb, k);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = part[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) t += part[w];
    epi.store(m, n, t, 0);
  }
}

template <typename T, int UNROLL, class VA, class VB, class EPI>
__global__ void __launch_bounds__(256) dot_thread_kernel(const VA va, const VB vb, const EPI epi, int M, int N, int K) {
  const int64_t o = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= int64_t(M) * N) return;
  const int m = int(o % M), n = int(o / M);
  const auto ra = va.row(m);
  const auto rb = vb.row(n);
  T s = T(0);
#pragma unroll UNROLL  // few threads: latency-bound, UNROLL k-steps of loads in flight (same summation order)
  for (int k = 0; k < K; ++k) s += va.at(ra, k) * vb.at(rb, k);
  epi.store(m, n, s, 0);
}

}  // namespace simt
}  // namespace cdnn
