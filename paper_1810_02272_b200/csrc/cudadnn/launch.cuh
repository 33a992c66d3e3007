// launch.cuh — host-side planning and launch of the two implicit-GEMM engines.
//
// run_tc:   float  -> tcgen05 TF32 engine (gemm_tc.cuh), TMA for eligible operands
// run_simt: double -> SIMT FP64 engine (gemm_simt.cuh)
// Both split K over blockIdx.z when the output has too few tiles to fill the
// 148 SMs; partial tiles go to the stream's workspace and a second kernel
// reduces them in fixed split order (deterministic, no float atomics) while
// applying the op's epilogue.
#pragma once

#include <cstring>
#include <type_traits>

#include "gemm_simt.cuh"
#include "gemm_tc.cuh"
#include "internal.hpp"

namespace cdnn {

constexpr int kNumSMs = 148;

// A request to load a K-contiguous fp32 operand with TMA.
struct TmaReq {
  const float* p = nullptr;
  int rows = 0, K = 0;
  int64_t ld = 0;
  const float* p_lo = nullptr;  // TmaSplitView: the lo copy (same layout)
};

inline bool tma_eligible(const float* p, int rows, int K, int64_t ld, int box_rows) {
  return p && (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * 4) % 16 == 0) && K >= 32 &&
         rows >= box_rows && ld >= K;
}

// Split-K reduction: block (32 m) x (8 split groups); group g sums splits
// z = g, g+8, ... (loads coalesced along m), then the 8 partials are added in
// fixed order -> deterministic.  grid = (ceil(M/32), N).
template <typename T, class EPI>
__global__ void __launch_bounds__(256) reduce_splits_kernel(const T* __restrict__ ws, int M, int N, int splits,
                                                            EPI epi) {
  __shared__ T part[8][33];
  const int mi = threadIdx.x & 31, gi = threadIdx.x >> 5;
  const int m = blockIdx.x * 32 + mi, n = blockIdx.y;
  T s = T(0);
  if (m < M) {
    const T* p = ws + int64_t(n) * M + m;
    const int64_t zs = int64_t(N) * M;
#pragma unroll 4
    for (int z = gi; z < splits; z += 8) s += p[z * zs];
  }
  part[gi][mi] = s;
  __syncthreads();
  if (gi == 0 && m < M) {
    T t = part[0][mi];
#pragma unroll
    for (int g = 1; g < 8; ++g) t += part[g][mi];
    epi.store(m, n, t, 0);
  }
}

// Few splits (<= 8): block = 32 m x 8 n, each thread adds its splits in order.
template <typename T, class EPI>
__global__ void __launch_bounds__(256) reduce_few_splits_kernel(const T* __restrict__ ws, int M, int N, int splits,
                                                                EPI epi) {
  const int m = blockIdx.x * 32 + (threadIdx.x & 31), n = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (m >= M || n >= N) return;
  const T* p = ws + int64_t(n) * M + m;
  const int64_t zs = int64_t(N) * M;
  T s = p[0];
  for (int z = 1; z < splits; ++z) s += p[z * zs];
  epi.store(m, n, s, 0);
}

template <typename T, class EPI>
void launch_reduce(Ctx* c, cudaStream_t st, const T* ws, int M, int N, int splits, const EPI& epi) {
  if (splits <= 8) {
    dim3 grid((M + 31) / 32, (N + 7) / 8);
    reduce_few_splits_kernel<T, EPI><<<grid, 256, 0, st>>>(ws, M, N, splits, epi);
    check_launch("reduce_few_splits_kernel");
    count_launch(c);
    return;
  }
  dim3 grid((M + 31) / 32, N);
  reduce_splits_kernel<T, EPI><<<grid, 256, 0, st>>>(ws, M, N, splits, epi);
  check_launch("reduce_splits_kernel");
  count_launch(c);
}

inline int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return int(std::min<int64_t>(b, int64_t(kNumSMs) * 32));
}

template <int BN, bool SPLIT, class VA, class VB, class EPI>
void launch_tc_kernel(Ctx* c, cudaStream_t st, dim3 grid, const CUtensorMap& ta,
                      const CUtensorMap& tb, const CUtensorMap& ta_lo, const CUtensorMap& tb_lo, const VA& va,
                      const VB& vb, const EPI& epi, int M, int N, int K, int kt_per_split) {
  constexpr int smem = tc::smem_bytes<BN, SPLIT>();
  auto kern = tc::tc_gemm_kernel<BN, SPLIT, VA, VB, EPI>;
  static bool attr_set[16] = {};
  if (!attr_set[c->device & 15]) {
    CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set[c->device & 15] = true;
  }
  kern<<<grid, tc::kThreads, smem, st>>>(ta, tb, ta_lo, tb_lo, va, vb, epi, M, N, K, kt_per_split);
  check_launch("tc_gemm_kernel");
  count_launch(c);
}

template <int BN, bool SPLIT, class VA, class VB, class EPI>
void run_tc_bn(Ctx* c, cudaStream_t st, Workspace& ws, const GemmPlan& pl, int M, int N, int K,
               const VA& va, const VB& vb, const EPI& epi, const TmaReq& ra, const TmaReq& rb) {
  if constexpr (SPLIT && BN == 128 && tc::is_presplit<VA>::value && tc::is_presplit<VB>::value &&
                std::is_same_v<EPI, StoreEpi<float>>) {
    // both operands pre-split and many tiles: the persistent kernel (epilogue of tile i
    // under the MMAs of tile i+1)
    const int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + BN - 1) / BN);
    if (pl.splits == 1 && tiles >= 2 * kNumSMs) {
      const CUtensorMap ta = *tmap_k_major(c, ra.p, ra.rows, ra.K, ra.ld, tc::BM);
      const CUtensorMap tb = *tmap_k_major(c, rb.p, rb.rows, rb.K, rb.ld, BN);
      const CUtensorMap tal = *tmap_k_major(c, ra.p_lo, ra.rows, ra.K, ra.ld, tc::BM);
      const CUtensorMap tbl = *tmap_k_major(c, rb.p_lo, rb.rows, rb.K, rb.ld, BN);
      constexpr int smem = tc::persist_smem_bytes<BN>();
      auto kern = tc::tc_gemm_persist_kernel<BN>;
      static bool attr_set[16] = {};
      if (!attr_set[c->device & 15]) {
        CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set[c->device & 15] = true;
      }
      kern<<<std::min(tiles, kNumSMs), tc::kThreads, smem, st>>>(ta, tb, tal, tbl, epi, M, N, K);
      check_launch("tc_gemm_persist_kernel");
      count_launch(c);
      return;
    }
  }
  CUtensorMap ta, tb, tal, tbl;
  std::memset(&ta, 0, sizeof ta);
  std::memset(&tb, 0, sizeof tb);
  std::memset(&tal, 0, sizeof tal);
  std::memset(&tbl, 0, sizeof tbl);
  if (tc::is_tma<VA>::value) ta = *tmap_k_major(c, ra.p, ra.rows, ra.K, ra.ld, tc::BM);
  if (tc::is_tma<VB>::value) tb = *tmap_k_major(c, rb.p, rb.rows, rb.K, rb.ld, BN);
  if (tc::is_presplit<VA>::value) tal = *tmap_k_major(c, ra.p_lo, ra.rows, ra.K, ra.ld, tc::BM);
  if (tc::is_presplit<VB>::value) tbl = *tmap_k_major(c, rb.p_lo, rb.rows, rb.K, rb.ld, BN);
  dim3 grid((M + tc::BM - 1) / tc::BM, (N + BN - 1) / BN, pl.splits);
  if (pl.splits == 1) {
    launch_tc_kernel<BN, SPLIT>(c, st, grid, ta, tb, tal, tbl, va, vb, epi, M, N, K, pl.kt_per_split);
  } else {
    float* wsp = static_cast<float*>(ws.get(size_t(pl.splits) * M * N * sizeof(float), c->device));
    PartialEpi<float> pe{wsp, M, N};
    launch_tc_kernel<BN, SPLIT>(c, st, grid, ta, tb, tal, tbl, va, vb, pe, M, N, K, pl.kt_per_split);
    launch_reduce<float>(c, st, wsp, M, N, pl.splits, epi);
  }
}

// Picks the tile width and the numerics mode: 3xTF32 (context default) or
// plain TF32.
template <class VA, class VB, class EPI>
void run_tc(Ctx* c, cudaStream_t st, Workspace& ws, const GemmPlan& pl, int M, int N, int K,
            const VA& va, const VB& vb, const EPI& epi, const TmaReq& ra = {}, const TmaReq& rb = {}) {
  constexpr bool any_tma = tc::is_tma<VA>::value || tc::is_tma<VB>::value;
  auto go = [&](auto split_tag) {
    constexpr bool S = decltype(split_tag)::value;
    switch (pl.bn) {
      case 32: run_tc_bn<32, S>(c, st, ws, pl, M, N, K, va, vb, epi, ra, rb); break;
      case 64: run_tc_bn<64, S>(c, st, ws, pl, M, N, K, va, vb, epi, ra, rb); break;
      default: run_tc_bn<128, S>(c, st, ws, pl, M, N, K, va, vb, epi, ra, rb); break;
    }
  };
  (void)any_tma;  // TMA operands are split in the kernel in 3xTF32 mode
  if (c->math_mode == CDNN_MATH_TF32X3) go(std::true_type{});
  else go(std::false_type{});
}

// Dense fp32 operand -> TMA when it is K-contiguous and aligned (3xTF32: the
// producers split the landed tile); the gather producers otherwise.
template <class F>
void with_operand(Ctx* c, const DenseView<float>& v, int box_rows, TmaReq& req, F&& f) {
  if (!v.mcontig && v.sk == 1 &&
      tma_eligible(v.p, v.rows, v.K, v.sr, box_rows)) {
    req = TmaReq{v.p, v.rows, v.K, v.sr};
    f(TmaView{});
  } else {
    f(v);
  }
}

template <typename T, class VA, class VB, class EPI>
void run_simt(Ctx* c, cudaStream_t st, Workspace& ws, const GemmPlan& pl, int M, int N, int K,
              const VA& va, const VB& vb, const EPI& epi) {
  dim3 grid((M + simt::TBM - 1) / simt::TBM, (N + simt::TBN - 1) / simt::TBN, pl.splits);
  if (pl.splits == 1) {
    simt::simt_gemm_kernel<T, VA, VB, EPI><<<grid, simt::kThreads, 0, st>>>(va, vb, epi, M, N, K, pl.kt_per_split);
    check_launch("simt_gemm_kernel");
    count_launch(c);
  } else {
    T* wsp = static_cast<T*>(ws.get(size_t(pl.splits) * M * N * sizeof(T), c->device));
    PartialEpi<T> pe{wsp, M, N};
    simt::simt_gemm_kernel<T, VA, VB, PartialEpi<T>><<<grid, simt::kThreads, 0, st>>>(va, vb, pe, M, N, K, pl.kt_per_split);
    check_launch("simt_gemm_kernel");
    count_launch(c);
    launch_reduce<T>(c, st, wsp, M, N, pl.splits, epi);
  }
}

}  // namespace cdnn
