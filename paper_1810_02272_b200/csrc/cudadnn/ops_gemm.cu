// ops_gemm.cu — kernels::gemm (backend.cpp:169-197) and the InnerProduct layer
// (layers.cpp:124-169) on the implicit-GEMM engines.
//
// Orientation: the engines store D with lanes walking m, so every op maps the
// output's contiguous index to m:
//   gemm     C[i][j]   (row-major)      m = j, n = i
//   ip fwd   top[b][o] = x W^T + bias  m = o, n = b, K = input_dim
//   ip wgrad dW[o][k] += dY^T X        m = k, n = o, K = batch
//   ip dgrad dX[b][k]  = dY W           m = k, n = b, K = num_output
#include <string>

#include "launch.cuh"

namespace cdnn {

// fp32 GEMMs up to this many multiply-adds take the SIMT engine
constexpr int64_t kSimtMaxMacs = int64_t(1) << 26;

GemmPlan plan_tc(int M, int N, int K) {
  GemmPlan p;
  p.bn = N <= 32 ? 32 : (N <= 64 ? 64 : 128);
  const int tiles = ((M + tc::BM - 1) / tc::BM) * ((N + p.bn - 1) / p.bn);
  const int kt = (K + tc::BK - 1) / tc::BK;
  int splits = 1;
  // resident CTA slots: one per SM, two for the 32-wide tiles (tc::ctas_per_sm)
  const int slots = kNumSMs * (p.bn == 32 ? tc::ctas_per_sm<32, true>() : 1);
  if (tiles < slots && kt >= 8) {
    // pick the split count with the best whole-wave occupancy of the resident
    // slots up to ~2 waves, fewest splits on ties
    const int smax = std::max(1, std::min(kt / 4, (2 * slots + tiles - 1) / tiles));
    double best = 0.0;
    for (int sp = 1; sp <= smax; ++sp) {
      const int ctas = tiles * sp, waves = (ctas + slots - 1) / slots;
      const double eff = double(ctas) / (double(waves) * slots);
      if (eff > best + 1e-9) { best = eff; splits = sp; }
    }
  }
  p.kt_per_split = (kt + splits - 1) / splits;
  p.splits = (kt + p.kt_per_split - 1) / p.kt_per_split;
  return p;
}

GemmPlan plan_simt(int M, int N, int K) {
  GemmPlan p;
  p.bn = simt::TBN;
  const int tiles = ((M + simt::TBM - 1) / simt::TBM) * ((N + simt::TBN - 1) / simt::TBN);
  const int kt = (K + simt::TBK - 1) / simt::TBK;
  int splits = 1;
  if (tiles < 2 * kNumSMs && kt >= 4) {  // small grids: split K down to 2 slabs per CTA
    splits = std::min(kt / 2, (2 * kNumSMs + tiles - 1) / tiles);
    splits = std::max(splits, 1);
  }
  p.kt_per_split = (kt + splits - 1) / splits;
  p.splits = (kt + p.kt_per_split - 1) / p.kt_per_split;
  return p;
}

// Tiled transpose: in [R][C] (leading dimension ld) -> out [C][R] (leading dimension R).
// A block moves four 32 x 32 tiles (a 32 x 128 strip of the input): every load of the
// strip is issued before the barrier (16 per thread in flight), four times fewer blocks
// than one tile each (AlexNet fc6's 4096 x 9216 weight: 36864 latency-bound blocks,
// 2.5 TB/s).
constexpr int kTrTiles = 4;
// SPLIT: the output is written as its tf32 hi part and the tf32 residual lo
// (3xTF32 operands pre-split once in HBM; the GEMM's TMA then brings both).
template <bool SPLIT>
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                        float* __restrict__ out_lo, int R, int C, int64_t ld) {
  __shared__ float tile[kTrTiles][32][33];
  const int c0 = blockIdx.x * 32 * kTrTiles, r0 = blockIdx.y * 32;
  float v[kTrTiles][4];
#pragma unroll
  for (int t = 0; t < kTrTiles; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = r0 + threadIdx.y + 8 * i, c = c0 + t * 32 + threadIdx.x;
      v[t][i] = (r < R && c < C) ? __ldg(in + int64_t(r) * ld + c) : 0.f;
    }
#pragma unroll
  for (int t = 0; t < kTrTiles; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) tile[t][threadIdx.y + 8 * i][threadIdx.x] = v[t][i];
  __syncthreads();
#pragma unroll
  for (int t = 0; t < kTrTiles; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int c = c0 + t * 32 + threadIdx.y + 8 * i, r = r0 + threadIdx.x;
      if (c < C && r < R) {
        const float x = tile[t][threadIdx.x][threadIdx.y + 8 * i];
        if constexpr (SPLIT) {
          const float hi = ptx::tf32_hi(x);
          out[int64_t(c) * R + r] = hi;
          out_lo[int64_t(c) * R + r] = ptx::tf32_lo(x, hi);
        } else {
          out[int64_t(c) * R + r] = x;
        }
      }
    }
}

// An MN-contiguous operand of a large tensor-core GEMM, copied K-major: the
// producers then load 16-byte K vectors instead of scalars (one extra HBM pass,
// repaid many times by the contraction).  In 3xTF32 mode the copy is written
// pre-split (hi at offset_elems, lo right after it): the GEMM does no conversion.
struct KCopy {
  DenseView<float> v;
  const float* lo = nullptr;
};
KCopy k_major_copy(Ctx* c, cudaStream_t st, Workspace& scratch, size_t offset_elems, const DenseView<float>& v,
                   bool split) {
  float* out = static_cast<float*>(scratch.ptr) + offset_elems;
  float* lo = split ? out + ((size_t(v.rows) * v.K + 3) & ~size_t(3)) : nullptr;  // 16-byte aligned
  dim3 grid((v.rows + 32 * kTrTiles - 1) / (32 * kTrTiles), (v.K + 31) / 32);
  if (split) transpose_kernel<true><<<grid, dim3(32, 8), 0, st>>>(v.p, out, lo, v.K, v.rows, v.sk);
  else transpose_kernel<false><<<grid, dim3(32, 8), 0, st>>>(v.p, out, nullptr, v.K, v.rows, v.sk);
  check_launch("transpose");
  count_launch(c);
  return KCopy{DenseView<float>{out, int64_t(v.K), 1, v.rows, v.K, false}, lo};
}

// A K-contiguous operand written pre-split (hi, lo; rows of K, compact) so the GEMM's
// producers convert only the other operand (the large InnerProducts' activations and
// top diffs: 2.4 M elements against a 37.7 M-element weight for AlexNet fc6).
__global__ void __launch_bounds__(256) split_rows_kernel(const float* __restrict__ in, float* __restrict__ hi,
                                                         float* __restrict__ lo, int rows, int K, int64_t ld) {
  const int64_t total = int64_t(rows) * K;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / K, k = i - r * K;
    const float x = __ldg(in + r * ld + k);
    const float h = ptx::tf32_hi(x);
    hi[i] = h;
    lo[i] = ptx::tf32_lo(x, h);
  }
}
KCopy split_copy(Ctx* c, cudaStream_t st, Workspace& scratch, size_t offset_elems, const DenseView<float>& v) {
  float* out = static_cast<float*>(scratch.ptr) + offset_elems;
  float* lo = out + ((size_t(v.rows) * v.K + 3) & ~size_t(3));
  const int64_t total = int64_t(v.rows) * v.K;
  const int blocks = int(std::min<int64_t>((total + 255) / 256, int64_t(kNumSMs) * 8));
  split_rows_kernel<<<blocks, 256, 0, st>>>(v.p, out, lo, v.rows, v.K, v.sr);
  check_launch("split_rows");
  count_launch(c);
  return KCopy{DenseView<float>{out, int64_t(v.K), 1, v.rows, v.K, false}, lo};
}

// A K-major copy as a GEMM operand: pre-split TMA when it carries a lo copy (the copy
// is only made pre-split when TMA can take it, see dense_gemm).
template <class F>
void with_copy(Ctx* c, const KCopy& k, int box_rows, TmaReq& req, F&& f) {
  if (k.lo) {
    req = TmaReq{k.v.p, k.v.rows, k.v.K, k.v.sr, k.lo};
    f(TmaSplitView{});
  } else {
    with_operand(c, k.v, box_rows, req, f);
  }
}

// One GEMM D[m][n] = sum_k A(m,k) B(n,k) with dense views, routed by dtype.
// Small products in a single launch (gemm_simt.cuh dot kernels); false = not small.
template <typename T>
static bool small_gemm(Ctx* c, cudaStream_t st, int M, int N, int K, const DenseView<T>& va, const DenseView<T>& vb,
                       const StoreEpi<T>& epi) {
  const int64_t outs = int64_t(M) * N;
  // K in [64, 256): warp-per-output up to this many outputs (LeNet ip2 dW, 5000, measured faster per thread)
  constexpr int64_t warp_outs = 2048;
  // very few outputs, long K (PG-MLP dW over 1024 rows: a warp per output was 9.5 us):
  // a block per output
  if (outs <= 2 * kNumSMs && K >= 512) {
    simt::dot_block_kernel<T><<<int(outs), 256, 0, st>>>(va, vb, epi, M, N, K);
  } else
  // few outputs: a warp per output (CIFAR ip2 dW 640 x K=100: 29 -> 5.5 us)
  if (outs <= 16384 && (K >= 256 || (K >= 64 && outs <= warp_outs))) {
    const int64_t threads = outs * 32;
    simt::dot_warp_kernel<T><<<int((threads + 255) / 256), 256, 0, st>>>(va, vb, epi, M, N, K);
  } else if (K <= 128 && outs <= (int64_t(1) << 20)) {
    if (outs <= (int64_t(1) << 17))  // few threads (CIFAR ip1 dW 65536 x K=100: 27 -> 15 us)
      simt::dot_thread_kernel<T, 16><<<int((outs + 255) / 256), 256, 0, st>>>(va, vb, epi, M, N, K);
    else  // enough threads to hide the latency (LeNet ip1 dW 400000 x K=64)
      simt::dot_thread_kernel<T, 4><<<int((outs + 255) / 256), 256, 0, st>>>(va, vb, epi, M, N, K);
  } else {
    return false;
  }
  check_launch("small_gemm");
  count_launch(c);
  return true;
}

template <typename T>
static void dense_gemm(Ctx* c, cdnn_handle stream, int M, int N, int K, const DenseView<T>& va,
                       const DenseView<T>& vb, const StoreEpi<T>& epi) {
  cudaStream_t st = stream_of(c, stream);
  if (small_gemm<T>(c, st, M, N, K, va, vb, epi)) return;
  Workspace& ws = workspace_of(c, stream);
  if constexpr (std::is_same_v<T, float>) {
    // Small contractions (the CIFAR / LeNet / PG InnerProducts) are latency
    // bound: a tensor-core tile pipeline with a handful of CTAs loses to the
    // exact-fp32 SIMT engine split wide over K.
    if (int64_t(M) * N * K <= kSimtMaxMacs) {
      run_simt<T>(c, st, ws, plan_simt(M, N, K), M, N, K, va, vb, epi);
      return;
    }
    const GemmPlan pl = plan_tc(M, N, K);
    const bool split = c->math_mode == CDNN_MATH_TF32X3;
    // the copy of an operand with `rows` rows is TMA-eligible (aligned, K >= 32, rows >= box)
    auto presplit = [&](const DenseView<float>& v, int box) { return split && v.K >= 32 && v.K % 4 == 0 && v.rows >= box; };
    // a K-contiguous operand at most a quarter the size of the other one: pre-split copy
    // (one cheap pass) so only the large operand is converted in the kernel
    auto small_split = [&](const DenseView<float>& v, const DenseView<float>& o, int box) {
      return !v.mcontig && presplit(v, box) && v.sk == 1 && 4 * int64_t(v.rows) <= int64_t(o.rows);
    };
    // (contractions of >= 2^32 MACs: below that the extra launch does not pay, AlexNet fc8)
    const bool big = int64_t(M) * N * K >= (int64_t(1) << 32);
    const bool sa = big && small_split(va, vb, tc::BM), sb = big && small_split(vb, va, pl.bn);
    if (int64_t(M) * N * K >= (int64_t(1) << 28) && (va.mcontig || vb.mcontig || sa || sb)) {
      Workspace& aux = ws.aux();
      const size_t f = split ? 2 : 1;
      // 16-byte aligned halves (row counts are multiples of 4 elements only by chance)
      auto round4 = [](size_t n) { return (n + 3) & ~size_t(3); };
      const size_t na = (va.mcontig || sa) ? round4(size_t(va.rows) * va.K) : 0;
      const size_t nb = (vb.mcontig || sb) ? round4(size_t(vb.rows) * vb.K) : 0;
      aux.get((na + nb) * f * sizeof(float), c->device);
      const KCopy ka = va.mcontig ? k_major_copy(c, st, aux, 0, va, presplit(va, tc::BM))
                       : sa       ? split_copy(c, st, aux, 0, va)
                                  : KCopy{va, nullptr};
      const KCopy kb = vb.mcontig ? k_major_copy(c, st, aux, na * f, vb, presplit(vb, pl.bn))
                       : sb       ? split_copy(c, st, aux, na * f, vb)
                                  : KCopy{vb, nullptr};
      TmaReq ra2, rb2;
      with_copy(c, ka, tc::BM, ra2, [&](const auto& a) {
        with_copy(c, kb, pl.bn, rb2, [&](const auto& b) { run_tc(c, st, ws, pl, M, N, K, a, b, epi, ra2, rb2); });
      });
      return;
    }
    TmaReq ra, rb;
    with_operand(c, va, tc::BM, ra, [&](const auto& a) {
      with_operand(c, vb, pl.bn, rb, [&](const auto& b) { run_tc(c, st, ws, pl, M, N, K, a, b, epi, ra, rb); });
    });
  } else {
    const GemmPlan pl = plan_simt(M, N, K);
    run_simt<T>(c, st, ws, pl, M, N, K, va, vb, epi);
  }
}

template <typename T>
static void gemm_t(Ctx* c, int ta, int tb, int m, int n, int k, double alpha, const BufferSlot& A,
                   const BufferSlot& B, double beta, BufferSlot& C, cdnn_handle stream) {
  const T* a = reinterpret_cast<const T*>(A.dev);
  const T* b = reinterpret_cast<const T*>(B.dev);
  T* cc = reinterpret_cast<T*>(C.dev);
  // kernel A(mm=j, p) = opB[p][j]
  DenseView<T> va = tb ? DenseView<T>{b, int64_t(k), 1, n, k, false}
                       : DenseView<T>{b, 1, int64_t(n), n, k, true};
  // kernel B(nn=i, p) = opA[i][p]
  DenseView<T> vb = ta ? DenseView<T>{a, 1, int64_t(m), m, k, true}
                       : DenseView<T>{a, int64_t(k), 1, m, k, false};
  StoreEpi<T> epi{cc, 1, int64_t(n), T(alpha), T(beta), nullptr, false, false};
  dense_gemm<T>(c, stream, n, m, k, va, vb, epi);
}

// db[j] += sum_r dy[r][j] (layers.cpp:157-163): 32 columns x 8 row strands per
// block, fixed-shape tree over the strands (deterministic), coalesced rows.
template <typename T>
__global__ void __launch_bounds__(256) colsum_accum_kernel(const T* __restrict__ dy, T* __restrict__ db, int rows,
                                                           int cols) {
  __shared__ T part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  T s = T(0);
  if (j < cols)
    for (int r = ty; r < rows; r += 8) s += dy[int64_t(r) * cols + j];
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < cols) {
    T t = part[0][tx];
#pragma unroll
    for (int k = 1; k < 8; ++k) t += part[k][tx];
    db[j] += t;
  }
}

// Few columns, many rows (the PG-MLP's 10 / 2 bias columns over 1024 rows: the 32-column
// kernel above walked 128 rows per thread, 13 us): a block per column, threads stride
// the rows, fixed-shape tree in shared memory (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) colsum_accum_col_kernel(const T* __restrict__ dy, T* __restrict__ db, int rows,
                                                               int cols) {
  __shared__ T part[256];
  const int j = blockIdx.x;
  T s = T(0);
  for (int r = threadIdx.x; r < rows; r += 256) s += dy[int64_t(r) * cols + j];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) db[j] += part[0];
}

}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_gemm(cdnn_ctx ctx, int trans_a, int trans_b, int m, int n, int k, double alpha,
              cdnn_handle a, cdnn_handle b, double beta, cdnn_handle c, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    if (m <= 0 || n <= 0 || k <= 0) fail(CDNN_INVALID_ARGUMENT, "gemm: m, n, k must be positive");
    BufferSlot& A = buffer(cx, a, "gemm A");
    BufferSlot& B = buffer(cx, b, "gemm B");
    BufferSlot& C = buffer(cx, c, "gemm C");
    require_len(A, uint64_t(m) * k, "gemm A");
    require_len(B, uint64_t(k) * n, "gemm B");
    require_len(C, uint64_t(m) * n, "gemm C");
    require_dtype(B, A.dtype, "gemm B");
    require_dtype(C, A.dtype, "gemm C");
    DeviceGuard g(cx);
    if (A.dtype == CDNN_F32) gemm_t<float>(cx, trans_a, trans_b, m, n, k, alpha, A, B, beta, C, stream);
    else if (A.dtype == CDNN_F64) gemm_t<double>(cx, trans_a, trans_b, m, n, k, alpha, A, B, beta, C, stream);
    else fail(CDNN_INVALID_ARGUMENT, "gemm: floating buffers required");
  });
}

int cdnn_ip_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle w, cdnn_handle bias, cdnn_handle top,
                    int rows, int k, int o, int relu, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    if (rows <= 0 || k <= 0 || o <= 0) fail(CDNN_INVALID_ARGUMENT, "ip_forward: extents must be positive");
    BufferSlot& X = buffer(c, x, "ip_forward x");
    BufferSlot& W = buffer(c, w, "ip_forward w");
    BufferSlot& Y = buffer(c, top, "ip_forward top");
    BufferSlot* Bi = buffer_or_null(c, bias, "ip_forward bias");
    require_len(X, uint64_t(rows) * k, "ip_forward x");
    require_len(W, uint64_t(o) * k, "ip_forward w");
    require_len(Y, uint64_t(rows) * o, "ip_forward top");
    if (Bi) { require_len(*Bi, uint64_t(o), "ip_forward bias"); require_dtype(*Bi, X.dtype, "ip bias"); }
    require_dtype(W, X.dtype, "ip w");
    require_dtype(Y, X.dtype, "ip top");
    DeviceGuard g(c);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      DenseView<T> va{reinterpret_cast<const T*>(W.dev), int64_t(k), 1, o, k, false};
      DenseView<T> vb{reinterpret_cast<const T*>(X.dev), int64_t(k), 1, rows, k, false};
      StoreEpi<T> epi{reinterpret_cast<T*>(Y.dev), 1, int64_t(o), T(1), T(0),
                      Bi ? reinterpret_cast<const T*>(Bi->dev) : nullptr, true, relu != 0};
      dense_gemm<T>(c, stream, o, rows, k, va, vb, epi);
    };
    if (X.dtype == CDNN_F32) run(float{});
    else if (X.dtype == CDNN_F64) run(double{});
    else fail(CDNN_INVALID_ARGUMENT, "ip_forward: floating buffers required");
  });
}

int cdnn_ip_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle w, cdnn_handle dy, cdnn_handle dw,
                     cdnn_handle db, cdnn_handle dx, int rows, int k, int o, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    if (rows <= 0 || k <= 0 || o <= 0) fail(CDNN_INVALID_ARGUMENT, "ip_backward: extents must be positive");
    BufferSlot& X = buffer(c, x, "ip_backward x");
    BufferSlot& W = buffer(c, w, "ip_backward w");
    BufferSlot& DY = buffer(c, dy, "ip_backward dy");
    BufferSlot* DW = buffer_or_null(c, dw, "ip_backward dw");
    BufferSlot* DB = buffer_or_null(c, db, "ip_backward db");
    BufferSlot* DX = buffer_or_null(c, dx, "ip_backward dx");
    require_len(X, uint64_t(rows) * k, "ip_backward x");
    require_len(W, uint64_t(o) * k, "ip_backward w");
    require_len(DY, uint64_t(rows) * o, "ip_backward dy");
    if (DW) require_len(*DW, uint64_t(o) * k, "ip_backward dw");
    if (DB) require_len(*DB, uint64_t(o), "ip_backward db");
    if (DX) require_len(*DX, uint64_t(rows) * k, "ip_backward dx");
    for (BufferSlot* b : {&W, &DY, DW, DB, DX})
      if (b) require_dtype(*b, X.dtype, "ip_backward");
    DeviceGuard g(c);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      const T* xp = reinterpret_cast<const T*>(X.dev);
      const T* wp = reinterpret_cast<const T*>(W.dev);
      const T* dyp = reinterpret_cast<const T*>(DY.dev);
      if (DW) {  // dW += dY^T X   (layers.cpp:153-155, beta = 1)
        DenseView<T> va{xp, 1, int64_t(k), k, rows, true};
        DenseView<T> vb{dyp, 1, int64_t(o), o, rows, true};
        StoreEpi<T> epi{reinterpret_cast<T*>(DW->dev), 1, int64_t(k), T(1), T(1), nullptr, false, false};
        dense_gemm<T>(c, stream, k, o, rows, va, vb, epi);
      }
      if (DB) {  // db += column sums of dY (layers.cpp:157-163)
        if (o <= 64 && rows >= 512)
          colsum_accum_col_kernel<T><<<o, 256, 0, stream_of(c, stream)>>>(dyp, reinterpret_cast<T*>(DB->dev), rows, o);
        else
          colsum_accum_kernel<T><<<(o + 31) / 32, 256, 0, stream_of(c, stream)>>>(
              dyp, reinterpret_cast<T*>(DB->dev), rows, o);
        check_launch("colsum");
        count_launch(c);
      }
      if (DX) {  // dX = dY W   (layers.cpp:166-168, beta = 0)
        DenseView<T> va{wp, 1, int64_t(k), k, o, true};
        DenseView<T> vb{dyp, int64_t(o), 1, rows, o, false};
        StoreEpi<T> epi{reinterpret_cast<T*>(DX->dev), 1, int64_t(k), T(1), T(0), nullptr, false, false};
        dense_gemm<T>(c, stream, k, rows, o, va, vb, epi);
      }
    };
    if (X.dtype == CDNN_F32) run(float{});
    else if (X.dtype == CDNN_F64) run(double{});
    else fail(CDNN_INVALID_ARGUMENT, "ip_backward: floating buffers required");
  });
}

}  // extern "C"
