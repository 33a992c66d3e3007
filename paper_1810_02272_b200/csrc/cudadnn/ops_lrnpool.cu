// ops_lrnpool.cu — LRN (ACROSS_CHANNELS) fused with the MAX pooling that consumes
// its top (AlexNet norm1 -> pool1, norm2 -> pool2).  Neither layer exists in the
// reference; the semantics are Caffe's, exactly those of the unfused kernels
// (ops_layers.cu lrn_fwd_ring / lrn_bwd_ring, ops_pool.cu max_pool_fwd /
// max_pool_bwd_k): the same expressions in the same order, so the LRN top, the
// pooled top, the int32 argmax mask and the bottom gradient are bit-identical
// to LRN followed by Pooling (tests/test_gpu_kernels.py checks that).
//
// HBM traffic per element of the LRN bottom x (f32; AlexNet conv1: 74.3 M):
//   unfused forward   x + y + scale (LRN) + y + pool/mask (1/4.5 each)   ~ 18 B
//   fused forward     x + y (kept: the blob stays observable) + pool/mask ~  9.8 B
//   unfused backward  pool dy/mask, norm dy (LRN: x, y, scale, dy, dx)   ~ 25.8 B
//   fused backward    x + pool dy/mask + dx (scale, y and the LRN top diff are
//                     recomputed in registers; nothing else is stored)   ~  9.8 B
// The scale tensor is not stored at all.
//
// Forward: one block per (image, band of TR pooled rows); one thread per input
// pixel of the band's (TR-1)*S+K input rows walks the channels with the x ring
// of lrn_fwd_ring, G channels per step, and parks the normalised values in a
// double-buffered shared tile from which the block's pool threads take the
// 3x3 / 2x2 window maxima (one __syncthreads per G channels).  Halo rows between
// bands are computed twice (12% more x reads, from L2) and stored once.
// Backward: one thread per input pixel walks the channels; for the entering
// channel e = c + pre it recomputes scale(e) = k + alpha/n * sum x^2, y(e) and the
// LRN top diff (the pool backward gather over the <= R x R windows holding the
// pixel, in max_pool_bwd_k's order), then dx(c) from the rings of lrn_bwd_ring.
#include "launch.cuh"
#include "lrn_math.cuh"
#include "ptx.cuh"

namespace cdnn {
namespace {

constexpr int kCB = 16;       // LRN channels per block (the channel halos are loaded / computed twice)
constexpr int kThreads = 256;
constexpr int kMaxItems = 12;  // pooled (mask, dy) pairs one thread holds in the backward scatter

struct LrnPoolGeom {
  int N, C, H, W, PH, PW;
  int TRP;    // pooled rows per band
  int bands;
  int segs;   // channel segments of kCB
};

// channels [cfirst, cfirst + n) x npix consecutive elements of each plane -> smem tile
// [n][npix], by cp.async (no register round trip: every load of the tile is in flight
// at once); channels outside [0, C) are zero-filled.
template <typename T>
__device__ __forceinline__ void tile_async(T* tile, const T* base, int cfirst, int n, int C, uint32_t plane,
                                           int npix) {
  const uint32_t s0 = ptx::smem_u32(tile);
  for (int cl = 0; cl < n; ++cl) {
    const int c = cfirst + cl;
    const bool in = c >= 0 && c < C;
    const T* src = base + uint32_t(in ? c : 0) * plane;
    for (int p = threadIdx.x; p < npix; p += kThreads) {
      const uint32_t dst = s0 + uint32_t(cl * npix + p) * uint32_t(sizeof(T));
      if constexpr (sizeof(T) == 4) ptx::cp_async_4(dst, src + p, in ? 4u : 0u);
      else ptx::cp_async_8(dst, src + p, in ? 8u : 0u);
    }
  }
}

// Forward: block (band of TRP pooled rows, channel segment, image).
//   A  x tile: channels [c0-pre, c1+post) x the band's input rows -> smem (coalesced rows)
//   B  LRN top for [c0, c1) from the tile (window sum in lrn_fwd_ring's order) -> smem,
//      and to HBM for the rows this band owns (halo rows belong to the next band)
//   C  the pooled maxima / argmax of the band from the smem tile
template <typename T, int SIZE, int K, int S>
__global__ void __launch_bounds__(kThreads) lrn_maxpool_fwd(const T* __restrict__ x, T* __restrict__ ynorm,
                                                            T* __restrict__ ypool, int* __restrict__ mask,
                                                            LrnPoolGeom g, T alpha, T beta, T k, bool relu) {
  constexpr int pre = (SIZE - 1) / 2;
  extern __shared__ uint8_t smem_raw[];
  const int band = blockIdx.x, img = blockIdx.z;
  const int c0 = blockIdx.y * kCB, c1 = min(g.C, c0 + kCB), nc = c1 - c0;
  const int pr0 = band * g.TRP, pr1 = min(g.PH, pr0 + g.TRP);
  const int r0 = pr0 * S, r1 = min(g.H, (pr1 - 1) * S + K);
  const int own1 = band + 1 == g.bands ? g.H : min(g.H, pr1 * S);
  const int npix = (r1 - r0) * g.W, nown = (own1 - r0) * g.W;
  const uint32_t HW = uint32_t(g.H * g.W), PHW = uint32_t(g.PH * g.PW);
  T* xs = reinterpret_cast<T*>(smem_raw);       // [nc + SIZE - 1][npix]
  T* ys = xs + (kCB + SIZE - 1) * npix;         // [nc][npix]
  tile_async(xs, x + size_t(img) * g.C * HW + uint32_t(r0 * g.W), c0 - pre, nc + SIZE - 1, g.C, HW, npix);
  ptx::cp_async_wait_all();
  __syncthreads();
  const T aN = alpha / T(SIZE);
  T* yb = ynorm + size_t(img) * g.C * HW + uint32_t(r0 * g.W);
  for (int cl = 0; cl < nc; ++cl) {
    T* dst = yb + uint32_t(c0 + cl) * HW;
    for (int p = threadIdx.x; p < npix; p += kThreads) {
      T sum = T(0);
#pragma unroll
      for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xs[(cl + j) * npix + p]);
      const T sc = lrn::scale(sum, aN, k);
      const T yv = lrn::top(xs[(cl + pre) * npix + p], lrn::neg_pow(sc, beta));
      ys[cl * npix + p] = yv;
      if (p < nown) dst[p] = yv;
    }
  }
  __syncthreads();
  const int prows = pr1 - pr0, per_c = prows * g.PW;
  for (int it = threadIdx.x; it < nc * per_c; it += kThreads) {
    const int cl = it / per_c, rem = it - cl * per_c;
    const int prl = rem / g.PW, pw = rem - prl * g.PW;
    const int hs = (pr0 + prl) * S, ws = pw * S;
    const T* t = ys + cl * npix + (hs - r0) * g.W;
    T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
    int arg = -1;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b)
        if (hs + a < g.H && ws + b < g.W) {
          const T v = t[a * g.W + ws + b];
          if (v > best) { best = v; arg = (hs + a) * g.W + ws + b; }
        }
    const uint32_t o = (uint32_t(img) * g.C + c0 + cl) * PHW + uint32_t((pr0 + prl) * g.PW + pw);
    ypool[o] = relu ? (best > T(0) ? best : T(0)) : best;
    mask[o] = arg;
  }
}

// Backward: block (band of TRP pooled rows = the pixel rows it owns, channel segment, image).
//   0  LRN top diff of channels [c0-post, c1+pre) on the owned pixels by a deterministic
//      scatter of the pooled diffs through the argmax mask: four passes in the order
//      max_pool_bwd_k's gather adds a pixel's windows ((a, b) = (0,0), (0,1), (1,0), (1,1)
//      relative to its first window), so the sums are bit-identical; within a pass no
//      two windows share a pixel
//   1  x tile: channels [c0-(SIZE-1), c1+(SIZE-1)) on the owned pixels
//   2  t = dy*y/scale for [c0-post, c1+pre); p1 = dy*scale^-beta kept for [c0, c1)
//   3  dx for [c0, c1) (ring sum in lrn_bwd_ring's order), gated, coalesced stores
template <typename T, int SIZE, int K, int S>
__global__ void __launch_bounds__(kThreads) lrn_maxpool_bwd(const T* __restrict__ x, const T* __restrict__ pdy,
                                                            const int* __restrict__ mask, T* __restrict__ dx,
                                                            LrnPoolGeom g, T alpha, T beta, T k, bool gate_x) {
  constexpr int pre = (SIZE - 1) / 2, post = SIZE - 1 - pre;
  extern __shared__ uint8_t smem_raw[];
  const int band = blockIdx.x, img = blockIdx.z;
  const int c0 = blockIdx.y * kCB, c1 = min(g.C, c0 + kCB), nc = c1 - c0;
  const int pr0 = band * g.TRP, pr1 = min(g.PH, pr0 + g.TRP);
  const int r0 = pr0 * S, r1 = band + 1 == g.bands ? g.H : min(g.H, pr1 * S);  // owned pixel rows
  const int npix = (r1 - r0) * g.W;
  const uint32_t HW = uint32_t(g.H * g.W), PHW = uint32_t(g.PH * g.PW);
  const int ndc = nc + SIZE - 1;            // channels with a top diff / t
  T* nd = reinterpret_cast<T*>(smem_raw);   // [ndc][npix]: LRN top diff, then p1 (own channels)
  T* xs = nd + (kCB + SIZE - 1) * npix;     // [nc + 2(SIZE-1)][npix]
  T* ts = xs + (kCB + 2 * (SIZE - 1)) * npix;  // [ndc][npix]
  // the x tile flies (cp.async) while the pooled diffs are scattered
  tile_async(xs, x + size_t(img) * g.C * HW + uint32_t(r0 * g.W), c0 - (SIZE - 1), nc + 2 * (SIZE - 1), g.C, HW,
             npix);
  for (int i = threadIdx.x; i < ndc * npix; i += kThreads) nd[i] = T(0);
  // pooled rows whose windows reach the owned rows
  const int ph0 = max(0, (r0 - K + S) / S), ph1 = min(g.PH, (r1 - 1) / S + 1);
  const int per_c = (ph1 - ph0) * g.PW, nitems = ndc * per_c;
  const int* mb = mask + size_t(img) * g.C * PHW;
  const T* db0 = pdy + size_t(img) * g.C * PHW;
  // one pooled element -> (tile cell of its argmax or -1, pass); the pass is the
  // position of this window in max_pool_bwd_k's gather order for that pixel
  auto locate = [&](int it, int& cell, int& pass, T& v) {
    const int cl = it / per_c, rem = it - cl * per_c;
    const int c = c0 - post + cl;
    cell = -1;
    pass = 0;
    v = T(0);
    if (c < 0 || c >= g.C) return;
    const uint32_t o = uint32_t(c) * PHW + uint32_t(ph0 * g.PW + rem);
    const int m = __ldg(mb + o);
    v = __ldg(db0 + o);
    if (m < 0) return;
    const int mh = m / g.W;
    if (mh < r0 || mh >= r1) return;
    const int prl = rem / g.PW, ph = ph0 + prl, pw = rem - prl * g.PW, mw = m - mh * g.W;
    const int a = (K > S && mh == ph * S && ph > 0) ? 1 : 0;  // second window of that row
    const int b = (K > S && mw == pw * S && pw > 0) ? 1 : 0;
    cell = cl * npix + (m - r0 * g.W);
    pass = a * 2 + b;
  };
  int icell[kMaxItems], ipass[kMaxItems];
  T iv[kMaxItems];
#pragma unroll
  for (int q = 0; q < kMaxItems; ++q) {
    const int it = threadIdx.x + q * kThreads;
    icell[q] = -1;
    ipass[q] = 0;
    iv[q] = T(0);
    if (it < nitems) locate(it, icell[q], ipass[q], iv[q]);
  }
  for (int pass = 0; pass < 4; ++pass) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kMaxItems; ++q)
      if (icell[q] >= 0 && ipass[q] == pass) nd[icell[q]] += iv[q];
    for (int it = threadIdx.x + kMaxItems * kThreads; it < nitems; it += kThreads) {  // beyond the registers
      int cell, ps;
      T v;
      locate(it, cell, ps, v);
      if (cell >= 0 && ps == pass) nd[cell] += v;
    }
  }
  ptx::cp_async_wait_all();
  __syncthreads();
  const T aN = alpha / T(SIZE);
  for (int cl = 0; cl < ndc; ++cl) {  // channel c' = c0 - post + cl
    const int c = c0 - post + cl;
    const bool in = c >= 0 && c < g.C;
    const bool own = c >= c0 && c < c1;
    for (int p = threadIdx.x; p < npix; p += kThreads) {
      T t = T(0);
      if (in) {
        T sum = T(0);
#pragma unroll
        for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xs[(cl + j) * npix + p]);
        const T sc = lrn::scale(sum, aN, k);
        const T np = lrn::neg_pow(sc, beta);
        const T d = nd[cl * npix + p];
        t = lrn::term(d, lrn::top(xs[(cl + pre) * npix + p], np), sc);
        if (own) nd[cl * npix + p] = lrn::mul_(d, np);
      }
      ts[cl * npix + p] = t;
    }
  }
  __syncthreads();
  const T coef = T(2) * alpha * beta / T(SIZE);
  T* db = dx + size_t(img) * g.C * HW + uint32_t(r0 * g.W);
  for (int cl = 0; cl < nc; ++cl) {
    T* dst = db + uint32_t(c0 + cl) * HW;
    for (int p = threadIdx.x; p < npix; p += kThreads) {
      T acc = T(0);
#pragma unroll
      for (int j = 0; j < SIZE; ++j) acc = lrn::add_(acc, ts[(cl + j) * npix + p]);
      const T xc = xs[(cl + SIZE - 1) * npix + p];
      const T gv = lrn::sub_(nd[(cl + post) * npix + p], lrn::mul_(lrn::mul_(coef, xc), acc));
      dst[p] = (!gate_x || xc > T(0)) ? gv : T(0);
    }
  }
}

// owned pixel rows of the widest band
int bwd_rows(const LrnPoolGeom& g, int S) { return std::max(g.TRP * S, g.H - (g.bands - 1) * g.TRP * S); }

size_t fwd_smem_bytes(const LrnPoolGeom& g, int size, int K, int S, size_t es) {
  return size_t(2 * kCB + size - 1) * size_t((g.TRP - 1) * S + K) * g.W * es;
}
size_t bwd_smem_bytes(const LrnPoolGeom& g, int size, int S, size_t es) {
  return size_t(3 * kCB + 4 * (size - 1)) * size_t(bwd_rows(g, S)) * g.W * es;
}

// Bands of TRP pooled rows: as many as keep both tiles within ~100 KB (two blocks per
// SM), at most ~512 owned pixels; TRP = 0 when not even one pooled row fits.
LrnPoolGeom lrn_pool_geom(const PoolDescSlot& d, int size, size_t es) {
  const auto& p = d.p;
  LrnPoolGeom g{p.n, p.c, p.h, p.w, d.PH, d.PW, 1, 0, (p.c + kCB - 1) / kCB};
  const int K = p.kernel_h, S = p.stride_h;
  for (int trp = std::max(1, std::min(d.PH, 512 / std::max(1, S * p.w))); trp >= 1; --trp) {
    g.TRP = trp;
    g.bands = (d.PH + trp - 1) / trp;
    if (bwd_smem_bytes(g, size, S, es) <= 100 * 1024 && fwd_smem_bytes(g, size, K, S, es) <= 100 * 1024) return g;
  }
  g.TRP = 0;
  return g;
}

bool fusable(const PoolDescSlot& d, int size, size_t es) {
  const auto& p = d.p;
  const bool window = p.kernel_h == p.kernel_w && p.stride_h == p.stride_w &&
                      ((p.kernel_h == 3 && p.stride_h == 2) || (p.kernel_h == 2 && p.stride_h == 2));
  return p.method == CDNN_POOL_MAX && !p.global_pooling && p.pad_h == 0 && p.pad_w == 0 && window &&
         (size == 3 || size == 5) && uint64_t(p.n) * p.c * p.h * p.w < (1ull << 31) &&
         lrn_pool_geom(d, size, es).TRP > 0;
}

template <typename T, int SIZE, int K, int S>
void launch_fwd(Ctx* c, cudaStream_t st, const PoolDescSlot& d, const T* x, T* yn, T* yp, int* m, double alpha,
                double beta, double k, bool relu) {
  const LrnPoolGeom g = lrn_pool_geom(d, SIZE, sizeof(T));
  const size_t smem = fwd_smem_bytes(g, SIZE, K, S, sizeof(T));
  auto kern = lrn_maxpool_fwd<T, SIZE, K, S>;
  CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<dim3(g.bands, g.segs, g.N), kThreads, smem, st>>>(x, yn, yp, m, g, T(alpha), T(beta), T(k), relu);
  check_launch("lrn_maxpool_fwd");
  count_launch(c);
}

template <typename T, int SIZE, int K, int S>
void launch_bwd(Ctx* c, cudaStream_t st, const PoolDescSlot& d, const T* x, const T* pdy, const int* m, T* dx,
                double alpha, double beta, double k, bool gate_x) {
  const LrnPoolGeom g = lrn_pool_geom(d, SIZE, sizeof(T));
  const size_t smem = bwd_smem_bytes(g, SIZE, S, sizeof(T));
  auto kern = lrn_maxpool_bwd<T, SIZE, K, S>;
  CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<dim3(g.bands, g.segs, g.N), kThreads, smem, st>>>(x, pdy, m, dx, g, T(alpha), T(beta), T(k), gate_x);
  check_launch("lrn_maxpool_bwd");
  count_launch(c);
}

template <class F>
void dispatch_shape(const PoolDescSlot& d, int size, F&& f) {
  const int K = d.p.kernel_h;
  if (size == 5 && K == 3) f(std::integral_constant<int, 5>{}, std::integral_constant<int, 3>{});
  else if (size == 5 && K == 2) f(std::integral_constant<int, 5>{}, std::integral_constant<int, 2>{});
  else if (size == 3 && K == 3) f(std::integral_constant<int, 3>{}, std::integral_constant<int, 3>{});
  else f(std::integral_constant<int, 3>{}, std::integral_constant<int, 2>{});
}

}  // namespace
}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_lrn_pool_supported(cdnn_ctx ctx, cdnn_handle pool_desc_h, int local_size, int* out) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    // the float path decides for the net; the double tiles are checked at launch
    *out = fusable(pool_desc(c, pool_desc_h), local_size, sizeof(float)) ? 1 : 0;
  });
}

int cdnn_lrn_pool_forward(cdnn_ctx ctx, cdnn_handle pool_desc_h, cdnn_handle x, cdnn_handle lrn_top,
                          cdnn_handle pool_top, cdnn_handle mask, int local_size, double alpha, double beta, double k,
                          int flags, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    const PoolDescSlot d = pool_desc(c, pool_desc_h);
    BufferSlot& X = buffer(c, x, "lrn_pool x");
    if (!fusable(d, local_size, dtype_size(X.dtype)))
      fail(CDNN_INVALID_ARGUMENT, "lrn_pool: unsupported LRN / pooling combination");
    BufferSlot& YN = buffer(c, lrn_top, "lrn_pool lrn top");
    BufferSlot& YP = buffer(c, pool_top, "lrn_pool pool top");
    BufferSlot& M = buffer(c, mask, "lrn_pool mask");
    const uint64_t nin = uint64_t(d.p.n) * d.p.c * d.p.h * d.p.w, nout = uint64_t(d.p.n) * d.p.c * d.PH * d.PW;
    require_len(X, nin, "lrn_pool x");
    require_len(YN, nin, "lrn_pool lrn top");
    require_len(YP, nout, "lrn_pool pool top");
    require_len(M, nout, "lrn_pool mask");
    require_dtype(YN, X.dtype, "lrn_pool");
    require_dtype(YP, X.dtype, "lrn_pool");
    require_dtype(M, CDNN_I32, "lrn_pool mask");
    DeviceGuard dg(c);
    cudaStream_t st = stream_of(c, stream);
    const bool relu = (flags & CDNN_POOL_RELU) != 0;
    dispatch_shape(d, local_size, [&](auto sz, auto kk) {
      constexpr int SIZE = decltype(sz)::value, K = decltype(kk)::value;
      if (X.dtype == CDNN_F32)
        launch_fwd<float, SIZE, K, 2>(c, st, d, reinterpret_cast<const float*>(X.dev), reinterpret_cast<float*>(YN.dev),
                                      reinterpret_cast<float*>(YP.dev), reinterpret_cast<int*>(M.dev), alpha, beta, k,
                                      relu);
      else if (X.dtype == CDNN_F64)
        launch_fwd<double, SIZE, K, 2>(c, st, d, reinterpret_cast<const double*>(X.dev),
                                       reinterpret_cast<double*>(YN.dev), reinterpret_cast<double*>(YP.dev),
                                       reinterpret_cast<int*>(M.dev), alpha, beta, k, relu);
      else
        fail(CDNN_INVALID_ARGUMENT, "lrn_pool: floating buffers required");
    });
  });
}

int cdnn_lrn_pool_backward(cdnn_ctx ctx, cdnn_handle pool_desc_h, cdnn_handle x, cdnn_handle pool_dy,
                           cdnn_handle mask, cdnn_handle dx, cdnn_handle gate, int local_size, double alpha,
                           double beta, double k, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    const PoolDescSlot d = pool_desc(c, pool_desc_h);
    if (gate && gate != x) fail(CDNN_INVALID_ARGUMENT, "lrn_pool backward: the ReLU gate must be the LRN bottom x");
    BufferSlot& X = buffer(c, x, "lrn_pool_bwd x");
    if (!fusable(d, local_size, dtype_size(X.dtype)))
      fail(CDNN_INVALID_ARGUMENT, "lrn_pool: unsupported LRN / pooling combination");
    BufferSlot& DY = buffer(c, pool_dy, "lrn_pool_bwd pool dy");
    BufferSlot& M = buffer(c, mask, "lrn_pool_bwd mask");
    BufferSlot& DX = buffer(c, dx, "lrn_pool_bwd dx");
    const uint64_t nin = uint64_t(d.p.n) * d.p.c * d.p.h * d.p.w, nout = uint64_t(d.p.n) * d.p.c * d.PH * d.PW;
    require_len(X, nin, "lrn_pool_bwd x");
    require_len(DX, nin, "lrn_pool_bwd dx");
    require_len(DY, nout, "lrn_pool_bwd pool dy");
    require_len(M, nout, "lrn_pool_bwd mask");
    require_dtype(DX, X.dtype, "lrn_pool_bwd");
    require_dtype(DY, X.dtype, "lrn_pool_bwd");
    require_dtype(M, CDNN_I32, "lrn_pool_bwd mask");
    DeviceGuard dg(c);
    cudaStream_t st = stream_of(c, stream);
    dispatch_shape(d, local_size, [&](auto sz, auto kk) {
      constexpr int SIZE = decltype(sz)::value, K = decltype(kk)::value;
      if (X.dtype == CDNN_F32)
        launch_bwd<float, SIZE, K, 2>(c, st, d, reinterpret_cast<const float*>(X.dev),
                                      reinterpret_cast<const float*>(DY.dev), reinterpret_cast<const int*>(M.dev),
                                      reinterpret_cast<float*>(DX.dev), alpha, beta, k, gate != 0);
      else if (X.dtype == CDNN_F64)
        launch_bwd<double, SIZE, K, 2>(c, st, d, reinterpret_cast<const double*>(X.dev),
                                       reinterpret_cast<const double*>(DY.dev), reinterpret_cast<const int*>(M.dev),
                                       reinterpret_cast<double*>(DX.dev), alpha, beta, k, gate != 0);
      else
        fail(CDNN_INVALID_ARGUMENT, "lrn_pool: floating buffers required");
    });
  });
}

}  // extern "C"
