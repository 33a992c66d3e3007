// ops_pool.cu — Caffe pooling (absent from the reference).
//
// MAX: window scanned h-major then w, strict `>` so the first maximum wins;
//      the int32 mask holds the flat h*W+w index of the winner (bit-exact
//      integer output).  Backward gathers: each bottom element sums the top
//      diffs of the windows whose mask points at it (no atomics, deterministic).
// AVE: Caffe's divisor counts padded positions but not the overhang past
//      H+pad; backward spreads top_diff/pool_size over the clipped window.
// One thread per output (forward) / input (backward) element; NCHW planes.
#include <cstdlib>

#include "launch.cuh"

namespace cdnn {
namespace {

struct PoolGeom {
  int N, C, H, W, PH, PW, kh, kw, sh, sw, ph, pw;
  // 32-bit index decomposition without hardware division (SASS integer division
  // is a ~20-instruction sequence; these kernels are issue-bound otherwise)
  FastDiv divW, divHW, divPW, divPHW, divSH, divSW, divH;
};

// (plane, h, w) of a flat NCHW index within planes of H x W
struct Idx3 {
  uint32_t plane, h, w;
};
__device__ __forceinline__ Idx3 split3(uint32_t i, const FastDiv& dhw, const FastDiv& dw, uint32_t HW, uint32_t W) {
  const uint32_t plane = dhw.div(i);
  const uint32_t r = i - plane * HW;
  const uint32_t h = dw.div(r);
  return {plane, h, r - h * W};
}

template <typename T>
__global__ void __launch_bounds__(256) max_pool_fwd(const T* __restrict__ x, T* __restrict__ y, int* __restrict__ mask,
                                                    PoolGeom g, uint32_t total, bool relu) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, g.divPHW, g.divPW, uint32_t(g.PH * g.PW), uint32_t(g.PW));
    int hs = int(q.h) * g.sh - g.ph, ws = int(q.w) * g.sw - g.pw;
    const int he = min(hs + g.kh, g.H), we = min(ws + g.kw, g.W);
    hs = max(hs, 0);
    ws = max(ws, 0);
    const T* plane = x + size_t(q.plane) * uint32_t(g.H * g.W);
    T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
    int arg = -1;
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) {
        const T v = __ldg(plane + h * g.W + w);
        if (v > best) { best = v; arg = h * g.W + w; }
      }
    y[i] = relu ? (best > T(0) ? best : T(0)) : best;  // fused in-place ReLU on the pooled top
    if (mask) mask[i] = arg;
  }
}

// gather: every bottom element sums the top diffs of the windows whose argmax is it
template <typename T>
__global__ void __launch_bounds__(256) max_pool_bwd(const T* __restrict__ dy, const int* __restrict__ mask,
                                                    T* __restrict__ dx, PoolGeom g, uint32_t total4,
                                                    const T* __restrict__ gate) {
  // four consecutive bottom elements of one row per thread: the row's window range
  // (and the plane / row decomposition) is computed once per thread
  const uint32_t W4 = uint32_t(g.W + 3) >> 2;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += gridDim.x * blockDim.x) {
    const uint32_t row = i / W4, w0 = (i - row * W4) * 4;  // row = plane*H + h (W4 small: cheap)
    const uint32_t plane = g.divH.div(row), hq = row - plane * uint32_t(g.H);
    const int h = int(hq) + g.ph;
    const int phs = h < g.kh ? 0 : int(g.divSH.div(uint32_t(h - g.kh))) + 1;
    const int phe = min(int(g.divSH.div(uint32_t(h))) + 1, g.PH);
    const size_t base = size_t(plane) * uint32_t(g.PH * g.PW);
    const size_t out = size_t(row) * uint32_t(g.W);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int wq = int(w0) + e;
      if (wq >= g.W) break;
      const int w = wq + g.pw;
      const int pws = w < g.kw ? 0 : int(g.divSW.div(uint32_t(w - g.kw))) + 1;
      const int pwe = min(int(g.divSW.div(uint32_t(w))) + 1, g.PW);
      const int me = int(hq) * g.W + wq;
      T s = T(0);
      for (int ph = phs; ph < phe; ++ph)
        for (int pw = pws; pw < pwe; ++pw) {
          const size_t o = base + ph * g.PW + pw;
          if (__ldg(mask + o) == me) s += __ldg(dy + o);
        }
      // fused backward of an in-place ReLU on the pooling's bottom (gate = its data)
      dx[out + wq] = (gate && !(__ldg(gate + out + wq) > T(0))) ? T(0) : s;
    }
  }
}

// Fixed-window MAX backward over S x S blocks of bottom elements: with K <= 2S the
// block (padded rows S*j .. S*j+S-1, columns S*k ..) is covered only by the windows
// (j-D .. j) x (k-D .. k), D = (K-1)/S, so one thread loads those (D+1)^2 mask entries
// and top diffs once for S*S elements (AlexNet 3x3/2: 4 windows for 4 elements instead
// of 4 per element) and decomposes one index.  A window whose argmax is the element
// covers it, so the mask test alone selects the contributions; they are added in
// ascending (ph, pw) order like max_pool_bwd, so the sums are bit-identical.
template <typename T, int K, int S>
__global__ void __launch_bounds__(256) max_pool_bwd_blk(const T* __restrict__ dy, const int* __restrict__ mask,
                                                        T* __restrict__ dx, PoolGeom g, FastDiv div_bw,
                                                        FastDiv div_bhw, uint32_t BW, uint32_t BHW, uint32_t total,
                                                        const T* __restrict__ gate) {
  constexpr int D = (K - 1) / S;
  static_assert(K <= 2 * S, "block covers at most (D+1)^2 windows");
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, div_bhw, div_bw, BHW, BW);
    const int j = int(q.h), k = int(q.w);
    const size_t base = size_t(q.plane) * uint32_t(g.PH * g.PW);
    int m[D + 1][D + 1];
    T v[D + 1][D + 1];
#pragma unroll
    for (int a = 0; a <= D; ++a)
#pragma unroll
      for (int b = 0; b <= D; ++b) {
        const int ph = j - D + a, pw = k - D + b;
        const bool ok = ph >= 0 && ph < g.PH && pw >= 0 && pw < g.PW;
        const size_t o = base + ph * g.PW + pw;
        m[a][b] = ok ? __ldg(mask + o) : -1;
        v[a][b] = ok ? __ldg(dy + o) : T(0);
      }
    const size_t pbase = size_t(q.plane) * uint32_t(g.H * g.W);
    bool in[S][S];
    T gv[S][S];
#pragma unroll
    for (int r = 0; r < S; ++r)
#pragma unroll
      for (int c = 0; c < S; ++c) {
        const int h = j * S + r - g.ph, w = k * S + c - g.pw;
        in[r][c] = h >= 0 && h < g.H && w >= 0 && w < g.W;
        gv[r][c] = (gate && in[r][c]) ? __ldg(gate + pbase + h * g.W + w) : T(1);
      }
#pragma unroll
    for (int r = 0; r < S; ++r)
#pragma unroll
      for (int c = 0; c < S; ++c) {
        if (!in[r][c]) continue;
        const int h = j * S + r - g.ph, w = k * S + c - g.pw;
        const int me = h * g.W + w;
        T s = T(0);
#pragma unroll
        for (int a = 0; a <= D; ++a)
#pragma unroll
          for (int b = 0; b <= D; ++b)
            if (m[a][b] == me) s += v[a][b];
        dx[pbase + me] = gv[r][c] > T(0) ? s : T(0);
      }
  }
}

// Fixed-window MAX forward, two vertically adjacent outputs per thread (S < K: the
// shared window rows are loaded once; consecutive threads take consecutive output
// columns, so every store is coalesced); every load issued before the scan, which
// keeps max_pool_fwd's h-major order and strict '>' (bit-identical).
template <typename T, int K, int S>
__global__ void __launch_bounds__(256) max_pool_fwd_k2(const T* __restrict__ x, T* __restrict__ y,
                                                       int* __restrict__ mask, PoolGeom g, FastDiv div_pw,
                                                       FastDiv div_phw2, uint32_t PHW2, uint32_t total, bool relu) {
  constexpr int RW = K + S;  // input rows of the two windows
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, div_phw2, div_pw, PHW2, uint32_t(g.PW));
    const int oh = int(q.h) * 2, ow = int(q.w);
    const int hs = oh * S - g.ph, ws = ow * S - g.pw;
    const T* plane = x + size_t(q.plane) * uint32_t(g.H * g.W);
    T v[RW][K];
    bool ok[RW][K];
    // interior (the whole 2-window block inside the plane, the common case): no bounds
    // tests, one row pointer per window row and immediate column offsets -- the general
    // path's integer work was ~2/3 of this issue-bound kernel's instructions
    const bool interior = hs >= 0 && ws >= 0 && hs + RW <= g.H && ws + K <= g.W && oh + 1 < g.PH;
    if (interior) {
      const T* r0 = plane + (hs * g.W + ws);
#pragma unroll
      for (int a = 0; a < RW; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          ok[a][b] = true;
          v[a][b] = __ldg(r0 + a * g.W + b);
        }
    } else {
#pragma unroll
      for (int a = 0; a < RW; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          const int h = hs + a, w = ws + b;
          ok[a][b] = h >= 0 && h < g.H && w >= 0 && w < g.W;
          v[a][b] = ok[a][b] ? __ldg(plane + h * g.W + w) : T(0);
        }
    }
    const size_t ob = size_t(q.plane) * uint32_t(g.PH * g.PW) + size_t(oh) * g.PW + ow;
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      if (oh + o >= g.PH) break;
      T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
      int arg = -1;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b)
          if (ok[o * S + a][b] && v[o * S + a][b] > best) {
            best = v[o * S + a][b];
            arg = (hs + o * S + a) * g.W + ws + b;
          }
      y[ob + o * g.PW] = relu ? (best > T(0) ? best : T(0)) : best;
      if (mask) mask[ob + o * g.PW] = arg;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) ave_pool_fwd(const T* __restrict__ x, T* __restrict__ y, PoolGeom g,
                                                    uint32_t total, bool relu) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, g.divPHW, g.divPW, uint32_t(g.PH * g.PW), uint32_t(g.PW));
    int hs = int(q.h) * g.sh - g.ph, ws = int(q.w) * g.sw - g.pw;
    int he = min(hs + g.kh, g.H + g.ph), we = min(ws + g.kw, g.W + g.pw);
    const int pool = (he - hs) * (we - ws);
    hs = max(hs, 0); ws = max(ws, 0);
    he = min(he, g.H); we = min(we, g.W);
    const T* plane = x + size_t(q.plane) * uint32_t(g.H * g.W);
    T s = T(0);
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) s += __ldg(plane + h * g.W + w);
    const T v = s / T(pool);
    y[i] = relu ? (v > T(0) ? v : T(0)) : v;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) ave_pool_bwd(const T* __restrict__ dy, T* __restrict__ dx, PoolGeom g,
                                                    uint32_t total, const T* __restrict__ gate) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, g.divHW, g.divW, uint32_t(g.H * g.W), uint32_t(g.W));
    const int h = int(q.h) + g.ph, w = int(q.w) + g.pw;
    const int phs = h < g.kh ? 0 : int(g.divSH.div(uint32_t(h - g.kh))) + 1;
    const int phe = min(int(g.divSH.div(uint32_t(h))) + 1, g.PH);
    const int pws = w < g.kw ? 0 : int(g.divSW.div(uint32_t(w - g.kw))) + 1;
    const int pwe = min(int(g.divSW.div(uint32_t(w))) + 1, g.PW);
    const size_t base = size_t(q.plane) * uint32_t(g.PH * g.PW);
    T s = T(0);
    for (int ph = phs; ph < phe; ++ph)
      for (int pw = pws; pw < pwe; ++pw) {
        const int hs = ph * g.sh - g.ph, ws = pw * g.sw - g.pw;
        const int he = min(hs + g.kh, g.H + g.ph), we = min(ws + g.kw, g.W + g.pw);
        s += __ldg(dy + base + ph * g.PW + pw) / T((he - hs) * (we - ws));
      }
    dx[i] = (gate && !(__ldg(gate + i) > T(0))) ? T(0) : s;
  }
}

// Fixed-window AVE pooling: unrolled K x K window, same h-major summation order
// and Caffe divisor (padded positions counted, overhang past H+pad not) as
// ave_pool_fwd, so outputs are bit-identical.
template <typename T, int K, int S>
__global__ void __launch_bounds__(256) ave_pool_fwd_k(const T* __restrict__ x, T* __restrict__ y, PoolGeom g,
                                                      uint32_t total, bool relu) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, g.divPHW, g.divPW, uint32_t(g.PH * g.PW), uint32_t(g.PW));
    const int hs = int(q.h) * S - g.ph, ws = int(q.w) * S - g.pw;
    const int pool = (min(hs + K, g.H + g.ph) - hs) * (min(ws + K, g.W + g.pw) - ws);
    const T* plane = x + size_t(q.plane) * uint32_t(g.H * g.W);
    T v[K][K];
    bool ok[K][K];
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b) {
        const int h = hs + a, w = ws + b;
        ok[a][b] = h >= 0 && h < g.H && w >= 0 && w < g.W;
        v[a][b] = ok[a][b] ? __ldg(plane + h * g.W + w) : T(0);
      }
    T s = T(0);
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b)
        if (ok[a][b]) s += v[a][b];
    const T r = s / T(pool);
    y[i] = relu ? (r > T(0) ? r : T(0)) : r;
  }
}

// Fixed-window AVE backward: one bottom element per thread, at most ceil(K/S)^2
// covering windows, visited in ave_pool_bwd's (ph, pw) order (bit-identical sums).
template <typename T, int K, int S>
__global__ void __launch_bounds__(256) ave_pool_bwd_k(const T* __restrict__ dy, T* __restrict__ dx, PoolGeom g,
                                                      uint32_t total, const T* __restrict__ gate) {
  constexpr int R = (K + S - 1) / S;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const Idx3 q = split3(i, g.divHW, g.divW, uint32_t(g.H * g.W), uint32_t(g.W));
    const int h = int(q.h) + g.ph, w = int(q.w) + g.pw;
    const int phs = h < K ? 0 : (h - K) / S + 1, phe = min(h / S + 1, g.PH);
    const int pws = w < K ? 0 : (w - K) / S + 1, pwe = min(w / S + 1, g.PW);
    const size_t base = size_t(q.plane) * uint32_t(g.PH * g.PW);
    const bool open = !gate || __ldg(gate + i) > T(0);
    T v[R][R];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b)
        v[a][b] = (phs + a < phe && pws + b < pwe) ? __ldg(dy + base + (phs + a) * g.PW + pws + b) : T(0);
    T s = T(0);
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b)
        if (phs + a < phe && pws + b < pwe) {
          const int hs0 = (phs + a) * S - g.ph, ws0 = (pws + b) * S - g.pw;
          const int pool = (min(hs0 + K, g.H + g.ph) - hs0) * (min(ws0 + K, g.W + g.pw) - ws0);
          s += v[a][b] / T(pool);
        }
    dx[i] = open ? s : T(0);
  }
}

// 32 / 22 for square 3x3 / 2x2 windows of stride 2 (the unrolled kernels, MAX and
// AVE), else 0; CDNN_POOL_GENERIC=1 forces the dynamic-window kernels (A/B checks)
int fixed_window(const PoolGeom& g) {
  static const bool generic = [] {
    const char* e = std::getenv("CDNN_POOL_GENERIC");
    return e && e[0] == '1';
  }();
  if (generic || g.sh != 2 || g.sw != 2 || g.kh != g.kw) return 0;
  return g.kh == 3 ? 32 : g.kh == 2 ? 22 : 0;
}

PoolGeom geom_of(const PoolDescSlot& d) {
  const auto& p = d.p;
  PoolGeom g{p.n, p.c, p.h, p.w, d.PH, d.PW, p.kernel_h, p.kernel_w, p.stride_h, p.stride_w, p.pad_h, p.pad_w,
             FastDiv(uint32_t(p.w)), FastDiv(uint32_t(p.h * p.w)), FastDiv(uint32_t(d.PW)),
             FastDiv(uint32_t(d.PH * d.PW)), FastDiv(uint32_t(p.stride_h)), FastDiv(uint32_t(p.stride_w)),
             FastDiv(uint32_t(p.h))};
  if (uint64_t(p.n) * p.c * p.h * p.w >= (1ull << 31))
    fail(CDNN_INVALID_ARGUMENT, "pool: tensors of 2^31 elements or more are not supported");
  return g;
}

}  // namespace
}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_pool_forward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle y, cdnn_handle mask,
                      cdnn_handle stream) {
  return cdnn_pool_forward_ex(ctx, desc, x, y, mask, 0, stream);
}

int cdnn_pool_forward_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle y, cdnn_handle mask, int flags,
                         cdnn_handle stream) {
  return guarded([&] {
    const bool relu = (flags & CDNN_POOL_RELU) != 0;
    Ctx* c = need_ctx(ctx);
    PoolDescSlot d = pool_desc(c, desc);
    BufferSlot& X = buffer(c, x, "pool x");
    BufferSlot& Y = buffer(c, y, "pool y");
    BufferSlot* M = buffer_or_null(c, mask, "pool mask");
    const PoolGeom g = geom_of(d);
    const uint64_t nin = uint64_t(g.N) * g.C * g.H * g.W, nout = uint64_t(g.N) * g.C * g.PH * g.PW;
    require_len(X, nin, "pool x");
    require_len(Y, nout, "pool y");
    require_dtype(Y, X.dtype, "pool");
    if (M) { require_len(*M, nout, "pool mask"); require_dtype(*M, CDNN_I32, "pool mask"); }
    DeviceGuard dg(c);
    cudaStream_t st = stream_of(c, stream);
    const int blocks = grid_for(int64_t(nout), 256);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      const T* xp = reinterpret_cast<const T*>(X.dev);
      T* yp = reinterpret_cast<T*>(Y.dev);
      int* mp = M ? reinterpret_cast<int*>(M->dev) : nullptr;
      if (d.p.method == CDNN_POOL_MAX) {
        const int fw = fixed_window(g);
        if (fw) {  // two outputs per thread
          const uint32_t PH2 = uint32_t(g.PH + 1) / 2, PHW2 = PH2 * uint32_t(g.PW);
          const uint64_t n2 = uint64_t(g.N) * g.C * PHW2;
          const int b2 = grid_for(int64_t(n2), 256);
          if (fw == 32)
            max_pool_fwd_k2<T, 3, 2><<<b2, 256, 0, st>>>(xp, yp, mp, g, g.divPW, FastDiv(PHW2), PHW2, uint32_t(n2),
                                                         relu);
          else
            max_pool_fwd_k2<T, 2, 2><<<b2, 256, 0, st>>>(xp, yp, mp, g, g.divPW, FastDiv(PHW2), PHW2, uint32_t(n2),
                                                         relu);
        } else {
          max_pool_fwd<T><<<blocks, 256, 0, st>>>(xp, yp, mp, g, uint32_t(nout), relu);
        }
      } else {
        switch (fixed_window(g)) {
          case 32: ave_pool_fwd_k<T, 3, 2><<<blocks, 256, 0, st>>>(xp, yp, g, uint32_t(nout), relu); break;
          case 22: ave_pool_fwd_k<T, 2, 2><<<blocks, 256, 0, st>>>(xp, yp, g, uint32_t(nout), relu); break;
          default: ave_pool_fwd<T><<<blocks, 256, 0, st>>>(xp, yp, g, uint32_t(nout), relu);
        }
      }
    };
    if (X.dtype == CDNN_F32) run(float{});
    else if (X.dtype == CDNN_F64) run(double{});
    else fail(CDNN_INVALID_ARGUMENT, "pool: floating buffers required");
    check_launch("pool_fwd");
    count_launch(c);
  });
}

int cdnn_pool_backward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle dy, cdnn_handle mask, cdnn_handle dx,
                       cdnn_handle stream) {
  return cdnn_pool_backward_ex(ctx, desc, dy, mask, dx, 0, stream);
}

int cdnn_pool_backward_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle dy, cdnn_handle mask, cdnn_handle dx,
                          cdnn_handle gate, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    PoolDescSlot d = pool_desc(c, desc);
    BufferSlot& DY = buffer(c, dy, "pool_bwd dy");
    BufferSlot& DX = buffer(c, dx, "pool_bwd dx");
    BufferSlot* M = buffer_or_null(c, mask, "pool_bwd mask");
    BufferSlot* G = buffer_or_null(c, gate, "pool_bwd gate");
    const PoolGeom g = geom_of(d);
    const uint64_t nin = uint64_t(g.N) * g.C * g.H * g.W, nout = uint64_t(g.N) * g.C * g.PH * g.PW;
    require_len(DY, nout, "pool_bwd dy");
    require_len(DX, nin, "pool_bwd dx");
    require_dtype(DX, DY.dtype, "pool_bwd");
    if (G) { require_len(*G, nin, "pool_bwd gate"); require_dtype(*G, DY.dtype, "pool_bwd gate"); }
    if (d.p.method == CDNN_POOL_MAX) {
      if (!M) fail(CDNN_INVALID_ARGUMENT, "pool_bwd: MAX pooling needs the argmax mask");
      require_len(*M, nout, "pool_bwd mask");
      require_dtype(*M, CDNN_I32, "pool_bwd mask");
    }
    DeviceGuard dg(c);
    cudaStream_t st = stream_of(c, stream);
    const int blocks = grid_for(int64_t(nin), 256);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      const int fw = fixed_window(g);
      const T* dyp = reinterpret_cast<const T*>(DY.dev);
      T* dxp = reinterpret_cast<T*>(DX.dev);
      const T* gp = G ? reinterpret_cast<const T*>(G->dev) : nullptr;
      if (fw && d.p.method == CDNN_POOL_MAX) {
        const int* mp = reinterpret_cast<const int*>(M->dev);
        // S x S blocks of bottom elements per thread (S = 2 for both fixed windows)
        const uint32_t BW = uint32_t(g.W + g.pw + 1) / 2, BH = uint32_t(g.H + g.ph + 1) / 2;
        const uint64_t nb = uint64_t(g.N) * g.C * BH * BW;
        const int bb = grid_for(int64_t(nb), 256);
        if (fw == 32)
          max_pool_bwd_blk<T, 3, 2><<<bb, 256, 0, st>>>(dyp, mp, dxp, g, FastDiv(BW), FastDiv(BH * BW), BW, BH * BW,
                                                         uint32_t(nb), gp);
        else
          max_pool_bwd_blk<T, 2, 2><<<bb, 256, 0, st>>>(dyp, mp, dxp, g, FastDiv(BW), FastDiv(BH * BW), BW, BH * BW,
                                                         uint32_t(nb), gp);
      } else if (fw) {
        if (fw == 32) ave_pool_bwd_k<T, 3, 2><<<blocks, 256, 0, st>>>(dyp, dxp, g, uint32_t(nin), gp);
        else ave_pool_bwd_k<T, 2, 2><<<blocks, 256, 0, st>>>(dyp, dxp, g, uint32_t(nin), gp);
      } else if (d.p.method == CDNN_POOL_MAX) {
        const uint64_t n4 = uint64_t(g.N) * g.C * g.H * ((g.W + 3) / 4);
        max_pool_bwd<T><<<grid_for(int64_t(n4), 256), 256, 0, st>>>(
            reinterpret_cast<const T*>(DY.dev), reinterpret_cast<const int*>(M->dev), reinterpret_cast<T*>(DX.dev), g,
            uint32_t(n4), G ? reinterpret_cast<const T*>(G->dev) : nullptr);
      }
      else
        ave_pool_bwd<T><<<blocks, 256, 0, st>>>(reinterpret_cast<const T*>(DY.dev), reinterpret_cast<T*>(DX.dev), g,
                                                 uint32_t(nin), G ? reinterpret_cast<const T*>(G->dev) : nullptr);
    };
    if (DY.dtype == CDNN_F32) run(float{});
    else if (DY.dtype == CDNN_F64) run(double{});
    else fail(CDNN_INVALID_ARGUMENT, "pool_bwd: floating buffers required");
    check_launch("pool_bwd");
    count_launch(c);
  });
}

}  // extern "C"
