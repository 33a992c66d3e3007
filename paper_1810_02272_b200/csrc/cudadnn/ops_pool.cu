// ops_pool.cu — Caffe pooling (absent from the reference).
//
// MAX: window scanned h-major then w, strict `>` so the first maximum wins;
//      the int32 mask holds the flat h*W+w index of the winner (bit-exact
//      integer output).  Backward gathers: each bottom element sums the top
//      diffs of the windows whose mask points at it (no atomics, deterministic).
// AVE: Caffe's divisor counts padded positions but not the overhang past
//      H+pad; backward spreads top_diff/pool_size over the clipped window.
// One thread per output (forward) / input (backward) element; NCHW planes.
#include "launch.cuh"

namespace cdnn {
namespace {

struct PoolGeom {
  int N, C, H, W, PH, PW, kh, kw, sh, sw, ph, pw;
};

template <typename T>
__global__ void max_pool_fwd(const T* __restrict__ x, T* __restrict__ y, int* __restrict__ mask, PoolGeom g) {
  const int64_t total = int64_t(g.N) * g.C * g.PH * g.PW;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int pw = int(i % g.PW);
    const int ph = int((i / g.PW) % g.PH);
    const int64_t nc = i / (int64_t(g.PW) * g.PH);
    int hs = ph * g.sh - g.ph, ws = pw * g.sw - g.pw;
    const int he = min(hs + g.kh, g.H), we = min(ws + g.kw, g.W);
    hs = max(hs, 0);
    ws = max(ws, 0);
    const T* plane = x + nc * g.H * g.W;
    T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
    int arg = -1;
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) {
        const T v = plane[h * g.W + w];
        if (v > best) { best = v; arg = h * g.W + w; }
      }
    y[i] = best;
    if (mask) mask[i] = arg;
  }
}

template <typename T>
__global__ void max_pool_bwd(const T* __restrict__ dy, const int* __restrict__ mask, T* __restrict__ dx, PoolGeom g) {
  const int64_t total = int64_t(g.N) * g.C * g.H * g.W;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int w = int(i % g.W);
    const int h = int((i / g.W) % g.H);
    const int64_t nc = i / (int64_t(g.W) * g.H);
    // windows [ph*sh - pad, +kh) that contain h
    const int phs = (h + g.ph < g.kh) ? 0 : (h + g.ph - g.kh) / g.sh + 1;
    const int phe = min((h + g.ph) / g.sh + 1, g.PH);
    const int pws = (w + g.pw < g.kw) ? 0 : (w + g.pw - g.kw) / g.sw + 1;
    const int pwe = min((w + g.pw) / g.sw + 1, g.PW);
    const int me = h * g.W + w;
    const int64_t base = nc * g.PH * g.PW;
    T s = T(0);
    for (int ph = phs; ph < phe; ++ph)
      for (int pw = pws; pw < pwe; ++pw)
        if (mask[base + ph * g.PW + pw] == me) s += dy[base + ph * g.PW + pw];
    dx[i] = s;
  }
}

template <typename T>
__global__ void ave_pool_fwd(const T* __restrict__ x, T* __restrict__ y, PoolGeom g) {
  const int64_t total = int64_t(g.N) * g.C * g.PH * g.PW;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int pw = int(i % g.PW);
    const int ph = int((i / g.PW) % g.PH);
    const int64_t nc = i / (int64_t(g.PW) * g.PH);
    int hs = ph * g.sh - g.ph, ws = pw * g.sw - g.pw;
    int he = min(hs + g.kh, g.H + g.ph), we = min(ws + g.kw, g.W + g.pw);
    const int pool = (he - hs) * (we - ws);
    hs = max(hs, 0); ws = max(ws, 0);
    he = min(he, g.H); we = min(we, g.W);
    const T* plane = x + nc * g.H * g.W;
    T s = T(0);
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) s += plane[h * g.W + w];
    y[i] = s / T(pool);
  }
}

template <typename T>
__global__ void ave_pool_bwd(const T* __restrict__ dy, T* __restrict__ dx, PoolGeom g) {
  const int64_t total = int64_t(g.N) * g.C * g.H * g.W;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int w = int(i % g.W) + g.pw;
    const int h = int((i / g.W) % g.H) + g.ph;
    const int64_t nc = i / (int64_t(g.W) * g.H);
    const int phs = (h < g.kh) ? 0 : (h - g.kh) / g.sh + 1;
    const int phe = min(h / g.sh + 1, g.PH);
    const int pws = (w < g.kw) ? 0 : (w - g.kw) / g.sw + 1;
    const int pwe = min(w / g.sw + 1, g.PW);
    const int64_t base = nc * g.PH * g.PW;
    T s = T(0);
    for (int ph = phs; ph < phe; ++ph)
      for (int pw = pws; pw < pwe; ++pw) {
        const int hs = ph * g.sh - g.ph, ws = pw * g.sw - g.pw;
        const int he = min(hs + g.kh, g.H + g.ph), we = min(ws + g.kw, g.W + g.pw);
        s += dy[base + ph * g.PW + pw] / T((he - hs) * (we - ws));
      }
    dx[i] = s;
  }
}

PoolGeom geom_of(const PoolDescSlot& d) {
  const auto& p = d.p;
  return PoolGeom{p.n, p.c, p.h, p.w, d.PH, d.PW, p.kernel_h, p.kernel_w, p.stride_h, p.stride_w, p.pad_h, p.pad_w};
}

}  // namespace
}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_pool_forward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle y, cdnn_handle mask,
                      cdnn_handle stream) {
  return guarded([&] {
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
      if (d.p.method == CDNN_POOL_MAX)
        max_pool_fwd<T><<<blocks, 256, 0, st>>>(reinterpret_cast<const T*>(X.dev), reinterpret_cast<T*>(Y.dev),
                                                 M ? reinterpret_cast<int*>(M->dev) : nullptr, g);
      else
        ave_pool_fwd<T><<<blocks, 256, 0, st>>>(reinterpret_cast<const T*>(X.dev), reinterpret_cast<T*>(Y.dev), g);
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
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    PoolDescSlot d = pool_desc(c, desc);
    BufferSlot& DY = buffer(c, dy, "pool_bwd dy");
    BufferSlot& DX = buffer(c, dx, "pool_bwd dx");
    BufferSlot* M = buffer_or_null(c, mask, "pool_bwd mask");
    const PoolGeom g = geom_of(d);
    const uint64_t nin = uint64_t(g.N) * g.C * g.H * g.W, nout = uint64_t(g.N) * g.C * g.PH * g.PW;
    require_len(DY, nout, "pool_bwd dy");
    require_len(DX, nin, "pool_bwd dx");
    require_dtype(DX, DY.dtype, "pool_bwd");
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
      if (d.p.method == CDNN_POOL_MAX)
        max_pool_bwd<T><<<blocks, 256, 0, st>>>(reinterpret_cast<const T*>(DY.dev), reinterpret_cast<const int*>(M->dev),
                                                 reinterpret_cast<T*>(DX.dev), g);
      else
        ave_pool_bwd<T><<<blocks, 256, 0, st>>>(reinterpret_cast<const T*>(DY.dev), reinterpret_cast<T*>(DX.dev), g);
    };
    if (DY.dtype == CDNN_F32) run(float{});
    else if (DY.dtype == CDNN_F64) run(double{});
    else fail(CDNN_INVALID_ARGUMENT, "pool_bwd: floating buffers required");
    check_launch("pool_bwd");
    count_launch(c);
  });
}

}  // extern "C"
