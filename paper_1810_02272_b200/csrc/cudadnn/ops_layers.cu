// ops_layers.cu — the remaining Caffe layers of the configs (absent from the
// reference): LRN (AlexNet), Dropout (AlexNet), BatchNorm + Scale + Eltwise
// (ResNet-20).  NCHW, one thread per element for the elementwise parts and one
// block per channel (fixed-shape tree -> deterministic) for the reductions.
//
// Dropout draws its mask from a counter-based hash of (seed, iteration, index)
// — identical on the CPU oracle and the GPU, recomputed in backward (no mask
// buffer), and the iteration counter lives in device memory so a captured CUDA
// graph draws a fresh mask on every replay.
#include "launch.cuh"
#include "lrn_math.cuh"

namespace cdnn {
namespace {

constexpr int kT = 256;

template <typename T>
T* P(const BufferSlot& b) { return reinterpret_cast<T*>(b.dev); }

template <class F>
void by_dtype(int dtype, const char* what, F&& f) {
  if (dtype == CDNN_F32) f(float{});
  else if (dtype == CDNN_F64) f(double{});
  else fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": floating buffers required");
}

int blocks(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, int64_t(kNumSMs) * 16))); }

// ---- LRN (ACROSS_CHANNELS): scale = k + alpha/n * sum_{window} x^2 ; y = x * scale^-beta
// One thread per pixel (img, hw) walks the channels with a running window sum
// (entering square added, leaving square subtracted; the leaving value is an
// L1 hit), so the tensor is read ~once, coalesced across threads (consecutive hw).
// (the arithmetic itself is lrn_math.cuh, shared with the fused LRN + pooling kernels)

// Forward: channels are processed in groups of four, the group's entering,
// leaving and own values loaded together before any arithmetic (12 independent
// loads in flight per thread; norm1 of AlexNet 267 -> 244 us).  The same
// restructuring of the backward measured slower (563 -> 777 us) and is not used.
constexpr int kLrnU = 4;

template <typename T>
__global__ void lrn_fwd(const T* __restrict__ x, T* __restrict__ y, T* __restrict__ scale, int N, int C, int HW,
                        int size, T alpha, T beta, T k) {
  const int64_t pixels = int64_t(N) * HW;
  const int pre = (size - 1) / 2, post = size - 1 - pre;
  const T aN = alpha / T(size);
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < pixels; p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t img = p / HW, hw = p - img * HW;
    const T* xb = x + img * C * HW + hw;
    const int64_t ob = img * C * HW + hw;
    T s = T(0);  // sum of squares over [c - pre, c + post]
    for (int cc = 0; cc < post && cc < C; ++cc) {
      const T v = __ldg(xb + int64_t(cc) * HW);
      s = lrn::sq_acc(s, v);
    }
    for (int c0 = 0; c0 < C; c0 += kLrnU) {
      T vin[kLrnU], vout[kLrnU], vx[kLrnU];
#pragma unroll
      for (int u = 0; u < kLrnU; ++u) {
        const int c = c0 + u, cin = c + post, cout = c - pre - 1;
        vin[u] = (c < C && cin < C) ? __ldg(xb + int64_t(cin) * HW) : T(0);
        vout[u] = (c < C && cout >= 0) ? __ldg(xb + int64_t(cout) * HW) : T(0);
        vx[u] = c < C ? __ldg(xb + int64_t(c) * HW) : T(0);
      }
#pragma unroll
      for (int u = 0; u < kLrnU; ++u) {
        const int c = c0 + u;
        if (c >= C) break;
        s = lrn::sq_acc(s, vin[u]);
        s = lrn::fma_(-vout[u], vout[u], s);
        s = s > T(0) ? s : T(0);
        const int64_t o = ob + int64_t(c) * HW;
        const T sc = lrn::scale(s, aN, k);
        scale[o] = sc;
        y[o] = lrn::top(vx[u], lrn::neg_pow(sc, beta));
      }
    }
  }
}

// dx = dy * scale^-beta - 2*alpha*beta/n * x * sum_{c' : c in window(c')} dy*y/scale
template <typename T>
__global__ void lrn_bwd(const T* __restrict__ x, const T* __restrict__ y, const T* __restrict__ scale,
                        const T* __restrict__ dy, T* __restrict__ dx, int N, int C, int HW, int size, T alpha, T beta,
                        const T* __restrict__ gate) {
  const int64_t pixels = int64_t(N) * HW;
  const int pre = (size - 1) / 2, post = size - 1 - pre;
  const T coef = T(2) * alpha * beta / T(size);
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < pixels; p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t img = p / HW, hw = p - img * HW;
    const int64_t base = img * C * HW + hw;
    auto t = [&](int cc) {
      const int64_t o = base + int64_t(cc) * HW;
      return lrn::term(dy[o], y[o], scale[o]);
    };
    T acc = T(0);  // sum of t over [c - post, c + pre]
    for (int cc = 0; cc < pre && cc < C; ++cc) acc = lrn::add_(acc, t(cc));
    for (int c = 0; c < C; ++c) {
      const int cin = c + pre, cout = c - post - 1;
      if (cin < C) acc = lrn::add_(acc, t(cin));
      if (cout >= 0) acc = lrn::sub_(acc, t(cout));
      const int64_t o = base + int64_t(c) * HW;
      const T g = lrn::grad(dy[o], lrn::neg_pow(scale[o], beta), coef, x[o], acc);
      dx[o] = (gate && !(gate[o] > T(0))) ? T(0) : g;
    }
  }
}

// Compile-time window (local_size 3 / 5, AlexNet uses 5): the window's values
// live in a register ring, so every tensor is read exactly once per pixel
// (forward: x; backward: x, y, scale, dy) and the leaving channel is never
// re-fetched; the entering channel's loads are issued kLrnU channels ahead.
template <typename T, int SIZE>
__global__ void lrn_fwd_ring(const T* __restrict__ x, T* __restrict__ y, T* __restrict__ scale, int N, int C, int HW,
                             T alpha, T beta, T k) {
  constexpr int pre = (SIZE - 1) / 2, post = SIZE - 1 - pre;
  const int64_t pixels = int64_t(N) * HW;
  const T aN = alpha / T(SIZE);
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < pixels; p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t img = p / HW, hw = p - img * HW;
    const int64_t base = img * C * HW + hw;
    T xr[SIZE];  // x of channels c - pre .. c + post (0 outside [0, C))
#pragma unroll
    for (int j = 0; j < SIZE; ++j) {
      const int cc = j - pre;
      xr[j] = (cc >= 0 && cc < C) ? __ldg(x + base + int64_t(cc) * HW) : T(0);
    }
    for (int c0 = 0; c0 < C; c0 += kLrnU) {
      T nx[kLrnU];  // entering channels c + post + 1 for the group's kLrnU channels
#pragma unroll
      for (int u = 0; u < kLrnU; ++u) {
        const int cin = c0 + u + post + 1;
        nx[u] = cin < C ? __ldg(x + base + int64_t(cin) * HW) : T(0);
      }
#pragma unroll
      for (int u = 0; u < kLrnU; ++u) {
        const int c = c0 + u;
        if (c >= C) break;
        T sum = T(0);
#pragma unroll
        for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xr[j]);
        const int64_t o = base + int64_t(c) * HW;
        const T sc = lrn::scale(sum, aN, k);
        scale[o] = sc;
        y[o] = lrn::top(xr[pre], lrn::neg_pow(sc, beta));
#pragma unroll
        for (int j = 0; j + 1 < SIZE; ++j) xr[j] = xr[j + 1];
        xr[SIZE - 1] = nx[u];
      }
    }
  }
}

template <typename T, int SIZE>
__global__ void lrn_bwd_ring(const T* __restrict__ x, const T* __restrict__ y, const T* __restrict__ scale,
                             const T* __restrict__ dy, T* __restrict__ dx, int N, int C, int HW, T alpha, T beta,
                             const T* __restrict__ gate) {
  constexpr int pre = (SIZE - 1) / 2, post = SIZE - 1 - pre;
  const int64_t pixels = int64_t(N) * HW;
  const T coef = T(2) * alpha * beta / T(SIZE);
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < pixels; p += int64_t(gridDim.x) * blockDim.x) {
    const int64_t img = p / HW, hw = p - img * HW;
    const int64_t base = img * C * HW + hw;
    // rings over channels c - post .. c + pre: t = dy*y/scale, and dy, scale for the output
    T tr[SIZE], dyr[SIZE], scr[SIZE];
#pragma unroll
    for (int j = 0; j < SIZE; ++j) {
      const int cc = j - post;
      if (cc >= 0 && cc < C) {
        const int64_t o = base + int64_t(cc) * HW;
        dyr[j] = __ldg(dy + o);
        scr[j] = __ldg(scale + o);
        tr[j] = lrn::term(dyr[j], __ldg(y + o), scr[j]);
      } else {
        dyr[j] = T(0); scr[j] = T(1); tr[j] = T(0);
      }
    }
    for (int c0 = 0; c0 < C; c0 += kLrnU) {
      T ndy[kLrnU], ny[kLrnU], nsc[kLrnU], xv[kLrnU];
#pragma unroll
      for (int u = 0; u < kLrnU; ++u) {
        const int c = c0 + u, cin = c + pre + 1;
        const bool in = cin < C;
        const int64_t oi = base + int64_t(in ? cin : 0) * HW;
        ndy[u] = in ? __ldg(dy + oi) : T(0);
        ny[u] = in ? __ldg(y + oi) : T(0);
        nsc[u] = in ? __ldg(scale + oi) : T(1);
        xv[u] = c < C ? __ldg(x + base + int64_t(c) * HW) : T(0);
      }
#pragma unroll
      for (int u = 0; u < kLrnU; ++u) {
        const int c = c0 + u;
        if (c >= C) break;
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < SIZE; ++j) acc = lrn::add_(acc, tr[j]);
        const T g = lrn::grad(dyr[post], lrn::neg_pow(scr[post], beta), coef, xv[u], acc);
        // fused backward of an in-place ReLU on this layer's bottom (gate = its data:
        // normally the very buffer x, whose value is already in a register)
        const bool open = !gate || (gate == x ? xv[u] > T(0) : __ldg(gate + base + int64_t(c) * HW) > T(0));
        dx[base + int64_t(c) * HW] = open ? g : T(0);
#pragma unroll
        for (int j = 0; j + 1 < SIZE; ++j) { tr[j] = tr[j + 1]; dyr[j] = dyr[j + 1]; scr[j] = scr[j + 1]; }
        dyr[SIZE - 1] = ndy[u];
        scr[SIZE - 1] = nsc[u];
        tr[SIZE - 1] = lrn::term(ndy[u], ny[u], nsc[u]);
      }
    }
  }
}

// ---- Dropout --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t drop_hash(uint64_t seed, uint64_t iter, uint64_t idx) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull ^ (iter + 1) * 0xBF58476D1CE4E5B9ull ^ (idx + 1) * 0x94D049BB133111EBull;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return uint32_t(z >> 32);
}

template <typename T>
__global__ void dropout_kernel(const T* __restrict__ in, T* __restrict__ out, uint64_t n, uint32_t threshold, T scale,
                               uint64_t seed, const unsigned long long* __restrict__ iter) {
  const uint64_t it = *iter;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = drop_hash(seed, it, i) > threshold ? in[i] * scale : T(0);
}

__global__ void bump_kernel(unsigned long long* iter) { *iter += 1; }

// ---- BatchNorm (training statistics), Scale, Eltwise ----------------------------------
// Per-channel sums over (N, HW) are two-level and deterministic: grid (C, splits),
// each block reduces a fixed range of images into one double pair (fixed-shape
// tree), then one thread per channel adds the split partials in order.  The
// elementwise passes index by plane (blockIdx.y = img*C + c): no per-element
// division, float4 when HW % 4 == 0.

enum ChanOp { kSumSq = 0, kSumDot = 1 };  // (x, x*x) | (a, a*b)

// 16-byte packs (4 floats / 2 doubles): the per-channel passes walk a block's planes as
// one flat run of packs (HW % W == 0: no pack crosses a plane), so every thread is busy
// even on 8 x 8 planes (a thread per plane element left 3/4 of a 256-thread block idle)
template <typename T>
struct alignas(16) Pk {
  static constexpr int W = 16 / int(sizeof(T));
  T v[W];
};
template <typename T>
__device__ __forceinline__ bool packable(const T* p, int HW) {
  return HW % Pk<T>::W == 0 && (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

template <typename T, int OP>
__global__ void __launch_bounds__(kT) chan_partials(const T* __restrict__ u, const T* __restrict__ w, double2* part,
                                                    int N, int C, int HW, int splits) {
  __shared__ double sh0[kT], sh1[kT];
  const int c = blockIdx.x, sp = blockIdx.y;
  const int n0 = int(int64_t(N) * sp / splits), n1 = int(int64_t(N) * (sp + 1) / splits);
  double s0 = 0, s1 = 0;
  constexpr int W = Pk<T>::W;
  if (packable(u, HW) && (OP == kSumSq || packable(w, HW))) {
    const uint32_t hwv = uint32_t(HW / W), total = uint32_t(n1 - n0) * hwv;
    const Pk<T>* up = reinterpret_cast<const Pk<T>*>(u);
    const Pk<T>* wp = reinterpret_cast<const Pk<T>*>(w);
    for (uint32_t j = threadIdx.x; j < total; j += kT) {
      const uint32_t k = j / hwv, i = j - k * hwv;
      const int64_t off = (int64_t(n0 + int(k)) * C + c) * hwv + i;
      const Pk<T> a = up[off];
      if (OP == kSumSq) {
#pragma unroll
        for (int e = 0; e < W; ++e) { const double v = double(a.v[e]); s0 += v; s1 += v * v; }
      } else {
        const Pk<T> b = wp[off];
#pragma unroll
        for (int e = 0; e < W; ++e) { const double v = double(a.v[e]); s0 += v; s1 += v * double(b.v[e]); }
      }
    }
  } else {
    for (int n = n0; n < n1; ++n) {
      const int64_t off = (int64_t(n) * C + c) * HW;
      for (int i = threadIdx.x; i < HW; i += kT) {
        const double a = double(u[off + i]);
        if (OP == kSumSq) { s0 += a; s1 += a * a; }
        else { s0 += a; s1 += a * double(w[off + i]); }
      }
    }
  }
  sh0[threadIdx.x] = s0;
  sh1[threadIdx.x] = s1;
  __syncthreads();
  for (int k = kT / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) { sh0[threadIdx.x] += sh0[threadIdx.x + k]; sh1[threadIdx.x] += sh1[threadIdx.x + k]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[int64_t(c) * splits + sp] = make_double2(sh0[0], sh1[0]);
}

// A channel-major elementwise pass: block (c, sp) covers channel c of images
// [n0, n1) (the chan_partials split), f(base offset, count) applied pack by pack
template <typename T, class F>
__device__ __forceinline__ void chan_apply(int N, int C, int HW, int splits, bool packed, F f) {
  const int c = blockIdx.x, sp = blockIdx.y;
  const int n0 = int(int64_t(N) * sp / splits), n1 = int(int64_t(N) * (sp + 1) / splits);
  if (packed) {
    constexpr int W = Pk<T>::W;
    const uint32_t hwv = uint32_t(HW / W), total = uint32_t(n1 - n0) * hwv;
    for (uint32_t j = threadIdx.x; j < total; j += kT) {
      const uint32_t k = j / hwv, i = j - k * hwv;
      f((int64_t(n0 + int(k)) * C + c) * hwv + i, std::integral_constant<bool, true>{});
    }
  } else {
    for (int n = n0; n < n1; ++n)
      for (int i = threadIdx.x; i < HW; i += kT) f((int64_t(n) * C + c) * HW + i, std::integral_constant<bool, false>{});
  }
}

__device__ __forceinline__ double2 sum_parts(const double2* part, int c, int splits) {
  double s0 = 0, s1 = 0;
  for (int k = 0; k < splits; ++k) { s0 += part[int64_t(c) * splits + k].x; s1 += part[int64_t(c) * splits + k].y; }
  return make_double2(s0, s1);
}

template <typename T>
__global__ void bn_finalize(const double2* part, int splits, int C, double cnt, double eps, T* mean, T* invstd) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double2 s = sum_parts(part, c, splits);
  const double m = s.x / cnt, var = s.y / cnt - m * m;
  mean[c] = T(m);
  invstd[c] = T(1.0 / sqrt(var + eps));
}

// a = mean(dy), b = mean(dy*y)
template <typename T>
__global__ void bn_bwd_finalize(const double2* part, int splits, int C, double cnt, T* a, T* b) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double2 s = sum_parts(part, c, splits);
  a[c] = T(s.x / cnt);
  b[c] = T(s.y / cnt);
}

// dbeta += sum dy ; dgamma += sum dy*x
template <typename T>
__global__ void scale_finalize(const double2* part, int splits, int C, T* dg, T* db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double2 s = sum_parts(part, c, splits);
  if (db) db[c] += T(s.x);
  if (dg) dg[c] += T(s.y);
}

// Plane-indexed elementwise: out = f(i, c) over plane (img, c); F(v0, v1, c) per element.
template <typename T, class F>
__device__ __forceinline__ void plane_apply(T* __restrict__ out, int64_t off, int HW, F f) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += gridDim.x * blockDim.x) out[off + i] = f(off + i);
}

template <typename T>
__global__ void bn_apply(const T* __restrict__ x, const T* __restrict__ mean, const T* __restrict__ invstd,
                         T* __restrict__ y, int C, int HW) {
  const int c = blockIdx.y % C;
  const T m = mean[c], is = invstd[c];
  const int64_t off = int64_t(blockIdx.y) * HW;
  plane_apply(y, off, HW, [&](int64_t i) { return (x[i] - m) * is; });
}

template <typename T>
__global__ void bn_bwd_apply(const T* __restrict__ y, const T* __restrict__ dy, const T* __restrict__ a,
                             const T* __restrict__ b, const T* __restrict__ invstd, T* __restrict__ dx, int C, int HW) {
  const int c = blockIdx.y % C;
  const T ac = a[c], bc = b[c], is = invstd[c];
  const int64_t off = int64_t(blockIdx.y) * HW;
  plane_apply(dx, off, HW, [&](int64_t i) { return (dy[i] - ac - y[i] * bc) * is; });
}

template <typename T>
__global__ void scale_fwd(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ bta,
                          T* __restrict__ y, int C, int HW) {
  const int c = blockIdx.y % C;
  const T gc = g[c], bc = bta ? bta[c] : T(0);
  const int64_t off = int64_t(blockIdx.y) * HW;
  plane_apply(y, off, HW, [&](int64_t i) { return x[i] * gc + bc; });
}

template <typename T>
__global__ void scale_bwd_data(const T* __restrict__ dy, const T* __restrict__ g, T* __restrict__ dx, int C, int HW) {
  const int c = blockIdx.y % C;
  const T gc = g[c];
  const int64_t off = int64_t(blockIdx.y) * HW;
  plane_apply(dx, off, HW, [&](int64_t i) { return dy[i] * gc; });
}

// ---- fused BatchNorm + Scale (z = gamma*xn + beta, xn = (x - mean)*invstd) ----------
// backward sums (S0 = sum dz, S1 = sum dz*xn): dbeta += S0, dgamma += S1,
// a = S0/M, b = S1/M for dx = gamma*invstd*(dz - a - xn*b)
template <typename T>
__global__ void bn_scale_finalize(const double2* part, int splits, int C, double cnt, T* dg, T* db, T* a, T* b) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double2 s = sum_parts(part, c, splits);
  if (db) db[c] += T(s.x);
  if (dg) dg[c] += T(s.y);
  a[c] = T(s.x / cnt);
  b[c] = T(s.y / cnt);
}

// The channel's split partials summed by warp 0 (lane-strided, then a fixed xor tree):
// one round of parallel loads instead of `splits` dependent ones; deterministic.
__device__ __forceinline__ double2 sum_parts_warp(const double2* part, int c, int splits) {
  double s0 = 0, s1 = 0;
  for (int k = int(threadIdx.x); k < splits; k += 32) {
    const double2 v = part[int64_t(c) * splits + k];
    s0 += v.x;
    s1 += v.y;
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, m);
    s1 += __shfl_xor_sync(0xffffffffu, s1, m);
  }
  return make_double2(s0, s1);
}

// Fused BatchNorm + Scale passes on the chan_partials grid with the finalize folded in:
// each block sums the channel's split partials (bn_finalize's / bn_scale_finalize's
// formulas), block (c, 0) stores the statistics / accumulates dgamma,
// dbeta -- two launches per pass instead of three.
template <typename T>
__global__ void __launch_bounds__(kT) bn_scale_apply_c(const T* __restrict__ x, const double2* __restrict__ part,
                                                       int splits, double cnt, double eps, T* __restrict__ mean,
                                                       T* __restrict__ invstd, const T* __restrict__ g,
                                                       const T* __restrict__ bta, T* __restrict__ xn,
                                                       T* __restrict__ z, int N, int C, int HW, bool relu) {
  __shared__ T st[2];
  const int c = blockIdx.x;
  if (threadIdx.x < 32) {
    const double2 s = sum_parts_warp(part, c, splits);
    if (threadIdx.x == 0) {
      const double m = s.x / cnt, var = s.y / cnt - m * m;
      st[0] = T(m);
      st[1] = T(1.0 / sqrt(var + eps));
      if (blockIdx.y == 0) { mean[c] = st[0]; invstd[c] = st[1]; }
    }
  }
  __syncthreads();
  const T m = st[0], is = st[1], gc = g[c], bc = bta ? bta[c] : T(0);
  const bool packed = packable(x, HW) && packable(xn, HW) && packable(z, HW);
  chan_apply<T>(N, C, HW, splits, packed, [&](int64_t o, auto pk) {
    if constexpr (decltype(pk)::value) {
      Pk<T> a = reinterpret_cast<const Pk<T>*>(x)[o], b;
#pragma unroll
      for (int e = 0; e < Pk<T>::W; ++e) {
        a.v[e] = (a.v[e] - m) * is;
        b.v[e] = a.v[e] * gc + bc;
        if (relu) b.v[e] = b.v[e] > T(0) ? b.v[e] : T(0);
      }
      reinterpret_cast<Pk<T>*>(xn)[o] = a;
      reinterpret_cast<Pk<T>*>(z)[o] = b;
    } else {
      const T v = (x[o] - m) * is;
      xn[o] = v;
      const T zv = v * gc + bc;
      z[o] = relu ? (zv > T(0) ? zv : T(0)) : zv;
    }
  });
}

template <typename T>
__global__ void __launch_bounds__(kT) bn_scale_bwd_apply_c(const T* __restrict__ xn, const T* __restrict__ dz,
                                                           const double2* __restrict__ part, int splits, double cnt,
                                                           const T* __restrict__ invstd, const T* __restrict__ g,
                                                           T* __restrict__ dg, T* __restrict__ db,
                                                           T* __restrict__ dx, int N, int C, int HW) {
  __shared__ T st[2];
  const int c = blockIdx.x;
  if (threadIdx.x < 32) {
    const double2 s = sum_parts_warp(part, c, splits);
    if (threadIdx.x == 0) {
      if (blockIdx.y == 0) {
        if (db) db[c] += T(s.x);
        if (dg) dg[c] += T(s.y);
      }
      st[0] = T(s.x / cnt);
      st[1] = T(s.y / cnt);
    }
  }
  __syncthreads();
  const T ac = st[0], bc = st[1], k = invstd[c] * g[c];
  const bool packed = packable(xn, HW) && packable(dz, HW) && packable(dx, HW);
  chan_apply<T>(N, C, HW, splits, packed, [&](int64_t o, auto pk) {
    if constexpr (decltype(pk)::value) {
      const Pk<T> a = reinterpret_cast<const Pk<T>*>(xn)[o];
      Pk<T> d = reinterpret_cast<const Pk<T>*>(dz)[o];
#pragma unroll
      for (int e = 0; e < Pk<T>::W; ++e) d.v[e] = (d.v[e] - ac - a.v[e] * bc) * k;
      reinterpret_cast<Pk<T>*>(dx)[o] = d;
    } else {
      dx[o] = (dz[o] - ac - xn[o] * bc) * k;
    }
  });
}

// ---- policy-gradient diff injection (trainer.cpp:42-113 restated on the device) ----------
// softmax: dlogit[r][c] = (p[r][c] - [c == a_r]) * G_r        (dlogps_softmax, sign +1)
// sigmoid: dlogit[r][0] = -((a_r == 0 ? 1 - p : -p) * G_r)    (dlogps_sigmoid, sign -1)
// rows >= n (padding of a fixed-batch net) get 0, so they add nothing to the gradients.
template <typename T>
__global__ void pg_diff_kernel(const T* __restrict__ prob, const T* __restrict__ act, const T* __restrict__ ret,
                               T* __restrict__ dlogit, int rows, int n, int classes, int sigmoid) {
  const int64_t total = int64_t(rows) * classes;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int r = int(i / classes), c = int(i - int64_t(r) * classes);
    T v = T(0);
    if (r < n) {
      const int a = int(act[r]);
      const T p = prob[i], g = ret[r];
      if (sigmoid) v = -((a == 0 ? T(1) - p : T(0) - p) * g);
      else v = (p - (c == a ? T(1) : T(0))) * g;
    }
    dlogit[i] = v;
  }
}

// launch helpers: splits so each partial block covers ~32k elements; plane grid
inline int chan_splits(int N, int C, int HW) {
  // >= 4 blocks per SM in total, >= 2048 elements per block, <= N
  const int64_t want = (4 * kNumSMs + C - 1) / C;
  const int64_t cap = std::max<int64_t>(1, int64_t(N) * HW / 2048);
  return int(std::max<int64_t>(1, std::min<int64_t>({int64_t(N), want, cap})));
}
inline dim3 plane_grid(int N, int C, int HW) {
  return dim3(unsigned(std::max(1, std::min((HW + kT - 1) / kT, 64))), unsigned(N * C));
}

template <typename T>
__global__ void axpby_kernel(const T* __restrict__ x, T* __restrict__ y, uint64_t n, T a, T b, bool read_y) {
  constexpr int W = Pk<T>::W;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u) == 0) {  // 16-byte packs
    for (uint64_t j = i; j < n / W; j += stride) {
      const Pk<T> xv = reinterpret_cast<const Pk<T>*>(x)[j];
      Pk<T> yv;
      if (read_y) yv = reinterpret_cast<const Pk<T>*>(y)[j];
#pragma unroll
      for (int e = 0; e < W; ++e) yv.v[e] = read_y ? a * xv.v[e] + b * yv.v[e] : a * xv.v[e];
      reinterpret_cast<Pk<T>*>(y)[j] = yv;
    }
    i += n / W * W;
  }
  for (; i < n; i += stride) y[i] = read_y ? a * x[i] + b * y[i] : a * x[i];
}

}  // namespace
}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_lrn_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle scale, int n, int c, int hw,
                     int local_size, double alpha, double beta, double k, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    if (n < 1 || c < 1 || hw < 1 || local_size < 1 || local_size % 2 == 0)
      fail(CDNN_INVALID_ARGUMENT, "lrn: bad extents or even local_size");
    BufferSlot& X = buffer(cx, x, "lrn x");
    BufferSlot& Y = buffer(cx, y, "lrn y");
    BufferSlot& S = buffer(cx, scale, "lrn scale");
    const uint64_t cnt = uint64_t(n) * c * hw;
    for (BufferSlot* b : {&X, &Y, &S}) { require_len(*b, cnt, "lrn"); require_dtype(*b, X.dtype, "lrn"); }
    DeviceGuard g(cx);
    by_dtype(X.dtype, "lrn", [&](auto tag) {
      using T = decltype(tag);
      cudaStream_t st = stream_of(cx, stream);
      const int nb = blocks(int64_t(n) * hw);
      if (local_size == 5)
        lrn_fwd_ring<T, 5><<<nb, kT, 0, st>>>(P<T>(X), P<T>(Y), P<T>(S), n, c, hw, T(alpha), T(beta), T(k));
      else if (local_size == 3)
        lrn_fwd_ring<T, 3><<<nb, kT, 0, st>>>(P<T>(X), P<T>(Y), P<T>(S), n, c, hw, T(alpha), T(beta), T(k));
      else
        lrn_fwd<T><<<nb, kT, 0, st>>>(P<T>(X), P<T>(Y), P<T>(S), n, c, hw, local_size, T(alpha), T(beta), T(k));
    });
    check_launch("lrn_fwd");
    count_launch(cx);
  });
}

int cdnn_lrn_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle scale, cdnn_handle dy, cdnn_handle dx,
                      int n, int c, int hw, int local_size, double alpha, double beta, cdnn_handle stream) {
  return cdnn_lrn_backward_ex(ctx, x, y, scale, dy, dx, n, c, hw, local_size, alpha, beta, 0, stream);
}

int cdnn_lrn_backward_ex(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle scale, cdnn_handle dy, cdnn_handle dx,
                         int n, int c, int hw, int local_size, double alpha, double beta, cdnn_handle gate,
                         cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "lrn_bwd x");
    BufferSlot& Y = buffer(cx, y, "lrn_bwd y");
    BufferSlot& S = buffer(cx, scale, "lrn_bwd scale");
    BufferSlot& DY = buffer(cx, dy, "lrn_bwd dy");
    BufferSlot& DX = buffer(cx, dx, "lrn_bwd dx");
    BufferSlot* G = buffer_or_null(cx, gate, "lrn_bwd gate");
    const uint64_t cnt = uint64_t(n) * c * hw;
    for (BufferSlot* b : {&X, &Y, &S, &DY, &DX, G})
      if (b) { require_len(*b, cnt, "lrn_bwd"); require_dtype(*b, X.dtype, "lrn_bwd"); }
    DeviceGuard g(cx);
    by_dtype(X.dtype, "lrn_bwd", [&](auto tag) {
      using T = decltype(tag);
      cudaStream_t st = stream_of(cx, stream);
      const int nb = blocks(int64_t(n) * hw);
      const T* gp = G ? reinterpret_cast<const T*>(G->dev) : nullptr;
      if (local_size == 5)
        lrn_bwd_ring<T, 5><<<nb, kT, 0, st>>>(P<T>(X), P<T>(Y), P<T>(S), P<T>(DY), P<T>(DX), n, c, hw, T(alpha), T(beta), gp);
      else if (local_size == 3)
        lrn_bwd_ring<T, 3><<<nb, kT, 0, st>>>(P<T>(X), P<T>(Y), P<T>(S), P<T>(DY), P<T>(DX), n, c, hw, T(alpha), T(beta), gp);
      else
        lrn_bwd<T><<<nb, kT, 0, st>>>(P<T>(X), P<T>(Y), P<T>(S), P<T>(DY), P<T>(DX), n, c, hw, local_size, T(alpha),
                                      T(beta), gp);
    });
    check_launch("lrn_bwd");
    count_launch(cx);
  });
}

int cdnn_dropout(cdnn_ctx ctx, cdnn_handle in, cdnn_handle out, uint64_t n, double ratio, uint64_t seed,
                 cdnn_handle counter, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    if (!(ratio >= 0.0 && ratio < 1.0)) fail(CDNN_INVALID_ARGUMENT, "dropout: ratio must be in [0, 1)");
    BufferSlot& I = buffer(cx, in, "dropout in");
    BufferSlot& O = buffer(cx, out, "dropout out");
    BufferSlot& K = buffer(cx, counter, "dropout counter");
    require_len(I, n, "dropout");
    require_len(O, n, "dropout");
    require_dtype(O, I.dtype, "dropout");
    if (K.len * dtype_size(K.dtype) < 8) fail(CDNN_INVALID_ARGUMENT, "dropout: counter buffer needs 8 bytes");
    DeviceGuard g(cx);
    const uint32_t thr = uint32_t(std::min(4294967295.0, ratio * 4294967296.0));
    by_dtype(I.dtype, "dropout", [&](auto tag) {
      using T = decltype(tag);
      dropout_kernel<T><<<blocks(int64_t(n)), kT, 0, stream_of(cx, stream)>>>(
          P<T>(I), P<T>(O), n, thr, T(1.0 / (1.0 - ratio)), seed, reinterpret_cast<unsigned long long*>(K.dev));
    });
    check_launch("dropout");
    count_launch(cx);
  });
}

int cdnn_counter_increment(cdnn_ctx ctx, cdnn_handle counter, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& K = buffer(cx, counter, "counter");
    if (K.len * dtype_size(K.dtype) < 8) fail(CDNN_INVALID_ARGUMENT, "counter buffer needs 8 bytes");
    DeviceGuard g(cx);
    bump_kernel<<<1, 1, 0, stream_of(cx, stream)>>>(reinterpret_cast<unsigned long long*>(K.dev));
    check_launch("counter");
    count_launch(cx);
  });
}

int cdnn_batchnorm_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle mean, cdnn_handle invstd, int n,
                           int c, int hw, double eps, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "bn x");
    BufferSlot& Y = buffer(cx, y, "bn y");
    BufferSlot& M = buffer(cx, mean, "bn mean");
    BufferSlot& V = buffer(cx, invstd, "bn invstd");
    const uint64_t cnt = uint64_t(n) * c * hw;
    require_len(X, cnt, "bn"); require_len(Y, cnt, "bn"); require_len(M, uint64_t(c), "bn"); require_len(V, uint64_t(c), "bn");
    for (BufferSlot* b : {&Y, &M, &V}) require_dtype(*b, X.dtype, "bn");
    if (n * c > 65535) fail(CDNN_INVALID_ARGUMENT, "bn: n*c must be <= 65535");
    DeviceGuard g(cx);
    cudaStream_t st = stream_of(cx, stream);
    const int splits = chan_splits(n, c, hw);
    double2* part = static_cast<double2*>(workspace_of(cx, stream).get(size_t(c) * splits * sizeof(double2), cx->device));
    by_dtype(X.dtype, "bn", [&](auto tag) {
      using T = decltype(tag);
      chan_partials<T, kSumSq><<<dim3(c, splits), kT, 0, st>>>(P<T>(X), nullptr, part, n, c, hw, splits);
      bn_finalize<T><<<(c + 127) / 128, 128, 0, st>>>(part, splits, c, double(n) * hw, eps, P<T>(M), P<T>(V));
      bn_apply<T><<<plane_grid(n, c, hw), kT, 0, st>>>(P<T>(X), P<T>(M), P<T>(V), P<T>(Y), c, hw);
    });
    check_launch("bn_fwd");
    count_launch(cx, 3);
  });
}

int cdnn_batchnorm_backward(cdnn_ctx ctx, cdnn_handle y, cdnn_handle invstd, cdnn_handle dy, cdnn_handle dx,
                            cdnn_handle scratch, int n, int c, int hw, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& Y = buffer(cx, y, "bn_bwd y");
    BufferSlot& V = buffer(cx, invstd, "bn_bwd invstd");
    BufferSlot& DY = buffer(cx, dy, "bn_bwd dy");
    BufferSlot& DX = buffer(cx, dx, "bn_bwd dx");
    BufferSlot& S = buffer(cx, scratch, "bn_bwd scratch");
    const uint64_t cnt = uint64_t(n) * c * hw;
    require_len(Y, cnt, "bn_bwd"); require_len(DY, cnt, "bn_bwd"); require_len(DX, cnt, "bn_bwd");
    require_len(V, uint64_t(c), "bn_bwd"); require_len(S, 2 * uint64_t(c), "bn_bwd scratch");
    for (BufferSlot* b : {&V, &DY, &DX, &S}) require_dtype(*b, Y.dtype, "bn_bwd");
    if (n * c > 65535) fail(CDNN_INVALID_ARGUMENT, "bn_bwd: n*c must be <= 65535");
    DeviceGuard g(cx);
    cudaStream_t st = stream_of(cx, stream);
    const int splits = chan_splits(n, c, hw);
    double2* part = static_cast<double2*>(workspace_of(cx, stream).get(size_t(c) * splits * sizeof(double2), cx->device));
    by_dtype(Y.dtype, "bn_bwd", [&](auto tag) {
      using T = decltype(tag);
      T* a = P<T>(S);
      T* b = a + c;
      chan_partials<T, kSumDot><<<dim3(c, splits), kT, 0, st>>>(P<T>(DY), P<T>(Y), part, n, c, hw, splits);
      bn_bwd_finalize<T><<<(c + 127) / 128, 128, 0, st>>>(part, splits, c, double(n) * hw, a, b);
      bn_bwd_apply<T><<<plane_grid(n, c, hw), kT, 0, st>>>(P<T>(Y), P<T>(DY), a, b, P<T>(V), P<T>(DX), c, hw);
    });
    check_launch("bn_bwd");
    count_launch(cx, 3);
  });
}

int cdnn_scale_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle gamma, cdnn_handle beta, cdnn_handle y, int n, int c,
                       int hw, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "scale x");
    BufferSlot& G = buffer(cx, gamma, "scale gamma");
    BufferSlot* B = buffer_or_null(cx, beta, "scale beta");
    BufferSlot& Y = buffer(cx, y, "scale y");
    const uint64_t cnt = uint64_t(n) * c * hw;
    require_len(X, cnt, "scale"); require_len(Y, cnt, "scale"); require_len(G, uint64_t(c), "scale");
    if (B) { require_len(*B, uint64_t(c), "scale"); require_dtype(*B, X.dtype, "scale"); }
    require_dtype(G, X.dtype, "scale"); require_dtype(Y, X.dtype, "scale");
    if (n * c > 65535) fail(CDNN_INVALID_ARGUMENT, "scale: n*c must be <= 65535");
    DeviceGuard g(cx);
    by_dtype(X.dtype, "scale", [&](auto tag) {
      using T = decltype(tag);
      scale_fwd<T><<<plane_grid(n, c, hw), kT, 0, stream_of(cx, stream)>>>(P<T>(X), P<T>(G),
                                                                          B ? P<T>(*B) : nullptr, P<T>(Y), c, hw);
    });
    check_launch("scale_fwd");
    count_launch(cx);
  });
}

int cdnn_scale_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle gamma, cdnn_handle dy, cdnn_handle dgamma,
                        cdnn_handle dbeta, cdnn_handle dx, int n, int c, int hw, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "scale_bwd x");
    BufferSlot& G = buffer(cx, gamma, "scale_bwd gamma");
    BufferSlot& DY = buffer(cx, dy, "scale_bwd dy");
    BufferSlot* DG = buffer_or_null(cx, dgamma, "scale_bwd dgamma");
    BufferSlot* DB = buffer_or_null(cx, dbeta, "scale_bwd dbeta");
    BufferSlot* DX = buffer_or_null(cx, dx, "scale_bwd dx");
    const uint64_t cnt = uint64_t(n) * c * hw;
    require_len(X, cnt, "scale_bwd"); require_len(DY, cnt, "scale_bwd"); require_len(G, uint64_t(c), "scale_bwd");
    if (DX) require_len(*DX, cnt, "scale_bwd dx");
    if (n * c > 65535) fail(CDNN_INVALID_ARGUMENT, "scale_bwd: n*c must be <= 65535");
    DeviceGuard g(cx);
    cudaStream_t st = stream_of(cx, stream);
    by_dtype(X.dtype, "scale_bwd", [&](auto tag) {
      using T = decltype(tag);
      if (DG || DB) {
        const int splits = chan_splits(n, c, hw);
        double2* part =
            static_cast<double2*>(workspace_of(cx, stream).get(size_t(c) * splits * sizeof(double2), cx->device));
        chan_partials<T, kSumDot><<<dim3(c, splits), kT, 0, st>>>(P<T>(DY), P<T>(X), part, n, c, hw, splits);
        scale_finalize<T><<<(c + 127) / 128, 128, 0, st>>>(part, splits, c, DG ? P<T>(*DG) : nullptr,
                                                          DB ? P<T>(*DB) : nullptr);
        count_launch(cx, 2);
      }
      if (DX) {
        scale_bwd_data<T><<<plane_grid(n, c, hw), kT, 0, st>>>(P<T>(DY), P<T>(G), P<T>(*DX), c, hw);
        count_launch(cx);
      }
    });
    check_launch("scale_bwd");
  });
}

int cdnn_batchnorm_scale_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle xnorm, cdnn_handle z, cdnn_handle mean,
                                 cdnn_handle invstd, cdnn_handle gamma, cdnn_handle beta, int n, int c, int hw,
                                 double eps, cdnn_handle stream) {
  return cdnn_batchnorm_scale_forward_ex(ctx, x, xnorm, z, mean, invstd, gamma, beta, n, c, hw, eps, 0, stream);
}

int cdnn_batchnorm_scale_forward_ex(cdnn_ctx ctx, cdnn_handle x, cdnn_handle xnorm, cdnn_handle z, cdnn_handle mean,
                                    cdnn_handle invstd, cdnn_handle gamma, cdnn_handle beta, int n, int c, int hw,
                                    double eps, int flags, cdnn_handle stream) {
  return guarded([&] {
    const bool relu = (flags & CDNN_BN_RELU) != 0;
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "bn_scale x");
    BufferSlot& XN = buffer(cx, xnorm, "bn_scale xnorm");
    BufferSlot& Z = buffer(cx, z, "bn_scale z");
    BufferSlot& M = buffer(cx, mean, "bn_scale mean");
    BufferSlot& V = buffer(cx, invstd, "bn_scale invstd");
    BufferSlot& G = buffer(cx, gamma, "bn_scale gamma");
    BufferSlot* B = buffer_or_null(cx, beta, "bn_scale beta");
    const uint64_t cnt = uint64_t(n) * c * hw;
    for (BufferSlot* b : {&X, &XN, &Z}) require_len(*b, cnt, "bn_scale");
    for (BufferSlot* b : {&M, &V, &G}) require_len(*b, uint64_t(c), "bn_scale");
    if (B) require_len(*B, uint64_t(c), "bn_scale");
    for (BufferSlot* b : {&XN, &Z, &M, &V, &G, B}) if (b) require_dtype(*b, X.dtype, "bn_scale");
    if (n * c > 65535) fail(CDNN_INVALID_ARGUMENT, "bn_scale: n*c must be <= 65535");
    DeviceGuard g(cx);
    cudaStream_t st = stream_of(cx, stream);
    const int splits = chan_splits(n, c, hw);
    double2* part = static_cast<double2*>(workspace_of(cx, stream).get(size_t(c) * splits * sizeof(double2), cx->device));
    by_dtype(X.dtype, "bn_scale", [&](auto tag) {
      using T = decltype(tag);
      chan_partials<T, kSumSq><<<dim3(c, splits), kT, 0, st>>>(P<T>(X), nullptr, part, n, c, hw, splits);
      bn_scale_apply_c<T><<<dim3(c, splits), kT, 0, st>>>(P<T>(X), part, splits, double(n) * hw, eps, P<T>(M), P<T>(V),
                                                         P<T>(G), B ? P<T>(*B) : nullptr, P<T>(XN), P<T>(Z), n, c, hw,
                                                         relu);
    });
    check_launch("bn_scale_fwd");
    count_launch(cx, 2);
  });
}

int cdnn_batchnorm_scale_backward(cdnn_ctx ctx, cdnn_handle xnorm, cdnn_handle invstd, cdnn_handle gamma,
                                  cdnn_handle dz, cdnn_handle dx, cdnn_handle dgamma, cdnn_handle dbeta,
                                  cdnn_handle scratch, int n, int c, int hw, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& XN = buffer(cx, xnorm, "bn_scale_bwd xnorm");
    BufferSlot& V = buffer(cx, invstd, "bn_scale_bwd invstd");
    BufferSlot& G = buffer(cx, gamma, "bn_scale_bwd gamma");
    BufferSlot& DZ = buffer(cx, dz, "bn_scale_bwd dz");
    BufferSlot* DX = buffer_or_null(cx, dx, "bn_scale_bwd dx");
    BufferSlot* DG = buffer_or_null(cx, dgamma, "bn_scale_bwd dgamma");
    BufferSlot* DB = buffer_or_null(cx, dbeta, "bn_scale_bwd dbeta");
    BufferSlot& S = buffer(cx, scratch, "bn_scale_bwd scratch");
    const uint64_t cnt = uint64_t(n) * c * hw;
    require_len(XN, cnt, "bn_scale_bwd"); require_len(DZ, cnt, "bn_scale_bwd");
    if (DX) require_len(*DX, cnt, "bn_scale_bwd");
    require_len(V, uint64_t(c), "bn_scale_bwd"); require_len(G, uint64_t(c), "bn_scale_bwd");
    require_len(S, 2 * uint64_t(c), "bn_scale_bwd scratch");
    for (BufferSlot* b : {&V, &G, &DZ, &S, DX, DG, DB}) if (b) require_dtype(*b, XN.dtype, "bn_scale_bwd");
    if (n * c > 65535) fail(CDNN_INVALID_ARGUMENT, "bn_scale_bwd: n*c must be <= 65535");
    DeviceGuard g(cx);
    cudaStream_t st = stream_of(cx, stream);
    const int splits = chan_splits(n, c, hw);
    double2* part = static_cast<double2*>(workspace_of(cx, stream).get(size_t(c) * splits * sizeof(double2), cx->device));
    by_dtype(XN.dtype, "bn_scale_bwd", [&](auto tag) {
      using T = decltype(tag);
      T* a = P<T>(S);
      T* b = a + c;
      chan_partials<T, kSumDot><<<dim3(c, splits), kT, 0, st>>>(P<T>(DZ), P<T>(XN), part, n, c, hw, splits);
      if (DX)
        bn_scale_bwd_apply_c<T><<<dim3(c, splits), kT, 0, st>>>(P<T>(XN), P<T>(DZ), part, splits, double(n) * hw,
                                                               P<T>(V), P<T>(G), DG ? P<T>(*DG) : nullptr,
                                                               DB ? P<T>(*DB) : nullptr, P<T>(*DX), n, c, hw);
      else
        bn_scale_finalize<T><<<(c + 127) / 128, 128, 0, st>>>(part, splits, c, double(n) * hw, DG ? P<T>(*DG) : nullptr,
                                                             DB ? P<T>(*DB) : nullptr, a, b);
    });
    check_launch("bn_scale_bwd");
    count_launch(cx, 2);
  });
}

int cdnn_pg_diff(cdnn_ctx ctx, cdnn_handle prob, cdnn_handle actions, cdnn_handle returns, cdnn_handle dlogit,
                 int rows, int n, int classes, int sigmoid, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& Pb = buffer(cx, prob, "pg_diff prob");
    BufferSlot& A = buffer(cx, actions, "pg_diff actions");
    BufferSlot& R = buffer(cx, returns, "pg_diff returns");
    BufferSlot& D = buffer(cx, dlogit, "pg_diff dlogit");
    if (rows < 1 || classes < 1 || n < 0 || n > rows) fail(CDNN_INVALID_ARGUMENT, "pg_diff: bad extents");
    if (sigmoid && classes != 1) fail(CDNN_INVALID_ARGUMENT, "pg_diff: the sigmoid variant has one logit per row");
    if (!sigmoid && classes < 2) fail(CDNN_INVALID_ARGUMENT, "pg_diff: the softmax variant needs >= 2 logits");
    const uint64_t cnt = uint64_t(rows) * classes;
    require_len(Pb, cnt, "pg_diff"); require_len(D, cnt, "pg_diff");
    require_len(A, uint64_t(std::max(n, 1)), "pg_diff actions"); require_len(R, uint64_t(std::max(n, 1)), "pg_diff returns");
    for (BufferSlot* b : {&A, &R, &D}) require_dtype(*b, Pb.dtype, "pg_diff");
    DeviceGuard g(cx);
    by_dtype(Pb.dtype, "pg_diff", [&](auto tag) {
      using T = decltype(tag);
      pg_diff_kernel<T><<<blocks(int64_t(cnt)), kT, 0, stream_of(cx, stream)>>>(P<T>(Pb), P<T>(A), P<T>(R), P<T>(D),
                                                                               rows, n, classes, sigmoid);
    });
    check_launch("pg_diff");
    count_launch(cx);
  });
}

// y = a*x (+ b*y when accumulate): Eltwise SUM forward terms and backward copies
int cdnn_axpby(cdnn_ctx ctx, uint64_t n, double a, cdnn_handle x, double b, cdnn_handle y, int accumulate,
               cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "axpby x");
    BufferSlot& Y = buffer(cx, y, "axpby y");
    require_len(X, n, "axpby"); require_len(Y, n, "axpby"); require_dtype(Y, X.dtype, "axpby");
    if (n == 0) return;
    DeviceGuard g(cx);
    by_dtype(X.dtype, "axpby", [&](auto tag) {
      using T = decltype(tag);
      axpby_kernel<T><<<blocks(int64_t(n)), kT, 0, stream_of(cx, stream)>>>(P<T>(X), P<T>(Y), n, T(a), T(b),
                                                                           accumulate != 0);
    });
    check_launch("axpby");
    count_launch(cx);
  });
}

}  // extern "C"
