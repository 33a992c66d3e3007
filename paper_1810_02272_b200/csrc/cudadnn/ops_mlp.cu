// ops_mlp.cu — the whole policy-gradient update of a small two-layer perceptron
// (the reference's pg_softmax graph: InnerProduct -> ReLU -> InnerProduct ->
// Softmax, proj/models/pg_softmax.prototxt) in ONE kernel.
//
// The layered path runs this update as thirteen launches (three GEMM-shaped
// InnerProduct products per layer, bias sums, ReLU, Softmax, the modulated
// log-prob gradient of trainer.cpp:42-113 and the solver of solver.cpp:24-57);
// at batch 1024 each of them is a few microseconds of launch latency around
// nanoseconds of math, so the step is latency bound.  Here one CTA does it all:
//
//   pass over rows (one thread per row, staged in shared memory):
//     a   = ReLU(x W1^T + b1)                    (layers.cpp InnerProduct / ReLU)
//     l   = a W2^T + b2 ; p = softmax(l)          (logits / prob tops written)
//     dl  = (p - onehot(action)) * return         (rows >= count: 0; cdnn_pg_diff)
//     dh  = (dl W2) * [pre-activation > 0]
//   every parameter gradient is a sum over rows: one warp per gradient element,
//   lanes stride the rows, a fixed xor tree, a per-element accumulator across
//   passes (deterministic order; no atomics);
//   then the solver rule of cdnn_solver_apply on the arena (the existing
//   gradient is added first, and zeroed, like the layered update).
//
// Numerics: the same operations as the layered path in a different summation
// order (FP32 / FP64 CUDA-core arithmetic, no tensor cores): parity against the
// oracle is the tolerance bar of north_star, not bit identity with the layered
// path (tests/test_gpu_pg.py checks both).
#include "launch.cuh"

namespace cdnn {
namespace {

constexpr int kMlpThreads = 1024;
constexpr int kMlpMaxParams = 4096;   // gradient elements (accumulators in shared memory)
constexpr int kMlpMaxClasses = 16;
constexpr int kMlpSmemBudget = 200 * 1024;

template <typename T>
T* dp(const BufferSlot& b) { return reinterpret_cast<T*>(b.dev); }

template <typename T> __device__ __forceinline__ T mlp_mul(T a, T b);
template <> __device__ __forceinline__ float mlp_mul(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mlp_mul(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T mlp_add(T a, T b);
template <> __device__ __forceinline__ float mlp_add(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double mlp_add(double a, double b) { return __dadd_rn(a, b); }
template <typename T> __device__ __forceinline__ T mlp_sub(T a, T b);
template <> __device__ __forceinline__ float mlp_sub(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ double mlp_sub(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
struct MlpArgs {
  const T* x;      // rows x in (device, or page-locked host memory read over the bus)
  const T* act;    // count actions (class indices as reals; device or page-locked host)
  const T* ret;    // count returns (device or page-locked host)
  T* x_copy;       // when x is host memory: the feed blob, filled with the states read
  T* prob_host;    // optional page-locked host copy of prob (the policy's action sampling)
  T* w;            // weight arena
  T* g;            // gradient arena
  T* hist;         // solver history (momentum / RMSProp cache) or null
  uint64_t oW1, ob1, oW2, ob2;  // parameter offsets in the arenas
  T* hidden;       // optional rows x hid ReLU top
  T* logits;       // rows x cls
  T* prob;         // rows x cls
  int rows, count, in, hid, cls;
  int rows_per_pass;
  int solver;      // CDNN_SOLVER_SGD / CDNN_SOLVER_RMSPROP
  T lr, mom, wd, rms_decay, eps;
};

// arena offset of gradient element p (W1 | b1 | W2 | b2 order)
template <typename T>
__device__ __forceinline__ uint64_t mlp_param_offset(const MlpArgs<T>& a, int p) {
  const int nW1 = a.hid * a.in, nW2 = a.cls * a.hid;
  if (p < nW1) return a.oW1 + p;
  if (p < nW1 + a.hid) return a.ob1 + (p - nW1);
  if (p < nW1 + a.hid + nW2) return a.oW2 + (p - nW1 - a.hid);
  return a.ob2 + (p - nW1 - a.hid - nW2);
}

// cdnn_solver_apply's rule for one element (w, arena gradient g, history h) with the
// batch gradient gsum added to g first; the arena gradient is left zero.
template <typename T>
__device__ __forceinline__ void mlp_solver_rule(const MlpArgs<T>& a, uint64_t off, T wi, T g0, T h0, T gsum) {
  T gi = mlp_add(g0, gsum);
  if (a.solver == CDNN_SOLVER_SGD) {
    if (a.wd != T(0)) gi = mlp_add(gi, mlp_mul(a.wd, wi));
    T step = mlp_mul(a.lr, gi);
    if (a.hist) {
      if (a.mom != T(0)) step = mlp_add(mlp_mul(a.mom, h0), step);
      a.hist[off] = step;
    }
    wi = mlp_sub(wi, step);
  } else {
    const T ci = mlp_add(mlp_mul(a.rms_decay, h0), mlp_mul(mlp_mul(mlp_sub(T(1), a.rms_decay), gi), gi));
    a.hist[off] = ci;
    wi = mlp_sub(wi, mlp_mul(a.lr, gi) / mlp_add(sqrt(ci), a.eps));
  }
  a.w[off] = wi;
  a.g[off] = T(0);
}

template <typename T>
__global__ void __launch_bounds__(kMlpThreads, 1) mlp_pg_step_kernel(const MlpArgs<T> a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  const int in = a.in, hid = a.hid, cls = a.cls, R = a.rows_per_pass;
  const int nW1 = hid * in, nW2 = cls * hid;
  const int P = nW1 + hid + nW2 + cls;
  // shared layout: parameters (W1 | b1 | W2 | b2), accumulators [P], then per-row
  // staging x [R][in], a [R][hid], pre / dh [R][hid], dl [R][cls]
  T* sW1 = sm;
  T* sb1 = sW1 + nW1;
  T* sW2 = sb1 + hid;
  T* sb2 = sW2 + nW2;
  T* acc = sb2 + cls;
  T* sx = acc + P;
  T* sa = sx + R * in;
  T* sd = sa + R * hid;
  T* sl = sd + R * hid;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  for (int i = tid; i < nW1; i += blockDim.x) sW1[i] = a.w[a.oW1 + i];
  for (int i = tid; i < hid; i += blockDim.x) sb1[i] = a.w[a.ob1 + i];
  for (int i = tid; i < nW2; i += blockDim.x) sW2[i] = a.w[a.oW2 + i];
  for (int i = tid; i < cls; i += blockDim.x) sb2[i] = a.w[a.ob2 + i];
  for (int i = tid; i < P; i += blockDim.x) acc[i] = T(0);
  __syncthreads();

  for (int r0 = 0; r0 < a.rows; r0 += R) {
    const int nr = min(R, a.rows - r0);
    // ---- forward + output gradient + hidden gradient, one row per thread
    for (int t = tid; t < nr; t += blockDim.x) {
      const int r = r0 + t;
      T* xs = sx + t * in;
      T* as = sa + t * hid;
      T* ds = sd + t * hid;
      T* ls = sl + t * cls;
      for (int k = 0; k < in; ++k) xs[k] = a.x[int64_t(r) * in + k];  // loads before the copy's stores
      if (a.x_copy)
        for (int k = 0; k < in; ++k) a.x_copy[int64_t(r) * in + k] = xs[k];
      for (int h = 0; h < hid; ++h) {
        const T* wr = sW1 + h * in;
        T s = T(0);
        for (int k = 0; k < in; ++k) s = fma(xs[k], wr[k], s);
        s = mlp_add(s, sb1[h]);
        ds[h] = s;                       // pre-activation (its sign gates dh)
        const T v = s > T(0) ? s : T(0);
        as[h] = v;
        if (a.hidden) a.hidden[int64_t(r) * hid + h] = v;
      }
      T l[kMlpMaxClasses];
      T m = T(0);
#pragma unroll
      for (int c = 0; c < kMlpMaxClasses; ++c) {
        if (c < cls) {
          const T* wr = sW2 + c * hid;
          T s = T(0);
          for (int h = 0; h < hid; ++h) s = fma(as[h], wr[h], s);
          s = mlp_add(s, sb2[c]);
          l[c] = s;
          m = c == 0 ? s : max(m, s);
          a.logits[int64_t(r) * cls + c] = s;
        }
      }
      T se = T(0);
#pragma unroll
      for (int c = 0; c < kMlpMaxClasses; ++c)
        if (c < cls) { l[c] = exp(l[c] - m); se += l[c]; }
      const bool live = r < a.count;
      const int act = live ? int(a.act[r]) : -1;
      const T gret = live ? a.ret[r] : T(0);
#pragma unroll
      for (int c = 0; c < kMlpMaxClasses; ++c)
        if (c < cls) {
          const T p = l[c] / se;
          a.prob[int64_t(r) * cls + c] = p;
          if (a.prob_host) a.prob_host[int64_t(r) * cls + c] = p;
          ls[c] = live ? mlp_mul(mlp_sub(p, c == act ? T(1) : T(0)), gret) : T(0);
        }
      for (int h = 0; h < hid; ++h) {
        T s = T(0);
        for (int c = 0; c < cls; ++c) s = fma(ls[c], sW2[c * hid + h], s);
        ds[h] = ds[h] > T(0) ? s : T(0);
      }
    }
    __syncthreads();
    // ---- parameter gradients: warp per element, lanes over the rows of the pass
    for (int p = warp; p < P; p += nwarps) {
      T s = T(0);
      if (p < nW1) {
        const int h = p / in, k = p - h * in;
        for (int j = lane; j < nr; j += 32) s = fma(sd[j * hid + h], sx[j * in + k], s);
      } else if (p < nW1 + hid) {
        const int h = p - nW1;
        for (int j = lane; j < nr; j += 32) s = mlp_add(s, sd[j * hid + h]);
      } else if (p < nW1 + hid + nW2) {
        const int q = p - nW1 - hid, c = q / hid, h = q - c * hid;
        for (int j = lane; j < nr; j += 32) s = fma(sl[j * cls + c], sa[j * hid + h], s);
      } else {
        const int c = p - nW1 - hid - nW2;
        for (int j = lane; j < nr; j += 32) s = mlp_add(s, sl[j * cls + c]);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) acc[p] = mlp_add(acc[p], s);
    }
    __syncthreads();
  }
  // ---- solver rule (cdnn_solver_apply semantics), gradients zeroed
  for (int p = tid; p < P; p += blockDim.x) {
    const uint64_t off = mlp_param_offset(a, p);
    mlp_solver_rule(a, off, a.w[off], a.g[off], a.hist ? a.hist[off] : T(0), acc[p]);
  }
}

// ---- compile-time extents (the reference's 4-10-2 policy): everything in registers.
// 256 threads (255 registers each: the 96 gradient partials stay in registers); a chunk of rows (states, actions, returns) is staged in shared memory
// with coalesced loads (one bus round trip when the inputs are host memory), each
// thread runs its rows fully unrolled and keeps its share of every parameter
// gradient in registers; a warp reduce-scatter (five xor-shuffle stages, each
// halving the vector: N/32 values per lane) and a fixed-order sum over the warps
// give each gradient element in a deterministic order.
constexpr int kFixThreads = 256;

template <int N, typename T>
__device__ __forceinline__ void warp_reduce_scatter(T (&v)[N], int lane) {
  static_assert(N % 32 == 0, "reduce-scatter over 32 lanes");
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int off = 16 >> s, half = N >> (s + 1);
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      if (i < half) {
        const T lo = v[i], hi = v[i + half];
        const T keep = up ? hi : lo, send = up ? lo : hi;
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
  }
}
template <int N>
__device__ __forceinline__ int reduce_scatter_base(int lane) {
  int b = 0;
#pragma unroll
  for (int s = 0; s < 5; ++s)
    if (lane & (16 >> s)) b += N >> (s + 1);
  return b;
}

template <typename T, int IN, int HID, int CLS>
__global__ void __launch_bounds__(kFixThreads, 1) mlp_pg_fixed_kernel(const MlpArgs<T> a) {
  constexpr int nW1 = HID * IN, nW2 = CLS * HID, NP = nW1 + HID + nW2 + CLS;
  constexpr int NPP = (NP + 31) / 32 * 32;
  constexpr int NWARP = kFixThreads / 32;
  constexpr int kFixChunk = sizeof(T) == 4 ? 1024 : 512;  // staged rows (static shared memory < 48 KB)
  __shared__ T sw[NP];
  __shared__ T red[NWARP][NPP];
  __shared__ T sx[kFixChunk * IN];
  __shared__ T sact[kFixChunk], sret[kFixChunk];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the solver's operands, loaded up front (one latency with the weights)
  T w0 = T(0), g0 = T(0), h0 = T(0);
  uint64_t off = 0;
  if (tid < NP) {
    off = mlp_param_offset(a, tid);
    w0 = a.w[off];
    g0 = a.g[off];
    if (a.hist) h0 = a.hist[off];
    sw[tid] = w0;
  }
  const T* W1 = sw;
  const T* b1 = sw + nW1;
  const T* W2 = b1 + HID;
  const T* b2 = W2 + nW2;
  T gp[NPP];
#pragma unroll
  for (int i = 0; i < NPP; ++i) gp[i] = T(0);
  for (int r0 = 0; r0 < a.rows; r0 += kFixChunk) {
    const int nr = min(kFixChunk, a.rows - r0);
    // every load of the chunk issued before any store (the stores may alias the
    // sources as far as the compiler knows): one memory / bus round trip, in flight
    // together with the weight loads of the first chunk
    constexpr int XPT = kFixChunk * IN / kFixThreads, RPT = kFixChunk / kFixThreads;
    T xv[XPT], av_[RPT], rv[RPT];
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int i = tid + u * kFixThreads;
      xv[u] = i < nr * IN ? a.x[int64_t(r0) * IN + i] : T(0);
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + u * kFixThreads;
      const bool live = i < nr && r0 + i < a.count;
      av_[u] = live ? a.act[r0 + i] : T(-1);
      rv[u] = live ? a.ret[r0 + i] : T(0);
    }
    __syncthreads();  // weights visible / previous chunk consumed
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int i = tid + u * kFixThreads;
      if (i < nr * IN) {
        sx[i] = xv[u];
        if (a.x_copy) a.x_copy[int64_t(r0) * IN + i] = xv[u];
      }
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = tid + u * kFixThreads;
      if (i < nr) { sact[i] = av_[u]; sret[i] = rv[u]; }
    }
    __syncthreads();
    for (int t = tid; t < nr; t += kFixThreads) {
      const int r = r0 + t;
      T x[IN];
#pragma unroll
      for (int k = 0; k < IN; ++k) x[k] = sx[t * IN + k];
      T pre[HID], av[HID];
#pragma unroll
      for (int h = 0; h < HID; ++h) {
        T s = T(0);
#pragma unroll
        for (int k = 0; k < IN; ++k) s = fma(x[k], W1[h * IN + k], s);
        s = mlp_add(s, b1[h]);
        pre[h] = s;
        av[h] = s > T(0) ? s : T(0);
      }
      if (a.hidden) {
#pragma unroll
        for (int h = 0; h < HID; ++h) a.hidden[int64_t(r) * HID + h] = av[h];
      }
      T l[CLS];
      T m = T(0);
#pragma unroll
      for (int c = 0; c < CLS; ++c) {
        T s = T(0);
#pragma unroll
        for (int h = 0; h < HID; ++h) s = fma(av[h], W2[c * HID + h], s);
        s = mlp_add(s, b2[c]);
        l[c] = s;
        m = c == 0 ? s : max(m, s);
        a.logits[int64_t(r) * CLS + c] = s;
      }
      T se = T(0);
#pragma unroll
      for (int c = 0; c < CLS; ++c) { l[c] = exp(l[c] - m); se += l[c]; }
      const int act = int(sact[t]);
      const T gret = sret[t];
      const bool live = r < a.count;
      T dl[CLS];
#pragma unroll
      for (int c = 0; c < CLS; ++c) {
        const T p = l[c] / se;
        a.prob[int64_t(r) * CLS + c] = p;
        if (a.prob_host) a.prob_host[int64_t(r) * CLS + c] = p;
        dl[c] = live ? mlp_mul(mlp_sub(p, c == act ? T(1) : T(0)), gret) : T(0);
      }
#pragma unroll
      for (int h = 0; h < HID; ++h) {
        T s = T(0);
#pragma unroll
        for (int c = 0; c < CLS; ++c) s = fma(dl[c], W2[c * HID + h], s);
        const T dh = pre[h] > T(0) ? s : T(0);
#pragma unroll
        for (int k = 0; k < IN; ++k) gp[h * IN + k] = fma(dh, x[k], gp[h * IN + k]);
        gp[nW1 + h] = mlp_add(gp[nW1 + h], dh);
      }
#pragma unroll
      for (int c = 0; c < CLS; ++c) {
#pragma unroll
        for (int h = 0; h < HID; ++h) gp[nW1 + HID + c * HID + h] = fma(dl[c], av[h], gp[nW1 + HID + c * HID + h]);
        gp[nW1 + HID + nW2 + c] = mlp_add(gp[nW1 + HID + nW2 + c], dl[c]);
      }
    }
  }
  warp_reduce_scatter<NPP>(gp, lane);
  const int base = reduce_scatter_base<NPP>(lane);
#pragma unroll
  for (int j = 0; j < NPP / 32; ++j) red[warp][base + j] = gp[j];
  __syncthreads();
  if (tid < NP) {
    T s = T(0);
#pragma unroll
    for (int w = 0; w < NWARP; ++w) s = mlp_add(s, red[w][tid]);
    mlp_solver_rule(a, off, w0, g0, h0, s);
  }
}

// rows staged per pass within the shared-memory budget (0: the net does not fit)
int mlp_rows_per_pass(int esz, int in, int hid, int cls) {
  const int64_t P = int64_t(hid) * in + hid + int64_t(cls) * hid + cls;
  const int64_t fixed = 2 * P * esz;
  const int64_t per_row = int64_t(in + 2 * hid + cls) * esz;
  if (fixed + 32 * per_row > kMlpSmemBudget) return 0;
  return int(std::min<int64_t>(kMlpThreads, (kMlpSmemBudget - fixed) / per_row));
}

bool mlp_supported(int esz, int rows, int in, int hid, int cls) {
  if (rows < 1 || in < 1 || hid < 1 || cls < 2 || cls > kMlpMaxClasses) return false;
  const int64_t P = int64_t(hid) * in + hid + int64_t(cls) * hid + cls;
  if (P > kMlpMaxParams) return false;
  return mlp_rows_per_pass(esz, in, hid, cls) > 0;
}

// A page-locked host pointer as the device sees it (UVA: cudaMallocHost memory is
// mapped); null stays null.
template <typename T>
T* mapped(const void* host, const char* what) {
  if (!host) return nullptr;
  cudaPointerAttributes at{};
  CDNN_CUDA(cudaPointerGetAttributes(&at, host));
  if (at.type != cudaMemoryTypeHost || !at.devicePointer)
    fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": host buffer is not page-locked (cudaMallocHost)");
  return static_cast<T*>(at.devicePointer);
}

}  // namespace
}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_mlp_pg_supported(cdnn_ctx ctx, int dtype, int rows, int in, int hidden, int classes, int* out) {
  return guarded([&] {
    need_ctx(ctx);
    if (!out) fail(CDNN_INVALID_ARGUMENT, "mlp_pg_supported: null out");
    if (dtype != CDNN_F32 && dtype != CDNN_F64) fail(CDNN_INVALID_ARGUMENT, "mlp_pg_supported: real dtype required");
    *out = mlp_supported(dtype == CDNN_F32 ? 4 : 8, rows, in, hidden, classes) ? 1 : 0;
  });
}

int cdnn_mlp_pg_step(cdnn_ctx ctx, cdnn_handle x, cdnn_handle actions, cdnn_handle returns, int rows, int count,
                     int in, int hidden, int classes, cdnn_handle weights, cdnn_handle grads, cdnn_handle history,
                     const uint64_t param_offsets[4], int solver, double lr, double momentum, double weight_decay,
                     double rms_decay, double epsilon, cdnn_handle hidden_top, cdnn_handle logits, cdnn_handle prob,
                     cdnn_handle stream) {
  return cdnn_mlp_pg_step_host(ctx, x, actions, returns, nullptr, nullptr, nullptr, nullptr, rows, count, in, hidden,
                               classes, weights, grads, history, param_offsets, solver, lr, momentum, weight_decay,
                               rms_decay, epsilon, hidden_top, logits, prob, stream);
}

int cdnn_mlp_pg_step_host(cdnn_ctx ctx, cdnn_handle x, cdnn_handle actions, cdnn_handle returns,
                          const void* host_x, const void* host_actions, const void* host_returns, void* host_prob,
                          int rows, int count, int in, int hidden, int classes, cdnn_handle weights, cdnn_handle grads,
                          cdnn_handle history, const uint64_t param_offsets[4], int solver, double lr,
                          double momentum, double weight_decay, double rms_decay, double epsilon,
                          cdnn_handle hidden_top, cdnn_handle logits, cdnn_handle prob, cdnn_handle stream) {
  return guarded([&] {
    Ctx* cx = need_ctx(ctx);
    BufferSlot& X = buffer(cx, x, "mlp_pg x");
    if ((host_actions == nullptr) != (host_returns == nullptr))
      fail(CDNN_INVALID_ARGUMENT, "mlp_pg: actions and returns come from the same side");
    BufferSlot* A = host_actions ? nullptr : &buffer(cx, actions, "mlp_pg actions");
    BufferSlot* Rt = host_returns ? nullptr : &buffer(cx, returns, "mlp_pg returns");
    BufferSlot& W = buffer(cx, weights, "mlp_pg weights");
    BufferSlot& G = buffer(cx, grads, "mlp_pg grads");
    BufferSlot& L = buffer(cx, logits, "mlp_pg logits");
    BufferSlot& Pb = buffer(cx, prob, "mlp_pg prob");
    BufferSlot* Hs = history ? &buffer(cx, history, "mlp_pg history") : nullptr;
    BufferSlot* Ht = hidden_top ? &buffer(cx, hidden_top, "mlp_pg hidden") : nullptr;
    if (!param_offsets) fail(CDNN_INVALID_ARGUMENT, "mlp_pg: null parameter offsets");
    if (solver != CDNN_SOLVER_SGD && solver != CDNN_SOLVER_RMSPROP) fail(CDNN_INVALID_ARGUMENT, "mlp_pg: unknown solver");
    if (solver == CDNN_SOLVER_RMSPROP && !Hs) fail(CDNN_INVALID_ARGUMENT, "mlp_pg: RMSProp needs its cache");
    if (count < 0 || count > rows) fail(CDNN_INVALID_ARGUMENT, "mlp_pg: count exceeds the batch");
    const int esz = X.dtype == CDNN_F64 ? 8 : 4;
    if (!mlp_supported(esz, rows, in, hidden, classes)) fail(CDNN_INVALID_ARGUMENT, "mlp_pg: unsupported extents");
    require_len(X, uint64_t(rows) * in, "mlp_pg x");
    require_len(L, uint64_t(rows) * classes, "mlp_pg logits");
    require_len(Pb, uint64_t(rows) * classes, "mlp_pg prob");
    if (A) require_len(*A, uint64_t(std::max(count, 1)), "mlp_pg actions");
    if (Rt) require_len(*Rt, uint64_t(std::max(count, 1)), "mlp_pg returns");
    if (Ht) require_len(*Ht, uint64_t(rows) * hidden, "mlp_pg hidden");
    const uint64_t sizes[4] = {uint64_t(hidden) * in, uint64_t(hidden), uint64_t(classes) * hidden, uint64_t(classes)};
    for (int i = 0; i < 4; ++i) {
      require_len(W, param_offsets[i] + sizes[i], "mlp_pg weights");
      require_len(G, param_offsets[i] + sizes[i], "mlp_pg grads");
      if (Hs) require_len(*Hs, param_offsets[i] + sizes[i], "mlp_pg history");
    }
    for (BufferSlot* b : {A, Rt, &W, &G, &L, &Pb, Hs, Ht})
      if (b) require_dtype(*b, X.dtype, "mlp_pg");
    DeviceGuard dg(cx);
    const int R = mlp_rows_per_pass(esz, in, hidden, classes);
    const int64_t nparams = int64_t(hidden) * in + hidden + int64_t(classes) * hidden + classes;
    const size_t smem = size_t(2 * nparams + int64_t(R) * (in + 2 * hidden + classes)) * esz;
    auto go = [&](auto tag) {
      using T = decltype(tag);
      const T* xs = host_x ? mapped<const T>(host_x, "mlp_pg states") : dp<T>(X);
      MlpArgs<T> args{xs,
                      A ? dp<T>(*A) : mapped<const T>(host_actions, "mlp_pg actions"),
                      Rt ? dp<T>(*Rt) : mapped<const T>(host_returns, "mlp_pg returns"),
                      host_x ? dp<T>(X) : nullptr,
                      mapped<T>(host_prob, "mlp_pg prob"),
                      dp<T>(W), dp<T>(G), Hs ? dp<T>(*Hs) : nullptr,
                      param_offsets[0], param_offsets[1], param_offsets[2], param_offsets[3],
                      Ht ? dp<T>(*Ht) : nullptr, dp<T>(L), dp<T>(Pb),
                      rows, count, in, hidden, classes, R, solver,
                      T(lr), T(momentum), T(weight_decay), T(rms_decay), T(epsilon)};
      // the reference's pg_softmax policy in fp32: the register kernel (fp64 partials
      // would not fit the register file: the shared-memory kernel)
      if constexpr (std::is_same_v<T, float>) {
        if (in == 4 && hidden == 10 && classes == 2) {
          mlp_pg_fixed_kernel<T, 4, 10, 2><<<1, kFixThreads, 0, stream_of(cx, stream)>>>(args);
          return;
        }
      }
      auto kern = mlp_pg_step_kernel<T>;
      CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      kern<<<1, kMlpThreads, smem, stream_of(cx, stream)>>>(args);
    };
    if (X.dtype == CDNN_F32) go(float{});
    else if (X.dtype == CDNN_F64) go(double{});
    else fail(CDNN_INVALID_ARGUMENT, "mlp_pg: floating buffers required");
    check_launch("mlp_pg_step");
    count_launch(cx);
  });
}

}  // extern "C"
