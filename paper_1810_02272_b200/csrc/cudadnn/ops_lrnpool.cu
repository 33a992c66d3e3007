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

constexpr int kG = 4;     // channels per step (loads in flight; one block barrier per step)
// forward fast path: x prefetched kPF - 1 steps ahead into a per-thread shared-memory ring
// by cp.async (the loads hold no registers while in flight; one step of register
// lookahead left too few bytes in flight at two 512-thread blocks per SM).  AlexNet
// norm1+pool1 / norm2+pool2 forward, ms: register lookahead 0.205 / 0.150; ring depth
// 2: 0.194 / 0.142, 3: 0.183 / 0.129, 4: 0.187 / 0.131, 6: 0.199 / 0.133, 8: 0.205 / 0.140
constexpr int kPF = 3;
#ifndef CDNN_LRN_FWD_SEG
#define CDNN_LRN_FWD_SEG 128
#endif
constexpr int kSeg = CDNN_LRN_FWD_SEG;  // forward: channels per block segment (segments run in parallel)
#ifndef CDNN_LRN_BWD_SEG
#define CDNN_LRN_BWD_SEG 128
#endif
constexpr int kSegB = CDNN_LRN_BWD_SEG;  // backward: channels per thread (each segment re-primes SIZE-1 channels)

// a pointer the optimiser cannot see through (keeps base + 32-bit offset addressing)
template <class P>
__device__ __forceinline__ P* opaque(P* p) {
  asm("" : "+l"(p));
  return p;
}

struct LrnPoolGeom {
  int N, C, H, W, PH, PW;
  int TR, rows_in;  // pooled rows per band, input rows per band
  int bands;
  int segs;         // channel segments of kSeg
};

// Forward: block (band, channel segment, image).  The x loads of step i+1 are issued
// before step i's arithmetic and barrier (lookahead of one step).
template <typename T, int SIZE, int K, int S>
__global__ void __launch_bounds__(1024) lrn_maxpool_fwd(const T* __restrict__ x, T* __restrict__ ynorm,
                                                        T* __restrict__ ypool, int* __restrict__ mask,
                                                        LrnPoolGeom g, T alpha, T beta, T k, bool relu) {
  constexpr int pre = (SIZE - 1) / 2, post = SIZE - 1 - pre;
  extern __shared__ uint8_t smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // [2][kG][rows_in * W]
  const int band = blockIdx.x, img = blockIdx.z;
  const int cs0 = blockIdx.y * kSeg, cs1 = min(g.C, cs0 + kSeg);
  const int pr0 = band * g.TR, pr1 = min(g.PH, pr0 + g.TR);
  const int r0 = pr0 * S, r1 = min(g.H, (pr1 - 1) * S + K);
  // rows whose LRN top this band stores (halo rows belong to the next band)
  const int own1 = band + 1 == g.bands ? g.H : min(g.H, pr1 * S);
  const int npix = (r1 - r0) * g.W, tsz = g.rows_in * g.W;
  const int HW = g.H * g.W, PHW = g.PH * g.PW;
  const T aN = alpha / T(SIZE);
  const int p = threadIdx.x;
  const bool active = p < npix;
  const int h = r0 + (active ? p / g.W : 0);
  const size_t base = size_t(img) * g.C * HW + size_t(h) * g.W + (active ? p % g.W : 0);
  const T* xp = opaque(x + base);
  T* yp = opaque(ynorm + base);
  const bool own = active && h < own1;
  T xr[SIZE];  // x(c - pre .. c + post)
#pragma unroll
  for (int j = 0; j < SIZE; ++j) {
    const int cc = cs0 + j - pre;
    xr[j] = (active && cc >= 0 && cc < g.C) ? __ldg(xp + uint32_t(cc) * uint32_t(HW)) : T(0);
  }
  auto load_step = [&](int c0, T (&nx)[kG]) {
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const int cin = c0 + u + post + 1;
      nx[u] = (active && c0 + u < cs1 && cin < g.C) ? __ldg(xp + uint32_t(cin) * uint32_t(HW)) : T(0);
    }
  };
  T nxt[kG];
  load_step(cs0, nxt);
  const int prows = pr1 - pr0;
  // the thread's first pool item (channel u0 of the step, pooled row / column) is the
  // same every step: its window origin, output offset and bounds are computed once
  // (two integer divisions per step and item otherwise; items beyond blockDim, if
  // any, take the general loop below)
  const int per_u = prows * g.PW;
  const int it0 = threadIdx.x;
  const bool has0 = it0 < kG * per_u;
  int u0 = 0, toff0 = 0, po0 = 0, abase0 = 0;
  uint32_t wbits0 = 0;
  if (has0) {
    u0 = it0 / per_u;
    const int rem = it0 - u0 * per_u;
    const int prl = rem / g.PW, pw = rem - prl * g.PW;
    const int hs = (pr0 + prl) * S, ws = pw * S;
    toff0 = u0 * tsz + (hs - r0) * g.W + ws;
    po0 = (pr0 + prl) * g.PW + pw;
    abase0 = hs * g.W + ws;
#pragma unroll
    for (int a = 0; a < K; ++a)
#pragma unroll
      for (int b = 0; b < K; ++b)
        if (hs + a < g.H && ws + b < g.W) wbits0 |= 1u << (a * K + b);
  }
  int c0 = cs0, step = 0;
  // Fast path (block-uniform: depends on the segment only): steps whose channels and
  // next loads are all in range run without bounds tests, with running 32-bit offsets,
  // unrolled over SIZE steps so the x ring rotates back to its registers.  Same values,
  // same operations and barriers as the general loop below: bit-identical.
  auto fast_ok = [&](int cc) {
    return cc + (SIZE + 1) * kG <= cs1 && cc + (SIZE + kPF - 1) * kG + post < g.C;
  };
  const bool extra_items = kG * per_u > int(blockDim.x);
  if (!extra_items && fast_ok(c0)) {
    // prefetch ring: slot j holds a step's kG entering channels, [slot][u][thread]
    T* pf = tile + 2 * kG * tsz;
    const uint32_t pf0 = ptx::smem_u32(pf) + uint32_t(threadIdx.x) * uint32_t(sizeof(T));
    const uint32_t pf_u = uint32_t(blockDim.x) * uint32_t(sizeof(T)), pf_slot = uint32_t(kG) * pf_u;
    const uint32_t pbytes = active ? uint32_t(sizeof(T)) : 0u;  // zero-fill for idle threads
    uint32_t oxn = uint32_t(c0 + kG + post + 1) * uint32_t(HW);  // step c0 + kG's first entering channel
    auto prefetch = [&](uint32_t slot) {  // the step at oxn into `slot`, one cp.async group
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const uint32_t dst = pf0 + slot * pf_slot + uint32_t(u) * pf_u;
        const T* src = xp + (oxn + uint32_t(u) * uint32_t(HW));
        if constexpr (sizeof(T) == 4) ptx::cp_async_4(dst, src, pbytes);
        else ptx::cp_async_8(dst, src, pbytes);
      }
      ptx::cp_async_commit();
      oxn += uint32_t(kG) * uint32_t(HW);
    };
    // slot 0: step c0 (already in registers); slots 1 .. kPF-1: the next steps
#pragma unroll
    for (int u = 0; u < kG; ++u) pf[u * blockDim.x + threadIdx.x] = nxt[u];
#pragma unroll
    for (int j = 1; j < kPF; ++j) prefetch(uint32_t(j));
    uint32_t slot = 0;
    uint32_t oy = uint32_t(c0) * uint32_t(HW);
    uint32_t opool = (uint32_t(img) * g.C + c0 + u0) * uint32_t(PHW) + uint32_t(po0);
    while (fast_ok(c0)) {
#pragma unroll
      for (int st = 0; st < SIZE; ++st) {
        T cur[kG];
        ptx::cp_async_wait<kPF - 2>();  // this step's group has landed
#pragma unroll
        for (int u = 0; u < kG; ++u) cur[u] = pf[(slot * kG + u) * blockDim.x + threadIdx.x];
        prefetch(slot);  // the step kPF - 1 ahead into the slot just read
        slot = slot + 1 == uint32_t(kPF) ? 0u : slot + 1;
        T* buf = tile + (step & 1) * kG * tsz;
        if (active) {
#pragma unroll
          for (int u = 0; u < kG; ++u) {
            T sum = T(0);
#pragma unroll
            for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xr[j]);
            const T sc = lrn::scale(sum, aN, k);
            const T yv = lrn::top(xr[pre], lrn::neg_pow(sc, beta));
            buf[u * tsz + p] = yv;
            if (own) yp[oy + uint32_t(u) * uint32_t(HW)] = yv;
#pragma unroll
            for (int j = 0; j + 1 < SIZE; ++j) xr[j] = xr[j + 1];
            xr[SIZE - 1] = cur[u];
          }
        }
        oy += uint32_t(kG) * uint32_t(HW);
        __syncthreads();
        if (has0) {
          const T* t = buf + toff0;
          T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
          int arg = -1;
#pragma unroll
          for (int a = 0; a < K; ++a)
#pragma unroll
            for (int b = 0; b < K; ++b) {
              if (wbits0 & (1u << (a * K + b))) {
                const T v = t[a * g.W + b];
                if (v > best) { best = v; arg = abase0 + a * g.W + b; }
              }
            }
          ypool[opool] = relu ? (best > T(0) ? best : T(0)) : best;
          mask[opool] = arg;
        }
        opool += uint32_t(kG) * uint32_t(PHW);
        c0 += kG;
        ++step;
      }
    }
    // the general loop continues with step c0's values in registers
    ptx::cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < kG; ++u) nxt[u] = pf[(slot * kG + u) * blockDim.x + threadIdx.x];
  }
  for (; c0 < cs1; c0 += kG, ++step) {
    T cur[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) cur[u] = nxt[u];
    if (c0 + kG < cs1) load_step(c0 + kG, nxt);
    T* buf = tile + (step & 1) * kG * tsz;
    if (active) {
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const int c = c0 + u;
        if (c >= cs1) break;
        T sum = T(0);
#pragma unroll
        for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xr[j]);
        const T sc = lrn::scale(sum, aN, k);
        const T yv = lrn::top(xr[pre], lrn::neg_pow(sc, beta));
        buf[u * tsz + p] = yv;
        if (own) yp[uint32_t(c) * uint32_t(HW)] = yv;
#pragma unroll
        for (int j = 0; j + 1 < SIZE; ++j) xr[j] = xr[j + 1];
        xr[SIZE - 1] = cur[u];
      }
    }
    __syncthreads();
    const int nu = min(kG, cs1 - c0);
    if (has0 && u0 < nu) {
      const T* t = buf + toff0;
      T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
      int arg = -1;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          if (wbits0 & (1u << (a * K + b))) {
            const T v = t[a * g.W + b];
            if (v > best) { best = v; arg = abase0 + a * g.W + b; }
          }
        }
      const uint32_t o = (uint32_t(img) * g.C + c0 + u0) * uint32_t(PHW) + uint32_t(po0);
      ypool[o] = relu ? (best > T(0) ? best : T(0)) : best;
      mask[o] = arg;
    }
    const int items = nu * per_u;
    for (int it = threadIdx.x + blockDim.x; it < items; it += blockDim.x) {
      const int u = it / (prows * g.PW);
      const int rem = it - u * (prows * g.PW);
      const int prl = rem / g.PW, pw = rem - prl * g.PW;
      const int hs = (pr0 + prl) * S, ws = pw * S;
      const T* t = buf + u * tsz + (hs - r0) * g.W;
      T best = sizeof(T) == 4 ? T(-3.402823466e+38f) : T(-1.7976931348623157e+308);
      int arg = -1;
#pragma unroll
      for (int a = 0; a < K; ++a)
#pragma unroll
        for (int b = 0; b < K; ++b) {
          if (hs + a < g.H && ws + b < g.W) {
            const T v = t[a * g.W + ws + b];
            if (v > best) { best = v; arg = (hs + a) * g.W + ws + b; }
          }
        }
      const uint32_t o = (uint32_t(img) * g.C + c0 + u) * uint32_t(PHW) + uint32_t((pr0 + prl) * g.PW + pw);
      ypool[o] = relu ? (best > T(0) ? best : T(0)) : best;
      mask[o] = arg;
    }
    // the next step writes the other buffer; the one after waits at its barrier
  }
}

// Backward: one thread per (pixel, channel segment).  32-bit element offsets (the
// tensors are < 2^31 elements: fusable()); the pixel's <= R x R window offsets into
// the pooled plane are computed once.
template <typename T, int SIZE, int K, int S>
__global__ void __launch_bounds__(256, 2) lrn_maxpool_bwd(const T* __restrict__ x, const T* __restrict__ pdy,
                                                       const int* __restrict__ mask, T* __restrict__ dx,
                                                       LrnPoolGeom g, T alpha, T beta, T k, bool gate_x) {
  constexpr int pre = (SIZE - 1) / 2, post = SIZE - 1 - pre;
  constexpr int R = (K + S - 1) / S;
  const uint32_t HW = uint32_t(g.H * g.W), PHW = uint32_t(g.PH * g.PW);
  const uint32_t pixels = uint32_t(g.N) * HW;
  const uint32_t segs = uint32_t((g.C + kSegB - 1) / kSegB);
  const uint32_t work = pixels * segs;
  const T aN = alpha / T(SIZE);
  const T coef = T(2) * alpha * beta / T(SIZE);
  for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < work; wi += gridDim.x * blockDim.x) {
    // consecutive threads: consecutive pixels of one segment (coalesced)
    const uint32_t seg = wi / pixels;
    const uint32_t pix = wi - seg * pixels;
    const int cs0 = int(seg) * kSegB, cs1 = min(g.C, cs0 + kSegB);
    const uint32_t img = pix / HW, hw = pix - img * HW;
    const int h = int(hw) / g.W, w = int(hw) - h * g.W;
    const int phs = h < K ? 0 : (h - K) / S + 1, phe = min(h / S + 1, g.PH);
    const int pws = w < K ? 0 : (w - K) / S + 1, pwe = min(w / S + 1, g.PW);
    // opaque per-image base pointers: element offsets are then one IMAD.WIDE each
    // (otherwise the compiler re-associates the 64-bit image offset into every
    // address: ~6 integer ops per load)
    const T* xp = opaque(x + size_t(img) * g.C * HW + hw);
    T* dxp = opaque(dx + size_t(img) * g.C * HW + hw);
    const int* mp = opaque(mask + size_t(img) * g.C * PHW);
    const T* dp = opaque(pdy + size_t(img) * g.C * PHW);
    // the pixel's <= R x R pooling windows: rows phs.., columns pws.. of the pooled
    // plane, i.e. element offsets woff0 + a*PW + b (one base pointer per window row,
    // the column step an immediate offset)
    bool wok[R][R];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) wok[a][b] = phs + a < phe && pws + b < pwe;
    const uint32_t woff0 = uint32_t(phs * g.PW + pws);
    auto xat = [&](int cc) { return (cc >= 0 && cc < g.C) ? __ldg(xp + uint32_t(cc) * HW) : T(0); };
    // the LRN top diff of channel cc at this pixel: max_pool_bwd_k's gather, in its order
    auto gather = [&](int cc, int (&m)[R][R], T (&v)[R][R]) {
      const bool live = cc < g.C;
      const uint32_t o0 = (live ? uint32_t(cc) : 0u) * PHW + woff0;
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const int* mr = mp + (o0 + uint32_t(a * g.PW));
        const T* dr = dp + (o0 + uint32_t(a * g.PW));
#pragma unroll
        for (int b = 0; b < R; ++b) {
          const bool ok = live && wok[a][b];
          m[a][b] = ok ? __ldg(mr + b) : -1;
          v[a][b] = ok ? __ldg(dr + b) : T(0);
        }
      }
    };
    auto ndy_of = [&](const int (&m)[R][R], const T (&v)[R][R]) {
      T sdy = T(0);
#pragma unroll
      for (int a = 0; a < R; ++a)
#pragma unroll
        for (int b = 0; b < R; ++b)
          if (m[a][b] == int(hw)) sdy += v[a][b];
      return sdy;
    };
    // rings over channels c - post .. c + pre: t = dy*y/scale, dy, scale^-beta (lrn_bwd_ring;
    // scale^-beta is the same function of the same scale, computed once per channel).
    // Ahead of the step for channel c they hold c-1-post .. c-1+pre (index 0 shifts out first).
    T tr[SIZE], dyr[SIZE], npr[SIZE];
#pragma unroll
    for (int j = 0; j < SIZE; ++j) { dyr[j] = T(0); npr[j] = T(1); tr[j] = T(0); }
#pragma unroll
    for (int j = 1; j < SIZE; ++j) {
      const int cc = cs0 + j - 1 - post;
      if (cc >= 0 && cc < g.C) {
        T sum = T(0);
#pragma unroll
        for (int q = 0; q < SIZE; ++q) sum = lrn::sq_acc(sum, xat(cc - pre + q));
        const T sc = lrn::scale(sum, aN, k);
        const T np = lrn::neg_pow(sc, beta);
        const T yv = lrn::top(xat(cc), np);
        int m[R][R];
        T v[R][R];
        gather(cc, m, v);
        const T d = ndy_of(m, v);
        dyr[j] = d;
        npr[j] = np;
        tr[j] = lrn::term(d, yv, sc);
      }
    }
    // x ring: x(c .. c + SIZE - 1), the window of the entering channel c + pre
    T xr[SIZE];
#pragma unroll
    for (int j = 0; j < SIZE - 1; ++j) xr[j] = xat(cs0 + j);
    xr[SIZE - 1] = T(0);
    // x (the HBM stream) two steps ahead, the pooled gather (mostly cache hits) one step
    auto load_x = [&](int c0, T (&nx)[kG]) {
#pragma unroll
      for (int u = 0; u < kG; ++u) nx[u] = c0 + u < cs1 ? xat(c0 + u + SIZE - 1) : T(0);
    };
    auto load_g = [&](int c0, int (&nm)[kG][R][R], T (&nv)[kG][R][R]) {
#pragma unroll
      for (int u = 0; u < kG; ++u) gather(c0 + u < cs1 ? c0 + u + pre : g.C, nm[u], nv[u]);
    };
    T nx[kG], nx2[kG];
    int nm[kG][R][R];
    T nv[kG][R][R];
    load_x(cs0, nx);
    load_x(cs0 + kG, nx2);
    load_g(cs0, nm, nv);
    int c0 = cs0;
    // Fast path (the interior of the segment): steps whose channels, entering channels and
    // prefetches are all in range run without bounds tests, address the tensors with
    // running 32-bit offsets, and are unrolled over SIZE steps so the rings rotate back
    // to their registers (no moves).  Same values, same operations as the general loop
    // below (which finishes the segment): bit-identical.  The general loop's integer and
    // move work was ~half of this issue-bound kernel's instructions.
    {
      uint32_t ox = uint32_t(c0 + 2 * kG + SIZE - 1) * HW;  // next x prefetch (channel c0 + 2kG + SIZE - 1)
      uint32_t og = uint32_t(c0 + kG + pre) * PHW + woff0;  // next gather (channel c0 + kG + pre)
      uint32_t od = uint32_t(c0) * HW;                      // dx of channel c0
      while (c0 + (SIZE + 2) * kG <= cs1 && c0 + (SIZE + 2) * kG + SIZE - 2 < g.C) {
#pragma unroll
        for (int st = 0; st < SIZE; ++st) {
          T cx[kG];
          int cm[kG][R][R];
          T cv[kG][R][R];
#pragma unroll
          for (int u = 0; u < kG; ++u) {
            cx[u] = nx[u];
            nx[u] = nx2[u];
#pragma unroll
            for (int a = 0; a < R; ++a)
#pragma unroll
              for (int b = 0; b < R; ++b) { cm[u][a][b] = nm[u][a][b]; cv[u][a][b] = nv[u][a][b]; }
          }
#pragma unroll
          for (int u = 0; u < kG; ++u) nx2[u] = __ldg(xp + (ox + uint32_t(u) * HW));
#pragma unroll
          for (int u = 0; u < kG; ++u)
#pragma unroll
            for (int a = 0; a < R; ++a)
#pragma unroll
              for (int b = 0; b < R; ++b) {
                const uint32_t o = og + uint32_t(u) * PHW + uint32_t(a * g.PW + b);
                nm[u][a][b] = wok[a][b] ? __ldg(mp + o) : -1;
                nv[u][a][b] = wok[a][b] ? __ldg(dp + o) : T(0);
              }
          ox += uint32_t(kG) * HW;
          og += uint32_t(kG) * PHW;
#pragma unroll
          for (int u = 0; u < kG; ++u) {
            xr[SIZE - 1] = cx[u];
#pragma unroll
            for (int j = 0; j + 1 < SIZE; ++j) { tr[j] = tr[j + 1]; dyr[j] = dyr[j + 1]; npr[j] = npr[j + 1]; }
            T sum = T(0);
#pragma unroll
            for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xr[j]);
            const T sc = lrn::scale(sum, aN, k);
            const T np = lrn::neg_pow(sc, beta);
            const T yv = lrn::top(xr[pre], np);
            const T d = ndy_of(cm[u], cv[u]);
            dyr[SIZE - 1] = d;
            npr[SIZE - 1] = np;
            tr[SIZE - 1] = lrn::term(d, yv, sc);
            T acc = T(0);
#pragma unroll
            for (int j = 0; j < SIZE; ++j) acc = lrn::add_(acc, tr[j]);
            const T xc = xr[0];
            const T gval = lrn::grad(dyr[post], npr[post], coef, xc, acc);
            dxp[od] = (!gate_x || xc > T(0)) ? gval : T(0);
            od += HW;
#pragma unroll
            for (int j = 0; j + 1 < SIZE; ++j) xr[j] = xr[j + 1];
          }
          c0 += kG;
        }
      }
    }
    for (; c0 < cs1; c0 += kG) {
      T cx[kG];
      int cm[kG][R][R];
      T cv[kG][R][R];
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        cx[u] = nx[u];
        nx[u] = nx2[u];
#pragma unroll
        for (int a = 0; a < R; ++a)
#pragma unroll
          for (int b = 0; b < R; ++b) { cm[u][a][b] = nm[u][a][b]; cv[u][a][b] = nv[u][a][b]; }
      }
      if (c0 + 2 * kG < cs1) load_x(c0 + 2 * kG, nx2);  // in flight during this step and the next
      if (c0 + kG < cs1) load_g(c0 + kG, nm, nv);
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const int c = c0 + u;
        if (c >= cs1) break;
        xr[SIZE - 1] = cx[u];  // x(c .. c + SIZE - 1)
#pragma unroll
        for (int j = 0; j + 1 < SIZE; ++j) { tr[j] = tr[j + 1]; dyr[j] = dyr[j + 1]; npr[j] = npr[j + 1]; }
        if (c + pre < g.C) {
          T sum = T(0);
#pragma unroll
          for (int j = 0; j < SIZE; ++j) sum = lrn::sq_acc(sum, xr[j]);
          const T sc = lrn::scale(sum, aN, k);
          const T np = lrn::neg_pow(sc, beta);
          const T yv = lrn::top(xr[pre], np);
          const T d = ndy_of(cm[u], cv[u]);
          dyr[SIZE - 1] = d;
          npr[SIZE - 1] = np;
          tr[SIZE - 1] = lrn::term(d, yv, sc);
        } else {
          dyr[SIZE - 1] = T(0); npr[SIZE - 1] = T(1); tr[SIZE - 1] = T(0);
        }
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < SIZE; ++j) acc = lrn::add_(acc, tr[j]);
        const T xc = xr[0];
        const T gval = lrn::grad(dyr[post], npr[post], coef, xc, acc);
        dxp[uint32_t(c) * HW] = (!gate_x || xc > T(0)) ? gval : T(0);
#pragma unroll
        for (int j = 0; j + 1 < SIZE; ++j) xr[j] = xr[j + 1];
      }
    }
  }
}

LrnPoolGeom lrn_pool_geom(const PoolDescSlot& d, int smem_cap_elems) {
  const auto& p = d.p;
  LrnPoolGeom g{p.n, p.c, p.h, p.w, d.PH, d.PW, 1, 0, 0, (p.c + kSeg - 1) / kSeg};
  const int K = p.kernel_h, S = p.stride_h;
  // band height: about 512 input pixels per block
  int tr = std::max(1, ((512 / std::max(1, p.w)) - K) / S + 1);
  tr = std::min(tr, d.PH);
  while (tr > 1 && ((tr - 1) * S + K) * p.w > std::min(1024, smem_cap_elems)) --tr;
  g.TR = tr;
  g.rows_in = (tr - 1) * S + K;
  g.bands = (d.PH + tr - 1) / tr;
  return g;
}

bool fusable(const PoolDescSlot& d, int size) {
  const auto& p = d.p;
  const bool window = p.kernel_h == p.kernel_w && p.stride_h == p.stride_w &&
                      ((p.kernel_h == 3 && p.stride_h == 2) || (p.kernel_h == 2 && p.stride_h == 2));
  return p.method == CDNN_POOL_MAX && !p.global_pooling && p.pad_h == 0 && p.pad_w == 0 && window &&
         (size == 3 || size == 5) && p.kernel_h * p.w <= 1024 &&
         uint64_t(p.n) * p.c * p.h * p.w < (1ull << 31) &&
         uint64_t(p.n) * p.h * p.w * ((p.c + kSeg - 1) / kSeg) < (1ull << 31);
}

template <typename T, int SIZE, int K, int S>
void launch_fwd(Ctx* c, cudaStream_t st, const PoolDescSlot& d, const T* x, T* yn, T* yp, int* m, double alpha,
                double beta, double k, bool relu) {
  const LrnPoolGeom g = lrn_pool_geom(d, 1024);
  const int threads = ((g.rows_in * g.W + 31) / 32) * 32;
  const size_t smem = (size_t(2) * kG * g.rows_in * g.W + size_t(kPF) * kG * threads) * sizeof(T);
  static size_t attr_smem[16] = {};
  if (smem > 48 * 1024 && attr_smem[c->device & 15] < smem) {
    CDNN_CUDA(cudaFuncSetAttribute(lrn_maxpool_fwd<T, SIZE, K, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
    attr_smem[c->device & 15] = smem;
  }
  lrn_maxpool_fwd<T, SIZE, K, S><<<dim3(g.bands, g.segs, g.N), threads, smem, st>>>(x, yn, yp, m, g, T(alpha),
                                                                                    T(beta), T(k), relu);
  check_launch("lrn_maxpool_fwd");
  count_launch(c);
}

template <typename T, int SIZE, int K, int S>
void launch_bwd(Ctx* c, cudaStream_t st, const PoolDescSlot& d, const T* x, const T* pdy, const int* m, T* dx,
                double alpha, double beta, double k, bool gate_x) {
  const LrnPoolGeom g = lrn_pool_geom(d, 1024);
  const int64_t work = int64_t(g.N) * g.H * g.W * ((g.C + kSegB - 1) / kSegB);
  lrn_maxpool_bwd<T, SIZE, K, S><<<grid_for(work, 256), 256, 0, st>>>(x, pdy, m, dx, g, T(alpha), T(beta), T(k),
                                                                       gate_x);
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
    *out = fusable(pool_desc(c, pool_desc_h), local_size) ? 1 : 0;
  });
}

int cdnn_lrn_pool_forward(cdnn_ctx ctx, cdnn_handle pool_desc_h, cdnn_handle x, cdnn_handle lrn_top,
                          cdnn_handle pool_top, cdnn_handle mask, int local_size, double alpha, double beta, double k,
                          int flags, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    const PoolDescSlot d = pool_desc(c, pool_desc_h);
    if (!fusable(d, local_size)) fail(CDNN_INVALID_ARGUMENT, "lrn_pool: unsupported LRN / pooling combination");
    BufferSlot& X = buffer(c, x, "lrn_pool x");
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
    if (!fusable(d, local_size)) fail(CDNN_INVALID_ARGUMENT, "lrn_pool: unsupported LRN / pooling combination");
    if (gate && gate != x) fail(CDNN_INVALID_ARGUMENT, "lrn_pool backward: the ReLU gate must be the LRN bottom x");
    BufferSlot& X = buffer(c, x, "lrn_pool_bwd x");
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
