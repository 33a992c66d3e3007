// operands.cuh — operand "views" for the implicit-GEMM engines.
//
// Every GEMM-shaped op of the hot path is expressed as
//     D[m][n] = sum_k A(m, k) * B(n, k)
// where A and B are *views*: a `row(r)` step that precomputes per-row state
// once, and an `at(row, k)` fetch that returns the element (0 outside the
// matrix, so tile tails contribute nothing).  The views below cover the dense
// row-major matrices of InnerProduct / gemm (any transpose) and the three
// convolution contractions (forward im2col, backward-data, backward-filter)
// without materialising im2col buffers.  The epilogues turn the fp32/fp64
// accumulator of D into the op's output layout.
#pragma once

#include <cstdint>

namespace cdnn {

// Granlund–Montgomery division by an invariant positive divisor < 2^31:
// q = mulhi(n, magic) >> shift, exact for 0 <= n < 2^31.
struct FastDiv {
  uint32_t d = 1, magic = 0, shift = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (d == 1) { magic = 0; shift = 0; return; }
    uint32_t s = 0;
    while ((1u << s) < d) ++s;           // s = ceil(log2 d)
    const uint64_t one = 1;
    magic = static_cast<uint32_t>(((one << 32) * ((one << s) - d)) / d + 1);
    shift = s - 1;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    if (d == 1) return n;
    const uint32_t t = __umulhi(n, magic);
    return (t + ((n - t) >> 1)) >> shift;
  }
};

// ---------------------------------------------------------------------------
// Dense strided matrix: A(r, k) = p[r*sr + k*sk].  `mcontig` says which index
// is memory-contiguous; it only picks the thread->element map of the gather
// (lanes walk the contiguous index so global loads coalesce).
template <typename T>
struct DenseView {
  const T* p;
  int64_t sr, sk;
  int rows, K;
  bool mcontig;
  struct Row { int64_t off; bool ok; };
  __device__ __forceinline__ Row row(int r) const { return Row{int64_t(r) * sr, r < rows}; }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    return (rw.ok && k < K) ? __ldg(p + rw.off + int64_t(k) * sk) : T(0);
  }
  __device__ __forceinline__ bool m_contig() const { return mcontig; }
};

// Marker: the operand is K-contiguous and 16-byte aligned, loaded by TMA.
struct TmaView {
  struct Row { int dummy; };
  __device__ __forceinline__ Row row(int) const { return Row{0}; }
  __device__ __forceinline__ float at(const Row&, int) const { return 0.f; }
  __device__ __forceinline__ bool m_contig() const { return false; }
};

// Per-k offsets of a convolution filter tap, shared by forward (A, k = (ci,kr,ks))
// and backward-filter (A, rows = (ci,kr,ks)):  x_off = ci*H*W + kr*dh*W + ks*dw.
struct ConvTap { int off; int dh; int dw; int pad_; };

// Convolution geometry shared by all three views (one group).
struct ConvGeom {
  int N, C, H, W;        // bottom
  int Co, P, Q;          // top channels / extents
  int R, S;              // kernel
  int sh, sw, ph, pw, dh, dw;
  int group, Cg, Cog;    // C/group, Co/group
  FastDiv div_PQ, div_Q, div_HW, div_W;
};

// Forward A: rows m = output pixel (img, p, q); k = (ci, kr, ks) within the group.
template <typename T>
struct ConvFwdA {
  const T* x;            // bottom data, offset to the group's first channel
  const ConvTap* taps;   // Cg*R*S entries
  ConvGeom g;
  int rows, K;
  struct Row { int64_t base; int h0, w0; bool ok; };
  __device__ __forceinline__ Row row(int r) const {
    Row rw; rw.ok = r < rows;
    const uint32_t img = g.div_PQ.div(r), pq = r - img * g.P * g.Q;
    const uint32_t pp = g.div_Q.div(pq), qq = pq - pp * g.Q;
    rw.h0 = int(pp) * g.sh - g.ph; rw.w0 = int(qq) * g.sw - g.pw;
    rw.base = int64_t(img) * g.C * g.H * g.W + int64_t(rw.h0) * g.W + rw.w0;
    return rw;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    if (!rw.ok || k >= K) return T(0);
    const ConvTap t = taps[k];
    const int h = rw.h0 + t.dh, w = rw.w0 + t.dw;
    if (unsigned(h) >= unsigned(g.H) || unsigned(w) >= unsigned(g.W)) return T(0);
    return __ldg(x + rw.base + t.off);
  }
  __device__ __forceinline__ bool m_contig() const { return true; }
};

// Backward-data A: rows m = bottom pixel (img, h, w); k = (co, kr, ks) in the group.
// A(m,k) = dy[img][co][(h+ph-kr*dh)/sh][(w+pw-ks*dw)/sw] when integral and in range.
struct DgradTap { int off; int dh; int dw; int pad_; };  // off = co*P*Q
template <typename T>
struct ConvDgradA {
  const T* dy;           // top diff, offset to the group's first channel
  const DgradTap* taps;  // Cog*R*S entries
  ConvGeom g;
  int rows, K;
  struct Row { int64_t base; int hp, wp; bool ok; };
  __device__ __forceinline__ Row row(int r) const {
    Row rw; rw.ok = r < rows;
    const uint32_t img = g.div_HW.div(r), hw = r - img * g.H * g.W;
    const uint32_t h = g.div_W.div(hw), w = hw - h * g.W;
    rw.hp = int(h) + g.ph; rw.wp = int(w) + g.pw;
    rw.base = int64_t(img) * g.Co * g.P * g.Q;
    return rw;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    if (!rw.ok || k >= K) return T(0);
    const DgradTap t = taps[k];
    int pn = rw.hp - t.dh, qn = rw.wp - t.dw;
    if (pn < 0 || qn < 0) return T(0);
    if (g.sh != 1) { if (pn % g.sh) return T(0); pn /= g.sh; }
    if (g.sw != 1) { if (qn % g.sw) return T(0); qn /= g.sw; }
    if (pn >= g.P || qn >= g.Q) return T(0);
    return __ldg(dy + rw.base + t.off + pn * g.Q + qn);
  }
  __device__ __forceinline__ bool m_contig() const { return true; }
};

// Backward-data B: rows n = ci in the group; k = (co, kr, ks):
// B(ci, k) = w[co][ci][kr][ks]  (weights offset to the group's first filter).
template <typename T>
struct ConvDgradB {
  const T* w;
  const int* koff;       // per k: co*Cg*R*S + kr*S + ks
  int RS;
  int rows, K;
  struct Row { int64_t off; bool ok; };
  __device__ __forceinline__ Row row(int r) const { return Row{int64_t(r) * RS, r < rows}; }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    return (rw.ok && k < K) ? __ldg(w + rw.off + koff[k]) : T(0);
  }
  __device__ __forceinline__ bool m_contig() const { return false; }
};

// Backward-filter A: rows m = tap (ci, kr, ks); k = output pixel (img, p, q).
template <typename T>
struct ConvWgradA {
  const T* x;            // bottom data, offset to the group's first channel
  const ConvTap* taps;   // Cg*R*S
  ConvGeom g;
  int rows, K;           // rows = Cg*R*S, K = N*P*Q
  struct Row { int off, dh, dw; bool ok; };
  __device__ __forceinline__ Row row(int r) const {
    Row rw; rw.ok = r < rows;
    if (rw.ok) { const ConvTap t = taps[r]; rw.off = t.off; rw.dh = t.dh; rw.dw = t.dw; }
    else { rw.off = 0; rw.dh = 0; rw.dw = 0; }
    return rw;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    if (!rw.ok || k >= K) return T(0);
    const uint32_t img = g.div_PQ.div(k), pq = k - img * g.P * g.Q;
    const uint32_t pp = g.div_Q.div(pq), qq = pq - pp * g.Q;
    const int h = int(pp) * g.sh - g.ph + rw.dh, w = int(qq) * g.sw - g.pw + rw.dw;
    if (unsigned(h) >= unsigned(g.H) || unsigned(w) >= unsigned(g.W)) return T(0);
    return __ldg(x + int64_t(img) * g.C * g.H * g.W + int64_t(h) * g.W + w +
                 (rw.off - rw.dh * g.W - rw.dw));
  }
  __device__ __forceinline__ bool m_contig() const { return false; }
};

// Backward-filter B: rows n = co in the group; k = output pixel (img, p, q).
template <typename T>
struct ConvWgradB {
  const T* dy;           // top diff, offset to the group's first channel
  ConvGeom g;
  int rows, K;
  struct Row { int64_t off; bool ok; };
  __device__ __forceinline__ Row row(int r) const { return Row{int64_t(r) * g.P * g.Q, r < rows}; }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    if (!rw.ok || k >= K) return T(0);
    const uint32_t img = g.div_PQ.div(k), pq = k - img * g.P * g.Q;
    return __ldg(dy + int64_t(img) * g.Co * g.P * g.Q + rw.off + pq);
  }
  __device__ __forceinline__ bool m_contig() const { return false; }
};

// ---------------------------------------------------------------------------
// Epilogues.  store(m, n, acc, split) is called once per in-range element.

// out[m*sm + n*sn] = alpha*acc + beta*out (beta==0 never reads) + bias[m|n], opt. ReLU
template <typename T>
struct StoreEpi {
  T* out;
  int64_t sm, sn;
  T alpha, beta;
  const T* bias;         // may be null
  bool bias_on_m;
  bool relu;
  __device__ __forceinline__ void store(int m, int n, T acc, int) const {
    T* o = out + int64_t(m) * sm + int64_t(n) * sn;
    T v = alpha * acc;
    if (beta != T(0)) v += beta * *o;
    if (bias) v += bias[bias_on_m ? m : n];
    if (relu) v = v > T(0) ? v : T(0);
    *o = v;
  }
};

// split-K partials: ws[split][n][m] (m contiguous so lanes coalesce)
template <typename T>
struct PartialEpi {
  T* ws;
  int M, N;
  __device__ __forceinline__ void store(int m, int n, T acc, int split) const {
    ws[(int64_t(split) * N + n) * M + m] = acc;
  }
};

// conv forward: y[img][co][p][q] = acc + bias[co]  (m = img*P*Q + pq, n = co in group)
template <typename T>
struct ConvFwdEpi {
  T* y;                  // offset to the group's first output channel
  const T* bias;         // offset to the group's first channel, may be null
  ConvGeom g;
  __device__ __forceinline__ void store(int m, int n, T acc, int) const {
    const uint32_t img = g.div_PQ.div(m), pq = m - img * g.P * g.Q;
    T v = acc;
    if (bias) v += bias[n];
    y[(int64_t(img) * g.Co + n) * g.P * g.Q + pq] = v;
  }
};

// conv backward-data: dx[img][ci][h][w] = acc  (m = img*H*W + hw, n = ci in group)
template <typename T>
struct ConvDgradEpi {
  T* dx;                 // offset to the group's first channel
  ConvGeom g;
  __device__ __forceinline__ void store(int m, int n, T acc, int) const {
    const uint32_t img = g.div_HW.div(m), hw = m - img * g.H * g.W;
    dx[(int64_t(img) * g.C + n) * g.H * g.W + hw] = acc;
  }
};

}  // namespace cdnn
