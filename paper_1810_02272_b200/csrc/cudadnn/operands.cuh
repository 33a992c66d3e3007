// operands.cuh — operand "views" for the implicit-GEMM engines.
//
// Every GEMM-shaped op of the hot path is expressed as
//     D[m][n] = sum_k A(m, k) * B(n, k)
// where A and B are *views* that never materialise im2col buffers.  A view
// factors element addressing into a per-row part and a per-k part so the
// gather producers can compute all addresses of a slab first and then issue
// every load independently (memory-level parallelism):
//     Row row(r)      per-row state  (e.g. output pixel -> image, h0, w0)
//     Kx  kx(k)       per-k state    (e.g. filter tap -> channel offset, dh, dw)
//     bool addr(Row, Kx, int& off)   element offset from base(), false = zero
// Offsets are 32-bit: every tensor on the path is < 2^31 elements (checked by
// the host).  The epilogues turn the fp32/fp64 accumulator of D into the op's
// output layout.
#pragma once

#include <cstdint>
#include <type_traits>

namespace cdnn {

// Granlund–Montgomery division by an invariant positive divisor < 2^31:
// q = (t + ((n - t) >> 1)) >> (l - 1), t = mulhi(n, magic), exact for n < 2^32.
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

// Generic scalar fetch on top of the address API (SIMT engine, tails).
template <class V, class R>
__device__ __forceinline__ auto view_at(const V& v, const R& rw, int k) {
  using E = std::remove_const_t<std::remove_pointer_t<decltype(v.base())>>;
  int off;
  const auto kx = v.kx(k);
  return v.addr(rw, kx, off) ? __ldg(v.base() + off) : E(0);
}

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
  struct Row { int off; bool ok; };
  struct Kx { int off; bool ok; };
  __device__ __forceinline__ const T* base() const { return p; }
  __device__ __forceinline__ Row row(int r) const { return Row{int(r * sr), r < rows}; }
  __device__ __forceinline__ Kx kx(int k) const { return Kx{int(k * sk), k < K}; }
  __device__ __forceinline__ bool addr(const Row& rw, const Kx& x, int& off) const {
    off = rw.off + x.off;
    return rw.ok && x.ok;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    return (rw.ok && k < K) ? __ldg(p + rw.off + int(k * sk)) : T(0);
  }
  __device__ __forceinline__ bool m_contig() const { return mcontig; }
};

// Marker: the operand is K-contiguous and 16-byte aligned, loaded by TMA.
// Marks an operand pre-split into tf32 hi / lo copies in HBM (3xTF32): TMA loads both
// halves, the producer warps do no conversion.
struct TmaSplitView;
struct TmaView {
  struct Row { int off; bool ok; };
  struct Kx { int off; bool ok; };
  __device__ __forceinline__ const float* base() const { return nullptr; }
  __device__ __forceinline__ Row row(int) const { return Row{0, false}; }
  __device__ __forceinline__ Kx kx(int) const { return Kx{0, false}; }
  __device__ __forceinline__ bool addr(const Row&, const Kx&, int& off) const { off = 0; return false; }
  __device__ __forceinline__ float at(const Row&, int) const { return 0.f; }
  __device__ __forceinline__ bool m_contig() const { return false; }
};
struct TmaSplitView : TmaView {};

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
  struct Row { int base; int h0, w0; bool ok; };
  struct Kx { int off; int dh, dw; bool ok; };
  __device__ __forceinline__ const T* base() const { return x; }
  __device__ __forceinline__ Row row(int r) const {
    Row rw;
    rw.ok = r < rows;
    const uint32_t img = g.div_PQ.div(r), pq = r - img * g.P * g.Q;
    const uint32_t pp = g.div_Q.div(pq), qq = pq - pp * g.Q;
    rw.h0 = int(pp) * g.sh - g.ph;
    rw.w0 = int(qq) * g.sw - g.pw;
    rw.base = int(img) * g.C * g.H * g.W + rw.h0 * g.W + rw.w0;
    return rw;
  }
  __device__ __forceinline__ Kx kx(int k) const {
    if (k >= K) return Kx{0, 0, 0, false};
    const int4 t = __ldg(reinterpret_cast<const int4*>(taps) + k);
    return Kx{t.x, t.y, t.z, true};
  }
  __device__ __forceinline__ bool addr(const Row& rw, const Kx& t, int& off) const {
    const int h = rw.h0 + t.dh, w = rw.w0 + t.dw;
    off = rw.base + t.off;
    return rw.ok && t.ok && unsigned(h) < unsigned(g.H) && unsigned(w) < unsigned(g.W);
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const { return view_at(*this, rw, k); }
  __device__ __forceinline__ bool m_contig() const { return true; }
};

// Backward-data A: rows m = bottom pixel (img, h, w); k = (co, kr, ks) in the group.
// A(m,k) = dy[img][co][(h+ph-kr*dh)/sh][(w+pw-ks*dw)/sw] when integral and in range.
struct DgradTap { int off; int dh; int dw; int pad_; };  // off = co*P*Q
template <typename T, bool UNIT_STRIDE = false>
struct ConvDgradA {
  const T* dy;           // top diff, offset to the group's first channel
  const DgradTap* taps;  // Cog*R*S entries
  ConvGeom g;
  int rows, K;
  struct Row { int base; int hp, wp; bool ok; };
  struct Kx { int off; int dh, dw; bool ok; };
  __device__ __forceinline__ const T* base() const { return dy; }
  __device__ __forceinline__ Row row(int r) const {
    Row rw;
    rw.ok = r < rows;
    const uint32_t img = g.div_HW.div(r), hw = r - img * g.H * g.W;
    const uint32_t h = g.div_W.div(hw), w = hw - h * g.W;
    rw.hp = int(h) + g.ph;
    rw.wp = int(w) + g.pw;
    rw.base = int(img) * g.Co * g.P * g.Q;
    return rw;
  }
  __device__ __forceinline__ Kx kx(int k) const {
    if (k >= K) return Kx{0, 0, 0, false};
    const int4 t = __ldg(reinterpret_cast<const int4*>(taps) + k);
    return Kx{t.x, t.y, t.z, true};
  }
  __device__ __forceinline__ bool addr(const Row& rw, const Kx& t, int& off) const {
    int pn = rw.hp - t.dh, qn = rw.wp - t.dw;
    bool ok = rw.ok && t.ok && pn >= 0 && qn >= 0;
    if constexpr (!UNIT_STRIDE) {
      const int ps = pn / g.sh, qs = qn / g.sw;
      ok = ok && ps * g.sh == pn && qs * g.sw == qn;
      pn = ps;
      qn = qs;
    }
    ok = ok && pn < g.P && qn < g.Q;
    off = rw.base + t.off + pn * g.Q + qn;
    return ok;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const { return view_at(*this, rw, k); }
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
  struct Row { int off; bool ok; };
  struct Kx { int off; bool ok; };
  __device__ __forceinline__ const T* base() const { return w; }
  __device__ __forceinline__ Row row(int r) const { return Row{r * RS, r < rows}; }
  __device__ __forceinline__ Kx kx(int k) const { return k < K ? Kx{__ldg(koff + k), true} : Kx{0, false}; }
  __device__ __forceinline__ bool addr(const Row& rw, const Kx& x, int& off) const {
    off = rw.off + x.off;
    return rw.ok && x.ok;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const { return view_at(*this, rw, k); }
  __device__ __forceinline__ bool m_contig() const { return false; }
};

// Backward-filter A: rows m = tap (ci, kr, ks); k = output pixel (img, p, q).
// With `ones_row` an extra row m = rows holds 1.0 for every valid k, so the
// GEMM also produces D[rows][co] = sum_k dy(co, k): the bias gradient rides
// along on the tensor cores (no separate reduction kernel).
template <typename T>
struct ConvWgradA {
  const T* x;            // bottom data, offset to the group's first channel
  const ConvTap* taps;   // Cg*R*S
  ConvGeom g;
  int rows, K;           // rows = Cg*R*S, K = N*P*Q
  bool ones_row;
  struct Row { int off, dh, dw; bool ok; bool one; };
  struct Kx { int base; int h0, w0; bool ok; };
  static constexpr bool kHasOnes = true;
  __device__ __forceinline__ const T* base() const { return x; }
  __device__ __forceinline__ Row row(int r) const {
    if (r >= rows) return Row{0, 0, 0, false, ones_row && r == rows};
    const int4 t = __ldg(reinterpret_cast<const int4*>(taps) + r);
    return Row{t.x, t.y, t.z, true, false};
  }
  __device__ __forceinline__ bool is_one(const Row& rw) const { return rw.one; }
  __device__ __forceinline__ Kx kx(int k) const {
    Kx p;
    p.ok = k < K;
    const uint32_t img = g.div_PQ.div(k), pq = k - img * g.P * g.Q;
    const uint32_t pp = g.div_Q.div(pq), qq = pq - pp * g.Q;
    p.h0 = int(pp) * g.sh - g.ph;
    p.w0 = int(qq) * g.sw - g.pw;
    p.base = int(img) * g.C * g.H * g.W + p.h0 * g.W + p.w0;
    return p;
  }
  __device__ __forceinline__ bool addr(const Row& rw, const Kx& p, int& off) const {
    const int h = p.h0 + rw.dh, w = p.w0 + rw.dw;
    off = p.base + rw.off;
    return rw.ok && p.ok && unsigned(h) < unsigned(g.H) && unsigned(w) < unsigned(g.W);
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const {
    if (rw.one) return k < K ? T(1) : T(0);
    return view_at(*this, rw, k);
  }
  __device__ __forceinline__ bool m_contig() const { return false; }
};

// backward-filter epilogue: dw[co][tap] += D[tap][co]; the ones row adds
// D[Kc][co] into db[co] (param diffs accumulate, layers.hpp:84-86).
template <typename T>
struct ConvWgradEpi {
  T* dw;                 // offset to the group's first filter
  T* db;                 // offset to the group's first channel, may be null
  int Kc;
  __device__ __forceinline__ void store(int m, int n, T acc, int) const {
    if (m < Kc) {
      if (!dw) return;
      T* o = dw + int64_t(n) * Kc + m;
      *o = *o + acc;
    } else if (db) {
      db[n] = db[n] + acc;
    }
  }
};

// Reduce epilogue of the tap-shift backward-filter partials: m' = tap*Cg + c
// (channel innermost) -> Caffe filter index c*R*S + tap; m' == Kc -> bias.
template <typename T>
struct ConvWgradPermEpi {
  T* dw;                 // offset to the group's first filter, may be null
  T* db;                 // offset to the group's first channel, may be null
  int Kc, Cg, RS;
  __device__ __forceinline__ void store(int m, int n, T acc, int) const {
    if (m < Kc) {
      if (!dw) return;
      const int tap = m / Cg, c = m - tap * Cg;
      T* o = dw + int64_t(n) * Kc + c * RS + tap;
      *o = *o + acc;
    } else if (db) {
      db[n] = db[n] + acc;
    }
  }
};

// Backward-filter B: rows n = co in the group; k = output pixel (img, p, q).
template <typename T>
struct ConvWgradB {
  const T* dy;           // top diff, offset to the group's first channel
  ConvGeom g;
  int rows, K;
  struct Row { int off; bool ok; };
  struct Kx { int base; bool ok; };
  __device__ __forceinline__ const T* base() const { return dy; }
  __device__ __forceinline__ Row row(int r) const { return Row{r * g.P * g.Q, r < rows}; }
  __device__ __forceinline__ Kx kx(int k) const {
    const uint32_t img = g.div_PQ.div(k), pq = k - img * g.P * g.Q;
    return Kx{int(img) * g.Co * g.P * g.Q + int(pq), k < K};
  }
  __device__ __forceinline__ bool addr(const Row& rw, const Kx& p, int& off) const {
    off = p.base + rw.off;
    return rw.ok && p.ok;
  }
  __device__ __forceinline__ T at(const Row& rw, int k) const { return view_at(*this, rw, k); }
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
  // 16 consecutive n of one m (a tcgen05.ld row): every read of the old C is
  // issued before the first store (the compiler cannot reorder loads past
  // possibly-aliasing stores, which serialised one memory latency per element).
  __device__ __forceinline__ void store16(int m, int n0, const uint32_t (&r)[16], int N) const {
    T* o = out + int64_t(m) * sm + int64_t(n0) * sn;
    T prev[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) prev[j] = (beta != T(0) && n0 + j < N) ? o[int64_t(j) * sn] : T(0);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (n0 + j < N) {
        T v = alpha * T(__uint_as_float(r[j]));
        if (beta != T(0)) v += beta * prev[j];
        if (bias) v += bias[bias_on_m ? m : n0 + j];
        if (relu) v = v > T(0) ? v : T(0);
        o[int64_t(j) * sn] = v;
      }
    }
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
  bool relu = false;     // fused in-place ReLU (max(v, 0), strict > like layers.cpp:184)
  __device__ __forceinline__ void store(int m, int n, T acc, int) const {
    const uint32_t img = g.div_PQ.div(m), pq = m - img * g.P * g.Q;
    T v = acc;
    if (bias) v += bias[n];
    if (relu) v = v > T(0) ? v : T(0);
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
