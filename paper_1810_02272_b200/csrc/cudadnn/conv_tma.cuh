// conv_tma.cuh — TMA-fed direct convolution on tcgen05 (stride 1, dilation 1, NCHW fp32).
//
//   out[img][n][p][q] = sum_{tap=(kr,ks)} sum_{c} Wt[tap][n][c] * in[img][c][p - oh + kr][q - ow + ks]
//
// Forward:       in = x,  out = y,  Wt = W repacked [tap][co][ci],  (oh, ow) = (pad_h, pad_w)
// Backward-data: in = dy, out = dx, Wt = W repacked [tap][ci][co] with the
//                tap flipped, (oh, ow) = (R-1-pad_h, S-1-pad_w)
//
// GEMM view per output tile: M = 128 output pixels (four 32-pixel atoms of
// 32/TW image rows, NB images x TH rows x TW columns), N = BN output
// channels, K = taps x input channels.  For every (tap, channel block) TMA
// brings, per atom, the input window displaced by the tap offset into a
// staging buffer; out-of-range coordinates are zero-filled by TMA, which
// implements the padding.  TMA only accepts 16-byte aligned innermost
// coordinates, so the window starts at the aligned column below the tap's
// column and the converter warps apply the remaining 0..3-element shift while
// writing the UMMA MN-major tf32 layout (128B_BASE32B: rows of 32 pixels per
// channel, 32-byte units XOR-swizzled by row) — in 3xTF32 mode they also
// split every value into tf32 hi + lo.  The weight slice
// Wt[tap][n0:n0+BN][c0:c0+CB] arrives by a second TMA, K-major and pre-split
// by the repack kernel.  No thread computes an im2col address.
#pragma once

#include <cstdint>

#include "gemm_tc.cuh"
#include "ptx.cuh"

namespace cdnn {
namespace tcconv {

constexpr int kThreads = 192;  // warp0 TMA, warp1 MMA/TMEM, warps 2-5 convert + epilogue

struct ConvTmaArgs {
  int N, Cin, Hin, Win;     // input of the direct conv (x for fwd, dy for dgrad)
  int Cout, P, Q;           // output extents
  int R, S, oh, ow;         // taps and the coordinate offset of tap (0,0)
  int TH, NB;               // tile rows per image and images per tile (TW, CB are template params)
  int cblocks;              // ceil(Cin / CB)
  int tiles_q, tiles_p;     // tiles along q and p
  const float* bias;        // may be null (fwd only)
  float* out;
  int relu;                 // fused in-place ReLU (fwd only)
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(ptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// UMMA smem descriptor with explicit layout type and byte offsets.
__device__ __forceinline__ uint64_t make_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7) << 61;
  return d;
}

// per stage: A hi/lo tiles (128 px x CB), B hi/lo (BN x CB), staging window
template <int TW, int CB>
__host__ __device__ constexpr uint32_t stg_bytes() { return 4u * CB * (32 / TW) * (TW + 4) * 4u; }
template <int CB>
__host__ __device__ constexpr uint32_t a_bytes() { return 128u * CB * 4u; }
template <int BN, int CB>
__host__ __device__ constexpr uint32_t b_bytes() { return uint32_t(BN) * CB * 4u; }
__host__ __device__ constexpr uint32_t round1k(uint32_t b) { return (b + 1023u) & ~1023u; }

template <int BN, bool SPLIT, int TW, int CB>
__host__ __device__ constexpr uint32_t stage_bytes() {
  return round1k((a_bytes<CB>() + b_bytes<BN, CB>()) * (SPLIT ? 2 : 1) + stg_bytes<TW, CB>());
}

template <int BN, bool SPLIT, int TW, int CB>
__host__ __device__ constexpr int stages() {
  // as many stages as fit in ~200 KB (2..6)
  return int(200u * 1024u / stage_bytes<BN, SPLIT, TW, CB>()) > 6 ? 6
         : int(200u * 1024u / stage_bytes<BN, SPLIT, TW, CB>()) < 2 ? 2
                                                                     : int(200u * 1024u / stage_bytes<BN, SPLIT, TW, CB>());
}

template <int BN, bool SPLIT, int TW, int CB>
__host__ __device__ constexpr int smem_bytes() {
  return 1024 + stages<BN, SPLIT, TW, CB>() * int(stage_bytes<BN, SPLIT, TW, CB>()) +
         (3 * stages<BN, SPLIT, TW, CB>() + 1) * 8 + 16;
}

// ATOM_32B swizzle of the MN-major tf32 UMMA layout (128B_BASE32B): 32-byte
// units of a 128-byte row XOR'd with the row index mod 4.
__device__ __forceinline__ uint32_t atom32_off(uint32_t row, uint32_t col) {
  return row * 128u + ((((col >> 3) ^ row) & 3u) << 5) + ((col & 7u) << 2);
}

template <int BN, bool SPLIT, int TW, int CB>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tma_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_w_hi,
                    const __grid_constant__ CUtensorMap tm_w_lo, const ConvTmaArgs a) {
  constexpr int ST = stages<BN, SPLIT, TW, CB>();
  constexpr int RB = 32 / TW;          // image rows per 32-pixel atom
  constexpr int SW = TW + 4;           // staged window width (shift 0..3)
  constexpr uint32_t A_BYTES = a_bytes<CB>(), B_BYTES = b_bytes<BN, CB>();
  constexpr uint32_t STAGE = stage_bytes<BN, SPLIT, TW, CB>();
  constexpr uint32_t BOX = uint32_t(SW * RB * CB) * 4u;  // one atom's staged window
  constexpr uint32_t TMEM_COLS = tc::tmem_cols_for(BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage: [A hi | B hi | A lo | B lo | staging]
  auto a_hi = [&](int s) { return smem + s * STAGE; };
  auto b_hi = [&](int s) { return smem + s * STAGE + A_BYTES; };
  auto a_lo = [&](int s) { return smem + s * STAGE + A_BYTES + B_BYTES; };
  auto b_lo = [&](int s) { return smem + s * STAGE + 2 * A_BYTES + B_BYTES; };
  auto stg = [&](int s) { return smem + s * STAGE + (A_BYTES + B_BYTES) * (SPLIT ? 2 : 1); };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
  uint64_t* conv = full + ST;
  uint64_t* empty = conv + ST;
  uint64_t* accum = empty + ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x;
  const int tq = t % a.tiles_q;
  t /= a.tiles_q;
  const int tp = t % a.tiles_p;
  const int tn = t / a.tiles_p;
  const int q0 = tq * TW, p0 = tp * a.TH, img0 = tn * a.NB;
  const int n0 = blockIdx.y * BN;
  const int nk = a.R * a.S * a.cblocks;
  const int hgroups = a.TH / RB;
  const int nat = min(4, a.NB * hgroups);  // 32-pixel atoms in this tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&conv[s], 4);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accum, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tm_in);
      ptx::tma_prefetch_desc(&tm_w_hi);
      if constexpr (SPLIT) ptx::tma_prefetch_desc(&tm_w_lo);
      int stage = 0;
      uint32_t phase = 0;
      int cb = 0, kr = 0, ks = 0;
      for (int kt = 0; kt < nk; ++kt) {
        const int tap = kr * a.S + ks;
        const int x0a = ((q0 - a.ow + ks) >> 2) << 2;  // TMA needs 16-byte aligned inner coordinates
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], BOX * nat + B_BYTES * (SPLIT ? 2 : 1));
        for (int bi = 0; bi < nat; ++bi) {
          const int nb = bi / hgroups, hg = bi - nb * hgroups;
          tma_load_4d(stg(stage) + bi * BOX, &tm_in, &full[stage], x0a, p0 - a.oh + kr + hg * RB, cb * CB, img0 + nb);
        }
        const int wrow = tap * a.Cout + n0;
        ptx::tma_load_2d(b_hi(stage), &tm_w_hi, &full[stage], cb * CB, wrow);
        if constexpr (SPLIT) ptx::tma_load_2d(b_lo(stage), &tm_w_lo, &full[stage], cb * CB, wrow);
        if (++stage == ST) { stage = 0; phase ^= 1; }
        if (++cb == a.cblocks) { cb = 0; if (++ks == a.S) { ks = 0; ++kr; } }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
    {
      // A: MN-major tf32 => 128B_BASE32B layout: rows of 32 pixels (128 B) per
      // channel, 4-channel groups 512 B apart (SBO), atoms CB*128 B apart (LBO)
      constexpr uint32_t a_lbo = uint32_t(CB) * 128u, a_kgrp = 8u * 128u;
      // B: K-major rows of CB fp32 (CB=32 -> SW128, CB=8 -> SW32)
      constexpr uint32_t b_layout = CB == 32 ? 2u : 6u;
      constexpr uint32_t b_sbo = 8u * CB * 4u;
      constexpr uint32_t idesc = tc::make_idesc_tf32(BN) | (1u << 15);  // A MN-major, B K-major
      int stage = 0;
      uint32_t phase = 0;
      for (int kt = 0; kt < nk; ++kt) {
        ptx::mbar_wait(&conv[stage], phase);
        ptx::tc_fence_after();
        const uint32_t ah = ptx::smem_u32(a_hi(stage)), bh = ptx::smem_u32(b_hi(stage));
        const uint32_t al = ptx::smem_u32(a_lo(stage)), bl = ptx::smem_u32(b_lo(stage));
#pragma unroll
        for (int j = 0; j < CB / 8; ++j) {
          const uint64_t dA_hi = make_desc(ah + j * a_kgrp, a_lbo, 512u, 1u);
          const uint64_t dB_hi = make_desc(bh + j * 32u, 16u, b_sbo, b_layout);
          uint32_t acc = (kt > 0 || j > 0) ? 1u : 0u;
          if constexpr (SPLIT) {
            const uint64_t dA_lo = make_desc(al + j * a_kgrp, a_lbo, 512u, 1u);
            const uint64_t dB_lo = make_desc(bl + j * 32u, 16u, b_sbo, b_layout);
            ptx::mma_tf32_elect(tmem, dA_lo, dB_hi, idesc, acc);
            ptx::mma_tf32_elect(tmem, dA_hi, dB_lo, idesc, 1u);
            acc = 1u;
          }
          ptx::mma_tf32_elect(tmem, dA_hi, dB_hi, idesc, acc);
        }
        ptx::mma_commit_elect(&empty[stage]);
        if (++stage == ST) { stage = 0; phase ^= 1; }
      }
      ptx::mma_commit_elect(accum);
    }
    __syncwarp();
  } else {
    // ---------------- converters: shift + swizzle (+ 3xTF32 split) ----------------
    // Thread t handles 16-byte output granules (row, col4) with col4 = t & 7
    // fixed, rows (t >> 3) + 16*i; row = atom*CB + channel.  The staged source
    // of granule element e sits at row*(RB*SW) + (j/TW)*SW + j%TW + shift,
    // j = col4*4 + e, so everything but the row term is loop invariant.
    const int tid = threadIdx.x - 64;
    const int col4 = tid & 7, row0 = tid >> 3;
    constexpr int ROWS = 4 * CB;  // atom rows in the A tile
    int src_e[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = col4 * 4 + e;
      src_e[e] = (j / TW) * SW + (j % TW);
    }
    int stage = 0;
    uint32_t phase = 0;
    int cb = 0, ks = 0;
    for (int kt = 0; kt < nk; ++kt) {
      const int x0 = q0 - a.ow + ks;
      const int delta = x0 - ((x0 >> 2) << 2);
      ptx::mbar_wait(&full[stage], phase);
      const float* src = reinterpret_cast<const float*>(stg(stage)) + delta;
      const uint32_t hi = ptx::smem_u32(a_hi(stage)), lo = ptx::smem_u32(a_lo(stage));
#pragma unroll
      for (int i = 0; i < ROWS / 16; ++i) {
        const int row = row0 + 16 * i;
        const float* s = src + row * (RB * SW);
        float v0 = s[src_e[0]], v1 = s[src_e[1]], v2 = s[src_e[2]], v3 = s[src_e[3]];
        if (row >= nat * CB) v0 = v1 = v2 = v3 = 0.f;  // atoms past the tile (partial tiles)
        const uint32_t off = atom32_off(uint32_t(row), uint32_t(col4 * 4));
        const float h0 = ptx::tf32_major<SPLIT>(v0), h1 = ptx::tf32_major<SPLIT>(v1), h2 = ptx::tf32_major<SPLIT>(v2),
                    h3 = ptx::tf32_major<SPLIT>(v3);
        ptx::st_shared_v4(hi + off, h0, h1, h2, h3);
        if constexpr (SPLIT)
          ptx::st_shared_v4(lo + off, ptx::tf32_lo(v0, h0), ptx::tf32_lo(v1, h1), ptx::tf32_lo(v2, h2),
                            ptx::tf32_lo(v3, h3));
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&conv[stage]);
      if (++stage == ST) { stage = 0; phase ^= 1; }
      if (++cb == a.cblocks) { cb = 0; if (++ks == a.S) ks = 0; }
    }
    // ---------------- epilogue: TMEM lane m = atom*32 + hl*TW + w ----------------
    ptx::mbar_wait(accum, 0);
    ptx::tc_fence_after();
    const int q = warp & 3;
    const int m = q * 32 + lane;
    const int bi = m >> 5, within = m & 31;
    const int nimg = bi / hgroups, hrow = (bi - nimg * hgroups) * RB + within / TW, w = within % TW;
    const int pp = p0 + hrow, qq = q0 + w, img = img0 + nimg;
    const bool valid = bi < nat && img < a.N && pp < a.P && qq < a.Q;
    const int64_t PQ = int64_t(a.P) * a.Q;
    float* outp = a.out + (int64_t(img) * a.Cout) * PQ + int64_t(pp) * a.Q + qq;
#pragma unroll 1
    for (int cc = 0; cc < BN; cc += 16) {
      uint32_t r[16];
      ptx::tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(cc), r);
      ptx::tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int n = n0 + cc + j;
          if (n < a.Cout) {
            float v = __uint_as_float(r[j]);
            if (a.bias) v += a.bias[n];
            if (a.relu) v = v > 0.f ? v : 0.f;
            outp[int64_t(n) * PQ] = v;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// Repack W[co][ci][kr][ks] into the per-tap K-major GEMM operand, padded to kpad
// channels, optionally split into (hi, lo) TF32 halves:
//   forward   : dst[tap][co][ci]                      tap = kr*S + ks
//   backward  : dst[tap][ci][co] from W[co][ci][R-1-kr][S-1-ks]
__global__ void repack_weights_kernel(const float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo,
                                      int Co, int Ci, int R, int S, int rows_per_tap, int kpad, bool backward,
                                      bool split) {
  const int total = R * S * rows_per_tap * kpad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int k = i % kpad;
    const int row = (i / kpad) % rows_per_tap;
    const int tap = i / (kpad * rows_per_tap);
    const int kr = tap / S, ks = tap % S;
    float v = 0.f;
    if (!backward) {  // row = co, k = ci
      if (k < Ci && row < Co) v = w[((row * Ci + k) * R + kr) * S + ks];
    } else {          // row = ci, k = co, flipped tap
      if (k < Co && row < Ci) v = w[((k * Ci + row) * R + (R - 1 - kr)) * S + (S - 1 - ks)];
    }
    if (split) {
      const float h = ptx::tf32_hi(v);
      hi[i] = h;
      lo[i] = ptx::tf32_lo(v, h);
    } else {
      hi[i] = v;
    }
  }
}

}  // namespace tcconv
}  // namespace cdnn
