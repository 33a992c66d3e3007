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
  int TW, TH, NB, CB;       // tile geometry: TW*TH*NB <= 128 pixels, CB channels per stage
  int cblocks;              // ceil(Cin / CB)
  int tiles_q, tiles_p;     // tiles along q and p
  const float* bias;        // may be null (fwd only)
  float* out;
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

// swizzle layout code of an MN-major row of TW fp32 (TMA swizzle span = TW*4 bytes)
__host__ __device__ constexpr uint32_t layout_for_row_bytes(int bytes) {
  return bytes == 128 ? 2u : bytes == 64 ? 4u : 6u;  // SW128 / SW64 / SW32
}

// per stage: staging (aligned activation window, no swizzle), A hi/lo tiles, B hi/lo
__host__ __device__ constexpr uint32_t a_bytes() { return 128 * 32 * 4; }           // 128 px x 32 ch
__host__ __device__ constexpr uint32_t stg_bytes() { return 32 * 4 * (32 + 16) * 4; }  // 4 atoms x 32 ch x (32 + 4*rb)
template <int BN>
__host__ __device__ constexpr uint32_t b_bytes() { return BN * 32 * 4; }

template <int BN>
__host__ __device__ constexpr int stages() { return BN >= 128 ? 2 : 3; }

template <int BN, bool SPLIT>
__host__ __device__ constexpr uint32_t stage_bytes() {
  return stg_bytes() + (a_bytes() + b_bytes<BN>()) * (SPLIT ? 2 : 1);
}

template <int BN, bool SPLIT>
__host__ __device__ constexpr int smem_bytes() {
  return 1024 + stages<BN>() * int(stage_bytes<BN, SPLIT>()) + (3 * stages<BN>() + 1) * 8 + 16;
}

// ATOM_32B swizzle of the MN-major tf32 UMMA layout (128B_BASE32B): 32-byte
// units of a 128-byte row XOR'd with the row index mod 4.
__device__ __forceinline__ uint32_t atom32_off(uint32_t row, uint32_t col) {
  return row * 128u + ((((col >> 3) ^ row) & 3u) << 5) + ((col & 7u) << 2);
}

template <int BN, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tma_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_w_hi,
                    const __grid_constant__ CUtensorMap tm_w_lo, const ConvTmaArgs a) {
  constexpr int ST = stages<BN>();
  constexpr uint32_t A_BYTES = a_bytes(), B_BYTES = b_bytes<BN>(), STG = stg_bytes();
  constexpr uint32_t STAGE = stage_bytes<BN, SPLIT>();
  constexpr uint32_t TMEM_COLS = tc::tmem_cols_for(BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage: [A hi | B hi | A lo | B lo | staging]; every tile 1024-B aligned
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
  const int q0 = tq * a.TW, p0 = tp * a.TH, img0 = tn * a.NB;
  const int n0 = blockIdx.y * BN;
  const int nk = a.R * a.S * a.cblocks;
  const int rb = 32 / a.TW, hgroups = a.TH / rb;
  const int nat = min(4, a.NB * hgroups);          // 32-pixel atoms in this tile
  const int sw_w = a.TW + 4;                        // staged window width (shift 0..3)
  const uint32_t box_bytes = uint32_t(sw_w * rb * a.CB) * 4u;
  const uint32_t b_box_bytes = uint32_t(BN * a.CB) * 4u;

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
      for (int kt = 0; kt < nk; ++kt) {
        const int cb = kt % a.cblocks, tap = kt / a.cblocks;
        const int kr = tap / a.S, ks = tap - kr * a.S;
        const int x0 = q0 - a.ow + ks;
        const int x0a = (x0 >> 2) << 2;  // TMA needs 16-byte aligned inner coordinates
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], box_bytes * nat + b_box_bytes * (SPLIT ? 2 : 1));
        for (int bi = 0; bi < nat; ++bi) {
          const int nb = bi / hgroups, hg = bi - nb * hgroups;
          tma_load_4d(stg(stage) + bi * box_bytes, &tm_in, &full[stage], x0a, p0 - a.oh + kr + hg * rb, cb * a.CB,
                      img0 + nb);
        }
        const int wrow = tap * a.Cout + n0;
        ptx::tma_load_2d(b_hi(stage), &tm_w_hi, &full[stage], cb * a.CB, wrow);
        if constexpr (SPLIT) ptx::tma_load_2d(b_lo(stage), &tm_w_lo, &full[stage], cb * a.CB, wrow);
        if (++stage == ST) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      // A: MN-major tf32 => 128B_BASE32B layout: rows of 32 pixels (128 B) per
      // channel, 4-channel groups 512 B apart (SBO), atoms CB*128 B apart (LBO)
      const uint32_t a_lbo = uint32_t(a.CB) * 128u, a_kgrp = 8u * 128u;
      // B: K-major rows of CB fp32 (CB=32 -> SW128, CB=8 -> SW32)
      const uint32_t b_row = uint32_t(a.CB) * 4u;
      const uint32_t b_layout = b_row == 128 ? 2u : 6u;
      const uint32_t b_sbo = 8u * b_row;
      const uint32_t idesc = tc::make_idesc_tf32(BN) | (1u << 15);  // A MN-major, B K-major
      int stage = 0;
      uint32_t phase = 0;
      for (int kt = 0; kt < nk; ++kt) {
        ptx::mbar_wait(&conv[stage], phase);
        ptx::tc_fence_after();
        const uint32_t ah = ptx::smem_u32(a_hi(stage)), bh = ptx::smem_u32(b_hi(stage));
        const uint32_t al = ptx::smem_u32(a_lo(stage)), bl = ptx::smem_u32(b_lo(stage));
        for (int j = 0; j < a.CB / 8; ++j) {
          const uint64_t dA_hi = make_desc(ah + j * a_kgrp, a_lbo, 512u, 1u);
          const uint64_t dB_hi = make_desc(bh + j * 32u, 16u, b_sbo, b_layout);
          uint32_t acc = (kt > 0 || j > 0) ? 1u : 0u;
          if constexpr (SPLIT) {
            const uint64_t dA_lo = make_desc(al + j * a_kgrp, a_lbo, 512u, 1u);
            const uint64_t dB_lo = make_desc(bl + j * 32u, 16u, b_sbo, b_layout);
            ptx::mma_tf32(tmem, dA_lo, dB_hi, idesc, acc);
            ptx::mma_tf32(tmem, dA_hi, dB_lo, idesc, 1u);
            acc = 1u;
          }
          ptx::mma_tf32(tmem, dA_hi, dB_hi, idesc, acc);
        }
        ptx::mma_commit(&empty[stage]);
        if (++stage == ST) { stage = 0; phase ^= 1; }
      }
      ptx::mma_commit(accum);
    }
    __syncwarp();
  } else {
    // ---------------- converters: shift + swizzle (+ 3xTF32 split) ----------------
    const int tid = threadIdx.x - 64;
    const int granules = 32 * a.CB;  // 128 px x CB ch / 4
    int stage = 0;
    uint32_t phase = 0;
    for (int kt = 0; kt < nk; ++kt) {
      const int tap = kt / a.cblocks;
      const int ks = tap % a.S;
      const int x0 = q0 - a.ow + ks;
      const int delta = x0 - ((x0 >> 2) << 2);
      ptx::mbar_wait(&full[stage], phase);
      const float* src = reinterpret_cast<const float*>(stg(stage));
      const uint32_t hi = ptx::smem_u32(a_hi(stage)), lo = ptx::smem_u32(a_lo(stage));
      for (int gidx = tid; gidx < granules; gidx += 128) {
        // granule = 4 consecutive tile pixels j..j+3 of channel c in atom bi
        const int col4 = gidx & 7, rowi = gidx >> 3;  // rowi = bi*CB + c
        const int bi = rowi / a.CB, c = rowi - bi * a.CB;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = col4 * 4 + e;
          const int hl = j / a.TW, w = j - hl * a.TW;
          v[e] = bi < nat ? src[((bi * a.CB + c) * rb + hl) * sw_w + delta + w] : 0.f;
        }
        const uint32_t off = atom32_off(uint32_t(rowi), uint32_t(col4 * 4));
        const float h0 = ptx::to_tf32(v[0]), h1 = ptx::to_tf32(v[1]), h2 = ptx::to_tf32(v[2]), h3 = ptx::to_tf32(v[3]);
        ptx::st_shared_v4(hi + off, h0, h1, h2, h3);
        if constexpr (SPLIT)
          ptx::st_shared_v4(lo + off, ptx::to_tf32(v[0] - h0), ptx::to_tf32(v[1] - h1), ptx::to_tf32(v[2] - h2),
                            ptx::to_tf32(v[3] - h3));
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&conv[stage]);
      if (++stage == ST) { stage = 0; phase ^= 1; }
    }
    // ---------------- epilogue: TMEM lane m = atom*32 + hl*TW + w ----------------
    ptx::mbar_wait(accum, 0);
    ptx::tc_fence_after();
    const int q = warp & 3;
    const int m = q * 32 + lane;
    const int bi = m >> 5, within = m & 31;
    const int nimg = bi / hgroups, hrow = (bi - nimg * hgroups) * rb + within / a.TW, w = within % a.TW;
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

// Repack W[co][ci][kr][ks] into the per-tap K-major GEMM operand, padded to cip
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
      const float h = ptx::to_tf32(v);
      hi[i] = h;
      lo[i] = ptx::to_tf32(v - h);
    } else {
      hi[i] = v;
    }
  }
}

}  // namespace tcconv
}  // namespace cdnn
