// conv_tap.cuh — "tap-shift" implicit-GEMM convolution on tcgen05 (stride 1,
// any dilation, one group per launch), fp32 NCHW in/out, tf32 / 3xTF32 math.
//
//   out[img][n][p][q] = sum_{r,s,c} Wt[r*S+s][n][c] * in_pad[img][c][p + r*dh][q + s*dw]
//
// Forward:       in = x,  out = y,  Wt[tap][co][ci],          in_pad offset (ph, pw)
// Backward-data: in = dy, out = dx,  Wt[tap][ci][co] flipped,  offset (dh(R-1)-ph, dw(S-1)-pw)
//
// Virtual pixel grid: every image is laid out as Hv x Wv rows (Hv = P + dh(R-1),
// Wv = Q + dw(S-1)), row v = img*Hv*Wv + hp*Wv + wp holding the padded input
// pixel (hp, wp).  Output pixel (p, q) is virtual row p*Wv + q, and the input
// pixel its tap (r, s) reads is that row plus the constant r*dh*Wv + s*dw.  So
// a tile stages the input rows [m0, m0 + 128 + halo) ONCE per 32-channel block
// — channels-last, K-major, 128B-swizzled, split into tf32 hi/lo — and every
// tap is the same smem tile with its UMMA descriptor start moved by whole
// 128-byte rows (the 128B swizzle is address based, so arbitrary row offsets
// are legal: profiles/dbg/umma_rowshift.cu).  The per-tap conversion work of
// an im2col / window-staging design (R*S times the input) disappears; rows
// whose (p, q) fall in the padding columns are computed and dropped by the
// epilogue.  Weights arrive per (block, tap) by TMA, pre-split K-major.
//
// Persistent CTAs (one per SM; two for the staging-bound small-channel convs)
// walk the tiles; every stage is pipelined
// against the others: A tiles double-buffered, weights in an mbarrier ring,
// two TMEM accumulators so the epilogue of tile i overlaps the MMAs of i+1.
// Warp roles (320 threads): warp 0 TMA producer of the weights, warp 1 TMEM
// owner + single-thread MMA issuer, warps 2-5 stage input tiles, warps 6-9
// epilogue (TMEM -> registers -> coalesced NCHW stores, + bias).
#pragma once

#include <cstdint>

#include "gemm_tc.cuh"
#include "operands.cuh"
#include "ptx.cuh"

namespace cdnn {
namespace tctap {

constexpr int kThreads = 320;
// Output-channel tiles 48..128 wide run a second MMA-issuing warp (warp 10): the two
// issuers take alternate weight-ring stages into two TMEM accumulators (summed by the
// epilogue), so each one's per-stage mbarrier wait and tcgen05.commit overlap the other
// one's MMAs.  (192-wide tiles need the TMEM for double buffering; 32-wide tiles run
// two CTAs per SM instead.)
template <int BN>
__host__ __device__ constexpr bool dual_issue() { return BN > 32 && BN <= 128; }
template <int BN>
__host__ __device__ constexpr int threads_for() { return dual_issue<BN>() ? 352 : 320; }
constexpr int kMaxStages = 16;

struct TapArgs {
  const float* in;
  const float* bias;  // fwd only, may be null
  float* out;
  int N, Cin, Hin, Win;  // direct-conv input (x or dy) of this group
  int Cout, P, Q;        // direct-conv output extents of this group
  int R, S, dh, dw, oh, ow;
  int Hv, Wv;            // virtual grid
  int Mv;                // N * Hv * Wv
  int rows;              // staged rows per tile (multiple of 8)
  int cblocks;           // ceil(Cin / 32)
  int wrows;             // rows per tap in the repacked weights
  int n0_base;           // first repacked-weight row of this group
  int tiles_m, tiles;    // m tiles, m tiles x n blocks
  int in_cstride;        // channel stride of `in` (Hin*Win)
  int64_t in_nstride;    // image stride of `in`
  int64_t out_nstride;   // image stride of `out`
  int nbuf, stages;      // A buffers (1|2), weight ring depth
  int tps;               // filter taps per weight-ring stage (one mbarrier wait + one commit per stage)
  int dual;              // two MMA issuers (dual_issue<BN>() and >= 2 ring stages per tile)
  int relu;              // fused in-place ReLU in the epilogue (forward)
  int fold;              // S folded into the channels (k = s*Cin + c, Cin*S <= 32): R taps of K = S*Cin
  const float* gate;     // backward-data: fused in-place ReLU backward, out = gate > 0 ? out : 0 (same layout)
  FastDiv div_hwv, div_wv;
  unsigned long long* trace;  // debug timeline (CDNN_TAP_TRACE), null in production
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slots per CTA: 0 start, 1 setup done, 2+3*i: tile i {A staged, MMAs issued, epilogue done}
constexpr int kTraceSlots = 32;
#define TAP_TRACE(slot) \
  do { if (a.trace && (slot) < kTraceSlots) a.trace[blockIdx.x * kTraceSlots + (slot)] = gtime(); } while (0)

__host__ __device__ constexpr uint32_t b_stage_bytes(int bn, bool split) { return uint32_t(bn) * 128u * (split ? 2u : 1u); }
__host__ __device__ constexpr uint32_t a_buf_bytes(int rows, bool split) { return uint32_t(rows) * 128u * (split ? 2u : 1u); }

inline int smem_bytes(int rows, int nbuf, int stages, int bn, bool split, int tps = 1) {
  return 1024 + nbuf * int(a_buf_bytes(rows, split)) + stages * tps * int(b_stage_bytes(bn, split)) +
         (2 * kMaxStages + 8 + 1) * 8 + 16;
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;              // LBO (unused for swizzled K-major) = 16 B
  d |= uint64_t(1024 >> 4) << 32;      // SBO = 8 rows x 128 B
  d |= uint64_t(1) << 46;              // descriptor version
  d |= uint64_t(2) << 61;              // SWIZZLE_128B
  return d;
}

// Stage 8 channels (two 16-byte granules) of one virtual row: hi (and lo) tf32.
template <bool SPLIT>
__device__ __forceinline__ void put_row8(uint32_t rbase, uint32_t lo_off, int row, int g8, const float (&x)[8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int g4 = g8 * 2 + h;
    const uint32_t off = rbase + (uint32_t((g4 ^ (row & 7)) & 7) << 4);
    const float h0 = ptx::tf32_major<SPLIT>(x[4 * h]), h1 = ptx::tf32_major<SPLIT>(x[4 * h + 1]);
    const float h2 = ptx::tf32_major<SPLIT>(x[4 * h + 2]), h3 = ptx::tf32_major<SPLIT>(x[4 * h + 3]);
    ptx::st_shared_v4(off, h0, h1, h2, h3);
    if constexpr (SPLIT)
      ptx::st_shared_v4(off + lo_off, ptx::tf32_lo(x[4 * h], h0), ptx::tf32_lo(x[4 * h + 1], h1),
                        ptx::tf32_lo(x[4 * h + 2], h2), ptx::tf32_lo(x[4 * h + 3], h3));
  }
}

template <int BN, bool SPLIT>
__global__ void __launch_bounds__(threads_for<BN>(), BN <= 32 ? 2 : 1)
    conv_tap_kernel(const __grid_constant__ CUtensorMap tm_w_hi, const __grid_constant__ CUtensorMap tm_w_lo,
                    const TapArgs a) {
  // 3xTF32 with BN <= 64: one MMA against [B_hi | B_lo] (N = 2*BN) gives A_hi*B_hi
  // and A_hi*B_lo in two column halves, a second adds A_lo*B_hi into the first;
  // the epilogue sums the halves.  2 MMAs per k-step instead of 3 and a third
  // less A traffic (the A operand's shared-memory reads bound N <= 64 tiles).
  constexpr bool CAT = SPLIT && BN <= 64;
  constexpr int ACC = CAT ? 2 * BN : BN;  // accumulator columns per buffer
  constexpr bool DUAL = dual_issue<BN>();
  const int NI = DUAL && a.dual ? 2 : 1;  // MMA issuers = accumulators per TMEM buffer
  constexpr uint32_t TMEM_COLS = tc::tmem_cols_for(2 * ACC * (DUAL ? 2 : 1));
  constexpr uint32_t B_STAGE = b_stage_bytes(BN, SPLIT);
  constexpr uint32_t B_HALF = uint32_t(BN) * 128u;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t A_BUF = a_buf_bytes(a.rows, SPLIT), A_HALF = uint32_t(a.rows) * 128u;
  uint8_t* abase = smem;
  uint8_t* bbase = smem + a.nbuf * A_BUF;
  const uint32_t B_RING = uint32_t(a.tps) * B_STAGE;  // one ring stage = tps taps' weights
  uint64_t* full = reinterpret_cast<uint64_t*>(bbase + a.stages * B_RING);
  uint64_t* empty = full + kMaxStages;
  uint64_t* a_full = empty + kMaxStages;
  uint64_t* a_empty = a_full + 2;
  uint64_t* t_full = a_empty + 2;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int taps = a.fold ? a.R : a.R * a.S;
  // Concurrent CTAs walk the taps from different starting points, so the 148
  // weight streams hit different L2 lines instead of the same ones at once.
  const int rot = int(blockIdx.x % uint32_t(taps));

  if (threadIdx.x == 0) {
    TAP_TRACE(0);
    for (int s = 0; s < a.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&a_full[b], 4);
      ptx::mbar_init(&a_empty[b], NI);
      ptx::mbar_init(&t_full[b], NI);
      ptx::mbar_init(&t_empty[b], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TAP_TRACE(1);

  if (warp == 0) {
    // ---------------- weights: TMA per (tile, channel block, tap) ----------------
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tm_w_hi);
      if constexpr (SPLIT) ptx::tma_prefetch_desc(&tm_w_lo);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        const int n0 = a.n0_base + (t / a.tiles_m) * BN;
        for (int cb = 0; cb < a.cblocks; ++cb)
          for (int it = 0; it < taps; it += a.tps) {
            const int cnt = min(a.tps, taps - it);
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full[stage], uint32_t(cnt) * B_STAGE);
            for (int j = 0; j < cnt; ++j) {
              const int tap = it + j + rot < taps ? it + j + rot : it + j + rot - taps;
              uint8_t* b = bbase + stage * B_RING + j * B_STAGE;
              ptx::tma_load_2d(b, &tm_w_hi, &full[stage], cb * 32, tap * a.wrows + n0);
              if constexpr (SPLIT) ptx::tma_load_2d(b + B_HALF, &tm_w_lo, &full[stage], cb * 32, tap * a.wrows + n0);
            }
            if (++stage == a.stages) { stage = 0; phase ^= 1; }
          }
      }
    }
  } else if (warp == 1 || (DUAL && warp == 10)) {
    // ---------------- MMA issuer(s) (whole warp, one elected lane issues) ----------------
    // Issuer pi takes the global ring stages g with g % NI == pi into accumulator pi.
    const int pi = warp == 1 ? 0 : 1;
    if (pi < NI) {
      constexpr uint32_t idesc = tc::make_idesc_tf32(BN);  // A, B K-major
      constexpr uint32_t idesc_cat = tc::make_idesc_tf32(2 * BN);
      // Everything the loop needs is derived from kernel parameters and loop
      // counters (uniform registers); the tap's row shift advances by adds.
      const uint32_t s_step = uint32_t(a.dw) * 8u;                     // one filter column, 16 B units
      const uint32_t r_step = uint32_t(a.dh * a.Wv) * 8u;              // one filter row
      const int S_eff = a.fold ? 1 : a.S;
      const int r_rot = rot / S_eff, s_rot = rot - r_rot * S_eff;
      const uint32_t shift_rot = uint32_t(r_rot) * r_step + uint32_t(s_rot) * s_step;
      const uint32_t a0 = ptx::smem_u32(abase), b0 = ptx::smem_u32(bbase);
      int stage = 0;
      uint32_t phase = 0;
      int gsel = 0;  // global stage counter modulo NI
      int aseq = 0, ts = 0;
      for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++ts) {
        const int acc_buf = ts & 1;
        if (ts >= 2) ptx::mbar_wait(&t_empty[acc_buf], uint32_t((ts >> 1) - 1) & 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t((acc_buf * NI + pi) * ACC);
        uint32_t acc0 = 0u;  // first MMA of the tile overwrites the accumulator
        for (int cb = 0; cb < a.cblocks; ++cb, ++aseq) {
          const int buf = aseq % a.nbuf;
          ptx::mbar_wait(&a_full[buf], uint32_t(aseq / a.nbuf) & 1u);
          ptx::tc_fence_after();
          const int nk8 = ((a.fold ? a.S * a.Cin : min(32, a.Cin - cb * 32)) + 7) >> 3;
          // descriptors are built once; per MMA only the 16-byte-unit start
          // address in the low word moves (smem < 256 KB: no carry out of 14 bits)
          const uint64_t dA = desc_sw128(a0 + uint32_t(buf) * A_BUF);
          const uint64_t dAl = dA + (A_HALF >> 4);
          uint32_t shift = shift_rot;
          int r = r_rot, s = s_rot;
          bool used = false;
          for (int it = 0; it < taps; it += a.tps) {
            const int cnt = min(a.tps, taps - it);
            const bool mine = gsel == pi;
            if (mine) {
              ptx::mbar_wait(&full[stage], phase);
              ptx::tc_fence_after();
            }
            for (int j = 0; j < cnt; ++j) {
              if (mine) {
                const uint64_t dB = desc_sw128(b0 + uint32_t(stage) * B_RING + uint32_t(j) * B_STAGE);
                const uint64_t dBl = dB + (B_HALF >> 4);
                const uint64_t ah = dA + shift, al = dAl + shift;
                auto k8 = [&](int jj, uint32_t acc) {
                  const uint64_t kj = uint64_t(jj) * 2u;  // +32 B per k8 step
                  if constexpr (CAT) {
                    // [B_hi | B_lo] are contiguous BN-row blocks: one N = 2*BN operand
                    ptx::mma_tf32_elect(d_tmem, ah + kj, dB + kj, idesc_cat, acc);
                    ptx::mma_tf32_elect(d_tmem, al + kj, dB + kj, idesc, 1u);
                  } else {
                    if constexpr (SPLIT) {
                      ptx::mma_tf32_elect(d_tmem, al + kj, dB + kj, idesc, acc);
                      ptx::mma_tf32_elect(d_tmem, ah + kj, dBl + kj, idesc, 1u);
                      acc = 1u;
                    }
                    ptx::mma_tf32_elect(d_tmem, ah + kj, dB + kj, idesc, acc);
                  }
                };
                if (nk8 == 4) {
                  k8(0, acc0);
                  k8(1, 1u);
                  k8(2, 1u);
                  k8(3, 1u);
                } else {
                  k8(0, acc0);
                  for (int jj = 1; jj < nk8; ++jj) k8(jj, 1u);
                }
                acc0 = 1u;
              }
              // next tap (rotated order wraps to tap 0)
              if (++s == S_eff) {
                s = 0;
                if (++r == a.R) { r = 0; shift = 0; } else shift += r_step - uint32_t(S_eff - 1) * s_step;
              } else {
                shift += s_step;
              }
            }
            if (mine) {
              ptx::mma_commit_elect(&empty[stage]);
              used = true;
            }
            if (++stage == a.stages) { stage = 0; phase ^= 1; }
            if (++gsel == NI) gsel = 0;
          }
          if (used) ptx::mma_commit_elect(&a_empty[buf]);
          else if (lane == 0) ptx::mbar_arrive(&a_empty[buf]);  // this issuer read nothing of it
          __syncwarp();
        }
        ptx::mma_commit_elect(&t_full[acc_buf]);
        if (lane == 0 && pi == 0) TAP_TRACE(3 + 3 * ts);
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---------------- input tiles: channels-last, swizzled, hi/lo ----------------
    const int tid = threadIdx.x - 64;
    const int HWv = a.Hv * a.Wv;
    int aseq = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
      const int m0 = (t % a.tiles_m) * 128;
      for (int cb = 0; cb < a.cblocks; ++cb, ++aseq) {
        const int buf = aseq % a.nbuf;
        if (aseq >= a.nbuf) ptx::mbar_wait(&a_empty[buf], uint32_t(aseq / a.nbuf - 1) & 1u);
        const int c0 = cb * 32;
        const int kc = min(32, a.Cin - c0);
        const int g8n = (kc + 7) >> 3;  // 8-channel groups the MMAs read
        const uint32_t hi = ptx::smem_u32(abase + buf * A_BUF);
        if (a.fold) {
          // folded row: element k = s*Cin + c holds X_v[v + s*dw][c]; one index
          // decomposition per row, then (s, c) and the pixel advance incrementally
          const int kf = a.S * a.Cin, g8f = (kf + 7) >> 3;
          for (int row = tid; row < a.rows; row += 128) {
            const uint32_t rbase = hi + uint32_t(row) * 128u;
            int v = m0 + row;
            int img = int(a.div_hwv.div(uint32_t(v)));
            const int rem0 = v - img * HWv;
            int hp = int(a.div_wv.div(uint32_t(rem0)));
            int wp = rem0 - hp * a.Wv;
            auto tap_src = [&](bool& ok) {
              const int h = hp - a.oh, w = wp - a.ow;
              ok = v < a.Mv && h >= 0 && h < a.Hin && w >= 0 && w < a.Win;
              return a.in + int64_t(img) * a.in_nstride + h * a.Win + w;
            };
            bool ok;
            const float* src = tap_src(ok);
            int c = 0;
            float x[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              x[k] = (k < kf && ok) ? __ldg(src + int64_t(c) * a.in_cstride) : 0.f;
              if (++c == a.Cin) {
                c = 0;
                v += a.dw;
                wp += a.dw;
                while (wp >= a.Wv) {
                  wp -= a.Wv;
                  if (++hp == a.Hv) { hp = 0; ++img; }
                }
                src = tap_src(ok);
              }
            }
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8)
              if (g8 < g8f) {
                float xx[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) xx[e] = x[g8 * 8 + e];
                put_row8<SPLIT>(rbase, A_HALF, row, g8, xx);
              }
          }
        } else {
          // two rows per thread per round with every load (up to 64, partial blocks
          // predicated) issued before any conversion: one memory round trip per two
          // rows, instead of one per row (per 8 channels for a partial block) -- the
          // staging of tall tiles (AlexNet conv1's 57-wide grid: 244 rows per 128
          // pixels) otherwise outlasts the MMAs it feeds
          auto row_src = [&](int row, bool& inb) {
            const int v = m0 + row;
            inb = false;
            const float* src = a.in;
            if (row < a.rows && v < a.Mv) {
              const int img = int(a.div_hwv.div(uint32_t(v)));
              const int rem = v - img * HWv;
              const int hp = int(a.div_wv.div(uint32_t(rem)));
              const int h = hp - a.oh, w = rem - hp * a.Wv - a.ow;
              inb = h >= 0 && h < a.Hin && w >= 0 && w < a.Win;
              src = a.in + int64_t(img) * a.in_nstride + int64_t(c0) * a.in_cstride + h * a.Win + w;
            }
            return src;
          };
          auto load32 = [&](const float* src, bool inb, float (&x)[4][8]) {
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8)
#pragma unroll
              for (int e = 0; e < 8; ++e)
                x[g8][e] = (inb && g8 * 8 + e < kc) ? __ldg(src + int64_t(g8 * 8 + e) * a.in_cstride) : 0.f;
          };
          auto put32 = [&](int row, const float (&x)[4][8]) {
            const uint32_t rbase = hi + uint32_t(row) * 128u;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8)
              if (g8 < g8n) put_row8<SPLIT>(rbase, A_HALF, row, g8, x[g8]);
          };
          // (one row per round for BN <= 32: two CTAs share the SM's registers)
          constexpr int RPT = BN > 32 ? 2 : 1;
          for (int row = tid; row < a.rows; row += 128 * RPT) {
            bool ia, ib = false;
            const float* sa = row_src(row, ia);
            float xa[4][8], xb[4][8];
            load32(sa, ia, xa);
            if constexpr (RPT == 2) {
              const float* sb = row_src(row + 128, ib);
              load32(sb, ib, xb);
            }
            put32(row, xa);
            if (RPT == 2 && row + 128 < a.rows) put32(row + 128, xb);
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&a_full[buf]);
        if (tid == 0 && cb == a.cblocks - 1) TAP_TRACE(2 + 3 * (aseq / a.cblocks));
      }
    }
  } else {
    // ---------------- epilogue: TMEM lane m <-> virtual row m0 + m ----------------
    const int q4 = warp & 3;  // TMEM lane quadrant this warp may access
    const int HWv = a.Hv * a.Wv;
    const int64_t PQ = int64_t(a.P) * a.Q;
    int ts = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++ts) {
      const int acc_buf = ts & 1;
      const int m0 = (t % a.tiles_m) * 128;
      const int nc0 = (t / a.tiles_m) * BN;  // output channel of TMEM column 0 (within the group)
      const int v = m0 + q4 * 32 + lane;
      const int img = int(a.div_hwv.div(uint32_t(v)));
      const int rem = v - img * HWv;
      const int p = int(a.div_wv.div(uint32_t(rem)));
      const int q = rem - p * a.Wv;
      const bool valid = v < a.Mv && p < a.P && q < a.Q;
      float* outp = a.out + int64_t(img) * a.out_nstride + int64_t(p) * a.Q + q;
      const float* gatep = a.gate ? a.gate + (outp - a.out) : nullptr;  // dereferenced only for valid rows
      // One output chunk: 16 accumulator columns -> (+ bias, ReLU, gate) -> NCHW stores.
      auto store_chunk = [&](int cc, const float (&gv)[16]) {
        uint32_t r[16];
        const uint32_t lane_base = tmem + (uint32_t(q4 * 32) << 16) + uint32_t(acc_buf * NI * ACC + cc);
        ptx::tmem_ld16(lane_base, r);
        if constexpr (CAT) {
          uint32_t r2[16];
          ptx::tmem_ld16(lane_base + BN, r2);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
        }
        if (DUAL && NI == 2) {  // second issuer's accumulator (and its [hi | lo] halves)
          uint32_t r3[16];
          ptx::tmem_ld16(lane_base + ACC, r3);
          if constexpr (CAT) {
            uint32_t r4[16];
            ptx::tmem_ld16(lane_base + ACC + BN, r4);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) r3[j] = __float_as_uint(__uint_as_float(r3[j]) + __uint_as_float(r4[j]));
          }
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r3[j]));
        }
        ptx::tmem_ld_wait();
        if (valid) {
          // bias reads for the 16 columns issued before the first store (the stores
          // may alias them as far as the compiler knows)
          float bv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = nc0 + cc + j;
            bv[j] = (a.bias && n < a.Cout) ? __ldg(a.bias + n) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = nc0 + cc + j;
            if (n < a.Cout) {
              float o = __uint_as_float(r[j]) + bv[j];
              if (a.relu) o = o > 0.f ? o : 0.f;
              if (!(gv[j] > 0.f)) o = 0.f;
              outp[int64_t(n) * PQ] = o;
            }
          }
        }
      };
      // (warp-uniform branch: tcgen05.ld is warp-collective)
      if (a.gate == nullptr) {
        ptx::mbar_wait(&t_full[acc_buf], uint32_t(ts >> 1) & 1u);
        ptx::tc_fence_after();
        float ones[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) ones[j] = 1.f;
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 16) store_chunk(cc, ones);
      } else {
        // fused ReLU gate (backward-data): the reads do not depend on the accumulator,
        // so chunk 0's are issued before waiting for it and chunk i+1's before chunk i
        // is stored -- the gate adds no memory latency per chunk to the epilogue.
        float gnext[16];
        auto load_gate = [&](int cc, float (&g)[16]) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = nc0 + cc + j;
            g[j] = (valid && n < a.Cout) ? __ldg(gatep + int64_t(n) * PQ) : 1.f;
          }
        };
        load_gate(0, gnext);
        ptx::mbar_wait(&t_full[acc_buf], uint32_t(ts >> 1) & 1u);
        ptx::tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < BN; cc += 16) {
          float gv[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) gv[j] = gnext[j];
          if (cc + 16 < BN) load_gate(cc + 16, gnext);
          store_chunk(cc, gv);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&t_empty[acc_buf]);
      if (warp == 6 && lane == 0) TAP_TRACE(4 + 3 * ts);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace tctap
}  // namespace cdnn
