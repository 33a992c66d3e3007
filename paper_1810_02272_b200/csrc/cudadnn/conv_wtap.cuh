// conv_wtap.cuh — tap-shift backward-filter (weight gradient) on tcgen05 for
// stride-1 convolutions, fp32 NCHW, tf32 / 3xTF32 math.
//
//   dW[co][c][r][s] = sum_v dY_v[v][co] * X_v[v + r*dh*Wv + s*dw][c]
//
// on the virtual pixel grid of conv_tap.cuh (v = img*Hv*Wv + p*Wv + q; dY_v is
// zero on the padding rows/columns, X_v is the zero-padded input).  The GEMM
// per kernel row r and group of four taps s0..s0+3 is
//
//   D[(j, c)][co] += sum_k X_v[k + r*dh*Wv + (s0+j)*dw][c] * dY_v[k][co]
//
// with the A operand MN-major (rows = virtual pixels, 128-byte rows of 32
// channels, 128B_BASE32B swizzle) and its four 32-row M atoms placed a
// constant number of rows apart (LBO): one MMA covers four taps of the same
// staged tile (overlapping atoms, profiles/dbg/umma_m64.cu mode 1).  The host
// packs the R x S taps into such groups along kernel rows (stride dw) and the
// leftover columns along kernel columns (stride dh*Wv): 7 groups for 5x5.
// B = dY^T is K-major.
// Each CTA accumulates a contiguous range of virtual pixels (split-K) for one
// 32-channel block, a set of kernel rows and a block of output channels, and
// writes its partial dW (and the bias partial from the dY it staged) to
// ws[split][co][m'] with m' = (r*S + s)*Cg + c (channel innermost, so a warp's
// 32 TMEM lanes store one coalesced 128-byte row; m' = Kc for the bias); the
// deterministic reduce_splits_kernel adds the splits and permutes m' into the
// Caffe filter layout [co][c][r][s] while accumulating into dw / db.
//
// Warps (320 threads): warp 1 TMEM owner + MMA issuer, warps 2-9 stage the
// pixel chunks (double-buffered; eight warps for enough loads in flight),
// warps 2-5 also run the epilogue (one TMEM lane quadrant each), warp 0 idles.
#pragma once

#include <cstdint>

#include "gemm_tc.cuh"
#include "operands.cuh"
#include "ptx.cuh"

namespace cdnn {
namespace tcwtap {

constexpr int kThreads = 320;  // warp 1 MMA, warps 2-9 stage (2-5 also run the epilogue)
constexpr int kStagers = 256;
constexpr int kMaxGroups = 32;
constexpr int kMaxStages = 4;  // pipeline stages (chunks of KC virtual pixels) in shared memory

// Four taps whose X rows sit a constant number of virtual rows apart (along a
// kernel row: dw; along a kernel column: dh*Wv) form one MMA's M atoms.
struct TapGroup {
  int start;    // virtual-row offset of atom 0 (r*dh*Wv + s*dw)
  int stride;   // rows between atoms
  int tap[4];   // r*S + s per atom, -1 = unused atom
};

struct WtapArgs {
  const float* x;   // bottom data, offset to the group's first channel
  const float* dy;  // top diff, offset to the group's first channel
  float* ws;        // partials [split][Cog][Kc + 1]
  int N, Cg, H, W, Cog, P, Q, R, S, dh, dw, ph, pw;
  int Hv, Wv, Mv;
  int64_t x_nstride, dy_nstride;  // image strides (full tensors)
  int Kc;                         // Cg * R * S
  int cblocks, ggroups, coblocks;  // channel blocks, tap-group sets, co blocks
  int ngroups;
  TapGroup groups[kMaxGroups];
  int gbegin[kMaxGroups + 1];      // tap-group set i = groups[gbegin[i], gbegin[i+1])
  int rows_lo[kMaxGroups];         // per set: first staged row offset
  int splits, chunks_per_split, nchunks;
  int rowsA;                      // staged X rows per chunk (multiple of 8)
  int stages;                     // pipeline depth (2..kMaxStages)
  int want_bias;
  FastDiv div_hwv, div_wv;
};

__host__ __device__ constexpr uint32_t a_bytes(int rowsA, bool split) { return uint32_t(rowsA) * 128u * (split ? 2u : 1u); }
__host__ __device__ constexpr uint32_t b_bytes(int bn, bool split, int kc) {
  return uint32_t(bn) * uint32_t(kc) * 4u * (split ? 2u : 1u);
}
inline int smem_bytes(int rowsA, int bn, bool split, int kc, int stages) {
  return 1024 + stages * int(a_bytes(rowsA, split) + b_bytes(bn, split, kc)) + 2 * bn * 4 + (2 * kMaxStages + 2) * 8 +
         16;
}

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7) << 61;
  return d;
}

// KC: virtual pixels per pipeline chunk (64, or 32 with up to four stages when one CTA
// owns the SM: smaller stages, a deeper pipeline)
// CL: CTAs per thread-block cluster along the 32-channel blocks.  They share the
// chunk sequence and the output-channel block, so their B operand (the dY chunk) is
// identical: each CTA stages 1/CL of its output channels and writes them into every
// CTA's buffer (distributed shared memory), arriving on every CTA's `full` barrier;
// each MMA warp's commit arrives on every CTA's `empty` barrier (multicast), so a
// buffer is refilled only when all CL tensor cores have consumed it.  The dY loads,
// conversions and index math per CTA drop by CL.
template <int BN, bool SPLIT, int KC, int CL = 1>
__global__ void __launch_bounds__(kThreads, BN >= 96 ? 1 : 2) conv_wtap_kernel(const WtapArgs a) {
  constexpr int TM = 128;
  const int item = blockIdx.y;
  const int cb = item % a.cblocks;
  const int gg = (item / a.cblocks) % a.ggroups;
  const int cob = item / (a.cblocks * a.ggroups);
  const int g0 = a.gbegin[gg], ngroups = a.gbegin[gg + 1] - g0;
  const int rlo = a.rows_lo[gg];
  const int n0 = cob * BN;
  const int z = blockIdx.x;
  const int ch0 = z * a.chunks_per_split, ch1 = min(a.nchunks, ch0 + a.chunks_per_split);
  // bias partials: the first cluster of channel blocks, each CTA for its output-channel share
  const bool do_bias = a.want_bias && cb < CL && gg == 0;
  const uint32_t crank = CL > 1 ? ptx::cluster_ctarank() : 0u;
  constexpr int BNS = BN / CL;  // output channels this CTA stages (and whose bias it sums)

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t A_B = a_bytes(a.rowsA, SPLIT), A_H = uint32_t(a.rowsA) * 128u;
  constexpr uint32_t B_B = b_bytes(BN, SPLIT, KC);
  const uint32_t STAGE = A_B + B_B;  // multiple of 1024 (rowsA % 8 == 0, BN*KC*4 % 1024 == 0)
  const int NS = a.stages;
  float* bias_part = reinterpret_cast<float*>(smem + NS * STAGE);  // [pixel half][BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(bias_part + 2 * BN);
  uint64_t* empty = full + kMaxStages;
  uint64_t* accum = empty + kMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  // 3xTF32 with BN <= 64: [dY_hi | dY_lo] concatenated along N (one MMA gives
  // X_hi*dY_hi and X_hi*dY_lo in two column halves; X_lo*dY_hi adds into the
  // first), 2 MMAs per k-step instead of 3; the epilogue sums the halves.
  constexpr bool CAT = SPLIT && BN <= 64;
  constexpr int ACC = CAT ? 2 * BN : BN;
  // B layout per 32-pixel block: [hi rows BN | lo rows BN] (lo only when SPLIT)
  constexpr uint32_t B_KB = uint32_t(SPLIT ? 2 : 1) * BN * 128u;
  uint32_t tmem_cols = 32;
  while (tmem_cols < uint32_t(ngroups * ACC)) tmem_cols <<= 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) {
      ptx::mbar_init(&full[b], (kStagers / 32) * CL);
      ptx::mbar_init(&empty[b], CL);
    }
    ptx::mbar_init(accum, 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 2 * BN; i += kThreads) bias_part[i] = 0.f;
  if (warp == 1) ptx::tmem_alloc(tmem_slot, tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) ptx::cluster_sync_all();  // every CTA's barriers exist before remote arrivals
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int HWv = a.Hv * a.Wv;

  if (warp == 1) {
    if (ch1 > ch0) {  // whole warp runs the loop, one elected lane issues
      // A MN-major (bit 15), B K-major; M = 128 = four 32-channel tap atoms, N = BN output channels
      constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (uint32_t(BN >> 3) << 17) |
                                 (uint32_t(TM >> 4) << 24);
      constexpr uint32_t idesc_cat = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                                     (uint32_t((2 * BN) >> 3) << 17) | (uint32_t(TM >> 4) << 24);
      for (int ch = ch0, b = 0, ph = 0; ch < ch1; ++ch) {
        if constexpr (CL > 1) ptx::mbar_wait_cluster(&full[b], uint32_t(ph));
        else ptx::mbar_wait(&full[b], uint32_t(ph));
        ptx::tc_fence_after();
        const uint32_t abase = ptx::smem_u32(smem + b * STAGE), bbase = abase + A_B;
        for (int k8 = 0; k8 < KC / 8; ++k8) {
          const uint64_t dB = desc(bbase + uint32_t(k8 >> 2) * B_KB + uint32_t(k8 & 3) * 32u, 16, 1024, 2);
          const uint64_t dBl = dB + ((uint32_t(BN) * 128u) >> 4);
          for (int g = 0; g < ngroups; ++g) {
            const TapGroup& tg = a.groups[g0 + g];
            const uint32_t row = uint32_t(tg.start - rlo + k8 * 8);
            const uint64_t dA = desc(abase + row * 128u, uint32_t(tg.stride) * 128u, 512, 1);
            const uint32_t d_tmem = tmem + uint32_t(g * ACC);
            uint32_t acc = (ch > ch0 || k8 > 0) ? 1u : 0u;
            if constexpr (CAT) {
              ptx::mma_tf32_elect(d_tmem, dA, dB, idesc_cat, acc);
              ptx::mma_tf32_elect(d_tmem, dA + (A_H >> 4), dB, idesc, 1u);
            } else {
              if constexpr (SPLIT) {
                ptx::mma_tf32_elect(d_tmem, dA + (A_H >> 4), dB, idesc, acc);
                ptx::mma_tf32_elect(d_tmem, dA, dBl, idesc, 1u);
                acc = 1u;
              }
              ptx::mma_tf32_elect(d_tmem, dA, dB, idesc, acc);
            }
          }
        }
        if constexpr (CL > 1) ptx::mma_commit_mc_elect(&empty[b], uint16_t((1u << CL) - 1u));
        else ptx::mma_commit_elect(&empty[b]);
        if (++b == NS) { b = 0; ph ^= 1; }
      }
      ptx::mma_commit_elect(accum);
    }
    __syncwarp();
  } else if (warp >= 2) {
    const int tid = threadIdx.x - 64;
    const int c0 = cb * 32, kc = min(32, a.Cg - c0);
    const int64_t HW = int64_t(a.H) * a.W, PQ = int64_t(a.P) * a.Q;
    // B = dY^T [co][v0 .. v0+KC): lane = one virtual pixel (its index decomposed once per
    // chunk), warp = one 32-pixel half and a quarter of the BN output channels, so each
    // element costs one load at base + co*PQ and two 4-byte stores; a warp's 32 lanes
    // fill one 128-byte K-major row (conflict free).  A: one pixel row per thread (rows
    // beyond kStagers, if any, take the sequential path below).
    static_assert(KC == 64 || KC == 32, "one or two 32-pixel halves per chunk");
    constexpr int KH = KC / 32;        // 32-pixel halves per chunk
    constexpr int CPW = BNS * KH / 8;  // output channels per warp (of this CTA's BN / CL share)
    static_assert(BNS * KH % 8 == 0, "cluster share of the output channels per warp");
    const int sw = tid >> 5, khalf = sw % KH, cw0 = int(crank) * BNS + (sw / KH) * CPW;
    float bsum[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) bsum[c] = 0.f;
    // A row `row` of chunk v0: source pointer and bounds
    auto a_src = [&](int v0, int row, bool& inb) {
      const int v = v0 + rlo + row;
      inb = false;
      const float* src = a.x;
      if (v < a.Mv) {
        const int img = int(a.div_hwv.div(uint32_t(v)));
        const int rem = v - img * HWv;
        const int hp = int(a.div_wv.div(uint32_t(rem)));
        const int h = hp - a.ph, w = rem - hp * a.Wv - a.pw;
        inb = h >= 0 && h < a.H && w >= 0 && w < a.W;
        src = a.x + int64_t(img) * a.x_nstride + int64_t(c0) * HW + int64_t(h) * a.W + w;
      }
      return src;
    };
    auto a_load = [&](const float* src, bool inb, float (&xv)[4][8]) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[u][e] = (inb && u * 8 + e < kc) ? __ldg(src + (u * 8 + e) * HW) : 0.f;
    };
    // A: X_v rows, MN-major 128B_BASE32B, tf32 hi (and lo)
    auto a_store = [&](uint32_t abase, int row, const float (&xv)[4][8]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t off = uint32_t(row) * 128u + (uint32_t((u ^ (row & 3)) & 3) << 5);
        float hv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) hv[e] = ptx::tf32_major<SPLIT>(xv[u][e]);
        ptx::st_shared_v4(abase + off, hv[0], hv[1], hv[2], hv[3]);
        ptx::st_shared_v4(abase + off + 16, hv[4], hv[5], hv[6], hv[7]);
        if constexpr (SPLIT) {
          ptx::st_shared_v4(abase + A_H + off, ptx::tf32_lo(xv[u][0], hv[0]), ptx::tf32_lo(xv[u][1], hv[1]),
                            ptx::tf32_lo(xv[u][2], hv[2]), ptx::tf32_lo(xv[u][3], hv[3]));
          ptx::st_shared_v4(abase + A_H + off + 16, ptx::tf32_lo(xv[u][4], hv[4]), ptx::tf32_lo(xv[u][5], hv[5]),
                            ptx::tf32_lo(xv[u][6], hv[6]), ptx::tf32_lo(xv[u][7], hv[7]));
        }
      }
    };
    auto b_load = [&](int v0, float (&yv)[CPW]) {
      const int v = v0 + khalf * 32 + lane;
      const int img = int(a.div_hwv.div(uint32_t(v)));
      const int rem = v - img * HWv;
      const int p = int(a.div_wv.div(uint32_t(rem)));
      const int q = rem - p * a.Wv;
      const bool ok = v < a.Mv && p < a.P && q < a.Q;
      const float* src = a.dy + (ok ? int64_t(img) * a.dy_nstride + int64_t(p) * a.Q + q : 0) + int64_t(n0 + cw0) * PQ;
#pragma unroll
      for (int c = 0; c < CPW; ++c) yv[c] = (ok && n0 + cw0 + c < a.Cog) ? __ldg(src + c * PQ) : 0.f;
    };
    auto b_store = [&](uint32_t bbase, const float (&yv)[CPW]) {
      const uint32_t lane_off = uint32_t(khalf) * B_KB + uint32_t(lane & 3) * 4u;
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int col = cw0 + c;
        const uint32_t off = lane_off + uint32_t(col) * 128u + (uint32_t(((lane >> 2) ^ (col & 7)) & 7) << 4);
        const float h = ptx::tf32_major<SPLIT>(yv[c]);
        const float l = SPLIT ? ptx::tf32_lo(yv[c], h) : 0.f;
        ptx::st_shared_f32(bbase + off, h);
        if constexpr (SPLIT) ptx::st_shared_f32(bbase + off + uint32_t(BN) * 128u, l);
        if constexpr (CL > 1) {  // the same slot of every other CTA of the cluster
#pragma unroll
          for (uint32_t r = 1; r < uint32_t(CL); ++r) {
            const uint32_t peer = (crank + r) % uint32_t(CL);
            const uint32_t rb = ptx::mapa(bbase + off, peer);
            ptx::st_cluster_f32(rb, h);
            if constexpr (SPLIT) ptx::st_cluster_f32(rb + uint32_t(BN) * 128u, l);
          }
        }
        if (do_bias) bsum[c] += yv[c];
      }
    };
    for (int ch = ch0, b = 0, ph = 0; ch < ch1; ++ch) {
      const int v0 = ch * KC;
      // Every global load of this thread's share of the chunk is issued BEFORE waiting
      // for the buffer: the loads fly while the MMAs of the two previous chunks run,
      // and the conversion starts once with all data present (one memory round trip
      // per chunk instead of one per row / item).
      float xv[4][8];
      bool inb = false;
      const float* asrc = tid < a.rowsA ? a_src(v0, tid, inb) : a.x;
      a_load(asrc, inb && tid < a.rowsA, xv);
      float yv[CPW];
      b_load(v0, yv);
      if (ch - ch0 >= NS) {
        if constexpr (CL > 1) ptx::mbar_wait_cluster(&empty[b], uint32_t(ph ^ 1));
        else ptx::mbar_wait(&empty[b], uint32_t(ph ^ 1));
      }
      const uint32_t abase = ptx::smem_u32(smem + b * STAGE), bbase = abase + A_B;
      if (tid < a.rowsA) a_store(abase, tid, xv);
      b_store(bbase, yv);
      for (int row = tid + kStagers; row < a.rowsA; row += kStagers) {  // tall tiles only
        float xr[4][8];
        bool in2 = false;
        const float* s2 = a_src(v0, row, in2);
        a_load(s2, in2, xr);
        a_store(abase, row, xr);
      }
      if constexpr (CL > 1) {
        ptx::fence_proxy_async_all();  // local and remote generic stores -> the tensor cores' reads
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&full[b]);
          const uint32_t fb = ptx::smem_u32(&full[b]);
#pragma unroll
          for (uint32_t r = 1; r < uint32_t(CL); ++r) ptx::mbar_arrive_cluster(ptx::mapa(fb, (crank + r) % uint32_t(CL)));
        }
      } else {
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&full[b]);
      }
      if (++b == NS) { b = 0; ph ^= 1; }
    }
    if (do_bias) {  // per output channel: fixed xor tree over the warp's 32 pixels, then the two halves
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        float t = bsum[c];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
        if (lane == 0) bias_part[khalf * BN + cw0 + c] = t;
      }
    }
    ptx::named_bar_sync(1, kStagers);  // stager warps only: bias partials complete
    // ---- epilogue (warps 2-5): TMEM lane (j*32 + c) of group g = tap (r, s0 + j), channel c
    if (warp >= 6) goto done;
    {
    const int q4 = warp & 3;  // lane quadrant = tap atom j
    float* wsz = a.ws + int64_t(z) * a.Cog * (a.Kc + 1);
    if (ch1 > ch0) {
      ptx::mbar_wait(accum, 0);
      ptx::tc_fence_after();
    }
    const int c = c0 + lane;
    for (int g = 0; g < ngroups; ++g) {
      const int tap = a.groups[g0 + g].tap[q4];
#pragma unroll 1
      for (int cc = 0; cc < BN; cc += 16) {
        uint32_t rv[16];
        if (ch1 > ch0) {
          ptx::tmem_ld16(tmem + (uint32_t(q4 * 32) << 16) + uint32_t(g * ACC + cc), rv);
          if constexpr (CAT) {
            uint32_t r2[16];
            ptx::tmem_ld16(tmem + (uint32_t(q4 * 32) << 16) + uint32_t(g * ACC + BN + cc), r2);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) rv[j] = __float_as_uint(__uint_as_float(rv[j]) + __uint_as_float(r2[j]));
          }
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) rv[j] = 0u;
        }
        if (tap >= 0 && c < a.Cg) {
          const int m = tap * a.Cg + c;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int co = n0 + cc + j;
            if (co < a.Cog) wsz[int64_t(co) * (a.Kc + 1) + m] = __uint_as_float(rv[j]);
          }
        }
      }
    }
    if (do_bias && warp == 2) {
      for (int col = int(crank) * BNS + lane; col < int(crank + 1) * BNS; col += 32)
        if (n0 + col < a.Cog) wsz[int64_t(n0 + col) * (a.Kc + 1) + a.Kc] = bias_part[col] + bias_part[BN + col];
    }
    }
  }
done:
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) ptx::cluster_sync_all();  // no CTA leaves while peers may write or arrive into it
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, tmem_cols);
  }
}

}  // namespace tcwtap
}  // namespace cdnn
