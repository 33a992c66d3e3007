// ops_conv.cu — Caffe convolution (absent from the reference)
// as three implicit GEMMs on the tensor-core (float) / SIMT (double) engines,
// per group g (weights [Co][C/g][R][S], NCHW activations, no im2col buffer):
//
//   forward          m = out pixel (img,p,q)   n = co    k = (ci,kr,ks)
//   backward-data    m = in  pixel (img,h,w)   n = ci    k = (co,kr,ks)
//   backward-filter  m = tap (ci,kr,ks)        n = co    k = out pixel (split-K)
//
// m is always the output's contiguous index, so epilogue stores coalesce.
// Backward-filter accumulates into dw (param diffs accumulate, layers.hpp:84-86);
// its bias gradient is a deterministic per-channel reduction.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "conv_tap.cuh"
#include "conv_tma.cuh"
#include "conv_wtap.cuh"
#include "launch.cuh"

namespace cdnn {
namespace {

// Group-aware repack of W[Co][Cg][R][S] into the per-tap K-major operand, padded to
// kpad channels, (hi, lo) TF32 split:
//   forward : dst[tap][co][ci]      (ci within the group)
//   backward: dst[tap][ci][co]      (co within ci's group), taps flipped
//   fold    : the kernel row's S taps live in k = s*Cd + c (Cd = channels of the direct conv)
__global__ void repack_tap_kernel(const float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo, int Co,
                                  int C, int Cg, int Cog, int R, int S, int kpad, bool backward, bool split, bool fold) {
  const int rows = backward ? C : Co;
  const int taps = fold ? R : R * S;
  const int Cd = backward ? Cog : Cg;
  const int total = taps * rows * kpad;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    int k = i % kpad;
    const int row = (i / kpad) % rows;
    const int tap = i / (kpad * rows);
    int kr = fold ? tap : tap / S, ks = fold ? 0 : tap % S;
    bool ok = k < Cd;
    if (fold) {
      ks = k / Cd;
      k -= ks * Cd;
      ok = ks < S;
    }
    float v = 0.f;
    if (ok) {
      if (!backward) {
        v = w[((row * Cg + k) * R + kr) * S + ks];
      } else {
        const int grp = row / Cg;
        v = w[(((grp * Cog + k) * Cg + (row - grp * Cg)) * R + (R - 1 - kr)) * S + (S - 1 - ks)];
      }
    }
    const float h = split ? ptx::tf32_hi(v) : v;
    hi[i] = h;
    if (split) lo[i] = ptx::tf32_lo(v, h);
  }
}

template <int BN, bool SPLIT>
void launch_conv_tap(Ctx* c, cudaStream_t st, dim3 grid, int smem, const CUtensorMap& twh, const CUtensorMap& twl,
                     const tctap::TapArgs& a) {
  auto kern = tctap::conv_tap_kernel<BN, SPLIT>;
  static int attr_smem[16] = {};
  if (attr_smem[c->device & 15] < smem) {
    CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_smem[c->device & 15] = smem;
  }
  kern<<<grid, tctap::threads_for<BN>(), smem, st>>>(twh, twl, a);
  check_launch("conv_tap_kernel");
  count_launch(c);
}

// Virtual pixel grid of the tap-shift kernels.  Output (p, q) is row p*Wv + q; the input
// pixel tap (r, s) reads is that row + r*dh*Wv + s*dw, decoded back to (hv - oh, wv - ow)
// (zero outside the image).  The padded grid (Hv = P + dh(R-1), Wv = Q + dw(S-1)) never
// wraps; the compact one shares the pad columns / rows between neighbours: a read that
// wraps into the next row (or image) decodes to a column (row) left of (above) the
// image, i.e. a zero -- exactly what the true, out-of-image pixel holds -- as long as
//   Wv >= Win + ow   and   Hv >= Hin + oh + 1   (one extra row for the column wrap of the
// last row).  13x13 / pad 1 (AlexNet conv3-5): 15x15 = 225 -> 15x14 = 210 rows per
// image; 27x27 / pad 2 (conv2): 961 -> 870 -- 7-10% fewer MMAs and staged rows.
void virtual_grid(int Hin, int Win, int P, int Q, int oh, int ow, int R, int S, int dh, int dw, int& Hv, int& Wv) {
  Hv = P + dh * (R - 1);
  Wv = Q + dw * (S - 1);
  const int hc = Hin + oh + 1, wc = Win + ow;
  if (oh >= 0 && ow >= 0 && hc >= P && wc >= Q && hc <= Hv && wc <= Wv) {
    Hv = hc;
    Wv = wc;
  }
}

// Output-channel tile width: the candidate with the least padding (ceil(Cout/bn)*bn),
// ties to the wider tile; N = 48 / 96 tiles fit AlexNet's 48 (conv2 backward-data),
// 96 (conv1) and 192 (conv4 / conv5 groups) channels exactly, where 64 / 128 tiles
// padded 25% of the MMA work.  Narrower while the grid would not fill the SMs.
int pick_bn(int cout, int tiles_m, int groups, std::initializer_list<int> cands) {
  int best = 0;
  int64_t best_pad = 0;
  for (int bn : cands) {
    const int64_t pad = int64_t((cout + bn - 1) / bn) * bn;
    if (!best || pad < best_pad || (pad == best_pad && bn > best)) { best = bn; best_pad = pad; }
  }
  while (best > 32 && int64_t(tiles_m) * groups * ((cout + best - 1) / best) < kNumSMs) {
    int smaller = 0;
    for (int bn : cands)
      if (bn < best && bn > smaller) smaller = bn;
    if (!smaller) break;
    best = smaller;
  }
  return best;
}

// Tap-shift implicit GEMM (conv_tap.cuh): stride 1, any dilation, any group count.
// Returns false when the staged tile does not fit shared memory.
bool conv_tap(Ctx* c, const ConvDescSlot& dconst, bool backward_data, const float* in, const float* w,
              const float* bias, float* out, cdnn_handle stream, bool relu = false, const float* gate = nullptr) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  const ConvGeom& g = d.geom;
  if (g.sh != 1 || g.sw != 1) return false;
  // 2-7 input channels with wide filters (CIFAR conv1): the window-staging kernel
  // (conv_tma.cuh) measures faster (profiles/r01_conv_bench.txt); it takes them when eligible
  {
    const int cin = backward_data ? g.Cog : g.Cg, win = backward_data ? g.Q : g.W;
    if (g.group == 1 && g.dh == 1 && g.dw == 1 && cin > 1 && cin < 8 && cin * g.S > 8 && win % 4 == 0)
      return false;
  }
  const int G = g.group;
  const int Cin = backward_data ? g.Cog : g.Cg, Hin = backward_data ? g.P : g.H, Win = backward_data ? g.Q : g.W;
  const int Cout = backward_data ? g.Cg : g.Cog, P = backward_data ? g.H : g.P, Q = backward_data ? g.W : g.Q;
  const int CinT = backward_data ? g.Co : g.C, CoutT = backward_data ? g.C : g.Co;
  const int oh = backward_data ? g.dh * (g.R - 1) - g.ph : g.ph, ow = backward_data ? g.dw * (g.S - 1) - g.pw : g.pw;
  if (oh < 0 || ow < 0) return false;  // padding wider than the dilated kernel: not a plain shift
  tctap::TapArgs a{};
  a.N = g.N; a.Cin = Cin; a.Hin = Hin; a.Win = Win; a.Cout = Cout; a.P = P; a.Q = Q;
  a.R = g.R; a.S = g.S; a.dh = g.dh; a.dw = g.dw; a.oh = oh; a.ow = ow;
  a.relu = relu ? 1 : 0;
  virtual_grid(Hin, Win, P, Q, oh, ow, g.R, g.S, g.dh, g.dw, a.Hv, a.Wv);
  if (int64_t(g.N) * a.Hv * a.Wv >= (int64_t(1) << 31)) return false;
  a.Mv = g.N * a.Hv * a.Wv;
  a.fold = (Cin < 16 && Cin * g.S <= 32) ? 1 : 0;
  a.rows = (128 + g.dh * (g.R - 1) * a.Wv + (a.fold ? 0 : g.dw * (g.S - 1)) + 7) & ~7;
  a.cblocks = a.fold ? 1 : (Cin + 31) / 32;
  a.in_cstride = Hin * Win;
  a.in_nstride = int64_t(CinT) * Hin * Win;
  a.out_nstride = int64_t(CoutT) * P * Q;
  a.div_hwv = FastDiv(uint32_t(a.Hv * a.Wv));
  a.div_wv = FastDiv(uint32_t(a.Wv));
  const bool split = c->math_mode == CDNN_MATH_TF32X3;
  const int tiles = (a.Mv + 127) / 128;
  // 192-wide tiles for 192 / 384 output channels (AlexNet conv3-5): the N = 192 MMA
  // costs 96 cycles (full rate) where N = 96 costs 56, and the A tile is staged once
  // per 192 channels
  const int bn = pick_bn(Cout, tiles, G, {32, 48, 64, 96, 128, 192});
  // shared memory: A buffers (double-buffered over channel blocks when they fit) + B ring
  int budget = 227 * 1024;
  // 32-wide tiles (<= 32 output channels per block, the CIFAR / LeNet / ResNet stage-1
  // convolutions): size the CTA for two per SM.  The two CTAs' staging, MMA issue
  // and epilogues interleave on the SM's tensor core (CIFAR conv2 39.4 -> 35.3 us,
  // the column-folded conv1 53 -> 48.5 us); TMEM 2 x <= 256 columns.
  const bool staging_bound = a.cblocks == 1;
  int ctas_per_sm = 1;
  // (32-wide tiles only: their kernel is register-bounded for two CTAs per SM)
  if (staging_bound && bn == 32 && tctap::smem_bytes(a.rows, 1, 2, bn, split) <= 113 * 1024) {
    budget = 113 * 1024;
    ctas_per_sm = 2;
  }
  a.nbuf = 2;
  auto fits = [&](int nbuf, int stages, int tps) {
    return tctap::smem_bytes(a.rows, nbuf, stages, bn, split, tps) <= budget;
  };
  if (!fits(a.nbuf, 2, 1)) a.nbuf = 1;
  if (!fits(a.nbuf, 2, 1)) return false;
  // several taps per weight-ring stage: every stage costs the MMA issuer one mbarrier
  // wait and one tcgen05.commit, a few hundred cycles of issue that a small-N tap (N = 48:
  // 8 MMAs, ~400 tensor cycles) does not cover -- the largest tps <= 4 whose ring still
  // holds two stages and >= 4 taps (AlexNet conv2 backward-data 0.95 -> 0.74 ms, conv1
  // forward 0.49 -> 0.45; profiles/dbg/ab_tps.sh)
  const int taps_all = a.fold ? g.R : g.R * g.S;
  a.tps = 1;
  for (int t = std::min(4, taps_all); t > 1; --t) {
    int st = 0;
    while (st < tctap::kMaxStages && fits(a.nbuf, st + 1, t)) ++st;
    if (st >= 2 && st * t >= 4) {
      a.tps = t;
      break;
    }
  }
  a.stages = 2;
  while (a.stages < tctap::kMaxStages && fits(a.nbuf, a.stages + 1, a.tps)) ++a.stages;
  int smem = tctap::smem_bytes(a.rows, a.nbuf, a.stages, bn, split, a.tps);
  // two MMA issuers on alternate ring stages when every tile has at least two stages
  // (AlexNet conv2 backward-data 0.79 -> 0.68 ms, conv1 forward 0.48 -> 0.43, conv3
  // backward-data 0.39 -> 0.36; profiles/dbg/ab_dual.sh, iter_dual2.sh)
  const bool dual_bn = bn > 32 && bn <= 128;
  a.dual = dual_bn && a.cblocks * ((taps_all + a.tps - 1) / a.tps) >= 2 ? 1 : 0;
  // an even ring: issuer g % 2 always owns the same slots (slot % 2) and so waits on every
  // phase of them -- with an odd ring an issuer would skip phases, and a parity wait can
  // then return on a phase two fills old
  if (a.dual && (a.stages & 1)) {
    --a.stages;
    smem = tctap::smem_bytes(a.rows, a.nbuf, a.stages, bn, split, a.tps);
  }
  // weights: repacked per call (they change every step), pre-split
  const int kpad = a.cblocks * 32;
  a.wrows = CoutT;
  const int RS = a.fold ? g.R : g.R * g.S;  // taps of the repacked operand
  const size_t elems = size_t(RS) * CoutT * kpad;
  const int slot = backward_data ? 2 : 0;
  if (!d.repack[slot] || d.repack[slot]->bytes < elems * 4) {
    d.repack[slot] = device_alloc_shared(elems * 4, c->device);
    d.repack[slot + 1] = device_alloc_shared(elems * 4, c->device);
  }
  float* whi = static_cast<float*>(d.repack[slot]->ptr);
  float* wlo = static_cast<float*>(d.repack[slot + 1]->ptr);
  cudaStream_t st = stream_of(c, stream);
  repack_tap_kernel<<<grid_for(int64_t(elems), 256), 256, 0, st>>>(w, whi, wlo, g.Co, g.C, g.Cg, g.Cog, g.R, g.S,
                                                                   kpad, backward_data, split, a.fold != 0);
  check_launch("repack_tap");
  count_launch(c);
  const uint64_t wdims[2] = {uint64_t(kpad), uint64_t(RS) * CoutT};
  const uint64_t wstr[1] = {uint64_t(kpad)};
  const uint32_t wbox[2] = {32u, uint32_t(bn)};
  const CUtensorMap* twh = tmap_generic(c, whi, 2, wdims, wstr, wbox, 128);
  const CUtensorMap* twl = tmap_generic(c, wlo, 2, wdims, wstr, wbox, 128);
  a.tiles_m = tiles;
  a.tiles = tiles * ((Cout + bn - 1) / bn);
  dim3 grid(std::min(a.tiles, ctas_per_sm * kNumSMs));  // persistent: CTAs walk the tiles
  for (int grp = 0; grp < G; ++grp) {
    tctap::TapArgs ag = a;
    ag.in = in + int64_t(grp) * Cin * Hin * Win;
    ag.out = out + int64_t(grp) * Cout * P * Q;
    ag.gate = gate ? gate + int64_t(grp) * Cout * P * Q : nullptr;
    ag.bias = bias ? bias + grp * Cout : nullptr;
    ag.n0_base = grp * Cout;
    auto go = [&](auto split_tag) {
      constexpr bool SP = decltype(split_tag)::value;
      switch (bn) {
        case 32: launch_conv_tap<32, SP>(c, st, grid, smem, *twh, *twl, ag); break;
        case 48: launch_conv_tap<48, SP>(c, st, grid, smem, *twh, *twl, ag); break;
        case 64: launch_conv_tap<64, SP>(c, st, grid, smem, *twh, *twl, ag); break;
        case 96: launch_conv_tap<96, SP>(c, st, grid, smem, *twh, *twl, ag); break;
        case 192: launch_conv_tap<192, SP>(c, st, grid, smem, *twh, *twl, ag); break;
        default: launch_conv_tap<128, SP>(c, st, grid, smem, *twh, *twl, ag); break;
      }
    };
    if (split) go(std::true_type{});
    else go(std::false_type{});
  }
  return true;
}

template <int BN, bool SPLIT, int KC, int CL>
void launch_conv_wtap(Ctx* c, cudaStream_t st, dim3 grid, int smem, const tcwtap::WtapArgs& a) {
  auto kern = tcwtap::conv_wtap_kernel<BN, SPLIT, KC, CL>;
  static int attr_smem[16] = {};
  if (attr_smem[c->device & 15] < smem) {
    CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_smem[c->device & 15] = smem;
  }
  if constexpr (CL == 1) {
    kern<<<grid, tcwtap::kThreads, smem, st>>>(a);
  } else {
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = CL;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(tcwtap::kThreads);
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CDNN_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  }
  check_launch("conv_wtap_kernel");
  count_launch(c);
}

// Co-resident clusters of CL wtap CTAs (GPC packing: fewer than SMs / CL)
template <int BN, bool SPLIT, int KC, int CL>
int wtap_active_clusters(Ctx* c, int smem) {
  auto kern = tcwtap::conv_wtap_kernel<BN, SPLIT, KC, CL>;
  CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = CL;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, CL);
  cfg.blockDim = dim3(tcwtap::kThreads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  (void)c;
  return n;
}

// Tap-shift backward-filter (conv_wtap.cuh) for stride-1 convolutions with at
// least 16 channels per group; split-K partials + the deterministic reduce.
bool conv_wgrad_tap(Ctx* c, const ConvDescSlot& d, const float* x, const float* dy, float* dw, float* db,
                    cdnn_handle stream) {
  const ConvGeom& g = d.geom;
  if (g.sh != 1 || g.sw != 1 || g.Cg < 16) return false;
  const bool split = c->math_mode == CDNN_MATH_TF32X3;
  tcwtap::WtapArgs a{};
  a.N = g.N; a.Cg = g.Cg; a.H = g.H; a.W = g.W; a.Cog = g.Cog; a.P = g.P; a.Q = g.Q;
  a.R = g.R; a.S = g.S; a.dh = g.dh; a.dw = g.dw; a.ph = g.ph; a.pw = g.pw;
  virtual_grid(g.H, g.W, g.P, g.Q, g.ph, g.pw, g.R, g.S, g.dh, g.dw, a.Hv, a.Wv);
  if (int64_t(g.N) * a.Hv * a.Wv >= (int64_t(1) << 31)) return false;
  a.Mv = g.N * a.Hv * a.Wv;
  a.x_nstride = int64_t(g.C) * g.H * g.W;
  a.dy_nstride = int64_t(g.Co) * g.P * g.Q;
  a.Kc = g.Cg * g.R * g.S;
  a.div_hwv = FastDiv(uint32_t(a.Hv * a.Wv));
  a.div_wv = FastDiv(uint32_t(a.Wv));
  const int bn = pick_bn(g.Cog, 1 << 20, 1, {32, 64, 96, 128});  // (split-K fills the grid)
  a.cblocks = (g.Cg + 31) / 32;
  a.coblocks = (g.Cog + bn - 1) / bn;
  // pack the taps into groups of four equally spaced X rows: along kernel rows
  // (stride dw) while four columns remain, then the leftover columns along
  // kernel columns (stride dh*Wv), then what is left along its row
  std::vector<tcwtap::TapGroup> groups;
  auto add = [&](int r, int s, int dr, int ds, int n) {
    tcwtap::TapGroup tg{};
    tg.start = r * g.dh * a.Wv + s * g.dw;
    tg.stride = dr * g.dh * a.Wv + ds * g.dw;
    for (int j = 0; j < 4; ++j) tg.tap[j] = j < n ? (r + j * dr) * g.S + (s + j * ds) : -1;
    if (n == 1) tg.stride = g.dw;
    groups.push_back(tg);
  };
  const int sfull = g.S / 4 * 4, rfull = g.R / 4 * 4;
  for (int r = 0; r < g.R; ++r)
    for (int s = 0; s < sfull; s += 4) add(r, s, 0, 1, 4);
  for (int s = sfull; s < g.S; ++s)
    for (int r = 0; r < rfull; r += 4) add(r, s, 1, 0, 4);
  for (int r = rfull; r < g.R; ++r)
    if (sfull < g.S) add(r, sfull, 0, 1, g.S - sfull);
  if (int(groups.size()) > tcwtap::kMaxGroups) return false;
  a.ngroups = int(groups.size());
  for (int i = 0; i < a.ngroups; ++i) a.groups[i] = groups[i];
  // sets of groups per CTA: TMEM columns (groups x accumulator width) <= 256 lets two
  // CTAs share an SM; 3xTF32 with bn <= 64 accumulates [hi | lo] halves (2 x bn)
  constexpr int kBudget = 227 * 1024;
  const int acc_cols = (split && bn <= 64) ? 2 * bn : bn;
  int per_set = std::max(1, 256 / acc_cols);
  int smem = 0;
  bool widened = false;
  for (;;) {
    a.ggroups = (a.ngroups + per_set - 1) / per_set;
    int rows_max = 0;
    for (int i = 0; i < a.ggroups; ++i) {
      a.gbegin[i] = i * a.ngroups / a.ggroups;
      a.gbegin[i + 1] = (i + 1) * a.ngroups / a.ggroups;
      int lo = 1 << 30, hi = 0;
      for (int k = a.gbegin[i]; k < a.gbegin[i + 1]; ++k) {
        lo = std::min(lo, groups[k].start);
        hi = std::max(hi, groups[k].start + 3 * groups[k].stride);
      }
      a.rows_lo[i] = lo;
      rows_max = std::max(rows_max, hi - lo);
    }
    a.rowsA = (64 + rows_max + 7) & ~7;
    a.stages = 2;
    smem = tcwtap::smem_bytes(a.rowsA, bn, split, 64, 2);
    // one CTA per SM anyway (shared memory): use the whole 512-column TMEM
    if (!widened && smem > 113 * 1024 && per_set < 512 / acc_cols) {
      widened = true;
      per_set = std::max(1, 512 / acc_cols);
      continue;
    }
    if (smem <= kBudget) break;
    if (per_set == 1) return false;
    per_set = std::max(1, per_set / 2);
  }
  const int items = a.cblocks * a.ggroups * a.coblocks;
  const bool two_per_sm = smem <= 113 * 1024 && bn < 96;  // BN >= 96: one CTA per SM (registers)
  // (deeper pipelines -- three 64-pixel stages, or four 32-pixel ones -- measured slower
  // on AlexNet's weight gradients: 0.54 -> 0.61 ms for conv3; two 64-pixel stages stay)
  const int kc = 64;
  a.nchunks = (a.Mv + kc - 1) / kc;
  // pairs of CTAs along the channel blocks share the dY staging (conv_wtap.cuh, CL):
  // AlexNet's five weight gradients 2.96 -> 2.80 ms; clusters of four measured no
  // faster (conv3 slower: fewer co-resident clusters than whole waves need)
  int cl = 2;
  while (cl > 1 && (a.cblocks % cl != 0 || (bn / cl) * 2 % 8 != 0)) cl /= 2;
  int target = (two_per_sm ? 2 : 1) * kNumSMs;
  if (cl > 1) {
    auto q = [&](auto split_tag) {
      constexpr bool SP = decltype(split_tag)::value;
      auto pick = [&](auto cl_tag) {
        constexpr int CLc = decltype(cl_tag)::value;
        switch (bn) {
          case 32: return wtap_active_clusters<32, SP, 64, CLc>(c, smem);
          case 64: return wtap_active_clusters<64, SP, 64, CLc>(c, smem);
          case 96: return wtap_active_clusters<96, SP, 64, CLc>(c, smem);
          default: return wtap_active_clusters<128, SP, 64, CLc>(c, smem);
        }
      };
      return cl == 4 ? pick(std::integral_constant<int, 4>{}) : pick(std::integral_constant<int, 2>{});
    };
    const int nclusters = split ? q(std::true_type{}) : q(std::false_type{});
    if (nclusters <= 0) cl = 1;
    else target = nclusters * cl;
  }
  // whole waves: the largest split count whose grid still fits the resident slots
  // (a 168-CTA grid on 148 one-CTA SMs runs as two waves, the second one 20 CTAs wide)
  int splits = items >= target ? 1 : target / items;
  splits = std::max(1, std::min(a.nchunks, splits));
  a.chunks_per_split = (a.nchunks + splits - 1) / splits;
  a.splits = (a.nchunks + a.chunks_per_split - 1) / a.chunks_per_split;
  a.want_bias = db != nullptr;
  cudaStream_t st = stream_of(c, stream);
  Workspace& wsp = workspace_of(c, stream);
  const size_t ws_elems = size_t(a.splits) * g.Cog * (a.Kc + 1);
  float* ws = static_cast<float*>(wsp.get(ws_elems * sizeof(float), c->device));
  dim3 grid(a.splits, items);
  for (int grp = 0; grp < g.group; ++grp) {
    tcwtap::WtapArgs ag = a;
    ag.x = x + int64_t(grp) * g.Cg * g.H * g.W;
    ag.dy = dy + int64_t(grp) * g.Cog * g.P * g.Q;
    ag.ws = ws;
    auto go = [&](auto split_tag) {
      constexpr bool SP = decltype(split_tag)::value;
      auto launch = [&](auto cl_tag) {
        constexpr int CLc = decltype(cl_tag)::value;
        switch (bn) {
          case 32: launch_conv_wtap<32, SP, 64, CLc>(c, st, grid, smem, ag); break;
          case 64: launch_conv_wtap<64, SP, 64, CLc>(c, st, grid, smem, ag); break;
          case 96: launch_conv_wtap<96, SP, 64, CLc>(c, st, grid, smem, ag); break;
          default: launch_conv_wtap<128, SP, 64, CLc>(c, st, grid, smem, ag); break;
        }
      };
      if (cl == 4) launch(std::integral_constant<int, 4>{});
      else if (cl == 2) launch(std::integral_constant<int, 2>{});
      else launch(std::integral_constant<int, 1>{});
    };
    if (split) go(std::true_type{});
    else go(std::false_type{});
    ConvWgradPermEpi<float> epi{dw ? dw + int64_t(grp) * g.Cog * a.Kc : nullptr, db ? db + grp * g.Cog : nullptr,
                                a.Kc, g.Cg, g.R * g.S};
    launch_reduce(c, st, ws, a.Kc + 1, g.Cog, a.splits, epi);
  }
  return true;
}

template <int BN, bool SPLIT, int TW, int CB>
void launch_conv_tma(Ctx* c, cudaStream_t st, dim3 grid, const CUtensorMap& tin, const CUtensorMap& twh,
                     const CUtensorMap& twl, const tcconv::ConvTmaArgs& a) {
  constexpr int smem = tcconv::smem_bytes<BN, SPLIT, TW, CB>();
  static_assert(smem <= 227 * 1024, "conv_tma smem budget");
  auto kern = tcconv::conv_tma_kernel<BN, SPLIT, TW, CB>;
  static bool attr_set[16] = {};
  if (!attr_set[c->device & 15]) {
    CDNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set[c->device & 15] = true;
  }
  kern<<<grid, tcconv::kThreads, smem, st>>>(tin, twh, twl, a);
  check_launch("conv_tma_kernel");
  count_launch(c);
}

// Direct convolution through TMA tap windows (stride 1, dilation 1, one group).
// backward_data: out = dx, in = dy, flipped taps.  Returns false when the
// shape is not eligible (the implicit-GEMM gather path handles it).
bool conv_direct_tma(Ctx* c, const ConvDescSlot& dconst, bool backward_data, const float* in, const float* w,
                     const float* bias, float* out, cdnn_handle stream, bool relu = false) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  const ConvGeom& g = d.geom;
  if (g.group != 1 || g.sh != 1 || g.sw != 1 || g.dh != 1 || g.dw != 1) return false;
  // direct-conv extents
  const int Cin = backward_data ? g.Co : g.C, Hin = backward_data ? g.P : g.H, Win = backward_data ? g.Q : g.W;
  const int Cout = backward_data ? g.C : g.Co, P = backward_data ? g.H : g.P, Q = backward_data ? g.W : g.Q;
  const int oh = backward_data ? g.R - 1 - g.ph : g.ph, ow = backward_data ? g.S - 1 - g.pw : g.pw;
  if (Win % 4 != 0 || Cout > 4096 || Win > 65535) return false;
  const bool split = c->math_mode == CDNN_MATH_TF32X3;
  tcconv::ConvTmaArgs a{};
  a.N = g.N; a.Cin = Cin; a.Hin = Hin; a.Win = Win;
  a.Cout = Cout; a.P = P; a.Q = Q; a.R = g.R; a.S = g.S; a.oh = oh; a.ow = ow;
  // 32-pixel atoms of rb = 32/TW image rows; a tile = 4 atoms
  const int TW = Q <= 8 ? 8 : (Q <= 16 ? 16 : 32);
  const int rb = 32 / TW, rows = 128 / TW;
  a.TH = std::min(rows, (P + rb - 1) / rb * rb);
  a.NB = std::max(1, std::min(rows / a.TH, g.N));
  const int CB = Cin >= 16 ? 32 : 8;
  a.cblocks = (Cin + CB - 1) / CB;
  a.tiles_q = (Q + TW - 1) / TW;
  a.tiles_p = (P + a.TH - 1) / a.TH;
  const int tiles_n = (g.N + a.NB - 1) / a.NB;
  a.bias = bias;
  a.out = out;
  a.relu = relu ? 1 : 0;
  const int tiles = a.tiles_q * a.tiles_p * tiles_n;
  int bn = Cout <= 32 ? 32 : (Cout <= 64 ? 64 : 128);
  if (bn > 32 && tiles * ((Cout + bn - 1) / bn) < kNumSMs) bn = bn == 128 ? 64 : 32;
  const int kpad = a.cblocks * CB;
  const int RS = g.R * g.S;
  // repack (and pre-split) the weights into the per-tap K-major operand
  const size_t elems = size_t(RS) * Cout * kpad;
  const int slot = backward_data ? 2 : 0;
  if (!d.repack[slot] || d.repack[slot]->bytes < elems * 4) {
    d.repack[slot] = device_alloc_shared(elems * 4, c->device);
    d.repack[slot + 1] = device_alloc_shared(elems * 4, c->device);
  }
  float* whi = static_cast<float*>(d.repack[slot]->ptr);
  float* wlo = static_cast<float*>(d.repack[slot + 1]->ptr);
  cudaStream_t st = stream_of(c, stream);
  tcconv::repack_weights_kernel<<<grid_for(int64_t(elems), 256), 256, 0, st>>>(
      w, whi, wlo, g.Co, g.C, g.R, g.S, Cout, kpad, backward_data, split);
  check_launch("repack_weights");
  count_launch(c);
  // tensor maps: input NCHW {W, H, C, N} with box {TW, 1, CB, 1}; weights {kpad, RS*Cout} box {CB, BN}
  const uint64_t idims[4] = {uint64_t(Win), uint64_t(Hin), uint64_t(Cin), uint64_t(g.N)};
  const uint64_t istr[3] = {uint64_t(Win), uint64_t(Hin) * Win, uint64_t(Cin) * Hin * Win};
  // staged window: TW + 4 columns from the 16-byte aligned start (no swizzle)
  const uint32_t ibox[4] = {uint32_t(TW + 4), uint32_t(rb), uint32_t(CB), 1u};
  const CUtensorMap* tin = tmap_generic(c, in, 4, idims, istr, ibox, 0);
  const uint64_t wdims[2] = {uint64_t(kpad), uint64_t(RS) * Cout};
  const uint64_t wstr[1] = {uint64_t(kpad)};
  const uint32_t wbox[2] = {uint32_t(CB), uint32_t(bn)};
  const CUtensorMap* twh = tmap_generic(c, whi, 2, wdims, wstr, wbox, CB * 4);
  const CUtensorMap* twl = tmap_generic(c, wlo, 2, wdims, wstr, wbox, CB * 4);
  dim3 grid(tiles, (Cout + bn - 1) / bn);
  auto go_cb = [&](auto split_tag, auto tw_tag, auto cb_tag) {
    constexpr bool S = decltype(split_tag)::value;
    constexpr int W = decltype(tw_tag)::value, K = decltype(cb_tag)::value;
    switch (bn) {
      case 32: launch_conv_tma<32, S, W, K>(c, st, grid, *tin, *twh, *twl, a); break;
      case 64: launch_conv_tma<64, S, W, K>(c, st, grid, *tin, *twh, *twl, a); break;
      default: launch_conv_tma<128, S, W, K>(c, st, grid, *tin, *twh, *twl, a); break;
    }
  };
  auto go_tw = [&](auto split_tag, auto tw_tag) {
    if (CB == 32) go_cb(split_tag, tw_tag, std::integral_constant<int, 32>{});
    else go_cb(split_tag, tw_tag, std::integral_constant<int, 8>{});
  };
  auto go = [&](auto split_tag) {
    if (TW == 32) go_tw(split_tag, std::integral_constant<int, 32>{});
    else if (TW == 16) go_tw(split_tag, std::integral_constant<int, 16>{});
    else go_tw(split_tag, std::integral_constant<int, 8>{});
  };
  if (split) go(std::true_type{});
  else go(std::false_type{});
  return true;
}

// ---- space-to-depth: stride-s convolution == stride-1 convolution over C*s*s channels
// X'[n][(dy*s + dx)*C + c][h'][w'] = x_pad[n][c][s*h' + dy][s*w' + dx]
// W'[co][(dy*s + dx)*C + c][r'][t'] = W[co][c][s*r' + dy][s*t' + dx]   (0 past the filter)
// with kernel ceil(R/s) x ceil(S/s), no padding, same output P x Q.  AlexNet conv1
// (11x11, stride 4, 3 channels) becomes a 3x3 convolution over 48 channels that the
// tap-shift kernels run on the tensor cores.
bool s2d_eligible(const ConvGeom& g) {
  return g.sh == g.sw && g.sh >= 2 && g.dh == 1 && g.dw == 1 && g.group == 1 &&
         g.C * g.sh * g.sw <= 128 && (g.R + g.sh - 1) / g.sh <= 4 && (g.S + g.sw - 1) / g.sw <= 4;
}

ConvDescSlot& s2d_desc(Ctx* c, const ConvDescSlot& dconst) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  if (!d.s2d) {
    const ConvGeom& g = d.geom;
    const int s = g.sh;
    auto child = std::make_shared<ConvDescSlot>();
    ConvGeom& h = child->geom;
    h.N = g.N; h.C = g.C * s * s; h.Co = g.Co; h.P = g.P; h.Q = g.Q;
    h.R = (g.R + s - 1) / s; h.S = (g.S + s - 1) / s;
    h.H = g.P + h.R - 1; h.W = g.Q + h.S - 1;
    h.sh = h.sw = 1; h.ph = h.pw = 0; h.dh = h.dw = 1;
    h.group = 1; h.Cg = h.C; h.Cog = h.Co;
    h.div_PQ = FastDiv(uint32_t(h.P * h.Q)); h.div_Q = FastDiv(uint32_t(h.Q));
    h.div_HW = FastDiv(uint32_t(h.H * h.W)); h.div_W = FastDiv(uint32_t(h.W));
    child->P = h.P; child->Q = h.Q;
    child->Kc = h.Cg * h.R * h.S;
    child->Kd = h.Cog * h.R * h.S;
    d.s2d = child;
  }
  (void)c;
  return *d.s2d;
}

float* s2d_buffer(Ctx* c, const ConvDescSlot& dconst, int which, size_t elems) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  auto& b = d.s2d_buf[which];
  if (!b || b->bytes < elems * 4) b = device_alloc_shared(elems * 4, c->device);
  return static_cast<float*>(b->ptr);
}

// One warp-strided sweep per X' row (n, cc, h'): lanes walk w' (stores coalesced,
// loads a stride-s run of one input row); 32-bit index math (X' < 2^31 elements).
// Used for s < 4 (ResNet 3x3/2 downsampling: measured faster there than the
// grouped kernel below, 64 vs 71 us for res2_0 forward).
__global__ void s2d_input_rows_kernel(const float* __restrict__ x, float* __restrict__ xs, ConvGeom g, ConvGeom h) {
  const int s = g.sh;
  const int rows = h.N * h.C * h.H;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
    const int h2 = row % h.H;
    const int cc = (row / h.H) % h.C;
    const int n = row / (h.H * h.C);
    const int c = cc % g.C, ph = cc / g.C, dy = ph / s, dx = ph % s;
    const int y = s * h2 + dy - g.ph;
    float* out = xs + size_t(row) * h.W;
    const bool yok = y >= 0 && y < g.H;
    const float* in = x + (size_t(n) * g.C + c) * g.H * g.W + size_t(yok ? y : 0) * g.W;
    for (int w2 = lane; w2 < h.W; w2 += 32) {
      const int xx = s * w2 + dx - g.pw;
      out[w2] = (yok && xx >= 0 && xx < g.W) ? __ldg(in + xx) : 0.f;
    }
  }
}

// One warp per X' row group (n, c, dy, h'): the s rows X'[n][(dy*s + dx)*C + c][h']
// for dx = 0..s-1 all come from input row y = s*h' + dy - pad, so a lane issues
// the s loads of its w' together (they cover one contiguous run of the input row:
// every line is used by the group) before the s coalesced stores; one index
// decomposition per group, s x the loads in flight of a row-per-warp sweep
// (AlexNet conv1, s = 4: 335 -> 145 us).
__global__ void s2d_input_kernel(const float* __restrict__ x, float* __restrict__ xs, ConvGeom g, ConvGeom h) {
  const int s = g.sh;
  const int groups = h.N * g.C * s * h.H;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t plane = size_t(h.H) * h.W;
  for (int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; grp < groups; grp += warps) {
    const int h2 = grp % h.H;
    const int t = grp / h.H;
    const int dy = t % s, c = (t / s) % g.C, n = t / (s * g.C);
    const int y = s * h2 + dy - g.ph;
    const bool yok = y >= 0 && y < g.H;
    const float* in = x + (size_t(n) * g.C + c) * g.H * g.W + size_t(yok ? y : 0) * g.W;
    // X' row of dx = 0; the row of phase dx is dx*C planes further
    float* out = xs + (size_t(n) * h.C + size_t(dy) * s * g.C + c) * plane + size_t(h2) * h.W;
    const size_t step = size_t(g.C) * plane;
    for (int w2 = lane; w2 < h.W; w2 += 32)
      for (int d0 = 0; d0 < s; d0 += 8) {  // s <= 8 at every eligible AlexNet-like stem
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int xx = s * w2 + d0 + j - g.pw;
          v[j] = (d0 + j < s && yok && xx >= 0 && xx < g.W) ? __ldg(in + xx) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (d0 + j < s) out[(d0 + j) * step + w2] = v[j];
      }
  }
}

// Compile-time stride S (AlexNet's stem: 4) and X' rows of at most 64: a warp takes
// NG consecutive groups and issues every load of them (NG x 2 x S per lane) before any
// store -- the per-group kernel above kept one group's 2 x 8 loads in flight
// (AlexNet conv1: 318 MB in 146 us, 2.2 TB/s).
template <int S, int NG>
__global__ void __launch_bounds__(256) s2d_input_k(const float* __restrict__ x, float* __restrict__ xs, ConvGeom g,
                                                   ConvGeom h) {
  const int groups = h.N * g.C * S * h.H;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t plane = size_t(h.H) * h.W;
  const size_t step = size_t(g.C) * plane;
  for (int g0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NG; g0 < groups; g0 += warps * NG) {
    float v[NG][2][S];
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      const int grp = g0 + q;
      const int h2 = grp % h.H, t = grp / h.H;
      const int dy = t % S, c = (t / S) % g.C, n = t / (S * g.C);
      const int y = S * h2 + dy - g.ph;
      const bool ok = grp < groups && y >= 0 && y < g.H;
      const float* in = x + (size_t(n) * g.C + c) * g.H * g.W + size_t(ok ? y : 0) * g.W;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const int w2 = lane + 32 * r, xx = S * w2 + j - g.pw;
          v[q][r][j] = (ok && w2 < h.W && xx >= 0 && xx < g.W) ? __ldg(in + xx) : 0.f;
        }
    }
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      const int grp = g0 + q;
      if (grp >= groups) break;
      const int h2 = grp % h.H, t = grp / h.H;
      const int dy = t % S, c = (t / S) % g.C, n = t / (S * g.C);
      float* out = xs + (size_t(n) * h.C + size_t(dy) * S * g.C + c) * plane + size_t(h2) * h.W;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int w2 = lane + 32 * r;
        if (w2 < h.W)
#pragma unroll
          for (int j = 0; j < S; ++j) out[j * step + w2] = v[q][r][j];
      }
    }
  }
}

void s2d_input(const float* x, float* xs, const ConvGeom& g, const ConvGeom& h, cudaStream_t st) {
  if (g.sh == 4 && h.W <= 64) {
    constexpr int NG = 4;
    s2d_input_k<4, NG><<<grid_for(int64_t(h.N) * g.C * 4 * h.H * 32 / NG, 256), 256, 0, st>>>(x, xs, g, h);
  } else if (g.sh >= 4)
    s2d_input_kernel<<<grid_for(int64_t(h.N) * h.C * h.H * 32 / g.sh, 256), 256, 0, st>>>(x, xs, g, h);
  else
    s2d_input_rows_kernel<<<grid_for(int64_t(h.N) * h.C * h.H * 32, 256), 256, 0, st>>>(x, xs, g, h);
}

__global__ void s2d_weight_kernel(const float* __restrict__ w, float* __restrict__ ws, ConvGeom g, ConvGeom h) {
  const int s = g.sh;
  const int total = h.Co * h.C * h.R * h.S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int t2 = i % h.S, r2 = (i / h.S) % h.R, cc = (i / (h.S * h.R)) % h.C, co = i / (h.S * h.R * h.C);
    const int c = cc % g.C, ph = cc / g.C, dy = ph / s, dx = ph % s;
    const int r = s * r2 + dy, t = s * t2 + dx;
    ws[i] = (r < g.R && t < g.S) ? w[((co * g.C + c) * g.R + r) * g.S + t] : 0.f;
  }
}

// dW[co][c][r][t] += dW'[co][(dy*s + dx)*C + c][r/s][t/s]
__global__ void s2d_dweight_kernel(const float* __restrict__ dws, float* __restrict__ dw, ConvGeom g, ConvGeom h) {
  const int s = g.sh;
  const int total = g.Co * g.C * g.R * g.S;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int t = i % g.S, r = (i / g.S) % g.R, c = (i / (g.S * g.R)) % g.C, co = i / (g.S * g.R * g.C);
    const int cc = ((r % s) * s + (t % s)) * g.C + c;
    dw[i] += dws[((co * h.C + cc) * h.R + r / s) * h.S + t / s];
  }
}

// dX[n][c][y][x] = dX'[n][(dy*s + dx)*C + c][(y+ph)/s][(x+pw)/s]
__global__ void d2s_input_kernel(const float* __restrict__ dxs, float* __restrict__ dx, ConvGeom g, ConvGeom h) {
  const int s = g.sh;
  const int64_t total = int64_t(g.N) * g.C * g.H * g.W;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int xx = int(i % g.W);
    const int y = int((i / g.W) % g.H);
    const int c = int((i / (int64_t(g.W) * g.H)) % g.C);
    const int n = int(i / (int64_t(g.W) * g.H * g.C));
    const int yp = y + g.ph, xp = xx + g.pw;
    const int h2 = yp / s, w2 = xp / s;
    const int cc = ((yp % s) * s + (xp % s)) * g.C + c;
    dx[i] = (h2 < h.H && w2 < h.W) ? dxs[((int64_t(n) * h.C + cc) * h.H + h2) * h.W + w2] : 0.f;
  }
}

bool conv_wgrad_s2d(Ctx* c, const ConvDescSlot& d, const float* x, const float* dy, float* dw, float* db,
                    cdnn_handle stream, bool input_unchanged) {
  if (!s2d_eligible(d.geom)) return false;
  ConvDescSlot& e = s2d_desc(c, d);
  const ConvGeom &g = d.geom, &h = e.geom;
  if (h.C < 16) return false;
  cudaStream_t st = stream_of(c, stream);
  // the forward's rewrite of this very input, when the caller promises it is unchanged
  const bool reuse = input_unchanged && d.s2d_fwd_src == x && d.s2d_buf[0];
  float* xs = reuse ? static_cast<float*>(d.s2d_buf[0]->ptr) : s2d_buffer(c, d, 2, size_t(h.N) * h.C * h.H * h.W);
  float* dws = s2d_buffer(c, d, 3, size_t(h.Co) * h.C * h.R * h.S);
  if (!reuse) s2d_input(x, xs, g, h, st);
  CDNN_CUDA(cudaMemsetAsync(dws, 0, size_t(h.Co) * h.C * h.R * h.S * 4, st));
  check_launch("s2d");
  count_launch(c);
  if (!conv_wgrad_tap(c, e, xs, dy, dw ? dws : nullptr, db, stream)) return false;
  if (dw) {
    s2d_dweight_kernel<<<grid_for(int64_t(g.Co) * g.C * g.R * g.S, 256), 256, 0, st>>>(dws, dw, g, h);
    check_launch("s2d_dweight");
    count_launch(c);
  }
  return true;
}

bool conv_dgrad_s2d(Ctx* c, const ConvDescSlot& d, const float* w, const float* dy, float* dx, cdnn_handle stream) {
  if (!s2d_eligible(d.geom)) return false;
  ConvDescSlot& e = s2d_desc(c, d);
  const ConvGeom &g = d.geom, &h = e.geom;
  cudaStream_t st = stream_of(c, stream);
  float* wsb = s2d_buffer(c, d, 1, size_t(h.Co) * h.C * h.R * h.S);
  float* dxs = s2d_buffer(c, d, 4, size_t(h.N) * h.C * h.H * h.W);
  s2d_weight_kernel<<<grid_for(int64_t(h.Co) * h.C * h.R * h.S, 256), 256, 0, st>>>(w, wsb, g, h);
  check_launch("s2d");
  count_launch(c);
  if (!conv_tap(c, e, true, dy, wsb, nullptr, dxs, stream)) return false;
  d2s_input_kernel<<<grid_for(int64_t(g.N) * g.C * g.H * g.W, 256), 256, 0, st>>>(dxs, dx, g, h);
  check_launch("d2s");
  count_launch(c);
  return true;
}

bool conv_forward_s2d(Ctx* c, const ConvDescSlot& d, const float* x, const float* w, const float* bias, float* y,
                      cdnn_handle stream, bool relu = false) {
  if (!s2d_eligible(d.geom)) return false;
  ConvDescSlot& e = s2d_desc(c, d);
  const ConvGeom &g = d.geom, &h = e.geom;
  cudaStream_t st = stream_of(c, stream);
  float* xs = s2d_buffer(c, d, 0, size_t(h.N) * h.C * h.H * h.W);
  float* wsb = s2d_buffer(c, d, 1, size_t(h.Co) * h.C * h.R * h.S);
  s2d_input(x, xs, g, h, st);
  const_cast<ConvDescSlot&>(d).s2d_fwd_src = x;
  s2d_weight_kernel<<<grid_for(int64_t(h.Co) * h.C * h.R * h.S, 256), 256, 0, st>>>(w, wsb, g, h);
  check_launch("s2d");
  count_launch(c, 2);
  return conv_tap(c, e, false, xs, wsb, bias, y, stream, relu);
}

// ---- column fold: a stride-1 convolution over C < 16 channels (CIFAR / LeNet conv1)
// == an R x 1 convolution over C' = max(16, C*S) channels with the S filter columns
// folded into the channels (zero channels past C*S):
//   X'[n][s*C + c][y][q] = x[n][c][y][q + s - pw]          (0 outside), H' = H, W' = Q
//   W'[co][s*C + c][r][0] = W[co][c][r][s]
// Same output P x Q, row padding kept (ph), no column padding.  The 16+ channel
// operand runs on the tap-shift kernels at full 8-wide K steps (and the backward
// filter on conv_wtap, which needs >= 16 channels), instead of staging 3-channel
// rows with scalar gathers.
bool cf_eligible(const ConvGeom& g) {
  return g.sh == 1 && g.sw == 1 && g.dh == 1 && g.dw == 1 && g.group == 1 && g.C < 16 &&
         g.C * g.S <= 32 && g.S > 1 && g.pw < g.S;
}

ConvDescSlot& cf_desc(const ConvDescSlot& dconst) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  if (!d.cf) {
    const ConvGeom& g = d.geom;
    auto child = std::make_shared<ConvDescSlot>();
    ConvGeom& h = child->geom;
    h = g;
    h.C = std::max(16, g.C * g.S);
    h.W = g.Q;
    h.S = 1;
    h.pw = 0;
    h.Cg = h.C; h.Cog = h.Co;
    h.div_PQ = FastDiv(uint32_t(h.P * h.Q)); h.div_Q = FastDiv(uint32_t(h.Q));
    h.div_HW = FastDiv(uint32_t(h.H * h.W)); h.div_W = FastDiv(uint32_t(h.W));
    child->P = h.P; child->Q = h.Q;
    child->Kc = h.Cg * h.R * h.S;
    child->Kd = h.Cog * h.R * h.S;
    d.cf = child;
  }
  return *d.cf;
}

float* cf_buffer(Ctx* c, const ConvDescSlot& dconst, int which, size_t elems) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  auto& b = d.cf_buf[which];
  if (!b || b->bytes < elems * 4) b = device_alloc_shared(elems * 4, c->device);
  return static_cast<float*>(b->ptr);
}

// One warp-strided sweep per X' row (n, s*C + c, y): lanes walk q, so the loads
// of a row are one contiguous (shifted) run of the input row and the stores are
// coalesced; 32-bit index math (X' < 2^31 elements).
__global__ void cf_input_kernel(const float* __restrict__ x, float* __restrict__ xf, ConvGeom g, ConvGeom h) {
  const int rows = h.N * h.C * h.H;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += warps) {
    const int y = row % h.H;
    const int cc = (row / h.H) % h.C;
    const int n = row / (h.H * h.C);
    const int s = cc / g.C, c = cc - s * g.C;
    float* out = xf + size_t(row) * h.W;
    const bool live = s < g.S;
    const float* in = x + (size_t(n) * g.C + c) * g.H * g.W + size_t(y) * g.W;
    for (int q = lane; q < h.W; q += 32) {
      const int xx = q + s - g.pw;
      out[q] = (live && xx >= 0 && xx < g.W) ? __ldg(in + xx) : 0.f;
    }
  }
}

__global__ void cf_weight_kernel(const float* __restrict__ w, float* __restrict__ wf, ConvGeom g, ConvGeom h) {
  const int total = h.Co * h.C * h.R;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int r = i % h.R, cc = (i / h.R) % h.C, co = i / (h.R * h.C);
    const int s = cc / g.C, c = cc - s * g.C;
    wf[i] = s < g.S ? w[((co * g.C + c) * g.R + r) * g.S + s] : 0.f;
  }
}

bool conv_forward_cf(Ctx* c, const ConvDescSlot& d, const float* x, const float* w, const float* bias, float* y,
                     cdnn_handle stream, bool relu) {
  if (!cf_eligible(d.geom)) return false;
  ConvDescSlot& e = cf_desc(d);
  const ConvGeom &g = d.geom, &h = e.geom;
  cudaStream_t st = stream_of(c, stream);
  float* xf = cf_buffer(c, d, 0, size_t(h.N) * h.C * h.H * h.W);
  float* wf = cf_buffer(c, d, 1, size_t(h.Co) * h.C * h.R);
  cf_input_kernel<<<grid_for(int64_t(h.N) * h.C * h.H * 32, 256), 256, 0, st>>>(x, xf, g, h);
  cf_weight_kernel<<<grid_for(int64_t(h.Co) * h.C * h.R, 256), 256, 0, st>>>(w, wf, g, h);
  check_launch("column fold");
  count_launch(c, 2);
  return conv_tap(c, e, false, xf, wf, bias, y, stream, relu);
}

template <typename T>
void conv_forward_t(Ctx* c, const ConvDescSlot& d, const BufferSlot& X, const BufferSlot& Wt,
                    const BufferSlot* B, BufferSlot& Y, cdnn_handle stream, bool relu) {
  const ConvGeom& g = d.geom;
  cudaStream_t st = stream_of(c, stream);
  Workspace& ws = workspace_of(c, stream);
  const int M = g.N * g.P * g.Q, N = g.Cog, K = d.Kc;
  if constexpr (std::is_same_v<T, float>) {
    if (conv_forward_s2d(c, d, reinterpret_cast<const float*>(X.dev), reinterpret_cast<const float*>(Wt.dev),
                         B ? reinterpret_cast<const float*>(B->dev) : nullptr, reinterpret_cast<float*>(Y.dev), stream,
                         relu))
      return;
    if (conv_forward_cf(c, d, reinterpret_cast<const float*>(X.dev), reinterpret_cast<const float*>(Wt.dev),
                        B ? reinterpret_cast<const float*>(B->dev) : nullptr, reinterpret_cast<float*>(Y.dev), stream,
                        relu))
      return;
    if (conv_tap(c, d, false, reinterpret_cast<const float*>(X.dev), reinterpret_cast<const float*>(Wt.dev),
                 B ? reinterpret_cast<const float*>(B->dev) : nullptr, reinterpret_cast<float*>(Y.dev), stream, relu))
      return;
    if (conv_direct_tma(c, d, false, reinterpret_cast<const float*>(X.dev), reinterpret_cast<const float*>(Wt.dev),
                        B ? reinterpret_cast<const float*>(B->dev) : nullptr, reinterpret_cast<float*>(Y.dev), stream, relu))
      return;
  }
  for (int grp = 0; grp < g.group; ++grp) {
    const T* x = reinterpret_cast<const T*>(X.dev) + int64_t(grp) * g.Cg * g.H * g.W;
    const T* w = reinterpret_cast<const T*>(Wt.dev) + int64_t(grp) * g.Cog * K;
    ConvFwdA<T> va{x, d.taps, g, M, K};
    DenseView<T> vb{w, int64_t(K), 1, N, K, false};
    ConvFwdEpi<T> epi{reinterpret_cast<T*>(Y.dev) + int64_t(grp) * g.Cog * g.P * g.Q,
                      B ? reinterpret_cast<const T*>(B->dev) + grp * g.Cog : nullptr, g, relu};
    if constexpr (std::is_same_v<T, float>) {
      const GemmPlan pl = plan_tc(M, N, K);
      TmaReq rb;
      with_operand(c, vb, pl.bn, rb, [&](const auto& b) { run_tc(c, st, ws, pl, M, N, K, va, b, epi, TmaReq{}, rb); });
    } else {
      run_simt<T>(c, st, ws, plan_simt(M, N, K), M, N, K, va, vb, epi);
    }
  }
}

// Strided backward-data as a direct gather: one thread per bottom element
// (img, c, h, w) visits only the taps whose output pixel exists,
// p = (h + ph - r*dh) / sh with zero remainder, so none of the (sh*sw - 1)/(sh*sw)
// structurally-zero products of the implicit-GEMM view are computed.  Exact
// FMA accumulation in T, co-major order; consecutive threads walk w (dY loads
// near-coalesced, filter loads warp-uniform).
template <typename T>
__global__ void __launch_bounds__(256) conv_dgrad_direct_kernel(const T* __restrict__ w, const T* __restrict__ dy,
                                                                T* __restrict__ dx, ConvGeom g, int64_t total) {
  // columns in phase-major order: j -> x = (j / Wq) + (j % Wq) * sw, so a warp shares
  // one column phase (same valid taps, no divergence) and reads consecutive q
  const int Wq = (g.W + g.sw - 1) / g.sw, Wj = Wq * g.sw;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int j = int(i % Wj);
    const int x = j / Wq + (j % Wq) * g.sw;
    if (x >= g.W) continue;
    const int y = int((i / Wj) % g.H);
    const int c = int((i / (int64_t(Wj) * g.H)) % g.C);
    const int img = int(i / (int64_t(Wj) * g.H * g.C));
    const int grp = c / g.Cg, cg = c - grp * g.Cg;
    T acc = T(0);
    for (int r = 0; r < g.R; ++r) {
      const int ty = y + g.ph - r * g.dh;
      if (ty < 0 || ty % g.sh) continue;
      const int p = ty / g.sh;
      if (p >= g.P) continue;
      for (int s = 0; s < g.S; ++s) {
        const int tx = x + g.pw - s * g.dw;
        if (tx < 0 || tx % g.sw) continue;
        const int q = tx / g.sw;
        if (q >= g.Q) continue;
        const T* wp = w + ((int64_t(grp) * g.Cog * g.Cg + cg) * g.R + r) * g.S + s;
        const T* dp = dy + ((int64_t(img) * g.Co + int64_t(grp) * g.Cog) * g.P + p) * g.Q + q;
        const int64_t wstep = int64_t(g.Cg) * g.R * g.S, dstep = int64_t(g.P) * g.Q;
        for (int co = 0; co < g.Cog; ++co) acc = fma(__ldg(wp + co * wstep), __ldg(dp + co * dstep), acc);
      }
    }
    dx[((int64_t(img) * g.C + c) * g.H + y) * g.W + x] = acc;
  }
}

// dY of a strided convolution scattered onto the stride-1 output grid of the same
// filter (P1 = H + 2ph - dh(R-1) rows): up[t][u] = dY[t/sh][u/sw] on the stride
// lattice, 0 elsewhere.  Backward-data and backward-filter of the strided conv are
// then the stride-1 ones on `up` (sh*sw x the MACs, all on the tensor cores).
__global__ void zero_insert_kernel(const float* __restrict__ dy, float* __restrict__ up, int64_t planes, int P, int Q,
                                   int P1, int Q1, int sh, int sw) {
  // one warp-strided sweep per output row (plane, t): 32-bit math, coalesced stores
  const int64_t rows = planes * P1;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t row = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; row < rows; row += warps) {
    const int t = int(row % P1);
    const int64_t pl = row / P1;
    float* out = up + row * Q1;
    const bool trow = t % sh == 0 && t / sh < P;
    const float* in = dy + (pl * P + (trow ? t / sh : 0)) * Q;
    for (int u = lane; u < Q1; u += 32)
      out[u] = (trow && u % sw == 0 && u / sw < Q) ? __ldg(in + u / sw) : 0.f;
  }
}

// Runs `body(up)` with dY zero-inserted and the descriptor's geometry switched to
// the stride-1 equivalent; returns body's result (false = not handled).
template <class F>
bool with_zero_inserted(Ctx* c, const ConvDescSlot& dconst, const float* dy, cdnn_handle stream, int which, F body) {
  ConvDescSlot& d = const_cast<ConvDescSlot&>(dconst);
  const ConvGeom g = d.geom;
  const int P1 = g.H + 2 * g.ph - g.dh * (g.R - 1), Q1 = g.W + 2 * g.pw - g.dw * (g.S - 1);
  if (P1 < 1 || Q1 < 1) return false;
  const size_t elems = size_t(g.N) * g.Co * P1 * Q1;
  auto& buf = d.upsampled[which];
  if (!buf || buf->bytes < elems * 4) buf = device_alloc_shared(elems * 4, c->device);
  float* up = static_cast<float*>(buf->ptr);
  cudaStream_t st = stream_of(c, stream);
  zero_insert_kernel<<<grid_for(int64_t(g.N) * g.Co * P1 * 32, 256), 256, 0, st>>>(dy, up, int64_t(g.N) * g.Co, g.P, g.Q, P1, Q1,
                                                                     g.sh, g.sw);
  check_launch("zero_insert");
  count_launch(c);
  ConvGeom g1 = g;
  g1.sh = g1.sw = 1;
  g1.P = P1;
  g1.Q = Q1;
  d.geom = g1;
  bool ok = false;
  try {
    ok = body(static_cast<const float*>(up));
  } catch (...) {
    d.geom = g;
    throw;
  }
  d.geom = g;
  return ok;
}

// dx = gate > 0 ? dx : 0 in place (a fused ReLU backward the route could not apply
// in its epilogue)
template <typename T>
__global__ void relu_gate_kernel(const T* __restrict__ gate, T* __restrict__ dx, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (!(gate[i] > T(0))) dx[i] = T(0);
}

template <typename T>
void conv_backward_data_impl(Ctx* c, const ConvDescSlot& d, const BufferSlot& Wt, const BufferSlot& DY,
                             BufferSlot& DX, cdnn_handle stream, const T* gate, bool& gated);

template <typename T>
void conv_backward_data_t(Ctx* c, const ConvDescSlot& d, const BufferSlot& Wt, const BufferSlot& DY,
                          BufferSlot& DX, cdnn_handle stream, const T* gate = nullptr) {
  bool gated = false;
  conv_backward_data_impl<T>(c, d, Wt, DY, DX, stream, gate, gated);
  if (gate && !gated) {
    const ConvGeom& g = d.geom;
    const int64_t n = int64_t(g.N) * g.C * g.H * g.W;
    relu_gate_kernel<T><<<grid_for(n, 256), 256, 0, stream_of(c, stream)>>>(gate, reinterpret_cast<T*>(DX.dev), n);
    check_launch("relu_gate");
    count_launch(c);
  }
}

template <typename T>
void conv_backward_data_impl(Ctx* c, const ConvDescSlot& d, const BufferSlot& Wt, const BufferSlot& DY,
                             BufferSlot& DX, cdnn_handle stream, const T* gate, bool& gated) {
  const ConvGeom& g = d.geom;
  cudaStream_t st = stream_of(c, stream);
  Workspace& ws = workspace_of(c, stream);
  const int M = g.N * g.H * g.W, N = g.Cg, K = d.Kd;
  if constexpr (std::is_same_v<T, float>) {
    if ((g.sh > 1 || g.sw > 1) &&
        conv_dgrad_s2d(c, d, reinterpret_cast<const float*>(Wt.dev), reinterpret_cast<const float*>(DY.dev),
                       reinterpret_cast<float*>(DX.dev), stream))
      return;
    if ((g.sh > 1 || g.sw > 1) && g.sh <= 2 && g.sw <= 2 &&
        with_zero_inserted(c, d, reinterpret_cast<const float*>(DY.dev), stream, 0, [&](const float* up) {
          return conv_tap(c, d, true, up, reinterpret_cast<const float*>(Wt.dev), nullptr,
                          reinterpret_cast<float*>(DX.dev), stream);
        }))
      return;
  }
  if (g.sh > 1 || g.sw > 1) {
    const int64_t total = int64_t(g.N) * g.C * g.H * ((g.W + g.sw - 1) / g.sw * g.sw);
    conv_dgrad_direct_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(
        reinterpret_cast<const T*>(Wt.dev), reinterpret_cast<const T*>(DY.dev), reinterpret_cast<T*>(DX.dev), g, total);
    check_launch("conv_dgrad_direct");
    count_launch(c);
    return;
  }
  if constexpr (std::is_same_v<T, float>) {
    if (conv_tap(c, d, true, reinterpret_cast<const float*>(DY.dev), reinterpret_cast<const float*>(Wt.dev), nullptr,
                 reinterpret_cast<float*>(DX.dev), stream, false, gate)) {
      gated = gate != nullptr;
      return;
    }
    if (conv_direct_tma(c, d, true, reinterpret_cast<const float*>(DY.dev), reinterpret_cast<const float*>(Wt.dev),
                        nullptr, reinterpret_cast<float*>(DX.dev), stream))
      return;
  }
  for (int grp = 0; grp < g.group; ++grp) {
    const T* dy = reinterpret_cast<const T*>(DY.dev) + int64_t(grp) * g.Cog * g.P * g.Q;
    const T* w = reinterpret_cast<const T*>(Wt.dev) + int64_t(grp) * g.Cog * g.Cg * g.R * g.S;
    ConvDgradB<T> vb{w, d.koff, g.R * g.S, N, K};
    ConvDgradEpi<T> epi{reinterpret_cast<T*>(DX.dev) + int64_t(grp) * g.Cg * g.H * g.W, g};
    auto go = [&](const auto& va) {
      if constexpr (std::is_same_v<T, float>) run_tc(c, st, ws, plan_tc(M, N, K), M, N, K, va, vb, epi);
      else run_simt<T>(c, st, ws, plan_simt(M, N, K), M, N, K, va, vb, epi);
    };
    if (g.sh == 1 && g.sw == 1) go(ConvDgradA<T, true>{dy, d.dtaps, g, M, K});
    else go(ConvDgradA<T, false>{dy, d.dtaps, g, M, K});
  }
}

template <typename T>
void conv_backward_filter_t(Ctx* c, const ConvDescSlot& d, const BufferSlot& X, const BufferSlot& DY,
                            BufferSlot* DW, BufferSlot* DB, cdnn_handle stream, bool input_unchanged) {
  const ConvGeom& g = d.geom;
  cudaStream_t st = stream_of(c, stream);
  Workspace& ws = workspace_of(c, stream);
  if (!DW && !DB) return;
  // rows = taps (+1 all-ones row when the bias gradient is wanted)
  const int Kc = d.Kc, M = Kc + (DB ? 1 : 0), N = g.Cog, K = g.N * g.P * g.Q;
  if constexpr (std::is_same_v<T, float>) {
    float* dw = DW ? reinterpret_cast<float*>(DW->dev) : nullptr;
    float* db = DB ? reinterpret_cast<float*>(DB->dev) : nullptr;
    const float* x = reinterpret_cast<const float*>(X.dev);
    if (g.sh == 1 && g.sw == 1) {
      // (a column fold of the backward filter measured slower than the gather engine; forward only)
      if (conv_wgrad_tap(c, d, x, reinterpret_cast<const float*>(DY.dev), dw, db, stream)) return;
    } else if (conv_wgrad_s2d(c, d, x, reinterpret_cast<const float*>(DY.dev), dw, db, stream, input_unchanged)) {
      return;
    } else if (g.sh <= 2 && g.sw <= 2 && g.Cg >= 16 &&
               with_zero_inserted(c, d, reinterpret_cast<const float*>(DY.dev), stream, 1,
                                  [&](const float* up) { return conv_wgrad_tap(c, d, x, up, dw, db, stream); })) {
      return;
    }
  }
  for (int grp = 0; grp < g.group; ++grp) {
    const T* x = reinterpret_cast<const T*>(X.dev) + int64_t(grp) * g.Cg * g.H * g.W;
    const T* dy = reinterpret_cast<const T*>(DY.dev) + int64_t(grp) * g.Cog * g.P * g.Q;
    ConvWgradA<T> va{x, d.taps, g, Kc, K, DB != nullptr};
    ConvWgradB<T> vb{dy, g, N, K};
    // dw[co][tap] += D[tap][co] ; db[co] += D[Kc][co]
    ConvWgradEpi<T> epi{DW ? reinterpret_cast<T*>(DW->dev) + int64_t(grp) * g.Cog * Kc : nullptr,
                        DB ? reinterpret_cast<T*>(DB->dev) + grp * g.Cog : nullptr, Kc};
    if constexpr (std::is_same_v<T, float>) run_tc(c, st, ws, plan_tc(M, N, K), M, N, K, va, vb, epi);
    else run_simt<T>(c, st, ws, plan_simt(M, N, K), M, N, K, va, vb, epi);
  }
}

}  // namespace
}  // namespace cdnn

using namespace cdnn;

extern "C" {

int cdnn_conv_forward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle w, cdnn_handle bias,
                      cdnn_handle y, cdnn_handle stream) {
  return cdnn_conv_forward_ex(ctx, desc, x, w, bias, y, 0, stream);
}

int cdnn_conv_forward_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle w, cdnn_handle bias,
                         cdnn_handle y, int flags, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    const ConvDescSlot& d = conv_desc(c, desc);
    BufferSlot& X = buffer(c, x, "conv x");
    BufferSlot& W = buffer(c, w, "conv w");
    BufferSlot& Y = buffer(c, y, "conv y");
    BufferSlot* B = buffer_or_null(c, bias, "conv bias");
    const auto& g = d.geom;
    require_len(X, uint64_t(g.N) * g.C * g.H * g.W, "conv x");
    require_len(W, uint64_t(g.Co) * d.Kc, "conv w");
    require_len(Y, uint64_t(g.N) * g.Co * g.P * g.Q, "conv y");
    if (B) { require_len(*B, uint64_t(g.Co), "conv bias"); require_dtype(*B, X.dtype, "conv bias"); }
    require_dtype(W, X.dtype, "conv w");
    require_dtype(Y, X.dtype, "conv y");
    DeviceGuard dg(c);
    const bool relu = (flags & CDNN_CONV_RELU) != 0;
    if (X.dtype == CDNN_F32) conv_forward_t<float>(c, d, X, W, B, Y, stream, relu);
    else if (X.dtype == CDNN_F64) conv_forward_t<double>(c, d, X, W, B, Y, stream, relu);
    else fail(CDNN_INVALID_ARGUMENT, "conv: floating buffers required");
  });
}

int cdnn_conv_backward_data(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle w, cdnn_handle dy, cdnn_handle dx,
                            cdnn_handle stream) {
  return cdnn_conv_backward_data_ex(ctx, desc, w, dy, dx, 0, stream);
}

int cdnn_conv_backward_data_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle w, cdnn_handle dy, cdnn_handle dx,
                               cdnn_handle gate, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    const ConvDescSlot& d = conv_desc(c, desc);
    BufferSlot& W = buffer(c, w, "conv_bwd_data w");
    BufferSlot& DY = buffer(c, dy, "conv_bwd_data dy");
    BufferSlot& DX = buffer(c, dx, "conv_bwd_data dx");
    const auto& g = d.geom;
    require_len(W, uint64_t(g.Co) * d.Kc, "conv_bwd_data w");
    require_len(DY, uint64_t(g.N) * g.Co * g.P * g.Q, "conv_bwd_data dy");
    require_len(DX, uint64_t(g.N) * g.C * g.H * g.W, "conv_bwd_data dx");
    require_dtype(DY, W.dtype, "conv_bwd_data");
    require_dtype(DX, W.dtype, "conv_bwd_data");
    BufferSlot* G = buffer_or_null(c, gate, "conv_bwd_data gate");
    if (G) { require_len(*G, uint64_t(g.N) * g.C * g.H * g.W, "conv_bwd_data gate"); require_dtype(*G, W.dtype, "gate"); }
    DeviceGuard dg(c);
    if (W.dtype == CDNN_F32)
      conv_backward_data_t<float>(c, d, W, DY, DX, stream, G ? reinterpret_cast<const float*>(G->dev) : nullptr);
    else if (W.dtype == CDNN_F64)
      conv_backward_data_t<double>(c, d, W, DY, DX, stream, G ? reinterpret_cast<const double*>(G->dev) : nullptr);
    else fail(CDNN_INVALID_ARGUMENT, "conv_bwd_data: floating buffers required");
  });
}

int cdnn_conv_backward_filter(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle dy, cdnn_handle dw,
                              cdnn_handle db, cdnn_handle stream) {
  return cdnn_conv_backward_filter_ex(ctx, desc, x, dy, dw, db, 0, stream);
}

int cdnn_conv_backward_filter_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle dy, cdnn_handle dw,
                                 cdnn_handle db, int flags, cdnn_handle stream) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    const ConvDescSlot& d = conv_desc(c, desc);
    BufferSlot& X = buffer(c, x, "conv_bwd_filter x");
    BufferSlot& DY = buffer(c, dy, "conv_bwd_filter dy");
    BufferSlot* DW = buffer_or_null(c, dw, "conv_bwd_filter dw");
    BufferSlot* DB = buffer_or_null(c, db, "conv_bwd_filter db");
    const auto& g = d.geom;
    require_len(X, uint64_t(g.N) * g.C * g.H * g.W, "conv_bwd_filter x");
    require_len(DY, uint64_t(g.N) * g.Co * g.P * g.Q, "conv_bwd_filter dy");
    if (DW) { require_len(*DW, uint64_t(g.Co) * d.Kc, "conv_bwd_filter dw"); require_dtype(*DW, X.dtype, "conv dw"); }
    if (DB) { require_len(*DB, uint64_t(g.Co), "conv_bwd_filter db"); require_dtype(*DB, X.dtype, "conv db"); }
    require_dtype(DY, X.dtype, "conv_bwd_filter");
    DeviceGuard dg(c);
    const bool unchanged = (flags & CDNN_CONV_INPUT_UNCHANGED) != 0;
    if (X.dtype == CDNN_F32) conv_backward_filter_t<float>(c, d, X, DY, DW, DB, stream, unchanged);
    else if (X.dtype == CDNN_F64) conv_backward_filter_t<double>(c, d, X, DY, DW, DB, stream, unchanged);
    else fail(CDNN_INVALID_ARGUMENT, "conv_bwd_filter: floating buffers required");
  });
}

}  // extern "C"
