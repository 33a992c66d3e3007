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
#include "launch.cuh"

namespace cdnn {
namespace {

template <typename T>
void conv_forward_t(Ctx* c, const ConvDescSlot& d, const BufferSlot& X, const BufferSlot& Wt,
                    const BufferSlot* B, BufferSlot& Y, cdnn_handle stream) {
  const ConvGeom& g = d.geom;
  cudaStream_t st = stream_of(c, stream);
  Workspace& ws = workspace_of(c, stream);
  const int M = g.N * g.P * g.Q, N = g.Cog, K = d.Kc;
  for (int grp = 0; grp < g.group; ++grp) {
    const T* x = reinterpret_cast<const T*>(X.dev) + int64_t(grp) * g.Cg * g.H * g.W;
    const T* w = reinterpret_cast<const T*>(Wt.dev) + int64_t(grp) * g.Cog * K;
    ConvFwdA<T> va{x, d.taps, g, M, K};
    DenseView<T> vb{w, int64_t(K), 1, N, K, false};
    ConvFwdEpi<T> epi{reinterpret_cast<T*>(Y.dev) + int64_t(grp) * g.Cog * g.P * g.Q,
                      B ? reinterpret_cast<const T*>(B->dev) + grp * g.Cog : nullptr, g};
    if constexpr (std::is_same_v<T, float>) {
      const GemmPlan pl = plan_tc(M, N, K);
      TmaReq rb;
      with_operand(c, vb, pl.bn, rb, [&](const auto& b) { run_tc(c, st, ws, pl, M, N, K, va, b, epi, TmaReq{}, rb); });
    } else {
      run_simt<T>(c, st, ws, plan_simt(M, N, K), M, N, K, va, vb, epi);
    }
  }
}

template <typename T>
void conv_backward_data_t(Ctx* c, const ConvDescSlot& d, const BufferSlot& Wt, const BufferSlot& DY,
                          BufferSlot& DX, cdnn_handle stream) {
  const ConvGeom& g = d.geom;
  cudaStream_t st = stream_of(c, stream);
  Workspace& ws = workspace_of(c, stream);
  const int M = g.N * g.H * g.W, N = g.Cg, K = d.Kd;
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
                            BufferSlot* DW, BufferSlot* DB, cdnn_handle stream) {
  const ConvGeom& g = d.geom;
  cudaStream_t st = stream_of(c, stream);
  Workspace& ws = workspace_of(c, stream);
  if (!DW && !DB) return;
  // rows = taps (+1 all-ones row when the bias gradient is wanted)
  const int Kc = d.Kc, M = Kc + (DB ? 1 : 0), N = g.Cog, K = g.N * g.P * g.Q;
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
    if (X.dtype == CDNN_F32) conv_forward_t<float>(c, d, X, W, B, Y, stream);
    else if (X.dtype == CDNN_F64) conv_forward_t<double>(c, d, X, W, B, Y, stream);
    else fail(CDNN_INVALID_ARGUMENT, "conv: floating buffers required");
  });
}

int cdnn_conv_backward_data(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle w, cdnn_handle dy, cdnn_handle dx,
                            cdnn_handle stream) {
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
    DeviceGuard dg(c);
    if (W.dtype == CDNN_F32) conv_backward_data_t<float>(c, d, W, DY, DX, stream);
    else if (W.dtype == CDNN_F64) conv_backward_data_t<double>(c, d, W, DY, DX, stream);
    else fail(CDNN_INVALID_ARGUMENT, "conv_bwd_data: floating buffers required");
  });
}

int cdnn_conv_backward_filter(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle dy, cdnn_handle dw,
                              cdnn_handle db, cdnn_handle stream) {
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
    if (X.dtype == CDNN_F32) conv_backward_filter_t<float>(c, d, X, DY, DW, DB, stream);
    else if (X.dtype == CDNN_F64) conv_backward_filter_t<double>(c, d, X, DY, DW, DB, stream);
    else fail(CDNN_INVALID_ARGUMENT, "conv_bwd_filter: floating buffers required");
  });
}

}  // extern "C"
