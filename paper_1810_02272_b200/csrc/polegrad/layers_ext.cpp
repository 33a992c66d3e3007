// layers_ext.cpp — layers the reference lacks, Caffe
// semantics, on the CudaDnn C-ABI: Convolution (tcgen05 implicit GEMM),
// Pooling (MAX with int32 argmax / AVE), SoftmaxWithLoss, Split.
#include <cmath>
#include <string>

#include "polegrad/errors.hpp"
#include "polegrad/layers.hpp"

namespace polegrad {

namespace {

const ProtoNode* find_block(const LayerSpec& spec, const char* key) {
  for (const ProtoNode& n : spec.extras)
    if (n.key == key && n.kind == ProtoNode::Kind::kBlock) return &n;
  return nullptr;
}

int to_int(const ProtoNode& n, const LayerSpec& spec) {
  try {
    std::size_t used = 0;
    const int v = std::stoi(n.value, &used);
    if (used != n.value.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw ModelError("layer '" + spec.name + "': '" + n.key + "' must be an integer, got '" + n.value + "'");
  }
}

bool to_bool(const ProtoNode& n) { return n.value == "true" || n.value == "1"; }

}  // namespace

ConvolutionParam parse_convolution_param(const LayerSpec& spec) {
  ConvolutionParam p;
  const ProtoNode* b = find_block(spec, "convolution_param");
  if (!b) throw ModelError("layer '" + spec.name + "': convolution_param is required");
  int ks[2] = {0, 0}, nks = 0, st[2] = {1, 1}, nst = 0, pd[2] = {0, 0}, npd = 0;
  for (const ProtoNode& c : b->children) {
    if (c.kind == ProtoNode::Kind::kBlock) continue;  // weight_filler, bias_filler, ...
    if (c.key == "num_output") p.num_output = to_int(c, spec);
    else if (c.key == "kernel_size" && nks < 2) ks[nks++] = to_int(c, spec);
    else if (c.key == "kernel_h") p.kernel_h = to_int(c, spec);
    else if (c.key == "kernel_w") p.kernel_w = to_int(c, spec);
    else if (c.key == "stride" && nst < 2) st[nst++] = to_int(c, spec);
    else if (c.key == "stride_h") p.stride_h = to_int(c, spec);
    else if (c.key == "stride_w") p.stride_w = to_int(c, spec);
    else if (c.key == "pad" && npd < 2) pd[npd++] = to_int(c, spec);
    else if (c.key == "pad_h") p.pad_h = to_int(c, spec);
    else if (c.key == "pad_w") p.pad_w = to_int(c, spec);
    else if (c.key == "dilation") p.dilation = to_int(c, spec);
    else if (c.key == "group") p.group = to_int(c, spec);
    else if (c.key == "bias_term") p.bias_term = to_bool(c);
  }
  // Caffe: repeated kernel_size/stride/pad give (h, w); a single value applies to both
  if (nks) { p.kernel_h = ks[0]; p.kernel_w = nks == 2 ? ks[1] : ks[0]; }
  if (nst) { p.stride_h = st[0]; p.stride_w = nst == 2 ? st[1] : st[0]; }
  if (npd) { p.pad_h = pd[0]; p.pad_w = npd == 2 ? pd[1] : pd[0]; }
  if (p.num_output < 1 || p.kernel_h < 1 || p.kernel_w < 1 || p.stride_h < 1 || p.stride_w < 1 || p.pad_h < 0 ||
      p.pad_w < 0 || p.group < 1 || p.dilation < 1)
    throw ModelError("layer '" + spec.name + "': convolution_param needs positive num_output and kernel size");
  return p;
}

PoolingParam parse_pooling_param(const LayerSpec& spec) {
  PoolingParam p;
  const ProtoNode* b = find_block(spec, "pooling_param");
  if (!b) throw ModelError("layer '" + spec.name + "': pooling_param is required");
  for (const ProtoNode& c : b->children) {
    if (c.kind == ProtoNode::Kind::kBlock) continue;
    if (c.key == "pool") {
      if (c.value == "MAX" || c.value == "0") p.max = true;
      else if (c.value == "AVE" || c.value == "1") p.max = false;
      else throw ModelError("layer '" + spec.name + "': unsupported pool method '" + c.value + "'");
    } else if (c.key == "kernel_size") p.kernel_h = p.kernel_w = to_int(c, spec);
    else if (c.key == "kernel_h") p.kernel_h = to_int(c, spec);
    else if (c.key == "kernel_w") p.kernel_w = to_int(c, spec);
    else if (c.key == "stride") p.stride_h = p.stride_w = to_int(c, spec);
    else if (c.key == "stride_h") p.stride_h = to_int(c, spec);
    else if (c.key == "stride_w") p.stride_w = to_int(c, spec);
    else if (c.key == "pad") p.pad_h = p.pad_w = to_int(c, spec);
    else if (c.key == "pad_h") p.pad_h = to_int(c, spec);
    else if (c.key == "pad_w") p.pad_w = to_int(c, spec);
    else if (c.key == "global_pooling") p.global_pooling = to_bool(c);
  }
  if (!p.global_pooling && (p.kernel_h < 1 || p.kernel_w < 1))
    throw ModelError("layer '" + spec.name + "': pooling_param needs kernel_size or global_pooling");
  return p;
}

// ---- Convolution --------------------------------------------------------------------

ConvolutionLayer::~ConvolutionLayer() {
  if (reg_ && desc_) cdnn_desc_free(reg_->context(), desc_);
}

std::vector<Shape> ConvolutionLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry,
                                           Rng& rng) {
  if (s.size() != 1) throw ModelError("layer '" + spec_.name + "': expected exactly one bottom shape");
  reg_ = registry;
  const Shape& b = s[0];
  if (b.c() % p_.group || p_.num_output % p_.group)
    throw ModelError("layer '" + spec_.name + "': channels and num_output must be divisible by group");
  cdnn_conv_params cp{b.n(), b.c(), b.h(), b.w(), p_.num_output, p_.kernel_h, p_.kernel_w, p_.stride_h,
                      p_.stride_w, p_.pad_h, p_.pad_w, p_.dilation, p_.dilation, p_.group};
  const int st = cdnn_conv_desc_create(registry->context(), &cp, &desc_);
  if (st == CDNN_INVALID_ARGUMENT) throw ModelError("layer '" + spec_.name + "': " + cdnn_last_error());
  cdnn_ok(st, "Convolution setup");
  int out[4];
  cdnn_ok(cdnn_conv_output_shape(registry->context(), desc_, out), "Convolution setup");
  const int cg = b.c() / p_.group;
  const int kc = cg * p_.kernel_h * p_.kernel_w;
  params_.clear();
  params_.push_back(
      std::make_shared<Blob>(registry, Shape{{p_.num_output, cg, p_.kernel_h, p_.kernel_w}}, spec_.name + ".weight"));
  if (p_.bias_term)
    params_.push_back(std::make_shared<Blob>(registry, Shape{{1, 1, 1, p_.num_output}}, spec_.name + ".bias"));
  // InnerProduct's uniform Xavier on the [num_output x C/g*kh*kw] filter matrix
  const double limit = std::sqrt(6.0 / (kc + p_.num_output));
  for (real& v : params_[0]->data()) v = static_cast<real>(rng.uniform(-limit, limit));
  return {Shape{{out[0], out[1], out[2], out[3]}}};
}

void ConvolutionLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = *reg_;
  const cdnn_handle x = bottoms[0]->gpu_data(), w = params_[0]->gpu_data();
  const cdnn_handle b = p_.bias_term ? params_[1]->gpu_data() : 0;
  cdnn_ok(cdnn_conv_forward_ex(reg.context(), desc_, x, w, b, tops[0]->overwrite_gpu_data(),
                               fused_relu_ ? CDNN_CONV_RELU : 0, reg.stream()),
          "Convolution forward");
  fwd_input_ = x;
}

void ConvolutionLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  backward_weights(tops, bottoms);
  if (propagate_down(0)) backward_inputs(tops, bottoms);
}

void ConvolutionLayer::backward_weights(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Registry& reg = *reg_;
  const cdnn_handle dy = tops[0]->gpu_diff(), x = bottoms[0]->gpu_data();
  const cdnn_handle dw = params_[0]->mutable_gpu_diff();
  const cdnn_handle db = p_.bias_term ? params_[1]->mutable_gpu_diff() : 0;
  // the bottom is unchanged since this layer's forward (the net rewrites no blob a
  // convolution reads between its forward and its backward): input rewrites are reused
  const int flags = x == fwd_input_ && !bottom_clobbered_ ? CDNN_CONV_INPUT_UNCHANGED : 0;
  cdnn_ok(cdnn_conv_backward_filter_ex(reg.context(), desc_, x, dy, dw, db, flags, reg.stream()),
          "Convolution backward");
}

void ConvolutionLayer::backward_inputs(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Registry& reg = *reg_;
  const cdnn_handle w = params_[0]->gpu_data(), dy = tops[0]->gpu_diff();
  const cdnn_handle gate = relu_gate_ ? bottoms[0]->gpu_data() : 0;
  cdnn_ok(cdnn_conv_backward_data_ex(reg.context(), desc_, w, dy, bottoms[0]->overwrite_gpu_diff(), gate,
                                     reg.stream()),
          "Convolution backward");
}

// ---- Pooling ------------------------------------------------------------------------

PoolingLayer::~PoolingLayer() {
  if (reg_) {
    if (desc_) cdnn_desc_free(reg_->context(), desc_);
    if (mask_) cdnn_free(reg_->context(), mask_);
  }
}

std::vector<Shape> PoolingLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry, Rng&) {
  if (s.size() != 1) throw ModelError("layer '" + spec_.name + "': expected exactly one bottom shape");
  reg_ = registry;
  const Shape& b = s[0];
  cdnn_pool_params pp{b.n(), b.c(), b.h(), b.w(), p_.max ? CDNN_POOL_MAX : CDNN_POOL_AVE, p_.kernel_h, p_.kernel_w,
                      p_.stride_h, p_.stride_w, p_.pad_h, p_.pad_w, p_.global_pooling ? 1 : 0};
  const int st = cdnn_pool_desc_create(registry->context(), &pp, &desc_);
  if (st == CDNN_INVALID_ARGUMENT) throw ModelError("layer '" + spec_.name + "': " + cdnn_last_error());
  cdnn_ok(st, "Pooling setup");
  int out[4];
  cdnn_ok(cdnn_pool_output_shape(registry->context(), desc_, out), "Pooling setup");
  top_count_ = std::size_t(out[0]) * out[1] * out[2] * out[3];
  if (p_.max) cdnn_ok(cdnn_alloc(registry->context(), top_count_, CDNN_I32, &mask_), "Pooling setup");
  return {Shape{{out[0], out[1], out[2], out[3]}}};
}

void PoolingLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = *reg_;
  if (fused_lrn_) {  // LRN + pooling in one pass over the LRN's bottom (ops_lrnpool.cu)
    const LRNLayer& l = *fused_lrn_;
    cdnn_ok(cdnn_lrn_pool_forward(reg.context(), desc_, lrn_bottom_->gpu_data(), bottoms[0]->overwrite_gpu_data(),
                                  tops[0]->overwrite_gpu_data(), mask_, l.size(), l.alpha(), l.beta(), l.k(),
                                  fused_relu_ ? CDNN_POOL_RELU : 0, reg.stream()),
            "LRN + Pooling forward");
    return;
  }
  const cdnn_handle x = bottoms[0]->gpu_data();
  cdnn_ok(cdnn_pool_forward_ex(reg.context(), desc_, x, tops[0]->overwrite_gpu_data(), mask_,
                               fused_relu_ ? CDNN_POOL_RELU : 0, reg.stream()),
          "Pooling forward");
}

void PoolingLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down(0) || fused_lrn_) return;  // fused: runs inside LRNLayer::backward
  Registry& reg = *reg_;
  const cdnn_handle dy = tops[0]->gpu_diff();
  const cdnn_handle gate = relu_gate_ ? bottoms[0]->gpu_data() : 0;
  cdnn_ok(cdnn_pool_backward_ex(reg.context(), desc_, dy, mask_, bottoms[0]->overwrite_gpu_diff(), gate, reg.stream()),
          "Pooling backward");
}

std::vector<int> PoolingLayer::mask() const {
  std::vector<int> m(top_count_, -1);
  if (mask_) {
    reg_->synchronize();
    cdnn_ok(cdnn_read(reg_->context(), mask_, m.data(), m.size()), "Pooling mask");
  }
  return m;
}

// ---- SoftmaxWithLoss ------------------------------------------------------------------

std::vector<Shape> SoftmaxWithLossLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry,
                                               Rng&) {
  if (s.size() != 2) throw ModelError("layer '" + spec_.name + "': SoftmaxWithLoss takes {scores, label}");
  rows_ = s[0].n();
  classes_ = s[0].c() * s[0].h() * s[0].w();
  if (s[1].count() != std::size_t(rows_)) throw ModelError("layer '" + spec_.name + "': one label per sample required");
  prob_ = std::make_unique<Blob>(registry, s[0], spec_.name + ".prob");
  return {Shape{{1, 1, 1, 1}}};
}

void SoftmaxWithLossLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data(), lab = bottoms[1]->gpu_data();
  cdnn_ok(cdnn_softmax_loss_forward(reg.context(), x, lab, prob_->overwrite_gpu_data(), tops[0]->overwrite_gpu_data(),
                                    rows_, classes_, normalize_ ? 1 : 0, reg.stream()),
          "SoftmaxWithLoss forward");
}

void SoftmaxWithLossLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  (void)tops;
  if (!propagate_down(0)) return;
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle p = prob_->gpu_data(), lab = bottoms[1]->gpu_data();
  // loss weight 1 (Caffe default); kept on the host so backward is graph capturable
  cdnn_ok(cdnn_softmax_loss_backward(reg.context(), p, lab, bottoms[0]->overwrite_gpu_diff(), rows_, classes_,
                                     normalize_ ? 1 : 0, loss_scale_, reg.stream()),
          "SoftmaxWithLoss backward");
}

// ---- Split ----------------------------------------------------------------------------

std::vector<Shape> SplitLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  if (s.size() != 1) throw ModelError("layer '" + spec_.name + "': expected exactly one bottom shape");
  return std::vector<Shape>(spec_.tops.size(), s[0]);
}

void SplitLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data();
  if (tops.size() <= 8) {  // every copy from one read of x
    cdnn_handle d[8] = {};
    for (std::size_t t = 0; t < tops.size(); ++t) d[t] = tops[t]->overwrite_gpu_data();
    cdnn_ok(cdnn_fan_out(reg.context(), x, d, nullptr, int(tops.size()), bottoms[0]->count(), reg.stream()),
            "Split forward");
    return;
  }
  for (Blob* t : tops)
    cdnn_ok(cdnn_copy(reg.context(), x, t->overwrite_gpu_data(), t->count(), reg.stream()), "Split forward");
}

void SplitLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down(0)) return;
  Registry& reg = bottoms[0]->registry();
  const std::size_t n = bottoms[0]->count();
  const cdnn_handle dx = bottoms[0]->overwrite_gpu_diff();
  if (tops.size() <= 8) {  // the diffs summed in one pass (same order and roundings as copy + axpy)
    cdnn_handle d[8] = {};
    for (std::size_t t = 0; t < tops.size(); ++t) d[t] = tops[t]->gpu_diff();
    // (gated by the bottom's data when the in-place ReLU producing it has its backward fused here)
    cdnn_ok(cdnn_fan_in_ex(reg.context(), d, int(tops.size()), dx, n, 0, relu_gate_ ? bottoms[0]->gpu_data() : 0,
                           reg.stream()),
            "Split backward");
    return;
  }
  cdnn_ok(cdnn_copy(reg.context(), tops[0]->gpu_diff(), dx, n, reg.stream()), "Split backward");
  for (std::size_t t = 1; t < tops.size(); ++t)
    cdnn_ok(cdnn_axpy(reg.context(), n, 1.0, tops[t]->gpu_diff(), dx, reg.stream()), "Split backward");
}

}  // namespace polegrad
