// layers_caffe.cpp — the layers of configs 4-5 (AlexNet: LRN, Dropout;
// ResNet-20: BatchNorm, Scale, Eltwise), Caffe semantics, on the CudaDnn
// C-ABI (csrc/cudadnn/ops_layers.cu).  The reference has none of them
// (SURVEY §8(f)); the CPU oracle restates each in oracle/ext/ext_layers.cpp.
#include <algorithm>
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

double to_double(const ProtoNode& n, const LayerSpec& spec) {
  try {
    std::size_t used = 0;
    const double v = std::stod(n.value, &used);
    if (used != n.value.size()) throw std::invalid_argument("trailing");
    return v;
  } catch (const std::exception&) {
    throw ModelError("layer '" + spec.name + "': '" + n.key + "' must be a number, got '" + n.value + "'");
  }
}

bool to_bool(const ProtoNode& n) { return n.value == "true" || n.value == "1"; }

void one_bottom(const LayerSpec& spec, const std::vector<Shape>& s) {
  if (s.size() != 1) throw ModelError("layer '" + spec.name + "': expected exactly one bottom shape");
}

}  // namespace

std::unique_ptr<Layer> make_caffe_layer(const LayerSpec& spec) {
  switch (spec.type) {
    case LayerType::kLRN: {
      int size = 5;
      double alpha = 1.0, beta = 0.75, k = 1.0;
      if (const ProtoNode* b = find_block(spec, "lrn_param"))
        for (const ProtoNode& c : b->children) {
          if (c.key == "local_size") size = int(to_double(c, spec));
          else if (c.key == "alpha") alpha = to_double(c, spec);
          else if (c.key == "beta") beta = to_double(c, spec);
          else if (c.key == "k") k = to_double(c, spec);
          else if (c.key == "norm_region" && c.value != "ACROSS_CHANNELS" && c.value != "0")
            throw ModelError("layer '" + spec.name + "': only ACROSS_CHANNELS LRN is supported");
        }
      if (size < 1 || size % 2 == 0) throw ModelError("layer '" + spec.name + "': LRN local_size must be odd");
      return std::make_unique<LRNLayer>(spec, size, alpha, beta, k);
    }
    case LayerType::kDropout: {
      double ratio = 0.5;
      if (const ProtoNode* b = find_block(spec, "dropout_param"))
        for (const ProtoNode& c : b->children)
          if (c.key == "dropout_ratio") ratio = to_double(c, spec);
      if (!(ratio >= 0.0 && ratio < 1.0)) throw ModelError("layer '" + spec.name + "': dropout_ratio must be in [0, 1)");
      return std::make_unique<DropoutLayer>(spec, ratio);
    }
    case LayerType::kBatchNorm: {
      double eps = 1e-5;
      if (const ProtoNode* b = find_block(spec, "batch_norm_param"))
        for (const ProtoNode& c : b->children) {
          if (c.key == "eps") eps = to_double(c, spec);
          else if (c.key == "use_global_stats" && to_bool(c))
            throw ModelError("layer '" + spec.name + "': BatchNorm with use_global_stats is not a training layer");
        }
      return std::make_unique<BatchNormLayer>(spec, eps);
    }
    case LayerType::kScale: {
      bool bias = false;
      if (const ProtoNode* b = find_block(spec, "scale_param"))
        for (const ProtoNode& c : b->children) {
          if (c.key == "bias_term") bias = to_bool(c);
          else if ((c.key == "axis" && c.value != "1") || (c.key == "num_axes" && c.value != "1"))
            throw ModelError("layer '" + spec.name + "': Scale supports axis 1, num_axes 1");
        }
      if (spec.bottoms.size() != 1) throw ModelError("layer '" + spec.name + "': Scale takes exactly one bottom");
      return std::make_unique<ScaleLayer>(spec, bias);
    }
    case LayerType::kEltwise: {
      std::vector<double> coeff;
      if (const ProtoNode* b = find_block(spec, "eltwise_param"))
        for (const ProtoNode& c : b->children) {
          if (c.key == "operation" && c.value != "SUM" && c.value != "1")
            throw ModelError("layer '" + spec.name + "': only Eltwise SUM is supported");
          if (c.key == "coeff") coeff.push_back(to_double(c, spec));
        }
      if (!coeff.empty() && coeff.size() != spec.bottoms.size())
        throw ModelError("layer '" + spec.name + "': Eltwise needs one coeff per bottom");
      if (coeff.empty()) coeff.assign(spec.bottoms.size(), 1.0);
      return std::make_unique<EltwiseLayer>(spec, coeff);
    }
    default: break;
  }
  throw ModelError("layer '" + spec.name + "': not a Caffe extension layer");
}

// ---- LRN --------------------------------------------------------------------------------

std::vector<Shape> LRNLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry, Rng&) {
  one_bottom(spec_, s);
  n_ = s[0].n();
  c_ = s[0].c();
  hw_ = s[0].h() * s[0].w();
  scale_ = std::make_unique<Blob>(registry, s[0], spec_.name + ".scale");
  return {s[0]};
}

void LRNLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  if (top_clobbered_ || bottom_clobbered_)
    throw ModelError("layer '" + spec_.name + "': LRN data rewritten in place before backward is unsupported");
  if (fused_pool_) return;  // computed by the consuming pooling layer's forward
  Registry& reg = bottoms[0]->registry();
  cdnn_ok(cdnn_lrn_forward(reg.context(), bottoms[0]->gpu_data(), tops[0]->overwrite_gpu_data(),
                           scale_->overwrite_gpu_data(), n_, c_, hw_, size_, alpha_, beta_, k_, reg.stream()),
          "LRN forward");
}

void LRNLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down(0)) return;
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data();
  if (fused_pool_) {  // pooling backward + LRN backward in one pass (ops_lrnpool.cu)
    cdnn_ok(cdnn_lrn_pool_backward(reg.context(), fused_pool_->desc(), x, pool_top_->gpu_diff(),
                                   fused_pool_->mask_handle(), bottoms[0]->overwrite_gpu_diff(), relu_gate_ ? x : 0,
                                   size_, alpha_, beta_, k_, reg.stream()),
            "LRN + Pooling backward");
    return;
  }
  cdnn_ok(cdnn_lrn_backward_ex(reg.context(), x, tops[0]->gpu_data(), scale_->gpu_data(), tops[0]->gpu_diff(),
                               bottoms[0]->overwrite_gpu_diff(), n_, c_, hw_, size_, alpha_, beta_,
                               relu_gate_ ? x : 0, reg.stream()),
          "LRN backward");
}

// ---- Dropout ------------------------------------------------------------------------------

DropoutLayer::~DropoutLayer() {
  if (reg_ && counter_) cdnn_free(reg_->context(), counter_);
}

std::vector<Shape> DropoutLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry,
                                       Rng& rng) {
  one_bottom(spec_, s);
  reg_ = registry;
  seed_ = rng.next_u64();
  cdnn_ok(cdnn_alloc(registry->context(), 1, CDNN_F64, &counter_), "Dropout setup");
  cdnn_ok(cdnn_fill(registry->context(), counter_, 1, 0.0, registry->stream()), "Dropout setup");
  return {s[0]};
}

void DropoutLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = *reg_;
  cdnn_ok(cdnn_counter_increment(reg.context(), counter_, reg.stream()), "Dropout forward");
  const cdnn_handle x = bottoms[0]->gpu_data();
  const cdnn_handle y = tops[0] == bottoms[0] ? tops[0]->mutable_gpu_data() : tops[0]->overwrite_gpu_data();
  cdnn_ok(cdnn_dropout(reg.context(), x, y, tops[0]->count(), ratio_, seed_, counter_, reg.stream()),
          "Dropout forward");
}

void DropoutLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down(0)) return;
  Registry& reg = *reg_;
  const cdnn_handle dy = tops[0]->gpu_diff();
  const cdnn_handle dx = tops[0] == bottoms[0] ? bottoms[0]->mutable_gpu_diff() : bottoms[0]->overwrite_gpu_diff();
  cdnn_ok(cdnn_dropout(reg.context(), dy, dx, bottoms[0]->count(), ratio_, seed_, counter_, reg.stream()),
          "Dropout backward");
}

// ---- BatchNorm ----------------------------------------------------------------------------

std::vector<Shape> BatchNormLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry,
                                         Rng&) {
  one_bottom(spec_, s);
  n_ = s[0].n();
  c_ = s[0].c();
  hw_ = s[0].h() * s[0].w();
  mean_ = std::make_unique<Blob>(registry, Shape{{1, 1, 1, c_}}, spec_.name + ".mean");
  invstd_ = std::make_unique<Blob>(registry, Shape{{1, 1, 1, c_}}, spec_.name + ".invstd");
  scratch_ = std::make_unique<Blob>(registry, Shape{{1, 1, 1, 2 * c_}}, spec_.name + ".scratch");
  xnorm_ = std::make_unique<Blob>(registry, s[0], spec_.name + ".xnorm");
  return {s[0]};
}

void BatchNormLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = bottoms[0]->registry();
  if (fused_) {
    const cdnn_handle x = bottoms[0]->gpu_data();
    const cdnn_handle z = z_ == bottoms[0] ? z_->mutable_gpu_data() : z_->overwrite_gpu_data();
    Blob* beta = fused_->beta();
    cdnn_ok(cdnn_batchnorm_scale_forward_ex(reg.context(), x, xnorm_->overwrite_gpu_data(), z,
                                            mean_->overwrite_gpu_data(), invstd_->overwrite_gpu_data(),
                                            fused_->gamma().gpu_data(), beta ? beta->gpu_data() : 0, n_, c_, hw_,
                                            eps_, fused_relu_ ? CDNN_BN_RELU : 0, reg.stream()),
            "BatchNorm+Scale forward");
    (void)tops;
    return;
  }
  const cdnn_handle mean = mean_->overwrite_gpu_data(), inv = invstd_->overwrite_gpu_data();
  const bool in_place = tops[0] == bottoms[0];
  const cdnn_handle x = bottoms[0]->gpu_data();
  // keep y privately when a later layer rewrites the top before our backward
  const cdnn_handle y = top_clobbered_ ? xnorm_->overwrite_gpu_data()
                        : in_place     ? tops[0]->mutable_gpu_data()
                                       : tops[0]->overwrite_gpu_data();
  cdnn_ok(cdnn_batchnorm_forward(reg.context(), x, y, mean, inv, n_, c_, hw_, eps_, reg.stream()),
          "BatchNorm forward");
  if (top_clobbered_) {
    const cdnn_handle t = in_place ? tops[0]->mutable_gpu_data() : tops[0]->overwrite_gpu_data();
    cdnn_ok(cdnn_copy(reg.context(), y, t, tops[0]->count(), reg.stream()), "BatchNorm forward");
  }
}

void BatchNormLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Registry& reg = bottoms[0]->registry();
  if (fused_) {
    Blob* beta = fused_->beta();
    const cdnn_handle dz = z_->gpu_diff();
    const cdnn_handle dx = !propagate_down(0)   ? 0
                           : z_ == bottoms[0] ? bottoms[0]->mutable_gpu_diff()
                                              : bottoms[0]->overwrite_gpu_diff();
    cdnn_ok(cdnn_batchnorm_scale_backward(reg.context(), xnorm_->gpu_data(), invstd_->gpu_data(),
                                          fused_->gamma().gpu_data(), dz, dx, fused_->gamma().mutable_gpu_diff(),
                                          beta ? beta->mutable_gpu_diff() : 0, scratch_->overwrite_gpu_data(), n_, c_,
                                          hw_, reg.stream()),
            "BatchNorm+Scale backward");
    (void)tops;
    return;
  }
  if (!propagate_down(0)) return;
  const cdnn_handle inv = invstd_->gpu_data();
  const cdnn_handle y = top_clobbered_ ? xnorm_->gpu_data() : tops[0]->gpu_data();
  const cdnn_handle dy = tops[0]->gpu_diff();
  const cdnn_handle dx = tops[0] == bottoms[0] ? bottoms[0]->mutable_gpu_diff() : bottoms[0]->overwrite_gpu_diff();
  cdnn_ok(cdnn_batchnorm_backward(reg.context(), y, inv, dy, dx, scratch_->overwrite_gpu_data(), n_, c_, hw_,
                                  reg.stream()),
          "BatchNorm backward");
}

// ---- Scale --------------------------------------------------------------------------------

std::vector<Shape> ScaleLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>& registry, Rng&) {
  one_bottom(spec_, s);
  n_ = s[0].n();
  c_ = s[0].c();
  hw_ = s[0].h() * s[0].w();
  params_.clear();
  params_.push_back(std::make_shared<Blob>(registry, Shape{{1, 1, 1, c_}}, spec_.name + ".weight"));
  for (real& v : params_[0]->data()) v = real(1);  // Caffe scale filler default: constant 1
  if (bias_) params_.push_back(std::make_shared<Blob>(registry, Shape{{1, 1, 1, c_}}, spec_.name + ".bias"));
  x_ = std::make_unique<Blob>(registry, s[0], spec_.name + ".input");
  return {s[0]};
}

void ScaleLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  if (fused_) return;
  Registry& reg = bottoms[0]->registry();
  const bool in_place = tops[0] == bottoms[0];
  cdnn_handle x = bottoms[0]->gpu_data();
  if (in_place || bottom_clobbered_) {
    cdnn_ok(cdnn_copy(reg.context(), x, x_->overwrite_gpu_data(), x_->count(), reg.stream()), "Scale forward");
    x = x_->gpu_data();
  }
  const cdnn_handle y = in_place ? tops[0]->mutable_gpu_data() : tops[0]->overwrite_gpu_data();
  cdnn_ok(cdnn_scale_forward(reg.context(), x, params_[0]->gpu_data(), bias_ ? params_[1]->gpu_data() : 0, y, n_, c_,
                             hw_, reg.stream()),
          "Scale forward");
}

void ScaleLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (fused_) return;
  Registry& reg = bottoms[0]->registry();
  const bool in_place = tops[0] == bottoms[0];
  const cdnn_handle x = (in_place || bottom_clobbered_) ? x_->gpu_data() : bottoms[0]->gpu_data();
  const cdnn_handle dx = !propagate_down(0) ? 0
                         : in_place         ? bottoms[0]->mutable_gpu_diff()
                                            : bottoms[0]->overwrite_gpu_diff();
  cdnn_ok(cdnn_scale_backward(reg.context(), x, params_[0]->gpu_data(), tops[0]->gpu_diff(),
                              params_[0]->mutable_gpu_diff(), bias_ ? params_[1]->mutable_gpu_diff() : 0, dx, n_, c_,
                              hw_, reg.stream()),
          "Scale backward");
}

// ---- Eltwise ------------------------------------------------------------------------------

std::vector<Shape> EltwiseLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  if (s.size() < 2) throw ModelError("layer '" + spec_.name + "': Eltwise takes at least two bottoms");
  for (const Shape& b : s)
    if (!(b == s[0])) throw ModelError("layer '" + spec_.name + "': Eltwise bottoms must have equal shapes");
  return {s[0]};
}

bool EltwiseLayer::unit_sum() const {
  return coeff_.size() <= 8 && std::all_of(coeff_.begin(), coeff_.end(), [](double a) { return a == 1.0; });
}

void EltwiseLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = bottoms[0]->registry();
  const std::size_t n = tops[0]->count();
  const cdnn_handle y = tops[0]->overwrite_gpu_data();
  // plain sum (every coefficient 1, the ResNet shortcut): one pass over all bottoms with
  // the roundings of the axpby sequence below (products by 1 are exact, each partial sum
  // rounded once, in bottom order)
  if (unit_sum()) {
    cdnn_handle xs[8] = {};
    for (std::size_t k = 0; k < bottoms.size(); ++k) xs[k] = bottoms[k]->gpu_data();
    cdnn_ok(cdnn_fan_in_ex(reg.context(), xs, int(bottoms.size()), y, n, fused_relu_ ? CDNN_FAN_RELU : 0, 0,
                           reg.stream()),
            "Eltwise forward");
    return;
  }
  cdnn_ok(cdnn_axpby(reg.context(), n, coeff_[0], bottoms[0]->gpu_data(), 0.0, y, 0, reg.stream()), "Eltwise forward");
  for (std::size_t k = 1; k < bottoms.size(); ++k)
    cdnn_ok(cdnn_axpby(reg.context(), n, coeff_[k], bottoms[k]->gpu_data(), 1.0, y, 1, reg.stream()),
            "Eltwise forward");
}

void EltwiseLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Registry& reg = bottoms[0]->registry();
  const std::size_t n = tops[0]->count();
  const cdnn_handle dy = tops[0]->gpu_diff();
  if (bottoms.size() <= 8) {  // every bottom diff from one read of dy
    cdnn_handle d[8] = {};
    double a[8] = {};
    for (std::size_t k = 0; k < bottoms.size(); ++k) {
      a[k] = coeff_[k];
      d[k] = propagate_down(k) ? bottoms[k]->overwrite_gpu_diff() : 0;
    }
    cdnn_ok(cdnn_fan_out(reg.context(), dy, d, a, int(bottoms.size()), n, reg.stream()), "Eltwise backward");
    return;
  }
  for (std::size_t k = 0; k < bottoms.size(); ++k) {
    if (!propagate_down(k)) continue;
    cdnn_ok(cdnn_axpby(reg.context(), n, coeff_[k], dy, 0.0, bottoms[k]->overwrite_gpu_diff(), 0, reg.stream()),
            "Eltwise backward");
  }
}

}  // namespace polegrad
