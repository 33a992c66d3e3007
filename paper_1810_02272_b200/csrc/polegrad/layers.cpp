// layers.cpp — the reference layer set on the GPU (reference: layers.cpp).
//
// Every forward/backward is a CudaDnn C-ABI call on device-resident blobs;
// setup() keeps the reference's host-side parameter init (same Rng draws in
// the same order, layers.cpp:116-119) so initial weights are bit-identical.
#include "polegrad/layers.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>

#include "polegrad/errors.hpp"

namespace polegrad {

bool reference_compat() {
  static const bool on = [] {
    const char* v = std::getenv("POLEGRAD_REFERENCE_COMPAT");
    return v && *v && std::string(v) != "0";
  }();
  return on;
}

std::string_view to_string(LayerType type) {
  switch (type) {
    case LayerType::kInnerProduct: return "InnerProduct";
    case LayerType::kRelu: return "ReLU";
    case LayerType::kSigmoid: return "Sigmoid";
    case LayerType::kSoftmax: return "Softmax";
    case LayerType::kMemoryData: return "MemoryData";
    case LayerType::kMemoryLoss: return "MemoryLoss";
    case LayerType::kConvolution: return "Convolution";
    case LayerType::kPooling: return "Pooling";
    case LayerType::kSoftmaxWithLoss: return "SoftmaxWithLoss";
    case LayerType::kSplit: return "Split";
    case LayerType::kLRN: return "LRN";
    case LayerType::kDropout: return "Dropout";
    case LayerType::kBatchNorm: return "BatchNorm";
    case LayerType::kScale: return "Scale";
    case LayerType::kEltwise: return "Eltwise";
  }
  return "?";
}

std::optional<LayerType> layer_type_from_string(std::string_view name) {
  static constexpr LayerType kReference[] = {LayerType::kInnerProduct, LayerType::kRelu, LayerType::kSigmoid,
                                             LayerType::kSoftmax, LayerType::kMemoryData, LayerType::kMemoryLoss};
  static constexpr LayerType kAdded[] = {LayerType::kConvolution, LayerType::kPooling, LayerType::kSoftmaxWithLoss,
                                         LayerType::kSplit,       LayerType::kLRN,     LayerType::kDropout,
                                         LayerType::kBatchNorm,   LayerType::kScale,   LayerType::kEltwise};
  for (LayerType t : kReference)
    if (to_string(t) == name) return t;
  if (!reference_compat())
    for (LayerType t : kAdded)
      if (to_string(t) == name) return t;
  return std::nullopt;
}

const std::vector<std::shared_ptr<Blob>>& Layer::params() const {
  static const std::vector<std::shared_ptr<Blob>> kNone;
  return kNone;
}

void Layer::set_loss_hook(LossHook) {
  throw ModelError("layer '" + spec_.name + "': loss hooks require a MemoryLoss layer");
}

namespace {

void require_one_bottom(const LayerSpec& spec, const std::vector<Shape>& shapes) {
  if (shapes.size() != 1) throw ModelError("layer '" + spec.name + "': expected exactly one bottom shape");
}

struct Arity {
  std::size_t bottoms_min, bottoms_max, tops_min, tops_max;
};

Arity arity_of(LayerType t) {
  switch (t) {
    case LayerType::kMemoryData: return {0, 0, 1, reference_compat() ? 1u : 2u};
    case LayerType::kMemoryLoss: return {1, 1, 0, 0};
    case LayerType::kSoftmaxWithLoss: return {2, 2, 1, 1};
    case LayerType::kSplit: return {1, 1, 1, 64};
    case LayerType::kEltwise: return {2, 64, 1, 1};
    default: return {1, 1, 1, 1};
  }
}

}  // namespace

std::unique_ptr<Layer> make_layer(const LayerSpec& spec) {
  const Arity a = arity_of(spec.type);
  const std::size_t nb = spec.bottoms.size(), nt = spec.tops.size();
  if (nb < a.bottoms_min || nb > a.bottoms_max || nt < a.tops_min || nt > a.tops_max) {
    throw ModelError("layer '" + spec.name + "' (" + std::string(to_string(spec.type)) + "): expected " +
                     std::to_string(a.bottoms_min) + " bottom(s) and " + std::to_string(a.tops_min) +
                     " top(s), got " + std::to_string(nb) + " and " + std::to_string(nt));
  }
  switch (spec.type) {
    case LayerType::kInnerProduct:
      if (!spec.inner_product || spec.inner_product->num_output < 1)
        throw ModelError("layer '" + spec.name + "': inner_product_param.num_output >= 1 is required");
      return std::make_unique<InnerProductLayer>(spec);
    case LayerType::kRelu: return std::make_unique<ReluLayer>(spec);
    case LayerType::kSigmoid: return std::make_unique<SigmoidLayer>(spec);
    case LayerType::kSoftmax: return std::make_unique<SoftmaxLayer>(spec);
    case LayerType::kMemoryData: {
      const auto& p = spec.memory_data;
      if (!p || p->batch_size < 1 || p->channels < 1 || p->height < 1 || p->width < 1)
        throw ModelError("layer '" + spec.name +
                         "': memory_data_param with positive batch_size, channels, height, width is required");
      return std::make_unique<MemoryDataLayer>(spec);
    }
    case LayerType::kMemoryLoss: return std::make_unique<MemoryLossLayer>(spec);
    case LayerType::kConvolution: return std::make_unique<ConvolutionLayer>(spec, parse_convolution_param(spec));
    case LayerType::kPooling: return std::make_unique<PoolingLayer>(spec, parse_pooling_param(spec));
    case LayerType::kSoftmaxWithLoss: {
      bool normalize = true;
      for (const ProtoNode& n : spec.extras)
        if (n.key == "loss_param" && n.kind == ProtoNode::Kind::kBlock)
          for (const ProtoNode& c : n.children)
            if (c.key == "normalize") normalize = c.value == "true" || c.value == "1";
      return std::make_unique<SoftmaxWithLossLayer>(spec, normalize);
    }
    case LayerType::kSplit: return std::make_unique<SplitLayer>(spec);
    case LayerType::kLRN:
    case LayerType::kDropout:
    case LayerType::kBatchNorm:
    case LayerType::kScale:
    case LayerType::kEltwise: return make_caffe_layer(spec);
  }
  throw ModelError("layer '" + spec.name + "': unhandled layer type");
}

// ---- InnerProduct (layers.cpp:102-169) -------------------------------------------

std::vector<Shape> InnerProductLayer::setup(const std::vector<Shape>& bottom_shapes,
                                            const std::shared_ptr<Registry>& registry, Rng& rng) {
  require_one_bottom(spec_, bottom_shapes);
  const Shape& b = bottom_shapes[0];
  input_dim_ = b.c() * b.h() * b.w();
  num_output_ = spec_.inner_product->num_output;
  params_.clear();
  params_.push_back(std::make_shared<Blob>(registry, Shape{{1, 1, num_output_, input_dim_}}, spec_.name + ".weight"));
  params_.push_back(std::make_shared<Blob>(registry, Shape{{1, 1, 1, num_output_}}, spec_.name + ".bias"));
  // uniform Xavier, limit sqrt(6 / (fan_in + fan_out)), row-major draw order; bias 0
  const double limit = std::sqrt(6.0 / (input_dim_ + num_output_));
  for (real& v : params_[0]->data()) v = static_cast<real>(rng.uniform(-limit, limit));
  return {Shape{{b.n(), 1, 1, num_output_}}};
}

void InnerProductLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Blob& x = *bottoms[0];
  Blob& y = *tops[0];
  Registry& reg = x.registry();
  const cdnn_handle xh = x.gpu_data(), wh = weight().gpu_data(), bh = bias().gpu_data();
  cdnn_ok(cdnn_ip_forward(reg.context(), xh, wh, bh, y.overwrite_gpu_data(), x.shape().n(), input_dim_, num_output_,
                          fused_relu_ ? 1 : 0, reg.stream()),
          "InnerProduct forward");
}

void InnerProductLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Blob& x = *bottoms[0];
  Blob& y = *tops[0];
  Registry& reg = x.registry();
  const cdnn_handle xh = x.gpu_data(), wh = weight().gpu_data(), dyh = y.gpu_diff();
  // dW += dY^T X ; db += colsum(dY) ; dX = dY W  (the reference always writes dX)
  cdnn_ok(cdnn_ip_backward(reg.context(), xh, wh, dyh, weight().mutable_gpu_diff(), bias().mutable_gpu_diff(),
                           x.overwrite_gpu_diff(), x.shape().n(), input_dim_, num_output_, reg.stream()),
          "InnerProduct backward");
}

void InnerProductLayer::backward_weights(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Blob& x = *bottoms[0];
  Registry& reg = x.registry();
  cdnn_ok(cdnn_ip_backward(reg.context(), x.gpu_data(), weight().gpu_data(), tops[0]->gpu_diff(),
                           weight().mutable_gpu_diff(), bias().mutable_gpu_diff(), 0, x.shape().n(), input_dim_,
                           num_output_, reg.stream()),
          "InnerProduct backward");
}

void InnerProductLayer::backward_inputs(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Blob& x = *bottoms[0];
  Registry& reg = x.registry();
  cdnn_ok(cdnn_ip_backward(reg.context(), x.gpu_data(), weight().gpu_data(), tops[0]->gpu_diff(), 0, 0,
                           x.overwrite_gpu_diff(), x.shape().n(), input_dim_, num_output_, reg.stream()),
          "InnerProduct backward");
}

// ---- ReLU / Sigmoid / Softmax (layers.cpp:174-266) ---------------------------------

std::vector<Shape> ReluLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  require_one_bottom(spec_, s);
  return {s[0]};
}

void ReluLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  if (forward_fused_) return;
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data();
  cdnn_ok(cdnn_relu_forward(reg.context(), x, tops[0]->overwrite_gpu_data(), bottoms[0]->count(), reg.stream()),
          "ReLU forward");
}

void ReluLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (backward_fused_) return;  // the consumer's backward applied the gate
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data(), dy = tops[0]->gpu_diff();
  cdnn_ok(cdnn_relu_backward(reg.context(), x, dy, bottoms[0]->overwrite_gpu_diff(), bottoms[0]->count(), reg.stream()),
          "ReLU backward");
}

std::vector<Shape> SigmoidLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  require_one_bottom(spec_, s);
  return {s[0]};
}

void SigmoidLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data();
  cdnn_ok(cdnn_sigmoid_forward(reg.context(), x, tops[0]->overwrite_gpu_data(), bottoms[0]->count(), reg.stream()),
          "Sigmoid forward");
}

void SigmoidLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle y = tops[0]->gpu_data(), dy = tops[0]->gpu_diff();
  cdnn_ok(cdnn_sigmoid_backward(reg.context(), y, dy, bottoms[0]->overwrite_gpu_diff(), bottoms[0]->count(),
                                reg.stream()),
          "Sigmoid backward");
}

std::vector<Shape> SoftmaxLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  require_one_bottom(spec_, s);
  return {s[0]};
}

void SoftmaxLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  const Shape& s = bottoms[0]->shape();
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle x = bottoms[0]->gpu_data();
  cdnn_ok(cdnn_softmax_forward(reg.context(), x, tops[0]->overwrite_gpu_data(), s.n(), s.c() * s.h() * s.w(),
                               reg.stream()),
          "Softmax forward");
}

void SoftmaxLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  const Shape& s = bottoms[0]->shape();
  Registry& reg = bottoms[0]->registry();
  const cdnn_handle y = tops[0]->gpu_data(), dy = tops[0]->gpu_diff();
  cdnn_ok(cdnn_softmax_backward(reg.context(), y, dy, bottoms[0]->overwrite_gpu_diff(), s.n(), s.c() * s.h() * s.w(),
                                reg.stream()),
          "Softmax backward");
}

// ---- MemoryData (layers.cpp:271-306) --------------------------------------------------

std::vector<Shape> MemoryDataLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  if (!s.empty()) throw ModelError("layer '" + spec_.name + "': MemoryData takes no bottoms");
  const MemoryDataParam& p = *spec_.memory_data;
  batch_size_ = p.batch_size;
  sample_size_ = std::size_t(p.channels) * p.height * p.width;
  std::vector<Shape> tops{Shape{{p.batch_size, p.channels, p.height, p.width}}};
  if (spec_.tops.size() == 2) tops.push_back(Shape{{p.batch_size, 1, 1, 1}});
  return tops;
}

void MemoryDataLayer::enqueue(std::span<const real> sample) {
  if (sample.size() != sample_size_) {
    throw InvalidArgument("layer '" + spec_.name + "': enqueue of " + std::to_string(sample.size()) +
                          " values, expected " + std::to_string(sample_size_));
  }
  queue_.emplace_back(sample.begin(), sample.end());
}

void MemoryDataLayer::set_batch(Blob& data_top, Blob* label_top, const real* data, const real* labels) {
  Registry& reg = data_top.registry();
  const std::size_t n = std::size_t(batch_size_) * sample_size_;
  cdnn_ok(cdnn_write_async(reg.context(), data_top.overwrite_gpu_data(), 0, data, n, reg.stream()), "set_batch data");
  if (label_top && labels)
    cdnn_ok(cdnn_write_async(reg.context(), label_top->overwrite_gpu_data(), 0, labels, std::size_t(batch_size_),
                             reg.stream()),
            "set_batch labels");
  staged_ = true;
}

void MemoryDataLayer::set_batch_device(Blob& data_top, Blob* label_top, cdnn_handle staged) {
  Registry& reg = data_top.registry();
  const std::size_t n = std::size_t(batch_size_) * sample_size_;
  cdnn_ok(cdnn_copy_range(reg.context(), staged, 0, data_top.overwrite_gpu_data(), 0, n, reg.stream()),
          "set_batch_device data");
  if (label_top)
    cdnn_ok(cdnn_copy_range(reg.context(), staged, n, label_top->overwrite_gpu_data(), 0, std::size_t(batch_size_),
                            reg.stream()),
            "set_batch_device labels");
  staged_ = true;
}

void MemoryDataLayer::forward(std::span<Blob* const>, std::span<Blob* const> tops) {
  if (staged_) {  // batch already in HBM (set_batch); consumed by this forward
    staged_ = false;
    return;
  }
  if (queue_.size() < std::size_t(batch_size_)) {
    throw DataStarvation("layer '" + spec_.name + "': queue holds " + std::to_string(queue_.size()) +
                         " sample(s), batch needs " + std::to_string(batch_size_));
  }
  std::vector<real> batch(std::size_t(batch_size_) * sample_size_);
  for (int b = 0; b < batch_size_; ++b) {
    std::copy(queue_.front().begin(), queue_.front().end(), batch.begin() + std::ptrdiff_t(b * sample_size_));
    queue_.pop_front();
  }
  Registry& reg = tops[0]->registry();
  const cdnn_handle h = tops[0]->overwrite_gpu_data();
  if (reg.stream() != 0) reg.synchronize();
  cdnn_ok(cdnn_write(reg.context(), h, batch.data(), batch.size()), "MemoryData forward");
}

void MemoryDataLayer::backward(std::span<Blob* const>, std::span<Blob* const>) {}

// ---- MemoryLoss (layers.cpp:311-323) --------------------------------------------------

std::vector<Shape> MemoryLossLayer::setup(const std::vector<Shape>& s, const std::shared_ptr<Registry>&, Rng&) {
  require_one_bottom(spec_, s);
  return {};
}

void MemoryLossLayer::forward(std::span<Blob* const>, std::span<Blob* const>) {}

void MemoryLossLayer::backward(std::span<Blob* const>, std::span<Blob* const> bottoms) {
  if (hook_) hook_(*bottoms[0]);  // host callback writes the bottom gradient
}

// ---- softmax_xent_gradient (layers.cpp:327-357) -------------------------------------

std::vector<real> softmax_xent_gradient(std::span<const real> probs, std::span<const real> target) {
  if (probs.size() != target.size()) {
    throw InvalidArgument("softmax_xent_gradient: probs length " + std::to_string(probs.size()) +
                          " != target length " + std::to_string(target.size()));
  }
  if (probs.empty()) throw InvalidArgument("softmax_xent_gradient: empty input");
  real total = 0;
  for (real p : probs) total += p;
  if (std::abs(total - real(1)) > real(1e-6))
    throw InvalidArgument("softmax_xent_gradient: probs sum to " + std::to_string(total) + ", expected 1");
  int hot = 0;
  for (real t : target) {
    if (t == real(1)) ++hot;
    else if (t != real(0)) throw InvalidArgument("softmax_xent_gradient: target is not one-hot");
  }
  if (hot != 1) throw InvalidArgument("softmax_xent_gradient: target is not one-hot");
  std::vector<real> g(probs.size());
  for (std::size_t i = 0; i < probs.size(); ++i) g[i] = probs[i] - target[i];
  return g;
}

}  // namespace polegrad
