// polegrad/layers.hpp — layer interface, factory and the concrete layers.
//
// The Layer virtual interface, the six reference layer types with their
// parameter structs and accessors, make_layer and softmax_xent_gradient keep
// the reference signatures (layers.hpp:16-193).  Forward/backward now run on
// the GPU through the CudaDnn C-ABI.  Added (Caffe semantics, absent from the
// reference — SURVEY §8(a) X1-X5): Convolution, Pooling, SoftmaxWithLoss,
// Split, and a labelled MemoryData top.  Their parameters are read from the
// layer's opaque prototxt blocks (convolution_param, pooling_param,
// loss_param), so prototxt parse/print is unchanged.
//
// Setting the environment variable POLEGRAD_REFERENCE_COMPAT=1 hides the
// added layer types from layer_type_from_string (and therefore from the
// parser) and restores the reference's wiring rules in Net, so the
// reference's own test-suite assertions that "Convolution" is unknown hold.
#pragma once

#include <deque>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "polegrad/blob.hpp"
#include "polegrad/proto_node.hpp"
#include "polegrad/types.hpp"

namespace polegrad {

enum class LayerType {
  kInnerProduct,
  kRelu,
  kSigmoid,
  kSoftmax,
  kMemoryData,
  kMemoryLoss,
  // B200 additions (Caffe layer set needed by the CNN configs)
  kConvolution,
  kPooling,
  kSoftmaxWithLoss,
  kSplit,
  kLRN,
  kDropout,
  kBatchNorm,
  kScale,
  kEltwise,
};

std::string_view to_string(LayerType type);
std::optional<LayerType> layer_type_from_string(std::string_view name);
// True when POLEGRAD_REFERENCE_COMPAT is set (reference layer set and rules).
bool reference_compat();

struct InnerProductParam {
  int num_output = 0;
  std::vector<ProtoNode> extras;  // unrecognised fields, printed back verbatim
  bool operator==(const InnerProductParam&) const = default;
};

struct MemoryDataParam {
  int batch_size = 0;
  int channels = 0;
  int height = 0;
  int width = 0;
  std::vector<ProtoNode> extras;
  bool operator==(const MemoryDataParam&) const = default;
};

struct LayerSpec {
  std::string name;
  LayerType type = LayerType::kInnerProduct;
  std::vector<std::string> bottoms;
  std::vector<std::string> tops;
  std::optional<InnerProductParam> inner_product;
  std::optional<MemoryDataParam> memory_data;
  std::vector<ProtoNode> extras;
  bool operator==(const LayerSpec&) const = default;
};

// Backward-time callback of MemoryLoss: fills the gradient of its bottom.
using LossHook = std::function<void(Blob& bottom)>;

class Layer {
 public:
  explicit Layer(LayerSpec spec) : spec_(std::move(spec)) {}
  virtual ~Layer() = default;
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;

  const LayerSpec& spec() const { return spec_; }
  const std::string& name() const { return spec_.name; }
  LayerType type() const { return spec_.type; }

  // Checks bottom shapes, allocates and initialises parameters, returns tops.
  virtual std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes,
                                   const std::shared_ptr<Registry>& registry, Rng& rng) = 0;
  virtual void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) = 0;
  // Parameter gradients accumulate; bottom gradients are overwritten.
  virtual void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) = 0;
  virtual const std::vector<std::shared_ptr<Blob>>& params() const;
  virtual void set_loss_hook(LossHook hook);  // MemoryLoss only

  // B200: which bottoms need a gradient (Caffe propagate_down).  The six
  // reference layers always write their bottom diff, as the reference does.
  void set_propagate_down(std::vector<bool> pd) { propagate_down_ = std::move(pd); }
  bool propagate_down(std::size_t i) const { return i >= propagate_down_.size() || propagate_down_[i]; }
  // True when forward() may be captured into a CUDA graph (no host work).
  virtual bool graph_safe() const { return true; }
  // B200: backward() split into two independent halves that Net may run on two
  // streams (parameter gradients || bottom gradient).  Only layers that return
  // true implement them; backward() stays their sequential composition.
  virtual bool can_split_backward() const { return false; }
  virtual void backward_weights(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
    (void)tops;
    (void)bottoms;
  }
  virtual void backward_inputs(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
    (void)tops;
    (void)bottoms;
  }
  // B200: set by Net when a later layer rewrites this layer's top (top_clobbered)
  // or its bottom 0 (bottom_clobbered, including this layer itself running in
  // place) before backward reads it; layers whose backward needs that data keep
  // a private copy (Caffe BatchNorm x_norm_, Scale temp_).
  void set_clobbered(bool top, bool bottom) { top_clobbered_ = top; bottom_clobbered_ = bottom; }
  // B200: set by Net when this layer's backward also applies the backward of the
  // in-place ReLU on its bottom 0 (dx = bottom data > 0 ? dx : 0, layers.cpp:188-195
  // semantics); that ReLU's own backward pass then does not run.
  virtual bool supports_relu_gate() const { return false; }
  void set_relu_gate(bool on) { relu_gate_ = on; }

 protected:
  LayerSpec spec_;
  std::vector<bool> propagate_down_;
  bool top_clobbered_ = false, bottom_clobbered_ = false;
  bool relu_gate_ = false;
};

std::unique_ptr<Layer> make_layer(const LayerSpec& spec);
// LRN / Dropout / BatchNorm / Scale / Eltwise from their prototxt param blocks.
std::unique_ptr<Layer> make_caffe_layer(const LayerSpec& spec);

// ---- reference layer set -------------------------------------------------------

// top = bottom W^T + b (W: num_output x C*H*W, uniform Xavier init).
class InnerProductLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<std::shared_ptr<Blob>>& params() const override { return params_; }
  bool can_split_backward() const override { return true; }
  void backward_weights(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  void backward_inputs(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  Blob& weight() { return *params_[0]; }
  Blob& bias() { return *params_[1]; }
  // Fuse a following in-place ReLU into the GEMM epilogue (set by Net).
  void fuse_relu(bool on) { fused_relu_ = on; }
  bool fused_relu() const { return fused_relu_; }

 private:
  int input_dim_ = 0;
  int num_output_ = 0;
  bool fused_relu_ = false;
  std::vector<std::shared_ptr<Blob>> params_;
};

class ReluLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // Forward already applied by the producer's epilogue (in-place fusion).
  void set_forward_fused(bool on) { forward_fused_ = on; }
  // Backward applied by the consumer's backward (Layer::set_relu_gate).
  void set_backward_fused(bool on) { backward_fused_ = on; }

 private:
  bool forward_fused_ = false;
  bool backward_fused_ = false;
};

class SigmoidLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
};

// Softmax over each sample's whole C*H*W vector; backward is the full Jacobian.
class SoftmaxLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
};

// Input feed.  Reference behaviour: a FIFO of single samples, each forward
// consumes batch_size of them (DataStarvation otherwise).  B200 additions: an
// optional second `label` top, and set_batch() which stages a whole batch
// (data + labels) straight into HBM from host memory (pinned for async).
class MemoryDataLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  bool graph_safe() const override { return false; }

  void enqueue(std::span<const real> sample);
  std::size_t queued() const { return queue_.size(); }
  std::size_t sample_size() const { return sample_size_; }
  int batch_size() const { return batch_size_; }
  // Copies batch_size samples (and labels when the layer has a label top)
  // into the top blobs asynchronously; they are consumed by the next forward
  // instead of the FIFO.
  void set_batch(Blob& data_top, Blob* label_top, const real* data, const real* labels);
  // device-resident batch: `staged` holds the data then the labels (see Net::set_batch_device)
  void set_batch_device(Blob& data_top, Blob* label_top, cdnn_handle staged);
  bool has_staged_batch() const { return staged_; }
  void clear_staged() { staged_ = false; }
  void mark_staged() { staged_ = true; }

 private:
  std::size_t sample_size_ = 0;
  int batch_size_ = 0;
  std::deque<std::vector<real>> queue_;
  bool staged_ = false;
};

// Sink of the graph; backward calls the installed hook (host side).
class MemoryLossLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  void set_loss_hook(LossHook hook) override { hook_ = std::move(hook); }
  bool has_loss_hook() const { return static_cast<bool>(hook_); }
  bool graph_safe() const override { return !hook_; }

 private:
  LossHook hook_;
};

// ---- B200 additions ---------------------------------------------------------------

struct ConvolutionParam {
  int num_output = 0;
  int kernel_h = 0, kernel_w = 0;
  int stride_h = 1, stride_w = 1;
  int pad_h = 0, pad_w = 0;
  int dilation = 1;
  int group = 1;
  bool bias_term = true;
};
ConvolutionParam parse_convolution_param(const LayerSpec& spec);

// Caffe convolution as implicit GEMMs on the tensor cores (no im2col buffer).
// Weights [num_output][C/group][kh][kw]; uniform Xavier init with the
// InnerProduct rule on the [num_output x C/group*kh*kw] view; bias zero.
class ConvolutionLayer final : public Layer {
 public:
  ConvolutionLayer(LayerSpec spec, ConvolutionParam p) : Layer(std::move(spec)), p_(p) {}
  ~ConvolutionLayer() override;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<std::shared_ptr<Blob>>& params() const override { return params_; }
  const ConvolutionParam& param() const { return p_; }
  bool can_split_backward() const override { return propagate_down(0); }
  void backward_weights(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  void backward_inputs(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // Fuse a following in-place ReLU into the convolution epilogue (set by Net).
  void fuse_relu(bool on) { fused_relu_ = on; }
  bool supports_relu_gate() const override { return true; }

 private:
  cdnn_handle fwd_input_ = 0;  // bottom data of the last forward
  ConvolutionParam p_;
  std::shared_ptr<Registry> reg_;
  cdnn_handle desc_ = 0;
  bool fused_relu_ = false;
  std::vector<std::shared_ptr<Blob>> params_;
};

struct PoolingParam {
  bool max = true;  // MAX or AVE
  int kernel_h = 0, kernel_w = 0;
  int stride_h = 1, stride_w = 1;
  int pad_h = 0, pad_w = 0;
  bool global_pooling = false;
};
PoolingParam parse_pooling_param(const LayerSpec& spec);

// Caffe pooling (ceil output size); MAX keeps an int32 argmax mask.
class LRNLayer;
class PoolingLayer final : public Layer {
 public:
  PoolingLayer(LayerSpec spec, PoolingParam p) : Layer(std::move(spec)), p_(p) {}
  ~PoolingLayer() override;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // Flat h*W+w argmax per output element (MAX only); downloads from HBM.
  std::vector<int> mask() const;
  bool supports_relu_gate() const override { return true; }
  // Fuse a following in-place ReLU into the pooling output (set by Net).
  void fuse_relu(bool on) { fused_relu_ = on; }
  // The LRN producing this layer's bottom runs inside this layer's forward
  // (cdnn_lrn_pool_forward, reading the LRN's bottom `lrn_bottom`), and this
  // layer's backward runs inside the LRN's (set by Net, see LRNLayer::fuse_pool).
  void fuse_lrn(const LRNLayer* lrn, Blob* lrn_bottom) { fused_lrn_ = lrn; lrn_bottom_ = lrn_bottom; }
  bool is_max() const { return p_.max; }
  cdnn_handle desc() const { return desc_; }
  cdnn_handle mask_handle() const { return mask_; }
  bool relu_fused() const { return fused_relu_; }

 private:
  bool fused_relu_ = false;
  const LRNLayer* fused_lrn_ = nullptr;
  Blob* lrn_bottom_ = nullptr;
  PoolingParam p_;
  std::shared_ptr<Registry> reg_;
  cdnn_handle desc_ = 0;
  cdnn_handle mask_ = 0;  // I32 device buffer
  std::size_t top_count_ = 0;
};

// softmax + multinomial logistic loss; bottoms {scores, label}, top {loss}.
// loss = -sum_n log(max(p[n][label_n], FLT_MIN)) / N  (normalize, default)
class SoftmaxWithLossLayer final : public Layer {
 public:
  SoftmaxWithLossLayer(LayerSpec spec, bool normalize) : Layer(std::move(spec)), normalize_(normalize) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const Blob& prob() const { return *prob_; }
  // Extra factor on the gradient (1/nranks under data parallelism, so the
  // sum all-reduce of per-rank normalised gradients is the global mean).
  void set_loss_scale(double s) { loss_scale_ = s; }

 private:
  double loss_scale_ = 1.0;
  bool normalize_;
  int rows_ = 0, classes_ = 0;
  std::unique_ptr<Blob> prob_;
};

// Fan-out: tops are copies of the bottom; bottom diff = sum of top diffs.
class SplitLayer final : public Layer {
 public:
  using Layer::Layer;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // the one-pass backward (<= 8 tops) can gate its sum by the bottom's data
  bool supports_relu_gate() const override { return spec_.tops.size() <= 8; }
};

// ---- configs 4-5 (AlexNet, ResNet-20), Caffe semantics -------------

// LRN ACROSS_CHANNELS (lrn_param: local_size 5, alpha 1, beta 0.75, k 1 defaults).
class LRNLayer final : public Layer {
 public:
  LRNLayer(LayerSpec spec, int size, double alpha, double beta, double k)
      : Layer(std::move(spec)), size_(size), alpha_(alpha), beta_(beta), k_(k) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  bool supports_relu_gate() const override { return true; }
  // LRN -> MAX Pooling fusion (set by Net when the pooling is this layer's only
  // consumer and cdnn_lrn_pool_supported): this forward does nothing (the
  // pooling's forward computes both tops), and this backward takes the pooled
  // top's diff and mask directly (cdnn_lrn_pool_backward); the LRN top's diff and
  // the scale tensor are then never materialised.
  void fuse_pool(const PoolingLayer* pool, Blob* pool_top) { fused_pool_ = pool; pool_top_ = pool_top; }
  int size() const { return size_; }
  double alpha() const { return alpha_; }
  double beta() const { return beta_; }
  double k() const { return k_; }

 private:
  const PoolingLayer* fused_pool_ = nullptr;
  Blob* pool_top_ = nullptr;
  int size_;
  double alpha_, beta_, k_;
  int n_ = 0, c_ = 0, hw_ = 0;
  std::unique_ptr<Blob> scale_;
};

// Dropout (training): counter-hash mask (cdnn_dropout), seed drawn from the net
// Rng at setup, device-side iteration counter advanced by every forward, so a
// replayed CUDA graph draws a fresh mask each step.  In place allowed.
class DropoutLayer final : public Layer {
 public:
  DropoutLayer(LayerSpec spec, double ratio) : Layer(std::move(spec)), ratio_(ratio) {}
  ~DropoutLayer() override;
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // Device iteration counter (one F64) the mask hash reads; Net saves / restores it
  // around steps that must not advance the mask sequence (feed-ring warm-up).
  cdnn_handle counter() const { return counter_; }

 private:
  double ratio_;
  std::uint64_t seed_ = 0;
  std::shared_ptr<Registry> reg_;
  cdnn_handle counter_ = 0;
};

// BatchNorm with mini-batch statistics (use_global_stats false); no affine part
// (Caffe pairs it with Scale).  In place allowed.
class ScaleLayer;
class BatchNormLayer final : public Layer {
 public:
  BatchNormLayer(LayerSpec spec, double eps) : Layer(std::move(spec)), eps_(eps) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // Fuse the following Scale layer (set by Net): forward writes the Scale's top
  // z = gamma*xnorm + beta directly, backward reads its top diff and produces the
  // Scale's parameter gradients too (one reduction pass each way).
  void fuse_scale(ScaleLayer* scale, Blob* scale_top) { fused_ = scale; z_ = scale_top; }
  // ... and an in-place ReLU on the Scale's top (set by Net): z is stored clamped at 0
  void fuse_relu(bool on) { fused_relu_ = on; }

 private:
  bool fused_relu_ = false;
  ScaleLayer* fused_ = nullptr;
  Blob* z_ = nullptr;
  double eps_;
  int n_ = 0, c_ = 0, hw_ = 0;
  std::unique_ptr<Blob> mean_, invstd_, scratch_;
  std::unique_ptr<Blob> xnorm_;  // private y when the top is rewritten later
};

// Scale along axis 1 with learnable gamma (filled with 1) and optional beta (0).
class ScaleLayer final : public Layer {
 public:
  ScaleLayer(LayerSpec spec, bool bias) : Layer(std::move(spec)), bias_(bias) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<std::shared_ptr<Blob>>& params() const override { return params_; }
  // Forward/backward done by the preceding BatchNorm (BatchNormLayer::fuse_scale).
  void set_fused(bool on) { fused_ = on; }
  Blob& gamma() { return *params_[0]; }
  Blob* beta() { return bias_ ? params_[1].get() : nullptr; }

 private:
  bool fused_ = false;
  bool bias_;
  int n_ = 0, c_ = 0, hw_ = 0;
  std::unique_ptr<Blob> x_;  // private input copy when in place / rewritten
  std::vector<std::shared_ptr<Blob>> params_;
};

// Eltwise SUM with optional per-bottom coefficients.
class EltwiseLayer final : public Layer {
 public:
  EltwiseLayer(LayerSpec spec, std::vector<double> coeff) : Layer(std::move(spec)), coeff_(std::move(coeff)) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottom_shapes, const std::shared_ptr<Registry>& registry,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  // a plain sum (every coefficient 1) of at most 8 bottoms: one pass, ReLU-fusable
  bool unit_sum() const;
  // an in-place ReLU on the top, applied by the one-pass sum (set by Net)
  void fuse_relu(bool on) { fused_relu_ = on; }

 private:
  std::vector<double> coeff_;
  bool fused_relu_ = false;
};

// Cross-entropy gradient at a softmax output: probs - one-hot target
// (validated: same length, non-empty, probs sum to 1 within 1e-6, one-hot).
std::vector<real> softmax_xent_gradient(std::span<const real> probs, std::span<const real> target);

}  // namespace polegrad
