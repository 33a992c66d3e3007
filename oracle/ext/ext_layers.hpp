// ORACLE — test infrastructure only.  Never linked into the product; only
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load it.
//
// Reference-style CPU extensions for the hot-path layers the reference
// (/root/reference/proj/core) does not have: Convolution, Pooling,
// SoftmaxWithLoss, Split and a labelled MemoryData feed, plus the momentum /
// weight-decay SGD solver.  They are written against the reference's own
// Layer / Blob / Registry interfaces (include/polegrad/layers.hpp:65-95) and
// do their arithmetic through the reference's kernels (kernels::gemm,
// backend.cpp:169-197), exactly as InnerProductLayer does (layers.cpp:124-169).
// Semantics follow Caffe (im2col convolution, ceil-mode pooling with int
// argmax masks, batch-normalised softmax loss) because the reference has
// none; parity for these is pinned by torch float64 cross-checks and
// finite-difference tests, not by reference tests.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "polegrad/blob.hpp"
#include "polegrad/layers.hpp"

namespace oracle {

using polegrad::Blob;
using polegrad::Handle;
using polegrad::LayerSpec;
using polegrad::Registry;
using polegrad::Rng;
using polegrad::Shape;
using polegrad::real;

struct ConvParam {
  int num_output = 0, kernel_h = 1, kernel_w = 1, stride_h = 1, stride_w = 1, pad_h = 0, pad_w = 0;
  int dilation_h = 1, dilation_w = 1, group = 1;
  bool bias_term = true;
};

struct PoolParam {
  bool max = true;
  int kernel_h = 1, kernel_w = 1, stride_h = 1, stride_w = 1, pad_h = 0, pad_w = 0;
  bool global = false;
};

// Layers whose bottom gradient is optional (Caffe propagate_down).  The
// reference's own six layers always write their bottom diff (layers.cpp).
class ExtLayer : public polegrad::Layer {
 public:
  using polegrad::Layer::Layer;
  std::vector<bool> propagate_down;  // set by the net before the first backward
};

class ConvolutionLayer final : public ExtLayer {
 public:
  ConvolutionLayer(LayerSpec spec, ConvParam p) : ExtLayer(std::move(spec)), p_(p) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<std::shared_ptr<Blob>>& params() const override { return params_; }

 private:
  void im2col(std::span<const real> img, std::span<real> col, int grp) const;
  void col2im(std::span<const real> col, std::span<real> img, int grp) const;
  ConvParam p_;
  int N_ = 0, C_ = 0, H_ = 0, W_ = 0, P_ = 0, Q_ = 0, Cg_ = 0, Cog_ = 0, Kc_ = 0;
  std::shared_ptr<Registry> reg_;
  std::vector<std::shared_ptr<Blob>> params_;
  Handle col_{}, wg_{}, yg_{};  // scratch buffers (reference gemm takes whole buffers)
};

class PoolingLayer final : public ExtLayer {
 public:
  PoolingLayer(LayerSpec spec, PoolParam p) : ExtLayer(std::move(spec)), p_(p) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<int>& mask() const { return mask_; }
  // test hook: replace the argmax decisions of the last forward (oracle-fed parity)
  void set_mask(const int* m) { std::copy(m, m + mask_.size(), mask_.begin()); }

 private:
  PoolParam p_;
  int N_ = 0, C_ = 0, H_ = 0, W_ = 0, PH_ = 0, PW_ = 0;
  std::vector<int> mask_;
};

class SoftmaxWithLossLayer final : public ExtLayer {
 public:
  SoftmaxWithLossLayer(LayerSpec spec, bool normalize) : ExtLayer(std::move(spec)), normalize_(normalize) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<real>& prob() const { return prob_; }

 private:
  bool normalize_;
  int rows_ = 0, classes_ = 0;
  std::vector<real> prob_;
};

class SplitLayer final : public ExtLayer {
 public:
  using ExtLayer::ExtLayer;
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
};

// ---- configs 4-5 (AlexNet, ResNet-20) — Caffe layer semantics, plain loops ----------

// LRN ACROSS_CHANNELS (Caffe lrn_layer.cpp CrossChannelForward/Backward_cpu):
// scale = k + alpha/size * sum_{c' in [c-(size-1)/2, c+(size-1)/2]} x^2 ; y = x*scale^-beta
class LRNLayer final : public ExtLayer {
 public:
  LRNLayer(LayerSpec spec, int size, double alpha, double beta, double k)
      : ExtLayer(std::move(spec)), size_(size), alpha_(alpha), beta_(beta), k_(k) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;

 private:
  int size_;
  double alpha_, beta_, k_;
  int N_ = 0, C_ = 0, HW_ = 0;
  std::vector<real> scale_;
};

// Dropout (train phase): keep iff hash(seed, iteration, i) > ratio * 2^32, kept values
// scaled by 1/(1-ratio).  The mask is a counter-based hash (same function as the CUDA
// kernel, ops_layers.cu) so oracle and device draw identical masks; seed = one draw of the
// net Rng at setup, iteration advanced at the start of every forward.
class DropoutLayer final : public ExtLayer {
 public:
  DropoutLayer(LayerSpec spec, double ratio) : ExtLayer(std::move(spec)), ratio_(ratio) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  static std::uint32_t hash(std::uint64_t seed, std::uint64_t iter, std::uint64_t idx);

 private:
  bool keep(std::size_t i) const;
  double ratio_;
  std::uint64_t seed_ = 0, iter_ = 0;
};

// BatchNorm with mini-batch statistics (use_global_stats false, Caffe batch_norm_layer.cpp):
// y = (x - mean_c) / sqrt(var_c + eps), biased variance over (N, H, W).
// Backward: dx = (dy - mean(dy) - y * mean(dy * y)) / sqrt(var + eps).
class BatchNormLayer final : public ExtLayer {
 public:
  BatchNormLayer(LayerSpec spec, double eps) : ExtLayer(std::move(spec)), eps_(eps) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;

 private:
  double eps_;
  int N_ = 0, C_ = 0, HW_ = 0;
  std::vector<real> xnorm_, invstd_;
};

// Scale (axis 1, one bottom): y = x * gamma_c (+ beta_c); gamma filled with 1, beta 0.
class ScaleLayer final : public ExtLayer {
 public:
  ScaleLayer(LayerSpec spec, bool bias) : ExtLayer(std::move(spec)), bias_(bias) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;
  const std::vector<std::shared_ptr<Blob>>& params() const override { return params_; }

 private:
  bool bias_;
  int N_ = 0, C_ = 0, HW_ = 0;
  std::vector<real> x_;  // input copy (in-place support, as Caffe's temp_)
  std::vector<std::shared_ptr<Blob>> params_;
};

// Eltwise SUM: y = sum_i coeff_i * x_i ; dx_i = coeff_i * dy.
class EltwiseLayer final : public ExtLayer {
 public:
  EltwiseLayer(LayerSpec spec, std::vector<double> coeff) : ExtLayer(std::move(spec)), coeff_(std::move(coeff)) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) override;

 private:
  std::vector<double> coeff_;
};

// Labelled batch feed: tops {data, label}; one whole batch per forward.
class LabelledDataLayer final : public ExtLayer {
 public:
  LabelledDataLayer(LayerSpec spec, int n, int c, int h, int w)
      : ExtLayer(std::move(spec)), n_(n), c_(c), h_(h), w_(w) {}
  std::vector<Shape> setup(const std::vector<Shape>& bottoms, const std::shared_ptr<Registry>& reg,
                           Rng& rng) override;
  void forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) override;
  void backward(std::span<Blob* const>, std::span<Blob* const>) override {}
  void set_batch(const double* data, const double* labels);
  int batch() const { return n_; }
  std::size_t sample_size() const { return std::size_t(c_) * h_ * w_; }

 private:
  int n_, c_, h_, w_;
  std::vector<real> data_, labels_;
  bool ready_ = false;
};

}  // namespace oracle
