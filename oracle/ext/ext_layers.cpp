// ORACLE — test infrastructure only (see ext_layers.hpp).
#include "ext_layers.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "polegrad/errors.hpp"

namespace oracle {

using polegrad::InvalidArgument;
using polegrad::ModelError;
namespace kernels = polegrad::kernels;

namespace {
void one_bottom(const LayerSpec& s, const std::vector<Shape>& b) {
  if (b.size() != 1) throw ModelError("layer '" + s.name + "': expected exactly one bottom shape");
}
// Copy n values between registry buffers at element offsets (host spans).
void copy_range(std::span<const real> src, std::size_t so, std::span<real> dst, std::size_t d0, std::size_t n) {
  std::copy(src.begin() + so, src.begin() + so + n, dst.begin() + d0);
}
}  // namespace

// ---------------------------------------------------------------------------
// Convolution: Caffe's im2col + gemm formulation, one image and group at a
// time, arithmetic through the reference kernels::gemm (backend.cpp:169-197).

std::vector<Shape> ConvolutionLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>& reg,
                                           Rng& rng) {
  one_bottom(spec_, b);
  reg_ = reg;
  N_ = b[0].n(); C_ = b[0].c(); H_ = b[0].h(); W_ = b[0].w();
  if (p_.num_output < 1 || p_.group < 1 || C_ % p_.group || p_.num_output % p_.group)
    throw ModelError("layer '" + spec_.name + "': bad convolution_param");
  const int ekh = p_.dilation_h * (p_.kernel_h - 1) + 1, ekw = p_.dilation_w * (p_.kernel_w - 1) + 1;
  P_ = (H_ + 2 * p_.pad_h - ekh) / p_.stride_h + 1;
  Q_ = (W_ + 2 * p_.pad_w - ekw) / p_.stride_w + 1;
  if (P_ < 1 || Q_ < 1) throw ModelError("layer '" + spec_.name + "': kernel larger than padded input");
  Cg_ = C_ / p_.group;
  Cog_ = p_.num_output / p_.group;
  Kc_ = Cg_ * p_.kernel_h * p_.kernel_w;
  params_.clear();
  params_.push_back(std::make_shared<Blob>(reg, Shape{{p_.num_output, Cg_, p_.kernel_h, p_.kernel_w}},
                                           spec_.name + ".weight"));
  if (p_.bias_term)
    params_.push_back(std::make_shared<Blob>(reg, Shape{{1, 1, 1, p_.num_output}}, spec_.name + ".bias"));
  // Same uniform Xavier rule as InnerProduct (layers.cpp:116-119) with the
  // filter viewed as a [num_output x Cg*kh*kw] matrix; bias stays zero.
  const double limit = std::sqrt(6.0 / (Kc_ + p_.num_output));
  for (auto& v : params_[0]->data()) v = static_cast<real>(rng.uniform(-limit, limit));
  col_ = reg->alloc_buffer(std::size_t(Kc_) * P_ * Q_);
  wg_ = reg->alloc_buffer(std::size_t(Cog_) * Kc_);
  yg_ = reg->alloc_buffer(std::size_t(Cog_) * P_ * Q_);
  return {Shape{{N_, p_.num_output, P_, Q_}}};
}

void ConvolutionLayer::im2col(std::span<const real> img, std::span<real> col, int grp) const {
  const int PQ = P_ * Q_;
  for (int c = 0; c < Cg_; ++c)
    for (int kr = 0; kr < p_.kernel_h; ++kr)
      for (int ks = 0; ks < p_.kernel_w; ++ks) {
        const int row = (c * p_.kernel_h + kr) * p_.kernel_w + ks;
        const real* plane = img.data() + std::size_t(grp * Cg_ + c) * H_ * W_;
        for (int p = 0; p < P_; ++p) {
          const int h = p * p_.stride_h - p_.pad_h + kr * p_.dilation_h;
          for (int q = 0; q < Q_; ++q) {
            const int w = q * p_.stride_w - p_.pad_w + ks * p_.dilation_w;
            col[std::size_t(row) * PQ + p * Q_ + q] =
                (h >= 0 && h < H_ && w >= 0 && w < W_) ? plane[h * W_ + w] : real(0);
          }
        }
      }
}

void ConvolutionLayer::col2im(std::span<const real> col, std::span<real> img, int grp) const {
  const int PQ = P_ * Q_;
  for (int c = 0; c < Cg_; ++c)
    for (int kr = 0; kr < p_.kernel_h; ++kr)
      for (int ks = 0; ks < p_.kernel_w; ++ks) {
        const int row = (c * p_.kernel_h + kr) * p_.kernel_w + ks;
        real* plane = img.data() + std::size_t(grp * Cg_ + c) * H_ * W_;
        for (int p = 0; p < P_; ++p) {
          const int h = p * p_.stride_h - p_.pad_h + kr * p_.dilation_h;
          if (h < 0 || h >= H_) continue;
          for (int q = 0; q < Q_; ++q) {
            const int w = q * p_.stride_w - p_.pad_w + ks * p_.dilation_w;
            if (w >= 0 && w < W_) plane[h * W_ + w] += col[std::size_t(row) * PQ + p * Q_ + q];
          }
        }
      }
}

void ConvolutionLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  Registry& reg = *reg_;
  const std::size_t PQ = std::size_t(P_) * Q_, img_in = std::size_t(C_) * H_ * W_,
                    img_out = std::size_t(p_.num_output) * PQ;
  Blob& w = *params_[0];
  for (int n = 0; n < N_; ++n) {
    for (int g = 0; g < p_.group; ++g) {
      im2col(bottoms[0]->data().subspan(n * img_in, img_in), reg.buffer(col_), g);
      Handle wh = w.data_handle();
      if (p_.group > 1) {
        copy_range(w.data(), std::size_t(g) * Cog_ * Kc_, reg.buffer(wg_), 0, std::size_t(Cog_) * Kc_);
        wh = wg_;
      }
      // Y_g[Cog][PQ] = W_g[Cog][Kc] * col[Kc][PQ]
      kernels::gemm(reg, false, false, Cog_, int(PQ), Kc_, real(1), wh, col_, real(0), yg_);
      auto y = tops[0]->data();
      auto yg = reg.buffer(yg_);
      for (int co = 0; co < Cog_; ++co) {
        const real bias = p_.bias_term ? params_[1]->data()[g * Cog_ + co] : real(0);
        for (std::size_t i = 0; i < PQ; ++i)
          y[n * img_out + (g * Cog_ + co) * PQ + i] = yg[co * PQ + i] + bias;
      }
    }
  }
}

void ConvolutionLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  Registry& reg = *reg_;
  const std::size_t PQ = std::size_t(P_) * Q_, img_in = std::size_t(C_) * H_ * W_,
                    img_out = std::size_t(p_.num_output) * PQ;
  Blob& w = *params_[0];
  const bool pd = propagate_down.empty() ? true : bool(propagate_down[0]);
  auto dy = tops[0]->diff();
  if (p_.bias_term) {
    auto db = params_[1]->diff();
    for (int n = 0; n < N_; ++n)
      for (int co = 0; co < p_.num_output; ++co) {
        real s = 0;
        for (std::size_t i = 0; i < PQ; ++i) s += dy[n * img_out + co * PQ + i];
        db[co] += s;
      }
  }
  if (pd) {
    auto dx = bottoms[0]->diff();
    std::fill(dx.begin(), dx.end(), real(0));
  }
  for (int n = 0; n < N_; ++n) {
    for (int g = 0; g < p_.group; ++g) {
      copy_range(tops[0]->diff(), n * img_out + std::size_t(g) * Cog_ * PQ, reg.buffer(yg_), 0, Cog_ * PQ);
      im2col(bottoms[0]->data().subspan(n * img_in, img_in), reg.buffer(col_), g);
      // dW_g += dY_g[Cog][PQ] * col^T   (beta = 1: parameter diffs accumulate)
      if (p_.group == 1) {
        kernels::gemm(reg, false, true, Cog_, Kc_, int(PQ), real(1), yg_, col_, real(1), w.diff_handle());
      } else {
        copy_range(w.diff(), std::size_t(g) * Cog_ * Kc_, reg.buffer(wg_), 0, std::size_t(Cog_) * Kc_);
        kernels::gemm(reg, false, true, Cog_, Kc_, int(PQ), real(1), yg_, col_, real(1), wg_);
        copy_range(reg.buffer(wg_), 0, w.diff(), std::size_t(g) * Cog_ * Kc_, std::size_t(Cog_) * Kc_);
      }
      if (pd) {
        Handle wh = w.data_handle();
        if (p_.group > 1) {
          copy_range(w.data(), std::size_t(g) * Cog_ * Kc_, reg.buffer(wg_), 0, std::size_t(Cog_) * Kc_);
          wh = wg_;
        }
        // dcol[Kc][PQ] = W_g^T * dY_g, then scatter-add back to the image
        kernels::gemm(reg, true, false, Kc_, int(PQ), Cog_, real(1), wh, yg_, real(0), col_);
        col2im(reg.buffer(col_), bottoms[0]->diff().subspan(n * img_in, img_in), g);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pooling (Caffe PoolingLayer::Forward_cpu / Backward_cpu semantics).

std::vector<Shape> PoolingLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng&) {
  one_bottom(spec_, b);
  N_ = b[0].n(); C_ = b[0].c(); H_ = b[0].h(); W_ = b[0].w();
  if (p_.global) {
    p_.kernel_h = H_; p_.kernel_w = W_; p_.stride_h = p_.stride_w = 1; p_.pad_h = p_.pad_w = 0;
  }
  if (p_.pad_h >= p_.kernel_h || p_.pad_w >= p_.kernel_w)
    throw ModelError("layer '" + spec_.name + "': pad must be smaller than kernel");
  PH_ = int(std::ceil(float(H_ + 2 * p_.pad_h - p_.kernel_h) / p_.stride_h)) + 1;
  PW_ = int(std::ceil(float(W_ + 2 * p_.pad_w - p_.kernel_w) / p_.stride_w)) + 1;
  if (p_.pad_h || p_.pad_w) {
    if ((PH_ - 1) * p_.stride_h >= H_ + p_.pad_h) --PH_;
    if ((PW_ - 1) * p_.stride_w >= W_ + p_.pad_w) --PW_;
  }
  mask_.assign(std::size_t(N_) * C_ * PH_ * PW_, -1);
  return {Shape{{N_, C_, PH_, PW_}}};
}

void PoolingLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto x = bottoms[0]->data();
  auto y = tops[0]->data();
  for (int nc = 0; nc < N_ * C_; ++nc) {
    const real* plane = x.data() + std::size_t(nc) * H_ * W_;
    for (int ph = 0; ph < PH_; ++ph)
      for (int pw = 0; pw < PW_; ++pw) {
        const std::size_t o = (std::size_t(nc) * PH_ + ph) * PW_ + pw;
        int hs = ph * p_.stride_h - p_.pad_h, ws = pw * p_.stride_w - p_.pad_w;
        if (p_.max) {
          const int he = std::min(hs + p_.kernel_h, H_), we = std::min(ws + p_.kernel_w, W_);
          hs = std::max(hs, 0); ws = std::max(ws, 0);
          real best = real(-FLT_MAX);
          int arg = -1;
          for (int h = hs; h < he; ++h)
            for (int w = ws; w < we; ++w)
              if (plane[h * W_ + w] > best) { best = plane[h * W_ + w]; arg = h * W_ + w; }
          y[o] = best;
          mask_[o] = arg;
        } else {
          int he = std::min(hs + p_.kernel_h, H_ + p_.pad_h), we = std::min(ws + p_.kernel_w, W_ + p_.pad_w);
          const int pool = (he - hs) * (we - ws);
          hs = std::max(hs, 0); ws = std::max(ws, 0);
          he = std::min(he, H_); we = std::min(we, W_);
          real s = 0;
          for (int h = hs; h < he; ++h)
            for (int w = ws; w < we; ++w) s += plane[h * W_ + w];
          y[o] = s / real(pool);
        }
      }
  }
}

void PoolingLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down.empty() && !propagate_down[0]) return;
  auto dy = tops[0]->diff();
  auto dx = bottoms[0]->diff();
  std::fill(dx.begin(), dx.end(), real(0));
  for (int nc = 0; nc < N_ * C_; ++nc) {
    real* plane = dx.data() + std::size_t(nc) * H_ * W_;
    for (int ph = 0; ph < PH_; ++ph)
      for (int pw = 0; pw < PW_; ++pw) {
        const std::size_t o = (std::size_t(nc) * PH_ + ph) * PW_ + pw;
        if (p_.max) {
          plane[mask_[o]] += dy[o];
        } else {
          int hs = ph * p_.stride_h - p_.pad_h, ws = pw * p_.stride_w - p_.pad_w;
          int he = std::min(hs + p_.kernel_h, H_ + p_.pad_h), we = std::min(ws + p_.kernel_w, W_ + p_.pad_w);
          const int pool = (he - hs) * (we - ws);
          hs = std::max(hs, 0); ws = std::max(ws, 0);
          he = std::min(he, H_); we = std::min(we, W_);
          for (int h = hs; h < he; ++h)
            for (int w = ws; w < we; ++w) plane[h * W_ + w] += dy[o] / real(pool);
        }
      }
  }
}

// ---------------------------------------------------------------------------
// SoftmaxWithLoss: prob = softmax over C*H*W of each sample (the reference
// Softmax rule, layers.cpp:232-247); loss = -sum log(max(p_label, FLT_MIN)) / N.

std::vector<Shape> SoftmaxWithLossLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&,
                                               Rng&) {
  if (b.size() != 2) throw ModelError("layer '" + spec_.name + "': SoftmaxWithLoss takes {logits, label}");
  rows_ = b[0].n();
  classes_ = b[0].c() * b[0].h() * b[0].w();
  if (b[1].count() != std::size_t(rows_)) throw ModelError("layer '" + spec_.name + "': one label per sample required");
  prob_.assign(std::size_t(rows_) * classes_, real(0));
  return {Shape{{1, 1, 1, 1}}};
}

void SoftmaxWithLossLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto x = bottoms[0]->data();
  auto lab = bottoms[1]->data();
  real loss = 0;
  for (int r = 0; r < rows_; ++r) {
    const std::size_t base = std::size_t(r) * classes_;
    real m = x[base];
    for (int i = 1; i < classes_; ++i) m = std::max(m, x[base + i]);
    real sum = 0;
    for (int i = 0; i < classes_; ++i) { prob_[base + i] = std::exp(x[base + i] - m); sum += prob_[base + i]; }
    for (int i = 0; i < classes_; ++i) prob_[base + i] /= sum;
    const int l = static_cast<int>(lab[r]);
    if (l < 0 || l >= classes_) throw InvalidArgument("layer '" + spec_.name + "': label out of range");
    loss -= std::log(std::max(prob_[base + l], real(FLT_MIN)));
  }
  tops[0]->data()[0] = normalize_ ? loss / real(rows_) : loss;
}

void SoftmaxWithLossLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down.empty() && !propagate_down[0]) return;
  const real weight = tops[0]->diff()[0];
  const real scale = weight / (normalize_ ? real(rows_) : real(1));
  auto dx = bottoms[0]->diff();
  auto lab = bottoms[1]->data();
  for (int r = 0; r < rows_; ++r) {
    const int l = static_cast<int>(lab[r]);
    for (int i = 0; i < classes_; ++i) {
      const std::size_t k = std::size_t(r) * classes_ + i;
      dx[k] = (prob_[k] - (i == l ? real(1) : real(0))) * scale;
    }
  }
}

// ---------------------------------------------------------------------------
// Split: every top is a copy of the bottom; the bottom diff is the sum of the
// top diffs (Caffe SplitLayer), which the reference's overwrite rule lacks.

std::vector<Shape> SplitLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng&) {
  one_bottom(spec_, b);
  return std::vector<Shape>(spec_.tops.size(), b[0]);
}

void SplitLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto x = bottoms[0]->data();
  for (Blob* t : tops) std::copy(x.begin(), x.end(), t->data().begin());
}

void SplitLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down.empty() && !propagate_down[0]) return;
  auto dx = bottoms[0]->diff();
  auto d0 = tops[0]->diff();
  std::copy(d0.begin(), d0.end(), dx.begin());
  for (std::size_t t = 1; t < tops.size(); ++t) {
    auto dt = tops[t]->diff();
    for (std::size_t i = 0; i < dx.size(); ++i) dx[i] += dt[i];
  }
}

// ---------------------------------------------------------------------------
// LRN across channels (Caffe lrn_layer.cpp, restated per element).

std::vector<Shape> LRNLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng&) {
  one_bottom(spec_, b);
  if (size_ < 1 || size_ % 2 == 0) throw ModelError("layer '" + spec_.name + "': LRN local_size must be odd");
  N_ = b[0].n(); C_ = b[0].c(); HW_ = b[0].h() * b[0].w();
  scale_.assign(b[0].count(), real(0));
  return {b[0]};
}

void LRNLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto x = bottoms[0]->data();
  auto y = tops[0]->data();
  const int pre = (size_ - 1) / 2;
  for (int n = 0; n < N_; ++n)
    for (int c = 0; c < C_; ++c)
      for (int i = 0; i < HW_; ++i) {
        real s = 0;
        for (int cc = std::max(c - pre, 0); cc < std::min(c - pre + size_, C_); ++cc) {
          const real v = x[(std::size_t(n) * C_ + cc) * HW_ + i];
          s += v * v;
        }
        const std::size_t at = (std::size_t(n) * C_ + c) * HW_ + i;
        scale_[at] = real(k_) + real(alpha_) / real(size_) * s;
        y[at] = x[at] * std::pow(scale_[at], real(-beta_));
      }
}

void LRNLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down.empty() && !propagate_down[0]) return;
  auto x = bottoms[0]->data();
  auto y = tops[0]->data();
  auto dy = tops[0]->diff();
  auto dx = bottoms[0]->diff();
  const int pre = (size_ - 1) / 2, post = size_ - 1 - pre;
  for (int n = 0; n < N_; ++n)
    for (int c = 0; c < C_; ++c)
      for (int i = 0; i < HW_; ++i) {
        real acc = 0;  // channels whose window contains c: c' in [c - post, c + pre]
        for (int cc = std::max(c - post, 0); cc < std::min(c + pre + 1, C_); ++cc) {
          const std::size_t j = (std::size_t(n) * C_ + cc) * HW_ + i;
          acc += dy[j] * y[j] / scale_[j];
        }
        const std::size_t at = (std::size_t(n) * C_ + c) * HW_ + i;
        dx[at] = dy[at] * std::pow(scale_[at], real(-beta_)) -
                 real(2) * real(alpha_) * real(beta_) / real(size_) * x[at] * acc;
      }
}

// ---------------------------------------------------------------------------
// Dropout with a counter-based mask (see ext_layers.hpp).

std::uint32_t DropoutLayer::hash(std::uint64_t seed, std::uint64_t iter, std::uint64_t idx) {
  std::uint64_t z = seed * 0x9E3779B97F4A7C15ull ^ (iter + 1) * 0xBF58476D1CE4E5B9ull ^ (idx + 1) * 0x94D049BB133111EBull;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return std::uint32_t(z >> 32);
}

bool DropoutLayer::keep(std::size_t i) const {
  const auto thr = std::uint32_t(std::min(4294967295.0, ratio_ * 4294967296.0));
  return hash(seed_, iter_, i) > thr;
}

std::vector<Shape> DropoutLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng& rng) {
  one_bottom(spec_, b);
  if (!(ratio_ >= 0.0 && ratio_ < 1.0)) throw ModelError("layer '" + spec_.name + "': dropout_ratio must be in [0, 1)");
  seed_ = rng.next_u64();
  return {b[0]};
}

void DropoutLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  ++iter_;
  auto x = bottoms[0]->data();
  auto y = tops[0]->data();
  const real scale = real(1.0 / (1.0 - ratio_));
  for (std::size_t i = 0; i < x.size(); ++i) y[i] = keep(i) ? x[i] * scale : real(0);
}

void DropoutLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down.empty() && !propagate_down[0]) return;
  auto dy = tops[0]->diff();
  auto dx = bottoms[0]->diff();
  const real scale = real(1.0 / (1.0 - ratio_));
  for (std::size_t i = 0; i < dy.size(); ++i) dx[i] = keep(i) ? dy[i] * scale : real(0);
}

// ---------------------------------------------------------------------------
// BatchNorm, training statistics (two-pass mean / biased variance in double).

std::vector<Shape> BatchNormLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng&) {
  one_bottom(spec_, b);
  N_ = b[0].n(); C_ = b[0].c(); HW_ = b[0].h() * b[0].w();
  xnorm_.assign(b[0].count(), real(0));
  invstd_.assign(std::size_t(C_), real(0));
  return {b[0]};
}

void BatchNormLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto x = bottoms[0]->data();
  auto y = tops[0]->data();
  const double cnt = double(N_) * HW_;
  for (int c = 0; c < C_; ++c) {
    double m = 0, v = 0;
    for (int n = 0; n < N_; ++n)
      for (int i = 0; i < HW_; ++i) m += double(x[(std::size_t(n) * C_ + c) * HW_ + i]);
    m /= cnt;
    for (int n = 0; n < N_; ++n)
      for (int i = 0; i < HW_; ++i) {
        const double d = double(x[(std::size_t(n) * C_ + c) * HW_ + i]) - m;
        v += d * d;
      }
    v /= cnt;
    const real mean = real(m);
    invstd_[c] = real(1.0 / std::sqrt(v + eps_));
    for (int n = 0; n < N_; ++n)
      for (int i = 0; i < HW_; ++i) {
        const std::size_t at = (std::size_t(n) * C_ + c) * HW_ + i;
        xnorm_[at] = (x[at] - mean) * invstd_[c];
      }
  }
  std::copy(xnorm_.begin(), xnorm_.end(), y.begin());
}

void BatchNormLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  if (!propagate_down.empty() && !propagate_down[0]) return;
  auto dy = tops[0]->diff();
  auto dx = bottoms[0]->diff();
  const double cnt = double(N_) * HW_;
  for (int c = 0; c < C_; ++c) {
    double a = 0, b = 0;
    for (int n = 0; n < N_; ++n)
      for (int i = 0; i < HW_; ++i) {
        const std::size_t at = (std::size_t(n) * C_ + c) * HW_ + i;
        a += double(dy[at]);
        b += double(dy[at]) * double(xnorm_[at]);
      }
    const real ma = real(a / cnt), mb = real(b / cnt);
    for (int n = 0; n < N_; ++n)
      for (int i = 0; i < HW_; ++i) {
        const std::size_t at = (std::size_t(n) * C_ + c) * HW_ + i;
        dx[at] = (dy[at] - ma - xnorm_[at] * mb) * invstd_[c];
      }
  }
}

// ---------------------------------------------------------------------------
// Scale (per channel, learnable gamma / beta).

std::vector<Shape> ScaleLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>& reg, Rng&) {
  one_bottom(spec_, b);
  N_ = b[0].n(); C_ = b[0].c(); HW_ = b[0].h() * b[0].w();
  params_.clear();
  params_.push_back(std::make_shared<Blob>(reg, Shape{{1, 1, 1, C_}}, spec_.name + ".weight"));
  for (real& v : params_[0]->data()) v = real(1);
  if (bias_) params_.push_back(std::make_shared<Blob>(reg, Shape{{1, 1, 1, C_}}, spec_.name + ".bias"));
  x_.assign(b[0].count(), real(0));
  return {b[0]};
}

void ScaleLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto x = bottoms[0]->data();
  std::copy(x.begin(), x.end(), x_.begin());
  auto y = tops[0]->data();
  auto g = params_[0]->data();
  for (std::size_t i = 0; i < x_.size(); ++i) {
    const std::size_t c = (i / HW_) % C_;
    y[i] = x_[i] * g[c] + (bias_ ? params_[1]->data()[c] : real(0));
  }
}

void ScaleLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  auto dy = tops[0]->diff();
  auto g = params_[0]->data();
  auto dg = params_[0]->diff();
  std::vector<double> sg(C_, 0.0), sb(C_, 0.0);
  for (std::size_t i = 0; i < x_.size(); ++i) {
    const std::size_t c = (i / HW_) % C_;
    sg[c] += double(dy[i]) * double(x_[i]);
    sb[c] += double(dy[i]);
  }
  for (int c = 0; c < C_; ++c) dg[c] += real(sg[c]);
  if (bias_) {
    auto db = params_[1]->diff();
    for (int c = 0; c < C_; ++c) db[c] += real(sb[c]);
  }
  if (!propagate_down.empty() && !propagate_down[0]) return;
  auto dx = bottoms[0]->diff();
  for (std::size_t i = 0; i < x_.size(); ++i) dx[i] = dy[i] * g[(i / HW_) % C_];
}

// ---------------------------------------------------------------------------
// Eltwise SUM.

std::vector<Shape> EltwiseLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng&) {
  if (b.size() < 2) throw ModelError("layer '" + spec_.name + "': Eltwise takes at least two bottoms");
  for (const Shape& s : b)
    if (!(s == b[0])) throw ModelError("layer '" + spec_.name + "': Eltwise bottoms must have equal shapes");
  if (coeff_.empty()) coeff_.assign(b.size(), 1.0);
  if (coeff_.size() != b.size()) throw ModelError("layer '" + spec_.name + "': one coeff per bottom required");
  return {b[0]};
}

void EltwiseLayer::forward(std::span<Blob* const> bottoms, std::span<Blob* const> tops) {
  auto y = tops[0]->data();
  for (std::size_t i = 0; i < y.size(); ++i) {
    real s = real(coeff_[0]) * bottoms[0]->data()[i];
    for (std::size_t k = 1; k < bottoms.size(); ++k) s = real(coeff_[k]) * bottoms[k]->data()[i] + s;
    y[i] = s;
  }
}

void EltwiseLayer::backward(std::span<Blob* const> tops, std::span<Blob* const> bottoms) {
  auto dy = tops[0]->diff();
  for (std::size_t k = 0; k < bottoms.size(); ++k) {
    if (!propagate_down.empty() && !propagate_down[k]) continue;
    auto dx = bottoms[k]->diff();
    for (std::size_t i = 0; i < dy.size(); ++i) dx[i] = real(coeff_[k]) * dy[i];
  }
}

// ---------------------------------------------------------------------------

std::vector<Shape> LabelledDataLayer::setup(const std::vector<Shape>& b, const std::shared_ptr<Registry>&, Rng&) {
  if (!b.empty()) throw ModelError("layer '" + spec_.name + "': data layers take no bottoms");
  if (n_ < 1 || c_ < 1 || h_ < 1 || w_ < 1) throw ModelError("layer '" + spec_.name + "': bad data shape");
  std::vector<Shape> tops{Shape{{n_, c_, h_, w_}}};
  if (spec_.tops.size() == 2) tops.push_back(Shape{{n_, 1, 1, 1}});
  return tops;
}

void LabelledDataLayer::set_batch(const double* data, const double* labels) {
  data_.resize(std::size_t(n_) * sample_size());
  for (std::size_t i = 0; i < data_.size(); ++i) data_[i] = static_cast<real>(data[i]);
  labels_.assign(std::size_t(n_), real(0));
  if (labels)
    for (int i = 0; i < n_; ++i) labels_[i] = static_cast<real>(labels[i]);
  ready_ = true;
}

void LabelledDataLayer::forward(std::span<Blob* const>, std::span<Blob* const> tops) {
  if (!ready_) throw polegrad::DataStarvation("layer '" + spec_.name + "': no batch was set");
  std::copy(data_.begin(), data_.end(), tops[0]->data().begin());
  if (tops.size() > 1) std::copy(labels_.begin(), labels_.end(), tops[1]->data().begin());
}

}  // namespace oracle
