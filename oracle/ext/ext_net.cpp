// ORACLE — test infrastructure only (see ext_layers.hpp).
#include "ext_net.hpp"

#include <bit>
#include <cmath>
#include <cstring>
#include <set>

#include "polegrad/errors.hpp"

namespace oracle {

using polegrad::FormatError;
using polegrad::InvalidArgument;
using polegrad::LayerType;
using polegrad::ModelError;
using polegrad::NotFound;

namespace {

bool is_inplace_ok(const std::string& type) {
  return type == "ReLU" || type == "Sigmoid" || type == "Dropout" || type == "BatchNorm" || type == "Scale";
}

// Caffe InsertSplits: a blob version read by more than one layer gets a Split
// layer right after its producer and each reader gets its own copy.
std::vector<LayerDef> insert_splits(const std::vector<LayerDef>& in) {
  struct Version { std::string name; int producer; std::vector<std::pair<int, int>> readers; };
  std::vector<Version> versions;
  std::map<std::string, int> current;
  for (int i = 0; i < int(in.size()); ++i) {
    for (int b = 0; b < int(in[i].bottoms.size()); ++b) {
      auto it = current.find(in[i].bottoms[b]);
      if (it != current.end()) versions[it->second].readers.push_back({i, b});
    }
    for (const auto& t : in[i].tops) {
      versions.push_back({t, i, {}});
      current[t] = int(versions.size()) - 1;
    }
  }
  std::map<std::pair<int, int>, std::string> rename;
  std::map<int, std::vector<LayerDef>> after;
  for (const auto& v : versions) {
    if (v.readers.size() < 2) continue;
    LayerDef split;
    split.type = "Split";
    split.name = v.name + "_" + in[v.producer].name + "_split";
    split.bottoms = {v.name};
    for (std::size_t j = 0; j < v.readers.size(); ++j) {
      const auto [li, bi] = v.readers[j];
      for (const auto& t : in[li].tops)
        if (t == v.name) throw ModelError("layer '" + in[li].name + "': in-place use of a fan-out blob '" + v.name + "'");
      const std::string nm = v.name + "_" + in[v.producer].name + "_" + std::to_string(j) + "_split";
      split.tops.push_back(nm);
      rename[{li, bi}] = nm;
    }
    after[v.producer].push_back(split);
  }
  std::vector<LayerDef> out;
  for (int i = 0; i < int(in.size()); ++i) {
    LayerDef d = in[i];
    for (int b = 0; b < int(d.bottoms.size()); ++b) {
      auto it = rename.find({i, b});
      if (it != rename.end()) d.bottoms[b] = it->second;
    }
    out.push_back(d);
    for (auto& s : after[i]) out.push_back(s);
  }
  return out;
}

polegrad::LayerSpec spec_of(const LayerDef& d, LayerType t) {
  polegrad::LayerSpec s;
  s.name = d.name;
  s.type = t;
  s.bottoms = d.bottoms;
  s.tops = d.tops;
  return s;
}

std::unique_ptr<polegrad::Layer> make(const LayerDef& d) {
  if (d.type == "InnerProduct") {
    auto s = spec_of(d, LayerType::kInnerProduct);
    s.inner_product = polegrad::InnerProductParam{int(d.get("num_output", 0)), {}};
    return polegrad::make_layer(s);
  }
  if (d.type == "ReLU") return polegrad::make_layer(spec_of(d, LayerType::kRelu));
  if (d.type == "Sigmoid") return polegrad::make_layer(spec_of(d, LayerType::kSigmoid));
  if (d.type == "Softmax") return polegrad::make_layer(spec_of(d, LayerType::kSoftmax));
  if (d.type == "MemoryLoss") return polegrad::make_layer(spec_of(d, LayerType::kMemoryLoss));
  if (d.type == "MemoryData") {
    const int n = int(d.get("batch_size", 0)), c = int(d.get("channels", 0)), h = int(d.get("height", 0)),
              w = int(d.get("width", 0));
    if (d.tops.size() == 1) {
      auto s = spec_of(d, LayerType::kMemoryData);
      s.memory_data = polegrad::MemoryDataParam{n, c, h, w, {}};
      return polegrad::make_layer(s);
    }
    if (d.tops.size() != 2 || !d.bottoms.empty()) throw ModelError("layer '" + d.name + "': MemoryData takes {data[, label]}");
    return std::make_unique<LabelledDataLayer>(spec_of(d, LayerType::kMemoryData), n, c, h, w);
  }
  if (d.bottoms.size() < 1) throw ModelError("layer '" + d.name + "': missing bottom");
  if (d.type == "Convolution") {
    ConvParam p;
    p.num_output = int(d.get("num_output", 0));
    p.kernel_h = int(d.get("kernel_h", d.get("kernel_size", 1)));
    p.kernel_w = int(d.get("kernel_w", d.get("kernel_size", 1)));
    p.stride_h = int(d.get("stride_h", d.get("stride", 1)));
    p.stride_w = int(d.get("stride_w", d.get("stride", 1)));
    p.pad_h = int(d.get("pad_h", d.get("pad", 0)));
    p.pad_w = int(d.get("pad_w", d.get("pad", 0)));
    p.dilation_h = p.dilation_w = int(d.get("dilation", 1));
    p.group = int(d.get("group", 1));
    p.bias_term = d.get("bias_term", 1) != 0;
    if (d.bottoms.size() != 1 || d.tops.size() != 1) throw ModelError("layer '" + d.name + "': Convolution is 1 -> 1");
    return std::make_unique<ConvolutionLayer>(spec_of(d, LayerType::kInnerProduct), p);
  }
  if (d.type == "Pooling") {
    PoolParam p;
    p.max = d.get("pool", 0) == 0;
    p.kernel_h = int(d.get("kernel_h", d.get("kernel_size", 1)));
    p.kernel_w = int(d.get("kernel_w", d.get("kernel_size", 1)));
    p.stride_h = int(d.get("stride_h", d.get("stride", 1)));
    p.stride_w = int(d.get("stride_w", d.get("stride", 1)));
    p.pad_h = int(d.get("pad_h", d.get("pad", 0)));
    p.pad_w = int(d.get("pad_w", d.get("pad", 0)));
    p.global = d.get("global_pooling", 0) != 0;
    if (d.bottoms.size() != 1 || d.tops.size() != 1) throw ModelError("layer '" + d.name + "': Pooling is 1 -> 1");
    return std::make_unique<PoolingLayer>(spec_of(d, LayerType::kInnerProduct), p);
  }
  if (d.type == "SoftmaxWithLoss") {
    if (d.bottoms.size() != 2 || d.tops.size() != 1) throw ModelError("layer '" + d.name + "': SoftmaxWithLoss is 2 -> 1");
    return std::make_unique<SoftmaxWithLossLayer>(spec_of(d, LayerType::kInnerProduct), d.get("normalize", 1) != 0);
  }
  if (d.type == "Split") return std::make_unique<SplitLayer>(spec_of(d, LayerType::kInnerProduct));
  if (d.type == "LRN") {
    if (d.get("norm_region", 0) != 0) throw ModelError("layer '" + d.name + "': only ACROSS_CHANNELS LRN");
    return std::make_unique<LRNLayer>(spec_of(d, LayerType::kInnerProduct), int(d.get("local_size", 5)),
                                      d.get("alpha", 1.0), d.get("beta", 0.75), d.get("k", 1.0));
  }
  if (d.type == "Dropout")
    return std::make_unique<DropoutLayer>(spec_of(d, LayerType::kInnerProduct), d.get("dropout_ratio", 0.5));
  if (d.type == "BatchNorm") {
    if (d.get("use_global_stats", 0) != 0) throw ModelError("layer '" + d.name + "': training BatchNorm only");
    return std::make_unique<BatchNormLayer>(spec_of(d, LayerType::kInnerProduct), d.get("eps", 1e-5));
  }
  if (d.type == "Scale") {
    if (d.bottoms.size() != 1) throw ModelError("layer '" + d.name + "': Scale takes one bottom");
    return std::make_unique<ScaleLayer>(spec_of(d, LayerType::kInnerProduct), d.get("bias_term", 0) != 0);
  }
  if (d.type == "Eltwise") {
    if (d.get("operation", 1) != 1) throw ModelError("layer '" + d.name + "': only Eltwise SUM");
    std::vector<double> coeff;
    for (int i = 0; d.p.count("coeff" + std::to_string(i)); ++i) coeff.push_back(d.get("coeff" + std::to_string(i), 1));
    return std::make_unique<EltwiseLayer>(spec_of(d, LayerType::kInnerProduct), coeff);
  }
  throw ModelError("layer '" + d.name + "': unknown layer type \"" + d.type + "\"");
}

}  // namespace

ExtNet::ExtNet(std::vector<LayerDef> defs, std::uint64_t seed, bool compat)
    : defs_(compat ? std::move(defs) : insert_splits(defs)), reg_(std::make_shared<Registry>()) {
  rng_ = reg_->create_rng(seed);
  Rng& rng = reg_->rng(rng_);
  std::map<std::string, bool> needs_bwd;
  for (const LayerDef& d : defs_) {
    auto layer = make(d);
    std::vector<Blob*> bottoms;
    std::vector<Shape> shapes;
    bool any_bottom_bwd = false;
    for (const auto& b : d.bottoms) {
      auto it = index_.find(b);
      if (it == index_.end()) throw ModelError("layer '" + d.name + "': undefined bottom '" + b + "'");
      bottoms.push_back(it->second);
      shapes.push_back(it->second->shape());
      any_bottom_bwd = any_bottom_bwd || needs_bwd[b];
    }
    auto top_shapes = layer->setup(shapes, reg_, rng);
    if (top_shapes.size() != d.tops.size())
      throw ModelError("layer '" + d.name + "': produced " + std::to_string(top_shapes.size()) + " top shape(s) for " +
                       std::to_string(d.tops.size()) + " top name(s)");
    const bool layer_bwd = any_bottom_bwd || !layer->params().empty();
    if (auto* ext = dynamic_cast<ExtLayer*>(layer.get())) {
      for (const auto& b : d.bottoms) ext->propagate_down.push_back(needs_bwd[b]);
    }
    std::vector<Blob*> tops;
    for (std::size_t t = 0; t < d.tops.size(); ++t) {
      const std::string& name = d.tops[t];
      const bool inplace = std::find(d.bottoms.begin(), d.bottoms.end(), name) != d.bottoms.end();
      if (inplace && !compat && is_inplace_ok(d.type)) {
        tops.push_back(index_.at(name));
        producer_[name] = layers_.size();
      } else {
        if (index_.count(name)) throw ModelError("layer '" + d.name + "': top '" + name + "' is already produced");
        blobs_.push_back(std::make_shared<Blob>(reg_, top_shapes[t], name));
        index_[name] = blobs_.back().get();
        producer_[name] = layers_.size();
        tops.push_back(blobs_.back().get());
      }
      needs_bwd[name] = layer_bwd;
      if (d.type == "SoftmaxWithLoss") {
        tops.back()->diff()[0] = real(1);  // loss_weight
        loss_tops_.push_back(tops.back());
      }
    }
    for (const auto& p : layer->params()) params_.push_back(p.get());
    layers_.push_back(std::move(layer));
    bottoms_.push_back(std::move(bottoms));
    tops_.push_back(std::move(tops));
  }
}

ExtNet::~ExtNet() {
  if (reg_ && rng_) reg_->free_subsystem(rng_);
}

double ExtNet::forward() {
  for (std::size_t i = 0; i < layers_.size(); ++i) layers_[i]->forward(bottoms_[i], tops_[i]);
  double loss = 0;
  for (Blob* b : loss_tops_) loss += static_cast<double>(b->data()[0]);
  return loss;
}

void ExtNet::backward() {
  for (std::size_t i = layers_.size(); i-- > 0;) layers_[i]->backward(tops_[i], bottoms_[i]);
}

void ExtNet::backward_from(const std::string& name) {
  auto it = producer_.find(name);
  if (it == producer_.end()) throw ModelError("backward_from: no layer produces blob '" + name + "'");
  for (std::size_t i = it->second + 1; i-- > 0;) layers_[i]->backward(tops_[i], bottoms_[i]);
}

Blob& ExtNet::blob(const std::string& name) {
  auto it = index_.find(name);
  if (it == index_.end()) throw NotFound("no blob named '" + name + "'");
  return *it->second;
}

polegrad::Layer* ExtNet::layer(const std::string& name) {
  for (auto& l : layers_)
    if (l->name() == name) return l.get();
  return nullptr;
}

void ExtNet::set_batch(const double* data, const double* labels) {
  for (auto& l : layers_) {
    if (auto* ld = dynamic_cast<LabelledDataLayer*>(l.get())) { ld->set_batch(data, labels); return; }
    if (auto* md = dynamic_cast<polegrad::MemoryDataLayer*>(l.get())) {
      const std::size_t ss = md->sample_size();
      const int n = md->spec().memory_data->batch_size;
      std::vector<real> s(ss);
      for (int i = 0; i < n; ++i) {
        for (std::size_t j = 0; j < ss; ++j) s[j] = static_cast<real>(data[i * ss + j]);
        md->enqueue(s);
      }
      return;
    }
  }
  throw ModelError("set_batch: net has no data layer");
}

// MCWT v1: "MCWT", u32 version, u32 count, per blob {u32 len, name, u32 dims[4],
// f64 values} — all little endian (net.cpp:144-152, 214-246).
std::vector<std::uint8_t> ExtNet::snapshot_weights() const {
  std::vector<std::uint8_t> out{'M', 'C', 'W', 'T'};
  auto u32 = [&](std::uint32_t v) { for (int i = 0; i < 4; ++i) out.push_back(std::uint8_t(v >> (8 * i))); };
  u32(1);
  u32(std::uint32_t(params_.size()));
  for (const Blob* p : params_) {
    u32(std::uint32_t(p->name().size()));
    out.insert(out.end(), p->name().begin(), p->name().end());
    for (int d : p->shape().d) u32(std::uint32_t(d));
    for (real v : p->data()) {
      const auto bits = std::bit_cast<std::uint64_t>(static_cast<double>(v));
      for (int i = 0; i < 8; ++i) out.push_back(std::uint8_t(bits >> (8 * i)));
    }
  }
  return out;
}

void ExtNet::restore_weights(const std::vector<std::uint8_t>& b) {
  std::size_t pos = 0;
  auto need = [&](std::size_t n) { if (b.size() - pos < n) throw FormatError("weight snapshot: truncated payload"); };
  auto u32 = [&] { need(4); std::uint32_t v = 0; for (int i = 0; i < 4; ++i) v |= std::uint32_t(b[pos + i]) << (8 * i); pos += 4; return v; };
  need(4);
  if (std::memcmp(b.data(), "MCWT", 4) != 0) throw FormatError("weight snapshot: bad magic");
  pos = 4;
  if (u32() != 1) throw FormatError("weight snapshot: unsupported version");
  if (u32() != params_.size()) throw FormatError("weight snapshot: blob count mismatch");
  for (Blob* p : params_) {
    const std::uint32_t len = u32();
    need(len);
    const std::string name(reinterpret_cast<const char*>(b.data() + pos), len);
    pos += len;
    if (name != p->name()) throw FormatError("weight snapshot: blob '" + name + "' does not match '" + p->name() + "'");
    Shape s;
    for (int i = 0; i < 4; ++i) s.d[i] = int(u32());
    if (!(s == p->shape())) throw FormatError("weight snapshot: shape mismatch for '" + name + "'");
    auto dst = p->data();
    for (auto& v : dst) {
      need(8);
      std::uint64_t bits = 0;
      for (int i = 0; i < 8; ++i) bits |= std::uint64_t(b[pos + i]) << (8 * i);
      pos += 8;
      v = static_cast<real>(std::bit_cast<double>(bits));
    }
  }
  if (pos != b.size()) throw FormatError("weight snapshot: trailing bytes");
}

ExtSolver::ExtSolver(int method, double lr, double mom, double wd, double decay, double eps)
    : method_(method), lr_(real(lr)), mom_(real(mom)), wd_(real(wd)), decay_(real(decay)), eps_(real(eps)) {
  if (!(lr_ > real(0))) throw InvalidArgument("solver: learning_rate must be > 0");
}

void ExtSolver::apply_update(const std::vector<Blob*>& params) {
  if (hist_.empty()) {
    for (Blob* p : params) hist_.emplace_back(p->count(), real(0));
  }
  if (hist_.size() != params.size()) throw polegrad::InvalidState("solver: net parameter count changed mid-run");
  for (std::size_t k = 0; k < params.size(); ++k) {
    auto w = params[k]->data();
    auto g = params[k]->diff();
    auto& h = hist_[k];
    for (std::size_t i = 0; i < w.size(); ++i) {
      if (method_ == 0) {
        real gi = g[i];
        if (wd_ != real(0)) gi = gi + wd_ * w[i];
        real step = lr_ * gi;
        if (mom_ != real(0)) step = mom_ * h[i] + step;
        h[i] = step;
        w[i] = w[i] - step;
      } else {
        h[i] = decay_ * h[i] + (real(1) - decay_) * g[i] * g[i];
        w[i] -= lr_ * g[i] / (std::sqrt(h[i]) + eps_);
      }
    }
    std::fill(g.begin(), g.end(), real(0));
  }
}

}  // namespace oracle
