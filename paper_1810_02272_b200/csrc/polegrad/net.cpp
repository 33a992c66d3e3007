// net.cpp — graph build, forward/backward and MCWT snapshots (reference:
// net.cpp:12-286), plus the Caffe wiring rules and the flat parameter arenas.
#include "polegrad/net.hpp"

#include <algorithm>
#include <cstdlib>
#include <bit>
#include <cstring>
#include <set>
#include <utility>

#include "polegrad/errors.hpp"

namespace polegrad {

namespace {

bool allows_in_place(LayerType t) {
  return t == LayerType::kRelu || t == LayerType::kSigmoid || t == LayerType::kDropout || t == LayerType::kBatchNorm ||
         t == LayerType::kScale;
}

// Caffe InsertSplits: each blob *version* read by more than one layer gets a
// Split layer right after its producer and every reader its own copy (the
// reference overwrites the shared diff instead).
std::vector<LayerSpec> with_splits(const std::vector<LayerSpec>& layers) {
  struct Version {
    std::string name;
    std::size_t producer;
    std::vector<std::pair<std::size_t, std::size_t>> readers;  // (layer, bottom slot)
  };
  std::vector<Version> versions;
  std::map<std::string, std::size_t> live;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    for (std::size_t b = 0; b < layers[i].bottoms.size(); ++b) {
      auto it = live.find(layers[i].bottoms[b]);
      if (it != live.end()) versions[it->second].readers.emplace_back(i, b);
    }
    for (const std::string& t : layers[i].tops) {
      versions.push_back({t, i, {}});
      live[t] = versions.size() - 1;
    }
  }
  std::map<std::pair<std::size_t, std::size_t>, std::string> renamed;
  std::map<std::size_t, std::vector<LayerSpec>> inserted;
  for (const Version& v : versions) {
    if (v.readers.size() < 2) continue;
    LayerSpec split;
    split.type = LayerType::kSplit;
    split.name = v.name + "_" + layers[v.producer].name + "_split";
    split.bottoms = {v.name};
    for (std::size_t j = 0; j < v.readers.size(); ++j) {
      const auto [li, bi] = v.readers[j];
      for (const std::string& t : layers[li].tops)
        if (t == v.name)
          throw ModelError("layer '" + layers[li].name + "': in-place use of the fan-out blob '" + v.name + "'");
      const std::string copy = v.name + "_" + layers[v.producer].name + "_" + std::to_string(j) + "_split";
      split.tops.push_back(copy);
      renamed[{li, bi}] = copy;
    }
    inserted[v.producer].push_back(std::move(split));
  }
  if (renamed.empty()) return layers;
  std::vector<LayerSpec> out;
  for (std::size_t i = 0; i < layers.size(); ++i) {
    LayerSpec s = layers[i];
    for (std::size_t b = 0; b < s.bottoms.size(); ++b) {
      auto it = renamed.find({i, b});
      if (it != renamed.end()) s.bottoms[b] = it->second;
    }
    out.push_back(std::move(s));
    for (LayerSpec& sp : inserted[i]) out.push_back(std::move(sp));
  }
  return out;
}

}  // namespace

Net::Net(const NetDef& def, std::uint64_t seed) { build(def, seed, 0); }
Net::Net(const NetDef& def, std::uint64_t seed, int device) { build(def, seed, device); }

void Net::build(const NetDef& def, std::uint64_t seed, int device) {
  registry_ = std::make_shared<Registry>(device);
  def_ = def;
  const bool compat = reference_compat();
  const std::vector<LayerSpec> specs = compat ? def.layers : with_splits(def.layers);
  rng_handle_ = registry_->create_rng(seed);
  Rng& rng = registry_->rng(rng_handle_);

  std::set<std::string> consumed;
  std::map<std::string, bool> needs_grad;  // Caffe blob_need_backward
  for (const LayerSpec& spec : specs) {
    auto layer = make_layer(spec);
    std::vector<Blob*> bottoms;
    std::vector<Shape> bottom_shapes;
    bool any_bottom_grad = false;
    std::vector<bool> pd;
    for (const std::string& name : spec.bottoms) {
      auto it = blob_index_.find(name);
      if (it == blob_index_.end()) throw ModelError("layer '" + spec.name + "': undefined bottom '" + name + "'");
      bottoms.push_back(it->second);
      bottom_shapes.push_back(it->second->shape());
      consumed.insert(name);
      any_bottom_grad = any_bottom_grad || needs_grad[name];
      pd.push_back(needs_grad[name]);
    }
    std::vector<Shape> top_shapes = layer->setup(bottom_shapes, registry_, rng);
    if (top_shapes.size() != spec.tops.size()) {
      throw ModelError("layer '" + spec.name + "': produced " + std::to_string(top_shapes.size()) +
                       " top shape(s) for " + std::to_string(spec.tops.size()) + " top name(s)");
    }
    if (!compat) layer->set_propagate_down(pd);
    const bool layer_grad = any_bottom_grad || !layer->params().empty();
    std::vector<Blob*> tops;
    for (std::size_t t = 0; t < spec.tops.size(); ++t) {
      const std::string& name = spec.tops[t];
      const bool in_place = std::find(spec.bottoms.begin(), spec.bottoms.end(), name) != spec.bottoms.end();
      if (blob_index_.contains(name)) {
        if (!(in_place && !compat && allows_in_place(spec.type)))
          throw ModelError("layer '" + spec.name + "': top '" + name + "' is already produced");
        tops.push_back(blob_index_.at(name));  // in-place: the top is the bottom blob
      } else {
        blobs_.push_back(std::make_shared<Blob>(registry_, top_shapes[t], name));
        blob_index_.emplace(name, blobs_.back().get());
        tops.push_back(blobs_.back().get());
      }
      producer_index_[name] = layers_.size();
      needs_grad[name] = layer_grad;
      if (spec.type == LayerType::kSoftmaxWithLoss) {
        tops.back()->diff()[0] = real(1);  // loss weight
        loss_tops_.push_back(tops.back());
      }
    }
    layer_param_begin_.push_back(params_.size());
    for (const auto& p : layer->params()) params_.push_back(p.get());
    layers_.push_back(std::move(layer));
    bottoms_.push_back(std::move(bottoms));
    tops_.push_back(std::move(tops));
  }
  for (const auto& blob : blobs_)
    if (!consumed.contains(blob->name())) output_names_.push_back(blob->name());

  // In-place rewrites after a layer ran: which layers must keep private copies
  // of data their backward reads (Caffe BatchNorm x_norm_, Scale temp_).
  for (std::size_t i = 0; i < layers_.size(); ++i) {
    auto rewritten_after = [&](const Blob* b) {
      for (std::size_t j = i + 1; j < layers_.size(); ++j)
        if (std::find(tops_[j].begin(), tops_[j].end(), b) != tops_[j].end() &&
            std::find(bottoms_[j].begin(), bottoms_[j].end(), b) != bottoms_[j].end())
          return true;
      return false;
    };
    const bool top = !tops_[i].empty() && rewritten_after(tops_[i][0]);
    const bool bottom = !bottoms_[i].empty() && rewritten_after(bottoms_[i][0]);
    layers_[i]->set_clobbered(top, bottom);
  }

  // Fuse BatchNorm + the Scale reading its top.
  for (std::size_t i = 0; i + 1 < layers_.size(); ++i) {
    auto* bn = dynamic_cast<BatchNormLayer*>(layers_[i].get());
    auto* sc = dynamic_cast<ScaleLayer*>(layers_[i + 1].get());
    if (bn && sc && bottoms_[i + 1][0] == tops_[i][0]) {
      bn->fuse_scale(sc, tops_[i + 1][0]);
      sc->set_fused(true);
      // ... and an in-place ReLU on the Scale's top: applied when z is stored
      auto* relu = i + 2 < layers_.size() ? dynamic_cast<ReluLayer*>(layers_[i + 2].get()) : nullptr;
      if (!compat && relu && bottoms_[i + 2][0] == tops_[i + 1][0] && tops_[i + 2][0] == tops_[i + 1][0]) {
        bn->fuse_relu(true);
        relu->set_forward_fused(true);
      }
    }
  }

  // Fuse a plain Eltwise sum + in-place ReLU: the one-pass sum stores max(sum, 0).
  for (std::size_t i = 0; !compat && i + 1 < layers_.size(); ++i) {
    auto* el = dynamic_cast<EltwiseLayer*>(layers_[i].get());
    auto* relu = dynamic_cast<ReluLayer*>(layers_[i + 1].get());
    if (el && relu && el->unit_sum() && bottoms_[i + 1][0] == tops_[i][0] && tops_[i + 1][0] == tops_[i][0]) {
      el->fuse_relu(true);
      relu->set_forward_fused(true);
    }
  }

  // Fuse InnerProduct / Convolution + in-place ReLU: the ReLU runs in the epilogue.
  for (std::size_t i = 0; i + 1 < layers_.size(); ++i) {
    auto* relu = dynamic_cast<ReluLayer*>(layers_[i + 1].get());
    if (!relu || bottoms_[i + 1][0] != tops_[i][0] || tops_[i + 1][0] != tops_[i][0]) continue;
    if (auto* ip = dynamic_cast<InnerProductLayer*>(layers_[i].get())) {
      ip->fuse_relu(true);
      relu->set_forward_fused(true);
    } else if (auto* conv = dynamic_cast<ConvolutionLayer*>(layers_[i].get()); conv && !compat) {
      conv->fuse_relu(true);
      relu->set_forward_fused(true);
    } else if (auto* pool = dynamic_cast<PoolingLayer*>(layers_[i].get()); pool && !compat) {
      pool->fuse_relu(true);
      relu->set_forward_fused(true);
    }
  }
  // Fuse an in-place ReLU's backward into the backward of the layer that consumes
  // its top (Pooling, LRN, Convolution dgrad): that layer writes the ReLU blob's
  // diff gated by the blob's data, and the ReLU pass disappears.  Only when the
  // consumer directly follows the ReLU and nothing else reads or rewrites the blob.
  for (std::size_t i = 0; !compat && i + 1 < layers_.size(); ++i) {
    auto* relu = dynamic_cast<ReluLayer*>(layers_[i].get());
    if (!relu || bottoms_[i].size() != 1 || tops_[i].size() != 1 || bottoms_[i][0] != tops_[i][0]) continue;
    Blob* b = tops_[i][0];
    Layer* consumer = layers_[i + 1].get();
    if (!consumer->supports_relu_gate() || bottoms_[i + 1].empty() || bottoms_[i + 1][0] != b) continue;
    bool other_use = false;
    for (std::size_t k = i + 1; k < layers_.size() && !other_use; ++k) {
      for (std::size_t q = 0; q < bottoms_[k].size(); ++q)
        if (bottoms_[k][q] == b && !(k == i + 1 && q == 0)) other_use = true;
      for (Blob* t : tops_[k])
        if (t == b) other_use = true;
    }
    if (other_use) continue;
    consumer->set_relu_gate(true);
    relu->set_backward_fused(true);
  }
  // Fuse LRN with the MAX pooling that is its top's only reader (AlexNet norm -> pool):
  // one pass over the LRN bottom forward and backward (ops_lrnpool.cu); the LRN top
  // stays materialised, its diff and the scale tensor are not.
  for (std::size_t i = 0; !compat && i + 1 < layers_.size(); ++i) {
    auto* lrn = dynamic_cast<LRNLayer*>(layers_[i].get());
    auto* pool = dynamic_cast<PoolingLayer*>(layers_[i + 1].get());
    if (!lrn || !pool || !pool->is_max() || bottoms_[i + 1].size() != 1 || bottoms_[i + 1][0] != tops_[i][0]) continue;
    Blob* t = tops_[i][0];
    bool other_use = t == bottoms_[i][0];
    for (std::size_t k = i + 2; k < layers_.size() && !other_use; ++k) {
      for (Blob* b : bottoms_[k])
        if (b == t) other_use = true;
      for (Blob* b : tops_[k])
        if (b == t) other_use = true;
    }
    int ok = 0;
    cdnn_ok(cdnn_lrn_pool_supported(registry_->context(), pool->desc(), lrn->size(), &ok), "LRN + Pooling fusion");
    if (other_use || !ok) continue;
    lrn->fuse_pool(pool, tops_[i + 1][0]);
    pool->fuse_lrn(lrn, bottoms_[i][0]);
  }
  pack_params();
}

// Move every parameter into two flat arenas (weights, gradients) so the solver
// is one kernel and data-parallel all-reduce works on contiguous buckets.
void Net::pack_params() {
  param_offsets_.clear();
  std::size_t total = 0;
  for (Blob* p : params_) {
    param_offsets_.push_back(total);
    total += (p->count() + 3) & ~std::size_t(3);  // 16-byte aligned views
  }
  param_total_ = total;
  if (total == 0) return;
  weight_arena_ = registry_->alloc_buffer(total);
  grad_arena_ = registry_->alloc_buffer(total);
  for (std::size_t i = 0; i < params_.size(); ++i) {
    Blob* p = params_[i];
    const Handle w = registry_->alloc_view(weight_arena_, param_offsets_[i], p->count());
    const Handle g = registry_->alloc_view(grad_arena_, param_offsets_[i], p->count());
    kernels::copy(*registry_, p->data_handle(), w, p->count());
    kernels::copy(*registry_, p->diff_handle(), g, p->count());
    p->rebind(w, g);
  }
}

Net::~Net() {
  if (registry_ && side_stream_) {
    try {
      registry_->synchronize();
      cdnn_stream_free(registry_->context(), side_stream_);
    } catch (...) {}
  }
  if (registry_ && rng_handle_) {
    try { registry_->free_subsystem(rng_handle_); } catch (...) {}
  }
}

Net& Net::operator=(Net&& o) noexcept {
  if (this != &o) {
    if (registry_ && rng_handle_) {
      try { registry_->free_subsystem(rng_handle_); } catch (...) {}
    }
    registry_ = std::move(o.registry_);
    rng_handle_ = std::exchange(o.rng_handle_, Handle{});
    side_stream_ = std::exchange(o.side_stream_, cdnn_handle{0});
    def_ = std::move(o.def_);
    layers_ = std::move(o.layers_);
    bottoms_ = std::move(o.bottoms_);
    tops_ = std::move(o.tops_);
    blobs_ = std::move(o.blobs_);
    blob_index_ = std::move(o.blob_index_);
    producer_index_ = std::move(o.producer_index_);
    params_ = std::move(o.params_);
    output_names_ = std::move(o.output_names_);
    loss_tops_ = std::move(o.loss_tops_);
    layer_param_begin_ = std::move(o.layer_param_begin_);
    param_offsets_ = std::move(o.param_offsets_);
    param_total_ = o.param_total_;
    weight_arena_ = o.weight_arena_;
    grad_arena_ = o.grad_arena_;
    backward_hook_ = std::move(o.backward_hook_);
  }
  return *this;
}

std::map<std::string, Blob*> Net::forward() {
  for (std::size_t i = 0; i < layers_.size(); ++i) layers_[i]->forward(bottoms_[i], tops_[i]);
  std::map<std::string, Blob*> outputs;
  for (const std::string& name : output_names_) outputs.emplace(name, blob_index_.at(name));
  return outputs;
}

// Layer i's backward.  Splittable layers (Convolution with a bottom gradient,
// InnerProduct) fork their parameter-gradient half onto the side stream: it
// only reads the top diff and bottom data and writes parameter diffs, none of
// which the remaining bottom-gradient chain touches; the solver joins it.
void Net::backward_layer(std::size_t i, bool& forked) {
  Layer& l = *layers_[i];
  const bool split = !reference_compat() && l.can_split_backward();
  if (!split) {
    l.backward(tops_[i], bottoms_[i]);
    return;
  }
  Registry& reg = *registry_;
  const cdnn_handle main = reg.stream();
  if (!side_stream_) cdnn_ok(cdnn_stream_create(reg.context(), &side_stream_), "backward side stream");
  // bring every operand current on the main stream before the fork
  for (Blob* t : tops_[i]) t->gpu_diff();
  for (Blob* b : bottoms_[i]) b->gpu_data();
  for (const auto& p : l.params()) {
    p->gpu_data();
    p->mutable_gpu_diff();
  }
  cdnn_ok(cdnn_stream_wait(reg.context(), side_stream_, main), "backward fork");
  reg.set_stream(side_stream_);
  try {
    l.backward_weights(tops_[i], bottoms_[i]);
  } catch (...) {
    reg.set_stream(main);
    throw;
  }
  reg.set_stream(main);
  l.backward_inputs(tops_[i], bottoms_[i]);
  forked = true;
}

void Net::backward() {
  bool forked = false;
  for (std::size_t i = layers_.size(); i-- > 0;) {
    backward_layer(i, forked);
    if (backward_hook_) backward_hook_(i);
  }
  if (forked) cdnn_ok(cdnn_stream_wait(registry_->context(), registry_->stream(), side_stream_), "backward join");
}

void Net::backward_from(const std::string& blob_name) {
  auto it = producer_index_.find(blob_name);
  if (it == producer_index_.end()) throw ModelError("backward_from: no layer produces blob '" + blob_name + "'");
  bool forked = false;
  for (std::size_t i = it->second + 1; i-- > 0;) {
    backward_layer(i, forked);
    if (backward_hook_) backward_hook_(i);
  }
  if (forked) cdnn_ok(cdnn_stream_wait(registry_->context(), registry_->stream(), side_stream_), "backward join");
}

bool Net::has_blob(const std::string& name) const { return blob_index_.contains(name); }

Blob& Net::blob(const std::string& name) {
  auto it = blob_index_.find(name);
  if (it == blob_index_.end()) throw NotFound("no blob named '" + name + "'");
  return *it->second;
}

const Blob& Net::blob(const std::string& name) const { return const_cast<Net*>(this)->blob(name); }

Layer* Net::find_layer(const std::string& name) {
  for (const auto& l : layers_)
    if (l->name() == name) return l.get();
  return nullptr;
}

std::vector<std::pair<std::string, Shape>> Net::blob_shapes() const {
  std::vector<std::pair<std::string, Shape>> out;
  out.reserve(blobs_.size());
  for (const auto& b : blobs_) out.emplace_back(b->name(), b->shape());
  return out;
}

double Net::loss() const {
  double s = 0;
  for (const Blob* b : loss_tops_) s += static_cast<double>(b->data()[0]);
  return s;
}

void Net::set_batch(const real* data, const real* labels) {
  for (std::size_t i = 0; i < layers_.size(); ++i) {
    if (auto* md = dynamic_cast<MemoryDataLayer*>(layers_[i].get())) {
      md->set_batch(*tops_[i][0], tops_[i].size() > 1 ? tops_[i][1] : nullptr, data, labels);
      return;
    }
  }
  throw ModelError("set_batch: net has no MemoryData layer");
}

void Net::set_batch_device(cdnn_handle staged) {
  for (std::size_t i = 0; i < layers_.size(); ++i) {
    if (auto* md = dynamic_cast<MemoryDataLayer*>(layers_[i].get())) {
      md->set_batch_device(*tops_[i][0], tops_[i].size() > 1 ? tops_[i][1] : nullptr, staged);
      return;
    }
  }
  throw ModelError("set_batch_device: net has no MemoryData layer");
}

void Net::pg_backward(const std::string& logit_blob, const std::string& prob_blob, std::span<const real> actions,
                      std::span<const real> returns, bool sigmoid) {
  Blob& logit = blob(logit_blob);
  Blob& prob = blob(prob_blob);
  const int rows = logit.shape().n();
  const int classes = int(logit.count() / std::size_t(rows));
  if (prob.count() != logit.count()) throw InvalidArgument("pg_backward: prob and logit blobs differ in size");
  if (actions.size() != returns.size()) throw InvalidArgument("pg_backward: one return per action required");
  if (actions.size() > std::size_t(rows))
    throw InvalidArgument("pg_backward: " + std::to_string(actions.size()) + " steps exceed the batch of " +
                          std::to_string(rows));
  Registry& reg = *registry_;
  const std::size_t n = actions.size();
  if (!pg_actions_) {
    pg_actions_ = reg.alloc_buffer(std::size_t(rows));
    pg_returns_ = reg.alloc_buffer(std::size_t(rows));
  }
  std::vector<real> a(std::size_t(rows), real(0)), g(std::size_t(rows), real(0));
  std::copy(actions.begin(), actions.end(), a.begin());
  std::copy(returns.begin(), returns.end(), g.begin());
  reg.write(pg_actions_, a);
  reg.write(pg_returns_, g);
  cdnn_ok(cdnn_pg_diff(reg.context(), prob.gpu_data(), reg.in(pg_actions_), reg.in(pg_returns_),
                       logit.overwrite_gpu_diff(), rows, int(n), classes, sigmoid ? 1 : 0, reg.stream()),
          "pg_backward");
  backward_from(logit_blob);
}

std::vector<double> Net::dropout_counters() {
  std::vector<double> out;
  registry_->synchronize();
  for (const auto& l : layers_)
    if (auto* d = dynamic_cast<DropoutLayer*>(l.get())) {
      double v = 0;
      cdnn_ok(cdnn_read(registry_->context(), d->counter(), &v, 1), "dropout_counters");
      out.push_back(v);
    }
  return out;
}

void Net::set_dropout_counters(const std::vector<double>& values) {
  std::size_t k = 0;
  registry_->synchronize();
  for (const auto& l : layers_)
    if (auto* d = dynamic_cast<DropoutLayer*>(l.get())) {
      if (k >= values.size()) throw InvalidArgument("set_dropout_counters: too few values");
      cdnn_ok(cdnn_write(registry_->context(), d->counter(), &values[k++], 1), "set_dropout_counters");
    }
  if (k != values.size()) throw InvalidArgument("set_dropout_counters: too many values");
}

void Net::pg_backward_async(const std::string& logit_blob, const std::string& prob_blob, const real* actions,
                            const real* returns, std::size_t n, bool sigmoid) {
  Blob& logit = blob(logit_blob);
  Blob& prob = blob(prob_blob);
  const int rows = logit.shape().n();
  const int classes = int(logit.count() / std::size_t(rows));
  if (prob.count() != logit.count()) throw InvalidArgument("pg_backward: prob and logit blobs differ in size");
  if (n > std::size_t(rows))
    throw InvalidArgument("pg_backward: " + std::to_string(n) + " steps exceed the batch of " + std::to_string(rows));
  Registry& reg = *registry_;
  if (!pg_actions_) {
    pg_actions_ = reg.alloc_buffer(std::size_t(rows));
    pg_returns_ = reg.alloc_buffer(std::size_t(rows));
  }
  if (n) {
    cdnn_ok(cdnn_write_async(reg.context(), reg.in(pg_actions_), 0, actions, n, reg.stream()), "pg_backward");
    cdnn_ok(cdnn_write_async(reg.context(), reg.in(pg_returns_), 0, returns, n, reg.stream()), "pg_backward");
  }
  // rows >= n get a zero diff (cdnn_pg_diff), so the buffers need no padding
  cdnn_ok(cdnn_pg_diff(reg.context(), prob.gpu_data(), reg.in(pg_actions_), reg.in(pg_returns_),
                       logit.overwrite_gpu_diff(), rows, int(n), classes, sigmoid ? 1 : 0, reg.stream()),
          "pg_backward");
  backward_from(logit_blob);
}

std::optional<Net::MlpPgPlan> Net::mlp_pg_plan(const std::string& logit_blob, const std::string& prob_blob) const {
  // exactly: MemoryData, InnerProduct, ReLU, InnerProduct, Softmax [, MemoryLoss(prob)]
  const std::size_t nl = layers_.size();
  if (nl != 5 && nl != 6) return std::nullopt;
  const LayerType want[6] = {LayerType::kMemoryData, LayerType::kInnerProduct, LayerType::kRelu,
                             LayerType::kInnerProduct, LayerType::kSoftmax, LayerType::kMemoryLoss};
  for (std::size_t i = 0; i < nl; ++i)
    if (layers_[i]->type() != want[i]) return std::nullopt;
  auto one = [&](const std::vector<Blob*>& v) { return v.size() == 1 ? v[0] : nullptr; };
  if (tops_[0].empty()) return std::nullopt;
  Blob* data = tops_[0][0];
  Blob* ip1 = one(tops_[1]);
  Blob* relu = one(tops_[2]);
  Blob* logits = one(tops_[3]);
  Blob* prob = one(tops_[4]);
  if (!ip1 || !relu || !logits || !prob) return std::nullopt;
  if (one(bottoms_[1]) != data || one(bottoms_[2]) != ip1 || one(bottoms_[3]) != relu || one(bottoms_[4]) != logits)
    return std::nullopt;
  if (nl == 6) {
    if (one(bottoms_[5]) != prob) return std::nullopt;
    const auto* loss = static_cast<const MemoryLossLayer*>(layers_[5].get());
    if (loss->has_loss_hook()) return std::nullopt;  // host-side gradient: not this update
  }
  if (logits->name() != logit_blob || prob->name() != prob_blob) return std::nullopt;
  MlpPgPlan p;
  p.data = data;
  p.hidden = relu;
  p.logits = logits;
  p.prob = prob;
  p.rows = data->shape().n();
  if (p.rows < 1) return std::nullopt;
  p.in = int(data->count() / std::size_t(p.rows));
  p.hidden_n = int(ip1->count() / std::size_t(p.rows));
  p.classes = int(logits->count() / std::size_t(p.rows));
  const std::size_t b1 = first_param_of_layer(1), b3 = first_param_of_layer(3);
  if (layers_[1]->params().size() != 2 || layers_[3]->params().size() != 2) return std::nullopt;
  p.params[0] = b1;
  p.params[1] = b1 + 1;
  p.params[2] = b3;
  p.params[3] = b3 + 1;
  if (params_[p.params[0]]->count() != std::size_t(p.hidden_n) * std::size_t(p.in) ||
      params_[p.params[2]]->count() != std::size_t(p.classes) * std::size_t(p.hidden_n))
    return std::nullopt;
  int ok = 0;
  cdnn_ok(cdnn_mlp_pg_supported(registry_->context(), sizeof(real) == 4 ? CDNN_F32 : CDNN_F64, p.rows, p.in,
                                p.hidden_n, p.classes, &ok),
          "mlp_pg_plan");
  if (!ok) return std::nullopt;
  return p;
}

void Net::pg_stage_async(const real* actions, const real* returns, std::size_t n) {
  Registry& reg = *registry_;
  const MemoryDataLayer* feed = nullptr;
  for (const auto& l : layers_)
    if (auto* md = dynamic_cast<const MemoryDataLayer*>(l.get())) { feed = md; break; }
  const std::size_t rows = feed ? std::size_t(feed->batch_size()) : n;
  if (n > rows) throw InvalidArgument("pg_stage: " + std::to_string(n) + " steps exceed the batch of " + std::to_string(rows));
  if (!pg_actions_) {
    pg_actions_ = reg.alloc_buffer(std::max<std::size_t>(rows, 1));
    pg_returns_ = reg.alloc_buffer(std::max<std::size_t>(rows, 1));
  }
  if (n) {
    cdnn_ok(cdnn_write_async(reg.context(), reg.in(pg_actions_), 0, actions, n, reg.stream()), "pg_stage");
    cdnn_ok(cdnn_write_async(reg.context(), reg.in(pg_returns_), 0, returns, n, reg.stream()), "pg_stage");
  }
}

void Net::zero_param_diffs() {
  if (!param_total_) return;
  Registry& reg = *registry_;
  cdnn_ok(cdnn_fill(reg.context(), reg.out(grad_arena_), param_total_, 0.0, reg.stream()), "zero_param_diffs");
  for (Blob* p : params_) p->overwrite_gpu_diff();
}

MemoryDataLayer* Net::feed_layer() {
  for (auto& l : layers_)
    if (auto* md = dynamic_cast<MemoryDataLayer*>(l.get())) return md;
  return nullptr;
}

void Net::mark_device_fresh() {
  for (auto& b : blobs_) {
    b->overwrite_gpu_data();
    b->overwrite_gpu_diff();
  }
  for (Blob* p : params_) {
    p->overwrite_gpu_data();
    p->overwrite_gpu_diff();
  }
}

void Net::reuse_resident_batch() {
  for (std::size_t i = 0; i < layers_.size(); ++i) {
    if (auto* md = dynamic_cast<MemoryDataLayer*>(layers_[i].get())) {
      for (Blob* t : tops_[i]) t->gpu_data();  // make sure the resident copy is current
      md->mark_staged();
      return;
    }
  }
  throw ModelError("reuse_resident_batch: net has no MemoryData layer");
}

void Net::profile_layers(std::vector<float>& fwd_ms, std::vector<float>& bwd_ms) {
  cdnn_ctx ctx = registry_->context();
  const cdnn_handle st = registry_->stream();
  const std::size_t n = layers_.size();
  std::vector<cdnn_handle> ev(2 * n + 2, 0);
  for (auto& e : ev) cdnn_ok(cdnn_event_create(ctx, &e), "profile");
  cdnn_ok(cdnn_event_record(ctx, ev[0], st), "profile");
  for (std::size_t i = 0; i < n; ++i) {
    layers_[i]->forward(bottoms_[i], tops_[i]);
    cdnn_ok(cdnn_event_record(ctx, ev[i + 1], st), "profile");
  }
  for (std::size_t k = 0; k < n; ++k) {
    const std::size_t i = n - 1 - k;
    layers_[i]->backward(tops_[i], bottoms_[i]);
    cdnn_ok(cdnn_event_record(ctx, ev[n + 1 + k], st), "profile");
  }
  fwd_ms.assign(n, 0.f);
  bwd_ms.assign(n, 0.f);
  for (std::size_t i = 0; i < n; ++i) cdnn_ok(cdnn_event_elapsed(ctx, ev[i], ev[i + 1], &fwd_ms[i]), "profile");
  for (std::size_t k = 0; k < n; ++k)
    cdnn_ok(cdnn_event_elapsed(ctx, ev[n + k], ev[n + 1 + k], &bwd_ms[n - 1 - k]), "profile");
  for (auto e : ev) cdnn_event_free(ctx, e);
}

void Net::set_loss_scale(double s) {
  for (auto& l : layers_)
    if (auto* sl = dynamic_cast<SoftmaxWithLossLayer*>(l.get())) sl->set_loss_scale(s);
}

bool Net::graph_safe() const {
  for (std::size_t i = 0; i < layers_.size(); ++i) {
    auto* md = dynamic_cast<const MemoryDataLayer*>(layers_[i].get());
    if (md ? !md->has_staged_batch() : !layers_[i]->graph_safe()) return false;
  }
  return true;
}

// ---- MCWT v1 weight snapshots (reference net.cpp:144-286) ------------------------------
// "MCWT" | u32 version=1 | u32 blob count | per blob: u32 name length, name,
// u32 dims[4] (NCHW), f64 values — little endian, f64 whatever `real` is.

std::vector<std::uint8_t> Net::snapshot_weights() const {
  std::vector<std::uint8_t> out = {'M', 'C', 'W', 'T'};
  auto put32 = [&](std::uint32_t v) {
    for (int s = 0; s < 32; s += 8) out.push_back(static_cast<std::uint8_t>(v >> s));
  };
  put32(1);
  put32(static_cast<std::uint32_t>(params_.size()));
  for (const Blob* p : params_) {
    put32(static_cast<std::uint32_t>(p->name().size()));
    out.insert(out.end(), p->name().begin(), p->name().end());
    for (int d : p->shape().d) put32(static_cast<std::uint32_t>(d));
    for (real v : p->data()) {
      const std::uint64_t bits = std::bit_cast<std::uint64_t>(static_cast<double>(v));
      for (int s = 0; s < 64; s += 8) out.push_back(static_cast<std::uint8_t>(bits >> s));
    }
  }
  return out;
}

void Net::restore_weights(std::span<const std::uint8_t> bytes) {
  std::size_t at = 0;
  auto need = [&](std::size_t n) {
    if (bytes.size() - at < n) throw FormatError("weight snapshot: truncated payload");
  };
  auto get32 = [&] {
    need(4);
    std::uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= std::uint32_t(bytes[at + i]) << (8 * i);
    at += 4;
    return v;
  };
  need(4);
  if (std::memcmp(bytes.data(), "MCWT", 4) != 0) throw FormatError("weight snapshot: bad magic");
  at = 4;
  const std::uint32_t version = get32();
  if (version != 1) throw FormatError("weight snapshot: unsupported version " + std::to_string(version));
  const std::uint32_t count = get32();
  if (count != params_.size())
    throw FormatError("weight snapshot: holds " + std::to_string(count) + " blob(s), net has " +
                      std::to_string(params_.size()));
  for (Blob* p : params_) {
    const std::uint32_t len = get32();
    need(len);
    const std::string name(reinterpret_cast<const char*>(bytes.data() + at), len);
    at += len;
    if (name != p->name()) throw FormatError("weight snapshot: blob '" + name + "' does not match '" + p->name() + "'");
    Shape s;
    for (int i = 0; i < 4; ++i) s.d[i] = static_cast<int>(get32());
    if (s != p->shape())
      throw FormatError("weight snapshot: blob '" + name + "' has shape " + to_string(s) + ", net expects " +
                        to_string(p->shape()));
    need(8 * p->count());
    auto dst = p->data();
    for (real& v : dst) {
      std::uint64_t bits = 0;
      for (int i = 0; i < 8; ++i) bits |= std::uint64_t(bytes[at + i]) << (8 * i);
      at += 8;
      v = static_cast<real>(std::bit_cast<double>(bits));
    }
  }
  if (at != bytes.size()) throw FormatError("weight snapshot: trailing bytes");
}

}  // namespace polegrad
