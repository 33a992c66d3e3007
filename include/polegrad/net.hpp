// polegrad/net.hpp — executable network over named blobs.
//
// Reference API (net.hpp:14-85) unchanged: NetDef, Net(def, seed), forward,
// backward, backward_from, blob lookup, params in layer order, MCWT weight
// snapshots.  B200 additions:
//  * all blobs live in HBM; parameters and their gradients are packed into two
//    contiguous arenas (one solver kernel, one all-reduce per bucket);
//  * Caffe wiring when not in reference-compat mode: in-place ReLU/Sigmoid
//    tops, automatic Split layers for fan-out, need-backward propagation
//    (no data gradient into the input), SoftmaxWithLoss loss tops;
//  * set_batch() feed, step capture into a CUDA graph, and an optional
//    data-parallel hook (polegrad::Parallel) that all-reduces gradient
//    buckets on a side stream as backward produces them.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "polegrad/layers.hpp"
#include "polegrad/proto_node.hpp"

namespace polegrad {

// Ordered model description: layer order is execution order.
struct NetDef {
  std::optional<std::string> name;
  std::vector<LayerSpec> layers;
  std::vector<ProtoNode> extras;  // unrecognised top-level fields
  bool operator==(const NetDef&) const = default;
};

class Net {
 public:
  Net() = default;
  Net(const NetDef& def, std::uint64_t seed);
  Net(const NetDef& def, std::uint64_t seed, int device);
  ~Net();
  Net(const Net&) = delete;
  Net& operator=(const Net&) = delete;
  Net(Net&&) noexcept = default;
  Net& operator=(Net&& other) noexcept;

  // Every layer in order; returns the blobs no layer consumes.
  std::map<std::string, Blob*> forward();
  // Every layer's backward in reverse order.
  void backward();
  // Backward of the named blob's producer and everything before it.
  void backward_from(const std::string& blob_name);

  bool has_blob(const std::string& name) const;
  Blob& blob(const std::string& name);
  const Blob& blob(const std::string& name) const;
  const std::vector<std::unique_ptr<Layer>>& layers() const { return layers_; }
  Layer* find_layer(const std::string& name);
  const std::vector<Blob*>& params() const { return params_; }
  std::vector<std::pair<std::string, Shape>> blob_shapes() const;
  const NetDef& def() const { return def_; }
  const std::shared_ptr<Registry>& registry() const { return registry_; }

  std::vector<std::uint8_t> snapshot_weights() const;
  void restore_weights(std::span<const std::uint8_t> bytes);

  // ---- B200 additions ---------------------------------------------------------
  // Sum of the loss tops (SoftmaxWithLoss) after the last forward (D2H read).
  double loss() const;
  const std::vector<Blob*>& loss_blobs() const { return loss_tops_; }
  // Stage one batch into the first MemoryData layer (see MemoryDataLayer::set_batch).
  void set_batch(const real* data, const real* labels = nullptr);
  // Same from a device buffer holding the batch's data followed by its labels (a
  // device-to-device copy, capturable; used by the feed ring's staged slots).
  void set_batch_device(cdnn_handle staged);
  // Flat arenas: params()[i] data/diff are views at param_offset(i).
  Handle weight_arena() const { return weight_arena_; }
  Handle grad_arena() const { return grad_arena_; }
  std::size_t param_offset(std::size_t i) const { return param_offsets_.at(i); }
  std::size_t param_total() const { return param_total_; }
  // Called after layer i's backward (reverse order); used by Parallel.
  using BackwardHook = std::function<void(std::size_t layer_index)>;
  void set_backward_hook(BackwardHook hook) { backward_hook_ = std::move(hook); }
  const BackwardHook& backward_hook() const { return backward_hook_; }
  // Dropout iteration counters (layer order; synchronous D2H / H2D): an eager
  // step that must leave no trace (FeedRing warm-up) restores them afterwards, so
  // ring training draws the same mask sequence as eager training.
  std::vector<double> dropout_counters();
  void set_dropout_counters(const std::vector<double>& values);
  // Index of the first parameter owned by layer i (params are in layer order).
  std::size_t first_param_of_layer(std::size_t i) const { return layer_param_begin_.at(i); }
  // True when forward/backward contain no host work (graph capturable).
  bool graph_safe() const;
  // Scale the gradient of every SoftmaxWithLoss layer (see Parallel).
  void set_loss_scale(double s);
  // Treat the data layer's current top contents as this step's batch (inputs
  // already resident in HBM; no feed copy).
  void reuse_resident_batch();
  // Policy-gradient step of a whole episode batch: after a
  // forward of the first n rows of the feed, write the modulated log-prob
  // gradients (trainer.cpp:42-113: softmax (p - onehot(a))*G, sigmoid -(dlogp*G))
  // into `logit_blob`'s diff on the device (rows >= n get 0) and run
  // backward_from(logit_blob) once -- the batched equivalent of the reference's
  // per-step accumulate_step (trainer.cpp:204-216).  One H2D of 2n values.
  void pg_backward(const std::string& logit_blob, const std::string& prob_blob, std::span<const real> actions,
                   std::span<const real> returns, bool sigmoid);
  // The same with the n actions / returns read asynchronously on the stream from host
  // memory that stays valid (page-locked for a CUDA-graph capture): no host
  // synchronisation, so a whole episode update can be captured and replayed.
  void pg_backward_async(const std::string& logit_blob, const std::string& prob_blob, const real* actions,
                         const real* returns, std::size_t n, bool sigmoid);
  // The pg_softmax shape (MemoryData -> InnerProduct -> ReLU -> InnerProduct ->
  // Softmax [-> MemoryLoss], proj/models/pg_softmax.prototxt) whose whole
  // policy-gradient update runs as one kernel (cdnn_mlp_pg_step, Solver::apply_mlp_pg).
  struct MlpPgPlan {
    Blob* data = nullptr;    // feed top (rows x in)
    Blob* hidden = nullptr;  // ReLU top (rows x hidden)
    Blob* logits = nullptr;  // second InnerProduct top (rows x classes)
    Blob* prob = nullptr;    // Softmax top
    int rows = 0, in = 0, hidden_n = 0, classes = 0;
    std::size_t params[4] = {0, 0, 0, 0};  // W1, b1, W2, b2 (indices into params())
  };
  // The plan when this net has that shape for (logit_blob, prob_blob) and the
  // extents fit the fused kernel; nullopt otherwise (the layered path runs).
  std::optional<MlpPgPlan> mlp_pg_plan(const std::string& logit_blob, const std::string& prob_blob) const;
  // The n actions / returns of an episode into the device buffers pg_backward uses
  // (async H2D from host memory that stays valid): the fused update's inputs.
  void pg_stage_async(const real* actions, const real* returns, std::size_t n);
  Handle pg_actions() const { return pg_actions_; }
  Handle pg_returns() const { return pg_returns_; }
  // Zero every parameter gradient on the device (one fill over the grad arena).
  void zero_param_diffs();
  // Stream of the parameter-gradient halves of the two-stream backward (0 until used).
  cdnn_handle side_stream() const { return side_stream_; }
  // First MemoryData layer (the feed), or nullptr.
  MemoryDataLayer* feed_layer();
  // After replaying a captured step: every blob's and parameter's device copy
  // is newest (replays bypass the host-side coherence records).
  void mark_device_fresh();
  // One eager step with device events between layers: per-layer forward and
  // backward milliseconds (layer order) — the kernel-share breakdown.
  void profile_layers(std::vector<float>& fwd_ms, std::vector<float>& bwd_ms);

 private:
  void build(const NetDef& def, std::uint64_t seed, int device);
  void pack_params();

  std::shared_ptr<Registry> registry_;
  Handle rng_handle_{};
  NetDef def_;
  std::vector<std::unique_ptr<Layer>> layers_;
  std::vector<std::vector<Blob*>> bottoms_;
  std::vector<std::vector<Blob*>> tops_;
  std::vector<std::shared_ptr<Blob>> blobs_;
  std::map<std::string, Blob*> blob_index_;
  std::map<std::string, std::size_t> producer_index_;
  std::vector<Blob*> params_;
  std::vector<std::string> output_names_;
  std::vector<Blob*> loss_tops_;
  std::vector<std::size_t> layer_param_begin_;
  std::vector<std::size_t> param_offsets_;
  std::size_t param_total_ = 0;
  Handle weight_arena_{}, grad_arena_{};
  BackwardHook backward_hook_;
  // parameter-gradient halves of splittable layers run here, in parallel with
  // the bottom-gradient chain on the registry stream (CDNN_SPLIT_BACKWARD=0 off)
  cdnn_handle side_stream_ = 0;
  Handle pg_actions_{}, pg_returns_{};  // pg_backward inputs (batch-sized)
  void backward_layer(std::size_t i, bool& forked);
};

}  // namespace polegrad
