// polegrad/feed.hpp — pinned-memory feed ring.
//
// The reference feeds MemoryData from a host FIFO, synchronously, every step
// (layers.cpp:282-304; callers main.cpp:275-281, trainer.cpp:182-189).  The
// ring owns `depth` pinned host slots (batch data, labels, loss) and one
// captured CUDA graph per slot whose first node is the H2D copy of that slot
// and whose last node is the D2H copy of the loss (forward -> backward ->
// update in between).  push() stages the next batch into a free slot on the
// host while earlier steps run on the device, then enqueues the slot's graph;
// pop_loss() returns losses in push order.  Every step still copies its own
// inputs and reads its own loss; only the host staging leaves the critical path.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "polegrad/imagedb.hpp"
#include "polegrad/net.hpp"
#include "polegrad/solver.hpp"

namespace polegrad {

class FeedRing {
 public:
  // The net must be graph-safe (no loss hooks / FIFO-fed MemoryData) and end in
  // a loss top; its first MemoryData layer is the feed.  depth >= 1.
  FeedRing(Net& net, Solver& solver, int depth = 2);
  ~FeedRing();
  FeedRing(const FeedRing&) = delete;
  FeedRing& operator=(const FeedRing&) = delete;

  // Copies one batch (data: batch*C*H*W values; labels: batch values or empty
  // when the feed has no label top) into the next slot and enqueues its step.
  // InvalidState when every slot holds a loss not yet popped.
  void push(std::span<const real> data, std::span<const real> labels);
  // Zero-copy variant: the batch already sits in page-locked host memory
  // (cdnn_host_alloc_pinned); its H2D is enqueued straight from there.  The
  // buffers must stay unchanged until this step's pop_loss().
  void push_pinned(std::span<const real> data, std::span<const real> labels);
  // Samples one batch from `dataset` (imagedb::Dataset::sample, one draw per image
  // from `rng`) and gathers the tensors and labels straight into the next pinned
  // slot, then enqueues its step.  InvalidArgument when a
  // sampled tensor does not match the feed's sample size.
  void push_sampled(const imagedb::Dataset& dataset, imagedb::SampleMethod method, bool use_boost, Rng& rng);
  // Waits for the oldest pushed step and returns its loss.  InvalidState when
  // nothing is in flight.
  double pop_loss();
  std::size_t in_flight() const { return pushed_ - popped_; }
  int depth() const { return int(slots_.size()); }

 private:
  void release() noexcept;
  struct Slot {
    real* data = nullptr;
    real* labels = nullptr;
    real* loss = nullptr;
    cdnn_handle graph = 0;
    cdnn_handle done = 0;     // event recorded after the slot's step
    cdnn_handle staged = 0;   // device copy of the slot's batch (data, then labels)
  };
  Slot& acquire();
  void launch(Slot& s, const real* data = nullptr, const real* labels = nullptr);
  Net& net_;
  Solver& solver_;
  std::vector<Slot> slots_;
  std::size_t data_len_ = 0, label_len_ = 0, batch_ = 0;
  cdnn_handle copy_stream_ = 0;  // H2D of the next batches, overlapping the running step
  std::uint64_t pushed_ = 0, popped_ = 0;
};

}  // namespace polegrad
