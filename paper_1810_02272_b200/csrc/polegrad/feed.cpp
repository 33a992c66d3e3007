// feed.cpp — pinned-memory feed ring (include/polegrad/feed.hpp).
#include "polegrad/feed.hpp"

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "polegrad/errors.hpp"
#include "polegrad/layers.hpp"

namespace polegrad {

FeedRing::FeedRing(Net& net, Solver& solver, int depth) : net_(net), solver_(solver) {
  if (depth < 1) throw InvalidArgument("feed ring: depth must be >= 1");
  MemoryDataLayer* feed = net.feed_layer();
  if (!feed) throw ModelError("feed ring: the net has no MemoryData layer");
  if (net.loss_blobs().empty()) throw InvalidState("feed ring: the net has no loss top");
  batch_ = std::size_t(feed->batch_size());
  data_len_ = batch_ * feed->sample_size();
  label_len_ = feed->spec().tops.size() > 1 ? std::size_t(feed->batch_size()) : 0;
  Registry& reg = *net.registry();
  cdnn_ctx ctx = reg.context();
  try {
    slots_.resize(std::size_t(depth));
    for (Slot& s : slots_) {
      void* p = nullptr;
      cdnn_ok(cdnn_host_alloc_pinned((data_len_ + label_len_ + 1) * sizeof(real), &p), "feed ring");
      s.data = static_cast<real*>(p);
      s.labels = label_len_ ? s.data + data_len_ : nullptr;
      s.loss = s.data + data_len_ + label_len_;
      std::memset(p, 0, (data_len_ + label_len_ + 1) * sizeof(real));
      cdnn_ok(cdnn_event_create(ctx, &s.done), "feed ring");
      cdnn_ok(cdnn_alloc(ctx, data_len_ + label_len_, kRealDtype, &s.staged), "feed ring");
    }
    cdnn_ok(cdnn_stream_create(ctx, &copy_stream_), "feed ring");
    // One eager forward/backward on a zero batch creates every lazily allocated
    // resource (workspaces, tensor maps, repacked weights) outside the capture;
    // its gradients are discarded and the solver history is allocated without
    // an update, so the weights are untouched.
    // The warm-up leaves no trace: the backward hook (Parallel's bucket
    // all-reduces) is detached, so no collective is launched on the comm stream
    // outside the captured steps (it would race zero_param_diffs and leave the
    // buckets marked launched for the first capture), and the Dropout
    // iteration counters are restored, so ring training draws the same masks as
    // eager training.
    net.set_batch(slots_[0].data, slots_[0].labels);
    if (!net.graph_safe()) throw InvalidState("feed ring: net has host-side layers (loss hooks / FIFO feed)");
    const std::vector<double> counters = net.dropout_counters();
    Net::BackwardHook hook = net.backward_hook();
    net.set_backward_hook(nullptr);
    try {
      net.forward();
      net.backward();
    } catch (...) {
      net.set_backward_hook(std::move(hook));
      throw;
    }
    net.set_backward_hook(std::move(hook));
    net.zero_param_diffs();
    solver.prepare(net);
    reg.synchronize();
    net.set_dropout_counters(counters);
    for (Slot& s : slots_) {
      // capture: D2D(slot's staged batch) -> forward -> backward -> update -> D2H(loss).
      // The slot's H2D runs on the copy stream at push time, overlapping the step
      // in flight (push() orders the graph after it).
      cdnn_ok(cdnn_graph_begin(ctx, reg.stream()), "feed ring capture");
      try {
        net.set_batch_device(s.staged);
        net.forward();
        net.backward();
        solver.apply_update(net);
        cdnn_ok(cdnn_read_async(ctx, net.loss_blobs()[0]->gpu_data(), 0, s.loss, 1, reg.stream()), "feed ring");
      } catch (...) {
        cdnn_handle dead = 0;
        cdnn_graph_end(ctx, reg.stream(), &dead);
        if (dead) cdnn_graph_free(ctx, dead);
        throw;
      }
      cdnn_ok(cdnn_graph_end(ctx, reg.stream(), &s.graph), "feed ring capture");
    }
    solver.uncount_updates(std::uint64_t(depth));  // captures are not updates
  } catch (...) {
    release();
    throw;
  }
}

FeedRing::~FeedRing() { release(); }

void FeedRing::release() noexcept {
  Registry& reg = *net_.registry();
  try { reg.synchronize(); } catch (...) {}
  for (Slot& s : slots_) {
    if (s.graph) cdnn_graph_free(reg.context(), s.graph);
    if (s.done) cdnn_event_free(reg.context(), s.done);
    if (s.staged) cdnn_free(reg.context(), s.staged);
    if (s.data) cdnn_host_free_pinned(s.data);
    s = Slot{};
  }
  slots_.clear();
  if (copy_stream_) cdnn_stream_free(reg.context(), copy_stream_);
  copy_stream_ = 0;
}

FeedRing::Slot& FeedRing::acquire() {
  if (pushed_ - popped_ >= slots_.size()) throw InvalidState("feed ring: full, pop_loss() first");
  // the slot's previous step was popped, so its graph has finished reading it
  return slots_[pushed_ % slots_.size()];
}

void FeedRing::launch(Slot& s, const real* data, const real* labels) {
  Registry& reg = *net_.registry();
  cdnn_ctx ctx = reg.context();
  // H2D of this slot's batch on the copy stream (the slot's previous step has
  // finished -- acquire() -- so nothing still reads its staged buffer), then the
  // step, ordered after the copy
  if (!data) {
    cdnn_ok(cdnn_write_async(ctx, s.staged, 0, s.data, data_len_ + label_len_, copy_stream_), "feed ring push");
  } else {
    cdnn_ok(cdnn_write_async(ctx, s.staged, 0, data, data_len_, copy_stream_), "feed ring push");
    if (label_len_) cdnn_ok(cdnn_write_async(ctx, s.staged, data_len_, labels, label_len_, copy_stream_), "feed ring push");
  }
  cdnn_ok(cdnn_stream_wait(ctx, reg.stream(), copy_stream_), "feed ring push");
  cdnn_ok(cdnn_graph_launch(ctx, s.graph, reg.stream()), "feed ring push");
  cdnn_ok(cdnn_event_record(reg.context(), s.done, reg.stream()), "feed ring push");
  ++pushed_;
  solver_.uncount_updates(-1);  // one real update
}

namespace {
// The caller's pageable batch into the slot's page-locked staging: one host thread moves
// ~5-10 GB/s, so large batches (AlexNet b256: 158 MB) are split over up to 8 threads
// in contiguous byte ranges (the bytes are the same whatever the split).
void copy_to_staging(void* dst, const void* src, std::size_t bytes) {
  constexpr std::size_t kChunk = std::size_t(8) << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const std::size_t nt = std::min<std::size_t>({8, std::size_t(hw), (bytes + kChunk - 1) / kChunk});
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(nt - 1);
  const std::size_t per = (bytes + nt - 1) / nt;
  try {
    for (std::size_t t = 1; t < nt; ++t) {
      const std::size_t b0 = t * per, b1 = std::min(bytes, b0 + per);
      if (b0 < b1)
        pool.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, b1 - b0); });
    }
  } catch (...) {  // no thread to spare: finish on this one
    for (std::thread& th : pool) th.join();
    std::memcpy(dst, src, bytes);
    return;
  }
  std::memcpy(dst, src, std::min(bytes, per));
  for (std::thread& th : pool) th.join();
}
}  // namespace

void FeedRing::push(std::span<const real> data, std::span<const real> labels) {
  if (data.size() != data_len_) throw InvalidArgument("feed ring: batch has the wrong number of values");
  if (labels.size() != label_len_) throw InvalidArgument("feed ring: wrong number of labels");
  Slot& s = acquire();
  copy_to_staging(s.data, data.data(), data_len_ * sizeof(real));
  if (label_len_) std::memcpy(s.labels, labels.data(), label_len_ * sizeof(real));
  launch(s);
}

void FeedRing::push_sampled(const imagedb::Dataset& dataset, imagedb::SampleMethod method, bool use_boost, Rng& rng) {
  Slot& s = acquire();
  const std::size_t per = data_len_ / batch_;
  for (std::size_t b = 0; b < batch_; ++b) {
    const imagedb::Entry& e = dataset.sample(method, use_boost, rng);
    if (e.tensor.size() != per)
      throw InvalidArgument("feed ring: sampled entry " + std::to_string(e.id) + " has " +
                            std::to_string(e.tensor.size()) + " values, the feed takes " + std::to_string(per));
    std::memcpy(s.data + b * per, e.tensor.data(), per * sizeof(real));
    if (label_len_) s.labels[b] = static_cast<real>(e.label);
  }
  launch(s);
}

void FeedRing::push_pinned(std::span<const real> data, std::span<const real> labels) {
  if (data.size() != data_len_) throw InvalidArgument("feed ring: batch has the wrong number of values");
  if (labels.size() != label_len_) throw InvalidArgument("feed ring: wrong number of labels");
  Slot& s = acquire();
  launch(s, data.data(), label_len_ ? labels.data() : nullptr);
}

double FeedRing::pop_loss() {
  if (pushed_ == popped_) throw InvalidState("feed ring: no step in flight");
  Slot& s = slots_[popped_ % slots_.size()];
  cdnn_ok(cdnn_event_sync(net_.registry()->context(), s.done), "feed ring pop");
  ++popped_;
  // the graph's kernels bypassed the blob coherence records: device is newest
  net_.mark_device_fresh();
  return static_cast<double>(*s.loss);
}

}  // namespace polegrad
