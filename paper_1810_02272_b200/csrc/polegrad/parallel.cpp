// parallel.cpp — bucketed NCCL gradient all-reduce overlapped with backward.
#include "polegrad/parallel.hpp"

#include <algorithm>

#include "polegrad/errors.hpp"

namespace polegrad {

std::vector<GradBucket> plan_buckets(const std::vector<std::size_t>& offsets, const std::vector<std::size_t>& counts,
                                     std::size_t total, std::size_t bucket_elems) {
  if (offsets.size() != counts.size()) throw InvalidArgument("plan_buckets: offsets/counts length mismatch");
  std::vector<GradBucket> out;
  if (offsets.empty()) return out;
  bucket_elems = std::max<std::size_t>(bucket_elems, 1);
  std::size_t end = total;  // buckets tile the arena from the back (padding included)
  std::size_t acc = 0;
  for (std::size_t i = offsets.size(); i-- > 0;) {
    acc += counts[i];
    if (acc >= bucket_elems || i == 0) {
      const std::size_t begin = i == 0 ? 0 : offsets[i];
      out.push_back(GradBucket{begin, end, i});
      end = begin;
      acc = 0;
    }
  }
  return out;
}

Parallel::UniqueId Parallel::unique_id() {
  UniqueId id{};
  cdnn_ok(cdnn_nccl_unique_id(id.data()), "Parallel::unique_id");
  return id;
}

Parallel::Parallel(Net& net, int nranks, int rank, const UniqueId& id, std::size_t bucket_bytes)
    : net_(&net), nranks_(nranks), rank_(rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("Parallel: bad rank / nranks");
  Registry& reg = *net.registry();
  cdnn_ok(cdnn_nccl_comm_create(reg.context(), nranks, rank, id.data(), &comm_), "Parallel");
  cdnn_ok(cdnn_stream_create(reg.context(), &comm_stream_), "Parallel");
  init_buckets(bucket_bytes);
}

Parallel::Parallel(Net& net, int nranks, int rank, HostTransport transport, std::size_t bucket_bytes)
    : net_(&net), nranks_(nranks), rank_(rank), transport_(std::move(transport)) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("Parallel: bad rank / nranks");
  if (!transport_) throw InvalidArgument("Parallel: empty host transport");
  init_buckets(bucket_bytes);
}

void Parallel::init_buckets(std::size_t bucket_bytes) {
  Net& net = *net_;
  std::vector<std::size_t> offs, counts;
  for (std::size_t i = 0; i < net.params().size(); ++i) {
    offs.push_back(net.param_offset(i));
    counts.push_back(net.params()[i]->count());
  }
  buckets_ = plan_buckets(offs, counts, net.param_total(), std::max<std::size_t>(bucket_bytes / sizeof(real), 1));
  launched_.assign(buckets_.size(), false);
  net.set_backward_hook([this](std::size_t layer) { on_layer_done(layer); });
  // Normalised losses average over the local batch; 1/nranks makes the SUM
  // all-reduce the global-batch mean (Caffe divides by solver_count).
  // MemoryLoss nets inject unnormalised diffs, for which the plain sum is exact.
  net.set_loss_scale(1.0 / nranks_);
}

std::pair<int, int> Parallel::comm_info() const {
  if (transport_) return {nranks_, rank_};
  int n = 0, r = 0;
  cdnn_ok(cdnn_nccl_comm_info(net_->registry()->context(), comm_, &n, &r), "Parallel::comm_info");
  return {n, r};
}

Parallel::~Parallel() {
  if (net_) net_->set_backward_hook(nullptr);
  Registry& reg = *net_->registry();
  if (comm_stream_) cdnn_stream_free(reg.context(), comm_stream_);
  if (comm_) cdnn_subsystem_free(reg.context(), comm_);
}

void Parallel::broadcast_weights() {
  Registry& reg = *net_->registry();
  for (Blob* p : net_->params()) p->gpu_data();  // upload any host-side edits first
  if (transport_) {
    std::vector<real> host(net_->param_total());
    cdnn_ok(cdnn_read_async(reg.context(), reg.in(net_->weight_arena()), 0, host.data(), host.size(), reg.stream()),
            "broadcast_weights");
    reg.synchronize();
    transport_(1, host.data(), 0, host.size());
    cdnn_ok(cdnn_write_async(reg.context(), reg.in(net_->weight_arena()), 0, host.data(), host.size(), reg.stream()),
            "broadcast_weights");
    reg.synchronize();
  } else {
    cdnn_ok(cdnn_broadcast(reg.context(), comm_, reg.in(net_->weight_arena()), net_->param_total(), 0, reg.stream()),
            "broadcast_weights");
  }
  for (Blob* p : net_->params()) p->overwrite_gpu_data();
}

void Parallel::launch(std::size_t b) {
  if (launched_[b]) return;
  launched_[b] = true;
  ++launches_;
  Registry& reg = *net_->registry();
  const GradBucket& k = buckets_[b];
  if (transport_) {
    // every gradient queued so far on the compute and side streams, then the host round trip
    if (net_->side_stream()) cdnn_ok(cdnn_stream_sync(reg.context(), net_->side_stream()), "allreduce");
    std::vector<real> host(k.end - k.begin);
    cdnn_ok(cdnn_read_async(reg.context(), reg.in(net_->grad_arena()), k.begin, host.data(), host.size(),
                            reg.stream()),
            "allreduce");
    reg.synchronize();
    transport_(0, host.data(), k.begin, host.size());
    cdnn_ok(cdnn_write_async(reg.context(), reg.in(net_->grad_arena()), k.begin, host.data(), host.size(),
                             reg.stream()),
            "allreduce");
    reg.synchronize();
    return;
  }
  // the comm stream waits for every gradient queued so far on the compute stream and
  // on the backward side stream (parameter-gradient halves, Net::backward_layer)
  cdnn_ok(cdnn_stream_wait(reg.context(), comm_stream_, reg.stream()), "allreduce");
  if (net_->side_stream()) cdnn_ok(cdnn_stream_wait(reg.context(), comm_stream_, net_->side_stream()), "allreduce");
  cdnn_ok(cdnn_allreduce_sum(reg.context(), comm_, reg.in(net_->grad_arena()), k.begin, k.end - k.begin, comm_stream_),
          "allreduce");
}

void Parallel::on_layer_done(std::size_t layer) {
  // backward runs layers in reverse: once layer `layer` is done, every
  // parameter with index >= first_param_of_layer(layer) has its gradient.
  const std::size_t ready_from = net_->first_param_of_layer(layer);
  for (std::size_t b = 0; b < buckets_.size(); ++b)
    if (!launched_[b] && buckets_[b].first_param >= ready_from) launch(b);
}

void Parallel::reduce_gradients(Net& net) {
  if (&net != net_) throw InvalidArgument("Parallel: solver applied to another net");
  for (Blob* p : net.params()) p->gpu_diff();  // host-side gradient edits go up first
  for (std::size_t b = 0; b < buckets_.size(); ++b) launch(b);
  Registry& reg = *net.registry();
  if (comm_stream_) cdnn_ok(cdnn_stream_wait(reg.context(), reg.stream(), comm_stream_), "allreduce join");
  launched_.assign(buckets_.size(), false);
}

}  // namespace polegrad
