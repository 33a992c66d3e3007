// polegrad/parallel.hpp — data-parallel training over NCCL (the paper's
// "Parallel object"; absent from the reference).
//
// One process (or thread) per GPU, each holding a replica Net built from the
// same definition and seed.  Each rank feeds its own slice of the batch; the
// gradient arena is SUM-all-reduced (the reference's losses are not
// normalised by rank count, so a sum keeps single-device parity) in buckets
// formed in reverse parameter order, each launched on a communication stream
// as soon as backward has produced every gradient in it, so the transfers
// overlap the rest of backward.  Solver::apply_update waits for the buckets
// before the fused update, after which weights stay bit-identical on all ranks.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <vector>

#include "polegrad/net.hpp"

namespace polegrad {

// Contiguous range [begin, end) of the gradient arena reduced as one unit,
// together with the lowest parameter index it contains.
struct GradBucket {
  std::size_t begin = 0, end = 0;
  std::size_t first_param = 0;
};

// Pure host planning (unit-testable without a GPU): walks parameters from the
// last to the first and closes a bucket once it holds >= bucket_elems.
std::vector<GradBucket> plan_buckets(const std::vector<std::size_t>& offsets, const std::vector<std::size_t>& counts,
                                     std::size_t total, std::size_t bucket_elems);

class Parallel {
 public:
  using UniqueId = std::array<std::uint8_t, 128>;
  static UniqueId unique_id();  // call on rank 0, share out of band

  Parallel(Net& net, int nranks, int rank, const UniqueId& id, std::size_t bucket_bytes = std::size_t(8) << 20);
  // Host-transport replica: the same buckets, backward hook, loss scale and join,
  // but each bucket is copied to the host, combined by `transport` across ranks
  // (op 0: in-place SUM all-reduce; op 1: broadcast from rank 0) and copied back,
  // synchronously.  For running the data-parallel protocol where NCCL cannot (several
  // ranks on one GPU, CPU-side collectives such as gloo); not graph-capturable.
  using HostTransport = std::function<void(int op, real* host, std::size_t offset, std::size_t n)>;
  Parallel(Net& net, int nranks, int rank, HostTransport transport, std::size_t bucket_bytes = std::size_t(8) << 20);
  ~Parallel();
  Parallel(const Parallel&) = delete;
  Parallel& operator=(const Parallel&) = delete;

  int nranks() const { return nranks_; }
  int rank() const { return rank_; }
  const std::vector<GradBucket>& buckets() const { return buckets_; }
  // Size and rank as the communicator reports them (NCCL: ncclCommCount /
  // ncclCommUserRank; host transport: the constructor's).
  std::pair<int, int> comm_info() const;
  // Bucket all-reduces issued so far (a captured step issues one per bucket).
  std::uint64_t launches() const { return launches_; }

  // Rank 0's weights to every rank (start of training).
  void broadcast_weights();
  // Launch every bucket not yet launched, then make the compute stream wait
  // for the communication stream (called by Solver before the update).
  void reduce_gradients(Net& net);

 private:
  void init_buckets(std::size_t bucket_bytes);
  void on_layer_done(std::size_t layer_index);
  void launch(std::size_t b);

  Net* net_;
  int nranks_, rank_;
  cdnn_handle comm_ = 0;
  cdnn_handle comm_stream_ = 0;
  HostTransport transport_;
  std::vector<GradBucket> buckets_;
  std::vector<bool> launched_;
  std::uint64_t launches_ = 0;
};

}  // namespace polegrad
