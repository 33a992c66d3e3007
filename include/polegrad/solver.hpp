// polegrad/solver.hpp — parameter update.
//
// Reference API (solver.hpp:10-39) with SolverConfig extended by Caffe's
// momentum and weight decay (both default 0, which is exactly the reference
// SGD step).  apply_update() is one fused sm_100a kernel over the net's flat
// parameter arena: it applies the rule and zeroes every gradient
// (solver.cpp:55).  With a Parallel attached it first waits for the gradient
// all-reduce (sum over ranks).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "polegrad/net.hpp"
#include "polegrad/types.hpp"

namespace polegrad {

enum class SolverMethod { kSgd, kRmsProp };

struct SolverConfig {
  SolverMethod method = SolverMethod::kRmsProp;
  real learning_rate = real(1e-3);
  real rms_decay = real(0.99);
  real epsilon = real(1e-8);
  // B200 additions (Caffe SGDSolver): g += weight_decay*w; v = momentum*v + lr*g; w -= v
  real momentum = real(0);
  real weight_decay = real(0);
};

class Parallel;

class Solver {
 public:
  explicit Solver(const SolverConfig& config);
  ~Solver();
  const SolverConfig& config() const { return config_; }

  // sgd:     w -= lr*diff            (+ momentum / weight decay when set)
  // rmsprop: cache = d*cache + (1-d)*diff^2 ; w -= lr*diff/(sqrt(cache)+eps)
  // Every parameter diff is zero afterwards.
  void apply_update(Net& net);

  // The whole policy-gradient update of the net's pg_softmax MLP (Net::mlp_pg_plan)
  // as one kernel: forward of the staged feed, the softmax gradient of the first
  // `count` rows at the logits with the actions / returns staged by
  // Net::pg_stage_async, backward and this solver's rule; every parameter diff is
  // zero afterwards, like apply_update.  Not with a Parallel attached.
  // With host pointers (page-locked, mapped) the kernel reads the states / actions /
  // returns over the bus (the states also land in the feed blob) and writes the
  // probabilities to host_prob: a captured update with no copy nodes.
  void apply_mlp_pg(Net& net, const Net::MlpPgPlan& plan, std::size_t count, const real* host_states = nullptr,
                    const real* host_actions = nullptr, const real* host_returns = nullptr,
                    real* host_prob = nullptr);
  bool has_parallel() const { return parallel_ != nullptr; }
  // Data-parallel training: all-reduce gradients through `parallel` before
  // each update (nullptr detaches).
  void set_parallel(Parallel* parallel) { parallel_ = parallel; }
  // Solver state for checkpoints (momentum / RMSProp history, arena order).
  std::vector<real> history() const;
  void set_history(std::span<const real> h);
  std::uint64_t iterations() const { return iterations_; }
  // Allocate the history (and install a restored one) without updating, so a
  // following graph capture performs no allocation.
  void prepare(Net& net);
  // Bookkeeping for captured updates: captures are not updates, replays are.
  void uncount_updates(std::int64_t n) { iterations_ = std::uint64_t(std::int64_t(iterations_) - n); }

  // Checkpoint of the solver state (the reference saves none):
  //   "MCSS", u32 version (1), u32 method (0 sgd, 1 rmsprop), u64 updates,
  //   u64 n, n x f64 history (arena order; n = 0 for a stateless solver or
  //   before the first update) — little endian, values widened to f64 like MCWT.
  // restore_state() may run before the first update (the history is then
  // installed on the next apply_update); FormatError on a malformed payload,
  // InvalidState when the method or the parameter count does not match.
  std::vector<std::uint8_t> snapshot_state() const;
  void restore_state(std::span<const std::uint8_t> bytes);

 private:
  SolverConfig config_;
  Parallel* parallel_ = nullptr;
  std::shared_ptr<Registry> hist_reg_;  // registry holding the history buffer
  Handle history_{};
  std::size_t history_len_ = 0;
  std::size_t history_params_ = 0;
  std::uint64_t iterations_ = 0;
  std::vector<real> pending_;  // restored history awaiting the first update
};

// True when every parameter gradient of the net is exactly zero.
bool diffs_are_zeroed(const Net& net);

}  // namespace polegrad
