// solver.cpp — one fused update kernel over the net's parameter arena
// (reference: solver.cpp:10-68).
#include "polegrad/solver.hpp"

#include "polegrad/errors.hpp"
#include "polegrad/parallel.hpp"

namespace polegrad {

Solver::Solver(const SolverConfig& config) : config_(config) {
  if (!(config_.learning_rate > real(0))) throw InvalidArgument("solver: learning_rate must be > 0");
  if (config_.method == SolverMethod::kRmsProp) {
    if (!(config_.rms_decay >= real(0)) || !(config_.rms_decay < real(1)))
      throw InvalidArgument("solver: rms_decay must be in [0, 1)");
    if (!(config_.epsilon > real(0))) throw InvalidArgument("solver: epsilon must be > 0");
  }
  if (!(config_.momentum >= real(0))) throw InvalidArgument("solver: momentum must be >= 0");
  if (!(config_.weight_decay >= real(0))) throw InvalidArgument("solver: weight_decay must be >= 0");
}

Solver::~Solver() {
  if (hist_reg_ && history_) {
    try { hist_reg_->free_buffer(history_); } catch (...) {}
  }
}

void Solver::apply_update(Net& net) {
  const auto& params = net.params();
  if (params.empty()) return;
  Registry& reg = *net.registry();
  const bool stateful = config_.method == SolverMethod::kRmsProp || config_.momentum != real(0);
  if (stateful) {
    if (!history_) {
      history_ = reg.alloc_buffer(net.param_total());  // zero-filled cache / momentum
      history_len_ = net.param_total();
      history_params_ = params.size();
      hist_reg_ = net.registry();
    } else if (net.param_total() != history_len_ || params.size() != history_params_) {
      throw InvalidState("solver: net parameter count changed mid-run");
    } else if (hist_reg_ != net.registry()) {
      // same shapes on another net: carry the state over (the reference shares it)
      const std::vector<real> h = hist_reg_->read(history_);
      hist_reg_->free_buffer(history_);
      hist_reg_ = net.registry();
      history_ = reg.alloc_buffer(history_len_);
      reg.write(history_, h);
    }
  }
  if (parallel_) parallel_->reduce_gradients(net);
  // Make every parameter view current on the device, run one kernel over the
  // arenas, then mark the views device-newest (their host mirrors are stale).
  for (Blob* p : params) {
    p->gpu_data();
    p->gpu_diff();
  }
  const auto& c = config_;
  cdnn_ok(cdnn_solver_apply(reg.context(),
                            c.method == SolverMethod::kRmsProp ? CDNN_SOLVER_RMSPROP : CDNN_SOLVER_SGD,
                            reg.in(net.weight_arena()), reg.in(net.grad_arena()), stateful ? reg.in(history_) : 0,
                            net.param_total(), static_cast<double>(c.learning_rate), static_cast<double>(c.momentum),
                            static_cast<double>(c.weight_decay), static_cast<double>(c.rms_decay),
                            static_cast<double>(c.epsilon), reg.stream()),
          "solver");
  for (Blob* p : params) {
    p->overwrite_gpu_data();
    p->overwrite_gpu_diff();
  }
}

std::vector<real> Solver::history() const {
  if (!history_) return {};
  return hist_reg_->read(history_);
}

void Solver::set_history(std::span<const real> h) {
  if (!history_ || h.size() != history_len_) throw InvalidState("solver: history size mismatch");
  hist_reg_->write(history_, h);
}

bool diffs_are_zeroed(const Net& net) {
  for (const Blob* p : net.params())
    for (real v : p->diff())
      if (v != real(0)) return false;
  return true;
}

}  // namespace polegrad
