// solver.cpp — one fused update kernel over the net's parameter arena
// (reference: solver.cpp:10-68).
#include "polegrad/solver.hpp"

#include <bit>
#include <cstring>

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

void Solver::prepare(Net& net) {
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
      if (!pending_.empty()) {
        if (pending_.size() != history_len_) throw InvalidState("solver: restored history does not match the net");
        reg.write(history_, pending_);
        pending_.clear();
      }
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
}

void Solver::apply_update(Net& net) {
  const auto& params = net.params();
  if (params.empty()) return;
  Registry& reg = *net.registry();
  const bool stateful = config_.method == SolverMethod::kRmsProp || config_.momentum != real(0);
  prepare(net);
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
                            reg.inout(net.weight_arena()), reg.inout(net.grad_arena()),
                            stateful ? reg.inout(history_) : 0,
                            net.param_total(), static_cast<double>(c.learning_rate), static_cast<double>(c.momentum),
                            static_cast<double>(c.weight_decay), static_cast<double>(c.rms_decay),
                            static_cast<double>(c.epsilon), reg.stream()),
          "solver");
  for (Blob* p : params) {
    p->overwrite_gpu_data();
    p->overwrite_gpu_diff();
  }
  ++iterations_;
}

void Solver::apply_mlp_pg(Net& net, const Net::MlpPgPlan& plan, std::size_t count, const real* host_states,
                          const real* host_actions, const real* host_returns, real* host_prob) {
  if (parallel_) throw InvalidState("apply_mlp_pg: the fused update does not all-reduce (detach the Parallel)");
  if (count > std::size_t(plan.rows)) throw InvalidArgument("apply_mlp_pg: count exceeds the batch");
  if ((host_actions == nullptr) != (host_returns == nullptr))
    throw InvalidArgument("apply_mlp_pg: actions and returns come from the same side");
  if (!host_actions && !net.pg_actions())
    throw InvalidState("apply_mlp_pg: stage the actions / returns first (Net::pg_stage_async)");
  Registry& reg = *net.registry();
  const bool stateful = config_.method == SolverMethod::kRmsProp || config_.momentum != real(0);
  prepare(net);
  const auto& params = net.params();
  for (Blob* p : params) {
    p->gpu_data();
    p->gpu_diff();
  }
  const std::uint64_t offs[4] = {net.param_offset(plan.params[0]), net.param_offset(plan.params[1]),
                                 net.param_offset(plan.params[2]), net.param_offset(plan.params[3])};
  const auto& c = config_;
  // host states: the kernel fills the feed blob; device states: it reads the staged batch
  cdnn_handle x = host_states ? plan.data->overwrite_gpu_data() : plan.data->gpu_data();
  cdnn_handle act = host_actions ? 0 : reg.in(net.pg_actions());
  cdnn_handle ret = host_returns ? 0 : reg.in(net.pg_returns());
  cdnn_ok(cdnn_mlp_pg_step_host(reg.context(), x, act, ret, host_states, host_actions, host_returns, host_prob,
                           plan.rows, int(count), plan.in, plan.hidden_n, plan.classes, reg.inout(net.weight_arena()),
                           reg.inout(net.grad_arena()), stateful ? reg.inout(history_) : 0, offs,
                           c.method == SolverMethod::kRmsProp ? CDNN_SOLVER_RMSPROP : CDNN_SOLVER_SGD,
                           static_cast<double>(c.learning_rate), static_cast<double>(c.momentum),
                           static_cast<double>(c.weight_decay), static_cast<double>(c.rms_decay),
                           static_cast<double>(c.epsilon), plan.hidden->overwrite_gpu_data(),
                           plan.logits->overwrite_gpu_data(), plan.prob->overwrite_gpu_data(), reg.stream()),
          "apply_mlp_pg");
  for (Blob* p : params) {
    p->overwrite_gpu_data();
    p->overwrite_gpu_diff();
  }
  ++iterations_;
}

std::vector<std::uint8_t> Solver::snapshot_state() const {
  std::vector<std::uint8_t> out{'M', 'C', 'S', 'S'};
  auto put = [&](std::uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) out.push_back(std::uint8_t(v >> (8 * i)));
  };
  put(1, 4);
  put(config_.method == SolverMethod::kRmsProp ? 1 : 0, 4);
  put(iterations_, 8);
  const std::vector<real> h = history_ ? hist_reg_->read(history_) : pending_;
  put(h.size(), 8);
  for (real v : h) put(std::bit_cast<std::uint64_t>(static_cast<double>(v)), 8);
  return out;
}

void Solver::restore_state(std::span<const std::uint8_t> b) {
  std::size_t pos = 0;
  auto need = [&](std::size_t n) {
    if (b.size() - pos < n) throw FormatError("solver state: truncated payload");
  };
  auto get = [&](int bytes) {
    need(std::size_t(bytes));
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= std::uint64_t(b[pos + i]) << (8 * i);
    pos += std::size_t(bytes);
    return v;
  };
  need(4);
  if (std::memcmp(b.data(), "MCSS", 4) != 0) throw FormatError("solver state: bad magic");
  pos = 4;
  if (get(4) != 1) throw FormatError("solver state: unsupported version");
  const std::uint64_t method = get(4);
  if (method != (config_.method == SolverMethod::kRmsProp ? 1u : 0u))
    throw InvalidState("solver state: saved by a different update rule");
  const std::uint64_t iters = get(8);
  const std::uint64_t n = get(8);
  if (n > (b.size() - pos) / 8) throw FormatError("solver state: truncated payload");
  std::vector<real> h(n);
  for (auto& v : h) v = static_cast<real>(std::bit_cast<double>(get(8)));
  if (pos != b.size()) throw FormatError("solver state: trailing bytes");
  if (history_) {
    if (n != history_len_) throw InvalidState("solver state: history length does not match the net");
    hist_reg_->write(history_, h);
  } else {
    pending_ = std::move(h);
  }
  iterations_ = iters;
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
