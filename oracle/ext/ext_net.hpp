// ORACLE — test infrastructure only (see ext_layers.hpp).
//
// ExtNet restates the reference Net (net.cpp:12-122) for layer lists that
// include the extension layers: same definition-order forward, reverse-order
// backward, backward_from, params in layer order, seeded init from one Rng and
// the MCWT weight snapshot format (net.cpp:154-286).  Added Caffe semantics:
// in-place tops for ReLU / Sigmoid, automatic Split insertion for fan-out,
// need-backward propagation (bottom diffs of extension layers are skipped
// when nothing upstream has parameters) and loss tops with diff = 1.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ext_layers.hpp"

namespace oracle {

struct LayerDef {
  std::string type, name;
  std::vector<std::string> bottoms, tops;
  std::map<std::string, double> p;  // numeric params (num_output, kernel_h, pool=0/1, ...)
  double get(const std::string& k, double d) const {
    auto it = p.find(k);
    return it == p.end() ? d : it->second;
  }
};

class ExtNet {
 public:
  ExtNet(std::vector<LayerDef> defs, std::uint64_t seed, bool reference_compat);
  ~ExtNet();

  double forward();  // returns the summed loss of the loss tops
  void backward();
  void backward_from(const std::string& blob);

  Blob& blob(const std::string& name);
  bool has_blob(const std::string& name) const { return index_.count(name) != 0; }
  const std::vector<Blob*>& params() const { return params_; }
  std::vector<std::uint8_t> snapshot_weights() const;
  void restore_weights(const std::vector<std::uint8_t>& bytes);

  void set_batch(const double* data, const double* labels);
  polegrad::Layer* layer(const std::string& name);
  const std::vector<LayerDef>& defs() const { return defs_; }
  std::shared_ptr<Registry> registry() const { return reg_; }

 private:
  std::vector<LayerDef> defs_;
  std::shared_ptr<Registry> reg_;
  Handle rng_{};
  std::vector<std::unique_ptr<polegrad::Layer>> layers_;
  std::vector<std::vector<Blob*>> bottoms_, tops_;
  std::vector<std::shared_ptr<Blob>> blobs_;
  std::map<std::string, Blob*> index_;
  std::map<std::string, std::size_t> producer_;
  std::vector<Blob*> params_;
  std::vector<Blob*> loss_tops_;
};

// Solver restated from solver.cpp:24-57 and extended with Caffe momentum and
// weight decay (g += wd*w; v = mom*v + lr*g; w -= v).  With mom = wd = 0 it is
// the reference SGD step w -= lr*g; RMSProp follows solver.cpp:50-52.  Every
// parameter diff is zeroed afterwards (solver.cpp:55).
class ExtSolver {
 public:
  ExtSolver(int method, double lr, double momentum, double weight_decay, double rms_decay, double eps);
  void apply_update(const std::vector<Blob*>& params);

 private:
  int method_;
  real lr_, mom_, wd_, decay_, eps_;
  std::vector<std::vector<real>> hist_;
};

}  // namespace oracle
