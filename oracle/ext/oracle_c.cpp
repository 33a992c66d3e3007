// ORACLE — test infrastructure only (see ext_layers.hpp).
//
// extern "C" driver over (a) the UNMODIFIED reference Net / Solver / prototxt
// parser compiled from /root/reference/proj/core/src, and (b) the reference-style
// extension ExtNet for nets with Convolution / Pooling / SoftmaxWithLoss.
// Values cross the boundary as double whatever `real` is.
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "ext_net.hpp"
#include "polegrad/errors.hpp"
#include "polegrad/net.hpp"
#include "polegrad/prototxt.hpp"
#include "polegrad/solver.hpp"

#define ORC_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

struct OrcNet {
  std::unique_ptr<polegrad::Net> ref;   // reference path
  std::unique_ptr<oracle::ExtNet> ext;  // extension path
  std::vector<polegrad::Blob*> params() const { return ref ? ref->params() : ext->params(); }
  polegrad::Blob& blob(const std::string& n) { return ref ? ref->blob(n) : ext->blob(n); }
};

struct OrcSolver {
  std::unique_ptr<polegrad::Solver> ref;
  std::unique_ptr<oracle::ExtSolver> ext;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const polegrad::InvalidArgument& e) { g_err = e.what(); return 1; }
  catch (const polegrad::DanglingHandle& e) { g_err = e.what(); return 2; }
  catch (const polegrad::UnknownFunction& e) { g_err = e.what(); return 3; }
  catch (const polegrad::ModelError& e) { g_err = e.what(); return 4; }
  catch (const polegrad::DataStarvation& e) { g_err = e.what(); return 5; }
  catch (const polegrad::FormatError& e) { g_err = e.what(); return 6; }
  catch (const polegrad::NotFound& e) { g_err = e.what(); return 7; }
  catch (const polegrad::InvalidState& e) { g_err = e.what(); return 8; }
  catch (const polegrad::ParseError& e) { g_err = e.what(); return 9; }
  catch (const std::exception& e) { g_err = e.what(); return 99; }
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  if (s.empty()) return out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, sep)) out.push_back(item);
  return out;
}

// one layer per line: type|name|bottoms(,)|tops(,)|k=v;k=v
std::vector<oracle::LayerDef> parse_spec(const std::string& text) {
  std::vector<oracle::LayerDef> defs;
  for (const auto& line : split(text, '\n')) {
    if (line.empty()) continue;
    auto f = split(line, '|');
    while (f.size() < 5) f.push_back("");
    oracle::LayerDef d;
    d.type = f[0];
    d.name = f[1];
    d.bottoms = split(f[2], ',');
    d.tops = split(f[3], ',');
    for (const auto& kv : split(f[4], ';')) {
      auto eq = kv.find('=');
      if (eq == std::string::npos) continue;
      d.p[kv.substr(0, eq)] = std::stod(kv.substr(eq + 1));
    }
    defs.push_back(std::move(d));
  }
  return defs;
}

}  // namespace

ORC_API const char* orc_last_error(void) { return g_err.c_str(); }
ORC_API int orc_real_size(void) { return int(sizeof(polegrad::real)); }

ORC_API int orc_refnet_create(const char* prototxt, uint64_t seed, void** out) {
  return guard([&] {
    auto n = std::make_unique<OrcNet>();
    n->ref = std::make_unique<polegrad::Net>(polegrad::prototxt::parse(prototxt), seed);
    *out = n.release();
  });
}

ORC_API int orc_extnet_create(const char* spec, uint64_t seed, int compat, void** out) {
  return guard([&] {
    auto n = std::make_unique<OrcNet>();
    n->ext = std::make_unique<oracle::ExtNet>(parse_spec(spec), seed, compat != 0);
    *out = n.release();
  });
}

ORC_API void orc_net_free(void* net) { delete static_cast<OrcNet*>(net); }

ORC_API int orc_set_batch(void* net, const double* data, const double* labels) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    if (n->ext) { n->ext->set_batch(data, labels); return; }
    for (const auto& l : n->ref->layers()) {
      if (auto* md = dynamic_cast<polegrad::MemoryDataLayer*>(l.get())) {
        const std::size_t ss = md->sample_size();
        std::vector<polegrad::real> s(ss);
        for (int i = 0; i < md->spec().memory_data->batch_size; ++i) {
          for (std::size_t j = 0; j < ss; ++j) s[j] = static_cast<polegrad::real>(data[i * ss + j]);
          md->enqueue(s);
        }
        return;
      }
    }
    throw polegrad::ModelError("set_batch: no MemoryData layer");
  });
}

ORC_API int orc_forward(void* net, double* loss) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    double l = 0;
    if (n->ext) l = n->ext->forward();
    else n->ref->forward();
    if (loss) *loss = l;
  });
}

ORC_API int orc_backward(void* net) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    if (n->ext) n->ext->backward(); else n->ref->backward();
  });
}

ORC_API int orc_backward_from(void* net, const char* blob) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    if (n->ext) n->ext->backward_from(blob); else n->ref->backward_from(blob);
  });
}

ORC_API int orc_blob_shape(void* net, const char* name, int shape[4]) {
  return guard([&] {
    auto& b = static_cast<OrcNet*>(net)->blob(name);
    for (int i = 0; i < 4; ++i) shape[i] = b.shape().d[i];
  });
}

ORC_API int orc_blob_get(void* net, const char* name, int diff, double* out) {
  return guard([&] {
    auto& b = static_cast<OrcNet*>(net)->blob(name);
    auto s = diff ? b.diff() : b.data();
    for (std::size_t i = 0; i < s.size(); ++i) out[i] = static_cast<double>(s[i]);
  });
}

ORC_API int orc_blob_set(void* net, const char* name, int diff, const double* in) {
  return guard([&] {
    auto& b = static_cast<OrcNet*>(net)->blob(name);
    auto s = diff ? b.diff() : b.data();
    for (std::size_t i = 0; i < s.size(); ++i) s[i] = static_cast<polegrad::real>(in[i]);
  });
}

ORC_API int orc_param_count(void* net) { return int(static_cast<OrcNet*>(net)->params().size()); }

ORC_API int orc_param_info(void* net, int i, char* name, int cap, int shape[4]) {
  return guard([&] {
    auto ps = static_cast<OrcNet*>(net)->params();
    if (i < 0 || i >= int(ps.size())) throw polegrad::InvalidArgument("param index out of range");
    std::snprintf(name, std::size_t(cap), "%s", ps[i]->name().c_str());
    for (int k = 0; k < 4; ++k) shape[k] = ps[i]->shape().d[k];
  });
}

ORC_API int orc_param_get(void* net, int i, int diff, double* out) {
  return guard([&] {
    auto ps = static_cast<OrcNet*>(net)->params();
    auto s = diff ? ps.at(i)->diff() : ps.at(i)->data();
    for (std::size_t k = 0; k < s.size(); ++k) out[k] = static_cast<double>(s[k]);
  });
}

ORC_API int orc_param_set(void* net, int i, int diff, const double* in) {
  return guard([&] {
    auto ps = static_cast<OrcNet*>(net)->params();
    auto s = diff ? ps.at(i)->diff() : ps.at(i)->data();
    for (std::size_t k = 0; k < s.size(); ++k) s[k] = static_cast<polegrad::real>(in[k]);
  });
}

ORC_API int orc_snapshot(void* net, uint8_t* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    const auto bytes = n->ext ? n->ext->snapshot_weights() : n->ref->snapshot_weights();
    *len = bytes.size();
    if (buf && cap >= bytes.size()) std::memcpy(buf, bytes.data(), bytes.size());
  });
}

ORC_API int orc_restore(void* net, const uint8_t* buf, uint64_t len) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    std::vector<std::uint8_t> v(buf, buf + len);
    if (n->ext) n->ext->restore_weights(v); else n->ref->restore_weights(v);
  });
}

ORC_API int orc_pool_mask(void* net, const char* layer, int* out, uint64_t n) {
  return guard([&] {
    auto* on = static_cast<OrcNet*>(net);
    if (!on->ext) throw polegrad::ModelError("pool_mask: reference nets have no pooling");
    auto* pl = dynamic_cast<oracle::PoolingLayer*>(on->ext->layer(layer));
    if (!pl) throw polegrad::NotFound(std::string("no pooling layer ") + layer);
    if (n < pl->mask().size()) throw polegrad::InvalidArgument("pool_mask: buffer too small");
    std::memcpy(out, pl->mask().data(), pl->mask().size() * sizeof(int));
  });
}

ORC_API int orc_set_pool_mask(void* net, const char* layer, const int* in, uint64_t n) {
  return guard([&] {
    auto* on = static_cast<OrcNet*>(net);
    if (!on->ext) throw polegrad::ModelError("set_pool_mask: reference nets have no pooling");
    auto* pl = dynamic_cast<oracle::PoolingLayer*>(on->ext->layer(layer));
    if (!pl) throw polegrad::NotFound(std::string("no pooling layer ") + layer);
    if (n < pl->mask().size()) throw polegrad::InvalidArgument("set_pool_mask: buffer too small");
    pl->set_mask(in);
  });
}

// method 0 = SGD, 1 = RMSProp.  Plain SGD / RMSProp on a reference net runs the
// unmodified polegrad::Solver; momentum / weight decay use the ExtSolver.
ORC_API int orc_solver_create(void* net, int method, double lr, double mom, double wd, double decay, double eps,
                              void** out) {
  return guard([&] {
    auto* n = static_cast<OrcNet*>(net);
    auto s = std::make_unique<OrcSolver>();
    if (n->ref && mom == 0 && wd == 0) {
      polegrad::SolverConfig c;
      c.method = method == 1 ? polegrad::SolverMethod::kRmsProp : polegrad::SolverMethod::kSgd;
      c.learning_rate = static_cast<polegrad::real>(lr);
      c.rms_decay = static_cast<polegrad::real>(decay);
      c.epsilon = static_cast<polegrad::real>(eps);
      s->ref = std::make_unique<polegrad::Solver>(c);
    } else {
      s->ext = std::make_unique<oracle::ExtSolver>(method, lr, mom, wd, decay, eps);
    }
    *out = s.release();
  });
}

ORC_API int orc_solver_apply(void* solver, void* net) {
  return guard([&] {
    auto* s = static_cast<OrcSolver*>(solver);
    auto* n = static_cast<OrcNet*>(net);
    if (s->ref) {
      if (!n->ref) throw polegrad::InvalidArgument("reference solver needs a reference net");
      s->ref->apply_update(*n->ref);
    } else {
      s->ext->apply_update(n->params());
    }
  });
}

ORC_API void orc_solver_free(void* s) { delete static_cast<OrcSolver*>(s); }

// The reference's own kernels on a private Registry (backend.cpp:169-197).
ORC_API int orc_gemm(int ta, int tb, int m, int n, int k, double alpha, const double* a, const double* b, double beta,
                     double* c) {
  return guard([&] {
    polegrad::Registry reg;
    auto up = [&](const double* p, std::size_t len) {
      auto h = reg.alloc_buffer(len);
      auto s = reg.buffer(h);
      for (std::size_t i = 0; i < len; ++i) s[i] = static_cast<polegrad::real>(p[i]);
      return h;
    };
    auto ha = up(a, std::size_t(m) * k), hb = up(b, std::size_t(k) * n), hc = up(c, std::size_t(m) * n);
    polegrad::kernels::gemm(reg, ta != 0, tb != 0, m, n, k, static_cast<polegrad::real>(alpha), ha, hb,
                            static_cast<polegrad::real>(beta), hc);
    auto s = reg.buffer(hc);
    for (std::size_t i = 0; i < s.size(); ++i) c[i] = static_cast<double>(s[i]);
  });
}

ORC_API int orc_xent_grad(const double* probs, const double* target, int n, double* out) {
  return guard([&] {
    std::vector<polegrad::real> p(probs, probs + n), t(target, target + n);
    auto g = polegrad::softmax_xent_gradient(p, t);
    for (int i = 0; i < n; ++i) out[i] = static_cast<double>(g[i]);
  });
}

// Parse + canonical print through the reference parser (boundary-input parity).
ORC_API int orc_prototxt_roundtrip(const char* text, char* out, uint64_t cap, uint64_t* len) {
  return guard([&] {
    const std::string s = polegrad::prototxt::print(polegrad::prototxt::parse(text));
    *len = s.size();
    if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  });
}
