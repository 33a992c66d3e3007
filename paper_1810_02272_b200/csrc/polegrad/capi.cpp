// capi.cpp — extern "C" surface of the C++ API (include/polegrad_c.h).
#include <cstring>
#include <memory>
#include <string>

#include "polegrad/errors.hpp"
#include "polegrad/net.hpp"
#include "polegrad/parallel.hpp"
#include "polegrad/prototxt.hpp"
#include "polegrad/solver.hpp"
#include "polegrad_c.h"
#include "polegrad/feed.hpp"
#include "polegrad/imagedb.hpp"

struct pg_net {
  std::unique_ptr<polegrad::Net> net;
};
struct pg_solver {
  std::unique_ptr<polegrad::Solver> solver;
};
struct pg_parallel {
  std::unique_ptr<polegrad::Parallel> par;
};

namespace {

thread_local std::string g_error;

template <class F>
int run(F&& f) {
  using namespace polegrad;
  try {
    f();
    return CDNN_OK;
  } catch (const InvalidArgument& e) { g_error = e.what(); return CDNN_INVALID_ARGUMENT; }
  catch (const DanglingHandle& e) { g_error = e.what(); return CDNN_DANGLING_HANDLE; }
  catch (const UnknownFunction& e) { g_error = e.what(); return CDNN_UNKNOWN_FUNCTION; }
  catch (const ModelError& e) { g_error = e.what(); return CDNN_MODEL_ERROR; }
  catch (const DataStarvation& e) { g_error = e.what(); return CDNN_DATA_STARVATION; }
  catch (const FormatError& e) { g_error = e.what(); return CDNN_FORMAT_ERROR; }
  catch (const NotFound& e) { g_error = e.what(); return CDNN_NOT_FOUND; }
  catch (const InvalidState& e) { g_error = e.what(); return CDNN_INVALID_STATE; }
  catch (const ParseError& e) { g_error = e.what(); return CDNN_PARSE_ERROR; }
  catch (const LoadError& e) { g_error = e.what(); return CDNN_LOAD_ERROR; }
  catch (const std::exception& e) { g_error = e.what(); return CDNN_CUDA_ERROR; }
}

polegrad::Net& net_of(pg_net* n) {
  if (!n || !n->net) throw polegrad::InvalidArgument("null net");
  return *n->net;
}

polegrad::MemoryDataLayer* data_layer(polegrad::Net& net, const char* name) {
  for (const auto& l : net.layers())
    if (auto* md = dynamic_cast<polegrad::MemoryDataLayer*>(l.get()))
      if (!name || !*name || l->name() == name) return md;
  throw polegrad::NotFound("no MemoryData layer");
}

using polegrad::cdnn_ok;
using polegrad::real;

}  // namespace

extern "C" {

const char* pg_last_error(void) { return g_error.c_str(); }
int pg_real_size(void) { return int(sizeof(real)); }

int pg_net_create(const char* prototxt, uint64_t seed, int device, pg_net** out) {
  return run([&] {
    auto n = std::make_unique<pg_net>();
    n->net = std::make_unique<polegrad::Net>(polegrad::prototxt::parse(prototxt), seed, device);
    *out = n.release();
  });
}

int pg_net_free(pg_net* n) {
  return run([&] { delete n; });
}

int pg_net_forward(pg_net* n) { return run([&] { net_of(n).forward(); }); }
int pg_net_backward(pg_net* n) { return run([&] { net_of(n).backward(); }); }
int pg_net_backward_from(pg_net* n, const char* b) { return run([&] { net_of(n).backward_from(b); }); }
int pg_net_loss(pg_net* n, double* out) { return run([&] { *out = net_of(n).loss(); }); }

int pg_net_set_batch(pg_net* n, const void* data, const void* labels) {
  return run([&] { net_of(n).set_batch(static_cast<const real*>(data), static_cast<const real*>(labels)); });
}

int pg_net_pg_backward(pg_net* n, const char* logit_blob, const char* prob_blob, const void* actions,
                       const void* returns, uint64_t count, int sigmoid) {
  return run([&] {
    net_of(n).pg_backward(logit_blob, prob_blob, std::span<const real>(static_cast<const real*>(actions), count),
                          std::span<const real>(static_cast<const real*>(returns), count), sigmoid != 0);
  });
}

int pg_net_enqueue(pg_net* n, const char* layer, const void* sample, uint64_t count) {
  return run([&] {
    data_layer(net_of(n), layer)->enqueue(std::span<const real>(static_cast<const real*>(sample), count));
  });
}

int pg_net_sync(pg_net* n) { return run([&] { net_of(n).registry()->synchronize(); }); }

int pg_net_context(pg_net* n, void** ctx) { return run([&] { *ctx = net_of(n).registry()->context(); }); }

int pg_net_num_layers(pg_net* n) {
  int k = -1;
  run([&] { k = int(net_of(n).layers().size()); });
  return k;
}

int pg_net_layer_name(pg_net* n, int i, char* buf, int cap) {
  return run([&] {
    const auto& ls = net_of(n).layers();
    if (i < 0 || i >= int(ls.size())) throw polegrad::InvalidArgument("layer index out of range");
    std::snprintf(buf, std::size_t(cap), "%s", ls[i]->name().c_str());
  });
}

int pg_blob_shape(pg_net* n, const char* name, int shape[4]) {
  return run([&] {
    const auto& s = net_of(n).blob(name).shape();
    for (int i = 0; i < 4; ++i) shape[i] = s.d[i];
  });
}

int pg_blob_get(pg_net* n, const char* name, int diff, void* out) {
  return run([&] {
    const polegrad::Blob& b = net_of(n).blob(name);
    auto s = diff ? b.diff() : b.data();
    std::memcpy(out, s.data(), s.size() * sizeof(real));
  });
}

int pg_blob_set(pg_net* n, const char* name, int diff, const void* in) {
  return run([&] {
    polegrad::Blob& b = net_of(n).blob(name);
    auto s = diff ? b.diff() : b.data();
    std::memcpy(s.data(), in, s.size() * sizeof(real));
  });
}

int pg_param_count(pg_net* n) {
  int k = -1;
  run([&] { k = int(net_of(n).params().size()); });
  return k;
}

int pg_param_info(pg_net* n, int i, char* name, int cap, int shape[4]) {
  return run([&] {
    const auto& ps = net_of(n).params();
    if (i < 0 || i >= int(ps.size())) throw polegrad::InvalidArgument("param index out of range");
    std::snprintf(name, std::size_t(cap), "%s", ps[i]->name().c_str());
    for (int k = 0; k < 4; ++k) shape[k] = ps[i]->shape().d[k];
  });
}

int pg_param_get(pg_net* n, int i, int diff, void* out) {
  return run([&] {
    const polegrad::Blob* b = net_of(n).params().at(std::size_t(i));
    auto s = diff ? b->diff() : b->data();
    std::memcpy(out, s.data(), s.size() * sizeof(real));
  });
}

int pg_param_set(pg_net* n, int i, int diff, const void* in) {
  return run([&] {
    polegrad::Blob* b = net_of(n).params().at(std::size_t(i));
    auto s = diff ? b->diff() : b->data();
    std::memcpy(s.data(), in, s.size() * sizeof(real));
  });
}

int pg_pool_mask(pg_net* n, const char* layer, int32_t* out, uint64_t count) {
  return run([&] {
    auto* pl = dynamic_cast<polegrad::PoolingLayer*>(net_of(n).find_layer(layer));
    if (!pl) throw polegrad::NotFound(std::string("no pooling layer '") + layer + "'");
    const std::vector<int> m = pl->mask();
    if (count < m.size()) throw polegrad::InvalidArgument("pool_mask: buffer too small");
    std::memcpy(out, m.data(), m.size() * sizeof(int));
  });
}

int pg_snapshot(pg_net* n, uint8_t* buf, uint64_t cap, uint64_t* len) {
  return run([&] {
    const auto bytes = net_of(n).snapshot_weights();
    *len = bytes.size();
    if (buf && cap >= bytes.size()) std::memcpy(buf, bytes.data(), bytes.size());
  });
}

int pg_restore(pg_net* n, const uint8_t* buf, uint64_t len) {
  return run([&] { net_of(n).restore_weights(std::span<const std::uint8_t>(buf, len)); });
}

int pg_solver_create(int method, double lr, double mom, double wd, double decay, double eps, pg_solver** out) {
  return run([&] {
    polegrad::SolverConfig c;
    c.method = method == 1 ? polegrad::SolverMethod::kRmsProp : polegrad::SolverMethod::kSgd;
    c.learning_rate = static_cast<real>(lr);
    c.momentum = static_cast<real>(mom);
    c.weight_decay = static_cast<real>(wd);
    c.rms_decay = static_cast<real>(decay);
    c.epsilon = static_cast<real>(eps);
    auto s = std::make_unique<pg_solver>();
    s->solver = std::make_unique<polegrad::Solver>(c);
    *out = s.release();
  });
}

int pg_solver_free(pg_solver* s) { return run([&] { delete s; }); }

int pg_solver_apply(pg_solver* s, pg_net* n) { return run([&] { s->solver->apply_update(net_of(n)); }); }

int pg_solver_snapshot(pg_solver* s, uint8_t* buf, uint64_t cap, uint64_t* len) {
  return run([&] {
    const auto bytes = s->solver->snapshot_state();
    *len = bytes.size();
    if (buf && cap >= bytes.size()) std::memcpy(buf, bytes.data(), bytes.size());
  });
}

int pg_solver_restore(pg_solver* s, const uint8_t* buf, uint64_t len) {
  return run([&] { s->solver->restore_state(std::span<const std::uint8_t>(buf, len)); });
}

int pg_solver_iterations(pg_solver* s, uint64_t* out) {
  return run([&] { *out = s->solver->iterations(); });
}

struct pg_feed_ring {
  std::unique_ptr<polegrad::FeedRing> ring;
};

int pg_feed_ring_create(pg_net* n, pg_solver* s, int depth, pg_feed_ring** out) {
  return run([&] {
    auto r = std::make_unique<pg_feed_ring>();
    r->ring = std::make_unique<polegrad::FeedRing>(net_of(n), *s->solver, depth);
    *out = r.release();
  });
}

int pg_feed_ring_free(pg_feed_ring* r) { return run([&] { delete r; }); }

int pg_feed_ring_push(pg_feed_ring* r, const void* data, uint64_t n_data, const void* labels, uint64_t n_labels) {
  return run([&] {
    r->ring->push(std::span<const real>(static_cast<const real*>(data), n_data),
                  std::span<const real>(static_cast<const real*>(labels), labels ? n_labels : 0));
  });
}

int pg_feed_ring_push_pinned(pg_feed_ring* r, const void* data, uint64_t n_data, const void* labels,
                             uint64_t n_labels) {
  return run([&] {
    r->ring->push_pinned(std::span<const real>(static_cast<const real*>(data), n_data),
                         std::span<const real>(static_cast<const real*>(labels), labels ? n_labels : 0));
  });
}

int pg_feed_ring_pop_loss(pg_feed_ring* r, double* loss) { return run([&] { *loss = r->ring->pop_loss(); }); }

struct pg_imagedb {
  polegrad::imagedb::Dataset db;
};
struct pg_rng {
  polegrad::Rng rng;
};

namespace {
polegrad::imagedb::SampleMethod sample_method(int method) {
  if (method != 0 && method != 1) throw polegrad::InvalidArgument("sample method must be 0 (uniform) or 1 (label balanced)");
  return method ? polegrad::imagedb::SampleMethod::kLabelBalanced : polegrad::imagedb::SampleMethod::kUniform;
}
}  // namespace

int pg_feed_ring_push_sampled(pg_feed_ring* r, const pg_imagedb* db, int method, int use_boost, pg_rng* rng) {
  return run([&] {
    if (!r || !db || !rng) throw polegrad::InvalidArgument("null ring, dataset or rng");
    r->ring->push_sampled(db->db, sample_method(method), use_boost != 0, rng->rng);
  });
}

int pg_imagedb_load(const char* index_path, pg_imagedb** out) {
  return run([&] {
    if (!index_path || !out) throw polegrad::InvalidArgument("null path or out");
    auto d = std::make_unique<pg_imagedb>();
    d->db = polegrad::imagedb::load(index_path);
    *out = d.release();
  });
}

int pg_imagedb_free(pg_imagedb* db) { return run([&] { delete db; }); }

int pg_imagedb_size(const pg_imagedb* db, uint64_t* out) { return run([&] { *out = db->db.size(); }); }

int pg_imagedb_set_boost(pg_imagedb* db, int64_t id, double boost) {
  return run([&] { db->db.set_boost(id, static_cast<real>(boost)); });
}

int pg_imagedb_sample(const pg_imagedb* db, int method, int use_boost, pg_rng* rng, uint64_t n, int64_t* ids) {
  return run([&] {
    if (!db || !rng || (n && !ids)) throw polegrad::InvalidArgument("null dataset, rng or ids");
    const auto m = sample_method(method);
    for (uint64_t i = 0; i < n; ++i) ids[i] = db->db.sample(m, use_boost != 0, rng->rng).id;
  });
}

int pg_rng_create(uint64_t seed, pg_rng** out) {
  return run([&] { *out = new pg_rng{polegrad::Rng(seed)}; });
}

int pg_rng_free(pg_rng* rng) { return run([&] { delete rng; }); }

int pg_step_capture(pg_net* n, pg_solver* s, const void* data, const void* labels, void* loss_out, uint64_t* graph) {
  return run([&] {
    polegrad::Net& net = net_of(n);
    polegrad::Registry& reg = *net.registry();
    reg.synchronize();
    cdnn_ok(cdnn_graph_begin(reg.context(), reg.stream()), "step capture");
    try {
      if (data) net.set_batch(static_cast<const real*>(data), static_cast<const real*>(labels));
      else net.reuse_resident_batch();  // inputs already in HBM
      if (!net.graph_safe()) throw polegrad::InvalidState("step capture: net has host-side layers (loss hooks / FIFO feed)");
      net.forward();
      net.backward();
      s->solver->apply_update(net);
      if (loss_out) {
        // loss top(s) of the net; the graph ends with their D2H copy
        if (net.loss_blobs().empty()) throw polegrad::InvalidState("step capture: net has no loss top");
        cdnn_ok(cdnn_read_async(reg.context(), net.loss_blobs()[0]->gpu_data(), 0, loss_out, 1, reg.stream()),
                "step capture");
      }
    } catch (...) {
      cdnn_handle dead = 0;
      cdnn_graph_end(reg.context(), reg.stream(), &dead);
      if (dead) cdnn_graph_free(reg.context(), dead);
      throw;
    }
    cdnn_handle g = 0;
    cdnn_ok(cdnn_graph_end(reg.context(), reg.stream(), &g), "step capture");
    *graph = g;
  });
}

namespace {
// the fused one-kernel update applies (PG_STEP_LAYERED not set, softmax head, no Parallel)
std::optional<polegrad::Net::MlpPgPlan> fused_plan(polegrad::Net& net, pg_solver* s, const char* logit_blob,
                                                   const char* prob_blob, int sigmoid, int flags) {
  if ((flags & PG_STEP_LAYERED) || sigmoid || s->solver->has_parallel()) return std::nullopt;
  return net.mlp_pg_plan(logit_blob, prob_blob);
}
}  // namespace

int pg_pg_step_fused(pg_net* n, pg_solver* s, const char* logit_blob, const char* prob_blob, int sigmoid,
                     int flags, int* out) {
  return run([&] {
    if (!out) throw polegrad::InvalidArgument("pg_pg_step_fused: null out");
    *out = fused_plan(net_of(n), s, logit_blob, prob_blob, sigmoid, flags).has_value() ? 1 : 0;
  });
}

int pg_pg_step_capture(pg_net* n, pg_solver* s, const void* states, const void* actions, const void* returns,
                       uint64_t count, const char* logit_blob, const char* prob_blob, int sigmoid, void* prob_out,
                       uint64_t* graph) {
  return pg_pg_step_capture_ex(n, s, states, actions, returns, count, logit_blob, prob_blob, sigmoid, 0, prob_out,
                               graph);
}

int pg_pg_step_capture_ex(pg_net* n, pg_solver* s, const void* states, const void* actions, const void* returns,
                          uint64_t count, const char* logit_blob, const char* prob_blob, int sigmoid, int flags,
                          void* prob_out, uint64_t* graph) {
  return run([&] {
    polegrad::Net& net = net_of(n);
    polegrad::Registry& reg = *net.registry();
    if (!states || !actions || !returns) throw polegrad::InvalidArgument("pg step capture: null input buffer");
    const auto plan = fused_plan(net, s, logit_blob, prob_blob, sigmoid, flags);
    if (plan) {  // the history and the action / return buffers exist before the capture
      s->solver->prepare(net);
      net.pg_stage_async(nullptr, nullptr, 0);
    }
    // one eager update first: lazily allocated buffers must exist before the capture
    reg.synchronize();
    cdnn_ok(cdnn_graph_begin(reg.context(), reg.stream()), "pg step capture");
    try {
      if (plan) {
        // ONE kernel node: states / actions / returns read from the page-locked host
        // buffers, forward, softmax gradient at the logits, backward, solver rule,
        // probabilities written to prob_out (no copy nodes)
        s->solver->apply_mlp_pg(net, *plan, count, static_cast<const real*>(states),
                                static_cast<const real*>(actions), static_cast<const real*>(returns),
                                static_cast<real*>(prob_out));
      } else {
        net.set_batch(static_cast<const real*>(states), nullptr);
        net.forward();
        net.pg_backward_async(logit_blob, prob_blob, static_cast<const real*>(actions),
                              static_cast<const real*>(returns), count, sigmoid != 0);
        s->solver->apply_update(net);
      }
      if (prob_out && !plan) {
        polegrad::Blob& prob = net.blob(prob_blob);
        cdnn_ok(cdnn_read_async(reg.context(), prob.gpu_data(), 0, prob_out, prob.count(), reg.stream()),
                "pg step capture");
      }
    } catch (...) {
      cdnn_handle dead = 0;
      cdnn_graph_end(reg.context(), reg.stream(), &dead);
      if (dead) cdnn_graph_free(reg.context(), dead);
      throw;
    }
    cdnn_handle g = 0;
    cdnn_ok(cdnn_graph_end(reg.context(), reg.stream(), &g), "pg step capture");
    *graph = g;
  });
}

int pg_net_profile(pg_net* n, float* fwd_ms, float* bwd_ms, int cap) {
  return run([&] {
    std::vector<float> f, b;
    net_of(n).profile_layers(f, b);
    if (cap < int(f.size())) throw polegrad::InvalidArgument("profile: buffer too small");
    std::copy(f.begin(), f.end(), fwd_ms);
    std::copy(b.begin(), b.end(), bwd_ms);
  });
}

int pg_step_replay(pg_net* n, uint64_t graph) {
  return run([&] {
    polegrad::Registry& reg = *net_of(n).registry();
    cdnn_ok(cdnn_graph_launch(reg.context(), graph, reg.stream()), "step replay");
    net_of(n).mark_device_fresh();
  });
}

int pg_graph_free(pg_net* n, uint64_t graph) {
  return run([&] { cdnn_ok(cdnn_graph_free(net_of(n).registry()->context(), graph), "graph free"); });
}

int pg_parallel_unique_id(uint8_t id[128]) {
  return run([&] {
    const auto u = polegrad::Parallel::unique_id();
    std::memcpy(id, u.data(), 128);
  });
}

int pg_parallel_create(pg_net* n, int nranks, int rank, const uint8_t id[128], uint64_t bucket_bytes,
                       pg_parallel** out) {
  return run([&] {
    polegrad::Parallel::UniqueId u;
    std::memcpy(u.data(), id, 128);
    auto p = std::make_unique<pg_parallel>();
    p->par = std::make_unique<polegrad::Parallel>(net_of(n), nranks, rank, u,
                                                  bucket_bytes ? bucket_bytes : (std::size_t(8) << 20));
    *out = p.release();
  });
}

int pg_parallel_create_host(pg_net* n, int nranks, int rank, pg_host_transport transport, void* user,
                            uint64_t bucket_bytes, pg_parallel** out) {
  return run([&] {
    if (!transport) throw polegrad::InvalidArgument("pg_parallel_create_host: null transport");
    auto fn = [transport, user](int op, polegrad::real* host, std::size_t offset, std::size_t count) {
      if (transport(user, op, host, offset, count) != 0)
        throw polegrad::InvalidState("Parallel host transport failed (op " + std::to_string(op) + ")");
    };
    auto p = std::make_unique<pg_parallel>();
    p->par = std::make_unique<polegrad::Parallel>(net_of(n), nranks, rank, fn,
                                                  bucket_bytes ? bucket_bytes : (std::size_t(8) << 20));
    *out = p.release();
  });
}

int pg_parallel_info(pg_parallel* p, int* nranks, int* rank, int* nbuckets, uint64_t* launches) {
  return run([&] {
    const auto [n, r] = p->par->comm_info();
    if (nranks) *nranks = n;
    if (rank) *rank = r;
    if (nbuckets) *nbuckets = int(p->par->buckets().size());
    if (launches) *launches = p->par->launches();
  });
}

int pg_parallel_free(pg_parallel* p) { return run([&] { delete p; }); }
int pg_parallel_broadcast(pg_parallel* p) { return run([&] { p->par->broadcast_weights(); }); }
int pg_solver_set_parallel(pg_solver* s, pg_parallel* p) {
  return run([&] { s->solver->set_parallel(p ? p->par.get() : nullptr); });
}

int pg_plan_buckets(const uint64_t* offsets, const uint64_t* counts, int n, uint64_t total, uint64_t bucket_elems,
                    int32_t* bucket_of, int32_t* nbuckets) {
  return run([&] {
    std::vector<std::size_t> o(offsets, offsets + n), c(counts, counts + n);
    const auto bs = polegrad::plan_buckets(o, c, total, bucket_elems);
    for (int i = 0; i < n; ++i) {
      bucket_of[i] = -1;
      for (std::size_t b = 0; b < bs.size(); ++b)
        if (o[i] >= bs[b].begin && o[i] < bs[b].end) bucket_of[i] = int32_t(b);
    }
    *nbuckets = int32_t(bs.size());
  });
}

int pg_prototxt_roundtrip(const char* text, char* out, uint64_t cap, uint64_t* len) {
  return run([&] {
    const std::string s = polegrad::prototxt::print(polegrad::prototxt::parse(text));
    *len = s.size();
    if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

}  // extern "C"
