// backend.cpp — Registry over the CudaDnn C-ABI (reference: backend.cpp).
//
// Registry ids are this object's own monotone counter (buffers and rngs
// share it, reference backend.cpp:18-26, 81-86); each buffer id maps to a
// cdnn buffer on the registry's device plus a lazily allocated host mirror.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <variant>

#include "polegrad/backend.hpp"
#include "polegrad/errors.hpp"

namespace polegrad {

// ---- errors -------------------------------------------------------------------
void throw_status(int status, const std::string& context) {
  const std::string msg = context.empty() ? std::string(cdnn_last_error())
                                          : context + ": " + cdnn_last_error();
  switch (status) {
    case CDNN_INVALID_ARGUMENT: throw InvalidArgument(msg);
    case CDNN_DANGLING_HANDLE: throw DanglingHandle(msg);
    case CDNN_UNKNOWN_FUNCTION: throw UnknownFunction(msg);
    case CDNN_MODEL_ERROR: throw ModelError(msg);
    case CDNN_DATA_STARVATION: throw DataStarvation(msg);
    case CDNN_FORMAT_ERROR: throw FormatError(msg);
    case CDNN_NOT_FOUND: throw NotFound(msg);
    case CDNN_INVALID_STATE: throw InvalidState(msg);
    case CDNN_PARSE_ERROR: throw ParseError(0, msg);
    case CDNN_LOAD_ERROR: throw LoadError(0, msg);
    default: throw DeviceError(msg);
  }
}

// ---- per-device contexts ------------------------------------------------------------
cdnn_ctx device_context(int device) {
  static std::mutex mu;
  static std::vector<cdnn_ctx> ctxs;
  std::lock_guard lock(mu);
  if (device < 0) throw InvalidArgument("device_context: negative device");
  if (ctxs.size() <= std::size_t(device)) ctxs.resize(std::size_t(device) + 1, nullptr);
  if (!ctxs[device]) {
    cdnn_ctx c = nullptr;
    cdnn_ok(cdnn_ctx_create(device, &c), "device_context");
    ctxs[device] = c;  // process lifetime: shared by every Registry on the device
  }
  return ctxs[device];
}

namespace {
std::string handle_label(std::uint64_t id) { return "handle " + std::to_string(id); }
}  // namespace

struct Registry::Slot {
  std::variant<Buffer, Rng> v;
};

Registry::Registry() : Registry(0) {}

Registry::Registry(int device) : device_(device), ctx_(device_context(device)) {}

Registry::~Registry() {
  std::lock_guard lock(mutex_);
  for (auto& [id, s] : slots_) {
    if (auto* b = std::get_if<Buffer>(&s->v)) cdnn_free(ctx_, b->dev);
  }
}

Registry::Slot& Registry::slot(std::uint64_t id) const {
  std::lock_guard lock(mutex_);
  auto it = slots_.find(id);
  if (id == 0 || it == slots_.end()) throw DanglingHandle(handle_label(id) + " is not live");
  return *it->second;
}

Registry::Buffer& Registry::record(Handle h) const {
  Slot& s = slot(h.id);
  auto* b = std::get_if<Buffer>(&s.v);
  if (!b) throw InvalidArgument(handle_label(h.id) + " is not a buffer");
  return *b;
}

Handle Registry::alloc_buffer(std::size_t length) {
  if (length == 0) throw InvalidArgument("alloc_buffer: length must be > 0");
  Buffer b;
  cdnn_ok(cdnn_alloc(ctx_, length, kRealDtype, &b.dev), "alloc_buffer");
  b.len = length;
  b.head = Buffer::Head::kDevice;  // device copy is zero-filled; host mirror not materialised
  auto s = std::make_unique<Slot>(Slot{std::move(b)});
  std::lock_guard lock(mutex_);
  const std::uint64_t id = next_id_++;
  slots_.emplace(id, std::move(s));
  return Handle{id, HandleKind::kBuffer};
}

Handle Registry::alloc_view(Handle parent, std::size_t offset, std::size_t length) {
  Buffer& p = record(parent);
  if (length == 0 || offset + length > p.len) throw InvalidArgument("alloc_view: range exceeds the parent buffer");
  Buffer b;
  cdnn_ok(cdnn_view(ctx_, in(p, ctx_), offset, length, &b.dev), "alloc_view");
  b.len = length;
  b.head = Buffer::Head::kDevice;
  auto s = std::make_unique<Slot>(Slot{std::move(b)});
  std::lock_guard lock(mutex_);
  const std::uint64_t id = next_id_++;
  slots_.emplace(id, std::move(s));
  return Handle{id, HandleKind::kBuffer};
}

void Registry::free_buffer(Handle h) {
  std::unique_ptr<Slot> dead;
  {
    std::lock_guard lock(mutex_);
    auto it = slots_.find(h.id);
    if (h.id == 0 || it == slots_.end()) throw DanglingHandle("free_buffer: " + handle_label(h.id) + " is not live");
    if (!std::holds_alternative<Buffer>(it->second->v))
      throw InvalidArgument("free_buffer: " + handle_label(h.id) + " is not a buffer");
    dead = std::move(it->second);
    slots_.erase(it);
  }
  cdnn_ok(cdnn_free(ctx_, std::get<Buffer>(dead->v).dev), "free_buffer");
}

std::size_t Registry::buffer_length(Handle h) const { return record(h).len; }

void Registry::to_host(Buffer& b, cdnn_ctx ctx) {
  if (b.host.empty()) b.host.resize(b.len);
  if (b.head == Buffer::Head::kDevice) {
    cdnn_ok(cdnn_read(ctx, b.dev, b.host.data(), b.len), "host sync");
    b.head = Buffer::Head::kSynced;
  }
}

cdnn_handle Registry::in(Buffer& b, cdnn_ctx ctx) {
  if (b.head == Buffer::Head::kHost) {
    cdnn_ok(cdnn_write(ctx, b.dev, b.host.data(), b.len), "device sync");
    b.head = Buffer::Head::kSynced;
  }
  return b.dev;
}

cdnn_handle Registry::inout(Buffer& b, cdnn_ctx ctx) {
  in(b, ctx);
  b.head = Buffer::Head::kDevice;
  return b.dev;
}

cdnn_handle Registry::out(Buffer& b) {
  b.head = Buffer::Head::kDevice;
  return b.dev;
}

cdnn_handle Registry::in(Handle h) const { return in(record(h), ctx_); }
cdnn_handle Registry::inout(Handle h) { return inout(record(h), ctx_); }
cdnn_handle Registry::out(Handle h) { return out(record(h)); }

void Registry::write(Handle h, std::span<const real> values) {
  Buffer& b = record(h);
  if (values.size() > b.len) {
    throw InvalidArgument("write: " + std::to_string(values.size()) + " values into a buffer of length " +
                          std::to_string(b.len));
  }
  if (values.empty()) return;
  if (b.head == Buffer::Head::kDevice) {
    // device copy is newest: write the prefix straight into HBM
    cdnn_ok(cdnn_write(ctx_, b.dev, values.data(), values.size()), "write");
    return;
  }
  std::copy(values.begin(), values.end(), b.host.begin());
  b.head = Buffer::Head::kHost;
}

std::vector<real> Registry::read(Handle h) const {
  Buffer& b = record(h);
  to_host(b, ctx_);
  return b.host;
}

std::span<real> Registry::buffer(Handle h) {
  Buffer& b = record(h);
  to_host(b, ctx_);
  b.head = Buffer::Head::kHost;
  return std::span<real>(b.host.data(), b.len);
}

std::span<const real> Registry::buffer(Handle h) const {
  Buffer& b = record(h);
  to_host(b, ctx_);
  return std::span<const real>(b.host.data(), b.len);
}

Handle Registry::create_rng(std::uint64_t seed) {
  auto s = std::make_unique<Slot>(Slot{Rng(seed)});
  std::lock_guard lock(mutex_);
  const std::uint64_t id = next_id_++;
  slots_.emplace(id, std::move(s));
  return Handle{id, HandleKind::kSubsystem};
}

Rng& Registry::rng(Handle h) {
  std::lock_guard lock(mutex_);
  auto it = slots_.find(h.id);
  if (h.id == 0 || it == slots_.end()) throw DanglingHandle("rng: " + handle_label(h.id) + " is not live");
  auto* r = std::get_if<Rng>(&it->second->v);
  if (!r) throw InvalidArgument("rng: " + handle_label(h.id) + " is not a rng subsystem");
  return *r;
}

void Registry::free_subsystem(Handle h) {
  std::lock_guard lock(mutex_);
  auto it = slots_.find(h.id);
  if (h.id == 0 || it == slots_.end()) throw DanglingHandle("free_subsystem: " + handle_label(h.id) + " is not live");
  if (!std::holds_alternative<Rng>(it->second->v))
    throw InvalidArgument("free_subsystem: " + handle_label(h.id) + " is not a subsystem");
  slots_.erase(it);
}

std::size_t Registry::live_slots() const {
  std::lock_guard lock(mutex_);
  return slots_.size();
}

void Registry::synchronize() const { cdnn_ok(cdnn_stream_sync(ctx_, stream_), "synchronize"); }

// ---- kernels --------------------------------------------------------------------------
namespace kernels {

namespace {
void check_length(const Registry& reg, Handle h, std::size_t n, const char* what) {
  const std::size_t len = reg.buffer_length(h);
  if (len < n) {
    throw InvalidArgument(std::string(what) + ": buffer of length " + std::to_string(len) + " is shorter than " +
                          std::to_string(n));
  }
}
}  // namespace

void fill(Registry& reg, Handle dst, std::size_t n, real value) {
  check_length(reg, dst, n, "fill");
  if (n == 0) return;
  cdnn_handle d = n == reg.buffer_length(dst) ? reg.out(dst) : reg.inout(dst);
  cdnn_ok(cdnn_fill(reg.context(), d, n, static_cast<double>(value), reg.stream()), "fill");
}

void copy(Registry& reg, Handle src, Handle dst, std::size_t n) {
  check_length(reg, src, n, "copy");
  check_length(reg, dst, n, "copy");
  if (n == 0) return;
  cdnn_handle s = reg.in(src);
  cdnn_handle d = n == reg.buffer_length(dst) ? reg.out(dst) : reg.inout(dst);
  cdnn_ok(cdnn_copy(reg.context(), s, d, n, reg.stream()), "copy");
}

void scal(Registry& reg, std::size_t n, real alpha, Handle x) {
  check_length(reg, x, n, "scal");
  if (n == 0) return;
  cdnn_ok(cdnn_scal(reg.context(), n, static_cast<double>(alpha), reg.inout(x), reg.stream()), "scal");
}

void axpy(Registry& reg, std::size_t n, real alpha, Handle x, Handle y) {
  check_length(reg, x, n, "axpy");
  check_length(reg, y, n, "axpy");
  if (n == 0) return;
  cdnn_handle xs = reg.in(x);
  cdnn_ok(cdnn_axpy(reg.context(), n, static_cast<double>(alpha), xs, reg.inout(y), reg.stream()), "axpy");
}

real dot(Registry& reg, std::size_t n, Handle x, Handle y) {
  check_length(reg, x, n, "dot");
  check_length(reg, y, n, "dot");
  if (n == 0) return real(0);
  double r = 0;
  cdnn_handle xs = reg.in(x), ys = reg.in(y);
  if (reg.stream() != 0) reg.synchronize();
  cdnn_ok(cdnn_dot(reg.context(), n, xs, ys, &r), "dot");
  return static_cast<real>(r);
}

void gemm(Registry& reg, bool trans_a, bool trans_b, int m, int n, int k, real alpha, Handle a, Handle b,
          real beta, Handle c) {
  if (m <= 0 || n <= 0 || k <= 0) throw InvalidArgument("gemm: m, n, k must be positive");
  check_length(reg, a, std::size_t(m) * std::size_t(k), "gemm A");
  check_length(reg, b, std::size_t(k) * std::size_t(n), "gemm B");
  check_length(reg, c, std::size_t(m) * std::size_t(n), "gemm C");
  cdnn_handle ah = reg.in(a), bh = reg.in(b);
  cdnn_handle ch = beta == real(0) && std::size_t(m) * n == reg.buffer_length(c) ? reg.out(c) : reg.inout(c);
  cdnn_ok(cdnn_gemm(reg.context(), trans_a, trans_b, m, n, k, static_cast<double>(alpha), ah, bh,
                    static_cast<double>(beta), ch, reg.stream()),
          "gemm");
}

void rng_uniform(Registry& reg, Handle rng_h, Handle dst, std::size_t n, real lo, real hi) {
  check_length(reg, dst, n, "rng_uniform");
  Rng& r = reg.rng(rng_h);
  if (n == 0) return;
  // Draw on the host in order (bit-exact stream), then upload the prefix.
  std::vector<real> v(n);
  for (auto& x : v) x = static_cast<real>(r.uniform(lo, hi));
  reg.write(dst, v);
}

}  // namespace kernels

// ---- dispatch (reference backend.cpp:213-305) ---------------------------------------
namespace {

Handle decode_handle(real v, HandleKind kind, const char* what) {
  if (!(v >= 0) || v != std::floor(v))
    throw InvalidArgument(std::string(what) + ": " + std::to_string(v) + " is not a handle id");
  return Handle{static_cast<std::uint64_t>(v), kind};
}
std::size_t decode_size(real v, const char* what) {
  if (!(v >= 0) || v != std::floor(v))
    throw InvalidArgument(std::string(what) + ": " + std::to_string(v) + " is not a valid count");
  return static_cast<std::size_t>(v);
}
int decode_int(real v, const char* what) {
  if (v != std::floor(v)) throw InvalidArgument(std::string(what) + ": " + std::to_string(v) + " is not an integer");
  return static_cast<int>(v);
}
void check_arity(int index, const char* name, std::span<const real> args, std::size_t expected) {
  if (args.size() != expected) {
    throw InvalidArgument("dispatch: function " + std::to_string(index) + " (" + name + ") expects " +
                          std::to_string(expected) + " arguments, got " + std::to_string(args.size()));
  }
}

}  // namespace

// Arity and argument decoding happen here with the reference's rules and
// messages; the decoded call then crosses the C-ABI through cdnn_dispatch with
// device handle ids, so dispatch() and the direct kernels::* call run the same
// device kernel and leave bit-identical buffers.
std::vector<real> Registry::dispatch(int fi, std::span<const real> args) {
  auto dev_in = [&](real v, const char* what) { return double(in(decode_handle(v, HandleKind::kBuffer, what))); };
  auto dev_io = [&](real v, const char* what) { return double(inout(decode_handle(v, HandleKind::kBuffer, what))); };
  std::vector<double> a;
  switch (fi) {
    case fn::kFill: {
      check_arity(fi, "fill", args, 3);
      const Handle d = decode_handle(args[0], HandleKind::kBuffer, "fill dst");
      const std::size_t n = decode_size(args[1], "fill n");
      if (buffer_length(d) < n)
        throw InvalidArgument("fill: buffer of length " + std::to_string(buffer_length(d)) + " is shorter than " +
                              std::to_string(n));
      a = {double(inout(d)), double(n), double(args[2])};
      break;
    }
    case fn::kCopy: {
      check_arity(fi, "copy", args, 3);
      const std::size_t n = decode_size(args[2], "copy n");
      const Handle s = decode_handle(args[0], HandleKind::kBuffer, "copy src");
      const Handle d = decode_handle(args[1], HandleKind::kBuffer, "copy dst");
      if (buffer_length(s) < n || buffer_length(d) < n)
        throw InvalidArgument("copy: buffer of length " + std::to_string(std::min(buffer_length(s), buffer_length(d))) +
                              " is shorter than " + std::to_string(n));
      a = {double(in(s)), double(inout(d)), double(n)};
      break;
    }
    case fn::kScal: {
      check_arity(fi, "scal", args, 3);
      a = {double(decode_size(args[0], "scal n")), double(args[1]), dev_io(args[2], "scal x")};
      break;
    }
    case fn::kAxpy: {
      check_arity(fi, "axpy", args, 4);
      a = {double(decode_size(args[0], "axpy n")), double(args[1]), dev_in(args[2], "axpy x"), dev_io(args[3], "axpy y")};
      break;
    }
    case fn::kDot: {
      check_arity(fi, "dot", args, 3);
      a = {double(decode_size(args[0], "dot n")), dev_in(args[1], "dot x"), dev_in(args[2], "dot y")};
      break;
    }
    case fn::kGemm: {
      check_arity(fi, "gemm", args, 10);
      const bool ta = decode_int(args[0], "gemm trans_a") != 0, tb = decode_int(args[1], "gemm trans_b") != 0;
      const int m = decode_int(args[2], "gemm m"), n = decode_int(args[3], "gemm n"), k = decode_int(args[4], "gemm k");
      const Handle ah = decode_handle(args[6], HandleKind::kBuffer, "gemm a");
      const Handle bh = decode_handle(args[7], HandleKind::kBuffer, "gemm b");
      const Handle chd = decode_handle(args[9], HandleKind::kBuffer, "gemm c");
      if (m <= 0 || n <= 0 || k <= 0) throw InvalidArgument("gemm: m, n, k must be positive");
      a = {double(ta), double(tb), double(m), double(n), double(k), double(args[5]), double(in(ah)), double(in(bh)),
           double(args[8]), double(inout(chd))};
      break;
    }
    case fn::kRngUniform: {
      check_arity(fi, "rng_uniform", args, 5);
      // The RNG subsystem lives host side (bit-exact stream); same path as the direct call.
      kernels::rng_uniform(*this, decode_handle(args[0], HandleKind::kSubsystem, "rng_uniform rng"),
                           decode_handle(args[1], HandleKind::kBuffer, "rng_uniform dst"),
                           decode_size(args[2], "rng_uniform n"), args[3], args[4]);
      return {};
    }
    default:
      throw UnknownFunction("dispatch: no function with index " + std::to_string(fi));
  }
  if (stream_ != 0) synchronize();
  double out[4] = {0, 0, 0, 0};
  std::uint64_t nout = 4;
  cdnn_ok(cdnn_dispatch(ctx_, fi, a.data(), a.size(), out, &nout), "dispatch");
  std::vector<real> result;
  for (std::uint64_t i = 0; i < nout; ++i) result.push_back(static_cast<real>(out[i]));
  return result;
}

}  // namespace polegrad
