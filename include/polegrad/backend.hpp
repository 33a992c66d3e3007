// polegrad/backend.hpp — handle registry and kernel entry points, now backed
// by the B200 CudaDnn C-ABI (include/cudadnn.h).
//
// Source-compatible with the reference backend (backend.hpp:14-144): Handle,
// HandleKind, Rng, fn::k* dispatch indices, Registry and kernels::*.  What
// changed underneath:
//  * every buffer lives in HBM behind a cdnn buffer handle; the host span
//    returned by buffer() is a lazily materialised mirror with Caffe
//    SyncedMemory semantics (paper "SyncMem object"): a mutable span marks the
//    host copy newest, device kernels upload it on next use, kernel outputs
//    mark the device copy newest and the next span access downloads it;
//  * kernels::* and dispatch() launch sm_100a kernels (TF32 tensor cores for
//    float, SIMT FP64 for double) on the registry's device;
//  * ids are still per-registry, monotone, never recycled, 0 = null.
// A span obtained before a device operation that writes the same buffer is
// stale afterwards: re-fetch it (Caffe's cpu_data() contract).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <random>
#include <span>
#include <unordered_map>
#include <vector>

#include "polegrad/types.hpp"

namespace polegrad {

enum class HandleKind { kBuffer, kSubsystem };

// Opaque id into a Registry; 0 is null and never names a slot.
struct Handle {
  std::uint64_t id = 0;
  HandleKind kind = HandleKind::kBuffer;

  explicit operator bool() const { return id != 0; }
  bool operator==(const Handle&) const = default;
};

// mt19937_64 with the top-53-bit [0,1) mapping: bit-identical draws on every
// platform (reference backend.hpp:27-45).  Weight init and synthetic inputs
// are drawn on the host in this exact order, then uploaded.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}
  std::uint64_t next_u64() { return engine_(); }
  double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }

 private:
  std::mt19937_64 engine_;
};

// Frozen dispatch indices (reference backend.hpp:47-69; new ones only append,
// see CDNN_FN_* in cudadnn.h for 8..13).
namespace fn {
inline constexpr int kFill = 1;        // dst, n, value
inline constexpr int kCopy = 2;        // src, dst, n
inline constexpr int kScal = 3;        // n, alpha, x
inline constexpr int kAxpy = 4;        // n, alpha, x, y
inline constexpr int kDot = 5;         // n, x, y -> result
inline constexpr int kGemm = 6;        // trans_a, trans_b, m, n, k, alpha, a, b, beta, c
inline constexpr int kRngUniform = 7;  // rng, dst, n, lo, hi
}  // namespace fn

// One device context per GPU, shared by every Registry on that device.
cdnn_ctx device_context(int device = 0);

class Registry {
 public:
  Registry();                    // device 0
  explicit Registry(int device);
  ~Registry();
  Registry(const Registry&) = delete;
  Registry& operator=(const Registry&) = delete;

  // ---- reference API ------------------------------------------------------
  Handle alloc_buffer(std::size_t length);  // zero-filled; length 0 -> InvalidArgument
  void free_buffer(Handle h);
  std::size_t buffer_length(Handle h) const;
  void write(Handle h, std::span<const real> values);  // into elements [0, size)
  std::vector<real> read(Handle h) const;
  std::span<real> buffer(Handle h);              // host view, marks host newest
  std::span<const real> buffer(Handle h) const;  // host view, read only
  Handle create_rng(std::uint64_t seed);
  Rng& rng(Handle h);
  void free_subsystem(Handle h);
  std::size_t live_slots() const;
  std::vector<real> dispatch(int function_index, std::span<const real> args);

  // ---- device side (B200) ---------------------------------------------------
  // Per-buffer coherence record.  Stable address for the buffer's lifetime.
  struct Buffer {
    cdnn_handle dev = 0;
    std::size_t len = 0;
    std::vector<real> host;  // empty until first host access
    enum class Head { kDevice, kHost, kSynced } head = Head::kDevice;
  };
  Buffer& record(Handle h) const;
  // cdnn handle of a buffer whose current contents a kernel will READ.
  cdnn_handle in(Handle h) const;
  // ... that a kernel will READ AND WRITE (e.g. beta = 1 accumulation).
  cdnn_handle inout(Handle h);
  // ... that a kernel will fully OVERWRITE (no upload of stale host data).
  cdnn_handle out(Handle h);
  static cdnn_handle in(Buffer& b, cdnn_ctx ctx);
  static cdnn_handle inout(Buffer& b, cdnn_ctx ctx);
  static cdnn_handle out(Buffer& b);
  static void to_host(Buffer& b, cdnn_ctx ctx);

  // A new buffer id aliasing elements [offset, offset+length) of `parent`
  // (flat parameter / gradient arenas).  The view has its own host mirror;
  // device kernels on the parent and on views see the same HBM.
  Handle alloc_view(Handle parent, std::size_t offset, std::size_t length);

  cdnn_ctx context() const { return ctx_; }
  int device() const { return device_; }
  // Stream every kernel of this registry is queued on (0 = context stream).
  cdnn_handle stream() const { return stream_; }
  void set_stream(cdnn_handle s) { stream_ = s; }
  void synchronize() const;

 private:
  struct Slot;
  Slot& slot(std::uint64_t id) const;

  int device_ = 0;
  cdnn_ctx ctx_ = nullptr;
  cdnn_handle stream_ = 0;
  mutable std::mutex mutex_;
  std::unordered_map<std::uint64_t, std::unique_ptr<Slot>> slots_;
  std::uint64_t next_id_ = 1;
};

namespace kernels {

void fill(Registry& reg, Handle dst, std::size_t n, real value);                  // dst[0,n) = value
void copy(Registry& reg, Handle src, Handle dst, std::size_t n);                  // dst[0,n) = src[0,n)
void scal(Registry& reg, std::size_t n, real alpha, Handle x);                    // x *= alpha
void axpy(Registry& reg, std::size_t n, real alpha, Handle x, Handle y);          // y += alpha x
real dot(Registry& reg, std::size_t n, Handle x, Handle y);
// Row-major C = alpha op(A) op(B) + beta C; beta == 0 never reads C.
void gemm(Registry& reg, bool trans_a, bool trans_b, int m, int n, int k, real alpha, Handle a, Handle b,
          real beta, Handle c);
// dst[0,n) = uniform draws in [lo, hi) from the rng subsystem, in order.
void rng_uniform(Registry& reg, Handle rng, Handle dst, std::size_t n, real lo, real hi);

}  // namespace kernels

}  // namespace polegrad
