// internal.hpp — CudaDnn context and handle look-up tables (paper Table 3).
//
// One cdnn_context per device.  Every resource lives in one table keyed by a
// monotone 64-bit id (never recycled, 0 = null; backend.hpp:17-25,
// backend.cpp:18-26).  Table mutation is serialised by the context mutex
// (backend.hpp:113); buffer contents are ordered by streams only.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <functional>
#include <cstdint>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <unordered_map>
#include <variant>
#include <vector>

#include "cudadnn.h"
#include "operands.cuh"

namespace cdnn {

struct Error {
  int status;
  std::string msg;
};
[[noreturn]] void fail(int status, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define CDNN_CUDA(x) ::cdnn::check_cuda((x), #x)

size_t dtype_size(int dtype);

struct DevAlloc {
  void* ptr = nullptr;
  size_t bytes = 0;
  int device = 0;
  ~DevAlloc();
};

struct BufferSlot {
  std::shared_ptr<DevAlloc> alloc;  // shared with views (arena sub-ranges)
  char* dev = nullptr;              // first element of this buffer / view
  uint64_t len = 0;
  int dtype = CDNN_F32;
};

// Split-K partial-sum scratch bound to one stream.  Grows by allocating a new
// block and retiring (not freeing) the old one, so CUDA graphs captured
// against an older block stay valid for the context's lifetime.
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
  std::vector<std::shared_ptr<DevAlloc>> blocks;
  void* get(size_t need, int device);
  // a second, independent scratch on the same stream (operand transposes that must
  // stay alive while the split-K partials use this one)
  std::unique_ptr<Workspace> second;
  Workspace& aux() {
    if (!second) second = std::make_unique<Workspace>();
    return *second;
  }
};

struct StreamSlot {
  cudaStream_t s = nullptr;
  std::shared_ptr<Workspace> ws;
};

struct ConvDescSlot {
  cdnn_conv_params p{};
  int P = 0, Q = 0;
  ConvGeom geom{};
  int Kc = 0;    // Cg*R*S   (forward reduction / backward-filter rows)
  int Kd = 0;    // Cog*R*S  (backward-data reduction)
  std::shared_ptr<DevAlloc> tables;  // taps | dtaps | koff
  ConvTap* taps = nullptr;
  DgradTap* dtaps = nullptr;
  int* koff = nullptr;
  // repacked per-tap weights for the TMA direct-conv path (lazily allocated):
  // [0] forward hi, [1] forward lo, [2] backward-data hi, [3] backward-data lo
  std::shared_ptr<DevAlloc> repack[4];
  // zero-inserted dY (strided backward through the stride-1 tap kernels), grow-only;
  // [0] backward-data, [1] backward-filter (they may run on two streams at once)
  std::shared_ptr<DevAlloc> upsampled[2];
  // space-to-depth rewrite of a strided convolution (stride s -> stride 1 over C*s*s
  // channels): the equivalent descriptor and its grow-only operand buffers
  // [0] X' forward, [1] W', [2] X' backward-filter, [3] dW', [4] dX'
  std::shared_ptr<ConvDescSlot> s2d;
  std::shared_ptr<DevAlloc> s2d_buf[5];
  const void* s2d_fwd_src = nullptr;  // input whose space-to-depth rewrite s2d_buf[0] holds
  // column fold of a small-channel stride-1 convolution (S filter columns folded
  // into C*S >= 16 channels, R x 1 kernel): descriptor and grow-only buffers
  // [0] X' forward, [1] W', [2] X' backward-filter, [3] dW'
  std::shared_ptr<ConvDescSlot> cf;
  std::shared_ptr<DevAlloc> cf_buf[4];
};

struct PoolDescSlot {
  cdnn_pool_params p{};
  int PH = 0, PW = 0;
};

struct RngSlot {
  std::mt19937_64 engine;
};

struct NcclSlot {
  void* comm = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0;
};

struct GraphSlot {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

struct EventSlot {
  cudaEvent_t ev = nullptr;
};

using Slot = std::variant<BufferSlot, StreamSlot, ConvDescSlot, PoolDescSlot, RngSlot, NcclSlot,
                          GraphSlot, EventSlot>;

}  // namespace cdnn

struct cdnn_context {
  int device = 0;
  cudaStream_t stream = nullptr;  // the context's own compute stream (handle 0)
  std::shared_ptr<cdnn::Workspace> ws;
  std::mutex mu;
  uint64_t next_id = 1;
  std::unordered_map<uint64_t, cdnn::Slot> slots;
  std::atomic<uint64_t> launches{0};
  int math_mode = CDNN_MATH_TF32X3;  // float GEMM numerics (cdnn_math_mode)
  std::mutex tmap_mu;
  std::unordered_map<std::string, CUtensorMap> tmaps;
};

namespace cdnn {

using Ctx = cdnn_context;

// RAII: make the context's device current for the duration of an entry point.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(Ctx* c);
  ~DeviceGuard();
};

uint64_t insert_slot(Ctx* c, Slot s);
BufferSlot& buffer(Ctx* c, cdnn_handle h, const char* what);
BufferSlot* buffer_or_null(Ctx* c, cdnn_handle h, const char* what);
ConvDescSlot& conv_desc(Ctx* c, cdnn_handle h);
PoolDescSlot& pool_desc(Ctx* c, cdnn_handle h);
RngSlot& rng(Ctx* c, cdnn_handle h);
NcclSlot& nccl(Ctx* c, cdnn_handle h);
cudaStream_t stream_of(Ctx* c, cdnn_handle h);
Workspace& workspace_of(Ctx* c, cdnn_handle h);
void require_len(const BufferSlot& b, uint64_t n, const char* what);
void require_dtype(const BufferSlot& b, int dtype, const char* what);

// Kernel launch bookkeeping + error check after every launch.
void count_launch(Ctx* c, int n = 1);
void check_launch(const char* what);

// Tensor map for a row-major fp32 matrix [rows][K] (row stride ld elements),
// box {32 k, box_rows}, 128B swizzle.  Cached per (ptr, shape, box).
const CUtensorMap* tmap_k_major(Ctx* c, const float* ptr, int rows, int K, int64_t ld,
                                int box_rows);
// Generic fp32 tensor map (rank <= 5): dims/strides in elements (innermost
// first, strides for dims 1..rank-1), box, swizzle span in bytes (32/64/128)
// or kSwizzle128Atom32 (SWIZZLE_128B_ATOM_32B: the MN-major tf32 UMMA layout).
constexpr int kSwizzle128Atom32 = 1;
const CUtensorMap* tmap_generic(Ctx* c, const float* ptr, int rank, const uint64_t* dims,
                                const uint64_t* strides_elems, const uint32_t* box, int swizzle_bytes);
std::shared_ptr<DevAlloc> device_alloc_shared(size_t bytes, int device);

// Plain GEMM-shaped launches shared by gemm / ip / conv (ops_gemm.cu).
struct GemmPlan {
  int bn = 128;
  int splits = 1;
  int kt_per_split = 1;
};
GemmPlan plan_tc(int M, int N, int K);
GemmPlan plan_simt(int M, int N, int K);

// Runs f under the C-ABI error guard; returns the cdnn_status.
int guarded(const std::function<void()>& f);
Ctx* need_ctx(cdnn_ctx c);

// nccl.cu: destroys a communicator held in an NcclSlot.
void nccl_destroy(void* comm);

}  // namespace cdnn
