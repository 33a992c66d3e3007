// context.cu — contexts, handle look-up tables, buffers, streams, graphs,
// events, the host RNG subsystem, descriptors and the C-ABI error plumbing.
//
// Reference behaviour mirrored here (paths under /root/reference/proj/core):
//   alloc zero-filled, length 0 rejected            src/backend.cpp:18-25
//   free of 0 / unknown / freed id -> DanglingHandle src/backend.cpp:27-38
//   wrong-kind handle -> InvalidArgument            src/backend.cpp:34-36, 46-48
//   write longer than the buffer -> InvalidArgument src/backend.cpp:62-69
//   monotone never-recycled ids                     include/polegrad/backend.hpp:17-25
//   mt19937_64 + (u64>>11)*2^-53 uniform mapping    include/polegrad/backend.hpp:31-45
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cudaTypedefs.h>

#include "internal.hpp"

namespace cdnn {

namespace {
thread_local std::string g_last_error;
}

void fail(int status, const std::string& msg) { throw Error{status, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? CDNN_NO_DEVICE
                                                                    : CDNN_CUDA_ERROR,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case CDNN_F32: return 4;
    case CDNN_F64: return 8;
    case CDNN_I32: return 4;
  }
  fail(CDNN_INVALID_ARGUMENT, "unknown dtype " + std::to_string(dtype));
}

DevAlloc::~DevAlloc() {
  if (ptr) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(ptr);
    if (prev >= 0) cudaSetDevice(prev);
  }
}

static std::shared_ptr<DevAlloc> device_alloc(size_t bytes, int device) {
  auto a = std::make_shared<DevAlloc>();
  a->device = device;
  a->bytes = bytes;
  CDNN_CUDA(cudaMalloc(&a->ptr, bytes));
  return a;
}

void* Workspace::get(size_t need, int device) {
  if (need <= bytes) return ptr;
  size_t want = std::max(need, bytes * 2);
  want = (want + (1 << 20) - 1) & ~size_t((1 << 20) - 1);
  auto blk = device_alloc(want, device);
  blocks.push_back(blk);  // older blocks are retired, not freed (graph safety)
  ptr = blk->ptr;
  bytes = want;
  return ptr;
}

DeviceGuard::DeviceGuard(Ctx* c) {
  cudaGetDevice(&prev);
  if (prev != c->device) CDNN_CUDA(cudaSetDevice(c->device));
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

uint64_t insert_slot(Ctx* c, Slot s) {
  std::lock_guard lock(c->mu);
  const uint64_t id = c->next_id++;
  c->slots.emplace(id, std::move(s));
  return id;
}

static std::string label(cdnn_handle h) { return "handle " + std::to_string(h); }

template <class T>
static T& slot_as(Ctx* c, cdnn_handle h, const char* what, const char* kind) {
  std::lock_guard lock(c->mu);
  auto it = c->slots.find(h);
  if (h == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, std::string(what) + ": " + label(h) + " is not live");
  T* p = std::get_if<T>(&it->second);
  if (!p) fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": " + label(h) + " is not a " + kind);
  return *p;
}

BufferSlot& buffer(Ctx* c, cdnn_handle h, const char* what) {
  return slot_as<BufferSlot>(c, h, what, "buffer");
}
BufferSlot* buffer_or_null(Ctx* c, cdnn_handle h, const char* what) {
  return h == 0 ? nullptr : &buffer(c, h, what);
}
ConvDescSlot& conv_desc(Ctx* c, cdnn_handle h) {
  return slot_as<ConvDescSlot>(c, h, "conv", "convolution descriptor");
}
PoolDescSlot& pool_desc(Ctx* c, cdnn_handle h) {
  return slot_as<PoolDescSlot>(c, h, "pool", "pooling descriptor");
}
RngSlot& rng(Ctx* c, cdnn_handle h) { return slot_as<RngSlot>(c, h, "rng", "rng subsystem"); }
NcclSlot& nccl(Ctx* c, cdnn_handle h) { return slot_as<NcclSlot>(c, h, "nccl", "nccl communicator"); }

cudaStream_t stream_of(Ctx* c, cdnn_handle h) {
  if (h == 0) return c->stream;
  return slot_as<StreamSlot>(c, h, "stream", "stream").s;
}
Workspace& workspace_of(Ctx* c, cdnn_handle h) {
  if (h == 0) return *c->ws;
  return *slot_as<StreamSlot>(c, h, "stream", "stream").ws;
}

void require_len(const BufferSlot& b, uint64_t n, const char* what) {
  if (b.len < n) {
    fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": buffer of length " + std::to_string(b.len) +
                                    " is shorter than " + std::to_string(n));
  }
}
void require_dtype(const BufferSlot& b, int dtype, const char* what) {
  if (b.dtype != dtype) {
    fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": dtype mismatch (" + std::to_string(b.dtype) +
                                    " vs " + std::to_string(dtype) + ")");
  }
}

void count_launch(Ctx* c, int n) { c->launches.fetch_add(uint64_t(n), std::memory_order_relaxed); }

void check_launch(const char* what) { CDNN_CUDA(cudaGetLastError()); (void)what; }

// ---- tensor maps ---------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CDNN_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) fail(CDNN_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

const CUtensorMap* tmap_k_major(Ctx* c, const float* ptr, int rows, int K, int64_t ld, int box_rows) {
  char key[128];
  std::snprintf(key, sizeof key, "%p/%d/%d/%lld/%d", static_cast<const void*>(ptr), rows, K,
                static_cast<long long>(ld), box_rows);
  std::lock_guard lock(c->tmap_mu);
  auto it = c->tmaps.find(key);
  if (it != c->tmaps.end()) return &it->second;
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  const cuuint32_t box[2] = {32, cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(CDNN_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  auto res = c->tmaps.emplace(key, m);
  return &res.first->second;
}

const CUtensorMap* tmap_generic(Ctx* c, const float* ptr, int rank, const uint64_t* dims,
                                const uint64_t* strides_elems, const uint32_t* box, int swizzle_bytes) {
  char key[256];
  int n = std::snprintf(key, sizeof key, "g%p/%d/%d", static_cast<const void*>(ptr), rank, swizzle_bytes);
  for (int i = 0; i < rank; ++i)
    n += std::snprintf(key + n, sizeof key - size_t(n), "/%llu:%llu:%u", static_cast<unsigned long long>(dims[i]),
                       static_cast<unsigned long long>(i ? strides_elems[i - 1] : 1), box[i]);
  std::lock_guard lock(c->tmap_mu);
  auto it = c->tmaps.find(key);
  if (it != c->tmaps.end()) return &it->second;
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
    if (i) gs[i - 1] = strides_elems[i - 1] * 4;
  }
  const CUtensorMapSwizzle sw = swizzle_bytes == kSwizzle128Atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                : swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_NONE;
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cuuint32_t(rank), const_cast<float*>(ptr), gd, gs,
                           bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(CDNN_CUDA_ERROR, "cuTensorMapEncodeTiled (generic) failed (" + std::to_string(int(r)) + ")");
  auto res = c->tmaps.emplace(key, m);
  return &res.first->second;
}

std::shared_ptr<DevAlloc> device_alloc_shared(size_t bytes, int device) { return device_alloc(bytes, device); }

}  // namespace cdnn

using namespace cdnn;

namespace {
template <class F>
int guard(F&& f) {
  try {
    f();
    return CDNN_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return CDNN_CUDA_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CDNN_CUDA_ERROR;
  }
}
}  // namespace

Ctx* cdnn::need_ctx(cdnn_ctx c) {
  if (!c) fail(CDNN_INVALID_ARGUMENT, "null context");
  return c;
}
int cdnn::guarded(const std::function<void()>& f) { return guard(f); }

extern "C" {

const char* cdnn_last_error(void) { return g_last_error.c_str(); }

const char* cdnn_status_name(int s) {
  switch (s) {
    case CDNN_OK: return "OK";
    case CDNN_INVALID_ARGUMENT: return "INVALID_ARGUMENT";
    case CDNN_DANGLING_HANDLE: return "DANGLING_HANDLE";
    case CDNN_UNKNOWN_FUNCTION: return "UNKNOWN_FUNCTION";
    case CDNN_MODEL_ERROR: return "MODEL_ERROR";
    case CDNN_DATA_STARVATION: return "DATA_STARVATION";
    case CDNN_FORMAT_ERROR: return "FORMAT_ERROR";
    case CDNN_NOT_FOUND: return "NOT_FOUND";
    case CDNN_INVALID_STATE: return "INVALID_STATE";
    case CDNN_PARSE_ERROR: return "PARSE_ERROR";
    case CDNN_LOAD_ERROR: return "LOAD_ERROR";
    case CDNN_CUDA_ERROR: return "CUDA_ERROR";
    case CDNN_NO_DEVICE: return "NO_DEVICE";
  }
  return "UNKNOWN_STATUS";
}

int cdnn_device_count(int* out) {
  return guard([&] {
    if (!out) fail(CDNN_INVALID_ARGUMENT, "null out");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) { cudaGetLastError(); n = 0; }
    *out = n;
  });
}

int cdnn_ctx_create(int device, cdnn_ctx* out) {
  return guard([&] {
    if (!out) fail(CDNN_INVALID_ARGUMENT, "null out");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      fail(CDNN_NO_DEVICE, "cdnn_ctx_create: no CUDA device is visible (the B200 library has no CPU path)");
    }
    if (device < 0 || device >= n) fail(CDNN_INVALID_ARGUMENT, "cdnn_ctx_create: device " + std::to_string(device) + " out of range");
    cudaDeviceProp prop;
    CDNN_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      fail(CDNN_NO_DEVICE, std::string("cdnn_ctx_create: device is sm_") + std::to_string(prop.major) +
                               std::to_string(prop.minor) + "; this library is built for sm_100a only");
    }
    auto c = std::make_unique<cdnn_context>();
    c->device = device;
    int prev = -1;
    cudaGetDevice(&prev);
    CDNN_CUDA(cudaSetDevice(device));
    CDNN_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->ws = std::make_shared<Workspace>();
    if (const char* m = std::getenv("CDNN_MATH")) {
      if (std::string(m) == "tf32") c->math_mode = CDNN_MATH_TF32;
    }
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
    *out = c.release();
  });
}

int cdnn_ctx_destroy(cdnn_ctx ctx) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    {
      DeviceGuard g(c);
      cudaStreamSynchronize(c->stream);
      for (auto& [id, s] : c->slots) {
        if (auto* st = std::get_if<StreamSlot>(&s)) { cudaStreamSynchronize(st->s); cudaStreamDestroy(st->s); }
        if (auto* gr = std::get_if<GraphSlot>(&s)) {
          if (gr->exec) cudaGraphExecDestroy(gr->exec);
          if (gr->graph) cudaGraphDestroy(gr->graph);
        }
        if (auto* ev = std::get_if<EventSlot>(&s)) cudaEventDestroy(ev->ev);
      }
      c->slots.clear();
      c->ws.reset();
      cudaStreamDestroy(c->stream);
    }
    delete c;
  });
}

int cdnn_ctx_device(cdnn_ctx ctx, int* out) {
  return guard([&] { *out = need_ctx(ctx)->device; });
}

int cdnn_live_slots(cdnn_ctx ctx, uint64_t* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    std::lock_guard lock(c->mu);
    *out = c->slots.size();
  });
}

int cdnn_launch_count(cdnn_ctx ctx, uint64_t* out) {
  return guard([&] { *out = need_ctx(ctx)->launches.load(); });
}

int cdnn_set_math_mode(cdnn_ctx ctx, int mode) {
  return guard([&] {
    if (mode != CDNN_MATH_TF32 && mode != CDNN_MATH_TF32X3) fail(CDNN_INVALID_ARGUMENT, "unknown math mode");
    need_ctx(ctx)->math_mode = mode;
  });
}

int cdnn_get_math_mode(cdnn_ctx ctx, int* out) {
  return guard([&] { *out = need_ctx(ctx)->math_mode; });
}

// ---- buffers ---------------------------------------------------------------------
int cdnn_alloc(cdnn_ctx ctx, uint64_t length, int dtype, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    if (length == 0) fail(CDNN_INVALID_ARGUMENT, "alloc_buffer: length must be > 0");
    const size_t es = dtype_size(dtype);
    DeviceGuard g(c);
    BufferSlot b;
    b.alloc = device_alloc(length * es, c->device);
    CDNN_CUDA(cudaMemsetAsync(b.alloc->ptr, 0, length * es, c->stream));
    CDNN_CUDA(cudaStreamSynchronize(c->stream));
    b.dev = static_cast<char*>(b.alloc->ptr);
    b.len = length;
    b.dtype = dtype;
    *out = insert_slot(c, std::move(b));
  });
}

int cdnn_free(cdnn_ctx ctx, cdnn_handle h) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    std::shared_ptr<DevAlloc> keep;
    {
      std::lock_guard lock(c->mu);
      auto it = c->slots.find(h);
      if (h == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, "free_buffer: " + label(h) + " is not live");
      auto* b = std::get_if<BufferSlot>(&it->second);
      if (!b) fail(CDNN_INVALID_ARGUMENT, "free_buffer: " + label(h) + " is not a buffer");
      keep = std::move(b->alloc);
      c->slots.erase(it);
    }
    if (keep && keep.use_count() == 1) {
      // pending work may still reference the memory
      DeviceGuard g(c);
      cudaStreamSynchronize(c->stream);
    }
  });
}

int cdnn_view(cdnn_ctx ctx, cdnn_handle h, uint64_t offset, uint64_t length, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    BufferSlot b = buffer(c, h, "view");
    if (length == 0) fail(CDNN_INVALID_ARGUMENT, "view: length must be > 0");
    if (offset + length > b.len) fail(CDNN_INVALID_ARGUMENT, "view: range exceeds buffer");
    b.dev += offset * dtype_size(b.dtype);
    b.len = length;
    *out = insert_slot(c, std::move(b));
  });
}

int cdnn_length(cdnn_ctx ctx, cdnn_handle h, uint64_t* out) {
  return guard([&] { *out = buffer(need_ctx(ctx), h, "buffer_length").len; });
}
int cdnn_buffer_dtype(cdnn_ctx ctx, cdnn_handle h, int* out) {
  return guard([&] { *out = buffer(need_ctx(ctx), h, "buffer_dtype").dtype; });
}
int cdnn_device_ptr(cdnn_ctx ctx, cdnn_handle h, void** out) {
  return guard([&] { *out = buffer(need_ctx(ctx), h, "device_ptr").dev; });
}

int cdnn_write(cdnn_ctx ctx, cdnn_handle h, const void* host, uint64_t n) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    BufferSlot& b = buffer(c, h, "write");
    if (n > b.len) {
      fail(CDNN_INVALID_ARGUMENT, "write: " + std::to_string(n) + " values into a buffer of length " + std::to_string(b.len));
    }
    if (n == 0) return;
    if (!host) fail(CDNN_INVALID_ARGUMENT, "write: null host pointer");
    DeviceGuard g(c);
    CDNN_CUDA(cudaMemcpyAsync(b.dev, host, n * dtype_size(b.dtype), cudaMemcpyHostToDevice, c->stream));
    CDNN_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int cdnn_read(cdnn_ctx ctx, cdnn_handle h, void* host, uint64_t n) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    BufferSlot& b = buffer(c, h, "read");
    if (n > b.len) fail(CDNN_INVALID_ARGUMENT, "read: " + std::to_string(n) + " values from a buffer of length " + std::to_string(b.len));
    if (n == 0) return;
    DeviceGuard g(c);
    CDNN_CUDA(cudaMemcpyAsync(host, b.dev, n * dtype_size(b.dtype), cudaMemcpyDeviceToHost, c->stream));
    CDNN_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int cdnn_write_async(cdnn_ctx ctx, cdnn_handle h, uint64_t offset, const void* host, uint64_t n,
                     cdnn_handle stream) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    BufferSlot& b = buffer(c, h, "write_async");
    if (offset + n > b.len) fail(CDNN_INVALID_ARGUMENT, "write_async: range exceeds buffer");
    if (n == 0) return;
    DeviceGuard g(c);
    const size_t es = dtype_size(b.dtype);
    CDNN_CUDA(cudaMemcpyAsync(b.dev + offset * es, host, n * es, cudaMemcpyHostToDevice, stream_of(c, stream)));
  });
}

int cdnn_read_async(cdnn_ctx ctx, cdnn_handle h, uint64_t offset, void* host, uint64_t n,
                    cdnn_handle stream) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    BufferSlot& b = buffer(c, h, "read_async");
    if (offset + n > b.len) fail(CDNN_INVALID_ARGUMENT, "read_async: range exceeds buffer");
    if (n == 0) return;
    DeviceGuard g(c);
    const size_t es = dtype_size(b.dtype);
    CDNN_CUDA(cudaMemcpyAsync(host, b.dev + offset * es, n * es, cudaMemcpyDeviceToHost, stream_of(c, stream)));
  });
}

int cdnn_host_alloc_pinned(uint64_t bytes, void** out) {
  return guard([&] { CDNN_CUDA(cudaMallocHost(out, bytes ? bytes : 1)); });
}
int cdnn_host_free_pinned(void* p) {
  return guard([&] { CDNN_CUDA(cudaFreeHost(p)); });
}

// ---- streams / graphs / events -------------------------------------------------------
int cdnn_stream_create(cdnn_ctx ctx, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    DeviceGuard g(c);
    StreamSlot s;
    CDNN_CUDA(cudaStreamCreateWithFlags(&s.s, cudaStreamNonBlocking));
    s.ws = std::make_shared<Workspace>();
    *out = insert_slot(c, std::move(s));
  });
}

int cdnn_stream_free(cdnn_ctx ctx, cdnn_handle h) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    cudaStream_t s = nullptr;
    std::shared_ptr<Workspace> ws;
    {
      std::lock_guard lock(c->mu);
      auto it = c->slots.find(h);
      if (h == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, "stream_free: " + label(h) + " is not live");
      auto* st = std::get_if<StreamSlot>(&it->second);
      if (!st) fail(CDNN_INVALID_ARGUMENT, "stream_free: " + label(h) + " is not a stream");
      s = st->s;
      ws = st->ws;
      c->slots.erase(it);
    }
    DeviceGuard g(c);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  });
}

int cdnn_stream_sync(cdnn_ctx ctx, cdnn_handle stream) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    DeviceGuard g(c);
    CDNN_CUDA(cudaStreamSynchronize(stream_of(c, stream)));
  });
}

int cdnn_stream_wait(cdnn_ctx ctx, cdnn_handle stream, cdnn_handle on) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    DeviceGuard g(c);
    cudaEvent_t ev;
    CDNN_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CDNN_CUDA(cudaEventRecord(ev, stream_of(c, on)));
    CDNN_CUDA(cudaStreamWaitEvent(stream_of(c, stream), ev, 0));
    cudaEventDestroy(ev);
  });
}

int cdnn_graph_begin(cdnn_ctx ctx, cdnn_handle stream) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    DeviceGuard g(c);
    CDNN_CUDA(cudaStreamBeginCapture(stream_of(c, stream), cudaStreamCaptureModeThreadLocal));
  });
}

int cdnn_graph_end(cdnn_ctx ctx, cdnn_handle stream, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    DeviceGuard g(c);
    GraphSlot gs;
    CDNN_CUDA(cudaStreamEndCapture(stream_of(c, stream), &gs.graph));
    CDNN_CUDA(cudaGraphInstantiate(&gs.exec, gs.graph, 0));
    *out = insert_slot(c, std::move(gs));
  });
}

int cdnn_graph_launch(cdnn_ctx ctx, cdnn_handle graph, cdnn_handle stream) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    GraphSlot& gs = slot_as<GraphSlot>(c, graph, "graph_launch", "graph");
    DeviceGuard g(c);
    CDNN_CUDA(cudaGraphLaunch(gs.exec, stream_of(c, stream)));
  });
}

int cdnn_graph_free(cdnn_ctx ctx, cdnn_handle graph) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    GraphSlot gs;
    {
      std::lock_guard lock(c->mu);
      auto it = c->slots.find(graph);
      if (graph == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, "graph_free: " + label(graph) + " is not live");
      auto* p = std::get_if<GraphSlot>(&it->second);
      if (!p) fail(CDNN_INVALID_ARGUMENT, "graph_free: " + label(graph) + " is not a graph");
      gs = *p;
      c->slots.erase(it);
    }
    DeviceGuard g(c);
    cudaDeviceSynchronize();
    if (gs.exec) cudaGraphExecDestroy(gs.exec);
    if (gs.graph) cudaGraphDestroy(gs.graph);
  });
}

int cdnn_event_create(cdnn_ctx ctx, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    DeviceGuard g(c);
    EventSlot e;
    CDNN_CUDA(cudaEventCreate(&e.ev));
    *out = insert_slot(c, e);
  });
}
int cdnn_event_record(cdnn_ctx ctx, cdnn_handle ev, cdnn_handle stream) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    EventSlot& e = slot_as<EventSlot>(c, ev, "event_record", "event");
    DeviceGuard g(c);
    CDNN_CUDA(cudaEventRecord(e.ev, stream_of(c, stream)));
  });
}
int cdnn_event_elapsed(cdnn_ctx ctx, cdnn_handle start, cdnn_handle end, float* ms) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    EventSlot& a = slot_as<EventSlot>(c, start, "event_elapsed", "event");
    EventSlot& b = slot_as<EventSlot>(c, end, "event_elapsed", "event");
    DeviceGuard g(c);
    CDNN_CUDA(cudaEventSynchronize(b.ev));
    CDNN_CUDA(cudaEventElapsedTime(ms, a.ev, b.ev));
  });
}
int cdnn_event_sync(cdnn_ctx ctx, cdnn_handle ev) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    EventSlot& e = slot_as<EventSlot>(c, ev, "event_sync", "event");
    DeviceGuard g(c);
    CDNN_CUDA(cudaEventSynchronize(e.ev));
  });
}
int cdnn_event_free(cdnn_ctx ctx, cdnn_handle ev) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    cudaEvent_t e;
    {
      std::lock_guard lock(c->mu);
      auto it = c->slots.find(ev);
      if (ev == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, "event_free: " + label(ev) + " is not live");
      auto* p = std::get_if<EventSlot>(&it->second);
      if (!p) fail(CDNN_INVALID_ARGUMENT, "event_free: " + label(ev) + " is not an event");
      e = p->ev;
      c->slots.erase(it);
    }
    DeviceGuard g(c);
    cudaEventDestroy(e);
  });
}

// ---- RNG subsystem -----------------------------------------------------------------------
int cdnn_rng_create(cdnn_ctx ctx, uint64_t seed, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    RngSlot r;
    r.engine.seed(seed);
    *out = insert_slot(c, std::move(r));
  });
}

int cdnn_rng_next_u64(cdnn_ctx ctx, cdnn_handle h, uint64_t* out) {
  return guard([&] { *out = rng(need_ctx(ctx), h).engine(); });
}

int cdnn_rng_uniform(cdnn_ctx ctx, cdnn_handle h, cdnn_handle dst, uint64_t n, double lo, double hi) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    BufferSlot& b = buffer(c, dst, "rng_uniform");
    require_len(b, n, "rng_uniform");
    RngSlot& r = rng(c, h);
    if (n == 0) return;
    // Host draws keep the exact sequential mt19937_64 stream (backend.cpp:199-207).
    DeviceGuard g(c);
    if (b.dtype == CDNN_F64) {
      std::vector<double> v(n);
      for (auto& x : v) x = lo + (hi - lo) * (static_cast<double>(r.engine() >> 11) * 0x1.0p-53);
      CDNN_CUDA(cudaMemcpyAsync(b.dev, v.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
      CDNN_CUDA(cudaStreamSynchronize(c->stream));
    } else if (b.dtype == CDNN_F32) {
      std::vector<float> v(n);
      for (auto& x : v) x = static_cast<float>(lo + (hi - lo) * (static_cast<double>(r.engine() >> 11) * 0x1.0p-53));
      CDNN_CUDA(cudaMemcpyAsync(b.dev, v.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
      CDNN_CUDA(cudaStreamSynchronize(c->stream));
    } else {
      fail(CDNN_INVALID_ARGUMENT, "rng_uniform: floating buffer required");
    }
  });
}

int cdnn_subsystem_free(cdnn_ctx ctx, cdnn_handle h) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    void* comm = nullptr;
    {
      std::lock_guard lock(c->mu);
      auto it = c->slots.find(h);
      if (h == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, "free_subsystem: " + label(h) + " is not live");
      if (auto* n = std::get_if<NcclSlot>(&it->second)) comm = n->comm;
      else if (!std::holds_alternative<RngSlot>(it->second))
        fail(CDNN_INVALID_ARGUMENT, "free_subsystem: " + label(h) + " is not a subsystem");
      c->slots.erase(it);
    }
    if (comm) nccl_destroy(comm);
  });
}

// ---- descriptors ----------------------------------------------------------------------
int cdnn_conv_desc_create(cdnn_ctx ctx, const cdnn_conv_params* pp, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    if (!pp) fail(CDNN_INVALID_ARGUMENT, "conv: null params");
    cdnn_conv_params p = *pp;
    if (p.dilation_h <= 0) p.dilation_h = 1;
    if (p.dilation_w <= 0) p.dilation_w = 1;
    if (p.group <= 0) p.group = 1;
    if (p.n < 1 || p.c < 1 || p.h < 1 || p.w < 1 || p.num_output < 1 || p.kernel_h < 1 ||
        p.kernel_w < 1 || p.stride_h < 1 || p.stride_w < 1 || p.pad_h < 0 || p.pad_w < 0)
      fail(CDNN_INVALID_ARGUMENT, "conv: non-positive extent");
    if (p.c % p.group || p.num_output % p.group)
      fail(CDNN_INVALID_ARGUMENT, "conv: channels and num_output must be divisible by group");
    const int ekh = p.dilation_h * (p.kernel_h - 1) + 1, ekw = p.dilation_w * (p.kernel_w - 1) + 1;
    ConvDescSlot d;
    d.p = p;
    d.P = (p.h + 2 * p.pad_h - ekh) / p.stride_h + 1;
    d.Q = (p.w + 2 * p.pad_w - ekw) / p.stride_w + 1;
    if (p.h + 2 * p.pad_h < ekh || p.w + 2 * p.pad_w < ekw || d.P < 1 || d.Q < 1)
      fail(CDNN_INVALID_ARGUMENT, "conv: kernel larger than padded input");
    const int64_t big = int64_t(p.n) * std::max(p.c, p.num_output) * std::max<int64_t>(int64_t(p.h) * p.w, int64_t(d.P) * d.Q);
    if (big >= (int64_t(1) << 31)) fail(CDNN_INVALID_ARGUMENT, "conv: tensor exceeds 2^31 elements");
    ConvGeom& g = d.geom;
    g.N = p.n; g.C = p.c; g.H = p.h; g.W = p.w;
    g.Co = p.num_output; g.P = d.P; g.Q = d.Q;
    g.R = p.kernel_h; g.S = p.kernel_w;
    g.sh = p.stride_h; g.sw = p.stride_w; g.ph = p.pad_h; g.pw = p.pad_w;
    g.dh = p.dilation_h; g.dw = p.dilation_w;
    g.group = p.group; g.Cg = p.c / p.group; g.Cog = p.num_output / p.group;
    g.div_PQ = FastDiv(uint32_t(d.P * d.Q));
    g.div_Q = FastDiv(uint32_t(d.Q));
    g.div_HW = FastDiv(uint32_t(p.h * p.w));
    g.div_W = FastDiv(uint32_t(p.w));
    const int RS = g.R * g.S;
    d.Kc = g.Cg * RS;
    d.Kd = g.Cog * RS;
    std::vector<ConvTap> taps(d.Kc);
    for (int ci = 0; ci < g.Cg; ++ci)
      for (int r = 0; r < g.R; ++r)
        for (int s = 0; s < g.S; ++s) {
          ConvTap& t = taps[(ci * g.R + r) * g.S + s];
          t.dh = r * g.dh; t.dw = s * g.dw;
          t.off = ci * g.H * g.W + t.dh * g.W + t.dw;
          t.pad_ = 0;
        }
    std::vector<DgradTap> dtaps(d.Kd);
    std::vector<int> koff(d.Kd);
    for (int co = 0; co < g.Cog; ++co)
      for (int r = 0; r < g.R; ++r)
        for (int s = 0; s < g.S; ++s) {
          const int k = (co * g.R + r) * g.S + s;
          dtaps[k] = DgradTap{co * g.P * g.Q, r * g.dh, s * g.dw, 0};
          koff[k] = co * g.Cg * RS + r * g.S + s;
        }
    const size_t b1 = taps.size() * sizeof(ConvTap), b2 = dtaps.size() * sizeof(DgradTap),
                 b3 = koff.size() * sizeof(int);
    DeviceGuard dg(c);
    d.tables = device_alloc(b1 + b2 + b3, c->device);
    char* base = static_cast<char*>(d.tables->ptr);
    CDNN_CUDA(cudaMemcpy(base, taps.data(), b1, cudaMemcpyHostToDevice));
    CDNN_CUDA(cudaMemcpy(base + b1, dtaps.data(), b2, cudaMemcpyHostToDevice));
    CDNN_CUDA(cudaMemcpy(base + b1 + b2, koff.data(), b3, cudaMemcpyHostToDevice));
    d.taps = reinterpret_cast<ConvTap*>(base);
    d.dtaps = reinterpret_cast<DgradTap*>(base + b1);
    d.koff = reinterpret_cast<int*>(base + b1 + b2);
    *out = insert_slot(c, std::move(d));
  });
}

int cdnn_conv_output_shape(cdnn_ctx ctx, cdnn_handle desc, int out[4]) {
  return guard([&] {
    ConvDescSlot& d = conv_desc(need_ctx(ctx), desc);
    out[0] = d.p.n; out[1] = d.p.num_output; out[2] = d.P; out[3] = d.Q;
  });
}

int cdnn_pool_desc_create(cdnn_ctx ctx, const cdnn_pool_params* pp, cdnn_handle* out) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    if (!pp) fail(CDNN_INVALID_ARGUMENT, "pool: null params");
    cdnn_pool_params p = *pp;
    if (p.n < 1 || p.c < 1 || p.h < 1 || p.w < 1) fail(CDNN_INVALID_ARGUMENT, "pool: non-positive bottom extent");
    if (p.method != CDNN_POOL_MAX && p.method != CDNN_POOL_AVE) fail(CDNN_INVALID_ARGUMENT, "pool: unknown method");
    if (p.global_pooling) {
      p.kernel_h = p.h; p.kernel_w = p.w; p.stride_h = p.stride_w = 1; p.pad_h = p.pad_w = 0;
    }
    if (p.kernel_h < 1 || p.kernel_w < 1 || p.stride_h < 1 || p.stride_w < 1 || p.pad_h < 0 || p.pad_w < 0)
      fail(CDNN_INVALID_ARGUMENT, "pool: bad kernel/stride/pad");
    if (p.pad_h >= p.kernel_h || p.pad_w >= p.kernel_w) fail(CDNN_INVALID_ARGUMENT, "pool: pad must be smaller than kernel");
    PoolDescSlot d;
    d.p = p;
    // Caffe: ceil((H + 2p - k) / s) + 1, then drop a window that would start in the padding
    d.PH = static_cast<int>(std::ceil(static_cast<float>(p.h + 2 * p.pad_h - p.kernel_h) / p.stride_h)) + 1;
    d.PW = static_cast<int>(std::ceil(static_cast<float>(p.w + 2 * p.pad_w - p.kernel_w) / p.stride_w)) + 1;
    if (p.pad_h || p.pad_w) {
      if ((d.PH - 1) * p.stride_h >= p.h + p.pad_h) --d.PH;
      if ((d.PW - 1) * p.stride_w >= p.w + p.pad_w) --d.PW;
    }
    if (d.PH < 1 || d.PW < 1) fail(CDNN_INVALID_ARGUMENT, "pool: kernel larger than padded input");
    *out = insert_slot(c, std::move(d));
  });
}

int cdnn_pool_output_shape(cdnn_ctx ctx, cdnn_handle desc, int out[4]) {
  return guard([&] {
    PoolDescSlot& d = pool_desc(need_ctx(ctx), desc);
    out[0] = d.p.n; out[1] = d.p.c; out[2] = d.PH; out[3] = d.PW;
  });
}

int cdnn_desc_free(cdnn_ctx ctx, cdnn_handle h) {
  return guard([&] {
    Ctx* c = need_ctx(ctx);
    std::shared_ptr<DevAlloc> keep;
    {
      std::lock_guard lock(c->mu);
      auto it = c->slots.find(h);
      if (h == 0 || it == c->slots.end()) fail(CDNN_DANGLING_HANDLE, "desc_free: " + label(h) + " is not live");
      if (auto* cd = std::get_if<ConvDescSlot>(&it->second)) keep = cd->tables;
      else if (!std::holds_alternative<PoolDescSlot>(it->second))
        fail(CDNN_INVALID_ARGUMENT, "desc_free: " + label(h) + " is not a descriptor");
      c->slots.erase(it);
    }
    if (keep) { DeviceGuard g(c); cudaStreamSynchronize(c->stream); }
  });
}

}  // extern "C"
