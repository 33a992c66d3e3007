/*
 * cudadnn.h — the B200 "CudaDnn" C-ABI: handle look-up tables for device
 * memory, streams, descriptors and subsystems (RNG, NCCL communicators),
 * the frozen function-index dispatch, and typed entry points for every op of
 * one SGD iteration.
 *
 * This is the device boundary of the hot path.  It replaces, one for one:
 *
 *   reference (/root/reference/proj/core)          this header
 *   ---------------------------------------------  -------------------------------
 *   Registry::alloc_buffer  backend.cpp:18-25      cdnn_alloc
 *   Registry::free_buffer   backend.cpp:27-38      cdnn_free
 *   Registry::buffer_length backend.cpp:58-60      cdnn_length
 *   Registry::write / read  backend.cpp:62-73      cdnn_write / cdnn_read
 *   Registry::buffer (span) backend.cpp:75-79      cdnn_device_ptr (device view)
 *   Registry::create_rng    backend.cpp:81-86      cdnn_rng_create
 *   Registry::free_subsystem backend.cpp:100-110   cdnn_subsystem_free
 *   Registry::live_slots    backend.cpp:112-115    cdnn_live_slots
 *   Registry::dispatch      backend.cpp:248-305    cdnn_dispatch (indices 1-7 frozen,
 *                                                  backend.hpp:47-69; new ops append)
 *   kernels::fill/copy/scal/axpy/dot backend.cpp:131-167   cdnn_fill/copy/scal/axpy/dot
 *   kernels::gemm           backend.cpp:169-197    cdnn_gemm (tcgen05 TF32 / SIMT FP64)
 *   kernels::rng_uniform    backend.cpp:199-207    cdnn_rng_uniform (host mt19937_64)
 *   InnerProductLayer fwd/bwd layers.cpp:124-169   cdnn_ip_forward / cdnn_ip_backward
 *   ReluLayer   layers.cpp:180-195                 cdnn_relu_forward / _backward
 *   SigmoidLayer layers.cpp:206-221                cdnn_sigmoid_forward / _backward
 *   SoftmaxLayer layers.cpp:232-266                cdnn_softmax_forward / _backward
 *   Solver::apply_update solver.cpp:24-57          cdnn_solver_apply
 *   (absent: Convolution, Pooling, SoftmaxWithLoss, momentum SGD, NCCL Parallel)
 *                                                  cdnn_conv_*, cdnn_pool_*,
 *                                                  cdnn_softmax_loss_*, cdnn_nccl_*
 *
 * Conventions:
 *  - The library owns all device memory; callers hold opaque 64-bit ids.
 *    Ids are monotone per context and never recycled; 0 is the null handle
 *    (backend.hpp:17-25).  Handle 0 as a *stream* argument means the
 *    context's own compute stream.
 *  - Every entry point returns a cdnn_status; the message of the last failure
 *    on the calling thread is available from cdnn_last_error().  Status codes
 *    map 1:1 onto the exception classes of errors.hpp:8-83.
 *  - Table mutation is serialised per context; buffer contents are ordered
 *    per stream.  Compute entry points are asynchronous on the
 *    given stream; cdnn_read/cdnn_write/cdnn_dot synchronise.
 *  - Element counts are in elements of the buffer's dtype.
 */
#ifndef CUDADNN_H_
#define CUDADNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDNN_API __attribute__((visibility("default")))

typedef uint64_t cdnn_handle;
typedef struct cdnn_context* cdnn_ctx;

typedef enum {
  CDNN_OK = 0,
  CDNN_INVALID_ARGUMENT = 1, /* InvalidArgument  errors.hpp:14 */
  CDNN_DANGLING_HANDLE = 2,  /* DanglingHandle   errors.hpp:20 */
  CDNN_UNKNOWN_FUNCTION = 3, /* UnknownFunction  errors.hpp:26 */
  CDNN_MODEL_ERROR = 4,      /* ModelError       errors.hpp:32 */
  CDNN_DATA_STARVATION = 5,  /* DataStarvation   errors.hpp:38 */
  CDNN_FORMAT_ERROR = 6,     /* FormatError      errors.hpp:44 */
  CDNN_NOT_FOUND = 7,        /* NotFound         errors.hpp:49 */
  CDNN_INVALID_STATE = 8,    /* InvalidState     errors.hpp:55 */
  CDNN_PARSE_ERROR = 9,      /* ParseError       errors.hpp:61 */
  CDNN_LOAD_ERROR = 10,      /* LoadError        errors.hpp:72 */
  CDNN_CUDA_ERROR = 11,      /* device / driver failure (no reference analog) */
  CDNN_NO_DEVICE = 12        /* no CUDA device: the library never falls back to the CPU */
} cdnn_status;

typedef enum { CDNN_F32 = 0, CDNN_F64 = 1, CDNN_I32 = 2 } cdnn_dtype;

/* handle kinds held in the look-up tables (paper Table 3) */
typedef enum {
  CDNN_KIND_BUFFER = 0,
  CDNN_KIND_STREAM = 1,
  CDNN_KIND_DESCRIPTOR = 2,
  CDNN_KIND_SUBSYSTEM = 3,
  CDNN_KIND_GRAPH = 4
} cdnn_kind;

/* Frozen dispatch indices (backend.hpp:47-69).  Indices only ever append. */
enum {
  CDNN_FN_FILL = 1,        /* dst, n, value */
  CDNN_FN_COPY = 2,        /* src, dst, n */
  CDNN_FN_SCAL = 3,        /* n, alpha, x */
  CDNN_FN_AXPY = 4,        /* n, alpha, x, y */
  CDNN_FN_DOT = 5,         /* n, x, y -> result */
  CDNN_FN_GEMM = 6,        /* trans_a, trans_b, m, n, k, alpha, a, b, beta, c */
  CDNN_FN_RNG_UNIFORM = 7, /* rng, dst, n, lo, hi */
  /* appended by this library */
  CDNN_FN_RELU_FWD = 8,    /* x, y, n */
  CDNN_FN_RELU_BWD = 9,    /* x, dy, dx, n */
  CDNN_FN_SIGMOID_FWD = 10,/* x, y, n */
  CDNN_FN_SIGMOID_BWD = 11,/* y, dy, dx, n */
  CDNN_FN_SOFTMAX_FWD = 12,/* x, y, rows, features */
  CDNN_FN_SOFTMAX_BWD = 13 /* y, dy, dx, rows, features */
};

/* ---- diagnostics / context ---------------------------------------------- */
CDNN_API const char* cdnn_last_error(void);
CDNN_API const char* cdnn_status_name(int status);
CDNN_API int cdnn_device_count(int* out);
CDNN_API int cdnn_ctx_create(int device, cdnn_ctx* out);
CDNN_API int cdnn_ctx_destroy(cdnn_ctx ctx);
CDNN_API int cdnn_ctx_device(cdnn_ctx ctx, int* out);
CDNN_API int cdnn_live_slots(cdnn_ctx ctx, uint64_t* out); /* backend.hpp:99-100 */
/* number of kernels this context has launched (the bench's gpu_launches claim) */
CDNN_API int cdnn_launch_count(cdnn_ctx ctx, uint64_t* out);

/* Numerics of F32 contractions (gemm / InnerProduct / Convolution):
 *   CDNN_MATH_TF32X3 (default)  split-precision 3xTF32 on the tensor cores:
 *                               x = hi + lo, D += A_lo B_hi + A_hi B_lo + A_hi B_hi,
 *                               FP32-level accuracy (gradient parity with the
 *                               FP32 reference through ReLU gates)
 *   CDNN_MATH_TF32              one TF32 MMA per product (fastest; TMA-fed operands)
 * The environment variable CDNN_MATH=tf32 selects TF32 for new contexts. */
typedef enum { CDNN_MATH_TF32 = 0, CDNN_MATH_TF32X3 = 1 } cdnn_math_mode;
CDNN_API int cdnn_set_math_mode(cdnn_ctx ctx, int mode);
CDNN_API int cdnn_get_math_mode(cdnn_ctx ctx, int* out);

/* ---- buffers ------------------------------------------------------------- */
/* zero-initialised; length 0 -> CDNN_INVALID_ARGUMENT (backend.cpp:18-21) */
CDNN_API int cdnn_alloc(cdnn_ctx ctx, uint64_t length, int dtype, cdnn_handle* out);
/* unknown, 0 or freed -> CDNN_DANGLING_HANDLE (backend.cpp:27-38) */
CDNN_API int cdnn_free(cdnn_ctx ctx, cdnn_handle h);
/* aliasing sub-range [offset, offset+length) of a buffer (flat param/grad arenas) */
CDNN_API int cdnn_view(cdnn_ctx ctx, cdnn_handle h, uint64_t offset, uint64_t length,
                       cdnn_handle* out);
CDNN_API int cdnn_length(cdnn_ctx ctx, cdnn_handle h, uint64_t* out);
CDNN_API int cdnn_buffer_dtype(cdnn_ctx ctx, cdnn_handle h, int* out);
CDNN_API int cdnn_device_ptr(cdnn_ctx ctx, cdnn_handle h, void** out);
/* synchronous host copies of elements [0, n); n > length -> INVALID_ARGUMENT */
CDNN_API int cdnn_write(cdnn_ctx ctx, cdnn_handle h, const void* host, uint64_t n);
CDNN_API int cdnn_read(cdnn_ctx ctx, cdnn_handle h, void* host, uint64_t n);
/* asynchronous copies at an element offset (host memory should be pinned) */
CDNN_API int cdnn_write_async(cdnn_ctx ctx, cdnn_handle h, uint64_t offset, const void* host,
                              uint64_t n, cdnn_handle stream);
CDNN_API int cdnn_read_async(cdnn_ctx ctx, cdnn_handle h, uint64_t offset, void* host,
                             uint64_t n, cdnn_handle stream);
CDNN_API int cdnn_host_alloc_pinned(uint64_t bytes, void** out);
CDNN_API int cdnn_host_free_pinned(void* p);

/* ---- streams / graphs ----------------------------------------------------- */
CDNN_API int cdnn_stream_create(cdnn_ctx ctx, cdnn_handle* out);
CDNN_API int cdnn_stream_free(cdnn_ctx ctx, cdnn_handle h);
CDNN_API int cdnn_stream_sync(cdnn_ctx ctx, cdnn_handle stream);
/* make `stream` wait for all work currently queued on `on` */
CDNN_API int cdnn_stream_wait(cdnn_ctx ctx, cdnn_handle stream, cdnn_handle on);
CDNN_API int cdnn_graph_begin(cdnn_ctx ctx, cdnn_handle stream);
CDNN_API int cdnn_graph_end(cdnn_ctx ctx, cdnn_handle stream, cdnn_handle* graph_out);
CDNN_API int cdnn_graph_launch(cdnn_ctx ctx, cdnn_handle graph, cdnn_handle stream);
CDNN_API int cdnn_graph_free(cdnn_ctx ctx, cdnn_handle graph);
/* events for device-side timing: elapsed ms between two records */
CDNN_API int cdnn_event_create(cdnn_ctx ctx, cdnn_handle* out);
CDNN_API int cdnn_event_record(cdnn_ctx ctx, cdnn_handle ev, cdnn_handle stream);
CDNN_API int cdnn_event_elapsed(cdnn_ctx ctx, cdnn_handle start, cdnn_handle end, float* ms);
CDNN_API int cdnn_event_free(cdnn_ctx ctx, cdnn_handle ev);
/* host waits until the work captured by the event's last record has completed */
CDNN_API int cdnn_event_sync(cdnn_ctx ctx, cdnn_handle ev);

/* ---- RNG subsystem (host mt19937_64, backend.hpp:31-45) ------------------ */
CDNN_API int cdnn_rng_create(cdnn_ctx ctx, uint64_t seed, cdnn_handle* out);
CDNN_API int cdnn_rng_next_u64(cdnn_ctx ctx, cdnn_handle rng, uint64_t* out);
/* dst[0..n) = lo + (hi-lo)*u, u = (u64>>11)*2^-53, drawn in order (backend.cpp:199-207) */
CDNN_API int cdnn_rng_uniform(cdnn_ctx ctx, cdnn_handle rng, cdnn_handle dst, uint64_t n,
                              double lo, double hi);
CDNN_API int cdnn_subsystem_free(cdnn_ctx ctx, cdnn_handle h);

/* ---- descriptors ---------------------------------------------------------- */
typedef struct {
  int n, c, h, w;          /* bottom NCHW */
  int num_output;          /* Cout */
  int kernel_h, kernel_w;
  int stride_h, stride_w;
  int pad_h, pad_w;
  int dilation_h, dilation_w;
  int group;
} cdnn_conv_params;

typedef enum { CDNN_POOL_MAX = 0, CDNN_POOL_AVE = 1 } cdnn_pool_method;

typedef struct {
  int n, c, h, w;          /* bottom NCHW */
  int method;              /* cdnn_pool_method */
  int kernel_h, kernel_w;
  int stride_h, stride_w;
  int pad_h, pad_w;
  int global_pooling;      /* kernel = full H x W */
} cdnn_pool_params;

/* Validates and derives output extents (Caffe conv: floor; pooling: ceil). */
CDNN_API int cdnn_conv_desc_create(cdnn_ctx ctx, const cdnn_conv_params* p, cdnn_handle* out);
CDNN_API int cdnn_conv_output_shape(cdnn_ctx ctx, cdnn_handle desc, int out_nchw[4]);
CDNN_API int cdnn_pool_desc_create(cdnn_ctx ctx, const cdnn_pool_params* p, cdnn_handle* out);
CDNN_API int cdnn_pool_output_shape(cdnn_ctx ctx, cdnn_handle desc, int out_nchw[4]);
CDNN_API int cdnn_desc_free(cdnn_ctx ctx, cdnn_handle h);

/* ---- legacy function-index dispatch (backend.cpp:248-305) ----------------- */
/* args are doubles, handle ids encoded as values; `out` receives up to
 * *nout results (dot).  Unknown index -> CDNN_UNKNOWN_FUNCTION; wrong arity
 * or non-integral handle/count -> CDNN_INVALID_ARGUMENT.  Synchronous. */
CDNN_API int cdnn_dispatch(cdnn_ctx ctx, int function_index, const double* args,
                           uint64_t nargs, double* out, uint64_t* nout);

/* ---- BLAS-like kernels (backend.cpp:131-197) ------------------------------ */
CDNN_API int cdnn_fill(cdnn_ctx ctx, cdnn_handle dst, uint64_t n, double value, cdnn_handle stream);
CDNN_API int cdnn_copy(cdnn_ctx ctx, cdnn_handle src, cdnn_handle dst, uint64_t n, cdnn_handle stream);
/* dst[dst_offset .. +n) = src[src_offset .. +n) on the stream (device to device, capturable) */
CDNN_API int cdnn_copy_range(cdnn_ctx ctx, cdnn_handle src, uint64_t src_offset, cdnn_handle dst,
                             uint64_t dst_offset, uint64_t n, cdnn_handle stream);
CDNN_API int cdnn_scal(cdnn_ctx ctx, uint64_t n, double alpha, cdnn_handle x, cdnn_handle stream);
CDNN_API int cdnn_axpy(cdnn_ctx ctx, uint64_t n, double alpha, cdnn_handle x, cdnn_handle y,
                       cdnn_handle stream);
CDNN_API int cdnn_dot(cdnn_ctx ctx, uint64_t n, cdnn_handle x, cdnn_handle y, double* result);
/* Fan-out in one pass (Split forward: dst_k = src when alpha is NULL; Eltwise SUM
 * backward: dst_k = alpha[k] * src); 1..8 destinations, 0 handles skipped. */
CDNN_API int cdnn_fan_out(cdnn_ctx ctx, cdnn_handle src, const cdnn_handle* dsts, const double* alpha, int ndst,
                          uint64_t n, cdnn_handle stream);
/* Fan-in in one pass (Split backward): dst = src_0 + src_1 + ... in order, rounded as
 * cdnn_copy followed by cdnn_axpy(1.0) per further source; 1..8 sources. */
CDNN_API int cdnn_fan_in(cdnn_ctx ctx, const cdnn_handle* srcs, int nsrc, cdnn_handle dst, uint64_t n,
                         cdnn_handle stream);
/* cdnn_fan_in with flags and a gate: CDNN_FAN_RELU stores max(sum, 0) (Eltwise SUM followed
 * by an in-place ReLU, whose forward pass then disappears); a nonzero gate stores
 * (gate > 0 ? sum : 0) (Split backward fused with the backward of the in-place ReLU whose
 * data is the gate) */
enum { CDNN_FAN_RELU = 1 };
CDNN_API int cdnn_fan_in_ex(cdnn_ctx ctx, const cdnn_handle* srcs, int nsrc, cdnn_handle dst, uint64_t n, int flags,
                            cdnn_handle gate, cdnn_handle stream);
/* Row-major C = alpha*op(A)*op(B) + beta*C; beta == 0 never reads C.
 * F32 buffers run on tcgen05 TF32 tensor cores, F64 on the SIMT FP64 path. */
CDNN_API int cdnn_gemm(cdnn_ctx ctx, int trans_a, int trans_b, int m, int n, int k, double alpha,
                       cdnn_handle a, cdnn_handle b, double beta, cdnn_handle c, cdnn_handle stream);

/* ---- layers ---------------------------------------------------------------- */
/* InnerProduct (layers.cpp:124-169).  x: rows x K, w: O x K, bias: O (0 = none)
 * top = x W^T + bias ; optional fused ReLU (relu != 0). */
CDNN_API int cdnn_ip_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle w, cdnn_handle bias,
                             cdnn_handle top, int rows, int k, int o, int relu,
                             cdnn_handle stream);
/* dW += dY^T X ; db += colsum(dY) (0 = skip) ; dX = dY W (0 = skip) */
CDNN_API int cdnn_ip_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle w, cdnn_handle dy,
                              cdnn_handle dw, cdnn_handle db, cdnn_handle dx, int rows, int k,
                              int o, cdnn_handle stream);

/* Convolution (Caffe semantics; absent from the reference).
 * bias may be 0.  backward_filter ACCUMULATES into dw/db (param diffs
 * accumulate, layers.hpp:84-86); backward_data OVERWRITES dx. */
CDNN_API int cdnn_conv_forward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle w,
                               cdnn_handle bias, cdnn_handle y, cdnn_handle stream);
/* cdnn_conv_forward with flags: CDNN_CONV_RELU applies max(y, 0) in the epilogue (a
 * following in-place ReLU fused, layers.cpp:184 semantics) */
enum { CDNN_CONV_RELU = 1 };
CDNN_API int cdnn_conv_forward_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle w,
                                  cdnn_handle bias, cdnn_handle y, int flags, cdnn_handle stream);
CDNN_API int cdnn_conv_backward_data(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle w,
                                     cdnn_handle dy, cdnn_handle dx, cdnn_handle stream);
/* cdnn_conv_backward_data with a fused ReLU gate (see cdnn_pool_backward_ex; 0 = none):
 * applied in the tap kernels' epilogue, else by a trailing gate pass */
CDNN_API int cdnn_conv_backward_data_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle w,
                                        cdnn_handle dy, cdnn_handle dx, cdnn_handle gate,
                                        cdnn_handle stream);
CDNN_API int cdnn_conv_backward_filter(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x,
                                       cdnn_handle dy, cdnn_handle dw, cdnn_handle db,
                                       cdnn_handle stream);
/* cdnn_conv_backward_filter with flags: CDNN_CONV_INPUT_UNCHANGED promises that x is the
 * very buffer, unmodified, of the last forward on this descriptor, so an input rewrite
 * the forward made (space-to-depth of a strided stem) is reused instead of redone */
enum { CDNN_CONV_INPUT_UNCHANGED = 2 };
CDNN_API int cdnn_conv_backward_filter_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x,
                                          cdnn_handle dy, cdnn_handle dw, cdnn_handle db, int flags,
                                          cdnn_handle stream);

/* Pooling (Caffe semantics).  mask: I32 buffer of top count
 * holding the flat h*W+w argmax (MAX only; first max wins, strict >). */
CDNN_API int cdnn_pool_forward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle y,
                               cdnn_handle mask, cdnn_handle stream);
/* cdnn_pool_forward with flags: CDNN_POOL_RELU clamps the pooled output at 0 (a following
 * in-place ReLU fused; the argmax mask is the pooling's, unchanged) */
enum { CDNN_POOL_RELU = 1 };
CDNN_API int cdnn_pool_forward_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle x, cdnn_handle y,
                                  cdnn_handle mask, int flags, cdnn_handle stream);
CDNN_API int cdnn_pool_backward(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle dy, cdnn_handle mask,
                                cdnn_handle dx, cdnn_handle stream);
/* Backward entry points with a fused ReLU gate: dx = gate > 0 ? grad : 0 elementwise,
 * gate = the data of the in-place ReLU on this layer's bottom (its backward,
 * layers.cpp:188-195, then no longer runs); gate 0 = the plain entry point. */
CDNN_API int cdnn_pool_backward_ex(cdnn_ctx ctx, cdnn_handle desc, cdnn_handle dy, cdnn_handle mask,
                                   cdnn_handle dx, cdnn_handle gate, cdnn_handle stream);

/* elementwise (layers.cpp:180-221); n elements */
CDNN_API int cdnn_relu_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, uint64_t n, cdnn_handle stream);
CDNN_API int cdnn_relu_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle dy, cdnn_handle dx,
                                uint64_t n, cdnn_handle stream);
CDNN_API int cdnn_sigmoid_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, uint64_t n,
                                  cdnn_handle stream);
CDNN_API int cdnn_sigmoid_backward(cdnn_ctx ctx, cdnn_handle y, cdnn_handle dy, cdnn_handle dx,
                                   uint64_t n, cdnn_handle stream);
/* whole-sample softmax over `features` values per row (layers.cpp:232-266) */
CDNN_API int cdnn_softmax_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, int rows,
                                  int features, cdnn_handle stream);
CDNN_API int cdnn_softmax_backward(cdnn_ctx ctx, cdnn_handle y, cdnn_handle dy, cdnn_handle dx,
                                   int rows, int features, cdnn_handle stream);
/* SoftmaxWithLoss (Caffe): prob = softmax(x) per row; loss[0] = -sum log p_label / norm.
 * label: same dtype as x, integral class ids.  norm = rows (normalize) or 1. */
CDNN_API int cdnn_softmax_loss_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle label,
                                       cdnn_handle prob, cdnn_handle loss, int rows, int classes,
                                       int normalize, cdnn_handle stream);
/* dx = loss_weight * (prob - onehot(label)) / norm */
CDNN_API int cdnn_softmax_loss_backward(cdnn_ctx ctx, cdnn_handle prob, cdnn_handle label,
                                        cdnn_handle dx, int rows, int classes, int normalize,
                                        double loss_weight, cdnn_handle stream);

/* ---- layers of configs 4-5 the reference lacks; Caffe semantics, NCHW,
 * hw = H*W.  No reference interface to replace: these follow the Caffe layer contracts. */
/* LRN ACROSS_CHANNELS: scale = k + alpha/size * sum_{window} x^2 ; y = x * scale^-beta.
 * `scale` (n*c*hw) is kept for backward. local_size odd. */
CDNN_API int cdnn_lrn_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle scale, int n,
                              int c, int hw, int local_size, double alpha, double beta, double k,
                              cdnn_handle stream);
/* dx = dy*scale^-beta - 2*alpha*beta/size * x * sum_{window} dy*y/scale */
CDNN_API int cdnn_lrn_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle scale,
                               cdnn_handle dy, cdnn_handle dx, int n, int c, int hw,
                               int local_size, double alpha, double beta, cdnn_handle stream);
/* cdnn_lrn_backward with a fused ReLU gate (see cdnn_pool_backward_ex; 0 = none) */
CDNN_API int cdnn_lrn_backward_ex(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle scale,
                                  cdnn_handle dy, cdnn_handle dx, int n, int c, int hw, int local_size,
                                  double alpha, double beta, cdnn_handle gate, cdnn_handle stream);
/* LRN fused with the MAX pooling that consumes its top (ops_lrnpool.cu): pool_desc
 * describes the pooling over the LRN's NCHW shape.  Supported (out = 1): local_size 3
 * or 5, MAX, no padding, square 3x3/2 or 2x2/2 windows.  Forward writes the LRN top
 * (kept observable), the pooled top and the argmax mask, bit-identical to
 * cdnn_lrn_forward + cdnn_pool_forward_ex (flags: CDNN_POOL_RELU); no scale tensor.
 * Backward takes the POOLED top's diff and mask and writes the LRN bottom diff,
 * bit-identical to cdnn_pool_backward + cdnn_lrn_backward_ex; gate 0 or x (the
 * in-place ReLU on the LRN bottom, fused). */
CDNN_API int cdnn_lrn_pool_supported(cdnn_ctx ctx, cdnn_handle pool_desc, int local_size, int* out);
CDNN_API int cdnn_lrn_pool_forward(cdnn_ctx ctx, cdnn_handle pool_desc, cdnn_handle x, cdnn_handle lrn_top,
                                   cdnn_handle pool_top, cdnn_handle mask, int local_size, double alpha,
                                   double beta, double k, int flags, cdnn_handle stream);
CDNN_API int cdnn_lrn_pool_backward(cdnn_ctx ctx, cdnn_handle pool_desc, cdnn_handle x, cdnn_handle pool_dy,
                                    cdnn_handle mask, cdnn_handle dx, cdnn_handle gate, int local_size,
                                    double alpha, double beta, double k, cdnn_handle stream);
/* Dropout (train): out[i] = in[i]/(1-ratio) if hash(seed, *counter, i) > ratio*2^32 else 0.
 * The same call maps forward data and backward diffs (same seed + counter -> same mask).
 * `counter` is an 8-byte device buffer (u64 iteration), read by the kernel so graph replays
 * draw fresh masks once cdnn_counter_increment advances it. */
CDNN_API int cdnn_dropout(cdnn_ctx ctx, cdnn_handle in, cdnn_handle out, uint64_t n, double ratio,
                          uint64_t seed, cdnn_handle counter, cdnn_handle stream);
CDNN_API int cdnn_counter_increment(cdnn_ctx ctx, cdnn_handle counter, cdnn_handle stream);
/* BatchNorm, training statistics over (n, hw) per channel: y = (x - mean) * invstd,
 * invstd = 1/sqrt(var + eps) (biased variance).  mean/invstd (c) kept for backward. */
CDNN_API int cdnn_batchnorm_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle y, cdnn_handle mean,
                                    cdnn_handle invstd, int n, int c, int hw, double eps,
                                    cdnn_handle stream);
/* dx = (dy - mean(dy) - y*mean(dy*y)) * invstd ; scratch holds 2*c values */
CDNN_API int cdnn_batchnorm_backward(cdnn_ctx ctx, cdnn_handle y, cdnn_handle invstd, cdnn_handle dy,
                                     cdnn_handle dx, cdnn_handle scratch, int n, int c, int hw,
                                     cdnn_handle stream);
/* BatchNorm followed by Scale, fused: xnorm = (x - mean)*invstd (kept for backward),
 * z = gamma*xnorm + beta (beta may be 0) */
CDNN_API int cdnn_batchnorm_scale_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle xnorm, cdnn_handle z,
                                          cdnn_handle mean, cdnn_handle invstd, cdnn_handle gamma,
                                          cdnn_handle beta, int n, int c, int hw, double eps,
                                          cdnn_handle stream);
/* cdnn_batchnorm_scale_forward with flags: CDNN_BN_RELU stores z = max(gamma*xnorm + beta, 0)
 * (an in-place ReLU on the Scale's top, whose forward pass then disappears); xnorm unchanged */
enum { CDNN_BN_RELU = 1 };
CDNN_API int cdnn_batchnorm_scale_forward_ex(cdnn_ctx ctx, cdnn_handle x, cdnn_handle xnorm, cdnn_handle z,
                                             cdnn_handle mean, cdnn_handle invstd, cdnn_handle gamma,
                                             cdnn_handle beta, int n, int c, int hw, double eps, int flags,
                                             cdnn_handle stream);
/* dbeta += sum dz ; dgamma += sum dz*xnorm ;
 * dx = gamma*invstd*(dz - mean(dz) - xnorm*mean(dz*xnorm)) (skipped when dx == 0); scratch 2*c */
CDNN_API int cdnn_batchnorm_scale_backward(cdnn_ctx ctx, cdnn_handle xnorm, cdnn_handle invstd,
                                           cdnn_handle gamma, cdnn_handle dz, cdnn_handle dx,
                                           cdnn_handle dgamma, cdnn_handle dbeta, cdnn_handle scratch,
                                           int n, int c, int hw, cdnn_handle stream);
/* Scale (per channel): y = x*gamma[c] (+ beta[c] when beta != 0) */
CDNN_API int cdnn_scale_forward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle gamma, cdnn_handle beta,
                                cdnn_handle y, int n, int c, int hw, cdnn_handle stream);
/* dgamma += sum dy*x ; dbeta += sum dy ; dx = dy*gamma (each skipped when its handle is 0) */
CDNN_API int cdnn_scale_backward(cdnn_ctx ctx, cdnn_handle x, cdnn_handle gamma, cdnn_handle dy,
                                 cdnn_handle dgamma, cdnn_handle dbeta, cdnn_handle dx, int n,
                                 int c, int hw, cdnn_handle stream);
/* y = a*x (accumulate = 0) or y = a*x + b*y: Eltwise SUM terms and their backward */
CDNN_API int cdnn_axpby(cdnn_ctx ctx, uint64_t n, double a, cdnn_handle x, double b, cdnn_handle y,
                        int accumulate, cdnn_handle stream);

/* ---- policy-gradient diff injection (trainer.cpp:42-113) ----
 * dlogit (rows x classes) = modulated log-prob gradient of n steps, 0 for rows >= n:
 *   softmax (sigmoid = 0): (prob - onehot(action)) * return
 *   sigmoid (sigmoid = 1, classes = 1): -((action == 0 ? 1 - p : -p) * return)
 * actions / returns: n values in the prob buffer's dtype. */
CDNN_API int cdnn_pg_diff(cdnn_ctx ctx, cdnn_handle prob, cdnn_handle actions, cdnn_handle returns,
                          cdnn_handle dlogit, int rows, int n, int classes, int sigmoid,
                          cdnn_handle stream);

/* ---- solver (solver.cpp:24-57 + Caffe momentum / weight decay) ----------- */
typedef enum { CDNN_SOLVER_SGD = 0, CDNN_SOLVER_RMSPROP = 1 } cdnn_solver_method;

/* ---- fused policy-gradient update of a two-layer perceptron (ops_mlp.cu) ----
 * The reference's pg_softmax graph (InnerProduct -> ReLU -> InnerProduct ->
 * Softmax, proj/models/pg_softmax.prototxt) trained by the batched policy
 * gradient (Net::pg_backward + Solver::apply_update, trainer.cpp:204-216) in one
 * kernel: forward of `rows` states x (rows x in), logits / prob tops (rows x
 * classes) and the optional ReLU top (rows x hidden) written, cdnn_pg_diff's
 * softmax gradient for the first `count` rows, backward, and the
 * cdnn_solver_apply rule on the arenas (weights, grads, history) at
 * param_offsets = {W1 (hidden x in), b1, W2 (classes x hidden), b2}; the arena
 * gradients are added to the batch gradient and left zero.  Deterministic; the
 * same operations as the layered path in another summation order.
 * cdnn_mlp_pg_supported: 1 when the extents fit the one-CTA kernel. */
CDNN_API int cdnn_mlp_pg_supported(cdnn_ctx ctx, int dtype, int rows, int in, int hidden, int classes,
                                   int* out);
CDNN_API int cdnn_mlp_pg_step(cdnn_ctx ctx, cdnn_handle x, cdnn_handle actions, cdnn_handle returns,
                              int rows, int count, int in, int hidden, int classes, cdnn_handle weights,
                              cdnn_handle grads, cdnn_handle history, const uint64_t param_offsets[4],
                              int solver, double lr, double momentum, double weight_decay,
                              double rms_decay, double epsilon, cdnn_handle hidden_top,
                              cdnn_handle logits, cdnn_handle prob, cdnn_handle stream);
/* The same reading the states / actions / returns straight from page-locked host
 * memory (cudaMallocHost: mapped under UVA) and writing prob to host_prob too, so a
 * captured episode update needs no copy nodes: host_x (rows x in) is read over the
 * bus and also stored into x (the feed blob); host_actions / host_returns (count
 * each) replace the actions / returns buffers (pass 0 handles); any host pointer may
 * be null (the device buffer is used). */
CDNN_API int cdnn_mlp_pg_step_host(cdnn_ctx ctx, cdnn_handle x, cdnn_handle actions, cdnn_handle returns,
                                   const void* host_x, const void* host_actions, const void* host_returns,
                                   void* host_prob, int rows, int count, int in, int hidden, int classes,
                                   cdnn_handle weights, cdnn_handle grads, cdnn_handle history,
                                   const uint64_t param_offsets[4], int solver, double lr, double momentum,
                                   double weight_decay, double rms_decay, double epsilon, cdnn_handle hidden_top,
                                   cdnn_handle logits, cdnn_handle prob, cdnn_handle stream);
/* One fused pass over n elements of (w, g, hist):
 *   SGD:      g' = g + wd*w ; v = mom*v + lr*g' ; w -= v      (hist may be 0 iff mom == 0)
 *             (mom = wd = 0 reproduces `w -= lr*g` bit for bit, solver.cpp:41-43)
 *   RMSProp:  c = d*c + (1-d)*g*g ; w -= lr*g/(sqrt(c)+eps)     (solver.cpp:50-52)
 * and then g = 0 (solver.cpp:55). */
CDNN_API int cdnn_solver_apply(cdnn_ctx ctx, int method, cdnn_handle w, cdnn_handle g,
                               cdnn_handle hist, uint64_t n, double lr, double momentum,
                               double weight_decay, double rms_decay, double epsilon,
                               cdnn_handle stream);

/* ---- NCCL data-parallel subsystem (paper "Parallel object") */
CDNN_API int cdnn_nccl_available(int* out);
CDNN_API int cdnn_nccl_unique_id(uint8_t id[128]);
CDNN_API int cdnn_nccl_comm_create(cdnn_ctx ctx, int nranks, int rank, const uint8_t id[128],
                                   cdnn_handle* out);
/* the communicator's size and this process's rank, as NCCL reports them
 * (ncclCommCount / ncclCommUserRank) */
CDNN_API int cdnn_nccl_comm_info(cdnn_ctx ctx, cdnn_handle comm, int* nranks, int* rank);
/* in-place sum all-reduce of elements [offset, offset+n) of buf */
CDNN_API int cdnn_allreduce_sum(cdnn_ctx ctx, cdnn_handle comm, cdnn_handle buf, uint64_t offset,
                                uint64_t n, cdnn_handle stream);
CDNN_API int cdnn_broadcast(cdnn_ctx ctx, cdnn_handle comm, cdnn_handle buf, uint64_t n, int root,
                            cdnn_handle stream);

#ifdef __cplusplus
}
#endif

#endif /* CUDADNN_H_ */
