// dispatch.cu — the frozen function-index boundary (paper's "Cuda Control":
// "parameters and a function index"), restating
// Registry::dispatch (backend.cpp:248-305) with its arity and decoding checks
// (backend.cpp:213-246).  Indices 1-7 keep the reference argument layout
// (backend.hpp:47-69); 8-13 are appended.  Handle ids travel as doubles
// exactly like the reference's `real` args.  Every call is synchronous so the
// buffer state afterwards equals the direct call's.
#include <cmath>
#include <string>

#include "internal.hpp"

using namespace cdnn;

namespace {

cdnn_handle decode_handle(double v, const char* what) {
  if (!(v >= 0) || v != std::floor(v))
    fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": " + std::to_string(v) + " is not a handle id");
  return static_cast<cdnn_handle>(v);
}
uint64_t decode_size(double v, const char* what) {
  if (!(v >= 0) || v != std::floor(v))
    fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": " + std::to_string(v) + " is not a valid count");
  return static_cast<uint64_t>(v);
}
int decode_int(double v, const char* what) {
  if (v != std::floor(v)) fail(CDNN_INVALID_ARGUMENT, std::string(what) + ": " + std::to_string(v) + " is not an integer");
  return static_cast<int>(v);
}
void check_arity(int index, const char* name, uint64_t n, uint64_t expected) {
  if (n != expected)
    fail(CDNN_INVALID_ARGUMENT, "dispatch: function " + std::to_string(index) + " (" + name + ") expects " +
                                    std::to_string(expected) + " arguments, got " + std::to_string(n));
}
void ok(int status) {
  if (status != CDNN_OK) throw Error{status, cdnn_last_error()};
}

}  // namespace

extern "C" int cdnn_dispatch(cdnn_ctx ctx, int fi, const double* a, uint64_t n, double* out, uint64_t* nout) {
  return guarded([&] {
    Ctx* c = need_ctx(ctx);
    if (n > 0 && !a) fail(CDNN_INVALID_ARGUMENT, "dispatch: null argument array");
    uint64_t produced = 0;
    switch (fi) {
      case CDNN_FN_FILL:
        check_arity(fi, "fill", n, 3);
        ok(cdnn_fill(c, decode_handle(a[0], "fill dst"), decode_size(a[1], "fill n"), a[2], 0));
        break;
      case CDNN_FN_COPY:
        check_arity(fi, "copy", n, 3);
        ok(cdnn_copy(c, decode_handle(a[0], "copy src"), decode_handle(a[1], "copy dst"), decode_size(a[2], "copy n"), 0));
        break;
      case CDNN_FN_SCAL:
        check_arity(fi, "scal", n, 3);
        ok(cdnn_scal(c, decode_size(a[0], "scal n"), a[1], decode_handle(a[2], "scal x"), 0));
        break;
      case CDNN_FN_AXPY:
        check_arity(fi, "axpy", n, 4);
        ok(cdnn_axpy(c, decode_size(a[0], "axpy n"), a[1], decode_handle(a[2], "axpy x"), decode_handle(a[3], "axpy y"), 0));
        break;
      case CDNN_FN_DOT: {
        check_arity(fi, "dot", n, 3);
        double r = 0;
        ok(cdnn_dot(c, decode_size(a[0], "dot n"), decode_handle(a[1], "dot x"), decode_handle(a[2], "dot y"), &r));
        if (out && nout && *nout >= 1) out[0] = r;
        produced = 1;
        break;
      }
      case CDNN_FN_GEMM:
        check_arity(fi, "gemm", n, 10);
        ok(cdnn_gemm(c, decode_int(a[0], "gemm trans_a") != 0, decode_int(a[1], "gemm trans_b") != 0,
                     decode_int(a[2], "gemm m"), decode_int(a[3], "gemm n"), decode_int(a[4], "gemm k"), a[5],
                     decode_handle(a[6], "gemm a"), decode_handle(a[7], "gemm b"), a[8], decode_handle(a[9], "gemm c"), 0));
        break;
      case CDNN_FN_RNG_UNIFORM:
        check_arity(fi, "rng_uniform", n, 5);
        ok(cdnn_rng_uniform(c, decode_handle(a[0], "rng_uniform rng"), decode_handle(a[1], "rng_uniform dst"),
                            decode_size(a[2], "rng_uniform n"), a[3], a[4]));
        break;
      case CDNN_FN_RELU_FWD:
        check_arity(fi, "relu_forward", n, 3);
        ok(cdnn_relu_forward(c, decode_handle(a[0], "relu x"), decode_handle(a[1], "relu y"), decode_size(a[2], "relu n"), 0));
        break;
      case CDNN_FN_RELU_BWD:
        check_arity(fi, "relu_backward", n, 4);
        ok(cdnn_relu_backward(c, decode_handle(a[0], "relu x"), decode_handle(a[1], "relu dy"),
                              decode_handle(a[2], "relu dx"), decode_size(a[3], "relu n"), 0));
        break;
      case CDNN_FN_SIGMOID_FWD:
        check_arity(fi, "sigmoid_forward", n, 3);
        ok(cdnn_sigmoid_forward(c, decode_handle(a[0], "sigmoid x"), decode_handle(a[1], "sigmoid y"),
                                decode_size(a[2], "sigmoid n"), 0));
        break;
      case CDNN_FN_SIGMOID_BWD:
        check_arity(fi, "sigmoid_backward", n, 4);
        ok(cdnn_sigmoid_backward(c, decode_handle(a[0], "sigmoid y"), decode_handle(a[1], "sigmoid dy"),
                                 decode_handle(a[2], "sigmoid dx"), decode_size(a[3], "sigmoid n"), 0));
        break;
      case CDNN_FN_SOFTMAX_FWD:
        check_arity(fi, "softmax_forward", n, 4);
        ok(cdnn_softmax_forward(c, decode_handle(a[0], "softmax x"), decode_handle(a[1], "softmax y"),
                                decode_int(a[2], "softmax rows"), decode_int(a[3], "softmax features"), 0));
        break;
      case CDNN_FN_SOFTMAX_BWD:
        check_arity(fi, "softmax_backward", n, 5);
        ok(cdnn_softmax_backward(c, decode_handle(a[0], "softmax y"), decode_handle(a[1], "softmax dy"),
                                 decode_handle(a[2], "softmax dx"), decode_int(a[3], "softmax rows"),
                                 decode_int(a[4], "softmax features"), 0));
        break;
      default:
        fail(CDNN_UNKNOWN_FUNCTION, "dispatch: no function with index " + std::to_string(fi));
    }
    if (fi != CDNN_FN_DOT && fi != CDNN_FN_RNG_UNIFORM) ok(cdnn_stream_sync(c, 0));
    if (nout) *nout = produced;
  });
}
