"""ctypes binding of the CudaDnn C-ABI (include/cudadnn.h).

This is the Python view of the device boundary: every call goes straight to
``lib/libcudadnn.so``.  There is no CPU fallback: without the built library or
without a CUDA device the calls raise ``CudnnError`` (status NO_DEVICE), so a
test or bench that passes has run the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libcudadnn.so")

OK = 0
STATUS = {
    0: "OK", 1: "INVALID_ARGUMENT", 2: "DANGLING_HANDLE", 3: "UNKNOWN_FUNCTION",
    4: "MODEL_ERROR", 5: "DATA_STARVATION", 6: "FORMAT_ERROR", 7: "NOT_FOUND",
    8: "INVALID_STATE", 9: "PARSE_ERROR", 10: "LOAD_ERROR", 11: "CUDA_ERROR", 12: "NO_DEVICE",
}
F32, F64, I32 = 0, 1, 2
MATH_TF32, MATH_TF32X3 = 0, 1
POOL_MAX, POOL_AVE = 0, 1
BN_RELU = 1  # cdnn_batchnorm_scale_forward_ex flags (CDNN_BN_RELU)
FAN_RELU = 1  # cdnn_fan_in_ex flags (CDNN_FAN_RELU)
SOLVER_SGD, SOLVER_RMSPROP = 0, 1
_NP = {F32: np.float32, F64: np.float64, I32: np.int32}

# every symbol include/cudadnn.h declares (checked by the CPU test suite)
EXPORTS = [
    "cdnn_last_error", "cdnn_status_name", "cdnn_device_count", "cdnn_ctx_create", "cdnn_ctx_destroy",
    "cdnn_ctx_device", "cdnn_live_slots", "cdnn_launch_count", "cdnn_set_math_mode", "cdnn_get_math_mode",
    "cdnn_alloc", "cdnn_free", "cdnn_view",
    "cdnn_length", "cdnn_buffer_dtype", "cdnn_device_ptr", "cdnn_write", "cdnn_read", "cdnn_write_async",
    "cdnn_read_async", "cdnn_host_alloc_pinned", "cdnn_host_free_pinned", "cdnn_stream_create",
    "cdnn_stream_free", "cdnn_stream_sync", "cdnn_stream_wait", "cdnn_graph_begin", "cdnn_graph_end",
    "cdnn_graph_launch", "cdnn_graph_free", "cdnn_event_create", "cdnn_event_record", "cdnn_event_elapsed",
    "cdnn_event_free", "cdnn_event_sync", "cdnn_rng_create", "cdnn_rng_next_u64", "cdnn_rng_uniform", "cdnn_subsystem_free",
    "cdnn_conv_desc_create", "cdnn_conv_output_shape", "cdnn_pool_desc_create", "cdnn_pool_output_shape",
    "cdnn_desc_free", "cdnn_dispatch", "cdnn_fill", "cdnn_copy", "cdnn_scal", "cdnn_axpy", "cdnn_dot", "cdnn_fan_out", "cdnn_fan_in", "cdnn_fan_in_ex",
    "cdnn_gemm", "cdnn_ip_forward", "cdnn_ip_backward", "cdnn_conv_forward", "cdnn_conv_backward_data", "cdnn_conv_backward_data_ex",
    "cdnn_conv_backward_filter", "cdnn_conv_backward_filter_ex", "cdnn_pool_forward", "cdnn_pool_backward", "cdnn_pool_backward_ex", "cdnn_relu_forward",
    "cdnn_relu_backward", "cdnn_sigmoid_forward", "cdnn_sigmoid_backward", "cdnn_softmax_forward",
    "cdnn_softmax_backward", "cdnn_softmax_loss_forward", "cdnn_softmax_loss_backward", "cdnn_solver_apply",
    "cdnn_nccl_available", "cdnn_nccl_unique_id", "cdnn_nccl_comm_create", "cdnn_nccl_comm_info", "cdnn_lrn_pool_supported", "cdnn_lrn_pool_forward",
    "cdnn_lrn_pool_backward", "cdnn_allreduce_sum",
    "cdnn_broadcast", "cdnn_copy_range", "cdnn_lrn_forward", "cdnn_lrn_backward", "cdnn_lrn_backward_ex", "cdnn_dropout", "cdnn_counter_increment",
    "cdnn_batchnorm_forward", "cdnn_batchnorm_backward", "cdnn_scale_forward", "cdnn_scale_backward",
    "cdnn_axpby", "cdnn_batchnorm_scale_forward", "cdnn_batchnorm_scale_forward_ex", "cdnn_batchnorm_scale_backward", "cdnn_conv_forward_ex",
    "cdnn_pool_forward_ex", "cdnn_pg_diff", "cdnn_mlp_pg_supported", "cdnn_mlp_pg_step", "cdnn_mlp_pg_step_host",
]


class CudnnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class ConvParams(C.Structure):
    _fields_ = [(f, C.c_int) for f in (
        "n", "c", "h", "w", "num_output", "kernel_h", "kernel_w", "stride_h", "stride_w",
        "pad_h", "pad_w", "dilation_h", "dilation_w", "group")]


class PoolParams(C.Structure):
    _fields_ = [(f, C.c_int) for f in (
        "n", "c", "h", "w", "method", "kernel_h", "kernel_w", "stride_h", "stride_w",
        "pad_h", "pad_w", "global_pooling")]


_lib: Optional[C.CDLL] = None


def load() -> C.CDLL:
    """Load libcudadnn.so (raises FileNotFoundError when it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} is not built; run `make -j8` or __graft_entry__.build()")
        lib = C.CDLL(LIB_PATH)
        u64, h, vp, i, d = C.c_uint64, C.c_uint64, C.c_void_p, C.c_int, C.c_double
        pu64, ph = C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)
        sig = {
            "cdnn_last_error": ([], C.c_char_p), "cdnn_status_name": ([i], C.c_char_p),
            "cdnn_device_count": ([C.POINTER(i)], i), "cdnn_ctx_create": ([i, C.POINTER(vp)], i),
            "cdnn_ctx_destroy": ([vp], i), "cdnn_ctx_device": ([vp, C.POINTER(i)], i),
            "cdnn_live_slots": ([vp, pu64], i), "cdnn_launch_count": ([vp, pu64], i),
            "cdnn_set_math_mode": ([vp, i], i), "cdnn_get_math_mode": ([vp, C.POINTER(i)], i),
            "cdnn_alloc": ([vp, u64, i, ph], i), "cdnn_free": ([vp, h], i),
            "cdnn_view": ([vp, h, u64, u64, ph], i), "cdnn_length": ([vp, h, pu64], i),
            "cdnn_buffer_dtype": ([vp, h, C.POINTER(i)], i), "cdnn_device_ptr": ([vp, h, C.POINTER(vp)], i),
            "cdnn_write": ([vp, h, vp, u64], i), "cdnn_read": ([vp, h, vp, u64], i),
            "cdnn_write_async": ([vp, h, u64, vp, u64, h], i), "cdnn_read_async": ([vp, h, u64, vp, u64, h], i),
            "cdnn_host_alloc_pinned": ([u64, C.POINTER(vp)], i), "cdnn_host_free_pinned": ([vp], i),
            "cdnn_stream_create": ([vp, ph], i), "cdnn_stream_free": ([vp, h], i),
            "cdnn_stream_sync": ([vp, h], i), "cdnn_stream_wait": ([vp, h, h], i),
            "cdnn_graph_begin": ([vp, h], i), "cdnn_graph_end": ([vp, h, ph], i),
            "cdnn_graph_launch": ([vp, h, h], i), "cdnn_graph_free": ([vp, h], i),
            "cdnn_event_create": ([vp, ph], i), "cdnn_event_record": ([vp, h, h], i),
            "cdnn_event_elapsed": ([vp, h, h, C.POINTER(C.c_float)], i), "cdnn_event_free": ([vp, h], i),
            "cdnn_event_sync": ([vp, h], i),
            "cdnn_rng_create": ([vp, u64, ph], i), "cdnn_rng_next_u64": ([vp, h, pu64], i),
            "cdnn_rng_uniform": ([vp, h, h, u64, d, d], i), "cdnn_subsystem_free": ([vp, h], i),
            "cdnn_conv_desc_create": ([vp, C.POINTER(ConvParams), ph], i),
            "cdnn_conv_output_shape": ([vp, h, C.POINTER(i)], i),
            "cdnn_pool_desc_create": ([vp, C.POINTER(PoolParams), ph], i),
            "cdnn_pool_output_shape": ([vp, h, C.POINTER(i)], i), "cdnn_desc_free": ([vp, h], i),
            "cdnn_dispatch": ([vp, i, C.POINTER(d), u64, C.POINTER(d), pu64], i),
            "cdnn_fill": ([vp, h, u64, d, h], i), "cdnn_copy": ([vp, h, h, u64, h], i),
            "cdnn_copy_range": ([vp, h, u64, h, u64, u64, h], i),
            "cdnn_scal": ([vp, u64, d, h, h], i), "cdnn_axpy": ([vp, u64, d, h, h, h], i),
            "cdnn_dot": ([vp, u64, h, h, C.POINTER(d)], i),
            "cdnn_fan_out": ([vp, h, C.POINTER(h), C.POINTER(d), i, u64, h], i),
            "cdnn_fan_in": ([vp, C.POINTER(h), i, h, u64, h], i),
            "cdnn_fan_in_ex": ([vp, C.POINTER(h), i, h, u64, i, h, h], i),
            "cdnn_gemm": ([vp, i, i, i, i, i, d, h, h, d, h, h], i),
            "cdnn_ip_forward": ([vp, h, h, h, h, i, i, i, i, h], i),
            "cdnn_ip_backward": ([vp, h, h, h, h, h, h, i, i, i, h], i),
            "cdnn_conv_forward": ([vp, h, h, h, h, h, h], i),
            "cdnn_conv_forward_ex": ([vp, h, h, h, h, h, i, h], i),
            "cdnn_conv_backward_data": ([vp, h, h, h, h, h], i),
            "cdnn_conv_backward_data_ex": ([vp, h, h, h, h, h, h], i),
            "cdnn_conv_backward_filter": ([vp, h, h, h, h, h, h], i),
            "cdnn_conv_backward_filter_ex": ([vp, h, h, h, h, h, i, h], i),
            "cdnn_pool_forward": ([vp, h, h, h, h, h], i), "cdnn_pool_forward_ex": ([vp, h, h, h, h, i, h], i), "cdnn_pool_backward": ([vp, h, h, h, h, h], i),
            "cdnn_pool_backward_ex": ([vp, h, h, h, h, h, h], i),
            "cdnn_relu_forward": ([vp, h, h, u64, h], i), "cdnn_relu_backward": ([vp, h, h, h, u64, h], i),
            "cdnn_sigmoid_forward": ([vp, h, h, u64, h], i), "cdnn_sigmoid_backward": ([vp, h, h, h, u64, h], i),
            "cdnn_softmax_forward": ([vp, h, h, i, i, h], i), "cdnn_softmax_backward": ([vp, h, h, h, i, i, h], i),
            "cdnn_softmax_loss_forward": ([vp, h, h, h, h, i, i, i, h], i),
            "cdnn_softmax_loss_backward": ([vp, h, h, h, i, i, i, d, h], i),
            "cdnn_solver_apply": ([vp, i, h, h, h, u64, d, d, d, d, d, h], i),
            "cdnn_nccl_available": ([C.POINTER(i)], i), "cdnn_nccl_unique_id": ([C.c_char_p], i),
            "cdnn_nccl_comm_create": ([vp, i, i, C.c_char_p, ph], i),
            "cdnn_nccl_comm_info": ([vp, u64, C.POINTER(i), C.POINTER(i)], i),
            "cdnn_lrn_pool_supported": ([vp, h, i, C.POINTER(i)], i),
            "cdnn_lrn_pool_forward": ([vp, h, h, h, h, h, i, d, d, d, i, h], i),
            "cdnn_lrn_pool_backward": ([vp, h, h, h, h, h, h, i, d, d, d, h], i),
            "cdnn_allreduce_sum": ([vp, h, h, u64, u64, h], i), "cdnn_broadcast": ([vp, h, h, u64, i, h], i),
            "cdnn_lrn_forward": ([vp, h, h, h, i, i, i, i, d, d, d, h], i),
            "cdnn_lrn_backward": ([vp, h, h, h, h, h, i, i, i, i, d, d, h], i),
            "cdnn_lrn_backward_ex": ([vp, h, h, h, h, h, i, i, i, i, d, d, h, h], i),
            "cdnn_dropout": ([vp, h, h, u64, d, u64, h, h], i), "cdnn_counter_increment": ([vp, h, h], i),
            "cdnn_batchnorm_forward": ([vp, h, h, h, h, i, i, i, d, h], i),
            "cdnn_batchnorm_backward": ([vp, h, h, h, h, h, i, i, i, h], i),
            "cdnn_scale_forward": ([vp, h, h, h, h, i, i, i, h], i),
            "cdnn_scale_backward": ([vp, h, h, h, h, h, h, i, i, i, h], i),
            "cdnn_axpby": ([vp, u64, d, h, d, h, i, h], i),
            "cdnn_pg_diff": ([vp, h, h, h, h, i, i, i, i, h], i),
            "cdnn_mlp_pg_supported": ([vp, i, i, i, i, i, C.POINTER(C.c_int)], i),
            "cdnn_mlp_pg_step": ([vp, h, h, h, i, i, i, i, i, h, h, h, C.POINTER(C.c_uint64), i, d, d, d, d, d,
                                  h, h, h, h], i),
            "cdnn_mlp_pg_step_host": ([vp, h, h, h, vp, vp, vp, vp, i, i, i, i, i, h, h, h, C.POINTER(C.c_uint64), i,
                                       d, d, d, d, d, h, h, h, h], i),
            "cdnn_batchnorm_scale_forward": ([vp, h, h, h, h, h, h, h, i, i, i, d, h], i),
            "cdnn_batchnorm_scale_forward_ex": ([vp, h, h, h, h, h, h, h, i, i, i, d, i, h], i),
            "cdnn_batchnorm_scale_backward": ([vp, h, h, h, h, h, h, h, h, i, i, i, h], i),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != OK:
        raise CudnnError(status, load().cdnn_last_error().decode(errors="replace"))


def device_count() -> int:
    n = C.c_int(0)
    check(load().cdnn_device_count(C.byref(n)))
    return n.value


class PinnedBuffer:
    """Page-locked host memory (cudaMallocHost) viewed as a numpy array; the
    feed / loss buffers of a captured step must be pinned."""

    def __init__(self, shape, dtype=np.float32):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        check(load().cdnn_host_alloc_pinned(max(self.nbytes, 1), C.byref(p)))
        self.ptr = p.value
        raw = (C.c_uint8 * max(self.nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(raw, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        if getattr(self, "ptr", None):
            load().cdnn_host_free_pinned(C.c_void_p(self.ptr))
            self.ptr = None


class Context:
    """One CudaDnn context (device + handle tables + compute stream)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        p = C.c_void_p()
        check(self.lib.cdnn_ctx_create(device, C.byref(p)))
        self.ptr = p

    def close(self) -> None:
        if self.ptr:
            check(self.lib.cdnn_ctx_destroy(self.ptr))
            self.ptr = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- call helper -----------------------------------------------------------
    def call(self, name: str, *args) -> None:
        check(getattr(self.lib, name)(self.ptr, *args))

    def _out_h(self, name: str, *args) -> int:
        h = C.c_uint64(0)
        check(getattr(self.lib, name)(self.ptr, *args, C.byref(h)))
        return h.value

    # -- tables ------------------------------------------------------------------
    def live_slots(self) -> int:
        v = C.c_uint64()
        check(self.lib.cdnn_live_slots(self.ptr, C.byref(v)))
        return v.value

    def launch_count(self) -> int:
        v = C.c_uint64()
        check(self.lib.cdnn_launch_count(self.ptr, C.byref(v)))
        return v.value

    def alloc(self, length: int, dtype: int = F32) -> int:
        return self._out_h("cdnn_alloc", length, dtype)

    def free(self, h: int) -> None:
        self.call("cdnn_free", h)

    def view(self, h: int, offset: int, length: int) -> int:
        return self._out_h("cdnn_view", h, offset, length)

    def length(self, h: int) -> int:
        v = C.c_uint64()
        self.call("cdnn_length", h, C.byref(v))
        return v.value

    def dtype(self, h: int) -> int:
        v = C.c_int()
        self.call("cdnn_buffer_dtype", h, C.byref(v))
        return v.value

    def device_ptr(self, h: int) -> int:
        v = C.c_void_p()
        self.call("cdnn_device_ptr", h, C.byref(v))
        return v.value or 0

    def upload(self, arr: np.ndarray, dtype: Optional[int] = None) -> int:
        """Allocate a buffer holding `arr` (dtype inferred from arr)."""
        if dtype is None:
            dtype = {np.dtype(np.float32): F32, np.dtype(np.float64): F64, np.dtype(np.int32): I32}[arr.dtype]
        a = np.ascontiguousarray(arr, dtype=_NP[dtype]).ravel()
        h = self.alloc(max(a.size, 1), dtype)
        if a.size:
            self.write(h, a)
        return h

    def write(self, h: int, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, dtype=_NP[self.dtype(h)]).ravel()
        self.call("cdnn_write", h, a.ctypes.data_as(C.c_void_p), a.size)

    def read(self, h: int, n: Optional[int] = None) -> np.ndarray:
        dt = self.dtype(h)
        n = self.length(h) if n is None else n
        out = np.empty(n, dtype=_NP[dt])
        self.call("cdnn_read", h, out.ctypes.data_as(C.c_void_p), n)
        return out

    def sync(self, stream: int = 0) -> None:
        self.call("cdnn_stream_sync", stream)

    # -- streams / graphs / events ----------------------------------------------------
    def stream_create(self) -> int:
        return self._out_h("cdnn_stream_create")

    def graph_begin(self, stream: int = 0) -> None:
        self.call("cdnn_graph_begin", stream)

    def graph_end(self, stream: int = 0) -> int:
        return self._out_h("cdnn_graph_end", stream)

    def graph_launch(self, g: int, stream: int = 0) -> None:
        self.call("cdnn_graph_launch", g, stream)

    def event(self) -> int:
        return self._out_h("cdnn_event_create")

    def record(self, ev: int, stream: int = 0) -> None:
        self.call("cdnn_event_record", ev, stream)

    def elapsed_ms(self, a: int, b: int) -> float:
        v = C.c_float()
        self.call("cdnn_event_elapsed", a, b, C.byref(v))
        return float(v.value)

    # -- rng ----------------------------------------------------------------------
    def rng_create(self, seed: int) -> int:
        return self._out_h("cdnn_rng_create", seed)

    def rng_uniform(self, rng: int, dst: int, n: int, lo: float, hi: float) -> None:
        self.call("cdnn_rng_uniform", rng, dst, n, lo, hi)

    def subsystem_free(self, h: int) -> None:
        self.call("cdnn_subsystem_free", h)

    # -- descriptors ---------------------------------------------------------------
    def conv_desc(self, n, c, h, w, num_output, kernel, stride=1, pad=0, dilation=1, group=1) -> int:
        kh, kw = (kernel, kernel) if isinstance(kernel, int) else kernel
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        dh, dw = (dilation, dilation) if isinstance(dilation, int) else dilation
        p = ConvParams(n, c, h, w, num_output, kh, kw, sh, sw, ph, pw, dh, dw, group)
        return self._out_h("cdnn_conv_desc_create", C.byref(p))

    def conv_output_shape(self, d: int) -> tuple:
        out = (C.c_int * 4)()
        self.call("cdnn_conv_output_shape", d, out)
        return tuple(out)

    def pool_desc(self, n, c, h, w, method, kernel, stride=1, pad=0, global_pooling=False) -> int:
        kh, kw = (kernel, kernel) if isinstance(kernel, int) else kernel
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        p = PoolParams(n, c, h, w, method, kh, kw, sh, sw, ph, pw, int(global_pooling))
        return self._out_h("cdnn_pool_desc_create", C.byref(p))

    def pool_output_shape(self, d: int) -> tuple:
        out = (C.c_int * 4)()
        self.call("cdnn_pool_output_shape", d, out)
        return tuple(out)

    # -- dispatch ------------------------------------------------------------------------
    def dispatch(self, index: int, args: Sequence[float]) -> list:
        a = (C.c_double * max(len(args), 1))(*args)
        out = (C.c_double * 4)()
        nout = C.c_uint64(4)
        check(self.lib.cdnn_dispatch(self.ptr, index, a, len(args), out, C.byref(nout)))
        return [out[i] for i in range(nout.value)]

    def dot(self, n: int, x: int, y: int) -> float:
        r = C.c_double()
        self.call("cdnn_dot", n, x, y, C.byref(r))
        return r.value
