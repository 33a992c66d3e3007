"""ctypes binding of include/polegrad_c.h — the reference-compatible Net /
Solver / Parallel API of the B200 library, in float (TF32 tensor cores) or
double (SIMT FP64) flavour.

    net = Net(open("models/cifar10_quick.prototxt").read(), seed=1, dtype="f32")
    solver = Solver(net, method="sgd", lr=1e-3, momentum=0.9, weight_decay=4e-3)
    net.set_batch(images, labels); net.forward(); net.backward(); solver.apply()

Everything runs on the GPU through libcudadnn.so; without a device the
constructor raises (status NO_DEVICE) — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import cudadnn

_HERE = os.path.dirname(os.path.abspath(__file__))
MODELS_DIR = os.path.join(_HERE, "models")
_LIBS: Dict[str, C.CDLL] = {}
NP_DTYPE = {"f32": np.float32, "f64": np.float64}

EXPORTS = [
    "pg_last_error", "pg_real_size", "pg_net_create", "pg_net_free", "pg_net_forward", "pg_net_backward",
    "pg_net_backward_from", "pg_net_loss", "pg_net_set_batch", "pg_net_enqueue", "pg_net_sync", "pg_net_context",
    "pg_net_num_layers", "pg_net_layer_name", "pg_blob_shape", "pg_blob_get", "pg_blob_set", "pg_param_count",
    "pg_param_info", "pg_param_get", "pg_param_set", "pg_pool_mask", "pg_snapshot", "pg_restore",
    "pg_solver_create", "pg_solver_free", "pg_solver_apply", "pg_step_capture", "pg_step_replay", "pg_graph_free",
    "pg_net_profile",
    "pg_parallel_unique_id", "pg_parallel_create", "pg_parallel_free", "pg_parallel_broadcast",
    "pg_solver_set_parallel", "pg_plan_buckets", "pg_prototxt_roundtrip", "pg_solver_snapshot",
    "pg_solver_restore", "pg_solver_iterations", "pg_feed_ring_create", "pg_feed_ring_free", "pg_feed_ring_push", "pg_feed_ring_push_pinned",
    "pg_feed_ring_pop_loss", "pg_net_pg_backward", "pg_feed_ring_push_sampled", "pg_imagedb_load",
    "pg_imagedb_free", "pg_imagedb_size", "pg_imagedb_set_boost", "pg_imagedb_sample", "pg_rng_create",
    "pg_rng_free", "pg_parallel_create_host", "pg_parallel_info", "pg_pg_step_capture",
    "pg_pg_step_capture_ex", "pg_pg_step_fused",
]

# int transport(void* user, int op, void* host, uint64_t offset, uint64_t n)
HOST_TRANSPORT = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_uint64)


def lib_path(dtype: str) -> str:
    return os.path.join(cudadnn.LIB_DIR, f"libpolegrad_b200_{dtype}.so")


def load(dtype: str = "f32") -> C.CDLL:
    if dtype not in ("f32", "f64"):
        raise ValueError("dtype must be 'f32' or 'f64'")
    if dtype not in _LIBS:
        path = lib_path(dtype)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} is not built; run `make -j8` or __graft_entry__.build()")
        cudadnn.load()  # libcudadnn.so first (rpath $ORIGIN resolves it anyway)
        lib = C.CDLL(path)
        vp, i, u64, d, cp = C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_char_p
        sig = {
            "pg_last_error": ([], cp), "pg_real_size": ([], i),
            "pg_net_create": ([cp, u64, i, C.POINTER(vp)], i), "pg_net_free": ([vp], i),
            "pg_net_forward": ([vp], i), "pg_net_backward": ([vp], i), "pg_net_backward_from": ([vp, cp], i),
            "pg_net_pg_backward": ([vp, cp, cp, vp, vp, u64, i], i),
            "pg_net_loss": ([vp, C.POINTER(d)], i), "pg_net_set_batch": ([vp, vp, vp], i),
            "pg_net_enqueue": ([vp, cp, vp, u64], i), "pg_net_sync": ([vp], i),
            "pg_net_context": ([vp, C.POINTER(vp)], i), "pg_net_num_layers": ([vp], i),
            "pg_net_layer_name": ([vp, i, cp, i], i), "pg_blob_shape": ([vp, cp, C.POINTER(i)], i),
            "pg_blob_get": ([vp, cp, i, vp], i), "pg_blob_set": ([vp, cp, i, vp], i),
            "pg_param_count": ([vp], i), "pg_param_info": ([vp, i, cp, i, C.POINTER(i)], i),
            "pg_param_get": ([vp, i, i, vp], i), "pg_param_set": ([vp, i, i, vp], i),
            "pg_pool_mask": ([vp, cp, C.POINTER(C.c_int32), u64], i),
            "pg_snapshot": ([vp, vp, u64, C.POINTER(u64)], i), "pg_restore": ([vp, vp, u64], i),
            "pg_solver_create": ([i, d, d, d, d, d, C.POINTER(vp)], i), "pg_solver_free": ([vp], i),
            "pg_solver_apply": ([vp, vp], i), "pg_solver_snapshot": ([vp, vp, u64, C.POINTER(u64)], i),
            "pg_solver_restore": ([vp, vp, u64], i), "pg_solver_iterations": ([vp, C.POINTER(u64)], i),
            "pg_feed_ring_create": ([vp, vp, i, C.POINTER(vp)], i), "pg_feed_ring_free": ([vp], i),
            "pg_feed_ring_push": ([vp, vp, u64, vp, u64], i),
            "pg_feed_ring_push_pinned": ([vp, vp, u64, vp, u64], i), "pg_feed_ring_pop_loss": ([vp, C.POINTER(d)], i),
            "pg_step_capture": ([vp, vp, vp, vp, vp, C.POINTER(u64)], i), "pg_step_replay": ([vp, u64], i),
            "pg_pg_step_capture": ([vp, vp, vp, vp, vp, u64, cp, cp, i, vp, C.POINTER(u64)], i),
            "pg_pg_step_capture_ex": ([vp, vp, vp, vp, vp, u64, cp, cp, i, i, vp, C.POINTER(u64)], i),
            "pg_pg_step_fused": ([vp, vp, cp, cp, i, i, C.POINTER(C.c_int)], i),
            "pg_graph_free": ([vp, u64], i), "pg_parallel_unique_id": ([cp], i),
            "pg_net_profile": ([vp, C.POINTER(C.c_float), C.POINTER(C.c_float), i], i),
            "pg_parallel_create": ([vp, i, i, cp, u64, C.POINTER(vp)], i), "pg_parallel_free": ([vp], i),
            "pg_parallel_broadcast": ([vp], i), "pg_solver_set_parallel": ([vp, vp], i),
            "pg_parallel_create_host": ([vp, i, i, HOST_TRANSPORT, vp, u64, C.POINTER(vp)], i),
            "pg_parallel_info": ([vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(u64)], i),
            "pg_plan_buckets": ([C.POINTER(u64), C.POINTER(u64), i, u64, u64, C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32)], i),
            "pg_prototxt_roundtrip": ([cp, cp, u64, C.POINTER(u64)], i),
            "pg_feed_ring_push_sampled": ([vp, vp, i, i, vp], i),
            "pg_imagedb_load": ([cp, C.POINTER(vp)], i), "pg_imagedb_free": ([vp], i),
            "pg_imagedb_size": ([vp, C.POINTER(u64)], i), "pg_imagedb_set_boost": ([vp, C.c_int64, d], i),
            "pg_imagedb_sample": ([vp, i, i, vp, u64, C.POINTER(C.c_int64)], i),
            "pg_rng_create": ([u64, C.POINTER(vp)], i), "pg_rng_free": ([vp], i),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes, fn.restype = args, res
        _LIBS[dtype] = lib
    return _LIBS[dtype]


class PolegradError(cudadnn.CudnnError):
    pass


def _check(lib: C.CDLL, status: int) -> None:
    if status != 0:
        raise PolegradError(status, lib.pg_last_error().decode(errors="replace"))


def prototxt_roundtrip(text: str, dtype: str = "f64") -> str:
    lib = load(dtype)
    n = C.c_uint64(0)
    _check(lib, lib.pg_prototxt_roundtrip(text.encode(), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib, lib.pg_prototxt_roundtrip(text.encode(), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def plan_buckets(offsets: List[int], counts: List[int], total: int, bucket_elems: int,
                 dtype: str = "f32") -> Tuple[List[int], int]:
    """Host-only bucket planner of polegrad::Parallel (no GPU needed)."""
    lib = load(dtype)
    n = len(offsets)
    o = (C.c_uint64 * max(n, 1))(*offsets)
    c = (C.c_uint64 * max(n, 1))(*counts)
    out = (C.c_int32 * max(n, 1))()
    nb = C.c_int32()
    _check(lib, lib.pg_plan_buckets(o, c, n, total, bucket_elems, out, C.byref(nb)))
    return [out[i] for i in range(n)], nb.value


def load_model(name: str, batch: Optional[int] = None) -> str:
    """Prototxt text of a bundled model; `batch` rewrites the MemoryData batch_size."""
    with open(os.path.join(MODELS_DIR, name if name.endswith(".prototxt") else name + ".prototxt")) as f:
        text = f.read()
    if batch is not None:
        import re
        text = re.sub(r"batch_size:\s*\d+", f"batch_size: {int(batch)}", text, count=1)
    return text


class Net:
    """polegrad::Net on a CUDA device (reference net.hpp API)."""

    def __init__(self, prototxt: str, seed: int = 1, dtype: str = "f32", device: int = 0):
        self.dtype = dtype
        self.np = NP_DTYPE[dtype]
        self.lib = load(dtype)
        p = C.c_void_p()
        _check(self.lib, self.lib.pg_net_create(prototxt.encode(), seed, device, C.byref(p)))
        self.ptr = p
        self._shapes: Dict[str, Tuple[int, ...]] = {}

    def close(self) -> None:
        if self.ptr:
            _check(self.lib, self.lib.pg_net_free(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, name: str, *args) -> None:
        _check(self.lib, getattr(self.lib, name)(self.ptr, *args))

    # ---- execution -------------------------------------------------------------------
    def forward(self) -> None:
        self._c("pg_net_forward")

    def backward(self) -> None:
        self._c("pg_net_backward")

    def backward_from(self, blob: str) -> None:
        self._c("pg_net_backward_from", blob.encode())

    def pg_backward(self, actions, returns, logit: str = "logits", prob: str = "prob", sigmoid: bool = False) -> None:
        """Policy-gradient episode batch on the device (Net::pg_backward)."""
        a = np.ascontiguousarray(actions, dtype=self.np)
        g = np.ascontiguousarray(returns, dtype=self.np)
        self._c("pg_net_pg_backward", logit.encode(), prob.encode(), a.ctypes.data, g.ctypes.data, a.size,
                1 if sigmoid else 0)

    def loss(self) -> float:
        v = C.c_double()
        self._c("pg_net_loss", C.byref(v))
        return v.value

    def set_batch(self, data: np.ndarray, labels: Optional[np.ndarray] = None) -> None:
        """Synchronous-safe staging: keeps references until the next sync."""
        self._staged = (np.ascontiguousarray(data, self.np),
                        None if labels is None else np.ascontiguousarray(labels, self.np))
        d, l = self._staged
        self._c("pg_net_set_batch", d.ctypes.data_as(C.c_void_p), None if l is None else l.ctypes.data_as(C.c_void_p))
        self.sync()

    def set_batch_ptr(self, data_ptr: int, labels_ptr: Optional[int]) -> None:
        self._c("pg_net_set_batch", C.c_void_p(data_ptr), C.c_void_p(labels_ptr) if labels_ptr else None)

    def enqueue(self, sample: np.ndarray, layer: str = "") -> None:
        s = np.ascontiguousarray(sample, self.np).ravel()
        self._c("pg_net_enqueue", layer.encode(), s.ctypes.data_as(C.c_void_p), s.size)

    def sync(self) -> None:
        self._c("pg_net_sync")

    def context_ptr(self) -> int:
        p = C.c_void_p()
        self._c("pg_net_context", C.byref(p))
        return p.value

    def layer_names(self) -> List[str]:
        n = self.lib.pg_net_num_layers(self.ptr)
        out = []
        buf = C.create_string_buffer(256)
        for i in range(n):
            self._c("pg_net_layer_name", i, buf, 256)
            out.append(buf.value.decode())
        return out

    # ---- blobs / params -------------------------------------------------------------------
    def blob_shape(self, name: str) -> Tuple[int, ...]:
        s = (C.c_int * 4)()
        self._c("pg_blob_shape", name.encode(), s)
        return tuple(s)

    def blob(self, name: str, diff: bool = False) -> np.ndarray:
        shape = self.blob_shape(name)
        out = np.empty(shape, self.np)
        self._c("pg_blob_get", name.encode(), int(diff), out.ctypes.data_as(C.c_void_p))
        return out

    def set_blob(self, name: str, values: np.ndarray, diff: bool = False) -> None:
        shape = self.blob_shape(name)
        v = np.ascontiguousarray(values, self.np).reshape(shape)
        self._c("pg_blob_set", name.encode(), int(diff), v.ctypes.data_as(C.c_void_p))

    def param_info(self) -> List[Tuple[str, Tuple[int, ...]]]:
        out = []
        buf = C.create_string_buffer(256)
        for i in range(self.lib.pg_param_count(self.ptr)):
            s = (C.c_int * 4)()
            self._c("pg_param_info", i, buf, 256, s)
            out.append((buf.value.decode(), tuple(s)))
        return out

    def param(self, i: int, diff: bool = False) -> np.ndarray:
        shape = self.param_info()[i][1]
        out = np.empty(shape, self.np)
        self._c("pg_param_get", i, int(diff), out.ctypes.data_as(C.c_void_p))
        return out

    def set_param(self, i: int, values: np.ndarray, diff: bool = False) -> None:
        shape = self.param_info()[i][1]
        v = np.ascontiguousarray(values, self.np).reshape(shape)
        self._c("pg_param_set", i, int(diff), v.ctypes.data_as(C.c_void_p))

    def pool_mask(self, layer: str) -> np.ndarray:
        # size from the layer's top: look it up through the layer list / blob shapes
        n = 1 << 26
        buf = np.empty(0, np.int32)
        for cap in (1 << 16, 1 << 20, 1 << 24, n):
            buf = np.empty(cap, np.int32)
            st = self.lib.pg_pool_mask(self.ptr, layer.encode(), buf.ctypes.data_as(C.POINTER(C.c_int32)), cap)
            if st == 0:
                return buf
            if st != 1:
                _check(self.lib, st)
        _check(self.lib, 1)
        return buf

    def snapshot(self) -> bytes:
        n = C.c_uint64()
        self._c("pg_snapshot", None, 0, C.byref(n))
        buf = (C.c_uint8 * n.value)()
        self._c("pg_snapshot", buf, n.value, C.byref(n))
        return bytes(buf)

    def restore(self, blob: bytes) -> None:
        b = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        self._c("pg_restore", b, len(blob))


class Solver:
    """polegrad::Solver (SGD / RMSProp + Caffe momentum & weight decay)."""

    def __init__(self, net: Net, method: str = "sgd", lr: float = 1e-3, momentum: float = 0.0,
                 weight_decay: float = 0.0, rms_decay: float = 0.99, epsilon: float = 1e-8):
        self.net = net
        self.lib = net.lib
        p = C.c_void_p()
        _check(self.lib, self.lib.pg_solver_create(1 if method == "rmsprop" else 0, lr, momentum, weight_decay,
                                                   rms_decay, epsilon, C.byref(p)))
        self.ptr = p

    def apply(self) -> None:
        _check(self.lib, self.lib.pg_solver_apply(self.ptr, self.net.ptr))

    def set_parallel(self, par: Optional["Parallel"]) -> None:
        _check(self.lib, self.lib.pg_solver_set_parallel(self.ptr, par.ptr if par else None))

    def snapshot(self) -> bytes:
        """Solver-state checkpoint ("MCSS": update count + momentum / RMSProp history)."""
        n = C.c_uint64()
        _check(self.lib, self.lib.pg_solver_snapshot(self.ptr, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _check(self.lib, self.lib.pg_solver_snapshot(self.ptr, buf, n.value, C.byref(n)))
        return bytes(buf)

    def restore(self, blob: bytes) -> None:
        b = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(self.lib, self.lib.pg_solver_restore(self.ptr, b, len(blob)))

    @property
    def iterations(self) -> int:
        v = C.c_uint64()
        _check(self.lib, self.lib.pg_solver_iterations(self.ptr, C.byref(v)))
        return v.value

    def close(self) -> None:
        if self.ptr:
            _check(self.lib, self.lib.pg_solver_free(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StepGraph:
    """One captured training step: H2D(pinned batch) -> fwd -> bwd -> update -> D2H(loss)."""

    def __init__(self, net: Net, solver: Solver, data_ptr: int, labels_ptr: Optional[int], loss_ptr: int):
        self.net = net
        g = C.c_uint64()
        _check(net.lib, net.lib.pg_step_capture(net.ptr, solver.ptr, C.c_void_p(data_ptr),
                                                C.c_void_p(labels_ptr) if labels_ptr else None,
                                                C.c_void_p(loss_ptr), C.byref(g)))
        self.graph = g.value

    def replay(self) -> None:
        _check(self.net.lib, self.net.lib.pg_step_replay(self.net.ptr, self.graph))


class PGStepGraph:
    """One captured policy-gradient update of an episode batch (pg_pg_step_capture):
    states -> forward -> device-side modulated log-prob gradients of `n` steps ->
    backward_from(logits) -> update -> probabilities to `prob`.  The buffers are
    cudadnn.PinnedBuffer of the net's real type; write the next episode into them and
    replay().  Capture after at least one eager update (lazy device buffers).

    fused=True (default): when the net is the pg_softmax MLP (InnerProduct -> ReLU ->
    InnerProduct -> Softmax) the update is one kernel (cdnn_mlp_pg_step) instead of
    the layer-by-layer launches; `self.fused` says which was captured."""

    LAYERED = 1  # PG_STEP_LAYERED

    def __init__(self, net: Net, solver: "Solver", states, actions, returns, n: int, prob=None,
                 logit: str = "logits", prob_blob: str = "prob", sigmoid: bool = False, fused: bool = True):
        self.net = net
        self._keep = (solver, states, actions, returns, prob)
        flags = 0 if fused else self.LAYERED
        ok = C.c_int(0)
        _check(net.lib, net.lib.pg_pg_step_fused(net.ptr, solver.ptr, logit.encode(), prob_blob.encode(),
                                                 int(sigmoid), flags, C.byref(ok)))
        self.fused = bool(ok.value)
        g = C.c_uint64()
        _check(net.lib, net.lib.pg_pg_step_capture_ex(net.ptr, solver.ptr, C.c_void_p(states.ptr),
                                                      C.c_void_p(actions.ptr), C.c_void_p(returns.ptr), n,
                                                      logit.encode(), prob_blob.encode(), int(sigmoid), flags,
                                                      C.c_void_p(prob.ptr) if prob is not None else None,
                                                      C.byref(g)))
        self.graph = g.value

    def replay(self) -> None:
        _check(self.net.lib, self.net.lib.pg_step_replay(self.net.ptr, self.graph))


class FeedRing:
    """polegrad::FeedRing — pinned-memory feed ring of `depth` captured steps
    (H2D(slot) -> forward -> backward -> update -> D2H(loss)); push() stages the
    next batch on the host while earlier steps run, pop_loss() returns losses
    in push order."""

    def __init__(self, net: Net, solver: "Solver", depth: int = 2):
        self.net = net
        self.lib = net.lib
        self._keep = solver
        p = C.c_void_p()
        _check(self.lib, self.lib.pg_feed_ring_create(net.ptr, solver.ptr, depth, C.byref(p)))
        self.ptr = p

    def push(self, data: np.ndarray, labels: Optional[np.ndarray] = None) -> None:
        x = np.ascontiguousarray(data, dtype=self.net.np)
        y = None if labels is None else np.ascontiguousarray(labels, dtype=self.net.np)
        _check(self.lib, self.lib.pg_feed_ring_push(self.ptr, x.ctypes.data, x.size,
                                                    None if y is None else y.ctypes.data,
                                                    0 if y is None else y.size))

    def push_pinned(self, data, labels=None) -> None:
        """Zero-copy push of batches already in page-locked memory (cudadnn.PinnedBuffer):
        the H2D is enqueued from them; keep them unchanged until this step's pop_loss().
        The buffers must hold the net's real type (float32 for the f32 library, float64
        for f64): the library copies count * sizeof(real) bytes from them."""
        for name, buf in (("data", data), ("labels", labels)):
            if buf is None:
                continue
            arr = buf.array
            if arr.dtype != np.dtype(self.net.np) or not arr.flags.c_contiguous:
                raise TypeError(f"push_pinned: {name} buffer is {arr.dtype}"
                                f"{'' if arr.flags.c_contiguous else ' (not C-contiguous)'}; "
                                f"the {self.net.dtype} library needs a C-contiguous {np.dtype(self.net.np)} "
                                f"PinnedBuffer")
        _check(self.lib, self.lib.pg_feed_ring_push_pinned(self.ptr, data.ptr, data.array.size,
                                                           None if labels is None else labels.ptr,
                                                           0 if labels is None else labels.array.size))

    def push_sampled(self, db: "ImageDB", rng: "Rng", method: str = "uniform", use_boost: bool = False) -> None:
        """Samples one batch from `db` (one `rng` draw per image) and gathers it
        straight into the next pinned slot (polegrad::FeedRing::push_sampled)."""
        _check(self.lib, self.lib.pg_feed_ring_push_sampled(self.ptr, db.ptr, _SAMPLE_METHODS[method],
                                                            int(use_boost), rng.ptr))

    def pop_loss(self) -> float:
        v = C.c_double()
        _check(self.lib, self.lib.pg_feed_ring_pop_loss(self.ptr, C.byref(v)))
        return v.value

    def close(self) -> None:
        if self.ptr:
            _check(self.lib, self.lib.pg_feed_ring_free(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_SAMPLE_METHODS = {"uniform": 0, "label_balanced": 1}


class _Owned:
    _free = ""

    def close(self) -> None:
        if getattr(self, "ptr", None):
            _check(self.lib, getattr(self.lib, self._free)(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rng(_Owned):
    """polegrad::Rng (mt19937_64, uniform01 = (next >> 11) * 2^-53)."""
    _free = "pg_rng_free"

    def __init__(self, seed: int, dtype: str = "f32"):
        self.lib = load(dtype)
        p = C.c_void_p()
        _check(self.lib, self.lib.pg_rng_create(seed, C.byref(p)))
        self.ptr = p


class ImageDB(_Owned):
    """polegrad::imagedb::Dataset loaded from an index file (reference imagedb.hpp:12-53;
    format in include/polegrad/imagedb.hpp, writer: write_imagedb)."""
    _free = "pg_imagedb_free"

    def __init__(self, index_path: str, dtype: str = "f32"):
        self.lib = load(dtype)
        p = C.c_void_p()
        _check(self.lib, self.lib.pg_imagedb_load(str(index_path).encode(), C.byref(p)))
        self.ptr = p

    def __len__(self) -> int:
        n = C.c_uint64()
        _check(self.lib, self.lib.pg_imagedb_size(self.ptr, C.byref(n)))
        return n.value

    def set_boost(self, entry_id: int, boost: float) -> None:
        _check(self.lib, self.lib.pg_imagedb_set_boost(self.ptr, entry_id, boost))

    def sample(self, rng: Rng, n: int, method: str = "uniform", use_boost: bool = False) -> np.ndarray:
        ids = np.zeros(n, dtype=np.int64)
        _check(self.lib, self.lib.pg_imagedb_sample(self.ptr, _SAMPLE_METHODS[method], int(use_boost), rng.ptr, n,
                                                    ids.ctypes.data_as(C.POINTER(C.c_int64))))
        return ids


def write_imagedb(directory: str, entries) -> str:
    """Writes `entries` = [(id, label, boost, tensor CxHxW float array), ...] in the
    index format polegrad::imagedb::load reads; returns the index path."""
    os.makedirs(directory, exist_ok=True)
    lines = []
    for eid, label, boost, tensor in entries:
        t = np.ascontiguousarray(tensor, dtype="<f4")
        if t.ndim != 3:
            raise ValueError("tensor must be C x H x W")
        name = f"{eid}.bin"
        with open(os.path.join(directory, name), "wb") as f:
            f.write(np.asarray(t.shape, dtype="<u4").tobytes())
            f.write(t.tobytes())
        lines.append(f"{eid},{label},{boost},{name}")
    index = os.path.join(directory, "index.csv")
    with open(index, "w") as f:
        f.write("\n".join(lines) + "\n")
    return index


class Parallel:
    """polegrad::Parallel — NCCL data parallelism, one rank per process."""

    @staticmethod
    def unique_id(dtype: str = "f32") -> bytes:
        lib = load(dtype)
        buf = C.create_string_buffer(128)
        _check(lib, lib.pg_parallel_unique_id(buf))
        return buf.raw[:128]

    def __init__(self, net: Net, nranks: int, rank: int, uid: bytes, bucket_bytes: int = 8 << 20):
        self.net = net
        p = C.c_void_p()
        _check(net.lib, net.lib.pg_parallel_create(net.ptr, nranks, rank, C.c_char_p(uid), bucket_bytes,
                                                   C.byref(p)))
        self.ptr = p

    @classmethod
    def host(cls, net: Net, nranks: int, rank: int, transport, bucket_bytes: int = 8 << 20) -> "Parallel":
        """Host-transport replica: `transport(op, array, offset)` combines one bucket
        (a numpy view of the host copy, the net's real type) across ranks in place:
        op 0 = SUM all-reduce, op 1 = broadcast from rank 0 (e.g. over gloo)."""
        self = cls.__new__(cls)
        self.net = net

        def tramp(_user, op, ptr, offset, n):
            try:
                arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float if net.np == np.float32
                                                                  else C.c_double)), shape=(n,))
                transport(op, arr, offset)
                return 0
            except Exception:  # reported to the caller as a failed transport
                import traceback
                traceback.print_exc()
                return 1

        self._tramp = HOST_TRANSPORT(tramp)  # keep alive as long as the Parallel
        p = C.c_void_p()
        _check(net.lib, net.lib.pg_parallel_create_host(net.ptr, nranks, rank, self._tramp, None, bucket_bytes,
                                                        C.byref(p)))
        self.ptr = p
        return self

    def info(self) -> dict:
        """Communicator size / rank as NCCL reports them, buckets, all-reduces issued."""
        n, r, nb, la = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
        _check(self.net.lib, self.net.lib.pg_parallel_info(self.ptr, C.byref(n), C.byref(r), C.byref(nb),
                                                           C.byref(la)))
        return {"nranks": n.value, "rank": r.value, "buckets": nb.value, "launches": la.value}

    def broadcast(self) -> None:
        _check(self.net.lib, self.net.lib.pg_parallel_broadcast(self.ptr))

    def close(self) -> None:
        if getattr(self, "ptr", None):
            _check(self.net.lib, self.net.lib.pg_parallel_free(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
