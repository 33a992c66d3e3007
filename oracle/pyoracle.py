"""ORACLE — test infrastructure only.

Python driver of oracle/_ref/liboracle_{f64,f32}.so: the UNMODIFIED reference
core (/root/reference/proj/core/src, compiled by oracle/Makefile) plus the
reference-style CPU extension layers in oracle/ext/.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg may use it, and only as
the checker / baseline — never as the product path.

Two net kinds:
  RefNet  — polegrad::Net built by the reference's own prototxt parser (MLPs);
  ExtNet  — the extension net for Convolution / Pooling / SoftmaxWithLoss nets,
            fed a layer list derived from the same prototxt by `to_spec`.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from typing import Dict, List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REFERENCE_LAYER_TYPES = {"InnerProduct", "ReLU", "Sigmoid", "Softmax", "MemoryData", "MemoryLoss"}

_libs: Dict[str, C.CDLL] = {}


def lib_path(dtype: str) -> str:
    return os.path.join(REF_DIR, f"liboracle_{dtype}.so")


def available(dtype: str = "f64") -> bool:
    return os.path.exists(lib_path(dtype))


def load(dtype: str = "f64") -> C.CDLL:
    if dtype not in _libs:
        lib = C.CDLL(lib_path(dtype))
        vp, i, u64, d, cp = C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_char_p
        pd = C.POINTER(C.c_double)
        sig = {
            "orc_last_error": ([], cp), "orc_real_size": ([], i),
            "orc_refnet_create": ([cp, u64, C.POINTER(vp)], i),
            "orc_extnet_create": ([cp, u64, i, C.POINTER(vp)], i), "orc_net_free": ([vp], None),
            "orc_set_batch": ([vp, pd, pd], i), "orc_forward": ([vp, pd], i), "orc_backward": ([vp], i),
            "orc_backward_from": ([vp, cp], i), "orc_blob_shape": ([vp, cp, C.POINTER(i)], i),
            "orc_blob_get": ([vp, cp, i, pd], i), "orc_blob_set": ([vp, cp, i, pd], i),
            "orc_param_count": ([vp], i), "orc_param_info": ([vp, i, cp, i, C.POINTER(i)], i),
            "orc_param_get": ([vp, i, i, pd], i), "orc_param_set": ([vp, i, i, pd], i),
            "orc_snapshot": ([vp, vp, u64, C.POINTER(u64)], i), "orc_restore": ([vp, vp, u64], i),
            "orc_pool_mask": ([vp, cp, C.POINTER(C.c_int), u64], i),
            "orc_set_pool_mask": ([vp, cp, C.POINTER(C.c_int), u64], i),
            "orc_solver_create": ([vp, i, d, d, d, d, d, C.POINTER(vp)], i),
            "orc_solver_apply": ([vp, vp], i), "orc_solver_free": ([vp], None),
            "orc_gemm": ([i, i, i, i, i, d, pd, pd, d, pd], i), "orc_xent_grad": ([pd, pd, i, pd], i),
            "orc_prototxt_roundtrip": ([cp, cp, u64, C.POINTER(u64)], i),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes, fn.restype = args, res
        _libs[dtype] = lib
    return _libs[dtype]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


def _check(lib, st):
    if st != 0:
        raise OracleError(st, lib.orc_last_error().decode(errors="replace"))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ---- minimal protobuf-text reader for building ExtNet layer lists ------------------
_TOKEN = re.compile(r'\s*(?:#[^\n]*\n?|("(?:[^"\\]|\\.)*")|([{}:])|([A-Za-z_][A-Za-z0-9_]*)|([-+.0-9][-+.0-9eExa-fA-F]*))')


def parse_blocks(text: str) -> list:
    """Parse prototxt into nested [(key, value-or-list)] (test helper)."""
    toks: List[str] = []
    pos = 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if not m or m.end() == pos:
            if text[pos:].strip() == "":
                break
            raise ValueError(f"cannot tokenize at {text[pos:pos + 20]!r}")
        pos = m.end()
        tok = next((g for g in m.groups() if g is not None), None)
        if tok is not None:
            toks.append(tok)
    it = iter(toks)

    def block(end_on_brace: bool) -> list:
        out = []
        for tok in it:
            if tok == "}":
                return out
            key = tok
            nxt = next(it)
            if nxt == ":":
                nxt = next(it)
            if nxt == "{":
                out.append((key, block(True)))
            else:
                out.append((key, nxt[1:-1] if nxt.startswith('"') else nxt))
        return out

    return block(False)


def _get(block: list, key: str, default=None):
    for k, v in block:
        if k == key:
            return v
    return default


def _all(block: list, key: str) -> list:
    return [v for k, v in block if k == key]


def to_spec(text: str) -> Tuple[str, Dict]:
    """prototxt -> oracle layer-list spec (type|name|bottoms|tops|k=v;...)."""
    lines = []
    info: Dict = {"data": None, "loss": None}
    for key, layer in parse_blocks(text):
        if key != "layer":
            continue
        t, name = _get(layer, "type"), _get(layer, "name")
        bottoms, tops = _all(layer, "bottom"), _all(layer, "top")
        p: Dict[str, float] = {}
        if t == "InnerProduct":
            p["num_output"] = float(_get(_get(layer, "inner_product_param", []), "num_output"))
        elif t == "MemoryData":
            md = _get(layer, "memory_data_param", [])
            for f in ("batch_size", "channels", "height", "width"):
                p[f] = float(_get(md, f))
            info["data"] = (name, tops, [int(p[f]) for f in ("batch_size", "channels", "height", "width")])
        elif t == "Convolution":
            cp = _get(layer, "convolution_param", [])
            p["num_output"] = float(_get(cp, "num_output"))
            ks = _all(cp, "kernel_size")
            if ks:
                p["kernel_h"], p["kernel_w"] = float(ks[0]), float(ks[-1])
            for f in ("kernel_h", "kernel_w", "stride_h", "stride_w", "pad_h", "pad_w", "dilation", "group"):
                if _get(cp, f) is not None:
                    p[f] = float(_get(cp, f))
            for f, (fh, fw) in (("stride", ("stride_h", "stride_w")), ("pad", ("pad_h", "pad_w"))):
                vs = _all(cp, f)
                if vs:
                    p[fh], p[fw] = float(vs[0]), float(vs[-1])
            if _get(cp, "bias_term") is not None:
                p["bias_term"] = 1.0 if _get(cp, "bias_term") in ("true", "1") else 0.0
        elif t == "Pooling":
            pp = _get(layer, "pooling_param", [])
            p["pool"] = 0.0 if _get(pp, "pool", "MAX") in ("MAX", "0") else 1.0
            for f in ("kernel_size", "stride", "pad", "kernel_h", "kernel_w", "stride_h", "stride_w", "pad_h",
                      "pad_w"):
                if _get(pp, f) is not None:
                    p[f] = float(_get(pp, f))
            if _get(pp, "global_pooling") in ("true", "1"):
                p["global_pooling"] = 1.0
        elif t == "SoftmaxWithLoss":
            lp = _get(layer, "loss_param", [])
            if _get(lp, "normalize") in ("false", "0"):
                p["normalize"] = 0.0
            info["loss"] = tops[0] if tops else None
        elif t == "LRN":
            lp = _get(layer, "lrn_param", [])
            for f in ("local_size", "alpha", "beta", "k"):
                if _get(lp, f) is not None:
                    p[f] = float(_get(lp, f))
            if _get(lp, "norm_region") not in (None, "ACROSS_CHANNELS", "0"):
                p["norm_region"] = 1.0
        elif t == "Dropout":
            dp = _get(layer, "dropout_param", [])
            if _get(dp, "dropout_ratio") is not None:
                p["dropout_ratio"] = float(_get(dp, "dropout_ratio"))
        elif t == "BatchNorm":
            bp = _get(layer, "batch_norm_param", [])
            if _get(bp, "eps") is not None:
                p["eps"] = float(_get(bp, "eps"))
            if _get(bp, "use_global_stats") in ("true", "1"):
                p["use_global_stats"] = 1.0
        elif t == "Scale":
            sp = _get(layer, "scale_param", [])
            p["bias_term"] = 1.0 if _get(sp, "bias_term") in ("true", "1") else 0.0
        elif t == "Eltwise":
            ep = _get(layer, "eltwise_param", [])
            p["operation"] = {"PROD": 0.0, "SUM": 1.0, "MAX": 2.0}.get(_get(ep, "operation", "SUM"), -1.0)
            for i, c in enumerate(_all(ep, "coeff")):
                p[f"coeff{i}"] = float(c)
        kv =";".join(f"{k}={v!r}" for k, v in p.items())
        lines.append(f"{t}|{name}|{','.join(bottoms)}|{','.join(tops)}|{kv}")
    return "\n".join(lines) + "\n", info


def is_reference_net(text: str) -> bool:
    layers = [l for k, l in parse_blocks(text) if k == "layer"]
    return all(_get(l, "type") in REFERENCE_LAYER_TYPES for l in layers) and all(
        len(_all(l, "top")) <= 1 for l in layers if _get(l, "type") == "MemoryData")


class OracleNet:
    """CPU oracle net.  `reference=None` picks RefNet when the model only uses
    reference layer types, ExtNet otherwise."""

    def __init__(self, prototxt: str, seed: int = 1, dtype: str = "f64", reference: Optional[bool] = None,
                 compat: bool = False):
        self.lib = load(dtype)
        self.dtype = dtype
        p = C.c_void_p()
        use_ref = is_reference_net(prototxt) if reference is None else reference
        self.kind = "reference" if use_ref else "extension"
        if use_ref:
            _check(self.lib, self.lib.orc_refnet_create(prototxt.encode(), seed, C.byref(p)))
        else:
            spec, _ = to_spec(prototxt)
            _check(self.lib, self.lib.orc_extnet_create(spec.encode(), seed, int(compat), C.byref(p)))
        self.ptr = p

    def __del__(self):
        if getattr(self, "ptr", None):
            self.lib.orc_net_free(self.ptr)
            self.ptr = None

    def set_batch(self, data: np.ndarray, labels: Optional[np.ndarray] = None) -> None:
        d = np.ascontiguousarray(data, np.float64).ravel()
        l = None if labels is None else np.ascontiguousarray(labels, np.float64).ravel()
        _check(self.lib, self.lib.orc_set_batch(self.ptr, _dp(d), None if l is None else _dp(l)))

    def forward(self) -> float:
        v = C.c_double()
        _check(self.lib, self.lib.orc_forward(self.ptr, C.byref(v)))
        return v.value

    def backward(self) -> None:
        _check(self.lib, self.lib.orc_backward(self.ptr))

    def backward_from(self, blob: str) -> None:
        _check(self.lib, self.lib.orc_backward_from(self.ptr, blob.encode()))

    def blob_shape(self, name: str):
        s = (C.c_int * 4)()
        _check(self.lib, self.lib.orc_blob_shape(self.ptr, name.encode(), s))
        return tuple(s)

    def blob(self, name: str, diff: bool = False) -> np.ndarray:
        out = np.empty(self.blob_shape(name), np.float64)
        _check(self.lib, self.lib.orc_blob_get(self.ptr, name.encode(), int(diff), _dp(out)))
        return out

    def set_blob(self, name: str, values: np.ndarray, diff: bool = False) -> None:
        v = np.ascontiguousarray(values, np.float64).reshape(self.blob_shape(name))
        _check(self.lib, self.lib.orc_blob_set(self.ptr, name.encode(), int(diff), _dp(v)))

    def param_info(self):
        out = []
        buf = C.create_string_buffer(256)
        for i in range(self.lib.orc_param_count(self.ptr)):
            s = (C.c_int * 4)()
            _check(self.lib, self.lib.orc_param_info(self.ptr, i, buf, 256, s))
            out.append((buf.value.decode(), tuple(s)))
        return out

    def param(self, i: int, diff: bool = False) -> np.ndarray:
        out = np.empty(self.param_info()[i][1], np.float64)
        _check(self.lib, self.lib.orc_param_get(self.ptr, i, int(diff), _dp(out)))
        return out

    def set_param(self, i: int, values: np.ndarray, diff: bool = False) -> None:
        v = np.ascontiguousarray(values, np.float64).reshape(self.param_info()[i][1])
        _check(self.lib, self.lib.orc_param_set(self.ptr, i, int(diff), _dp(v)))

    def snapshot(self) -> bytes:
        n = C.c_uint64()
        _check(self.lib, self.lib.orc_snapshot(self.ptr, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _check(self.lib, self.lib.orc_snapshot(self.ptr, buf, n.value, C.byref(n)))
        return bytes(buf)

    def restore(self, blob: bytes) -> None:
        b = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _check(self.lib, self.lib.orc_restore(self.ptr, b, len(blob)))

    def pool_mask(self, layer: str, n: int) -> np.ndarray:
        out = np.empty(n, np.int32)
        _check(self.lib, self.lib.orc_pool_mask(self.ptr, layer.encode(), out.ctypes.data_as(C.POINTER(C.c_int)), n))
        return out

    def set_pool_mask(self, layer: str, mask: np.ndarray) -> None:
        m = np.ascontiguousarray(mask, np.int32)
        _check(self.lib, self.lib.orc_set_pool_mask(self.ptr, layer.encode(), m.ctypes.data_as(C.POINTER(C.c_int)),
                                                    m.size))


def layer_tops(text: str):
    """(layer name, type, tops) in definition order (test helper)."""
    return [(_get(l, "name"), _get(l, "type"), _all(l, "top")) for k, l in parse_blocks(text) if k == "layer"]


class OracleSolver:
    def __init__(self, net: OracleNet, method: str = "sgd", lr: float = 1e-3, momentum: float = 0.0,
                 weight_decay: float = 0.0, rms_decay: float = 0.99, epsilon: float = 1e-8):
        self.net = net
        self.lib = net.lib
        p = C.c_void_p()
        _check(self.lib, self.lib.orc_solver_create(net.ptr, 1 if method == "rmsprop" else 0, lr, momentum,
                                                    weight_decay, rms_decay, epsilon, C.byref(p)))
        self.ptr = p

    def apply(self) -> None:
        _check(self.lib, self.lib.orc_solver_apply(self.ptr, self.net.ptr))

    def __del__(self):
        if getattr(self, "ptr", None):
            self.lib.orc_solver_free(self.ptr)
            self.ptr = None


def reference_gemm(ta, tb, m, n, k, alpha, A, B, beta, Cm, dtype="f64") -> np.ndarray:
    """kernels::gemm of the unmodified reference (backend.cpp:169-197)."""
    lib = load(dtype)
    a = np.ascontiguousarray(A, np.float64).ravel()
    b = np.ascontiguousarray(B, np.float64).ravel()
    c = np.ascontiguousarray(Cm, np.float64).ravel().copy()
    _check(lib, lib.orc_gemm(int(ta), int(tb), m, n, k, alpha, _dp(a), _dp(b), beta, _dp(c)))
    return c


def reference_prototxt_roundtrip(text: str) -> str:
    lib = load("f64")
    n = C.c_uint64()
    _check(lib, lib.orc_prototxt_roundtrip(text.encode(), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib, lib.orc_prototxt_roundtrip(text.encode(), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()
