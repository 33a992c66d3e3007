"""Solver-state checkpoint format ("MCSS") through the C-ABI
without a GPU: restoring before the first update is host-only (the history is
installed on the next apply), so the format, the round trip and the error
taxonomy are checked here; tests/test_gpu_checkpoint.py resumes training."""
import ctypes as C
import struct

import pytest

from paper_1810_02272_b200 import polegrad

FORMAT_ERROR, INVALID_STATE = 6, 8


def mcss(method=0, iters=7, hist=(0.5, -1.25, 3.0), magic=b"MCSS", version=1):
    return magic + struct.pack("<IIQQ", version, method, iters, len(hist)) + struct.pack(f"<{len(hist)}d", *hist)


@pytest.fixture(params=["f32", "f64"])
def solver(request):
    lib = polegrad.load(request.param)
    p = C.c_void_p()
    assert lib.pg_solver_create(0, 0.01, 0.9, 0.0, 0.99, 1e-8, C.byref(p)) == 0
    yield lib, p
    lib.pg_solver_free(p)


def restore(lib, p, blob):
    b = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
    return lib.pg_solver_restore(p, b, len(blob))


def snapshot(lib, p):
    n = C.c_uint64()
    assert lib.pg_solver_snapshot(p, None, 0, C.byref(n)) == 0
    buf = (C.c_uint8 * n.value)()
    assert lib.pg_solver_snapshot(p, buf, n.value, C.byref(n)) == 0
    return bytes(buf)


def test_fresh_solver_snapshot_is_empty(solver):
    lib, p = solver
    assert snapshot(lib, p) == mcss(iters=0, hist=())


def test_restore_before_first_update_round_trips(solver):
    lib, p = solver
    blob = mcss()  # values exactly representable in f32
    assert restore(lib, p, blob) == 0
    assert snapshot(lib, p) == blob
    it = C.c_uint64()
    assert lib.pg_solver_iterations(p, C.byref(it)) == 0 and it.value == 7


@pytest.mark.parametrize("bad,status,msg", [
    (mcss(magic=b"MCWT"), FORMAT_ERROR, "bad magic"),
    (mcss(version=2), FORMAT_ERROR, "unsupported version"),
    (mcss()[:-3], FORMAT_ERROR, "truncated"),
    (mcss() + b"\0", FORMAT_ERROR, "trailing"),
    (mcss(method=1), INVALID_STATE, "different update rule"),
    (b"MC", FORMAT_ERROR, "truncated"),
])
def test_restore_errors(solver, bad, status, msg):
    lib, p = solver
    assert restore(lib, p, bad) == status
    assert msg in lib.pg_last_error().decode()
