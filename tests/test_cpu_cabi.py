"""The C-ABI boundary without a GPU: both libraries load, export every symbol
their headers declare, fail loudly (NO_DEVICE) instead of falling back, and
the host-only pieces (prototxt boundary, DP bucket planner) behave."""
import os
import re

import pytest

from paper_1810_02272_b200 import cudadnn, polegrad

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header: str, prefix: str):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(" + prefix + r"[a-z0-9_]+)\s*\(", text)))


def test_cudadnn_exports_every_declared_symbol():
    lib = cudadnn.load()
    names = declared("cudadnn.h", "cdnn_")
    assert len(names) >= 60
    assert sorted(cudadnn.EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_polegrad_c_exports_every_declared_symbol(dtype):
    lib = polegrad.load(dtype)
    names = declared("polegrad_c.h", "pg_")
    assert sorted(polegrad.EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n
    assert lib.pg_real_size() == (4 if dtype == "f32" else 8)


def test_no_cpu_fallback_without_device():
    if cudadnn.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(cudadnn.CudnnError) as e:
        cudadnn.Context(0)
    assert e.value.name == "NO_DEVICE"
    with pytest.raises(polegrad.PolegradError):
        polegrad.Net(polegrad.load_model("pg_mlp"), 1, "f32")


def test_status_names():
    lib = cudadnn.load()
    for code, name in cudadnn.STATUS.items():
        assert lib.cdnn_status_name(code).decode() == name


@pytest.mark.parametrize("model", ["pg_mlp", "lenet", "cifar10_quick"])
def test_prototxt_canonical_form_is_idempotent(model):
    text = polegrad.load_model(model)
    once = polegrad.prototxt_roundtrip(text)
    assert polegrad.prototxt_roundtrip(once) == once
    assert "layer {" in once


def test_prototxt_matches_reference_printer():
    pyoracle = pytest.importorskip("oracle.pyoracle")
    if not pyoracle.available("f64"):
        pytest.skip("oracle not built")
    for name in ("pg_mlp",):
        text = polegrad.load_model(name)
        assert polegrad.prototxt_roundtrip(text) == pyoracle.reference_prototxt_roundtrip(text)
    # reference corpus, when present
    corpus = "/root/reference/proj/tests/corpus"
    if os.path.isdir(corpus):
        for f in sorted(os.listdir(corpus)):
            text = open(os.path.join(corpus, f)).read()
            try:
                want = pyoracle.reference_prototxt_roundtrip(text)
            except pyoracle.OracleError:
                continue
            assert polegrad.prototxt_roundtrip(text) == want, f


def test_bucket_planner_tiles_arena_back_to_front():
    # 5 params with 16-element-aligned offsets, buckets of >= 100 elements
    counts = [30, 64, 200, 10, 90]
    offs, o = [], 0
    for c in counts:
        offs.append(o)
        o += (c + 3) // 4 * 4
    of, nb = polegrad.plan_buckets(offs, counts, o, 100)
    # last param (90) + 10 -> bucket 0 closes at param 3; 200 -> bucket 1; 64 + 30 -> bucket 2
    assert nb == 3
    assert of == [2, 2, 1, 0, 0]
    of1, nb1 = polegrad.plan_buckets(offs, counts, o, 1 << 30)
    assert nb1 == 1 and of1 == [0] * 5
