"""The reference's own unit tests (/root/reference/proj/tests: backend, blob,
layers, net, solver, prototxt, imagedb; 88 cases), compiled unmodified against the
B200 library (oracle/_ref/reftests_b200, built by oracle/Makefile with a
doctest stand-in) and run on the GPU in reference-compat mode.  The prototxt
corpus case reads files under /root/reference, which does not exist on the
GPU box; it runs in the CPU suite instead (test_cpu_reference_suite.py)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "reftests_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="reftests_b200 not built (needs /root/reference at build time)")
def test_reference_unit_suite_on_b200():
    env = dict(os.environ, POLEGRAD_REFERENCE_COMPAT="1")
    args = [BIN]
    if not os.path.isdir("/root/reference/proj/tests/corpus"):
        args.append("-corpus files")
    r = subprocess.run(args, env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stdout
