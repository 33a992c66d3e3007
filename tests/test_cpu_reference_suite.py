"""Oracle pinning and boundary-input parity on the CPU (no GPU needed).

* reftests_ref  — the reference's own unit tests (backend, blob, layers, net,
  solver, prototxt, trainer, cartpole, imagedb: 111 cases / ~7.6k assertions, incl.
  the gemm / softmax / FD known-answer tests of SURVEY §8(c) and the episode
  finite-difference check trainer_test.cpp:242-290) compiled against the
  UNMODIFIED reference core: the oracle is the reference, and this proves the
  build is faithful.
* acceptance_ref — the reference's acceptance program (acceptance.cpp, included
  unmodified by oracle/acceptance_driver.cpp), criteria 1-7: the paper's Figure-6
  and Figure-9 worked-example tables, the 20-seed finite-difference checks,
  cart-pole learning, model round trips, sampler statistics, dynamics.
* reftests_b200 prototxt cases — the same unmodified prototxt tests compiled
  against the B200 library's parser/printer (host code, runs without a GPU),
  in reference-compat mode; in extended mode exactly one assertion (that
  "Convolution" is an unknown type) flips, by design.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "reftests_ref")
B200_BIN = os.path.join(ROOT, "oracle", "_ref", "reftests_b200")
HAVE_REF = os.path.isdir("/root/reference/proj")


def _run(args, env=None):
    r = subprocess.run(args, capture_output=True, text=True, timeout=600, env=env)
    return r.returncode, r.stdout + r.stderr


@pytest.mark.skipif(not (os.path.exists(REF_BIN) and HAVE_REF), reason="oracle reference suite not built here")
def test_reference_suite_passes_on_reference_core():
    rc, out = _run([REF_BIN])
    assert rc == 0, out[-3000:]
    assert "111 passed | 0 failed" in out


ACC_REF = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")


@pytest.mark.skipif(not (os.path.exists(ACC_REF) and HAVE_REF), reason="acceptance_ref not built here")
def test_reference_acceptance_criteria_pass_on_reference_core():
    rc, out = _run([ACC_REF, "1", "2", "3", "4", "5", "6", "7"])
    assert rc == 0, out[-3000:]
    for i in range(1, 8):
        assert f"PASS {i}/9" in out, out


@pytest.mark.skipif(not (os.path.exists(B200_BIN) and HAVE_REF), reason="reftests_b200 not built here")
def test_reference_prototxt_suite_on_b200_parser():
    env = dict(os.environ, POLEGRAD_REFERENCE_COMPAT="1")
    rc, out = _run([B200_BIN, "prototxt_test"], env)
    assert rc == 0, out[-3000:]
    assert "10 passed | 0 failed" in out


@pytest.mark.skipif(not (os.path.exists(B200_BIN) and HAVE_REF), reason="reftests_b200 not built here")
def test_extended_mode_only_flips_the_convolution_assertion():
    env = {k: v for k, v in os.environ.items() if k != "POLEGRAD_REFERENCE_COMPAT"}
    rc, out = _run([B200_BIN, "prototxt_test"], env)
    assert "9 passed | 1 failed" in out and "| 1 failed" in out, out[-2000:]
    # the one failing case is the reference's "Convolution is unknown" check
    assert "layer validation errors point at the offending line" in out, out[-2000:]


@pytest.mark.skipif(not (os.path.exists(B200_BIN) and HAVE_REF), reason="reftests_b200 not built here")
def test_reference_imagedb_suite_on_b200_library():
    """The reference's imagedb tests (dataset, label-balanced / boosted sampling
    statistics, index + tensor-file loading and its error lines) against the B200
    library's own imagedb (host-only)."""
    rc, out = _run([B200_BIN, "imagedb_test"])
    assert rc == 0, out[-3000:]
    assert "13 passed | 0 failed" in out
