"""imagedb sampling on CPU: the library's Dataset::sample
sequence (through the C API) against the pure-Python restatement of the reference
(oracle/imagedb_oracle.py, reference proj/core/src/imagedb.cpp:51-85), plus the
index-file loader's error lines.  The reference's own imagedb_test.cpp runs
against the same library in test_cpu_reference_suite.py."""
import os

import numpy as np
import pytest

from oracle.imagedb_oracle import MT19937_64, sample_ids
from paper_1810_02272_b200 import polegrad as pg


def test_mt19937_64_known_answer():
    # C++ standard [rand.predef]: 10000th output of a default-constructed mt19937_64
    rng = MT19937_64()
    for _ in range(9999):
        rng.next_u64()
    assert rng.next_u64() == 9981545732273789042


def make_entries(n=23, labels=5, seed=0):
    rs = np.random.RandomState(seed)
    out = []
    for k in range(n):
        eid = int(rs.randint(0, 10 ** 6)) * 7 + k  # unique, not insertion-sorted
        out.append((eid, int(rs.randint(0, labels)), float(1 + rs.randint(0, 4) * 0.75), rs.randn(2, 3, 3)))
    return out


@pytest.mark.parametrize("method", ["uniform", "label_balanced"])
@pytest.mark.parametrize("use_boost", [False, True])
def test_sample_sequence_matches_restatement(tmp_path, method, use_boost):
    entries = make_entries()
    db = pg.ImageDB(pg.write_imagedb(str(tmp_path), entries))
    assert len(db) == len(entries)
    got = db.sample(pg.Rng(1234), 400, method, use_boost)
    want = sample_ids([e[:3] for e in entries], 400, 1234, method, use_boost)
    assert got.tolist() == want


def test_set_boost_changes_weighted_draws(tmp_path):
    entries = make_entries(n=8, labels=2, seed=3)
    db = pg.ImageDB(pg.write_imagedb(str(tmp_path), entries))
    db.set_boost(entries[2][0], 40.0)
    moved = [(e[0], e[1], 40.0 if i == 2 else e[2]) for i, e in enumerate(entries)]
    got = db.sample(pg.Rng(9), 200, "uniform", True)
    assert got.tolist() == sample_ids(moved, 200, 9, "uniform", True)
    with pytest.raises(pg.PolegradError):
        db.set_boost(entries[0][0], 0.5)
    with pytest.raises(pg.PolegradError):
        db.set_boost(-1, 2.0)


@pytest.mark.parametrize("line,expect", [
    ("1,0,1.0", "line 2"),                # too few fields
    ("x,0,1.0,a.bin", "line 2"),          # id not a number
    ("2,0,0.5,a.bin", "boost must be >= 1"),
    ("3,0,1.0,missing.bin", "line 2"),
])
def test_load_errors_carry_line(tmp_path, line, expect):
    idx = pg.write_imagedb(str(tmp_path), [(0, 0, 1.0, np.zeros((1, 1, 1)))])
    with open(idx, "a") as f:
        f.write(line + "\n")
    with pytest.raises(pg.PolegradError) as e:
        pg.ImageDB(idx)
    assert e.value.args[0] == 10 or "LOAD" in str(e.value)
    assert expect in str(e.value)


def test_missing_index(tmp_path):
    with pytest.raises(pg.PolegradError) as e:
        pg.ImageDB(os.path.join(str(tmp_path), "nope.csv"))
    assert "line 0" in str(e.value)
