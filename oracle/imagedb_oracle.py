"""ORACLE — test infrastructure only (tests/ may import it; the product never does).

Pure-Python restatement of the reference's batch sampling
(/root/reference/proj/core/src/imagedb.cpp:51-85, Dataset::sample + pick) and of
its random source (polegrad::Rng, proj/core/include/polegrad/backend.hpp:31-40:
std::mt19937_64, uniform01 = (next >> 11) * 2^-53).  Pinned two ways:
  * MT19937_64 against the C++ standard's known answer (the 10000th output of a
    default-seeded engine, seed 5489, is 9981545732273789042);
  * the reference's own imagedb_test.cpp, compiled against the b200 library
    (tests/test_cpu_reference_suite.py), checks the library the restatement is
    compared with.
"""
from __future__ import annotations

from typing import Dict, List, Sequence

import numpy as np

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (n 312, m 156, r 31; tempering u 29 / s 17 / t 37 / l 43)."""

    N, M = 312, 156
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF
    MATRIX_A = 0xB5026F5AA96619E9

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self.N
        self.mt[0] = seed & MASK64
        for i in range(1, self.N):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & MASK64
        self.index = self.N

    def _twist(self) -> None:
        mt = self.mt
        for i in range(self.N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % self.N] & self.LOWER)
            y = x >> 1
            if x & 1:
                y ^= self.MATRIX_A
            mt[i] = mt[(i + self.M) % self.N] ^ y
        self.index = 0

    def next_u64(self) -> int:
        if self.index >= self.N:
            self._twist()
        y = self.mt[self.index]
        self.index += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53


def _pick(ids: Sequence[int], boost: Dict[int, float], use_boost: bool, rng: MT19937_64, real) -> int:
    """imagedb.cpp:51-69: uniform index floor(u * n), or the first id whose running
    boost sum (accumulated in `real`) exceeds real(u) * total."""
    if not use_boost:
        return ids[min(int(rng.uniform01() * len(ids)), len(ids) - 1)]
    total = real(0)
    for i in ids:
        total = real(total + real(boost[i]))
    target = real(real(rng.uniform01()) * total)
    run = real(0)
    for i in ids:
        run = real(run + real(boost[i]))
        if target < run:
            return i
    return ids[-1]


def sample_ids(entries: Sequence[tuple], n: int, seed: int, method: str = "uniform", use_boost: bool = False,
               real=np.float32) -> List[int]:
    """n draws of Dataset::sample (imagedb.cpp:71-85) over entries [(id, label, boost), ...]:
    uniform picks among all ids (ascending); label_balanced first picks a label group
    (ascending labels) by floor(u * groups), then an entry in insertion order."""
    rng = MT19937_64(seed)
    boost = {e[0]: e[2] for e in entries}
    all_ids = sorted(boost)
    groups: Dict[int, List[int]] = {}
    for eid, label, _ in entries:
        groups.setdefault(label, []).append(eid)
    labels = sorted(groups)
    out = []
    for _ in range(n):
        if method == "uniform":
            out.append(_pick(all_ids, boost, use_boost, rng, real))
        else:
            g = labels[min(int(rng.uniform01() * len(labels)), len(labels) - 1)]
            out.append(_pick(groups[g], boost, use_boost, rng, real))
    return out
