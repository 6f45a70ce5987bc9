"""Pins for the oracle's RNG and subset draw (readings c5-c7).

* Philox4x32-10 against the Random123 known-answer vectors (published) and
  against NVIDIA's ``curand_Philox4x32_10`` compiled for the host (a library
  routine with its own transcription of the round function).
* Floyd's subset map by exhaustive enumeration: every k-subset of [0, d) is
  produced equally often over all draw tuples (Bentley & Floyd 1987).
* The key packing by goldens computed independently in SURVEY.md 8(c).
"""
import itertools
import math
import os
import subprocess
import tempfile
from collections import Counter

import numpy as np
import pytest

import oracle
from conftest import golden_lines


def test_philox_random123_kat():
    n = 0
    for line in golden_lines("philox4x32_10_kat.txt"):
        lhs, rhs = line.split("->")
        w = [int(x, 16) for x in lhs.split()]
        expect = tuple(int(x, 16) for x in rhs.split())
        assert oracle.philox4x32_10(w[:4], w[4:6]) == expect
        n += 1
    assert n == 3


_CURAND_SRC = r"""
#include <cstdio>
#include <cstdint>
#include <vector_types.h>
#define QUALIFIERS static inline
#define __forceinline__
#include <curand_philox4x32_x.h>
int main() {
    unsigned c0, c1, c2, c3, k0, k1;
    while (scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
        uint4 c = {c0, c1, c2, c3};
        uint2 k = {k0, k1};
        uint4 o = curand_Philox4x32_10(c, k);
        printf("%08x %08x %08x %08x\n", o.x, o.y, o.z, o.w);
    }
    return 0;
}
"""


def _curand_host_binary():
    d = tempfile.mkdtemp(prefix="curand_host_")
    src = os.path.join(d, "p.cpp")
    exe = os.path.join(d, "p")
    with open(src, "w") as f:
        f.write(_CURAND_SRC)
    try:
        subprocess.check_call(["g++", "-O1", "-I/usr/local/cuda/include", "-o", exe, src],
                              stderr=subprocess.DEVNULL)
    except Exception:
        return None
    return exe


def test_philox_matches_curand_host_build():
    exe = _curand_host_binary()
    if exe is None:
        pytest.skip("curand header not host-compilable here")
    rng = np.random.default_rng(123)
    words = rng.integers(0, 2**32, size=(500, 6), dtype=np.uint64)
    words[0] = 0
    words[1] = 2**32 - 1
    inp = "\n".join(" ".join(f"{int(x):x}" for x in row) for row in words) + "\n"
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for row, line in zip(words, out):
        expect = tuple(int(x, 16) for x in line.split())
        assert oracle.philox4x32_10(row[:4], row[4:6]) == expect


def test_draw_and_floyd_keying_goldens():
    seen = 0
    for line in golden_lines("rng_keying.txt"):
        lhs, rhs = line.split("->")
        f = lhs.split()
        args = [int(x, 0) for x in f[1:]]
        if f[0] == "draw64":
            assert oracle.draw64(*args) == int(rhs.strip(), 16)
        else:
            d, k, seed, v, bid, h = args
            assert oracle.floyd(d, k, seed, v, bid, h) == [int(x) for x in rhs.split()]
        seen += 1
    assert seen == 6


def test_draw64_is_philox_of_packed_counter():
    # draw64 must be exactly Philox of the packed counter (reading c5), checked word by word
    seed, v, bid, h, s = 0x0123456789ABCDEF, 777, (5 << 32) | 9, 3, 41
    o = oracle.philox4x32_10([v, bid & 0xFFFFFFFF, (h << 16) | s, bid >> 32],
                             [seed & 0xFFFFFFFF, seed >> 32])
    assert oracle.draw64(seed, v, bid, h, s) == (o[1] << 32) | o[0]


@pytest.mark.parametrize("d", range(1, 8))
def test_floyd_exhaustive_uniform(d):
    """All prod(d-k+s+1) draw tuples give every k-subset equally often."""
    for k in range(1, d + 1):
        ranges = [range(d - k + s + 1) for s in range(k)]
        hist = Counter()
        total = 0
        for t in itertools.product(*ranges):
            sub = oracle.floyd_core(d, k, list(t))
            assert len(set(sub)) == k and sub == sorted(sub) and all(0 <= x < d for x in sub)
            hist[tuple(sub)] += 1
            total += 1
        assert len(hist) == math.comb(d, k)
        assert set(hist.values()) == {total // math.comb(d, k)}


def test_floyd_full_take_is_identity():
    assert oracle.floyd(5, 5, 9, 1, 2, 0) == [0, 1, 2, 3, 4]
    assert oracle.floyd(1, 1, 9, 1, 2, 0) == [0]
    assert oracle.floyd(9, 0, 9, 1, 2, 0) == []


def test_floyd_inclusion_frequency_chi2():
    """Each position appears with probability k/d over independent bids."""
    d, k, trials = 40, 7, 4000
    hits = np.zeros(d)
    for bid in range(trials):
        for p in oracle.floyd(d, k, 0xABCDEF, 31337, bid, 1):
            hits[p] += 1
    expect = trials * k / d
    chi2 = float(((hits - expect) ** 2 / expect).sum())
    # 39 dof: P(chi2 > 80) ~ 1e-4
    assert chi2 < 80, chi2


def test_floyd_large_degree_in_range():
    d = 10**9
    sub = oracle.floyd(d, 20, 1, 2, 3, 1)
    assert len(set(sub)) == 20 and sub == sorted(sub) and sub[-1] < d
