"""Pins for the oracle's packing page accounting (Sec. 5.2, Fig. 6; NEXT #3).

* Fig. 6 (golden fig6_packing.txt): individual packing reads 4 pages, batched 2.
* Brute force with Python sets on random fixtures: individual = per batch, per needed row, the
  pages the row spans; batched = whole partitions holding a needed row, clipped at the file end.
* Invariants: batched <= the file's pages; a partition covering the whole file reads it once.
"""
import numpy as np
import pytest

import oracle
from conftest import golden_lines

PAGE = 4096


def test_fig6():
    g = {"batch": []}
    for line in golden_lines("fig6_packing.txt"):
        k, *rest = line.split()
        if k == "batch":
            g["batch"].append([int(x) for x in rest])
        else:
            g[k] = int(rest[0])
    ind, bat = oracle.pack_pages(g["batch"], g["num_nodes"], g["row_bytes"], g["partition_rows"])
    assert (ind, bat) == (g["individual_pages"], g["batched_pages"])


def bf(plists, N, rb, part):
    ind = 0
    parts = set()
    for p in plists:
        for v in p:
            # brute force over the row's bytes (a 64-byte stride cannot skip a 4096-byte page)
            ind += len({o // PAGE for o in range(v * rb, (v + 1) * rb, 64)} | {((v + 1) * rb - 1) // PAGE})
            parts.add(v // part)
    file_pages = -(-N * rb // PAGE)
    bat = sum(min((q + 1) * part * rb // PAGE, file_pages) - q * part * rb // PAGE for q in parts)
    return ind, bat


@pytest.mark.parametrize("trial", range(20))
def test_brute_force(trial):
    rng = np.random.default_rng(trial)
    N = int(rng.integers(1, 3000))
    rb = int(rng.choice([400, 512, 1024, 4096, 12288, 100]))
    # partitions must not split a page: part_rows * rb a multiple of 4096
    base = PAGE // np.gcd(PAGE, rb)
    part = int(base * rng.integers(1, 40))
    pl = [rng.choice(N, size=int(rng.integers(0, min(N, 60) + 1)), replace=False) for _ in range(int(rng.integers(0, 8)))]
    ind, bat = oracle.pack_pages(pl, N, rb, part)
    assert (ind, bat) == bf(pl, N, rb, part)
    assert bat <= -(-N * rb // PAGE)
    if any(len(p) for p in pl):
        assert oracle.pack_pages(pl, N, rb, base * (-(-N // base)))[1] == -(-N * rb // PAGE)


def test_rejects_page_splitting_partitions():
    with pytest.raises(oracle.OracleError):
        oracle.pack_pages([[0]], 10, 512, 3)
