"""Host arithmetic of the layout's schedules behind the C ABI (runs without a GPU): the packing
groups (dgnn_packing_groups, the analogue of P:439's "C - 4N" sizing) and the assembler's runs
(dgnn_assembly_runs) against a plain transcription of their definitions, on random offsets incl.
empty batches, single huge batches and tiny budgets."""
import numpy as np
import pytest

from paper_2405_05231_b200 import _abi as A


def _groups_ref(po, rb, group_size, budget):
    out, g0, nb = [], 0, len(po) - 1
    while g0 < nb:
        g1 = g0 + 1
        while g1 < nb and (group_size <= 0 or g1 - g0 < group_size) and \
                (po[g1 + 1] - po[g0]) * rb + 4096 * (g1 + 1 - g0) <= budget:
            g1 += 1
        out.append((g0, g1))
        g0 = g1
    return out


def _runs_ref(no, max_rows, max_batches):
    out, b0, nb = [], 0, len(no) - 1
    while b0 < nb:
        b1 = int(np.searchsorted(no, no[b0] + max_rows, side="right")) - 1
        b1 = min(max(b1, b0 + 1), b0 + max_batches, nb)
        out.append((b0, b1))
        b0 = b1
    return out


@pytest.mark.parametrize("trial", range(40))
def test_packing_groups_and_runs_match_their_definitions(trial):
    rng = np.random.default_rng(trial)
    nb = int(rng.integers(0, 400))
    sizes = rng.integers(0, 5000, nb) * (rng.random(nb) < 0.9)  # some empty batches
    if nb and trial % 7 == 0:
        sizes[rng.integers(0, nb)] = 10_000_000  # one batch above any budget
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    rb = int(rng.choice([4, 400, 512, 4096]))
    budget = int(rng.choice([1, 4096, 1 << 20, 64 << 20, 4 << 30]))
    gs = int(rng.choice([0, 1, 3, 64]))
    assert A.dgnn_packing_groups(off, rb, gs, budget) == _groups_ref(off, rb, gs, budget)
    max_rows = int(rng.choice([1, 1000, 100_000, 1 << 30]))
    mb = int(rng.choice([1, 7, 1024]))
    assert A.dgnn_assembly_runs(off, max_rows, mb) == _runs_ref(off, max_rows, mb)


def test_bad_arguments():
    with pytest.raises(A.DgnnError):
        A.dgnn_assembly_runs(np.array([0, 5], np.int64), 0)


def _tables_ref(no, cst, crows, drows, sec, chunk_bytes, rb, runs):
    nb = len(no) - 1
    rows_pre = np.concatenate([[0], np.cumsum(crows)])
    tabs, spans = [], []
    for b0, b1 in runs:
        c_lo = int(cst[b0])
        c_hi = int(cst[b1]) if b1 < nb else int(chunk_bytes)
        chunk_off = np.concatenate([cst[b0:b1] - c_lo, [c_hi - c_lo]])
        if drows is None:
            tabs.append(np.concatenate([no[b0:b1 + 1] - no[b0], chunk_off, rows_pre[b0:b1 + 1] - rows_pre[b0]] +
                                       ([sec[b0:b1] - c_lo] if sec is not None else [])))
        else:
            dpre = np.concatenate([[0], np.cumsum(drows[b0:b1])])
            tabs.append(np.concatenate([no[b0:b1 + 1] - no[b0], dpre * rb, dpre, chunk_off]))
        spans.append((int(no[b0]), int(no[b1]), c_lo, c_hi))
    flat = np.concatenate(tabs).astype(np.int64) if tabs else np.zeros(0, np.int64)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in tabs])]).astype(np.int64)
    return flat, offs, spans


@pytest.mark.parametrize("trial", range(30))
def test_assembly_tables_match_their_definition(trial):
    rng = np.random.default_rng(1000 + trial)
    nb = int(rng.integers(1, 300))
    no = np.concatenate([[0], np.cumsum(rng.integers(1, 5000, nb))]).astype(np.int64)
    rb = int(rng.choice([400, 512, 4096]))
    crows = rng.integers(0, 3000, nb).astype(np.int64)
    cst = np.concatenate([[0], np.cumsum((crows * rb + 4095) // 4096 * 4096)])[:nb].astype(np.int64) + 4096
    chunk_bytes = int(cst[-1] + ((crows[-1] * rb + 4095) // 4096) * 4096) + 4096
    drows = rng.integers(0, 3000, nb).astype(np.int64) if trial % 3 == 0 else None
    sec = (cst + rng.integers(0, 4096, nb)).astype(np.int64) if (drows is None and trial % 2) else None
    runs = A.dgnn_assembly_runs(no, int(rng.choice([1000, 50_000, 1 << 30])), int(rng.choice([1, 5, 1024])))
    got = A.dgnn_assembly_tables(no, cst, crows, drows, sec, chunk_bytes, rb, runs)
    want = _tables_ref(no, cst, crows, drows, sec, chunk_bytes, rb, runs)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]) and got[2] == want[2]
