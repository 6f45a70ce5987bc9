"""The staging schedule of the window-ordered host tier (dgnn_host_order_schedule, host code: runs
without a GPU).

A simulation replays the schedule window by window with the assembler's timing -- window w is
prefetched (its copies land) while window w-1 still reads the arena -- and checks that (1) a copy
never overwrites a row that window w-1 or w still reads, (2) after its prefetch every physical row
window w needs is in the arena where window w's map says, (3) the map covers exactly window w's rows,
(4) every (group, run of consecutive windows) crosses PCIe at most once: rows copied <= sum over
groups of size x (number of runs of consecutive set bits in the mask), and at least once per group
a window reads; with room for every row, exactly once (gaps bridged).
"""
import ctypes

import numpy as np
import pytest

from paper_2405_05231_b200 import _abi as A


def _schedule(gs, gm, kh, nwin, capacity):
    L = A.load_library()
    gs = np.ascontiguousarray(gs, np.int64)
    gm = np.ascontiguousarray(gm, np.uint32)
    cap = 4 * max(len(gs), 1) * (nwin + 1) + 16
    co, mo = np.zeros(3 * cap, np.int64), np.zeros(3 * cap, np.int64)
    coff, moff = np.zeros(nwin + 1, np.int64), np.zeros(nwin + 1, np.int64)
    copied = ctypes.c_int64()
    rc = L.dgnn_host_order_schedule(A.P(gs.ctypes.data), A.P(gm.ctypes.data), len(gs), kh, nwin, capacity,
                                    A.P(co.ctypes.data), cap, A.P(coff.ctypes.data), A.P(mo.ctypes.data), cap,
                                    A.P(moff.ctypes.data), ctypes.byref(copied))
    return rc, co, coff, mo, moff, copied.value


def _runs(m, nwin):
    r, prev = 0, False
    for w in range(nwin):
        b = bool((m >> w) & 1)
        r += b and not prev
        prev = b
    return r


@pytest.mark.parametrize("trial", range(25))
def test_schedule_replays_correctly(trial):
    rng = np.random.default_rng(trial)
    nwin = int(rng.integers(1, 12))
    masks = np.unique(rng.integers(0, 1 << nwin, int(rng.integers(1, 60))).astype(np.uint32))
    sizes = rng.integers(1, 50, len(masks))
    gs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    kh = int(sizes.sum())
    phys_mask = np.repeat(masks, sizes)
    win_rows = [int(((phys_mask >> w) & 1).sum()) for w in range(nwin)]
    capacity = 2 * max(win_rows + [1])
    rc, co, coff, mo, moff, copied = _schedule(gs, masks, kh, nwin, capacity)
    assert rc == 0, A.load_library().dgnn_last_error()
    assert copied <= sum(int(s) * _runs(int(m), nwin) for m, s in zip(masks, sizes))
    assert copied >= sum(int(s) for m, s in zip(masks, sizes) if m)
    arena = np.full(capacity, -1, np.int64)  # physical row held by each staging row
    for w in range(nwin):
        reading = set()  # staging rows window w-1 still reads while w's copies land
        if w >= 1:
            m = mo[3 * moff[w - 1]:3 * moff[w]].reshape(-1, 3)
            for lo, hi, st in m:
                reading.update(range(st, st + hi - lo))
        c = co[3 * coff[w]:3 * coff[w + 1]].reshape(-1, 3)
        for lo, hi, st in c:
            for k in range(hi - lo):
                assert st + k not in reading, f"window {w}: copy overwrites a row window {w - 1} reads"
                arena[st + k] = lo + k
        m = mo[3 * moff[w]:3 * moff[w + 1]].reshape(-1, 3)
        assert np.all(np.diff(m[:, 0]) > 0) if len(m) > 1 else True
        covered = []
        for lo, hi, st in m:
            assert np.array_equal(arena[st:st + hi - lo], np.arange(lo, hi)), f"window {w}: stale rows"
            covered += list(range(lo, hi))
        assert sorted(covered) == list(np.nonzero((phys_mask >> w) & 1)[0]), f"window {w}: map != its rows"


def test_consecutive_windows_share_rows():
    """Rows needed by windows 0..3 cross once; rows needed by 0 and 2 (not 1) also cross once (a
    one-window gap is bridged at no extra room)."""
    gs, masks, kh = [0, 10], [0b1111, 0b0101], 15
    rc, co, coff, mo, moff, copied = _schedule(gs, masks, kh, 4, 40)
    assert rc == 0
    assert copied == 10 + 5


def test_gap_bridged_only_when_it_fits():
    """A group read by windows 0 and 3 stays resident through windows 1-2 only if the arena has
    room for it next to the groups of windows 1 and 2 (occupancy at window 2's prefetch: 40 of 40)."""
    gs, masks, kh = [0, 10, 30], [0b1001, 0b0010, 0b0100], 50
    rc, co, coff, mo, moff, copied = _schedule(gs, masks, kh, 4, 40)
    assert rc == 0
    assert copied == 10 * 2 + 20 + 20
    rc, co, coff, mo, moff, copied = _schedule(gs, masks, kh, 4, 50)
    assert rc == 0
    assert copied == 10 + 20 + 20


@pytest.mark.parametrize("trial", range(10))
def test_every_row_once_with_room(trial):
    rng = np.random.default_rng(100 + trial)
    nwin = int(rng.integers(2, 10))
    masks = np.unique(rng.integers(1, 1 << nwin, int(rng.integers(5, 60))).astype(np.uint32))
    sizes = rng.integers(1, 50, len(masks))
    gs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
    kh = int(sizes.sum())
    rc, co, coff, mo, moff, copied = _schedule(gs, masks, kh, nwin, kh)
    assert rc == 0
    assert copied == kh


def test_capacity_too_small_is_an_error():
    rc, *_ = _schedule([0], [0b11], 10, 2, 5)
    assert rc == A.DGNN_EINVAL
