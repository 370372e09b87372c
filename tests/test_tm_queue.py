"""Work distribution of the TMEM blind-rotation engine (csrc/tm_queue.h, the
functions br_fft_tm_kernel itself calls), run on the CPU
through the host emulation library: every (lane, CMux iteration) of a launch
is run exactly once, a slot's chunks are numbered in dependency order (the
kernel waits for chunk k - 1, which must be a smaller unit number for the wait
to terminate), an odd lane of the pair queue is the first unit and runs whole,
batches a little wider than the pipelines run as single-lane chunks, and
narrow batches fall back to the static contiguous split."""
import ctypes

import numpy as np
import pytest

from paper_1906_00148_b200 import build

STATIC, PAIRS, SINGLES = 0, 1, 2


def schedule(total, n, chunk, pipelines):
    L = ctypes.CDLL(build.build_emu())
    L.she_emu_tm_schedule.restype = ctypes.c_uint32
    cap = total * (n // max(1, min(chunk, n)) + 2) + pipelines + 8
    out = np.zeros((cap, 6), np.uint32)
    mode = ctypes.c_int(-1)
    rows = L.she_emu_tm_schedule(total, n, chunk, pipelines, cap,
                                 out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(mode))
    assert rows != 0xFFFFFFFF and rows <= cap
    return out[:rows], mode.value


def coverage(units, total, n):
    cov = np.zeros((total, n), np.int32)
    for base, nsl, i0, i1, _, _ in units:
        assert nsl in (1, 2) and i0 < i1 <= n and base + nsl <= total
        cov[base:base + nsl, i0:i1] += 1
    return cov


def check_queue(units, total, n, chunk, lanes_per_slot):
    """Chunks of a slot in increasing unit order, each continuing where the
    previous one ended; chunk-major over the slots."""
    seen = {}
    for base, nsl, i0, i1, slot, _ in units:
        if nsl != lanes_per_slot:
            continue
        assert base == lanes_per_slot * slot and i0 % chunk == 0 and i1 == min(n, i0 + chunk)
        assert seen.get(slot, 0) == i0
        seen[slot] = i1
    assert all(v == n for v in seen.values())
    k = [i0 // chunk for _, nsl, i0, _, _, _ in units if nsl == lanes_per_slot]
    assert k == sorted(k)
    return len(seen)


@pytest.mark.parametrize("total,n,chunk,pipelines", [
    (4797, 500, 32, 592),     # config 1: odd lane count, ragged last chunk
    (4796, 500, 32, 592),
    (1185, 500, 7, 592),      # just wide enough for the pair queue
    (2343, 500, 499, 592),    # chunks of 499 + 1
    (100, 128, 1, 16), (101, 128, 127, 16), (33, 5, 2, 4), (9, 3, 1, 4),
])
def test_pair_queue_covers_every_iteration_once_in_dependency_order(total, n, chunk, pipelines):
    units, mode = schedule(total, n, chunk, pipelines)
    assert mode == PAIRS
    assert (coverage(units, total, n) == 1).all()
    assert len(units) == (total // 2) * -(-n // chunk) + total % 2
    if total % 2:  # the odd lane: unit 0, all n iterations (the longest unit first)
        assert tuple(units[0][:4]) == (total - 1, 1, 0, n)
        units = units[1:]
    assert check_queue(units, total, n, chunk, 2) == total // 2


@pytest.mark.parametrize("total,n,chunk,pipelines", [
    (593, 500, 32, 592),      # one lane more than the pipelines
    (600, 500, 32, 592),      # a 512-gate rank shard of config 1 (8 ranks)
    (976, 500, 32, 592),      # the widest single-lane queue (1.65 lanes per pipeline)
    (700, 500, 7, 592), (5, 9, 2, 4), (26, 16, 5, 16),
])
def test_single_lane_queue(total, n, chunk, pipelines):
    units, mode = schedule(total, n, chunk, pipelines)
    assert mode == SINGLES
    assert (coverage(units, total, n) == 1).all()
    assert len(units) == total * -(-n // chunk)
    assert check_queue(units, total, n, chunk, 1) == total


@pytest.mark.parametrize("total,n,chunk,pipelines", [
    (0, 500, 32, 592), (1, 500, 32, 592), (46, 500, 32, 592), (591, 500, 32, 592),
    (592, 500, 32, 592),                                               # <= 1 lane per pipeline
    (977, 500, 32, 592), (1184, 500, 32, 592),                         # up to 2: one pair each
    (4797, 500, 500, 592), (4797, 500, 0xFFFFFFFF, 592), (600, 500, 500, 592),  # chunk >= n
    (37, 16, 4, 20), (9, 4, 2, 4 * 3),
])
def test_static_split_covers_every_lane_once(total, n, chunk, pipelines):
    units, mode = schedule(total, n, chunk, pipelines)
    assert mode == STATIC
    assert (coverage(units, total, n) == 1).all() if total else len(units) == 0
    for base, nsl, i0, i1, _, _ in units:
        assert (i0, i1) == (0, n)
    per = np.zeros(pipelines, np.int64)
    last_end = {}
    for base, nsl, _, _, _, gq in units:
        per[gq] += nsl
        assert last_end.get(gq, base) == base  # contiguous, in order
        last_end[gq] = base + nsl
    assert per.max() - per.min() <= 1  # balanced: at most one lane more than any other pipeline
    if total <= pipelines:  # narrow: every lane alone on a pipeline (all four warps on it)
        assert all(nsl == 1 for _, nsl, _, _, _, _ in units)
    # a pipeline runs pairs first and at most one single lane, last
    for gq in set(int(g) for g in units[:, 5]) if len(units) else ():
        mine = [int(nsl) for _, nsl, _, _, _, g in units if g == gq]
        assert mine == sorted(mine, reverse=True) and mine.count(1) <= 1


def test_mode_thresholds():
    """<= 1 lane per pipeline: static; up to 1.65: single-lane chunks; up to 2:
    static pairs; wider: the pair queue."""
    modes = {t: schedule(t, 500, 32, 592)[1] for t in (592, 593, 976, 977, 1184, 1185)}
    assert modes == {592: STATIC, 593: SINGLES, 976: SINGLES, 977: STATIC, 1184: STATIC, 1185: PAIRS}


def wrap_schedule(total, n, pipelines):
    L = ctypes.CDLL(build.build_emu())
    L.she_emu_tm_wrap_schedule.restype = ctypes.c_uint32
    cap = total + 3 * pipelines + 8
    out = np.zeros((cap, 6), np.uint32)
    mode = ctypes.c_int(-1)
    rows = L.she_emu_tm_wrap_schedule(total, n, pipelines, cap, out.ctypes.data_as(ctypes.c_void_p),
                                      ctypes.byref(mode))
    assert rows < 0xFFFFFFF0 and rows <= cap
    return out[:rows], mode.value


@pytest.mark.parametrize("total,n,pipelines,mode", [
    (4797, 500, 592, PAIRS), (4796, 500, 592, PAIRS), (1185, 500, 592, PAIRS), (1186, 500, 592, PAIRS),
    (9548, 500, 592, PAIRS), (131072, 500, 592, PAIRS), (2368, 500, 592, PAIRS),  # 2368 = 4 x 592: no cut at all
    (593, 500, 592, SINGLES), (612, 500, 592, SINGLES), (976, 500, 592, SINGLES),
    (33, 5, 4, PAIRS), (9, 3, 4, PAIRS), (5, 9, 4, SINGLES), (26, 16, 16, SINGLES), (101, 128, 16, PAIRS),
])
def test_wrap_around_schedule(total, n, pipelines, mode):
    """The default distribution of wide batches: every (lane, iteration) once;
    every pipeline the same number of iterations (+- 1); a unit is cut at most
    once; a pipeline runs a first part first and a last part last; and an
    execution that honours the progress words (a part with i0 > 0 waits until
    its slot has published i0) terminates whatever the pipelines' speeds."""
    units, m = wrap_schedule(total, n, pipelines)
    assert m == mode
    assert (coverage(units, total, n) == 1).all()
    lanes_per = 1 if mode == SINGLES else 2
    nunits = total if mode == SINGLES else (total + 1) // 2
    per = np.zeros(pipelines, np.int64)
    parts = {}
    order = {g: [] for g in range(pipelines)}
    for base, nsl, i0, i1, slot, gq in units:
        assert base == lanes_per * slot and slot < nunits
        assert nsl == (lanes_per if base + lanes_per <= total else 1)  # an odd last lane: a unit of one
        per[gq] += i1 - i0
        parts.setdefault(int(slot), []).append((int(i0), int(i1), int(gq)))
        order[int(gq)].append((int(slot), int(i0), int(i1)))
    assert per.max() - per.min() <= 1 and per.sum() == nunits * n
    for slot, ps in parts.items():
        ps.sort()
        assert len(ps) <= 2 and ps[0][0] == 0 and ps[-1][1] == n
        if len(ps) == 2:  # first part on one pipeline, last part on the next
            assert ps[0][1] == ps[1][0] and ps[1][2] == ps[0][2] + 1
    for gq, us in order.items():
        kinds = [0 if (i0 == 0 and i1 < n) else 2 if i0 > 0 else 1 for _, i0, i1 in us]
        assert kinds == sorted(kinds) and kinds.count(0) <= 1 and kinds.count(2) <= 1
    # adversarial execution: always advance the LAST pipeline that can move
    done = {s: 0 for s in parts}
    pos = {g: 0 for g in order}
    left = sum(len(v) for v in order.values())
    while left:
        moved = False
        for gq in sorted(order, reverse=True):
            if pos[gq] < len(order[gq]):
                slot, i0, i1 = order[gq][pos[gq]]
                if done[slot] >= i0:
                    assert done[slot] == i0
                    done[slot] = i1
                    pos[gq] += 1
                    left -= 1
                    moved = True
        assert moved, "deadlock"
    assert all(v == n for v in done.values())
