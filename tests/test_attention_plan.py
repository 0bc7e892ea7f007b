"""Host-side attention work plan (tc_attn.cu plan_attention through mpic_attention_plan; no
GPU needed): every (head, query tile) key range is covered exactly once, split partials map
onto their combine jobs one slot each, pairs share their first key block, the persistent
CTAs' item lists partition the items, and the longest-processing-time assignment is
balanced to within one item. Row layouts: the bench's MPIC-k selections (configs B, C, D,
E16), random sorted selections, and batched requests (per-row start of the row's request)."""
import ctypes as C

import numpy as np
import pytest

from paper_2502_01960_b200 import _lib

NO = 0xFFFFFFFF


def mpic_rows(imgs, T=2304, k=32):
    rows, at = [], 0
    for i in range(imgs):
        t = 32 + 7 * i
        rows += list(range(at, at + t))
        at += t
        rows += list(range(at, at + min(k, T)))
        at += T
    rows += list(range(at, at + 32))
    return np.array(rows, np.uint32)


def plan(rows, H, starts=None):
    L = _lib.lib()
    rows = np.ascontiguousarray(rows, np.uint32)
    st = None if starts is None else np.ascontiguousarray(starts, np.uint32)
    counts = np.zeros(4, np.uint32)
    _lib.check(L.mpic_attention_plan(rows.ctypes.data, len(rows), H, None if st is None else st.ctypes.data,
                                     counts.ctypes.data, None, 0, None, 0, None, 0))
    items, ctas, jobs, slots = (int(x) for x in counts)
    units = np.zeros((items, 10), np.uint32)
    offs = np.zeros(ctas + 1, np.uint32)
    jb = np.zeros((max(jobs, 1), 4), np.uint32)
    _lib.check(L.mpic_attention_plan(rows.ctypes.data, len(rows), H, None if st is None else st.ctypes.data,
                                     counts.ctypes.data, units.ctypes.data, items, offs.ctypes.data, ctas + 1,
                                     jb.ctypes.data, max(jobs, 1)))
    return units, offs, jb[:jobs], slots


def cost(u):  # tc_attn.cu plan_attention's estimate (0.1 us units)
    if u[3] == NO:
        return 16 * (u[4] - u[1]) + 20
    ln, both = max(u[4], u[5]) - u[1], min(u[4], u[5]) - u[1]
    return 27 * both + 20 * (ln - both) + 20


def check(rows, H, starts=None):
    units, offs, jobs, slots = plan(rows, H, starts)
    m = len(rows)
    shift = (-m) % 128
    tiles = (m + 127) // 128
    last = lambda t: (t + 1) * 128 - shift - 1
    first = lambda t: 0 if t == 0 else last(t - 1) + 1
    nblk = [int(rows[last(t)]) // 128 + 1 for t in range(tiles)]
    sblk = [0 if starts is None else min(int(starts[first(t)]) // 128, nblk[t] - 1) for t in range(tiles)]
    cover = {}
    seen_slots = set()
    for u in units:
        hd, b0 = int(u[0]), int(u[1])
        if u[3] != NO:
            assert u[2] != u[3]  # a pair holds two different tiles starting at the same block
        for x in range(2):
            t = int(u[2 + x])
            if t == NO:
                continue
            b1 = int(u[4 + x])
            assert b0 < b1
            for b in range(b0, b1):
                key = (hd, t, b)
                assert key not in cover, f"block covered twice: {key}"
                cover[key] = (int(u[6 + x]), int(u[8 + x]))
            if u[6 + x] != NO:
                assert u[6 + x] not in seen_slots
                seen_slots.add(int(u[6 + x]))
                j = jobs[u[8 + x]]
                assert (j[0], j[1]) == (t, hd) and j[2] <= u[6 + x] < j[2] + j[3]
    for hd in range(H):
        for t in range(tiles):
            got = [b for b in range(sblk[t], nblk[t]) if (hd, t, b) in cover]
            assert got == list(range(sblk[t], nblk[t])), f"head {hd} tile {t}: range not covered"
            assert not [b for (h2, t2, b) in cover if h2 == hd and t2 == t and not sblk[t] <= b < nblk[t]]
            direct = {cover[(hd, t, b)][0] == NO for b in range(sblk[t], nblk[t])}
            assert len(direct) == 1  # a tile is either written directly or only through partials
    assert seen_slots == set(range(slots))
    for j in jobs:
        assert 2 <= j[3] <= 16
    # persistent CTA lists partition the items; LPT keeps the loads within one item
    assert offs[0] == 0 and offs[-1] == len(units) and np.all(np.diff(offs.astype(np.int64)) >= 1)
    loads = [sum(cost(u) for u in units[offs[c]:offs[c + 1]]) for c in range(len(offs) - 1)]
    assert max(loads) - min(loads) <= max(cost(u) for u in units)
    return len(units), len(offs) - 1, len(jobs)


@pytest.mark.parametrize("imgs,T,H", [(1, 576, 32), (4, 2304, 32), (8, 2304, 32), (16, 2304, 32), (2, 576, 8)])
def test_plan_mpic_selections(imgs, T, H):
    items, ctas, jobs = check(mpic_rows(imgs, T), H)
    assert ctas == min(items, 148)


@pytest.mark.parametrize("m,n,H,seed", [(1, 50, 4, 0), (129, 1000, 3, 1), (330, 9418, 32, 2), (1896, 38248, 32, 3),
                                        (4000, 4000, 2, 4)])
def test_plan_random_rows(m, n, H, seed):
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(n - 1, m - 1, replace=False)).astype(np.uint32) if m > 1 else np.zeros(0, np.uint32)
    rows = np.append(rows, n - 1).astype(np.uint32)
    check(rows, H)


def test_plan_batched_starts():
    """Three requests in one pass: a row sees only its own request's rows (from its start)."""
    rows, starts, off = [], [], 0
    for imgs in (1, 3, 2):
        r = mpic_rows(imgs, 576)
        n = int(r[-1]) + 1
        rows += (r + off).tolist()
        starts += [off] * len(r)
        off += n
    check(np.array(rows, np.uint32), 32, np.array(starts, np.uint32))
