"""Host logic of the pair kernel's balanced unit schedule (tc_wide.cu
wide_schedule, exported as segconv_debug_wide_schedule): every unit of the
im2col forward is run exactly once -- whole, or as both feature halves -- and
the busiest pair's load does not exceed round-robin's.  No GPU needed."""
import ctypes as C

import numpy as np
import pytest

from paper_2209_03704_b200 import _capi as A


def unit_base(batch, n, cout, nt=256):
    """Class-major units of make_wide's im2col forward for k = 3, p = 0: class
    grids (n-1 | n-2)^2, 256 anchors per pair tile, ceil(cout / NT) feature tiles."""
    rows = [n - 1, n - 1, n - 2, n - 2]
    cols = [n - 1, n - 2, n - 1, n - 2]
    n_tiles = -(-cout // nt)
    base = [0]
    for q in range(4):
        base.append(base[-1] + -(-batch * rows[q] * cols[q] // 256) * n_tiles)
    return base


def schedule(base, taps, nkb, pairs, halves=1):
    cap = 4096
    out = np.zeros(cap, dtype=np.uint16)
    b = (C.c_longlong * 5)(*base)
    t = (C.c_int * 4)(*taps)
    slots = A.lib().segconv_debug_wide_schedule(b, t, nkb, pairs, halves,
                                                out.ctypes.data_as(C.POINTER(C.c_uint16)), cap)
    return int(slots), out[:pairs * slots].reshape(pairs, slots) if slots else None


def cost(base, taps, nkb, u):
    q = max(i for i in range(4) if base[i] <= u)
    return taps[q] * nkb


@pytest.mark.parametrize("batch,n,cin,cout,kst", [(1024, 4, 1024, 512, 2), (1024, 5, 512, 256, 2),
                                                 (512, 4, 1024, 512, 2), (64, 4, 1024, 512, 2),
                                                 (1024, 7, 256, 128, 1)])
@pytest.mark.parametrize("halves", [0, 1])
def test_every_unit_once_and_no_worse_than_round_robin(batch, n, cin, cout, kst, halves):
    pairs = 74
    base = unit_base(batch, n, cout)
    taps = [4, 2, 2, 1]
    nkb = cin // 64 // kst
    slots, tab = schedule(base, taps, nkb, pairs, halves)
    units = base[4]
    rr = max(sum(cost(base, taps, nkb, u) for u in range(i, units, pairs)) for i in range(pairs))
    if slots == 0:
        return  # round-robin kept
    seen = {}
    load = []
    for row in tab:
        ents = [int(e) for e in row]
        # a pair's list is a prefix; 0xFFFF only pads its end
        live = [e for e in ents if e != 0xFFFF]
        assert ents[:len(live)] == live
        l = 0.0
        for e in live:
            u, h = e & 0x3FFF, e >> 14
            assert 0 <= u < units and h in (0, 1, 2)
            assert halves or h == 0
            seen.setdefault(u, []).append(h)
            l += cost(base, taps, nkb, u) * (1.0 if h == 0 else 0.5)
        load.append(l)
    assert sorted(seen) == list(range(units))
    for u, hs in seen.items():
        assert sorted(hs) in ([0], [1, 2]), (u, hs)
    # MMA-time makespan (halves at half the cost) is below round-robin's
    assert max(load) < rr


def test_c5_layer_a_uses_halves():
    """C5 layer a at batch 1024 (the stack's longest layer): round-robin puts
    128 k-blocks on the busiest pair for a mean of 111; the table splits
    two-tap units into feature halves and gets within 6 % of the mean."""
    base = unit_base(1024, 4, 512)
    taps = [4, 2, 2, 1]
    nkb = 1024 // 64 // 2
    slots, tab = schedule(base, taps, nkb, 74)
    assert slots > 0
    halves = sum(1 for e in tab.ravel() if e != 0xFFFF and (e >> 14))
    assert halves > 0
    load = [sum(cost(base, taps, nkb, int(e) & 0x3FFF) * (0.5 if e >> 14 else 1.0)
                for e in row if e != 0xFFFF) for row in tab]
    mean = sum(cost(base, taps, nkb, u) for u in range(base[4])) / 74
    assert max(load) <= 1.06 * mean
