"""Host-side check of the temporally blocked pass's start-up-row cut (TSW_TB_STARTUP):
at input row i of an unclamped item, level m yields row s0 − K + i − m, and the kernel computes it
in the item's first SU_ROWS rows only when m ≤ ⌊i/2⌋.  Brute-force dependency propagation from the
item's outputs (level K rows [s0, s1), plus level K − 1 at the same rows, which the pass also
writes) back through the stencil's reads — rows r − 1, r, r + 1 of level m − 1 and row r of level
m − 2 (the u^{n−1} term) — must find every needed (level, row) computed and every skipped one
unneeded; with the fp32 y-flux cache every level must have run once before the plain rows."""
import pytest


def needed_rows(K, s0, s1):
    """{m: set of rows of level m that the pass's outputs depend on} (level 0 = input u^n)."""
    need = {m: set() for m in range(K + 1)}
    need[K] = set(range(s0, s1))
    need[K - 1] |= set(range(s0, s1))                 # u^{n+K−1} is written too
    for m in range(K, 0, -1):
        for r in need[m]:
            need[m - 1] |= {r - 1, r, r + 1}
            if m >= 2:
                need[m - 2].add(r)                    # p = level m − 2 at the same row
    return need


def su_rows(K, ycl):
    """The kernel's SU_ROWS for a y-flux cache on levels 1..ycl (fp32: ycl = K; fp64: 0, or
    TSW_TB_YCACHE_F64_LEVELS)."""
    return (2 * K // 3) * 3 if (2 * K // 3) * 3 >= 2 * ycl + 1 else (2 * ycl + 3) // 3 * 3


@pytest.mark.parametrize("K", [2, 3, 4, 5, 7, 8, 9, 10])
@pytest.mark.parametrize("ycl", [0, 2, 4, "K"])
def test_startup_cut_is_exact(K, ycl):
    ycl = K if ycl == "K" else min(ycl, K)
    cache = ycl > 0
    s0, s1 = 100, 137
    in_lo = s0 - K
    L = s1 + K - in_lo
    need = needed_rows(K, s0, s1)
    SU = su_rows(K, ycl)
    assert SU % 3 == 0                                 # the window phase of the next row is 0
    if ycl == K:                                       # the shortest such cut after row 2K
        assert SU == -(-(2 * K + 1) // 3) * 3
    for i in range(L):
        for m in range(1, K + 1):
            row = in_lo + i - m
            computed = (m <= i // 2) if i < SU else True
            if row in need[m]:
                assert computed, (K, i, m)
            if i < SU and not computed:
                assert row not in need[m], (K, i, m)
    # the plain rows after the cut read each level's cached flux from the previous row: every level
    # must have been computed at row SU − 1 (the cache variant) — and every needed row before the
    # cut is computed in both variants (checked above)
    if cache:   # every cached level ran at row SU − 1 (its first needed row is 2m ≤ SU − 1)
        assert (SU - 1) // 2 >= ycl


@pytest.mark.parametrize("K", [2, 5, 10])
def test_first_needed_row_is_2m(K):
    """The cut is tight: level m's first needed row is produced exactly at input row i = 2m."""
    s0, s1 = 50, 90
    need = needed_rows(K, s0, s1)
    for m in range(1, K + 1):
        first = min(need[m])
        assert first - (s0 - K) + m == 2 * m
