"""Seeded panel-pair generators for the parity tests.

Classes follow the reference's own test generators (PairGen,
proj/tests/test_kernels.cpp:47-79; selftest Gen, proj/include/gbem/selftest.hpp:60-161):
coplanar disjoint / adjacent / identical, parallel offset, orthogonal disjoint
/ edge-touching, plus far pairs of small panels (the regime where the
reference's corner sums lose digits) and pairs at
prescribed gap/diameter ratios that straddle the near/far switch.
Rows are (axis, level, a0, a1, b0, b1).
"""
from __future__ import annotations

import numpy as np

INPLANE = {0: (1, 2), 1: (0, 2), 2: (0, 1)}


def _span(rng, lo=-2.0, hi=2.0, wlo=0.3, whi=2.0):
    a = rng.uniform(lo, hi)
    return a, a + rng.uniform(wlo, whi)


def _crossing(a, b) -> bool:
    """Orthogonal rects cutting through each other (test_kernels.cpp:37-45)."""
    if int(a[0]) == int(b[0]):
        return False
    def ext(r, k):
        ax = int(r[0]); i0, i1 = INPLANE[ax]
        if k == ax:
            return r[1], r[1]
        return (r[2], r[3]) if k == i0 else (r[4], r[5])
    shared = 3 - int(a[0]) - int(b[0])
    ea, eb = ext(a, int(b[0])), ext(b, int(a[0]))
    sa, sb = ext(a, shared), ext(b, shared)
    return (ea[0] < b[1] < ea[1] and eb[0] < a[1] < eb[1] and min(sa[1], sb[1]) > max(sa[0], sb[0]))


def classic_pairs(rng, n):
    """PairGen classes: coplanar, parallel offset, orthogonal (no crossing)."""
    A, B = [], []
    while len(A) < n:
        ax = int(rng.integers(3))
        cls = int(rng.integers(3))
        a = [ax, rng.uniform(-1, 1), *_span(rng), *_span(rng)]
        if cls == 0:
            b = [ax, a[1], *_span(rng), *_span(rng)]
        elif cls == 1:
            b = [ax, a[1] + (1 if rng.random() < 0.5 else -1) * rng.uniform(0.3, 2), *_span(rng), *_span(rng)]
        else:
            bx = (ax + 1 + int(rng.integers(2))) % 3
            b = [bx, rng.uniform(-1, 1), *_span(rng), *_span(rng)]
        if not _crossing(a, b):
            A.append(a); B.append(b)
    return np.array(A), np.array(B)


def touching_pairs(rng, n):
    """Coplanar edge-adjacent, identical, and orthogonal edge-sharing pairs."""
    A, B = [], []
    for k in range(n):
        ax = int(rng.integers(3))
        lv = rng.normal()
        a = [ax, lv, *_span(rng), *_span(rng)]
        kind = k % 3
        if kind == 0:  # coplanar adjacent (selftest copAdjacent)
            b = [ax, lv, *_span(rng), *_span(rng)]
            along_a = rng.random() < 0.5
            hi = rng.random() < 0.5
            w = rng.uniform(0.3, 2.0)
            lo_i, hi_i = (2, 3) if along_a else (4, 5)
            if hi:
                b[lo_i], b[hi_i] = a[hi_i], a[hi_i] + w
            else:
                b[lo_i], b[hi_i] = a[lo_i] - w, a[lo_i]
        elif kind == 1:  # identical (self term)
            b = list(a)
        else:  # orthogonal sharing an edge: b's plane passes through a's edge
            bx = (ax + 1 + int(rng.integers(2))) % 3
            i0, i1 = INPLANE[ax]
            # a's extent along bx
            lo, hi = (a[2], a[3]) if bx == i0 else (a[4], a[5])
            lvl = hi if rng.random() < 0.5 else lo
            j0, j1 = INPLANE[bx]
            spans = {}
            for k2 in (j0, j1):
                if k2 == ax:  # b extends away from a's plane on one side
                    w = rng.uniform(0.3, 2.0)
                    spans[k2] = (lv, lv + w) if rng.random() < 0.5 else (lv - w, lv)
                else:  # shared axis: overlap with a's extent
                    ea = (a[2], a[3]) if k2 == i0 else (a[4], a[5])
                    c = rng.uniform(ea[0], ea[1])
                    spans[k2] = (c - rng.uniform(0.2, 1.5), c + rng.uniform(0.2, 1.5))
            b = [bx, lvl, *spans[j0], *spans[j1]]
        A.append(a); B.append(b)
    return np.array(A), np.array(B)


def ratio_pairs(rng, n, g_lo, g_hi):
    """Pairs with gap/max-diameter in [g_lo, g_hi], mixed classes, aspect up to 10,
    size ratio up to 8 (bisection on the offset along a random direction)."""
    A, B = [], []
    for _ in range(n):
        ax = int(rng.integers(3))
        la = rng.uniform(0.2, 1.2)
        lb = la * (1.0 if rng.random() < 0.4 else np.exp(rng.uniform(-np.log(10), np.log(10))))
        a = [ax, 0.0, -la / 2, la / 2, -lb / 2, lb / 2]
        cls = int(rng.integers(3))
        bx = ax if cls < 2 else (ax + 1 + int(rng.integers(2))) % 3
        s = np.exp(rng.uniform(-np.log(8), np.log(8)))
        lc = rng.uniform(0.2, 1.2) * s
        ld = lc * (1.0 if rng.random() < 0.4 else np.exp(rng.uniform(-np.log(10), np.log(10))))
        d = rng.normal(size=3)
        if cls == 0:
            d[ax] = 0.0
        d /= np.linalg.norm(d)
        g_target = rng.uniform(g_lo, g_hi)
        dm = max(np.hypot(la, lb), np.hypot(lc, ld))
        j0, j1 = INPLANE[bx]

        def place(t):
            c = d * t
            lvl = 0.0 if cls == 0 else c[bx]
            return [bx, lvl, c[j0] - lc / 2, c[j0] + lc / 2, c[j1] - ld / 2, c[j1] + ld / 2]

        lo, hi = 0.0, 500.0
        for _ in range(80):
            mid = 0.5 * (lo + hi)
            b = place(mid)
            if _gap(a, b) / dm < g_target:
                lo = mid
            else:
                hi = mid
        A.append(a); B.append(place(hi))
    return np.array(A), np.array(B)


def _ext(r, k):
    ax = int(r[0]); i0, i1 = INPLANE[ax]
    if k == ax:
        return r[1], r[1]
    return (r[2], r[3]) if k == i0 else (r[4], r[5])


def _gap(a, b):
    s = 0.0
    for k in range(3):
        la, ha = _ext(a, k); lb, hb = _ext(b, k)
        g = max(lb - ha, la - hb, 0.0)
        s += g * g
    return np.sqrt(s)


def small_far_pairs(rng, n, edge_lo=0.002, edge_hi=0.05, dist_lo=0.5, dist_hi=5.0):
    """Small panels far apart: the cancellation regime of the reference's corner sums."""
    A, B = [], []
    for _ in range(n):
        ax = int(rng.integers(3)); bx = int(rng.integers(3))
        def mk(axis, centre):
            la = np.exp(rng.uniform(np.log(edge_lo), np.log(edge_hi)))
            lb = la * rng.uniform(0.5, 2.0)
            i0, i1 = INPLANE[axis]
            return [axis, centre[axis], centre[i0] - la / 2, centre[i0] + la / 2, centre[i1] - lb / 2, centre[i1] + lb / 2]
        c1 = rng.uniform(-1, 1, size=3)
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        c2 = c1 + d * rng.uniform(dist_lo, dist_hi)
        if rng.random() < 0.3:  # coplanar variant
            bx = ax
            c2[ax] = c1[ax]
        A.append(mk(ax, c1)); B.append(mk(bx, c2))
    return np.array(A), np.array(B)


def near_contact_pairs(rng, n, g_lo, g_hi, kind, spacing=50.0):
    """Offset-parallel ("parallel"), orthogonal ("orthogonal") or coplanar
    ("coplanar": same plane, the closed form kernels.hpp:48-94) pairs at
    gap/max-diameter log-uniform in [g_lo, g_hi): the near-contact regime of the
    reference's reduced integrands (kernels.hpp:138-153, 175-214) and its
    Romberg (quadrature.hpp:70-113).  Pair k is translated to its own lattice
    site `spacing` apart (panels are at most
    ~20 long: size ratio and aspect up to 4), so the 2n panels [A0, B0, A1, B1, ...] also form a
    panel set whose cross pairs are all far (the assembly route test)."""
    A, B = [], []
    side = int(np.ceil(n ** (1.0 / 3.0)))
    while len(A) < n:
        ax = int(rng.integers(3))
        la = rng.uniform(0.2, 1.2)
        lb = la * (1.0 if rng.random() < 0.4 else np.exp(rng.uniform(-np.log(4), np.log(4))))
        a = [ax, 0.0, -la / 2, la / 2, -lb / 2, lb / 2]
        bx = ax if kind in ("parallel", "coplanar") else (ax + 1 + int(rng.integers(2))) % 3
        s = np.exp(rng.uniform(-np.log(4), np.log(4)))
        lc = rng.uniform(0.2, 1.2) * s
        ld = lc * (1.0 if rng.random() < 0.4 else np.exp(rng.uniform(-np.log(4), np.log(4))))
        d = rng.normal(size=3)
        if kind == "parallel" and abs(d[ax]) < 0.05:
            d[ax] = 0.05 if d[ax] >= 0 else -0.05  # keep the planes apart (offset-parallel, not coplanar)
        if kind == "coplanar":
            d[ax] = 0.0
        d /= np.linalg.norm(d)
        g_target = np.exp(rng.uniform(np.log(g_lo), np.log(g_hi)))
        dm = max(np.hypot(la, lb), np.hypot(lc, ld))
        j0, j1 = INPLANE[bx]

        def place(t):
            c = d * t
            return [bx, c[bx], c[j0] - lc / 2, c[j0] + lc / 2, c[j1] - ld / 2, c[j1] + ld / 2]

        lo, hi = 0.0, 500.0
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if _gap(a, place(mid)) / dm < g_target:
                lo = mid
            else:
                hi = mid
        b = place(hi)
        g = _gap(a, b) / dm
        if not (g_lo <= g < g_hi) or _crossing(a, b):
            continue
        k = len(A)
        site = np.array([k % side, (k // side) % side, k // (side * side)], dtype=float) * spacing

        def shift(r):
            axis = int(r[0]); i0, i1 = INPLANE[axis]
            return [axis, r[1] + site[axis], r[2] + site[i0], r[3] + site[i0], r[4] + site[i1], r[5] + site[i1]]

        A.append(shift(a)); B.append(shift(b))
    return np.array(A), np.array(B)
