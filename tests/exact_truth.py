"""Closed-form truth for parallel and orthogonal panel pairs, in arbitrary
precision (mpmath) — TEST INFRASTRUCTURE ONLY (golden-vector generation and
parity tests; never imported by the product).

The Galerkin single-layer pair integral (what `u_pair_integral`,
proj/include/gbem/kernels.hpp:270-291, returns) is

    U = 1/(4 pi) * integral_a integral_b dA dA' / |x - y|.

For axis-aligned rectangles it is a corner sum of a 4-fold antiderivative of
1/r, evaluated here with 50 significant digits so the sum does not cancel
(the reference evaluates near pairs by 1-D Romberg over reduced integrands,
kernels.hpp:96-214 and quadrature.hpp:27-113; this is an independent route):

* parallel planes at normal offset z (coplanar: z = 0):
    F(u, v) = (u^2 - z^2)/2 v ln(v + r) + (v^2 - z^2)/2 u ln(u + r)
              - u v z atan(u v / (z r)) - r (u^2 + v^2 - 2 z^2) / 6,
  with d^4 F / du^2 dv^2 = 1/r, u and v the in-plane coordinate differences;
* orthogonal planes, p = offset of a point of panel a from panel b's plane,
  q = offset of a point of panel b from panel a's plane, w = the difference
  along the shared axis:
    H(p, w, q) = (p w^2/2 - p^3/6) ln(q + r) + (q w^2/2 - q^3/6) ln(p + r)
                 + p q w ln(w + r) - w^3/6 atan(p q / (w r))
                 - q^2 w/2 atan(p w / (q r)) - p^2 w/2 atan(q w / (p r)) - p q r / 3,
  with d^4 H / dp dw^2 dq = 1/r.

Both were found by fitting an ansatz and verified symbolically
(tests/test_exact_truth.py re-checks the derivative identities and compares
against a direct mpmath quadrature).  The difference integrals use the
corner signs  G(a1 - c0) - G(a0 - c0) - G(a1 - c1) + G(a0 - c1).  For the
orthogonal case panel a is split at b's plane and panel b at a's plane, so
p and q keep one sign inside each piece (the atan terms are discontinuous
across p = 0 and q = 0).  Terms whose polynomial prefactor is exactly zero are
dropped (their limits are zero), which covers touching corners.
"""
from __future__ import annotations

import mpmath as mp

INPLANE = {0: (1, 2), 1: (0, 2), 2: (0, 1)}
DPS = 50


def _span(r, k):
    ax = int(r[0])
    i0, i1 = INPLANE[ax]
    if k == ax:
        return (mp.mpf(r[1]), mp.mpf(r[1]))
    return (mp.mpf(r[2]), mp.mpf(r[3])) if k == i0 else (mp.mpf(r[4]), mp.mpf(r[5]))


def _t(pref, f, *args):
    return mp.mpf(0) if pref == 0 else pref * f(*args)


def _F(u, v, z):
    r = mp.sqrt(u * u + v * v + z * z)
    s = _t((u * u - z * z) / 2 * v, lambda: mp.log(v + r) if v + r > 0 else mp.mpf(0))
    s += _t((v * v - z * z) / 2 * u, lambda: mp.log(u + r) if u + r > 0 else mp.mpf(0))
    s -= _t(u * v * z, lambda: mp.atan(u * v / (z * r)))
    return s - r * (u * u + v * v - 2 * z * z) / 6


def _H(p, w, q):
    r = mp.sqrt(p * p + w * w + q * q)
    lg = lambda x: mp.log(x + r) if x + r > 0 else mp.mpf(0)  # noqa: E731
    s = _t(p * w * w / 2 - p ** 3 / 6, lambda: lg(q))
    s += _t(q * w * w / 2 - q ** 3 / 6, lambda: lg(p))
    s += _t(p * q * w, lambda: lg(w))
    s -= _t(w ** 3 / 6, lambda: mp.atan(p * q / (w * r)))
    s -= _t(q * q * w / 2, lambda: mp.atan(p * w / (q * r)))
    s -= _t(p * p * w / 2, lambda: mp.atan(q * w / (p * r)))
    return s - p * q * r / 3


def _diff_corners(a, c):
    """(difference, sign) of the double integral of g(x1 - x2), x1 in a, x2 in c."""
    return ((a[1] - c[0], 1), (a[0] - c[0], -1), (a[1] - c[1], -1), (a[0] - c[1], 1))


def _split(lo, hi, at):
    return [(lo, at), (at, hi)] if lo < at < hi else [(lo, hi)]


def u_exact(a, b, dps: int = DPS) -> float:
    """U(a, b) for rows (axis, level, a0, a1, b0, b1)."""
    with mp.workdps(dps):
        ax, bx = int(a[0]), int(b[0])
        if ax == bx:
            i0, i1 = INPLANE[ax]
            z = mp.mpf(a[1]) - mp.mpf(b[1])
            tot = mp.mpf(0)
            for u, su in _diff_corners(_span(a, i0), _span(b, i0)):
                for v, sv in _diff_corners(_span(a, i1), _span(b, i1)):
                    tot += su * sv * _F(u, v, z)
        else:
            s = 3 - ax - bx
            xb, za = mp.mpf(b[1]), mp.mpf(a[1])
            Pa, Qb = _span(a, bx), _span(b, ax)
            tot = mp.mpf(0)
            for p0, p1 in _split(Pa[0], Pa[1], xb):
                for z0, z1 in _split(Qb[0], Qb[1], za):
                    pc = ((p1 - xb, 1), (p0 - xb, -1))
                    qc = ((za - z0, 1), (za - z1, -1))
                    for w, sw in _diff_corners(_span(a, s), _span(b, s)):
                        for p, sp in pc:
                            for q, sq in qc:
                                tot += sw * sp * sq * _H(p, w, q)
        return float(tot / (4 * mp.pi))


def u_quad(a, b, dps: int = 30) -> float:
    """Independent check: the same integral by 2-D mpmath quadrature of the
    tent-reduced form (x1 - x2 pushed forward to a trapezoid weight along each
    axis in-plane for both panels), split at the tent knees and at 0; for an
    orthogonal pair the integral along the offset from panel a's plane is done
    in closed form (asinh) and the other two numerically."""
    with mp.workdps(dps):
        ax, bx = int(a[0]), int(b[0])

        def tent(sa, sc):
            (a0, a1), (c0, c1) = sa, sc
            k = sorted([a0 - c1, a0 - c0, a1 - c1, a1 - c0])

            def T(w):
                return max(mp.mpf(0), min(a1, w + c1) - max(a0, w + c0))
            return T, k

        if ax == bx:
            i0, i1 = INPLANE[ax]
            z2 = (mp.mpf(a[1]) - mp.mpf(b[1])) ** 2
            Tu, ku = tent(_span(a, i0), _span(b, i0))
            Tv, kv = tent(_span(a, i1), _span(b, i1))
            ku = sorted(set(ku + [mp.mpf(0)])); kv = sorted(set(kv + [mp.mpf(0)]))
            ku = [x for x in ku if ku[0] <= x <= ku[-1]]; kv = [x for x in kv if kv[0] <= x <= kv[-1]]
            val = mp.quad(lambda u, v: Tu(u) * Tv(v) / mp.sqrt(u * u + v * v + z2), ku, kv)
        else:
            s = 3 - ax - bx
            xb, za = mp.mpf(b[1]), mp.mpf(a[1])
            Pa, Qb = _span(a, bx), _span(b, ax)
            Tw, kw = tent(_span(a, s), _span(b, s))
            kw = sorted(set(kw + [mp.mpf(0)])); kw = [x for x in kw if kw[0] <= x <= kw[-1]]
            pk = [x - xb for x in sorted(set([Pa[0], Pa[1]] + ([xb] if Pa[0] < xb < Pa[1] else [])))]
            q0, q1 = za - Qb[1], za - Qb[0]

            def inner(w, p):  # the q integral in closed form: asinh(q / rho) between the q limits
                rho = mp.sqrt(w * w + p * p)
                return Tw(w) * (mp.asinh(q1 / rho) - mp.asinh(q0 / rho))
            val = mp.quad(inner, kw, pk)
        return float(val / (4 * mp.pi))
