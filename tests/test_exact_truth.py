"""Pins the closed-form truth (tests/exact_truth.py) used by the near-contact
parity tests: the antiderivative identities, an independent mpmath quadrature,
the reference's frozen values, and the tight-tolerance reference on every
golden pair where the reference's Romberg converged."""
import json
import random
from pathlib import Path

import numpy as np
import pytest

import exact_truth as E

GOLD = Path(__file__).resolve().parent / "golden"


def test_antiderivative_identities():
    sp = pytest.importorskip("sympy")
    u, v, z, p, w, q = sp.symbols("u v z p w q", real=True)
    r3 = sp.sqrt(u ** 2 + v ** 2 + z ** 2)
    F = ((u ** 2 - z ** 2) / 2 * v * sp.log(v + r3) + (v ** 2 - z ** 2) / 2 * u * sp.log(u + r3)
         - u * v * z * sp.atan(u * v / (z * r3)) - r3 * (u ** 2 + v ** 2 - 2 * z ** 2) / 6)
    r = sp.sqrt(p ** 2 + w ** 2 + q ** 2)
    H = ((p * w ** 2 / 2 - p ** 3 / 6) * sp.log(q + r) + (q * w ** 2 / 2 - q ** 3 / 6) * sp.log(p + r)
         + p * q * w * sp.log(w + r) - w ** 3 / 6 * sp.atan(p * q / (w * r))
         - q ** 2 * w / 2 * sp.atan(p * w / (q * r)) - p ** 2 * w / 2 * sp.atan(q * w / (p * r)) - p * q * r / 3)
    dF = sp.lambdify((u, v, z), sp.diff(F, u, 2, v, 2) - 1 / r3, "mpmath")
    dH = sp.lambdify((p, w, q), sp.diff(H, p, 1, w, 2, q, 1) - 1 / r, "mpmath")
    import mpmath as mp
    mp.mp.dps = 40
    rnd = random.Random(5)
    for _ in range(20):
        a, b, c = [mp.mpf(rnd.uniform(0.1, 3)) * rnd.choice([-1, 1]) for _ in range(3)]
        assert abs(dF(a, b, c)) < mp.mpf(10) ** -30
        assert abs(dH(a, b, c)) < mp.mpf(10) ** -30


# proj/tests/test_kernels.cpp:166-215 (the reference's frozen U values)
FROZEN = [
    ((2, 0, 0, 1, 0, 1), (2, 0, 0, 1, 0, 1), 0.2366005022046692),
    ((0, 1, 0, 2, -0.25, 0.25), (0, 1, 0, 2, -0.25, 0.25), 0.21169029935491254),
    ((2, 0, 0, 1, 0, 1), (2, 0, 1, 2.3, 0, 0.7), 0.07287312340623026),
    ((1, -2, 0, 1.5, 0, 1), (1, -2, 2, 3, 0.5, 2.5), 0.12268222523420745),
    ((2, 1, 0, 1, 0, 1), (2, 0, 0, 1, 0, 1), 0.06993383553800263),
    ((0, 2.5, -1, 0.5, 0.3, 1.7), (0, 1, 0.2, 2, -0.5, 0.9), 0.18994761567034635),
    ((2, 0, 0, 1, 0, 1), (0, 2, 0.5, 1.5, 1, 2), 0.03625499787837069),
    ((2, 0, 0, 1, 0, 1), (1, 0, 0, 1, 0, 1), 0.10734127519843392),
    ((2, 0, 0, 2, -1, 1), (0, 1, -0.5, 0.5, 0, 1.5), 0.4790527168879336),
]


@pytest.mark.parametrize("a,b,val", FROZEN)
def test_frozen_reference_values(a, b, val):
    # the frozen values are the reference's own Romberg results (relTol 1e-8)
    assert abs(E.u_exact(a, b) - val) <= 1e-8 * val


def test_against_direct_quadrature():
    rng = np.random.default_rng(11)
    import pairgen as G
    A, B = G.classic_pairs(rng, 2)
    A2, B2 = G.near_contact_pairs(rng, 1, 1e-3, 1e-2, "orthogonal")
    A3, B3 = G.near_contact_pairs(rng, 1, 1e-2, 1e-1, "parallel")
    for a, b in zip(np.vstack([A, A2, A3]), np.vstack([B, B2, B3])):
        ex, qd = E.u_exact(a, b), E.u_quad(a, b, dps=17)
        assert abs(ex - qd) <= 1e-12 * abs(ex), (a, b, ex, qd)


def test_golden_exact_matches_converged_tight_reference():
    d = json.loads((GOLD / "near_contact_golden.json").read_text())
    ex, tight, tc = np.array(d["exact"]), np.array(d["tight"]), np.array(d["tight_converged"], bool)
    rel = np.abs(tight - ex) / ex
    assert tc.sum() >= 0.85 * len(tc)
    assert rel[tc].max() <= 1e-12, rel[tc].max()
    # the closed form is reproducible from the stored geometry
    A, B = np.array(d["A"]), np.array(d["B"])
    for k in range(0, len(A), 97):
        assert E.u_exact(A[k], B[k]) == ex[k]
