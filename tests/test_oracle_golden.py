"""Pins the CPU oracle (oracle/gbem_oracle.c) to the reference's own known answers
and, pair by pair, to the reference headers compiled in place (oracle/_ref).
CPU only."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import pairgen as G

GOLDEN_U = [  # proj/tests/test_kernels.cpp:166-215
    ((2, 0, (0, 1), (0, 1)), (2, 0, (0, 1), (0, 1)), 0.2366005022046692, 1e-9),
    ((0, 1, (0, 2), (-0.25, 0.25)), (0, 1, (0, 2), (-0.25, 0.25)), 0.21169029935491254, 1e-9),
    ((2, 0, (0, 1), (0, 1)), (2, 0, (1, 2.3), (0, 0.7)), 0.07287312340623026, 1e-9),
    ((1, -2, (0, 1.5), (0, 1)), (1, -2, (2, 3), (0.5, 2.5)), 0.12268222523420745, 1e-9),
    ((2, 1, (0, 1), (0, 1)), (2, 0, (0, 1), (0, 1)), 0.06993383553800263, 1e-6),
    ((0, 2.5, (-1, 0.5), (0.3, 1.7)), (0, 1, (0.2, 2), (-0.5, 0.9)), 0.18994761567034635, 1e-6),
    ((2, 0, (0, 1), (0, 1)), (0, 2, (0.5, 1.5), (1, 2)), 0.03625499787837069, 1e-6),
    ((2, 0, (0, 1), (0, 1)), (1, 0, (0, 1), (0, 1)), 0.10734127519843392, 1e-6),
    ((2, 0, (0, 2), (-1, 1)), (0, 1, (-0.5, 0.5), (0, 1.5)), 0.4790527168879336, 1e-6),
]


def test_frozen_single_layer_values():
    L = O.orc()
    for a, b, v, tol in GOLDEN_U:
        kv = L.orc_u_pair_integral(C.byref(O.rect(*a)), C.byref(O.rect(*b)), 1e-8, 16)
        assert kv.status == 0 and kv.converged
        assert abs(kv.value - v) <= tol * v


def test_frozen_values_tight_match():
    """Coplanar closed forms reproduce the frozen digits; Romberg paths to ~1e-11."""
    L = O.orc()
    for a, b, v, tol in GOLDEN_U:
        kv = L.orc_u_pair_integral(C.byref(O.rect(*a)), C.byref(O.rect(*b)), 1e-8, 16)
        assert abs(kv.value - v) <= (1e-15 if tol == 1e-9 else 2e-11) * v


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_bit_exact_vs_compiled_reference(seed):
    rng = np.random.default_rng(seed)
    A1, B1 = G.classic_pairs(rng, 400)
    A2, B2 = G.touching_pairs(rng, 60)
    A3, B3 = G.small_far_pairs(rng, 200)
    A = np.vstack([A1, A2, A3]); B = np.vstack([B1, B2, B3])
    o, oc, os_ = O.u_pairs("orc", A, B, nthreads=4)
    r, rc_, rs = O.u_pairs("ref", A, B, nthreads=4)
    assert os_ == rs == 0
    assert np.array_equal(o, r)            # bit-identical
    assert np.array_equal(oc, rc_)


def test_symmetry_and_positivity():
    """test_kernels.cpp:118-127 on the oracle."""
    rng = np.random.default_rng(424242)
    A, B = G.classic_pairs(rng, 100)
    u1, _, _ = O.u_pairs("orc", A, B)
    u2, _, _ = O.u_pairs("orc", B, A)
    assert np.all(u1 > 0)
    assert np.array_equal(u1, u2)  # canonical argument order makes it bitwise symmetric


def _aitken(v0, v1, v2):
    den = (v2 - v1) - (v1 - v0)
    if abs(den) < 1e-14 * max(abs(v2), 1e-300):
        return v2
    return v2 - (v2 - v1) ** 2 / den


def test_brute_force_oracle_reference_values():
    """test_oracle.cpp:60-88 on the restated recursive Gauss oracle."""
    L = O.orc()
    f = L.orc_oracle_pair_integral
    f.restype = C.c_double
    sq = O.rect(2, 0, (0, 1), (0, 1))
    acc = _aitken(*(f(C.byref(sq), C.byref(sq), d) for d in (3, 4, 5)))
    assert abs(acc - 0.2366005022046692) <= 1e-5 * 0.2366005022046692
    a, b = O.rect(2, 1, (0, 1), (0, 1)), O.rect(2, 0, (0, 1), (0, 1))
    assert abs(f(C.byref(a), C.byref(b), 6) - 0.06993383553800263) <= 1e-8 * 0.0699
    a, b = O.rect(2, 0, (0, 1), (0, 1)), O.rect(1, 0, (0, 1), (0, 1))
    acc = _aitken(*(f(C.byref(a), C.byref(b), d) for d in (3, 4, 5)))
    assert abs(acc - 0.10734127519843392) <= 1e-5 * 0.107


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_brute_force_oracle_matches_reference_oracle():
    rng = np.random.default_rng(5)
    A, B = G.classic_pairs(rng, 20)
    for k in range(len(A)):
        ra, rb = O.rect(A[k, 0], A[k, 1], A[k, 2:4], A[k, 4:6]), O.rect(B[k, 0], B[k, 1], B[k, 2:4], B[k, 4:6])
        assert O.orc().orc_oracle_pair_integral(C.byref(ra), C.byref(rb), 3) == \
            O.ref().ref_oracle_pair_integral(C.byref(ra), C.byref(rb), 3)


def test_far_truth_matches_brute_force_oracle():
    """The composite-Gauss far-field truth agrees with the reference's own
    brute-force oracle (oracle.hpp:191) to its depth-6 accuracy."""
    rng = np.random.default_rng(11)
    A, B = G.ratio_pairs(rng, 30, 1.5, 4.0)
    t = O.truth_pairs(A, B, sub=2)
    f = O.orc().orc_oracle_pair_integral
    for k in range(len(A)):
        ra, rb = O.rect(A[k, 0], A[k, 1], A[k, 2:4], A[k, 4:6]), O.rect(B[k, 0], B[k, 1], B[k, 2:4], B[k, 4:6])
        assert abs(f(C.byref(ra), C.byref(rb), 4) - t[k]) <= 1e-10 * t[k]


QUAD_CASES = [  # proj/tests/test_quadrature.cpp:11-79: (which, mode, a, b, singA, singB, exact, tol)
    (0, 0, 0.0, 1.0, 0, 0, 1.0 / 3.0, 1e-12),
    (1, 0, 0.0, 1.0, 0, 0, 1.0, 0.0),
    (2, 0, 0.0, 1.0, 0, 0, 2 * np.log(2) - 1, 1e-8 * (2 * np.log(2) - 1)),
    (3, 0, 2.0, 2.0, 0, 0, 0.0, 0.0),
    (4, 0, 0.0, 3.1, 0, 0, 1 - np.cos(3.1), 1e-10),
    (6, 1, 0.0, 1.0, 1, 0, 2.0, 1e-9),
    (7, 1, 0.0, 1.0, 1, 0, -1.0, 1e-8),
    (8, 1, 0.0, 1.0, 0, 1, 2.0, 1e-9),
    (9, 1, 0.0, 1.0, 1, 1, 4.0, 1e-8),
    (10, 2, -1.0, 1.0, 0, 0, 4.0, 1e-8),
    (11, 2, -1.0, 2.0, 0, 0, 3.0, 1e-10),
]


@pytest.mark.parametrize("case", QUAD_CASES)
def test_quadrature_known_answers(case):
    which, mode, a, b, sa, sb, exact, tol = case
    st, cv, ev = C.c_int(), C.c_int(), C.c_long()
    v = O.orc().orc_quad_test(which, mode, a, b, sa, sb, C.byref(st), C.byref(cv), C.byref(ev))
    assert st.value == 0
    assert abs(v - exact) <= tol


def test_quadrature_nonfinite_is_an_error():
    st, cv, ev = C.c_int(), C.c_int(), C.c_long()
    O.orc().orc_quad_test(5, 0, 0.0, 1.0, 0, 0, C.byref(st), C.byref(cv), C.byref(ev))
    assert st.value == 2  # NumericalError("non-finite integrand sample")


def _chol(A, B):
    n = A.shape[0]
    Bc = np.ascontiguousarray(np.atleast_2d(B.T))
    X = np.zeros_like(Bc)
    res = np.zeros(Bc.shape[0])
    piv = C.c_int64(-1)
    rc = O.orc().orc_cholesky_solve(n, np.ascontiguousarray(A).ctypes.data, Bc.shape[0], Bc.ctypes.data,
                                    X.ctypes.data, res.ctypes.data, C.byref(piv))
    return rc, X.T, res, piv.value


def test_cholesky_restatement():
    """test_solver.cpp:32-125 on the restated reference loop."""
    rc, x, res, _ = _chol(np.eye(4), np.arange(4.0)[:, None])
    assert rc == 0 and np.array_equal(x[:, 0], np.arange(4.0)) and res[0] == 0.0
    rc, x, _, _ = _chol(np.diag([4.0, 9.0]), np.array([[2.0], [3.0]]))
    assert abs(x[0, 0] - 0.5) < 1e-15 and abs(x[1, 0] - 1 / 3) < 1e-15
    rng = np.random.default_rng(11)
    M = rng.normal(size=(50, 50)); A = M.T @ M + np.eye(50); b = rng.normal(size=(50, 1))
    rc, x, res, _ = _chol(A, b)
    assert np.abs(x - np.linalg.solve(A, b)).max() <= 1e-9
    assert res[0] <= 1e-10
    rc, _, _, piv = _chol(np.array([[1.0, 2.0], [2.0, 1.0]]), np.ones((2, 1)))
    assert rc == 2 and piv == 1


# --- block-system pieces (kernels.hpp:319-355, solver.hpp:53-88) -------------------

def _random_point_cases(rng, k):
    R = np.zeros((k, 6)); X = np.zeros((k, 3))
    for t in range(k):
        ax = int(rng.integers(3)); lvl = rng.uniform(-1, 1)
        a0 = rng.uniform(-1, 1); b0 = rng.uniform(-1, 1)
        R[t] = [ax, lvl, a0, a0 + rng.uniform(0.01, 1.5), b0, b0 + rng.uniform(0.01, 1.5)]
        X[t] = rng.uniform(-2, 2, size=3)
        if t % 5 == 0:
            X[t, ax] = lvl  # in the panel plane: q vanishes, u keeps its log terms
        if t % 7 == 0:  # on an edge / corner line
            i0 = 1 if ax == 0 else 0
            X[t, i0] = R[t, 2]
    return X, R


@pytest.mark.skipif(not O.ref_available(), reason="reference headers not compiled here")
def test_point_kernels_bit_identical_to_reference():
    rng = np.random.default_rng(11)
    X, R = _random_point_cases(rng, 2000)
    ns = np.where(rng.random(len(R)) < 0.5, 1, -1)
    u1, q1 = O.point_kernels("orc", X, R, ns)
    u2, q2 = O.point_kernels("ref", X, R, ns)
    assert np.array_equal(u1, u2) and np.array_equal(q1, q2)
    assert np.all(np.isfinite(u1)) and np.all(q1[::5] == 0.0)


def test_point_kernels_known_answers():
    """Unit square seen from its own centre plane and from far away."""
    R = np.array([[2, 0.0, -0.5, 0.5, -0.5, 0.5]] * 3)
    X = np.array([[0, 0, 1e-12], [0, 0, 50.0], [0, 0, -50.0]])
    u, q = O.point_kernels("orc", X, R, np.array([1, 1, 1]))
    # solid angle of the square seen from just above its centre -> 1/2 of the sphere
    assert abs(q[0] - 0.5) < 1e-9
    # far field: u -> area / (4 pi r), q -> area / (4 pi r^2) (signed by the side)
    assert abs(u[1] - 1.0 / (4 * np.pi * 50.0)) < 1e-3 * u[1]  # finite-size correction O((a/r)^2)
    assert abs(q[1] - 1.0 / (4 * np.pi * 2500.0)) < 1e-3 * q[1] and abs(q[2] + q[1]) < 1e-15


@pytest.mark.parametrize("n", [1, 2, 7, 40])
def test_lu_oracle_matches_numpy(n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + 0.1 * np.eye(n)
    b = rng.standard_normal(n)
    x, res, st, _ = O.lu_solve(A, b)
    assert st == 0
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-12)
    assert res < 1e-13


def test_lu_oracle_singular_row():
    A = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 6.0], [1.0, 0.0, 1.0]])
    _, _, st, bad = O.lu_solve(A, np.ones(3))
    assert st == 2 and bad == 2


# Double layer (test rect, source rect, source normal sign, frozen value):
# proj/tests/test_kernels.cpp:217-241, checked there at 1e-6 relative.
QGOLD = [
    ((2, 1, (0, 1), (0, 1)), (2, 0, (-0.2, 1.3), (0.1, 0.8)), 1, 0.0554151455434669),
    ((2, 0, (0, 1), (0, 1)), (0, 2, (0.5, 1.5), (1, 2)), -1, 0.011324772441013004),
    ((2, 0, (0, 1), (0, 1)), (1, 0, (0, 1), (0, 1)), 1, 0.11113873320194041),
    ((1, -0.8575535635412491, (0.34410487297464243, 0.9076144923978153), (-0.622649673169549, 0.1631672183635413)),
     (0, 0.9076144923978153, (-1.6627438264788437, -0.8575535635412491), (-0.6769789681037953, 1.073134547946061)),
     1, -0.0733166487590698),
]


def _qrows(rs):
    return np.array([[r[0], r[1], r[2][0], r[2][1], r[3][0], r[3][1]] for r in rs], dtype=float)


def test_double_layer_frozen_values():
    A = _qrows([g[0] for g in QGOLD]); B = _qrows([g[1] for g in QGOLD]); ns = [g[2] for g in QGOLD]
    v, conv, st = O.q_pairs("orc", A, B, ns)
    assert (st == 0).all() and conv.all()
    for k, g in enumerate(QGOLD):
        assert abs(v[k] - g[3]) <= 1e-6 * abs(g[3]), (k, v[k], g[3])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [424242, 5])
def test_double_layer_bit_exact_vs_compiled_reference(seed):
    rng = np.random.default_rng(seed)
    A, B = G.classic_pairs(rng, 120)
    ns = rng.choice([-1, 1], size=len(A))
    vo, co, so = O.q_pairs("orc", A, B, ns)
    vr, cr, sr = O.q_pairs("ref", A, B, ns)
    assert (so == sr).all() and (co == cr).all()
    assert np.array_equal(vo, vr)
    Aq = _qrows([g[0] for g in QGOLD]); Bq = _qrows([g[1] for g in QGOLD]); nq = [g[2] for g in QGOLD]
    assert np.array_equal(O.q_pairs("orc", Aq, Bq, nq)[0], O.q_pairs("ref", Aq, Bq, nq)[0])


def test_double_layer_closed_surface_identity():
    """test_kernels.cpp:274-295: on a closed cube (2x2 panels per face, outward
    normals) the double-layer row sums equal -|I|/2."""
    rows, ns = [], []
    for axis in range(3):
        for side in range(2):
            for ia in range(2):
                for ib in range(2):
                    rows.append([axis, float(side), 0.5 * ia, 0.5 * (ia + 1), 0.5 * ib, 0.5 * (ib + 1)])
                    ns.append(1 if side else -1)
    P = np.array(rows)
    n = len(P)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v, _, st = O.q_pairs("orc", P[ii.ravel()], P[jj.ravel()], np.array(ns)[jj.ravel()])
    assert (st == 0).all()
    s = v.reshape(n, n).sum(axis=1)
    assert np.abs(s + 0.5 * 0.25).max() <= 1e-3 * 0.125


def _worst_q():
    return json.loads((Path(__file__).parent / "golden" / "selftest_worst_q.json").read_text())["cases"]


def test_selftest_worst_q_pairs_match_restatement():
    """The on-device selftest at 20000 pairs per class (tools/selftest_probe.py) misses the
    reference's tolerances on the two orthogonal double-layer classes.  The evaluator is
    not the cause: on every failing pair the GPU value equals the reference algorithm's
    q_pair_integral (kernels.hpp:295-315, restated in oracle/) to round-off."""
    for c in _worst_q():
        A, B = np.array([c["worst_test"]]), np.array([c["worst_source"]])
        v, conv, st = O.q_pairs("orc", A, B, [c["worst_nsign"]])
        assert st[0] == 0 and conv[0]
        assert abs(v[0] - c["worst_value"]) <= 1e-13 * abs(v[0]), c["name"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_selftest_worst_q_pairs_are_oracle_limited():
    """...and the miss is the brute-force oracle's (oracle.hpp:191): for the disjoint class
    the depth-6 value used by the selftest (selftest.hpp:47-49) is further from the
    semi-analytic value than depth 7; for the adjacent class the Aitken extrapolation of
    depths 3/4/5 (selftest.hpp:39-45) lands further off than the raw depth-7 value."""
    for c in _worst_q():
        A, B, ns = np.array([c["worst_test"]]), np.array([c["worst_source"]]), [c["worst_nsign"]]
        v = c["worst_value"]
        d7 = O.q_oracle(A, B, ns, 7)[0]
        assert abs(d7 - v) < abs(c["worst_oracle"] - v), c["name"]
        assert abs(d7 - v) / abs(d7) < c["tol"], c["name"]
