"""GPU pair-integral parity against the reference kernel and the far-field truth.

Gate (two-sided):
  (i)  |gpu - truth| <= 1e-10 |truth|   (1e-8 for touching / self pairs);
       truth = composite 6^4 Gauss (2x2 split per panel) for gap/diam >= 1.5,
       the reference kernel itself below that (well conditioned there);
  (ii) |gpu - ref| <= max(1e-10 |ref|, 2 |ref - truth|).
"""
import numpy as np
import pytest

import oracle_lib as O
import pairgen as G
from paper_2203_11733_b200._native import PanelArrays

pytestmark = pytest.mark.gpu

GOLDEN = [  # proj/tests/test_kernels.cpp:166-215 (value, rel tol used there)
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


def _rows(rs):
    return np.array([[r[0], r[1], r[2][0], r[2][1], r[3][0], r[3][1]] for r in rs], dtype=float)


def _gpu(ctx, A, B, **kw):
    out, conv, st = ctx.u_pair_integrals(PanelArrays.from_matrix(A), PanelArrays.from_matrix(B),
                                         ctx.quad(**kw) if kw else None)
    return out, conv, st


def test_golden_values(ctx):
    A = _rows([g[0] for g in GOLDEN]); B = _rows([g[1] for g in GOLDEN])
    out, conv, _ = _gpu(ctx, A, B)
    ref, _, _ = O.u_pairs("ref" if O.ref_available() else "orc", A, B)
    for k, g in enumerate(GOLDEN):
        assert abs(out[k] - g[2]) <= g[3] * g[2], (k, out[k], g[2])
        assert abs(out[k] - ref[k]) <= 1e-10 * abs(ref[k]), (k, out[k], ref[k])
    assert conv.all()


def _gate(gpu, ref, truth, g, touching, tol=1e-10, tol_sing=1e-8):
    tol_v = np.where(touching, tol_sing, tol)
    far = g >= 1.5
    t = np.where(far, truth, ref)
    e1 = np.abs(gpu - t) / np.abs(t)
    e2 = np.abs(gpu - ref)
    lim2 = np.maximum(tol_v * np.abs(ref), 2 * np.abs(ref - truth))
    bad = (e1 > tol_v) | ((e2 > lim2) & far)
    return bad, e1


@pytest.mark.parametrize("seed", [424242, 7])
def test_classic_pairs(ctx, seed):
    rng = np.random.default_rng(seed)
    A, B = G.classic_pairs(rng, 300)
    out, conv, st = _gpu(ctx, A, B)
    ref, rconv, _ = O.u_pairs("orc", A, B)
    g = O.gap_ratio(A, B)
    truth = np.where(g >= 1.5, O.truth_pairs(A, B), ref)
    bad, e1 = _gate(out, ref, truth, g, g == 0)
    assert not bad.any(), (np.flatnonzero(bad)[:10], e1[bad][:10], st.as_dict())
    # symmetry: U(a,b) == U(b,a)  (test_kernels.cpp:118-127)
    out2, _, _ = _gpu(ctx, B, A)
    assert np.all(np.abs(out2 - out) <= 1e-12 * np.abs(out))
    assert np.all(out > 0)


def test_touching_pairs(ctx):
    rng = np.random.default_rng(20260817)
    A, B = G.touching_pairs(rng, 150)
    out, conv, st = _gpu(ctx, A, B)
    ref, rconv, _ = O.u_pairs("orc", A, B)
    rel = np.abs(out - ref) / np.abs(ref)
    assert rel.max() <= 1e-8, (rel.argmax(), rel.max())
    assert (conv == rconv).all()


@pytest.mark.parametrize("lo,hi", [(0.3, 0.75), (0.75, 1.0), (1.0, 1.5), (1.5, 3.0), (3.0, 10.0), (10.0, 100.0)])
def test_ratio_bands(ctx, lo, hi):
    rng = np.random.default_rng(int(lo * 1000 + hi))
    A, B = G.ratio_pairs(rng, 200, lo, hi)
    out, conv, st = _gpu(ctx, A, B)
    ref, _, _ = O.u_pairs("orc", A, B, rel_tol=1e-13, max_levels=20)  # tight reference as near truth
    g = O.gap_ratio(A, B)
    truth = np.where(g >= 1.5, O.truth_pairs(A, B, sub=3), ref)
    rel = np.abs(out - truth) / truth
    assert rel.max() <= 1e-10, (rel.argmax(), rel.max(), g[rel.argmax()])


def test_small_far_pairs_beat_cancellation(ctx):
    """Far small panels: the GPU Gauss path stays near the truth where the
    reference's closed forms cancel (hazard #1)."""
    rng = np.random.default_rng(99)
    A, B = G.small_far_pairs(rng, 300)
    out, _, _ = _gpu(ctx, A, B)
    truth = O.truth_pairs(A, B, sub=1)
    ref, _, _ = O.u_pairs("orc", A, B)
    rel = np.abs(out - truth) / truth
    assert rel.max() <= 1e-11
    # two-sided gate (ii) against the reference
    assert np.all(np.abs(out - ref) <= np.maximum(1e-10 * np.abs(ref), 2 * np.abs(ref - truth)) + 1e-12 * truth)
