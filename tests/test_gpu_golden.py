"""GPU results against the committed golden fixtures (tests/golden/make_golden.py):
capacitance matrices of BASELINE configs 1-2 computed with the compiled reference
kernel + dense Cholesky, and a seeded pair list with reference / tight /
Gauss-truth values."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2203_11733_b200 as g
from paper_2203_11733_b200._native import PanelArrays

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("cfg", [1, 2])
def test_cmatrix_matches_reference_pipeline(ctx, cfg):
    fx = json.loads((GOLD / f"config{cfg}_cmatrix.json").read_text())
    m = g.config_model(cfg, seed=fx["seed"])
    ps = m.partition(1)
    ids = m.net_ids
    net = np.array([ids.index(v) if k == 0 else -1 for v, k in zip(ps.net, ps.kind)], dtype=np.int32)
    Cm, res, ast, sst = ctx.extract_cmatrix(ps.arrays(), net, len(ids), fx["eps_r"])
    ref = np.array(fx["cmatrix_F"])
    rel = np.abs(Cm - ref) / np.abs(ref)
    assert rel.max() <= 1e-6, rel.max()          # north-star capacitance gate
    assert rel.max() <= 1e-10, rel.max()         # what we actually reach
    assert res.max() <= 1e-12
    assert ast.pairs_total == len(ps) * (len(ps) + 1) // 2
    # the C-matrix of a free-space single dielectric: C11 > 0, couplings < 0, near symmetric
    assert np.all(np.diag(Cm) > 0) and np.all(Cm[~np.eye(len(ids), dtype=bool)] < 0)
    assert np.abs(Cm - Cm.T).max() <= 1e-12 * np.abs(Cm).max()


def test_pair_fixture_two_sided_gate(ctx):
    fx = json.loads((GOLD / "pairs_golden.json").read_text())
    A, B = np.array(fx["A"]), np.array(fx["B"])
    out, conv, _ = ctx.u_pair_integrals(PanelArrays.from_matrix(A), PanelArrays.from_matrix(B))
    ref, tight, gt, gr = (np.array(fx[k]) for k in ("ref", "tight", "gauss_truth", "gap_ratio"))
    truth = np.where(gr >= 1.5, gt, tight)
    tol = np.where(gr == 0.0, 1e-8, 1e-10)
    assert np.all(np.abs(out - truth) <= tol * np.abs(truth))
    lim = np.maximum(tol * np.abs(ref), 2 * np.abs(ref - truth))
    assert np.all(np.abs(out - ref) <= lim + 1e-13 * np.abs(truth))
