"""The block (mixed-unknown) system on the GPU: lu_solve (solver.hpp:53-88), the
Galerkin block system assemble_multi (assembly.hpp:110-175) and the collocation
baseline assemble_collocation (assembly.hpp:179-227), against the CPU oracle
restatement (oracle/gbem_oracle.c, its point and double-layer kernels pinned
bit-for-bit to the compiled reference in test_oracle_golden.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2203_11733_b200 as g
from paper_2203_11733_b200._native import GbemError

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
TWO = ROOT / "tests" / "golden" / "bench_two_layer.gbem"
SINGLE = ROOT / "tests" / "golden" / "bench_single.gbem"
EPS0 = 8.854187817e-12


@pytest.mark.parametrize("n", [1, 5, 63, 64, 65, 130, 500, 1100])
def test_lu_matches_oracle_and_numpy(ctx, n):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + 0.5 * np.eye(n)
    b = rng.standard_normal(n)
    x, res, st = ctx.lu_solve(A, b)
    xr = np.linalg.solve(A, b)
    assert np.abs(x - xr).max() <= 1e-9 * np.abs(xr).max()
    if n <= 500:
        xo, ro, sto, _ = O.lu_solve(A, b)
        assert sto == 0
        assert np.abs(x - xo).max() <= 1e-10 * np.abs(xo).max()
        # backward error of the same order as the reference algorithm's (both
        # grow with cond(A); seed 130 gives cond 5e4)
        assert res <= 4 * max(ro, 1e-14), (res, ro)
    else:
        assert res <= 1e-11


def test_lu_pivots_zero_diagonal(ctx):
    # needs a row exchange at every step
    A = np.array([[0.0, 2.0, 1.0], [1.0, 0.0, 3.0], [4.0, 1.0, 0.0]])
    b = np.array([1.0, 2.0, 3.0])
    x, res, _ = ctx.lu_solve(A, b)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-14)


def test_lu_singular_reports_row(ctx):
    A = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 6.0], [1.0, 0.0, 1.0]])
    _, _, st, bad = O.lu_solve(A, np.ones(3))
    with pytest.raises(GbemError) as e:
        ctx.lu_solve(A, np.ones(3))
    assert e.value.code == 2 and f"smallest pivot at row {bad}" in str(e.value)


def _oracle_system(ps, regions, main_net):
    return O.assemble_collocation(ps.matrix(), ps.nsign, ps.kind, ps.net, ps.regA, ps.regB, regions, main_net)


@pytest.mark.parametrize("scene,net", [(TWO, 1), (TWO, 2), (SINGLE, 1)])
def test_collocation_system_matches_oracle(ctx, scene, net):
    m = g.parse_model(scene.read_text())
    ps = m.partition(0, net)
    A, b, x, res = ctx.assemble_collocation(ps, m.regions, net, solve=True)
    Ao, bo, st = _oracle_system(ps, m.regions, net)
    assert st == 0 and A.shape == Ao.shape
    scale = np.abs(Ao).max()
    assert np.abs(A - Ao).max() <= 1e-13 * scale
    assert np.abs(b - bo).max() <= 1e-13 * max(np.abs(bo).max(), 1.0)
    xo, ro, sto, _ = O.lu_solve(Ao, bo)
    assert sto == 0
    assert np.abs(x - xo).max() <= 1e-9 * np.abs(xo).max()
    assert res <= 1e-12


def _oracle_cmatrix(m):
    """capacitance_matrix with the collocation baseline, all on the CPU oracle."""
    ids = m.net_ids
    eps = dict(m.regions)
    C = np.zeros((len(ids), len(ids)))
    for r, net in enumerate(ids):
        ps = m.partition(0, net)
        A, b, st = _oracle_system(ps, m.regions, net)
        x, _, _, _ = O.lu_solve(A, b)
        for k in range(len(ps)):
            if ps.kind[k] == 0:  # conductor: qCol = k (extraction.hpp:55-79)
                C[r, ids.index(int(ps.net[k]))] += eps[int(ps.regA[k])] * EPS0 * x[k] * 1e-6
    return C


def test_two_layer_cmatrix_collocation_end_to_end(ctx):
    m = g.parse_model(TWO.read_text())
    csv, js = m.extract(net=-1, mode=0, baseline="collocation")
    assert js["baseline"] == "collocation"
    assert [r["method"] for r in js["rows"]] == ["collocation", "collocation"]
    Cg = m.last_cap
    Co = _oracle_cmatrix(m)
    assert np.abs(Cg - Co).max() <= 1e-9 * np.abs(Co).max(), (Cg, Co)
    assert Cg[0, 0] > 0 and Cg[1, 1] > 0 and Cg[0, 1] < 0 and Cg[1, 0] < 0
    assert "# method net1=collocation net2=collocation" in csv


def _oracle_multi(ps, regions, net):
    return O.assemble_multi(ps.matrix(), ps.nsign, ps.kind, ps.net, ps.regA, ps.regB, regions, net)


@pytest.mark.parametrize("scene,net", [(TWO, 1), (TWO, 2)])
def test_galerkin_block_system_matches_oracle(ctx, scene, net):
    """assemble_multi (assembly.hpp:110-175) on the GPU against the CPU restatement
    (its q_pair_integral pinned bit-for-bit to the compiled reference): same
    reductions and Romberg rule, warp-parallel sample sums."""
    m = g.parse_model(scene.read_text())
    ps = m.partition(0, net)
    A, b, conv, x, res = ctx.assemble_multi(ps, m.regions, net, solve=True)
    Ao, bo, st, convo = _oracle_multi(ps, m.regions, net)
    assert st == 0 and A.shape == Ao.shape and conv == convo
    # entries agree to the quadrature tolerance (relTol 1e-8); most bit-for-bit close
    d = np.abs(A - Ao)
    assert d.max() <= 1e-8 * np.abs(Ao).max(), d.max() / np.abs(Ao).max()
    assert np.median(d[Ao != 0] / np.abs(Ao[Ao != 0])) <= 1e-13
    assert np.abs(b - bo).max() <= 1e-8 * max(np.abs(bo).max(), 1.0)
    xo, ro, sto, _ = O.lu_solve(Ao, bo)
    assert sto == 0
    assert np.abs(x - xo).max() <= 1e-6 * np.abs(xo).max()
    assert res <= 1e-12


def _oracle_cmatrix_multi(m):
    """capacitance_matrix through the Galerkin block system, all on the CPU oracle."""
    ids = m.net_ids
    eps = dict(m.regions)
    C = np.zeros((len(ids), len(ids)))
    for r, net in enumerate(ids):
        ps = m.partition(0, net)
        A, b, st, _ = _oracle_multi(ps, m.regions, net)
        assert st == 0
        x, _, _, _ = O.lu_solve(A, b)
        for k in range(len(ps)):
            if ps.kind[k] == 0:
                C[r, ids.index(int(ps.net[k]))] += eps[int(ps.regA[k])] * EPS0 * x[k] * 1e-6
    return C


def test_two_layer_cmatrix_galerkin_end_to_end(ctx):
    """The reference's default path for a two-dielectric scene
    (capacitance_row -> assemble_multi -> lu_solve, extraction.hpp:132-143)."""
    m = g.parse_model(TWO.read_text())
    csv, js = m.extract(net=-1, mode=0)
    assert [r["method"] for r in js["rows"]] == ["galerkin-block", "galerkin-block"]
    Cg = m.last_cap
    Co = _oracle_cmatrix_multi(m)
    assert np.abs(Cg - Co).max() <= 1e-6 * np.abs(Co).max(), (Cg, Co)
    assert Cg[0, 0] > 0 and Cg[1, 1] > 0 and Cg[0, 1] < 0 and Cg[1, 0] < 0
    assert "# method net1=galerkin-block net2=galerkin-block" in csv
    # the Galerkin and collocation block systems agree to the discretisation level
    m.extract(net=-1, baseline="collocation")
    assert np.abs(m.last_cap - Cg).max() <= 0.1 * np.abs(Cg).max()


def test_collocation_single_region_agrees_with_galerkin(ctx):
    """Cross-method check (SPEC.md:522 in SURVEY §8f): on the single-dielectric
    benchmark the collocation C-matrix agrees with the Galerkin one to the
    discretisation level."""
    m = g.parse_model(SINGLE.read_text())
    m.extract(net=-1)
    Cg = m.last_cap.copy()
    m.extract(net=-1, baseline="collocation")
    Cc = m.last_cap
    assert np.abs(Cc - Cg).max() <= 0.1 * np.abs(Cg).max()


def test_kernel_selftest_on_device(ctx):
    """run_selftest (selftest.hpp:184-245) on the GPU: the ten geometric classes
    against the recursive brute-force oracle, at the reference's tolerances."""
    cases = ctx.selftest(pairs=200)
    assert [c["name"] for c in cases][:3] == ["U coplanar disjoint", "U coplanar adjacent", "U coplanar identical"]
    assert len(cases) == 10
    for c in cases:
        assert c["passed"], c
        assert c["pairs"] == 200
        # the report carries the class's worst pair for follow-up (tools/selftest_recheck.py)
        assert int(c["worst_test"][0]) in (0, 1, 2) and int(c["worst_source"][0]) in (0, 1, 2), c
        assert np.isfinite(c["worst_value"]) and np.isfinite(c["worst_oracle"]), c
        if c["name"].startswith("Q"):
            assert c["worst_nsign"] in (-1, 1), c
        if c["name"] != "Q coplanar zero":
            rel = abs(c["worst_value"] - c["worst_oracle"]) / max(abs(c["worst_oracle"]), 1e-9)
            assert abs(rel - c["worst_rel"]) <= 1e-6 * max(c["worst_rel"], 1e-12) + 1e-15, c


def test_kernel_selftest_cli():
    import subprocess
    cli = ROOT / "paper_2203_11733_b200" / "lib" / "gbem"
    r = subprocess.run([str(cli), "kernels", "selftest", "--pairs", "64"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 10 and all(l.endswith("PASS") for l in lines), r.stdout


@pytest.mark.parametrize("depth", [3, 4, 5, 6])
def test_device_oracle_pinned_to_reference_oracle(ctx, depth):
    """The on-device brute-force oracle (k_st_oracle, the selftest's truth) is
    the reference's oracle_pair_integral (oracle.hpp:191-205, compiled in
    oracle/_ref) value for value at a fixed depth: single layer on disjoint and
    touching pairs, double layer on disjoint pairs."""
    import pairgen as G
    from paper_2203_11733_b200._native import PanelArrays
    rng = np.random.default_rng(600 + depth)
    A, B = G.classic_pairs(rng, 40)
    if depth <= 5:
        At, Bt = G.touching_pairs(rng, 9 if depth < 5 else 3)
        A, B = np.vstack([A, At]), np.vstack([B, Bt])
    gpu = ctx.oracle_pair_integrals(PanelArrays.from_matrix(A), PanelArrays.from_matrix(B), depth)
    lib = O.ref()
    ra, rb = O.rects_from_matrix(A), O.rects_from_matrix(B)
    ref = np.array([lib.ref_oracle_pair_integral(ra[k], rb[k], depth) for k in range(len(A))])
    rel = np.abs(gpu - ref) / np.abs(ref)
    assert rel.max() <= 1e-12, (rel.argmax(), rel.max())
    # double layer (recQ, oracle.hpp:105-131): non-coplanar pairs, both normal signs
    m = ~((A[:, 0] == B[:, 0]) & (A[:, 1] == B[:, 1]))
    ns = np.where(rng.random(len(A)) < 0.5, 1, -1).astype(np.int32)
    gq = ctx.oracle_pair_integrals(PanelArrays.from_matrix(A[m]), PanelArrays.from_matrix(B[m]), depth,
                                   double_layer=True, nsign=ns[m])
    rq = O.q_oracle(A[m], B[m], ns[m], depth)
    scale = np.abs(rq).max()
    # (the double-layer leaves cancel: an absolute floor at 1e-12 of the set's largest value)
    assert np.all(np.abs(gq - rq) <= 1e-11 * np.abs(rq) + 1e-12 * scale), np.abs(gq - rq).max()
