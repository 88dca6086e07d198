"""End-to-end extraction on the GPU through the C++ host: reference scene file in,
capacitance matrix out (proj/README.md:78-84 golden), plus the extraction
properties of proj/tests/test_extraction.cpp and the CLI contract."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2203_11733_b200 as g

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
BENCH = ROOT / "tests" / "golden" / "bench_single.gbem"
CLI = ROOT / "paper_2203_11733_b200" / "lib" / "gbem"

# proj/README.md:80-84 (printed with %.9g)
README_C = np.array([[2.2471839e-16, -5.80121909e-17], [-5.72842648e-17, 1.80198011e-16]])


def test_benchmark_matrix_matches_readme_golden():
    m = g.parse_model(BENCH.read_text())
    csv, js = m.extract(net=-1, mode=0)
    C = np.array([[js["rows"][r]["capacitance"][str(k)] for k in (1, 2)] for r in range(2)])
    assert np.all(np.abs(C - README_C) <= 5e-9 * np.abs(README_C)), C
    assert [r["panels"] for r in js["rows"]] == [83, 56]
    assert "# panels net1=83 net2=56" in csv
    assert "# method net1=galerkin-single net2=galerkin-single" in csv
    for r in js["rows"]:
        assert r["residual"] <= 1e-10
        assert 0 <= r["neutrality"] <= 0.005
        assert r["outerCharge"] < 0


def test_benchmark_matrix_matches_cpu_oracle_pipeline():
    """Same panels (reference partition), CPU oracle assembly + dense solve."""
    m = g.parse_model(BENCH.read_text())
    _, js = m.extract(net=-1, mode=0)
    for r, net in enumerate((1, 2)):
        ps = g.partition_scene(m, net)
        A, conv, rc = O.assemble("orc", ps.matrix(), nthreads=8)
        b = ((ps.kind == 0) & (ps.net == net)).astype(float)
        x = np.linalg.solve(A, b)
        q = 1.0 * 8.854187817e-12 * x * 1e-6
        for k in (1, 2):
            ref = q[(ps.kind == 0) & (ps.net == k)].sum()
            got = js["rows"][r]["capacitance"][str(k)]
            assert abs(got - ref) <= 1e-9 * abs(ref)


def test_capacitance_scales_linearly_with_permittivity():
    """test_extraction.cpp:93-109: exact 2x."""
    base = ("domain lo(-6,-6,0) hi(6,6,6)\nregion 1 {eps} lo(-6,-6,0) hi(6,6,6)\n"
            "net 1 cuboid lo(-1,-0.5,1) hi(1,0.5,2)\nnet 2 cuboid lo(-0.5,-1,3) hi(0.5,1,4)\nparams 3 4 1 1\n")
    m1, m2 = g.parse_model(base.format(eps=1.0)), g.parse_model(base.format(eps=2.0))
    m1.extract(net=1)
    m2.extract(net=1)
    assert np.array_equal(m2.last_cap, 2.0 * m1.last_cap)  # bit-exact, like the reference
    assert np.array_equal(m2.last_outer, 2.0 * m1.last_outer)


def test_mirror_symmetric_scene():
    """test_extraction.cpp:111-132."""
    text = ("domain lo(-8,-8,0) hi(8,8,5)\nregion 1 1.0 lo(-8,-8,0) hi(8,8,5)\n"
            "net 1 cuboid lo(-3,-1,1) hi(-1,1,3)\nnet 2 cuboid lo(1,-1,1) hi(3,1,3)\n")
    js = g.capacitance_matrix(g.parse_model(text))
    c11, c12 = js["rows"][0]["capacitance"]["1"], js["rows"][0]["capacitance"]["2"]
    c21, c22 = js["rows"][1]["capacitance"]["1"], js["rows"][1]["capacitance"]["2"]
    assert abs(c22 - c11) <= 1e-9 * c11 and abs(c21 - c12) <= 1e-9 * abs(c12)
    assert js["reciprocityDefect"] <= 1e-9
    assert c11 > 0 and c12 <= 1e-3 * c11


def test_config1_shared_matches_oracle():
    m = g.config_model(1)
    ps = m.partition(1)
    _, js = m.extract(net=-1, mode=1)
    A, conv, rc = O.assemble("orc", ps.matrix(), nthreads=16)
    B = np.stack([(ps.net == 1), (ps.net == 2)], axis=1).astype(float)
    X = np.linalg.solve(A, B)
    for r in range(2):
        for k in (1, 2):
            ref = 3.9 * 8.854187817e-12 * 1e-6 * X[ps.net == k, r].sum()
            got = js["rows"][r]["capacitance"][str(k)]
            assert abs(got - ref) <= 1e-6 * abs(ref), (r, k, got, ref)


def test_cli_extract_and_exit_codes(tmp_path):
    out = subprocess.run([str(CLI), "extract", "--input", str(BENCH), "--all"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("# gbem 1.0.0\n# params p1=1.5 p2=4 p3=1 p5=1\n")
    assert "net,1,2" in out.stdout
    js = subprocess.run([str(CLI), "extract", "--input", str(BENCH), "--net", "1", "--format", "json"],
                        capture_output=True, text=True)
    assert js.returncode == 0 and '"method": "galerkin-single"' in js.stdout and '"seconds"' in js.stdout
    bad = subprocess.run([str(CLI), "extract", "--input", str(tmp_path / "missing.gbem")], capture_output=True, text=True)
    assert bad.returncode == 1 and "cannot open" in bad.stderr
    both = subprocess.run([str(CLI), "extract", "--input", str(BENCH), "--all", "--net", "1"], capture_output=True,
                          text=True)
    assert both.returncode == 1 and "mutually exclusive" in both.stderr


def test_matrix_dump_round_trip(tmp_path):
    """--dump-matrix writes extraction.hpp:83-99's format; it equals the assembled matrix bit for bit."""
    p = tmp_path / "A.bin"
    m = g.parse_model(BENCH.read_text())
    m.extract(net=1, mode=0, dump_matrix=str(p))
    blob = p.read_bytes()
    n = int.from_bytes(blob[:8], "little")
    A = np.frombuffer(blob[8:], dtype="<f8").reshape(n, n)
    ps = g.partition_scene(m, 1)
    sysm = g.assemble_single(ps)
    assert n == len(ps) and np.array_equal(A, sysm.A)


@pytest.mark.parametrize("K", [1, 3, 6, 8, 9, 12, 16, 17, 24, 33, 48, 64])
def test_bordered_extraction_every_solve_path(ctx, K):
    """gbem_extract_cmatrix's bordered factorisation (C = B^T A^-1 B from the
    border corner, X from the backward substitution) across the right-hand-side
    widths that select the dataflow (K <= 16) and the look-ahead cluster (17..64: every
    right-hand-side-per-thread instantiation) backward substitutions; n = 2,832 = 22 * 128 + 16 has a
    ragged last block and also runs the SM-partitioned factorisation (n >= 2 * 1024).  Reference: the GPU-assembled A
    solved densely by numpy."""
    m = g.config_model(1, scale=1.4)
    ps = m.partition(1)
    n = len(ps)
    rng = np.random.default_rng(K)
    net = rng.integers(0, K, size=n).astype(np.int32)
    net[:K] = np.arange(K)  # every net has a panel
    Cm, res, ast, sst = ctx.extract_cmatrix(ps.arrays(), net, K, 3.9)
    A, _ = ctx.assemble_single(ps.arrays())
    B = (net[:, None] == np.arange(K)[None, :]).astype(float)
    Cref = 3.9 * 8.854187817e-12 * 1e-6 * (B.T @ np.linalg.solve(A, B))
    assert np.abs(Cm - Cref).max() <= 1e-9 * np.abs(Cref).max(), np.abs(Cm - Cref).max()
    assert np.array_equal(Cm, Cm.T)  # Y^T Y: exactly symmetric
    assert res.max() <= 1e-12, res


@pytest.mark.parametrize("K", [1, 6, 9, 16, 17, 40])
def test_spd_solve_every_width(ctx, K):
    """cholesky_solve with K right-hand sides on an assembled Galerkin matrix
    (n = 2,832: the SM-partitioned factorisation), forward + backward
    substitution (cooperative up to 8 columns, DMMA-blocked above) against numpy."""
    m = g.config_model(1, scale=1.4)
    ps = m.partition(1)
    A, _ = ctx.assemble_single(ps.arrays())
    rng = np.random.default_rng(100 + K)
    B = rng.standard_normal((len(ps), K))
    ctx.matrix_upload(A)
    X, res, st = ctx.spd_solve(B)
    Xr = np.linalg.solve(A, B)
    assert np.abs(X - Xr).max() <= 1e-10 * np.abs(Xr).max()
    assert np.max(res) <= 1e-12


def test_extract_more_than_64_nets(ctx):
    """K > 64: the bordered factorisation carries any number of
    border rows; 100 panel groups as nets, C = eps B^T A^-1 B against numpy."""
    import paper_2203_11733_b200 as g
    from paper_2203_11733_b200._native import PanelArrays
    m = g.config_model(1, scale=0.5)
    ps = m.partition(1)
    P = ps.matrix()
    n = len(P)
    K = 100
    rng = np.random.default_rng(100)
    net = (np.arange(n) % K).astype(np.int32)
    rng.shuffle(net)
    Cm, res, _, _ = ctx.extract_cmatrix(PanelArrays.from_matrix(P), net, K, 3.9)
    A, _ = ctx.assemble_single(PanelArrays.from_matrix(P))
    Bm = (net[:, None] == np.arange(K)[None, :]).astype(float)
    Cref = 3.9 * 8.854187817e-12 * 1e-6 * Bm.T @ np.linalg.solve(A, Bm)
    assert np.abs(Cm - Cref).max() <= 1e-9 * np.abs(Cref).max()
    assert res.max() <= 1e-10


@pytest.mark.skipif(not O.REF_GPU_SO.exists(), reason="oracle/_ref/libgbem_ref_gpu.so not built")
def test_reference_side_binding_reproduces_readme():
    """INTEGRATION.md's gbem::GpuBackend compiled against the unmodified reference
    headers (oracle/ref_gpu_backend.cpp): the reference's own Scene and
    partition_scene (partition.hpp:214) per main net, assemble + Cholesky through
    gbem_assemble_single / gbem_spd_solve, net_charges restated — the README
    capacitance matrix (proj/README.md:78-84) and the host path's rows."""
    text = BENCH.read_text()
    m = g.parse_model(text)
    p = m.params
    params = (p["p1"], p["p2"], p["p3"], p["p5"]) if isinstance(p, dict) else tuple(p)
    rows, panels = [], []
    for net in (1, 2):
        q, outer, npan, res, conv = O.ref_gpu_capacitance_row(text, net, params)
        rows.append(q)
        panels.append(npan)
        assert res <= 1e-10 and outer < 0
    Cb = np.array(rows)
    assert panels == [83, 56]
    assert np.all(np.abs(Cb - README_C) <= 5e-9 * np.abs(README_C)), Cb
    _, js = m.extract(net=-1, mode=0)
    Ch = np.array([[js["rows"][r]["capacitance"][str(k)] for k in (1, 2)] for r in range(2)])
    assert np.all(np.abs(Cb - Ch) <= 1e-9 * np.abs(Ch))  # same panels, different summation order of the charges


def test_shared_mode_pcg_solver_matches_direct():
    """The C++ host runs the sharded solve (gbem_pcg_extract_cmatrix) from the
    shared mode: CLI --solver pcg against --solver direct on the same panels."""
    args = [str(CLI), "extract", "--input", str(BENCH), "--all", "--mode", "shared", "--graded", "0.05,1.5,0.3",
            "--format", "json"]
    rd = subprocess.run(args + ["--solver", "direct"], capture_output=True, text=True, timeout=600)
    rp = subprocess.run(args + ["--solver", "pcg", "--jacobi-blocks", "3", "--pcg-tol", "1e-12"],
                        capture_output=True, text=True, timeout=600)
    assert rd.returncode == 0 and rp.returncode == 0, (rd.stderr, rp.stderr)
    jd, jp = json.loads(rd.stdout), json.loads(rp.stdout)
    for a, b in zip(jd["rows"], jp["rows"]):  # reports carry 9 significant digits
        assert b["method"] == "galerkin-shared-pcg" and a["method"] == "galerkin-shared"
        self_c = abs(a["capacitance"][str(a["net"])])
        for k, v in a["capacitance"].items():
            assert abs(b["capacitance"][k] - v) <= 2e-8 * self_c, (k, v, b["capacitance"][k])
        assert abs(b["outerCharge"] - a["outerCharge"]) <= 2e-8 * self_c
        assert b["residual"] <= 1e-11
