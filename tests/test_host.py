"""C++ host (libgbem_host.so): scene grammar, validation, faces, the reference
partition reproduced panel for panel, the net-independent partitions and the
BASELINE config generators.  CPU only (no GPU calls)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2203_11733_b200 as g
from paper_2203_11733_b200.api import ValidationError

ROOT = Path(__file__).resolve().parents[1]
BENCH = ROOT / "tests" / "golden" / "bench_single.gbem"
TWO_LAYER = ROOT / "tests" / "golden" / "bench_two_layer.gbem"


def test_parse_minimal_scene():
    m = g.parse_model("# toy scene\ndomain lo(0,0,0) hi(10,10,10)\nregion 1 3.9 lo(0,0,0) hi(10,10,10)\n"
                      "net 7 cuboid lo(4,4,4) hi(6,6,6)\n")
    assert m.net_ids == [7]
    assert m.info()["eps_r"] == 3.9
    assert m.params == (1.5, 4.0, 1.0, 1.0)  # partition.hpp:15-30 defaults


@pytest.mark.parametrize("text,needles", [  # test_model_io.cpp:84-136
    ("domain lo(0,0,0) hi(4,4,4)\nregion 1 lo(0,0,0) hi(4,4,4)\n", ["region 1", "missing permittivity", "line 2"]),
    ("domain lo(0,0,0) hi(4,4,4)\nwidget 3\n", ["line 2", "unknown key"]),
    ("domain lo(0,0,0) hi(4,4,4)\ndomain lo(0,0,0) hi(4,4,4)\n", ["duplicate domain"]),
    ("domain lo(0,0,0) hi(4,4,4)\nregion 1 1 lo(0,0,0) hi(4,4,4)\nbc +z robin\n", ["line 3", "dirichlet or neumann"]),
    ("domain lo(0,0,0) hi(4,4,4)\nregion 1 1 lo(0,0,0) hi(4,4,4)\nbc top neumann\n", ["expected face"]),
    ("domain lo(0,0) hi(4,4,4)\n", ["lo(x,y,z)"]),
    ("domain lo(0,0,0) hi(4,4,4)\nregion 1 abc lo(0,0,0) hi(4,4,4)\n", ["permittivity"]),
    ("region 1 1 lo(0,0,0) hi(4,4,4)\n", ["no domain"]),
])
def test_parse_errors(text, needles):
    with pytest.raises(ValidationError) as e:
        g.parse_model(text)
    for nd in needles:
        assert nd in str(e.value)


@pytest.mark.parametrize("body,needle", [  # geometry.hpp:237-324 messages
    ("net 1 cuboid lo(1,1,1) hi(3,3,3)\nnet 2 cuboid lo(2,2,2) hi(4,4,4)\n", "overlap"),
    ("net 1 cuboid lo(1,1,1) hi(2,2,2)\nnet 2 cuboid lo(2,1,1) hi(3,2,2)\n", "positive contact area"),
    ("net 1 cuboid lo(1,1,1) hi(1,2,2)\n", "degenerate"),
    ("net 1 cuboid lo(-1,1,1) hi(2,2,2)\n", "strictly interior"),
])
def test_scene_validation(body, needle):
    with pytest.raises(ValidationError) as e:
        g.parse_model("domain lo(0,0,0) hi(8,8,8)\nregion 1 1 lo(0,0,0) hi(8,8,8)\n" + body)
    assert needle in str(e.value)


def test_dump_round_trip_is_a_fixed_point():
    m = g.parse_model(TWO_LAYER.read_text())
    m.set_params(p1=1.25, p3=0.75)
    t1 = m.dump()
    m2 = g.parse_model(t1)
    assert m2.params == m.params
    assert m2.dump() == t1


def test_faces_of_benchmark():
    m = g.parse_model(BENCH.read_text())
    assert m.info()["faces"] == 18  # 12 conductor faces + 6 outer


def _ref_partition(model_text, net, params):
    """Run the reference partition_scene (compiled in oracle/_ref) on the same scene."""
    m = g.parse_model(model_text)
    lines = [l.split("#")[0].split() for l in model_text.splitlines()]
    def pt(tok):
        return [float(v) for v in tok[tok.index("(") + 1:-1].split(",")]
    dom = regs = None
    regs, cells, bc = [], [], [0] * 6
    faces = {"-x": 0, "+x": 1, "-y": 2, "+y": 3, "-z": 4, "+z": 5}
    for t in lines:
        if not t:
            continue
        if t[0] == "domain":
            dom = pt(t[1]) + pt(t[2])
        elif t[0] == "region":
            regs += [float(t[1]), float(t[2])] + pt(t[3]) + pt(t[4])
        elif t[0] == "net":
            cells += [float(t[1])] + pt(t[3]) + pt(t[4])
        elif t[0] == "bc":
            bc[faces[t[1]]] = 1 if t[2] == "neumann" else 0
    dom = np.array(dom); regs = np.array(regs); cells = np.array(cells)
    bc = np.array(bc, dtype=np.int32); par = np.array(params, dtype=float)
    cap = 200000
    ints = np.zeros(6 * cap, np.int32); dbl = np.zeros(7 * cap); fac = np.zeros(cap, np.int32)
    err = C.create_string_buffer(512)
    n = O.ref().ref_partition_scene(dom.ctypes.data, len(regs) // 8, regs.ctypes.data, len(cells) // 7,
                                    cells.ctypes.data, bc.ctypes.data, par.ctypes.data, net, cap,
                                    ints.ctypes.data, dbl.ctypes.data, fac.ctypes.data, err, 512)
    assert n >= 0, err.value
    return ints[:6 * n].reshape(n, 6), dbl[:7 * n].reshape(n, 7), fac[:n]


SCENES = {
    "bench": BENCH.read_text(),
    "two_layer": TWO_LAYER.read_text(),
    "stacked": "domain lo(-6,-6,0) hi(6,6,6)\nregion 1 1 lo(-6,-6,0) hi(6,6,6)\n"
               "net 1 cuboid lo(-1,-1,1) hi(1,1,2)\nnet 1 cuboid lo(-0.5,-0.5,2) hi(0.5,0.5,3)\n"
               "net 2 cuboid lo(2,-1,1) hi(3,1,4)\nbc +z neumann\n",
}


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", list(SCENES))
@pytest.mark.parametrize("params", [(1.5, 4, 1, 1), (0.75, 2, 0.5, 0.5), (3.0, 4, 4, 1)])
def test_partition_matches_reference_panel_for_panel(name, params):
    text = SCENES[name]
    m = g.parse_model(text)
    m.set_params(*params)
    for net in m.net_ids:
        ps = g.partition_scene(m, net)
        ints, dbl, fac = _ref_partition(text, net, params)
        assert len(ps) == len(ints)
        assert np.array_equal(ps.axis, ints[:, 0]) and np.array_equal(ps.nsign, ints[:, 1])
        assert np.array_equal(ps.kind, ints[:, 2]) and np.array_equal(ps.net, ints[:, 3])
        assert np.array_equal(ps.regA, ints[:, 4]) and np.array_equal(ps.regB, ints[:, 5])
        mine = np.stack([ps.level, ps.a0, ps.a1, ps.b0, ps.b1, ps.area, ps.dist], axis=1)
        assert np.array_equal(mine, dbl)  # bit-identical coordinates
        assert np.array_equal(ps.facing, fac)


def test_benchmark_panel_counts():
    """README.md:78-84: 83 / 56 panels for nets 1 / 2."""
    m = g.parse_model(BENCH.read_text())
    assert len(g.partition_scene(m, 1)) == 83
    assert len(g.partition_scene(m, 2)) == 56


def test_partition_covers_boundary_and_honours_bounds():
    m = g.parse_model(BENCH.read_text())
    ps = g.partition_scene(m, 1)
    # faces: 2 conductors + 40x40x10 box
    conductor = 2 * 2 * (4 * 1 + 4 * 1 + 1 * 1)
    box = 2 * (40 * 40 + 40 * 10 + 40 * 10)
    assert abs(ps.area.sum() - (conductor + box)) <= 1e-12 * (conductor + box)
    p1, p2, p3, p5 = m.params
    bound = np.where(ps.dist <= p5, np.where(ps.facing == 2, p1 * p2, p1),
                     np.where(ps.facing == 2, p1 * p2, p1) * p3 * (np.maximum(ps.dist, 1e-300) / p5) ** 3)
    assert np.all(ps.area <= bound * (1 + 1e-9))
    la, lb = ps.a1 - ps.a0, ps.b1 - ps.b0
    assert np.all(np.maximum(la, lb) / np.minimum(la, lb) <= 4 * (1 + 1e-9))


def test_unknown_main_net():
    m = g.parse_model(BENCH.read_text())
    with pytest.raises(ValidationError, match="unknown main net"):
        g.partition_scene(m, 99)


def test_partition_explosion_guard():
    m = g.parse_model(BENCH.read_text())
    m.set_params(p1=1e-9, p3=1e-9)
    with pytest.raises(ValidationError, match="partition bound too small"):
        g.partition_scene(m, 1)


@pytest.mark.parametrize("cfg,n", [(1, 1344), (2, 11340), (3, 33776), (5, 200000)])
def test_config_panel_counts_are_pinned(cfg, n):
    m = g.config_model(cfg, seed=1)
    ps = m.partition(1)
    assert len(ps) == n
    ps2 = g.config_model(cfg, seed=1).partition(1)
    assert np.array_equal(ps.matrix(), ps2.matrix())  # deterministic


def test_config1_uniform_panels():
    ps = g.config_model(1).partition(1)
    la, lb = ps.a1 - ps.a0, ps.b1 - ps.b0
    assert np.allclose(la, 0.025) and np.allclose(lb, 0.025)
    assert sorted(set(ps.net.tolist())) == [1, 2]
    assert np.sum(ps.net == 1) == 672


def test_config2_graded_edges():
    ps = g.config_model(2).partition(1)
    la, lb = ps.a1 - ps.a0, ps.b1 - ps.b0
    assert abs(min(la.min(), lb.min()) - 0.005) < 1e-12
    assert max(la.max(), lb.max()) <= 0.05 + 1e-12
    # every conductor face tiled exactly: 6 wires 2.0 x 0.1 x 0.1
    assert abs(ps.area.sum() - 6 * (4 * 2.0 * 0.1 + 2 * 0.01)) < 1e-12


def test_config5_geometry():
    ps = g.config_model(5, seed=3, scale=0.01).partition(1)
    la, lb = ps.a1 - ps.a0, ps.b1 - ps.b0
    assert len(ps) == 2000
    assert la.min() >= 0.002 - 1e-15 and la.max() <= 0.2 + 1e-15
    assert np.all(np.abs(ps.level * 1000 - np.round(ps.level * 1000)) < 1e-6)


@pytest.mark.parametrize("cfg", [1, 2])
def test_config_panel_lists_match_golden_fixture(cfg):
    """The committed C-matrix fixtures were computed on exactly these panel lists."""
    import hashlib
    import json
    fx = json.loads((ROOT / "tests" / "golden" / f"config{cfg}_cmatrix.json").read_text())
    P = g.config_model(cfg, seed=fx["seed"]).partition(1).matrix()
    assert len(P) == fx["panels"]
    assert hashlib.sha256(np.ascontiguousarray(P).tobytes()).hexdigest() == fx["panels_sha256"]


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_serialised_workloads_match_generator(cfg):
    """workloads/config*_panels.npz (what bench.py --impl reference reads) are
    the host generator's panel lists bit for bit."""
    import paper_2203_11733_b200 as g
    d = np.load(ROOT / "workloads" / f"config{cfg}_panels.npz")
    m = g.config_model(cfg, seed=1)
    ps = m.partition(1)
    assert np.array_equal(d["panels"], ps.matrix())
    assert int(d["nets"]) == len(m.net_ids) and float(d["eps_r"]) == m.info()["eps_r"]


def test_bench_arms_report_the_same_config():
    """bench.py: the reference arm (serialised panel list, no repo library) and
    the GPU arm describe the workload with identical `config` objects."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    for cfg in (2, 3):
        P, net, K, eps, seed = bench.serialized_workload(cfg)
        m = g.config_model(cfg, seed=1)
        assert bench.extract_config(cfg, len(P), K, eps, seed) == bench.extract_config(
            cfg, len(m.partition(1)), len(m.net_ids), m.info()["eps_r"], 1)
    P4, _, K4, _, _ = bench.serialized_workload(4)
    assert bench.sharded_config(8, len(P4), K4, 200000)["unique_entries"] == 96200 * 96201 // 2
