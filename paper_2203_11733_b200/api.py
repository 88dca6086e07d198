"""Python mirror of the reference's public API for the single-dielectric path.

Names, argument meaning and error behaviour follow proj/include/gbem/*.hpp:
    Span, Rect                       geometry.hpp:21-76
    QuadratureConfig                 quadrature.hpp:12-15
    u_pair_integral(Ii, Ij, cfg)     kernels.hpp:270   -> GPU (gbem_u_pair_integrals)
    assemble_single(panels, cfg)     assembly.hpp:82   -> GPU (gbem_assemble_single)
    cholesky_solve(A, b)             solver.hpp:24     -> GPU (gbem_spd_solve)
    parse_model(text)                model_io.hpp:127  -> C++ host
    partition_scene(model, net)      partition.hpp:214 -> C++ host
    capacitance_matrix(model, ...)   extraction.hpp:162 -> C++ host driving the GPU
ValidationError / NumericalError mirror errors.hpp:10-20.  Everything here
calls the native libraries; there is no Python or CPU compute path.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


class ValidationError(ValueError):
    pass


class NumericalError(ArithmeticError):
    pass


def _raise(code: int, msg: str):
    if code == 1:
        raise ValidationError(msg)
    if code == 2:
        raise NumericalError(msg)
    raise RuntimeError(msg)


@dataclass(frozen=True)
class Span:
    lo: float
    hi: float

    def length(self) -> float:
        return self.hi - self.lo

    def mid(self) -> float:
        return 0.5 * (self.lo + self.hi)


@dataclass(frozen=True)
class Rect:
    axis: int
    level: float
    spanA: Span
    spanB: Span
    normalSign: int = 1

    def area(self) -> float:
        return self.spanA.length() * self.spanB.length()

    def row(self):
        return (self.axis, self.level, self.spanA.lo, self.spanA.hi, self.spanB.lo, self.spanB.hi)


def rect(axis, level, a, b, ns=1) -> Rect:
    return Rect(int(axis), float(level), Span(*map(float, a)), Span(*map(float, b)), ns)


@dataclass
class QuadratureConfig:
    relTol: float = 1e-8
    maxLevels: int = 16

    def native(self) -> N.GbemQuadConfig:
        return N.GbemQuadConfig(self.relTol, self.maxLevels, 0.0, 0.0)


@dataclass
class KernelValue:
    value: float
    converged: bool


_ctx: N.Context | None = None


def context(device: int = 0) -> N.Context:
    """Process-wide GPU context (one process per GPU)."""
    global _ctx
    if _ctx is None:
        try:
            _ctx = N.Context(device)
        except N.GbemError as e:
            _raise(e.code, str(e))
    return _ctx


def _panels(rects) -> N.PanelArrays:
    if isinstance(rects, np.ndarray):
        return N.PanelArrays.from_matrix(rects)
    return N.PanelArrays.from_matrix(np.array([r.row() for r in rects], dtype=float))


def _call(fn, *a):
    try:
        return fn(*a)
    except N.GbemError as e:
        _raise(e.code, str(e))


def u_pair_integral(Ii: Rect, Ij: Rect, cfg: QuadratureConfig | None = None) -> KernelValue:
    out, conv, _ = _call(context().u_pair_integrals, _panels([Ii]), _panels([Ij]), (cfg or QuadratureConfig()).native())
    return KernelValue(float(out[0]), bool(conv[0]))


def u_pair_integrals(I, J, cfg: QuadratureConfig | None = None):
    """Batched u_pair_integral over two equal-length panel lists (Rects or (n,6) arrays)."""
    out, conv, st = _call(context().u_pair_integrals, _panels(I), _panels(J), (cfg or QuadratureConfig()).native())
    return out, conv, st.as_dict()


@dataclass
class GalerkinSystem:
    A: np.ndarray
    b: np.ndarray
    allConverged: bool
    stats: dict = field(default_factory=dict)


@dataclass
class Solution:
    x: np.ndarray
    residualNorm: float
    method: str = "cholesky"


def assemble_single(panel_set: "PanelSet", cfg: QuadratureConfig | None = None) -> GalerkinSystem:
    """assembly.hpp:82-104 on the GPU; b_i = 1 on the main net's conductor panels."""
    if panel_set.count_kind(2) or panel_set.count_kind(3):
        raise ValidationError("single-dielectric assembly requires one region with an all-Dirichlet boundary")
    A, st = _call(context().assemble_single, panel_set.arrays(), (cfg or QuadratureConfig()).native())
    b = ((panel_set.kind == 0) & (panel_set.net == panel_set.main_net)).astype(float)
    return GalerkinSystem(A, b, st.not_converged == 0, st.as_dict())


def cholesky_solve(A: np.ndarray, b: np.ndarray) -> Solution:
    """solver.hpp:24-50 on the GPU (blocked Cholesky, DMMA trailing update)."""
    A = np.asarray(A, dtype=float)
    b = np.asarray(b, dtype=float)
    if A.ndim != 2 or A.shape[0] != A.shape[1] or b.shape[0] != A.shape[0]:
        raise ValidationError("cholesky_solve: dimension mismatch")
    ctx = context()
    _call(ctx.matrix_upload, A)
    x, res, st = _call(ctx.spd_solve, b)
    return Solution(x, float(np.max(res)) if res.size else 0.0)


# ------------------------------------------------------------------ host library

_host = None


def host_lib() -> C.CDLL:
    global _host
    if _host is None:
        N.gpu_lib()  # resolve libgbem_gpu first (libgbem_host links it via $ORIGIN)
        path = N.LIB_DIR / "libgbem_host.so"
        if not path.exists():
            raise ImportError(f"{path} missing: run `python -m paper_2203_11733_b200.build`")
        L = C.CDLL(str(path))
        P = C.c_void_p
        sig = {
            "gbem_model_parse": (C.c_int, [C.c_char_p, C.POINTER(P), C.c_char_p, C.c_int]),
            "gbem_model_config": (C.c_int, [C.c_int, C.c_uint64, C.c_double, C.POINTER(P), C.c_char_p, C.c_int]),
            "gbem_model_free": (None, [P]),
            "gbem_model_dump": (C.c_int64, [P, C.c_char_p, C.c_int64]),
            "gbem_model_nets": (C.c_int, [P, P, C.c_int]),
            "gbem_model_regions": (C.c_int, [P, P, P, C.c_int]),
            "gbem_model_info": (C.c_int, [P, P, P, P, P]),
            "gbem_model_params": (C.c_int, [P, P]),
            "gbem_model_set_params": (C.c_int, [P, P, C.c_char_p, C.c_int]),
            "gbem_model_partition": (C.c_int64, [P, C.c_int, C.c_int32, P, C.c_char_p, C.c_int]),
            "gbem_model_panels": (C.c_int, [P] * 15),
            "gbem_model_extract": (C.c_int, [P, P, C.c_char_p, C.c_int64, P, C.c_char_p, C.c_int64, P,
                                             C.c_char_p, C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _host = L
    return _host


HOST_SYMBOLS = ["gbem_model_parse", "gbem_model_config", "gbem_model_free", "gbem_model_dump", "gbem_model_nets",
                "gbem_model_regions",
                "gbem_model_info", "gbem_model_params", "gbem_model_set_params", "gbem_model_partition",
                "gbem_model_panels", "gbem_model_extract"]


class ExtractOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("mode", C.c_int32), ("net", C.c_int32), ("rel_tol", C.c_double),
                ("max_levels", C.c_int32), ("dump_matrix", C.c_char_p), ("cap_out", C.c_void_p),
                ("outer_out", C.c_void_p), ("collocation", C.c_int32), ("solver", C.c_int32),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("nccl_id_file", C.c_char_p),
                ("jacobi_blocks", C.c_int32), ("pcg_tol", C.c_double)]


@dataclass
class PanelSet:
    """Panel list (partition.hpp:45-58) as arrays; rows = matrix rows."""
    axis: np.ndarray
    level: np.ndarray
    a0: np.ndarray
    a1: np.ndarray
    b0: np.ndarray
    b1: np.ndarray
    nsign: np.ndarray
    kind: np.ndarray
    net: np.ndarray
    regA: np.ndarray
    regB: np.ndarray
    area: np.ndarray
    dist: np.ndarray
    facing: np.ndarray
    main_net: int = -1

    def __len__(self):
        return len(self.axis)

    def count_kind(self, k: int) -> int:
        return int(np.sum(self.kind == k))

    def matrix(self) -> np.ndarray:
        return np.stack([self.axis.astype(float), self.level, self.a0, self.a1, self.b0, self.b1], axis=1)

    def arrays(self) -> N.PanelArrays:
        return N.PanelArrays(self.axis, self.level, self.a0, self.a1, self.b0, self.b1)


class Model:
    """Parsed scene + partition parameters (model_io.hpp ParsedModel), owned by the C++ host."""

    def __init__(self, handle):
        self.h = handle
        self.L = host_lib()

    def __del__(self):
        try:
            if self.h:
                self.L.gbem_model_free(self.h)
        except Exception:
            pass

    def dump(self) -> str:
        n = self.L.gbem_model_dump(self.h, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.L.gbem_model_dump(self.h, buf, n + 1)
        return buf.value.decode()

    @property
    def net_ids(self) -> list[int]:
        k = self.L.gbem_model_nets(self.h, None, 0)
        ids = np.zeros(max(k, 1), dtype=np.int32)
        self.L.gbem_model_nets(self.h, ids.ctypes.data, k)
        return [int(v) for v in ids[:k]]

    @property
    def regions(self) -> list[tuple[int, float]]:
        """[(region id, relative permittivity)], ascending id."""
        k = self.L.gbem_model_regions(self.h, None, None, 0)
        ids = np.zeros(max(k, 1), dtype=np.int32)
        eps = np.zeros(max(k, 1))
        self.L.gbem_model_regions(self.h, ids.ctypes.data, eps.ctypes.data, k)
        return [(int(ids[i]), float(eps[i])) for i in range(k)]

    def info(self) -> dict:
        nr, nf, fs = C.c_int32(), C.c_int32(), C.c_int32()
        eps = C.c_double()
        self.L.gbem_model_info(self.h, C.byref(nr), C.byref(nf), C.byref(eps), C.byref(fs))
        return {"regions": nr.value, "faces": nf.value, "eps_r": eps.value, "freespace": bool(fs.value)}

    @property
    def params(self) -> tuple:
        p = np.zeros(4)
        self.L.gbem_model_params(self.h, p.ctypes.data)
        return tuple(float(v) for v in p)

    def set_params(self, p1=None, p2=None, p3=None, p5=None):
        cur = list(self.params)
        for i, v in enumerate((p1, p2, p3, p5)):
            if v is not None:
                cur[i] = v
        arr = np.array(cur, dtype=float)
        err = C.create_string_buffer(512)
        rc = self.L.gbem_model_set_params(self.h, arr.ctypes.data, err, 512)
        if rc:
            _raise(rc, err.value.decode())

    def partition(self, mode: int, main_net: int = -1, args=None) -> PanelSet:
        err = C.create_string_buffer(1024)
        a = np.asarray(args if args is not None else [0.0], dtype=float)
        n = self.L.gbem_model_partition(self.h, mode, main_net, a.ctypes.data, err, 1024)
        if n < 0:
            _raise(1, err.value.decode())
        n = int(n)
        arrs = dict(axis=np.zeros(n, np.uint8), level=np.zeros(n), a0=np.zeros(n), a1=np.zeros(n), b0=np.zeros(n),
                    b1=np.zeros(n), nsign=np.zeros(n, np.int32), kind=np.zeros(n, np.int32), net=np.zeros(n, np.int32),
                    regA=np.zeros(n, np.int32), regB=np.zeros(n, np.int32), area=np.zeros(n), dist=np.zeros(n),
                    facing=np.zeros(n, np.int32))
        self.L.gbem_model_panels(self.h, *[arrs[k].ctypes.data for k in arrs])
        return PanelSet(**arrs, main_net=main_net)

    def extract(self, net: int = -1, mode: int = 0, device: int = 0, dump_matrix: str | None = None,
                rel_tol: float = 1e-8, max_levels: int = 16, baseline: str | None = None, solver: int = 0,
                jacobi_blocks: int = 1, pcg_tol: float = 1e-10) -> tuple[str, dict]:
        """Run capacitance_matrix (net=-1) or capacitance_row; returns (csv, json dict).
        Shared mode (mode=1): solver 0 auto / 1 direct / 2 block-Jacobi PCG.
        Full-precision values are left in self.last_cap (rows x nets) / self.last_outer."""
        ids = self.net_ids
        rows = 1 if net >= 0 else len(ids)
        self.last_cap = np.zeros((rows, len(ids)))
        self.last_outer = np.zeros(rows)
        if baseline not in (None, "collocation"):
            raise ValidationError("baseline must be 'collocation'")
        o = ExtractOpts(device, mode, net, rel_tol, max_levels, dump_matrix.encode() if dump_matrix else None,
                        self.last_cap.ctypes.data, self.last_outer.ctypes.data, 1 if baseline else 0, solver,
                        1, 0, None, jacobi_blocks, pcg_tol)
        cap = 1 << 20
        csv, js = C.create_string_buffer(cap), C.create_string_buffer(cap)
        cl, jl = C.c_int64(), C.c_int64()
        err = C.create_string_buffer(1024)
        rc = self.L.gbem_model_extract(self.h, C.byref(o), csv, cap, C.byref(cl), js, cap, C.byref(jl), err, 1024)
        if rc:
            _raise(rc, err.value.decode())
        return csv.value.decode(), json.loads(js.value.decode())


def parse_model(text: str) -> Model:
    L = host_lib()
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    rc = L.gbem_model_parse(text.encode(), C.byref(h), err, 1024)
    if rc:
        _raise(rc, err.value.decode())
    return Model(h)


def config_model(config: int, seed: int = 1, scale: float = 1.0) -> Model:
    """Synthetic BASELINE.json config (1..5) with its net-independent panel set."""
    L = host_lib()
    h = C.c_void_p()
    err = C.create_string_buffer(1024)
    rc = L.gbem_model_config(config, seed, scale, C.byref(h), err, 1024)
    if rc:
        _raise(rc, err.value.decode())
    return Model(h)


def partition_scene(model: Model, main_net: int) -> PanelSet:
    """partition.hpp:214 for one main net (reference panel order)."""
    return model.partition(0, main_net)


def capacitance_matrix(model: Model, **kw) -> dict:
    """extraction.hpp:162-184 (per-main-net partitions, one GPU solve per net)."""
    return model.extract(net=-1, mode=0, **kw)[1]


def capacitance_row(model: Model, main_net: int, **kw) -> dict:
    return model.extract(net=main_net, mode=0, **kw)[1]["rows"][0]
