"""ctypes bindings of the native libraries (include/gbem_gpu.h, include/gbem_host.h).

The product path is native only: if a library is missing the import of the
bound function raises, there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "lib"

GBEM_OK, GBEM_EINVAL, GBEM_ENUMERIC, GBEM_ECUDA = 0, 1, 2, 3


class GbemPanels(C.Structure):
    _fields_ = [("axis", C.POINTER(C.c_uint8)), ("level", C.POINTER(C.c_double)),
                ("a_lo", C.POINTER(C.c_double)), ("a_hi", C.POINTER(C.c_double)),
                ("b_lo", C.POINTER(C.c_double)), ("b_hi", C.POINTER(C.c_double))]


class GbemQuadConfig(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_levels", C.c_int32),
                ("near_ratio", C.c_double), ("far_tol", C.c_double)]


class GbemSelftestCase(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("pairs", C.c_int32), ("worst_rel", C.c_double), ("tol", C.c_double),
                ("pass_", C.c_int32), ("worst_test", C.c_double * 6), ("worst_source", C.c_double * 6),
                ("worst_nsign", C.c_int32), ("worst_value", C.c_double), ("worst_oracle", C.c_double)]


class GbemAssemblyStats(C.Structure):
    _fields_ = [("pairs_total", C.c_int64), ("pairs_coplanar", C.c_int64),
                ("pairs_parallel", C.c_int64), ("pairs_orthogonal", C.c_int64),
                ("pairs_far", C.c_int64), ("not_converged", C.c_int64),
                ("nonfinite", C.c_int64), ("near_evals", C.c_int64), ("far_evals", C.c_int64),
                ("far_flops", C.c_double), ("ms_classify", C.c_double), ("ms_far", C.c_double),
                ("ms_near", C.c_double), ("ms_total", C.c_double),
                ("pairs_near_romberg", C.c_int64), ("pairs_near_band", C.c_int64 * 4)]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["pairs_near_band"] = list(d["pairs_near_band"])
        return d


class GbemBlockPanels(C.Structure):
    _fields_ = [("geom", GbemPanels), ("nsign", C.c_void_p), ("kind", C.c_void_p), ("net", C.c_void_p),
                ("reg_a", C.c_void_p), ("reg_b", C.c_void_p)]


class GbemRegion(C.Structure):
    _fields_ = [("id", C.c_int32), ("eps", C.c_double)]


class GbemSolveStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nrhs", C.c_int64), ("bad_pivot", C.c_int64),
                ("max_residual", C.c_double), ("ms_factor", C.c_double),
                ("ms_solve", C.c_double), ("ms_residual", C.c_double)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


AllGatherFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
AllReduceFn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class GbemCollectives(C.Structure):
    _fields_ = [("user", C.c_void_p), ("all_gather", AllGatherFn), ("all_reduce_sum", AllReduceFn)]


class GbemPcgOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int32), ("jacobi_blocks", C.c_int32)]


class GbemPcgStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("rows_local", C.c_int64), ("row_begin", C.c_int64),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("iterations", C.c_int32), ("converged", C.c_int32),
                ("max_rel_resid", C.c_double), ("ms_assembly", C.c_double), ("ms_precond", C.c_double),
                ("ms_iterations", C.c_double), ("ms_matvec", C.c_double), ("ms_total", C.c_double),
                ("matvec_flops", C.c_double)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


# (name, restype, argtypes) for every symbol of include/gbem_gpu.h
_P = C.c_void_p
GPU_SYMBOLS = [
    ("gbem_ctx_create", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("gbem_ctx_destroy", None, [_P]),
    ("gbem_last_error", C.c_char_p, [_P]),
    ("gbem_ctx_set_stream", C.c_int, [_P, _P]),
    ("gbem_ctx_set_async", C.c_int, [_P, C.c_int]),
    ("gbem_ctx_sync", C.c_int, [_P]),
    ("gbem_ctx_launch_count", C.c_int64, [_P]),
    ("gbem_u_pair_integrals", C.c_int, [_P, C.POINTER(GbemPanels), C.POINTER(GbemPanels), C.c_int64,
                                        C.POINTER(GbemQuadConfig), _P, _P, C.POINTER(GbemAssemblyStats)]),
    ("gbem_assemble_single", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, C.POINTER(GbemQuadConfig),
                                       _P, C.c_int64, C.POINTER(GbemAssemblyStats)]),
    ("gbem_assemble_single_dev", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, C.POINTER(GbemQuadConfig),
                                           C.POINTER(GbemAssemblyStats)]),
    ("gbem_assemble_rows_dev", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, C.c_int64, C.c_int64,
                                         C.POINTER(GbemQuadConfig), _P, C.c_int64, C.POINTER(GbemAssemblyStats)]),
    ("gbem_assemble_rows_full_dev", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, C.c_int64, C.c_int64,
                                              C.POINTER(GbemQuadConfig), _P, C.c_int64, C.POINTER(GbemAssemblyStats)]),
    ("gbem_rowblock_matvec_dev", C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int64, _P, C.c_int64, C.c_int64, _P,
                                           C.c_int64]),
    ("gbem_spd_factor_dev", C.c_int, [_P, _P, C.c_int64, C.c_int64, C.POINTER(GbemSolveStats)]),
    ("gbem_matrix_apply_dev", C.c_int, [_P, _P, C.c_int64, _P]),
    ("gbem_spd_solve_factored_dev", C.c_int, [_P, _P, C.c_int64, _P, _P, C.POINTER(GbemSolveStats)]),
    ("gbem_assemble_collocation", C.c_int, [_P, C.POINTER(GbemBlockPanels), C.c_int64, C.POINTER(GbemRegion),
                                            C.c_int32, C.c_int32, _P, C.c_int64, _P, C.POINTER(C.c_int64)]),
    ("gbem_assemble_multi", C.c_int, [_P, C.POINTER(GbemBlockPanels), C.c_int64, C.POINTER(GbemRegion),
                                      C.c_int32, C.c_int32, C.POINTER(GbemQuadConfig), _P, C.c_int64, _P,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    ("gbem_lu_solve", C.c_int, [_P, _P, _P, _P, C.POINTER(GbemSolveStats)]),
    ("gbem_selftest", C.c_int, [_P, C.c_int32, C.c_uint64, C.POINTER(GbemQuadConfig), C.POINTER(GbemSelftestCase),
                                C.POINTER(C.c_int32)]),
    ("gbem_matrix_upload_general", C.c_int, [_P, _P, C.c_int64, C.c_int64]),
    ("gbem_matrix_download", C.c_int, [_P, _P, C.c_int64]),
    ("gbem_matrix_upload", C.c_int, [_P, _P, C.c_int64, C.c_int64]),
    ("gbem_matrix_device", C.c_int, [_P, C.POINTER(_P), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("gbem_spd_solve", C.c_int, [_P, _P, C.c_int64, _P, _P, C.POINTER(GbemSolveStats)]),
    ("gbem_spd_solve_dev", C.c_int, [_P, _P, C.c_int64, _P, _P, C.POINTER(GbemSolveStats)]),
    ("gbem_net_charges_dev", C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int32, C.c_double, _P, _P]),
    ("gbem_extract_cmatrix", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, _P, C.c_int32, C.c_double,
                                       C.POINTER(GbemQuadConfig), _P, _P, C.POINTER(GbemAssemblyStats),
                                       C.POINTER(GbemSolveStats)]),
    ("gbem_debug_fill_shared", C.c_int, [_P, C.c_double]),
    ("gbem_oracle_pair_integrals", C.c_int, [_P, C.POINTER(GbemPanels), C.POINTER(GbemPanels), _P, C.c_int64,
                                             C.c_int32, C.c_int32, _P]),
    ("gbem_nccl_unique_id", C.c_int, [_P]),
    ("gbem_ctx_init_nccl", C.c_int, [_P, C.c_int32, C.c_int32, _P]),
    ("gbem_ctx_set_collectives", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(GbemCollectives)]),
    ("gbem_pcg_extract_cmatrix_dev", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, _P, C.c_int32, C.c_double,
                                               C.POINTER(GbemQuadConfig), C.POINTER(GbemPcgOptions), _P, _P, _P,
                                               C.POINTER(GbemAssemblyStats), C.POINTER(GbemPcgStats)]),
    ("gbem_pcg_extract_cmatrix", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, _P, C.c_int32, C.c_double,
                                           C.POINTER(GbemQuadConfig), C.POINTER(GbemPcgOptions), _P, _P, _P,
                                           C.POINTER(GbemAssemblyStats), C.POINTER(GbemPcgStats)]),
    ("gbem_ctx_nranks", C.c_int32, [_P]),
    ("gbem_ctx_rank", C.c_int32, [_P]),
    ("gbem_extract_cmatrix_dev", C.c_int, [_P, C.POINTER(GbemPanels), C.c_int64, _P, C.c_int32, C.c_double,
                                           C.POINTER(GbemQuadConfig), _P, _P, C.POINTER(GbemAssemblyStats),
                                           C.POINTER(GbemSolveStats)]),
]

_gpu = None


def gpu_lib() -> C.CDLL:
    """Load libgbem_gpu.so (raises if it has not been built)."""
    global _gpu
    if _gpu is None:
        path = LIB_DIR / "libgbem_gpu.so"
        if not path.exists():
            raise ImportError(f"{path} missing: run `python -m paper_2203_11733_b200.build`")
        lib = C.CDLL(str(path))
        for name, res, args in GPU_SYMBOLS:
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _gpu = lib
    return _gpu


def ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class PanelArrays:
    """Contiguous SoA copies of a panel list + the gbem_panels view onto them."""

    def __init__(self, axis, level, a0, a1, b0, b1):
        self.axis = np.ascontiguousarray(axis, dtype=np.uint8)
        self.level = np.ascontiguousarray(level, dtype=np.float64)
        self.a0 = np.ascontiguousarray(a0, dtype=np.float64)
        self.a1 = np.ascontiguousarray(a1, dtype=np.float64)
        self.b0 = np.ascontiguousarray(b0, dtype=np.float64)
        self.b1 = np.ascontiguousarray(b1, dtype=np.float64)
        self.n = len(self.axis)

    @classmethod
    def from_matrix(cls, m: np.ndarray) -> "PanelArrays":
        """m: (n, 6) = axis, level, a0, a1, b0, b1."""
        m = np.asarray(m, dtype=np.float64)
        return cls(m[:, 0].astype(np.uint8), m[:, 1], m[:, 2], m[:, 3], m[:, 4], m[:, 5])

    def struct(self) -> GbemPanels:
        d = C.POINTER(C.c_double)
        return GbemPanels(self.axis.ctypes.data_as(C.POINTER(C.c_uint8)), self.level.ctypes.data_as(d),
                          self.a0.ctypes.data_as(d), self.a1.ctypes.data_as(d),
                          self.b0.ctypes.data_as(d), self.b1.ctypes.data_as(d))


class GbemError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Context:
    """One gbem_ctx on one CUDA device (one process per GPU)."""

    def __init__(self, device: int = 0):
        self.lib = gpu_lib()
        h = _P()
        rc = self.lib.gbem_ctx_create(device, C.byref(h))
        self.h = h
        if rc != GBEM_OK:
            msg = self.lib.gbem_last_error(h).decode() if h else "context creation failed"
            if h:
                self.lib.gbem_ctx_destroy(h)
            self.h = None
            raise GbemError(rc, msg)

    def close(self):
        if self.h:
            self.lib.gbem_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc != GBEM_OK:
            raise GbemError(rc, self.lib.gbem_last_error(self.h).decode())

    @property
    def launches(self) -> int:
        return int(self.lib.gbem_ctx_launch_count(self.h))

    def set_stream(self, stream_handle: int | None):
        """Order this context's work on a framework stream.  A handle of 0 is the
        legacy default stream (torch's default stream), passed as cudaStreamLegacy;
        None returns to the context's own stream."""
        h = None if stream_handle is None else (stream_handle or 1)
        self.check(self.lib.gbem_ctx_set_stream(self.h, _P(h)))

    @staticmethod
    def quad(rel_tol=1e-8, max_levels=16, near_ratio=1.0, far_tol=1e-12) -> GbemQuadConfig:
        return GbemQuadConfig(rel_tol, max_levels, near_ratio, far_tol)

    def u_pair_integrals(self, I: PanelArrays, J: PanelArrays, cfg: GbemQuadConfig | None = None):
        n = I.n
        out = np.zeros(n)
        conv = np.zeros(n, dtype=np.int32)
        st = GbemAssemblyStats()
        si, sj = I.struct(), J.struct()
        rc = self.lib.gbem_u_pair_integrals(self.h, C.byref(si), C.byref(sj), n,
                                            C.byref(cfg or self.quad()), ptr(out), ptr(conv), C.byref(st))
        self.check(rc)
        return out, conv.astype(bool), st

    def assemble_single(self, P: PanelArrays, cfg: GbemQuadConfig | None = None, download: bool = True):
        n = P.n
        A = np.empty((n, n)) if download else None
        st = GbemAssemblyStats()
        sp = P.struct()
        rc = self.lib.gbem_assemble_single(self.h, C.byref(sp), n, C.byref(cfg or self.quad()),
                                           ptr(A) if download else None, n, C.byref(st))
        self.check(rc)
        return A, st

    def extract_cmatrix(self, P: PanelArrays, net_of_panel: np.ndarray, K: int, eps_r: float,
                        cfg: GbemQuadConfig | None = None, stats: bool = True):
        """Host-buffer C-matrix extraction (assemble + factor + K solves + charges)."""
        net = np.ascontiguousarray(net_of_panel, dtype=np.int32)
        Cm = np.zeros((K, K))
        res = np.zeros(K)
        ast, sst = GbemAssemblyStats(), GbemSolveStats()
        sp = P.struct()
        rc = self.lib.gbem_extract_cmatrix(self.h, C.byref(sp), P.n, ptr(net), K, eps_r, C.byref(cfg or self.quad()),
                                           ptr(Cm), ptr(res), C.byref(ast) if stats else None,
                                           C.byref(sst) if stats else None)
        self.check(rc)
        return Cm, res, ast, sst

    def oracle_pair_integrals(self, I: PanelArrays, J: PanelArrays, depth: int, double_layer: bool = False,
                              nsign: np.ndarray | None = None) -> np.ndarray:
        """oracle_pair_integral (oracle.hpp:191) on the device, per pair."""
        out = np.zeros(I.n)
        ns = None if nsign is None else np.ascontiguousarray(nsign, dtype=np.int32)
        si, sj = I.struct(), J.struct()
        self.check(self.lib.gbem_oracle_pair_integrals(self.h, C.byref(si), C.byref(sj),
                                                       None if ns is None else ptr(ns), I.n,
                                                       1 if double_layer else 0, depth, ptr(out)))
        return out

    def fill_shared(self, value: float):
        """Diagnostic: leave `value` in every SM's shared memory."""
        self.check(self.lib.gbem_debug_fill_shared(self.h, value))

    def matrix_upload(self, A: np.ndarray):
        A = np.ascontiguousarray(A, dtype=np.float64)
        self.check(self.lib.gbem_matrix_upload(self.h, ptr(A), A.shape[0], A.shape[1]))

    def matrix_download(self, n: int) -> np.ndarray:
        A = np.empty((n, n))
        self.check(self.lib.gbem_matrix_download(self.h, ptr(A), n))
        return A

    def lu_solve(self, A: np.ndarray, b: np.ndarray):
        """lu_solve (solver.hpp:53-88) of a general matrix: (x, residual, stats)."""
        A = np.ascontiguousarray(A, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = len(b)
        self.check(self.lib.gbem_matrix_upload_general(self.h, ptr(A), n, A.shape[1]))
        x = np.zeros(n)
        res = np.zeros(1)
        st = GbemSolveStats()
        self.check(self.lib.gbem_lu_solve(self.h, ptr(b), ptr(x), ptr(res), C.byref(st)))
        return x, float(res[0]), st

    def assemble_collocation(self, ps, regions, main_net: int, solve: bool = False):
        """assemble_collocation (assembly.hpp:179-227) for an api.PanelSet and
        regions [(id, eps), ...]: (A (m, m) row-major, b (m,)) and, with solve,
        also the lu_solve solution and residual."""
        P = PanelArrays(ps.axis, ps.level, ps.a0, ps.a1, ps.b0, ps.b1)
        keep = [np.ascontiguousarray(ps.nsign, dtype=np.int8)] + [
            np.ascontiguousarray(v, dtype=np.int32) for v in (ps.kind, ps.net, ps.regA, ps.regB)]
        bp = GbemBlockPanels(P.struct(), *[ptr(v) for v in keep])
        regs = (GbemRegion * len(regions))(*[GbemRegion(int(i), float(e)) for i, e in regions])
        m = C.c_int64(0)
        self.check(self.lib.gbem_assemble_collocation(self.h, C.byref(bp), P.n, regs, len(regions), int(main_net),
                                                      None, 0, None, C.byref(m)))
        mm = m.value
        A = np.zeros((mm, mm))
        b = np.zeros(mm)
        self.check(self.lib.gbem_assemble_collocation(self.h, C.byref(bp), P.n, regs, len(regions), int(main_net),
                                                      ptr(A), mm, ptr(b), C.byref(m)))
        if not solve:
            return A, b
        x = np.zeros(mm)
        res = np.zeros(1)
        st = GbemSolveStats()
        self.check(self.lib.gbem_lu_solve(self.h, None, ptr(x), ptr(res), C.byref(st)))
        return A, b, x, float(res[0])

    def assemble_multi(self, ps, regions, main_net: int, solve: bool = False, cfg=None):
        """assemble_multi (assembly.hpp:110-175), the Galerkin block system, for an
        api.PanelSet and regions [(id, eps), ...]: (A (m, m) row-major, b (m,),
        all_converged) and, with solve, also the lu_solve solution and residual."""
        P = PanelArrays(ps.axis, ps.level, ps.a0, ps.a1, ps.b0, ps.b1)
        keep = [np.ascontiguousarray(ps.nsign, dtype=np.int8)] + [
            np.ascontiguousarray(v, dtype=np.int32) for v in (ps.kind, ps.net, ps.regA, ps.regB)]
        bp = GbemBlockPanels(P.struct(), *[ptr(v) for v in keep])
        regs = (GbemRegion * len(regions))(*[GbemRegion(int(i), float(e)) for i, e in regions])
        m = C.c_int64(0)
        conv = C.c_int32(0)
        q = cfg or self.quad()
        mmax = P.n + int(np.sum(keep[1] == 3))  # rows: panels + interfaces (two unknowns each)
        Abuf = np.zeros((mmax, mmax))
        bbuf = np.zeros(mmax)
        # the system stays in the context (for gbem_lu_solve); a row-major copy comes back
        self.check(self.lib.gbem_assemble_multi(self.h, C.byref(bp), P.n, regs, len(regions), int(main_net),
                                                C.byref(q), ptr(Abuf), mmax, ptr(bbuf), C.byref(m), C.byref(conv)))
        mm = m.value
        A = np.ascontiguousarray(Abuf[:mm, :mm])
        b = bbuf[:mm].copy()
        if not solve:
            return A, b, bool(conv.value)
        x = np.zeros(mm)
        res = np.zeros(1)
        st = GbemSolveStats()
        self.check(self.lib.gbem_lu_solve(self.h, None, ptr(x), ptr(res), C.byref(st)))
        return A, b, bool(conv.value), x, float(res[0])

    def selftest(self, pairs: int = 500, seed: int = 20260817):
        """run_selftest (selftest.hpp:184-245) on the GPU: [{name, pairs, worst_rel, tol, pass}] x 10."""
        cases = (GbemSelftestCase * 10)()
        nc = C.c_int32(0)
        self.check(self.lib.gbem_selftest(self.h, int(pairs), int(seed), C.byref(self.quad()), cases, C.byref(nc)))
        return [dict(name=c.name.decode(), pairs=c.pairs, worst_rel=c.worst_rel, tol=c.tol, passed=bool(c.pass_),
                     worst_test=list(c.worst_test), worst_source=list(c.worst_source), worst_nsign=c.worst_nsign,
                     worst_value=c.worst_value, worst_oracle=c.worst_oracle)
                for c in cases[:nc.value]]

    def spd_solve(self, B: np.ndarray):
        """B: (n,) or (n, k) right-hand sides; returns X like B, residuals (k,), stats."""
        B = np.asarray(B, dtype=np.float64)
        vec = B.ndim == 1
        Bc = np.ascontiguousarray((B[:, None] if vec else B).T)  # (k, n) rows = rhs columns
        k = Bc.shape[0]
        X = np.zeros_like(Bc)
        res = np.zeros(k)
        st = GbemSolveStats()
        rc = self.lib.gbem_spd_solve(self.h, ptr(Bc), k, ptr(X), ptr(res), C.byref(st))
        self.check(rc)
        Xo = X.T
        return (Xo[:, 0] if vec else np.ascontiguousarray(Xo)), res, st
