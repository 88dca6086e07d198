"""Test-side loader of the CPU checkers (oracle/): never imported by the product.

- `orc`: plain-C restatement (oracle/_build/libgbem_oracle.so)
- `ref`: the reference headers compiled in place (oracle/_ref/libgbem_ref.so)
Both are built by `make -C oracle` (and by __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORC_SO = ROOT / "oracle" / "_build" / "libgbem_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libgbem_ref.so"


class Rect(C.Structure):
    _fields_ = [("axis", C.c_int), ("level", C.c_double), ("a0", C.c_double), ("a1", C.c_double),
                ("b0", C.c_double), ("b1", C.c_double)]


class KV(C.Structure):
    _fields_ = [("value", C.c_double), ("converged", C.c_int), ("evals", C.c_long), ("status", C.c_int)]


RP = C.POINTER(Rect)


def _ensure_built():
    if not ORC_SO.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


def _bind(lib, prefix):
    f = getattr(lib, prefix + "_u_pair_integral")
    f.restype = KV
    f.argtypes = [RP, RP, C.c_double, C.c_int]
    f = getattr(lib, prefix + "_u_pairs")
    f.restype = C.c_int
    f.argtypes = [C.c_int64, RP, RP, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
    f = getattr(lib, prefix + "_assemble_single")
    f.restype = C.c_int
    f.argtypes = [C.c_int64, RP, C.c_double, C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_int]
    f = getattr(lib, prefix + "_oracle_pair_integral")
    f.restype = C.c_double
    f.argtypes = [RP, RP, C.c_int]


_orc = _ref = None


def orc():
    global _orc
    if _orc is None:
        _ensure_built()
        _orc = C.CDLL(str(ORC_SO))
        _bind(_orc, "orc")
        _orc.orc_gauss_pair.restype = C.c_double
        _orc.orc_gauss_pair.argtypes = [RP, RP, C.c_int]
        _orc.orc_rect_distance.restype = C.c_double
        _orc.orc_rect_distance.argtypes = [RP, RP]
        _orc.orc_rect_diameter.restype = C.c_double
        _orc.orc_rect_diameter.argtypes = [RP]
        _orc.orc_cholesky_solve.restype = C.c_int
        _orc.orc_cholesky_solve.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.POINTER(C.c_int64)]
        _orc.orc_quad_test.restype = C.c_double
        _orc.orc_quad_test.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                       C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_long)]
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        _ref = C.CDLL(str(REF_SO))
        _bind(_ref, "ref")
        _ref.ref_partition_scene.restype = C.c_int64
        _ref.ref_partition_scene.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_char_p, C.c_int]
    return _ref


def rect(axis, level, a, b) -> Rect:
    return Rect(int(axis), float(level), float(a[0]), float(a[1]), float(b[0]), float(b[1]))


def rects_from_matrix(m: np.ndarray):
    """(n, 6) matrix axis, level, a0, a1, b0, b1 -> ctypes Rect array."""
    n = len(m)
    arr = (Rect * n)()
    for k in range(n):
        arr[k] = Rect(int(m[k, 0]), *map(float, m[k, 1:6]))
    return arr


def u_pairs(lib_name: str, A: np.ndarray, B: np.ndarray, rel_tol=1e-8, max_levels=16, nthreads=8):
    lib = orc() if lib_name == "orc" else ref()
    ra, rb = rects_from_matrix(A), rects_from_matrix(B)
    out = np.zeros(len(A))
    conv = np.zeros(len(A), dtype=np.int32)
    f = lib.orc_u_pairs if lib_name == "orc" else lib.ref_u_pairs
    st = f(len(A), ra, rb, rel_tol, max_levels, out.ctypes.data, conv.ctypes.data, nthreads)
    return out, conv.astype(bool), st


def truth_pairs(A: np.ndarray, B: np.ndarray, sub=2):
    """Composite 6^4 Gauss (each panel split sub x sub), the far-field truth."""
    lib = orc()
    ra, rb = rects_from_matrix(A), rects_from_matrix(B)
    return np.array([lib.orc_gauss_pair(C.byref(ra[k]), C.byref(rb[k]), sub) for k in range(len(A))])


def gap_ratio(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    lib = orc()
    ra, rb = rects_from_matrix(A), rects_from_matrix(B)
    g = np.zeros(len(A))
    for k in range(len(A)):
        d = lib.orc_rect_distance(C.byref(ra[k]), C.byref(rb[k]))
        dm = max(lib.orc_rect_diameter(C.byref(ra[k])), lib.orc_rect_diameter(C.byref(rb[k])))
        g[k] = d / dm
    return g


def assemble(lib_name: str, P: np.ndarray, nthreads=8, rel_tol=1e-8, max_levels=16):
    lib = orc() if lib_name == "orc" else ref()
    n = len(P)
    rp = rects_from_matrix(P)
    A = np.zeros((n, n))
    conv = C.c_int(1)
    f = lib.orc_assemble_single if lib_name == "orc" else lib.ref_assemble_single
    st = f(n, rp, rel_tol, max_levels, A.ctypes.data, C.byref(conv), nthreads)
    return A, bool(conv.value), st
