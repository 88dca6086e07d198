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
    f = getattr(lib, prefix + "_u_point_rect")
    f.restype = C.c_double
    f.argtypes = [C.POINTER(C.c_double), RP]
    f = getattr(lib, prefix + "_q_point_rect")
    f.restype = C.c_double
    f.argtypes = [C.POINTER(C.c_double), RP, C.c_int]
    f = getattr(lib, prefix + "_q_pair_integral")
    f.restype = KV
    f.argtypes = [RP, RP, C.c_int, C.c_double, C.c_int]


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
        _orc.orc_assemble_collocation.restype = C.c_int
        _orc.orc_assemble_collocation.argtypes = [C.c_int64, C.c_void_p] + [C.c_void_p] * 5 + [
            C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
        _orc.orc_assemble_multi.restype = C.c_int
        _orc.orc_assemble_multi.argtypes = [C.c_int64, C.c_void_p] + [C.c_void_p] * 5 + [
            C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
            C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        _orc.orc_lu_solve.restype = C.c_int
        _orc.orc_lu_solve.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(C.c_int64)]
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


def point_kernels(lib_name: str, X: np.ndarray, R: np.ndarray, nsign: np.ndarray):
    """u_point_rect / q_point_rect at points X (k, 3) for rect rows R (k, 6)."""
    lib = orc() if lib_name == "orc" else ref()
    rr = rects_from_matrix(R)
    fu = getattr(lib, lib_name + "_u_point_rect")
    fq = getattr(lib, lib_name + "_q_point_rect")
    u = np.empty(len(X)); q = np.empty(len(X))
    for k in range(len(X)):
        x = (C.c_double * 3)(*map(float, X[k]))
        u[k] = fu(x, C.byref(rr[k]))
        q[k] = fq(x, C.byref(rr[k]), int(nsign[k]))
    return u, q


def lu_solve(A: np.ndarray, b: np.ndarray):
    """orc_lu_solve (solver.hpp:53-88): (x, resid, status, bad_row)."""
    A = np.ascontiguousarray(A, dtype=np.float64); b = np.ascontiguousarray(b, dtype=np.float64)
    n = len(b)
    x = np.zeros(n); res = np.zeros(1); bad = C.c_int64(-1)
    st = orc().orc_lu_solve(n, A.ctypes.data, b.ctypes.data, x.ctypes.data, res.ctypes.data, C.byref(bad))
    return x, float(res[0]), st, bad.value


def assemble_collocation(P: np.ndarray, nsign, kind, net, reg_a, reg_b, regions, main_net: int):
    """orc_assemble_collocation: (A (m, m), b (m,), status).  regions: [(id, eps), ...]."""
    n = len(P)
    rp = rects_from_matrix(P)
    ints = [np.ascontiguousarray(v, dtype=np.int32) for v in (nsign, kind, net, reg_a, reg_b)]
    rid = np.array([r[0] for r in regions], dtype=np.int32)
    reps = np.array([r[1] for r in regions], dtype=np.float64)
    mmax = n + int(np.sum(ints[1] == 3))
    A = np.zeros(mmax * mmax); b = np.zeros(mmax); m = C.c_int64(0)
    st = orc().orc_assemble_collocation(n, C.cast(rp, C.c_void_p), *[v.ctypes.data for v in ints], len(rid),
                                        rid.ctypes.data, reps.ctypes.data, int(main_net), A.ctypes.data,
                                        b.ctypes.data, C.byref(m))
    mm = m.value
    return A[:mm * mm].reshape(mm, mm), b[:mm], st


def q_pairs(lib_name: str, A: np.ndarray, B: np.ndarray, nsign, rel_tol=1e-8, max_levels=16):
    """q_pair_integral (kernels.hpp:295-315) of test rects A against source rects B
    (normal signs nsign): (values, converged, status)."""
    lib = orc() if lib_name == "orc" else ref()
    f = lib.orc_q_pair_integral if lib_name == "orc" else lib.ref_q_pair_integral
    ra, rb = rects_from_matrix(A), rects_from_matrix(B)
    out = np.zeros(len(A)); conv = np.zeros(len(A), dtype=np.int32); st = np.zeros(len(A), dtype=np.int32)
    for k in range(len(A)):
        kv = f(C.byref(ra[k]), C.byref(rb[k]), int(nsign[k]), rel_tol, max_levels)
        out[k], conv[k], st[k] = kv.value, kv.converged, kv.status
    return out, conv, st


def q_oracle(A: np.ndarray, B: np.ndarray, nsign, depth: int):
    """The reference's brute-force double-layer oracle (oracle.hpp:191, compiled in place)."""
    lib = ref()
    f = lib.ref_q_oracle_pair_integral
    f.restype = C.c_double
    f.argtypes = [RP, RP, C.c_int, C.c_int]
    ra, rb = rects_from_matrix(A), rects_from_matrix(B)
    return np.array([f(C.byref(ra[k]), C.byref(rb[k]), int(nsign[k]), depth) for k in range(len(A))])


def assemble_multi(P: np.ndarray, nsign, kind, net, reg_a, reg_b, regions, main_net: int, rel_tol=1e-8,
                   max_levels=16):
    """orc_assemble_multi (assembly.hpp:110-175): (A (m, m), b (m,), status, all_converged)."""
    n = len(P)
    rp = rects_from_matrix(P)
    ints = [np.ascontiguousarray(v, dtype=np.int32) for v in (nsign, kind, net, reg_a, reg_b)]
    rid = np.array([r[0] for r in regions], dtype=np.int32)
    reps = np.array([r[1] for r in regions], dtype=np.float64)
    mmax = n + int(np.sum(ints[1] == 3))
    A = np.zeros(mmax * mmax); b = np.zeros(mmax); m = C.c_int64(0); conv = C.c_int(0)
    st = orc().orc_assemble_multi(n, C.cast(rp, C.c_void_p), *[v.ctypes.data for v in ints], len(rid),
                                  rid.ctypes.data, reps.ctypes.data, int(main_net), rel_tol, max_levels,
                                  A.ctypes.data, b.ctypes.data, C.byref(m), C.byref(conv))
    mm = m.value
    return A[:mm * mm].reshape(mm, mm), b[:mm], st, bool(conv.value)


def assemble_ref_diag(P: np.ndarray, nthreads=8, rel_tol=1e-8, max_levels=16, nc_cap=1 << 20,
                      progress=None):
    """Reference assembly (oracle/_ref) plus the (i, j) of every pair the
    reference's Romberg reports as not converged (assembly.hpp:97)."""
    lib = ref()
    f = lib.ref_assemble_single_diag
    CB = C.CFUNCTYPE(None, C.c_int64)
    f.restype = C.c_int
    f.argtypes = [C.c_int64, RP, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_int64,
                  C.POINTER(C.c_int64), C.c_int, CB]
    n = len(P)
    rp = rects_from_matrix(P)
    A = np.empty((n, n))
    nc = np.zeros((nc_cap, 2), dtype=np.int64)
    cnt = C.c_int64(0)
    cb = CB(progress) if progress else CB(lambda d: None)
    st = f(n, rp, rel_tol, max_levels, A.ctypes.data, nc.ctypes.data, nc_cap, C.byref(cnt), nthreads, cb)
    k = min(cnt.value, nc_cap)
    return A, nc[:k].copy(), int(cnt.value), st


def flatten_scene(model_text: str):
    """Scene text (model_io.hpp grammar) -> the flat arrays the _ref entry points
    take: dom[6], regions (id, eps, lo, hi) x 8, cells (net, lo, hi) x 7, bc[6]."""
    lines = [l.split("#")[0].split() for l in model_text.splitlines()]

    def pt(tok):
        return [float(v) for v in tok[tok.index("(") + 1:-1].split(",")]
    dom = None
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
    return (np.array(dom, dtype=float), np.array(regs, dtype=float), np.array(cells, dtype=float),
            np.array(bc, dtype=np.int32))


REF_GPU_SO = ROOT / "oracle" / "_ref" / "libgbem_ref_gpu.so"


def ref_gpu_capacitance_row(model_text: str, main_net: int, params, rel_tol=1e-8, max_levels=16):
    """capacitance_row through the reference-side GPU binding (oracle/ref_gpu_backend.cpp):
    returns (charges per net in ascending id order, outer charge, panels, residual, converged)."""
    lib = C.CDLL(str(REF_GPU_SO))
    f = lib.refgpu_capacitance_row
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                  C.c_double, C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                  C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_char_p, C.c_int]
    dom, regs, cells, bc = flatten_scene(model_text)
    par = np.array(params, dtype=float)
    q = np.zeros(256)
    outer, res = C.c_double(0), C.c_double(0)
    npan, conv = C.c_int64(0), C.c_int(0)
    err = C.create_string_buffer(512)
    k = f(dom.ctypes.data, len(regs) // 8, regs.ctypes.data, len(cells) // 7, cells.ctypes.data, bc.ctypes.data,
          par.ctypes.data, main_net, rel_tol, max_levels, q.ctypes.data, 256, C.byref(outer), C.byref(npan),
          C.byref(res), C.byref(conv), err, 512)
    if k < 0:
        raise RuntimeError(f"refgpu_capacitance_row: {err.value.decode()} ({k})")
    return q[:k], outer.value, npan.value, res.value, bool(conv.value)
