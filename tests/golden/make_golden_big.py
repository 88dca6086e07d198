"""Generate the full-size C-matrix goldens (run here, on CPU; needs oracle/_ref):

  config3_cmatrix.json   BASELINE config 3 at full size (33,776 panels, K = 17)
  config4s_cmatrix.json  BASELINE config 4's generator at scale 0.2 (19,374 panels, K = 64)

Every one of the n(n+1)/2 entries is the reference kernel (oracle/_ref: the
reference headers compiled in place, `u_pair_integral` kernels.hpp:270 inside
the `assemble_single` loop assembly.hpp:88-102, on all host threads).  The
solve is LAPACK Cholesky (scipy; not the reference's loop order, which is
infeasible here: ~5 h at n = 33,776) and the charges follow net_charges
(extraction.hpp:55-79).  The file also records the reference's convergence
diagnostics: every pair its Romberg reports as not converged (assembly.hpp:97),
with the reference value, a tight-tolerance (relTol 1e-13) reference value and
the closed-form 50-digit value (tests/exact_truth.py), so the GPU can be
checked on exactly the pairs the reference is unsure of.

  python tests/golden/make_golden_big.py 3          # ~2.6 h on 8 threads
  python tests/golden/make_golden_big.py 4 0.2      # ~50 min
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import scipy.linalg as sla

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))
import exact_truth as E  # noqa: E402
import oracle_lib as O  # noqa: E402
import paper_2203_11733_b200 as g  # noqa: E402
from make_golden import EPS0, panels_digest  # noqa: E402

NC_KEEP = 4000


def run(cfg: int, scale: float, nthreads: int):
    m = g.config_model(cfg, seed=1, scale=scale)
    ps = m.partition(1)
    P = ps.matrix()
    n = len(P)
    ids = m.net_ids
    t0 = time.time()

    def prog(d):
        el = time.time() - t0
        # rows are dealt in order, so done rows carry less work than the average early on
        frac = 1.0 - (1.0 - d / n) ** 2
        print(f"  rows {d}/{n} ({100 * frac:.1f}% of pairs) {el:.0f}s", flush=True)

    A, nc, nnc, rc = O.assemble_ref_diag(P, nthreads=nthreads, progress=prog)
    assert rc == 0, rc
    t_asm = time.time() - t0
    print(f"assembly {t_asm:.0f}s, not converged {nnc}", flush=True)
    keep = nc[:NC_KEEP]
    if len(keep):
        ref_v, _, _ = O.u_pairs("ref", P[keep[:, 0]], P[keep[:, 1]], nthreads=nthreads)
        tight, _, _ = O.u_pairs("ref", P[keep[:, 0]], P[keep[:, 1]], rel_tol=1e-13, max_levels=20,
                                nthreads=nthreads)
    else:
        ref_v = tight = np.zeros(0)
    exact = np.array([E.u_exact(P[i], P[j]) for i, j in keep]) if len(keep) else np.zeros(0)
    B = np.stack([(ps.kind == 0) & (ps.net == nid) for nid in ids], axis=1).astype(float)
    if os.environ.get("GOLDEN_SAVE_A"):
        np.save(os.environ["GOLDEN_SAVE_A"], A)
    A_keep = A.copy()
    solve = "scipy LAPACK cho_factor/cho_solve (not the reference loop order)"
    spd_fail = None
    try:
        c, low = sla.cho_factor(A, lower=True, overwrite_a=True, check_finite=False)
        X = sla.cho_solve((c, low), B, check_finite=False)
        del c
    except np.linalg.LinAlgError as e:
        # the reference's cholesky_solve would throw "matrix not positive definite"
        # here (solver.hpp:29-33); capacitance_row's allowLuFallback path
        # (extraction.hpp:128-131) solves by partial-pivot LU instead
        spd_fail = str(e)
        print("Cholesky failed:", spd_fail, "-> LU (the reference's allowLuFallback)", flush=True)
        lu = sla.lu_factor(A_keep, check_finite=False)
        X = sla.lu_solve(lu, B, check_finite=False)
        del lu
        solve = "scipy LAPACK lu_factor/lu_solve (the reference's LU fallback: its Cholesky fails, " + spd_fail + ")"
    del A
    res = np.linalg.norm(A_keep @ X - B, axis=0) / np.linalg.norm(B, axis=0)
    eps = m.info()["eps_r"]
    Cm = np.array([[eps * EPS0 * 1e-6 * X[(ps.net == k), r].sum() for k in ids] for r in range(len(ids))])
    d = {"config": cfg, "scale": scale, "seed": 1, "panels": n, "panels_sha256": panels_digest(P),
         "net_ids": ids, "eps_r": eps, "kernel": "ref", "all_converged": nnc == 0,
         "not_converged_pairs": nnc,
         "not_converged_sample": {"ij": keep.tolist(), "ref": np.asarray(ref_v).tolist(),
                                  "tight": np.asarray(tight).tolist(), "exact": exact.tolist()},
         "cmatrix_F": Cm.tolist(), "max_residual": float(res.max()),
         "assembly_s": round(t_asm, 1), "threads": nthreads,
         "solve": solve, "reference_cholesky_fails": spd_fail}
    return d


if __name__ == "__main__":
    cfg = int(sys.argv[1])
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    nth = int(os.environ.get("GOLDEN_THREADS", os.cpu_count()))
    d = run(cfg, scale, nth)
    name = f"config{cfg}_cmatrix.json" if scale == 1.0 else f"config{cfg}s_cmatrix.json"
    (HERE / name).write_text(json.dumps(d, indent=1))
    print(name, d["panels"], d["cmatrix_F"][0][:2], d["max_residual"], d["not_converged_pairs"])


def add_exact(name: str):
    """Post-process an existing golden: closed-form values of its non-converged sample."""
    f = HERE / name
    d = json.loads(f.read_text())
    m = g.config_model(d["config"], seed=d["seed"], scale=d["scale"])
    P = m.partition(1).matrix()
    ij = d["not_converged_sample"]["ij"]
    d["not_converged_sample"]["exact"] = [E.u_exact(P[i], P[j]) for i, j in ij]
    f.write_text(json.dumps(d, indent=1))
