"""Generate the committed golden fixtures (run here, on CPU; needs oracle/_ref):

  config1_cmatrix.json, config2_cmatrix.json : capacitance matrices of BASELINE
      configs 1-2 (panel lists from the C++ host generator, which the tests
      regenerate bit-identically) computed with the reference kernel
      (oracle/_ref: the reference headers compiled in place) for every entry,
      the reference assembly loop, and a dense LAPACK Cholesky solve
      (scipy; the reference's own loop order is tested separately at small n).
  pairs_golden.json : seeded pair list with reference values (relTol 1e-8) and
      tight-tolerance values (relTol 1e-13) for the near-field gate.

  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np
import scipy.linalg as sla

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))
import oracle_lib as O  # noqa: E402
import pairgen as G  # noqa: E402
import paper_2203_11733_b200 as g  # noqa: E402

EPS0 = 8.854187817e-12


def panels_digest(P):
    return hashlib.sha256(np.ascontiguousarray(P).tobytes()).hexdigest()


def cmatrix(cfg):
    m = g.config_model(cfg, seed=1)
    ps = m.partition(1)
    P = ps.matrix()
    ids = m.net_ids
    lib = "ref" if O.ref_available() else "orc"
    A, conv, rc = O.assemble(lib, P, nthreads=os.cpu_count())
    assert rc == 0
    B = np.stack([(ps.kind == 0) & (ps.net == nid) for nid in ids], axis=1).astype(float)
    c, low = sla.cho_factor(A, lower=True)
    X = sla.cho_solve((c, low), B)
    eps = m.info()["eps_r"]
    C = np.array([[eps * EPS0 * 1e-6 * X[(ps.net == k), r].sum() for k in ids] for r in range(len(ids))])
    res = np.linalg.norm(A @ X - B, axis=0) / np.linalg.norm(B, axis=0)
    return {"config": cfg, "seed": 1, "panels": len(P), "panels_sha256": panels_digest(P), "net_ids": ids,
            "eps_r": eps, "kernel": lib, "all_converged": bool(conv), "cmatrix_F": C.tolist(),
            "max_residual": float(res.max())}


def pairs():
    rng = np.random.default_rng(20261020)
    parts = [G.classic_pairs(rng, 60), G.touching_pairs(rng, 30), G.ratio_pairs(rng, 60, 0.0, 1.0),
             G.small_far_pairs(rng, 30)]
    A = np.vstack([p[0] for p in parts]); B = np.vstack([p[1] for p in parts])
    lib = "ref" if O.ref_available() else "orc"
    ref, conv, _ = O.u_pairs(lib, A, B)
    tight, _, _ = O.u_pairs(lib, A, B, rel_tol=1e-13, max_levels=20)
    truth = O.truth_pairs(A, B, sub=2)
    return {"kernel": lib, "A": A.tolist(), "B": B.tolist(), "ref": ref.tolist(), "tight": tight.tolist(),
            "gauss_truth": truth.tolist(), "gap_ratio": O.gap_ratio(A, B).tolist()}


if __name__ == "__main__":
    (HERE / "pairs_golden.json").write_text(json.dumps(pairs()))
    for cfg in (1, 2):
        d = cmatrix(cfg)
        (HERE / f"config{cfg}_cmatrix.json").write_text(json.dumps(d, indent=1))
        print(cfg, d["panels"], d["cmatrix_F"][0][:2], d["max_residual"])
