"""Diagnostics of a reference-assembled matrix saved by make_golden_big.py
(GOLDEN_SAVE_A=path): accuracy of its far-field entries against the composite
6^4 Gauss truth (2 x 2 split) on a seeded sample, written into the golden's
JSON under "reference_matrix_diagnostics".  Config 3's reference matrix fails
LAPACK's Cholesky (the reference's cholesky_solve would throw); this records
how far its far entries are from the truth.

  python tests/golden/diag_reference_matrix.py /tmp/golden/A_c3.npy config3_cmatrix.json
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))
import oracle_lib as O  # noqa: E402
import paper_2203_11733_b200 as g  # noqa: E402


def main(a_path, name, nsample=8000):
    f = HERE / name
    d = json.loads(f.read_text())
    A = np.load(a_path, mmap_mode="r")
    P = g.config_model(d["config"], seed=d["seed"], scale=d["scale"]).partition(1).matrix()
    n = len(P)
    rng = np.random.default_rng(5)
    i = rng.integers(0, n, 4 * nsample)
    j = rng.integers(0, n, 4 * nsample)
    keep = i != j
    i, j = i[keep], j[keep]
    far = O.gap_ratio(P[i], P[j]) >= 1.5
    i, j = i[far][:nsample], j[far][:nsample]
    area = (P[:, 3] - P[:, 2]) * (P[:, 5] - P[:, 4])
    truth = O.truth_pairs(P[i], P[j], sub=2) / (area[i] * area[j])
    ref = np.array([A[a, b] for a, b in zip(i, j)])
    rel = np.abs(ref - truth) / np.abs(truth)
    d["reference_matrix_diagnostics"] = {
        "far_pairs_sampled": int(len(i)), "truth": "composite 6^4 Gauss, 2 x 2 split (orc_gauss_pair)",
        "rel_err_median": float(np.median(rel)), "rel_err_p99": float(np.percentile(rel, 99)),
        "rel_err_max": float(rel.max()), "frac_above_1e-10": float((rel > 1e-10).mean()),
        "frac_above_1e-8": float((rel > 1e-8).mean()), "frac_above_1e-7": float((rel > 1e-7).mean())}
    f.write_text(json.dumps(d, indent=1))
    print(d["reference_matrix_diagnostics"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
