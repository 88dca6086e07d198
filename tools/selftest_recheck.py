"""Re-evaluate the worst pairs dumped by tools/selftest_probe.py with the reference
compiled in place (oracle/_ref): its semi-analytic q_pair_integral / u_pair_integral
and its brute-force oracle at several depths.  Tells apart a GPU evaluator bug
(GPU value != reference value) from a reference-algorithm / oracle-depth limit
(GPU value == reference value, both != oracle)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle_lib as OL  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/st_probe.jsonl"
for line in open(path):
    c = json.loads(line)
    if c["passed"] and "--all" not in sys.argv:
        continue
    A = np.array([c["worst_test"]])
    B = np.array([c["worst_source"]])
    ns = [c["worst_nsign"]]
    q = c["name"].startswith("Q")
    if q:
        ref_v = OL.q_pairs("ref", A, B, ns)[0][0]
        orc = {d: OL.q_oracle(A, B, ns, d)[0] for d in (3, 4, 5, 6, 7)}
    else:
        ref_v = OL.u_pairs("ref", A, B)[0][0]
        orc = {d: OL.ref().ref_oracle_pair_integral(OL.rects_from_matrix(A), OL.rects_from_matrix(B), d)
               for d in (3, 4, 5, 6, 7)}
    print(f"{c['seed']} {c['name']}: gpu={c['worst_value']:.12e} ref={ref_v:.12e} "
          f"gpu-vs-ref={abs(c['worst_value'] - ref_v) / max(abs(ref_v), 1e-9):.2e} oracle_used={c['worst_oracle']:.12e}")
    print("   test", c["worst_test"], "source", c["worst_source"], "nsign", c["worst_nsign"])
    for d, v in orc.items():
        print(f"   oracle depth {d}: {v:.12e}  rel(ref)={abs(ref_v - v) / max(abs(v), 1e-9):.2e}")
