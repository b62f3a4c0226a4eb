"""Writes tests/golden/expected_<name>.json for the configs too large for the
oracle to rerun inside the test suite (C4r, C5).  Calls ONLY oracle/ (plain
exhaustive scans) on problems from gen/problems.py.

    python tests/golden/make_expected.py [threads]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from gen import problems as G  # noqa: E402
from oracle import oracle as O  # noqa: E402


def best_dict(b):
    return dict(index=b.index, T=b.T, u=b.u, U=b.U, n_feasible=b.n_feasible, n_scanned=b.n_scanned,
                hist=b.hist)


def main(threads):
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for cfg in (6, 5):
        prob = G.config_problems(cfg)[0]
        t = time.time()
        bm = O.search(prob, threads=threads)[0]
        t1 = time.time() - t
        lam = [[0.3 * bm.T] * prob.n_apps]
        t = time.time()
        rm = O.search(prob, "min_resource", loads=lam, threads=threads)[0]
        t2 = time.time() - t
        rec = dict(problem=prob.name, sha256=prob.sha256(), ntot=O.ntot(prob),
                   max_load=best_dict(bm), min_resource=dict(loads=lam, **best_dict(rm)),
                   oracle_seconds=dict(max_load=t1, min_resource=t2, threads=threads),
                   note="written by tests/golden/make_expected.py (oracle only)")
        with open(os.path.join(out_dir, f"expected_{prob.name}.json"), "w") as f:
            json.dump(rec, f, indent=1)
        print(prob.name, rec["max_load"]["index"], rec["min_resource"]["index"], t1, t2, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else os.cpu_count())
