"""Time-to-plan of every BASELINE.json config (development aid): C1 (4 problems),
C2 (27), C3 (max-load + the 20-level min-resource sweep in one pass), C4, C5."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return out, statistics.median(ts[1:])


for cfg in (1, 2, 3, 4, 5):
    probs = G.config_problems(cfg)
    tot_ml = tot_mr = 0.0
    for p in probs:
        nlev = 20 if cfg == 3 else 1
        s = api.Session(p, n_loads=nlev)
        r, t1 = timed(s.plan_max_load)
        lam = [[(k + 1) / nlev * r.objective * (1 if nlev > 1 else 0.3)] * p.n_apps for k in range(nlev)]
        _, t2 = timed(lambda: s.plan_min_resource(lam))
        tot_ml += t1
        tot_mr += t2
    print(f"C{cfg}: {len(probs)} problem(s), max-load {tot_ml / len(probs):.3f} ms, "
          f"min-resource ({20 if cfg == 3 else 1} level(s)) {tot_mr / len(probs):.3f} ms per problem", flush=True)
