"""Quick per-config timing probe (development aid): plan_max_load + plan_min_resource
with the library's own kernel timing.  python tools/probe.py 4 5 6"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

for cfg in [int(c) for c in sys.argv[1:]]:
    p = G.config_problems(cfg)[0]
    s = api.Session(p, n_loads=1)
    r = None
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = s.plan_max_load()
        dt = time.perf_counter() - t
        st = s.last_stats()
        print(p.name, "maxload", r.index, r.objective, "ms=%.2f" % (dt * 1e3), "kern_ms=%.3f" % (st["t_ns"] / 1e6), st, flush=True)
    lam = [[0.3 * r.objective] * p.n_apps]
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        m = s.plan_min_resource(lam)[0]
        dt = time.perf_counter() - t
        st = s.last_stats()
        print(p.name, "minres", m.index, m.gpus_used, m.quota_used, "ms=%.2f" % (dt * 1e3), "kern_ms=%.3f" % (st["t_ns"] / 1e6), st, flush=True)
