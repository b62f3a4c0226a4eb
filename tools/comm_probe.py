"""C4 / C5 with the NEXT-2 communication-aware QoS (flag COMM): plan times and
how the plans differ from the paper's Constraint-5 (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

for cfg in [int(c) for c in sys.argv[1:]] or [4]:
    base = G.config_problems(cfg)[0]
    for prob in (base, G.with_comm(base, cfg)):
        s = api.Session(prob, n_loads=1)
        for rep in range(3):
            r = s.plan_max_load()
            t1 = s.last_stats()["t_ns"] / 1e6
            m = s.plan_min_resource([[0.3 * r.objective] * prob.n_apps])[0]
            t2 = s.last_stats()["t_ns"] / 1e6
        print(prob.name, "COMM" if prob.flags & G.F_COMM else "paper", "maxload", r.index, r.objective,
              r.replicas, r.quota_pct, "comm", [round(v, 4) for v in (r.comm_ms or [])],
              "ms=%.3f" % t1, "| minres", m.index, m.gpus_used, m.quota_used, "ms=%.3f" % t2, flush=True)
torch.cuda.synchronize()
