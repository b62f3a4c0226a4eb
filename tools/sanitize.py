"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel of libcamelot.so runs at least once."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import _lib as L, api  # noqa: E402

probs = [G.config_problems(1)[0], G.config_problems(2)[4],
         G.random_small_problem(3, n_stages=4, n_gpus=9, n_apps=2, quota_step=25, batches=(1, 8))]
for p in probs:
    s = api.Session(p, n_loads=2)
    r = s.plan_max_load()
    m = s.plan_min_resource([[0.3 * max(r.objective, 1.0)] * p.n_apps, [0.5 * max(r.objective, 1.0)] * p.n_apps])
    s.predict_index(0, loads=[[1.0] * p.n_apps])
    s.score_range(0, min(5000, 1 << 12))
    ranks = [s, api.Session(p, n_loads=2)]   # one workspace per rank (finalize pairs with its search_local)
    keys = [ranks[k].search_local(0, rank=k, world=2).clone() for k in range(2)]
    red = torch.stack(keys).min(dim=0).values
    ranks[0].finalize(0, red, rank=0, world=2)
    f = api.Session(p, flags=p.flags | L.F_NO_FILTER).plan_max_load()
    g = api.Session(p, flags=p.flags | L.F_PAPER_GLOBAL).plan_max_load()
    print(p.name, r.index, m[0].index, f.index, g.index, flush=True)
# the newer paths: cascade sub-grid sweep + thread-per-parent passes (C4r), COMM,
# decision-tree tables, the tail simulator, simulated annealing
from gen import dt as D  # noqa: E402
c4r = G.config_problems(6)[0]
s = api.Session(c4r, n_loads=1)
r = s.plan_max_load()
m = s.plan_min_resource([[0.3 * r.objective]])
pc = G.with_comm(G.config_problems(2)[4], 1)
sc = api.Session(pc, n_loads=1)
rc = sc.plan_max_load()
fc = api.Session(pc, flags=pc.flags | L.F_NO_FILTER).plan_max_load()
tab = api.tables_from_trees(D.stage_trees(probs[0], 1), probs[0].batch, probs[0].quota_pct)
s1 = api.Session(probs[1])
rr = s1.plan_max_load()
sim = s1.simulate(rr.batch, rr.replicas, rr.quota_pct, [0.5 * rr.objective], 2000, 100, n_sims=2)
assert sim[0][0][0] > 0
sa = api.Session(probs[1], n_loads=1).sa(L.POLICY_MAX_LOAD, chains=256, iters=50)
print(c4r.name, r.index, m[0].index, rc.index, fc.index, float(tab.sum()), sim[0][0], sa.index, flush=True)
torch.cuda.synchronize()
print("sanitize workload ok")
