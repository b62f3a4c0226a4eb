"""One warm-up plan, then one measured plan of a config (for ncu captures).
python tools/ncu_one.py [config]   -- search_kernel launches per plan:
n passes for the coarse incumbent + n passes for the main search, per policy."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = G.config_problems(cfg)[0]
s = api.Session(p, n_loads=1)
for rep in range(2):
    r = s.plan_max_load()
    m = s.plan_min_resource([[0.3 * r.objective] * p.n_apps])[0]
torch.cuda.synchronize()
print(p.name, r.index, r.objective, m.index, m.gpus_used, m.quota_used)
