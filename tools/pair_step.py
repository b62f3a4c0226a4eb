"""A few fused C4 steps (camelot_plan_max_then_min) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

p = G.config_problems(int(sys.argv[1]) if len(sys.argv) > 1 else 4)[0]
s = api.Session(p, n_loads=1)
s.upload()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    pm, pr = s.plan_max_then_min(0.3, resident=True)
torch.cuda.synchronize()
print(p.name, pm.index, pr.index)
