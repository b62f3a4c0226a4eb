"""SA (the paper's solver) on the device: time and quality vs the exact search."""
import os
import struct
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = G.config_problems(cfg)[0]
s = api.Session(p)
ex = s.plan_max_load()
for chains, iters in [(4096, 500), (16384, 1000), (65536, 2000)]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = s.sa(0, seed=1, chains=chains, iters=iters, p0=0.3, cool=0.995)
    dt = time.perf_counter() - t
    print(p.name, "SA chains=%d iters=%d  %.1f ms  T_sa=%.4f  T*=%.4f  gap=%.2f%%" %
          (chains, iters, dt * 1e3, r.objective, ex.objective, 100 * (1 - r.objective / ex.objective)), flush=True)
