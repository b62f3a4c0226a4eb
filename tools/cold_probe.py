"""Cold-L2 penalty of the fused C4 call (development aid): device time of
camelot_plan_max_then_min (a) warm, (b) after a 256 MiB L2 flush, (c) after the
flush and a C4r call (same kernel instantiations: their code back in L2), (d)
after the flush and a touch of the workspace's first 64 MiB (data back in L2)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import problems as G
from paper_2005_02088_b200 import api
p = G.config_problems(4)[0]
s = api.Session(p, n_loads=1); s.upload()
w = api.Session(G.config_problems(6)[0], n_loads=1); w.upload()
st = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    s.plan_max_then_min(0.3, resident=True)
def timed(pre):
    out = []
    for i in range(15):
        pre(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.plan_max_then_min(0.3, resident=True)
        e1.record(st)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out), min(out)
def fl(i): flush.fill_(i & 0xFF)
def fl_code(i): fl(i); w.plan_max_then_min(0.3, resident=True)
def fl_data(i): fl(i); s.ws[: 64 << 20].sum()
for name, pre in [("warm", lambda i: None), ("flushed", fl), ("flushed+code", fl_code), ("flushed+data64M", fl_data)]:
    print(name, "median %.4f min %.4f ms" % timed(pre))
