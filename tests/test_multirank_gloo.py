"""The N > 1 host path on CPU: world_size-2 gloo process group, one
all_reduce(MIN) of sign-mapped packed keys (api.plan_distributed), checked
against the single-process oracle.  The per-rank shard search is emulated by
the oracle over the rank's chunks (chunk c = 2^15 consecutive indices, owned by
rank c mod W, the rule of the naive kernel); the collective, the key packing and
the combine are the product's."""
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CH = 1 << 15


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fbits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


class OracleShardSession:
    """Duck-typed Session: search_local / finalize backed by the CPU oracle."""

    def __init__(self, prob, oracle, api):
        self.prob, self.O, self.api = prob, oracle, api

    def _local_best(self, policy, loads, rank, world):
        nt = self.O.ntot(self.prob)
        best = None
        for c in range(rank, (nt + CH - 1) // CH, world):
            r = self.O.search(self.prob, "max_load" if policy == 0 else "min_resource", loads=loads,
                              lo=c * CH, hi=min(nt, (c + 1) * CH))[0]
            if r.index is None:
                continue
            key = (0xFFFFFFFF - fbits(r.T)) if policy == 0 else ((r.u << 24) | r.U)
            if best is None or (key, r.index) < best:
                best = (key, r.index)
        return best

    def search_local(self, policy, loads=None, rank=0, world=1, lo=0, hi=0, resident=False):
        b = self._local_best(policy, loads, rank, world)
        k = self.api.pack_key(0xFFFFFFFF, 0xFFFFFFFF) if b is None else self.api.pack_key(b[0], b[1])
        return torch.tensor([k], dtype=torch.int64)

    def finalize(self, policy, keys, loads=None, rank=0, world=1, lo=0, hi=0):
        obj, low = self.api.unpack_key(int(keys[0]))
        return [None if obj == 0xFFFFFFFF else low]


def worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from gen import problems as G
    from oracle import oracle as O
    from paper_2005_02088_b200 import api
    prob = G.config_problems(cfg)[0]
    s = OracleShardSession(prob, O, api)
    res = {}
    res["max"] = api.plan_distributed(s, 0)[0]
    ref = O.search(prob)[0]
    lam = [[0.3 * ref.T] * prob.n_apps]
    res["min"] = api.plan_distributed(s, 1, lam)[0]
    # edge keys: one rank infeasible, equal objectives, top-bit objective keys
    t = torch.tensor([api.pack_key(0xFFFFFFFF, 0xFFFFFFFF) if rank == 0 else api.pack_key(7, 5)])
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    res["edge1"] = api.unpack_key(int(t[0]))
    t = torch.tensor([api.pack_key(0xF0000000, 9 if rank == 0 else 4)])
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    res["edge2"] = api.unpack_key(int(t[0]))
    t = torch.tensor([api.pack_key(0x80000001 if rank == 0 else 0x7FFFFFFF, 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    res["edge3"] = api.unpack_key(int(t[0]))
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [1, 2])
def test_gloo_world2(cfg, oracle):
    from gen import problems as G
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(60)
    prob = G.config_problems(cfg)[0]
    ref = oracle.search(prob)[0]
    rm = oracle.search(prob, "min_resource", loads=[[0.3 * ref.T]])[0]
    for r in (0, 1):
        assert out[r]["max"] == ref.index
        assert out[r]["min"] == rm.index
        assert out[r]["edge1"] == (7, 5)
        assert out[r]["edge2"] == (0xF0000000, 4)
        assert out[r]["edge3"] == (0x7FFFFFFF, 1)
