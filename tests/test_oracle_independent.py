"""Pins of the oracle by independent computations (-m "not gpu").

* P-A: an independent numpy/itertools brute force over all
  four C1 problems, written here from the paper's definitions specialised to
  one GPU and one replica per stage (no code shared with oracle/), must give
  the oracle's argmax and objective bits for both policies.
* kappa over a split stage (tests/golden/kappa_split.json): kappa_i is the max
  over the GPUs hosting stage i (reading R17).
* min-resource priority (tests/golden/min_resource_priority.json): GPUs first,
  then quota (reading R11).
"""
import itertools
import json
import os
import struct

import numpy as np
import pytest

from gen import problems as G
from tests import helpers as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")
f32 = np.float32


def fbits(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def c1_brute_force(prob, lam=None):
    """Every C1 candidate scored from the paper's definitions with C = 1, Rmax = 1:
    both stages sit on the single GPU (the deployment scheme has one choice),
    Constraint-2 quota p1 + p2 <= R, Constraint-4 memory
    W1 + A1 s + W2 + A2 s <= F (L833), Constraint-3 bandwidth fl(bw1 + bw2) <= BW
    checked in placement order (L832; R2, R3), contention kappa_i =
    1 + gamma_i ((bw1 + bw2) - bw_i) / BW (R17), L_i = dur_i kappa_i,
    T_i = thr_i / kappa_i (N = 1; Eq. 1), QoS fl(L1 + L2) <= QoS (L834; R1),
    T = min(T1, T2).  Max-load: largest T, smallest index on ties (R20);
    min-resource at load lam: T >= lam (R10), smallest U = p1 + p2 (u = 1 always).
    Returns (index, T) or (index, U)."""
    Q = [int(q) for q in prob.quota_pct]
    S = [int(s) for s in prob.batch]
    cl = prob.cluster
    BW = f32(cl.bw_gbs)
    inv = f32(f32(1.0) / BW)
    best = None
    x = 0
    for b, t1, t2 in itertools.product(range(len(S)), range(len(Q)), range(len(Q))):
        idx = x
        x += 1
        e1, e2 = prob.table[0, b, t1], prob.table[1, b, t2]
        if Q[t1] > cl.quota_per_gpu:
            continue
        if Q[t1] + Q[t2] > cl.quota_per_gpu:
            continue
        s = S[b]
        if int(prob.weights_mib[0]) + int(prob.act_mib_per_item[0]) * s > cl.mem_mib:
            continue
        if sum(int(prob.weights_mib[i]) + int(prob.act_mib_per_item[i]) * s for i in (0, 1)) > cl.mem_mib:
            continue
        dem1 = f32(f32(0.0) + f32(f32(1.0) * e1[2]))
        if dem1 > BW:
            continue
        dem = f32(dem1 + f32(f32(1.0) * e2[2]))
        if dem > BW:
            continue
        T = None
        L = []
        Ts = []
        for e, g in ((e1, prob.bw_sensitivity[0]), (e2, prob.bw_sensitivity[1])):
            k = f32(f32(1.0) + f32(f32(g) * f32(f32(dem - e[2]) * inv)))
            L.append(f32(e[0] * k))
            Ts.append(f32(f32(f32(1.0) * e[1]) / k))
        if f32(L[0] + L[1]) > f32(prob.qos_ms[0]):
            continue
        T = min(Ts[0], Ts[1])
        if lam is None:
            if best is None or T > best[1]:
                best = (idx, T)
        else:
            if T < f32(lam):
                continue
            U = Q[t1] + Q[t2]
            if best is None or U < best[1]:
                best = (idx, U)
    return best


@pytest.mark.parametrize("j", range(4))
def test_c1_independent_brute_force(oracle, j):
    """P-A: oracle argmax and objective bits == the independent brute force."""
    prob = G.config_problems(1)[j]
    ref = oracle.search(prob)[0]
    bf = c1_brute_force(prob)
    assert bf is not None and ref.index == bf[0] and fbits(ref.T) == fbits(bf[1])
    for frac in (0.1, 0.3, 0.7, 1.0):
        lam = f32(f32(frac) * f32(ref.T))
        r = oracle.search(prob, "min_resource", loads=[[lam]])[0]
        bm = c1_brute_force(prob, lam)
        assert r.index == bm[0] and r.U == bm[1] and r.u == 1


def test_c1_brute_force_flags_and_qos(oracle):
    """P-A over perturbed C1 problems: tighter QoS, memory-tight GPU, bandwidth cap."""
    rng = np.random.default_rng(5)
    for j in range(4):
        base = G.config_problems(1)[j]
        for rho in (0.6, 0.9, 1.3):
            cl = G.Cluster(**{**base.cluster.__dict__, "mem_mib": int(rng.integers(3000, 12000)),
                              "bw_gbs": float(rng.uniform(300.0, 1200.0))})
            p = base.with_(qos_ms=(base.qos_ms * f32(rho)).astype(np.float32), cluster=cl)
            ref = oracle.search(p)[0]
            bf = c1_brute_force(p)
            if bf is None:
                assert ref.index is None
                continue
            assert ref.index == bf[0] and fbits(ref.T) == fbits(bf[1])


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "kappa_split.json")))["cases"],
                         ids=lambda c: c["name"])
def test_kappa_max_over_split_stage(oracle, case):
    """kappa of a stage split over GPUs is that of its worst GPU (golden)."""
    p = H.kappa_split_problem(case["bwA"])
    s = oracle.score(p, digits=([0], [0, 2], [0, 0]))
    assert s.verdict == 0 and s.u == 2
    assert s.gpu_of_instance == case["gpus"]
    assert s.dem == case["dem"]
    assert s.kappa == case["kappa"]
    assert s.L == case["L"] and s.Ti == case["Ti"]
    assert s.T == case["T"] and s.Lsum == [case["Lsum"]]
    assert oracle.encode(p, [0], [0, 2], [0, 0]) == 2
    b = oracle.search(p)[0]
    assert b.index == 2 and b.T == case["T"]


def test_min_resource_gpus_before_quota(oracle):
    """Lexicographic (u, U): a 1-GPU plan with larger sum N p beats a 2-GPU plan
    with a smaller one (golden)."""
    g = json.load(open(os.path.join(GOLD, "min_resource_priority.json")))
    p = H.min_resource_priority_problem()
    r = oracle.search(p, "min_resource", loads=[[g["setup"]["load"]]])[0]
    assert (r.index, r.u, r.U) == (g["expect"]["index"], g["expect"]["u"], g["expect"]["U"])
    w = g["u_first_would_give"]
    s = oracle.score(p, w["index"], loads=[[g["setup"]["load"]]])
    assert s.level_verdict == [0] and (s.u, s.U) == (w["u"], w["U"])
    # exhaustive listing: no feasible plan has u = 1 and U < 80
    for x in range(oracle.ntot(p)):
        s = oracle.score(p, x, loads=[[g["setup"]["load"]]])
        if s.level_verdict == [0]:
            assert (s.u, s.U) >= (1, 80)
