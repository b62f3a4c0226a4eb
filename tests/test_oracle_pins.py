"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it follows.  PAPER.md = /root/reference/PAPER.md,
SPEC.md = /root/reference/SPEC.md (test ideas only); readings Rnn = DESIGN.md.
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


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def fbits(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


# ----------------------------------------------------------------- enumeration
def test_ntot_and_digit_order(oracle):
    """V = [n1..nN, p1..pN] plus the batch (L858): the
    canonical index is mixed radix, batch digit(s) most significant (R-enum)."""
    for cfg in (1, 2, 3, 4, 5):
        p = G.config_problems(cfg)[0]
        nS, nQ, R, n, A = len(p.batch), len(p.quota_pct), p.max_replicas, p.n_stages, p.n_apps
        assert oracle.ntot(p) == nS ** A * (R * nQ) ** n
    # C1 by hand: x = beta*100 + theta1*10 + theta2 (Rmax = 1, |Q| = 10)
    p = G.config_problems(1)[0]
    assert oracle.decode(p, 0) == ([0], [0, 0], [0, 0])
    assert oracle.decode(p, 599) == ([5], [0, 0], [9, 9])
    assert oracle.decode(p, 347) == ([3], [0, 0], [4, 7])
    # C2 by hand: radices [7][2][20][2][20][2][20]
    p = G.config_problems(2)[0]
    x = ((((((3 * 2 + 1) * 20 + 7) * 2 + 0) * 20 + 19) * 2 + 1) * 20 + 4)
    assert oracle.decode(p, x) == ([3], [1, 0, 1], [7, 19, 4])


def test_decode_bijection(oracle):
    p = G.config_problems(1)[0]
    seen = set()
    prev = None
    for x in range(oracle.ntot(p)):
        d = oracle.decode(p, x)
        key = (tuple(d[0]), tuple(itertools.chain(*zip(d[1], d[2]))))
        assert key not in seen
        if prev is not None:
            assert key > prev          # index order == lexicographic digit order
        prev = key
        seen.add(key)
        assert oracle.encode(p, *d) == x
    rng = np.random.default_rng(0)
    for cfg in (4, 5):
        p = G.config_problems(cfg)[0]
        for x in rng.integers(0, oracle.ntot(p), 200):
            assert oracle.encode(p, *oracle.decode(p, int(x))) == int(x)


# ----------------------------------------------------------------- objective
def test_worked_example_1pct(oracle):
    """Eq. 1 on the 1% grid: f1=p, f2=2p -> optimum 66 at (66,33) (golden)."""
    g = gold("worked_example_1pct.json")
    p = H.linear_thr_problem([1.0, 2.0], list(range(1, 101)))
    b = oracle.search(p)[0]
    assert b.T == g["expected_T"]
    beta, rho, theta = oracle.decode(p, b.index)
    assert [int(p.quota_pct[t]) for t in theta] == g["expected_p"]
    # all tied optima are feasible with the same T, and every one has a larger index
    for opt in g["tied_optima"]:
        x = oracle.encode(p, [0], [0, 0], [opt[0] - 1, opt[1] - 1])
        s = oracle.score(p, x)
        assert s.verdict == 0 and s.T == g["expected_T"] and x >= b.index
    assert g["expected_T"] <= g["continuous_optimum"]
    # multi-threaded scan gives the same (index, T) and counters
    b8 = oracle.search(p, threads=8)[0]
    assert (b8.index, b8.T, b8.n_feasible) == (b.index, b.T, b.n_feasible)


def test_symmetric_closed_form(oracle):
    """Two identical stages with f(p) = k p on one GPU -> (50, 50) (
    symmetry of Eq. 1)."""
    for grid in (list(range(10, 101, 10)), list(range(5, 101, 5)), list(range(1, 101))):
        p = H.linear_thr_problem([3.0, 3.0], grid)
        b = oracle.search(p)[0]
        _, _, theta = oracle.decode(p, b.index)
        assert [grid[t] for t in theta] == [50, 50]
        assert b.T == np.float32(150.0)


def test_bottleneck_law(oracle):
    """Peak load is set by the slowest stage:
    T <= min_i N_i f(p_i), with equality when there is no contention."""
    rng = np.random.default_rng(1)
    for prob in G.config_problems(2)[:4] + G.config_problems(5):
        nt = oracle.ntot(prob)
        for x in rng.integers(0, nt, 300):
            x = int(x)
            s = oracle.score(prob, x)
            beta, rho, theta = oracle.decode(prob, x)
            ub = min(np.float32(r + 1) * prob.table[i, beta[prob.app_of_stage[i]], theta[i], 1]
                     for i, r in enumerate(rho))
            assert s.T <= ub
            s0 = oracle.score(prob, x, flags=G.F_NO_CONTENTION)
            assert s0.T == ub
            assert all(k == 1.0 for k in s0.kappa)
            assert s0.L == [float(prob.table[i, beta[prob.app_of_stage[i]], theta[i], 0])
                            for i in range(prob.n_stages)]


# ----------------------------------------------------------------- contention
def test_contention_golden(oracle):
    g = gold("contention_example.json")
    p = H.contention_problem(45.0)
    for xs, ls in g["Lsum"].items():
        s = oracle.score(p, int(xs))
        assert s.place_viol == 0
        assert s.Lsum[0] == ls
        assert s.kappa[1] == g["kappa2"][xs]
        assert s.kappa[0] == 1.0          # gamma = 0 stage is never inflated
    for x in g["quota_infeasible"]:
        assert oracle.score(p, x).verdict == oracle.V_QUOTA
    for case in g["cases"]:
        p = H.contention_problem(case["qos"], case["flags"])
        b = oracle.search(p)[0]
        assert b.index == case["expect_index"]
        if "expect_T_bits" in case:
            assert fbits(b.T) == int(case["expect_T_bits"], 16)
        if "expect_T" in case:
            assert b.T == case["expect_T"]


def test_contention_invariants(oracle):
    """Adding a co-located instance never decreases any kappa;
    a stage alone on its GPU has kappa 1; SAT only acts above BW."""
    # one GPU, stage 1 fixed, stage 2 replicas 1..3 -> dem grows -> kappa1 non-decreasing
    tab = H.table_from([[[10.0]], [[10.0]]], [[[5.0]], [[5.0]]], [[[30.0]], [[40.0]]])
    cl = H.cluster(C=1, BW=100.0)
    p = G.custom_problem("inv", tab, [10], [1], [1e9], cl, max_replicas=3,
                         bw_sensitivity=[0.7, 0.2], flags=G.F_NO_BW_CAP)
    k_prev = 0.0
    for r in range(3):
        s = oracle.score(p, digits=([0], [0, r], [0, 0]))
        assert s.kappa[0] >= k_prev
        k_prev = s.kappa[0]
    # dem = 30 + 3*40 = 150 > BW: SAT multiplies by dem/BW
    s = oracle.score(p, digits=([0], [0, 2], [0, 0]))
    ssat = oracle.score(p, digits=([0], [0, 2], [0, 0]), flags=G.F_NO_BW_CAP | G.F_SAT)
    assert ssat.kappa[0] == np.float32(np.float32(s.kappa[0]) * np.float32(np.float32(150.0) * np.float32(1 / np.float32(100.0))))
    s1 = oracle.score(p, digits=([0], [0, 0], [0, 0]))     # dem = 70 < BW
    s1sat = oracle.score(p, digits=([0], [0, 0], [0, 0]), flags=G.F_NO_BW_CAP | G.F_SAT)
    assert s1.kappa == s1sat.kappa
    # two GPUs, two stages forced apart by quota -> each alone -> kappa 1
    tab = H.table_from([[[10.0]], [[10.0]]], [[[5.0]], [[5.0]]], [[[30.0]], [[40.0]]])
    p = G.custom_problem("apart", tab, [60], [1], [1e9], H.cluster(C=2, BW=100.0),
                         bw_sensitivity=[1.0, 1.0])
    s = oracle.score(p, 0)
    assert s.verdict == 0 and s.gpu_of_instance == [[0], [1]] and s.kappa == [1.0, 1.0]


def test_float64_latency_bound(oracle):
    """binary32 predicted latencies stay within 1e-5 relative of the float64
    evaluation of the same placement (north_star tolerance)."""
    rng = np.random.default_rng(2)
    for prob in G.config_problems(3) + G.config_problems(5):
        for x in rng.integers(0, oracle.ntot(prob), 300):
            s = oracle.score(prob, int(x))
            if s.place_viol:
                continue
            for a, b in zip(s.L, s.L64):
                assert abs(a - b) <= 1e-5 * abs(b)
            for a, b in zip(s.Ti, s.T64):
                assert abs(a - b) <= 1e-5 * abs(b)
            for a, b in zip(s.Lsum, s.Lsum64):
                assert abs(a - b) <= 1e-5 * abs(b)


# ----------------------------------------------------------------- placement
@pytest.mark.parametrize("case", gold("placement_cases.json")["cases"], ids=lambda c: c["name"])
def test_placement_cases(oracle, case):
    prob, digits = H.placement_problem(case)
    s = oracle.score(prob, digits=digits)
    assert s.place_viol == case["expect_viol"]
    if case["expect_gpus"] is not None:
        assert s.gpu_of_instance == case["expect_gpus"]
        used = {g for gs in case["expect_gpus"] for g in gs}
        assert s.u == len(used)


def test_single_gpu_placement_is_aggregate(oracle):
    """With one GPU the deployment reduces to the aggregate Eq. 1 Constraints
    1-4 evaluated on that GPU (weights once per stage)."""
    rng = np.random.default_rng(3)
    for trial in range(300):
        n = int(rng.integers(1, 4))
        Rmax = 3
        Q = [10, 20, 30, 40, 50]
        bw = rng.uniform(0, 60, (n, 1, 5))
        tab = H.table_from(np.ones((n, 1, 5)), np.ones((n, 1, 5)), bw)
        W = rng.integers(0, 3000, n)
        Am = rng.integers(0, 800, n)
        cl = H.cluster(C=1, I=int(rng.integers(2, 8)), BW=100.0, FM=8000)
        p = G.custom_problem("agg", tab, Q, [2], [1e9], cl, max_replicas=Rmax,
                             weights_mib=W, act_mib_per_item=Am)
        rho = [int(v) for v in rng.integers(0, Rmax, n)]
        th = [int(v) for v in rng.integers(0, 5, n)]
        s = oracle.score(p, digits=([0], rho, th))
        # the aggregate check, stage by stage in pipeline order (first failing stage)
        q = ni = mem = 0
        dem = np.float32(0)
        ok = True
        for i in range(n):
            N = rho[i] + 1
            q += N * Q[th[i]]
            ni += N
            mem += int(W[i]) + N * int(Am[i]) * 2
            dem = np.float32(dem + np.float32(np.float32(N) * np.float32(bw[i, 0, th[i]])))
            if q > 100 or ni > cl.max_instances or mem > 8000 or dem > np.float32(100.0):
                ok = False
                break
        assert (s.place_viol == 0) == ok


# ----------------------------------------------------------------- constraint isolation
def test_constraint_isolation(oracle):
    """Each check of Eq. 1 / Eq. 3 can be the unique failing one."""
    one = lambda v: [[[v]]]
    base = dict(quota_pct=[50], batch=[1], max_replicas=2)

    def mk(cl, bw=0.0, W=0, A=0, qos=1e9, dur=10.0, thr=10.0, n=1, gamma=0.0):
        tab = H.table_from([[[dur]]] * n, [[[thr]]] * n, [[[bw]]] * n)
        return G.custom_problem("iso", tab, base["quota_pct"], base["batch"], [qos], cl,
                                max_replicas=2, weights_mib=[W] * n, act_mib_per_item=[A] * n,
                                bw_sensitivity=[gamma] * n)
    # quota: 3 x 50% on one GPU (two stages, second with 2 replicas)
    p = mk(H.cluster(C=1), n=2)
    assert oracle.score(p, digits=([0], [0, 1], [0, 0])).verdict == oracle.V_QUOTA
    # instances: I = 1, a stage with 2 replicas of 50% (quota OK)
    p = mk(H.cluster(C=1, I=1))
    assert oracle.score(p, digits=([0], [1], [0])).verdict == oracle.V_INST
    # memory
    p = mk(H.cluster(C=1, FM=1000), W=600, A=300)
    assert oracle.score(p, digits=([0], [1], [0])).verdict == oracle.V_MEM
    assert oracle.score(p, digits=([0], [0], [0])).verdict == 0
    # bandwidth (Constraint-3 per GPU): 2 x 60 GB/s on a 100 GB/s GPU
    p = mk(H.cluster(C=1, BW=100.0), bw=60.0)
    assert oracle.score(p, digits=([0], [1], [0])).verdict == oracle.V_BW
    assert oracle.score(p, digits=([0], [1], [0]), flags=G.F_NO_BW_CAP).verdict == 0
    # QoS (Constraint-5): two 10 ms stages vs QoS 19
    p = mk(H.cluster(C=1), qos=19.0, n=2)
    assert oracle.score(p, digits=([0], [0, 0], [0, 0])).verdict == oracle.V_QOS
    p = mk(H.cluster(C=1), qos=20.0, n=2)
    assert oracle.score(p, digits=([0], [0, 0], [0, 0])).verdict == 0     # <= is feasible
    # load floor (reading R10): T = 10 QPS vs lambda 10 (ok) / 10.5 (LOAD)
    p = mk(H.cluster(C=1))
    s = oracle.score(p, digits=([0], [0], [0]), loads=[[10.0], [10.5]])
    assert s.level_verdict == [0, oracle.V_LOAD]
    # EQ2 budget: u = 2 GPUs but y = 1
    p = mk(H.cluster(C=2), n=2).with_(quota_pct=np.asarray([60], np.int32),
                                      flags=G.F_EQ2_BUDGET)
    s = oracle.score(p, digits=([0], [0, 0], [0, 0]), loads=[[1.0]])
    assert s.u == 2 and s.eq2_y == [1] and s.level_verdict == [oracle.V_EQ2]


# ----------------------------------------------------------------- Eq. 2
def test_eq2_closed_form(oracle):
    """Eq. 2, rate reading R9; SPEC.md L274-276 examples."""
    tab = H.table_from([[[1.0]]] * 2, [[[1.0]]] * 2, [[[0.0]]] * 2)
    cl = H.cluster(C=8, FM=10000, G=1000.0)
    # memory bound: sum M = 5000 = 0.5 F -> 1 ; compute negligible
    p = G.custom_problem("e", tab, [10], [10], [1e9], cl, weights_mib=[2000, 2000],
                         act_mib_per_item=[50, 50], gflop_per_item=[0.001, 0.001])
    assert oracle.eq2_y(p, [0], [1.0]) == 1
    # sum M = 23000 = 2.3 F -> 3
    p = p.with_(weights_mib=np.asarray([11000, 11000], np.uint32),
                act_mib_per_item=np.asarray([50, 50], np.uint32))
    assert oracle.eq2_y(p, [0], [1.0]) == 3
    # compute bound: lambda * sum c / G = 700 * (2 + 3) / 1000 = 3.5 -> 4
    p = p.with_(weights_mib=np.asarray([0, 0], np.uint32),
                act_mib_per_item=np.asarray([0, 0], np.uint32),
                gflop_per_item=np.asarray([2.0, 3.0], np.float32))
    assert oracle.eq2_y(p, [0], [700.0]) == 4
    # clamp to C
    assert oracle.eq2_y(p, [0], [1e6]) == 8


def test_memory_limits_batch(oracle):
    """Footprint linear in batch makes large batches infeasible (PAPER.md
    L450-460, 'batch < 256 fits')."""
    tab = H.table_from([[[1.0], [1.0]]], [[[1.0], [1.0]]], [[[0.0], [0.0]]])
    p = G.custom_problem("mem", tab, [100], [128, 256], [1e9], H.cluster(C=1, FM=16000),
                         weights_mib=[2000], act_mib_per_item=[60])
    assert oracle.score(p, digits=([0], [0], [0])).verdict == 0          # 2000+60*128 = 9680
    assert oracle.score(p, digits=([1], [0], [0])).verdict == oracle.V_MEM  # 17360 > 16000


# ----------------------------------------------------------------- relaxations / policies
def test_qos_relaxation_monotone(oracle):
    """Raising QoS never lowers T* (QoS does not affect placement)."""
    for prob in G.config_problems(1) + G.config_problems(2)[:3]:
        prev = None
        for rho in (0.8, 1.0, 1.25, 1.5):
            p = prob.with_(qos_ms=(prob.qos_ms * np.float32(rho)).astype(np.float32))
            b = oracle.search(p, threads=8)[0]
            T = b.T if b.index is not None else 0.0
            if prev is not None:
                assert T >= prev
            prev = T


def test_exhaustive_beats_even_allocation(oracle):
    """Camelot >= EA: the exact optimum is at
    least the even allocation whenever EA is feasible."""
    for prob in G.config_problems(1) + G.config_problems(2)[:6]:
        n, Q = prob.n_stages, [int(q) for q in prob.quota_pct]
        share = prob.cluster.n_gpus * prob.cluster.quota_per_gpu // n
        N = 1
        while share > prob.cluster.quota_per_gpu and N < prob.max_replicas:
            N += 1
            share = prob.cluster.n_gpus * prob.cluster.quota_per_gpu // (n * N)
        th = max(k for k, q in enumerate(Q) if q <= min(share, prob.cluster.quota_per_gpu))
        best = oracle.search(prob, threads=8)[0]
        for b in range(len(prob.batch)):
            s = oracle.score(prob, digits=([b], [N - 1] * n, [th] * n))
            if s.verdict == 0:
                assert best.index is not None and best.T >= s.T


def test_min_resource_monotone_in_load(oracle):
    """Lower load never needs more resources; at lambda = T* the
    max-load plan is feasible, so (u*, U*) <= its (u, U)."""
    for prob in G.config_problems(1) + G.config_problems(2)[:4]:
        bm = oracle.search(prob, threads=8)[0]
        fr = [1.0, 0.7, 0.5, 0.3, 0.1]
        loads = [[np.float32(f) * np.float32(bm.T)] for f in fr]
        res = oracle.search(prob, "min_resource", loads=loads, threads=8)
        assert res[0].index is not None
        assert (res[0].u, res[0].U) <= (bm.u, bm.U)
        keys = [(r.u, r.U) for r in res]
        assert keys == sorted(keys, reverse=True)
        for r in res[1:]:
            assert r.n_feasible >= res[0].n_feasible


def test_min_resource_paper_global_limit(oracle):
    """PAPER_GLOBAL (Eq. 3 literal), lambda -> 0: every N_i = 1 and p is the
    minimum-sum QoS-feasible quota vector (p-only brute force)."""
    for prob in G.config_problems(2)[:5]:
        p = prob.with_(flags=G.F_PAPER_GLOBAL)
        r = oracle.search(p, "min_resource", loads=[[1e-3]], threads=8)[0]
        beta, rho, theta = oracle.decode(p, r.index)
        assert rho == [0] * p.n_stages
        Q = [int(q) for q in p.quota_pct]
        best = None
        for b in range(len(p.batch)):
            d = p.table[:, b, :, 0]
            for th in itertools.product(range(len(Q)), repeat=p.n_stages):
                ls = np.float32(0)
                for i, t in enumerate(th):
                    ls = np.float32(ls + d[i, t]) if i else d[i, t]
                if ls <= p.qos_ms[0]:
                    U = sum(Q[t] for t in th)
                    if best is None or U < best:
                        best = U
        assert r.U == best


def test_paper_constants(oracle):
    """MPS cap I = 48: 49 instances never fit one GPU."""
    tab = H.table_from([[[1.0]]], [[[1.0]]], [[[0.0]]])
    p = G.custom_problem("mps", tab, [1], [1], [1e9], H.cluster(C=1, I=48), max_replicas=16)
    p8 = p
    s = oracle.score(p8, digits=([0], [15], [0]))
    assert s.verdict == 0
    tab = H.table_from([[[1.0]]] * 4, [[[1.0]]] * 4, [[[0.0]]] * 4)
    p = G.custom_problem("mps", tab, [1], [1], [1e9], H.cluster(C=1, I=48), max_replicas=13)
    assert oracle.score(p, digits=([0], [11, 11, 11, 11], [0] * 4)).verdict == 0   # 48
    assert oracle.score(p, digits=([0], [11, 11, 11, 12], [0] * 4)).verdict == oracle.V_INST


def test_generator_identities():
    """Generator tables follow SPEC.md L62/L71/L76: Thr*Dur = 1000 s, Dur
    strictly decreasing in p and increasing in s, Bw < BW."""
    for cfg in (1, 2, 3, 4, 5):
        for prob in G.config_problems(cfg)[:3]:
            t = prob.table.astype(np.float64)
            s = prob.batch.astype(np.float64)[None, :, None]
            assert np.allclose(t[..., 0] * t[..., 1], 1000.0 * s, rtol=1e-6)
            assert (np.diff(t[..., 0], axis=2) < 0).all()
            assert (np.diff(t[..., 0], axis=1) > 0).all()
            assert (t[..., 2] < prob.cluster.bw_gbs).all()
            assert (prob.bw_sensitivity >= 0).all() and (prob.bw_sensitivity <= 1).all()


def test_validation(oracle):
    p = G.config_problems(1)[0]
    assert oracle.validate(p) == 0
    assert oracle.validate(p.with_(quota_pct=np.asarray([20, 10], np.int32))) != 0
    assert oracle.validate(p.with_(qos_ms=np.asarray([0.0], np.float32))) != 0
    bad = p.table.copy()
    bad[0, 0, 0, 0] = np.nan
    assert oracle.validate(p.with_(table=bad)) != 0
    assert oracle.validate(p.with_(bw_sensitivity=np.asarray([-1, 0], np.float32))) != 0
