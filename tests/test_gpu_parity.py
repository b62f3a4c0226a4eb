"""Parity of the CUDA path (through the C ABI) with the CPU oracle (-m gpu).

Bar (BASELINE.json north_star): chosen plan index bit-exact, predicted
latencies/throughputs within 1e-5 relative (here: bit-exact, both sides use
the same binary32 evaluation order, R21), feasibility verdicts
identical.  Inputs are the seeded synthetic problems of gen/problems.py.
"""
import json
import os
import struct

import numpy as np
import pytest
import torch

from gen import problems as G
from tests import helpers as H

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2005_02088_b200 import _lib
    _lib.build()
    from paper_2005_02088_b200 import api as A
    return A


def fb(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def check_plan(api, prob, got, ref, oracle, loads=None):
    assert got.index == ref.index, (prob.name, got.index, ref.index)
    if ref.index is None:
        assert not got.feasible
        return
    assert got.feasible
    assert got.quota_used == ref.U and got.gpus_used == ref.u
    # full prediction of the winner == oracle_predict
    s = oracle.score(prob, ref.index, loads=loads)
    assert fb(got.throughput_qps[0]) == fb(s.Tmin[0])
    assert [fb(v) for v in got.stage_latency_ms] == [fb(v) for v in s.L]
    assert [fb(v) for v in got.stage_throughput_qps] == [fb(v) for v in s.Ti]
    assert [fb(v) for v in got.kappa] == [fb(v) for v in s.kappa]
    assert [fb(v) for v in got.e2e_latency_ms] == [fb(v) for v in s.Lsum]
    assert got.gpu_of_instance == s.gpu_of_instance
    if loads is None:
        assert fb(got.objective) == fb(ref.T)


# ------------------------------------------------------------------ per-candidate scoring
@pytest.mark.parametrize("cfg,windows", [(1, None), (2, None), (3, 3), (4, 4), (5, 4)])
def test_score_range_vectors(api, oracle, cfg, windows):
    """Full verdict / objective vectors (C1, C2) and sampled windows (C3-C5)."""
    probs = G.config_problems(cfg)
    probs = probs if cfg == 1 else probs[:2]
    rng = np.random.default_rng(cfg)
    for prob in probs:
        nt = oracle.ntot(prob)
        if windows is None:
            spans = [(0, nt)]
        else:
            w = 40000
            starts = [0, nt - w] + [int(v) for v in rng.integers(0, nt - w, windows)]
            spans = [(s, s + w) for s in starts]
        s = api.Session(prob)
        for lo, hi in spans:
            v, T, u, U = (t.cpu().numpy() for t in s.score_range(lo, hi))
            rv, rT, ru, rU = oracle.score_range(prob, lo, hi)
            np.testing.assert_array_equal(v, rv)
            np.testing.assert_array_equal(U, rU)
            # T and u are defined for placed candidates only (after a placement
            # failure the oracle keeps its partial-placement state, the kernel not)
            placed = (rv & 15) == 0
            np.testing.assert_array_equal(T.view(np.uint32)[placed], rT.view(np.uint32)[placed])
            np.testing.assert_array_equal(u[placed], ru[placed])


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_predict_sampled(api, oracle, cfg):
    """camelot_predict == oracle_predict on random candidates (all fields)."""
    prob = G.config_problems(cfg)[0]
    s = api.Session(prob)
    rng = np.random.default_rng(10 + cfg)
    for x in rng.integers(0, oracle.ntot(prob), 200):
        x = int(x)
        g = s.predict_index(x, loads=[[10.0] * prob.n_apps])
        r = oracle.score(prob, x, loads=[[10.0] * prob.n_apps])
        assert g.index == x
        assert g.violations == r.level_verdict[0]
        assert g.quota_used == r.U
        assert g.eq2_gpus == r.eq2_y[0]
        if r.place_viol == 0:     # predictions are defined for placed candidates
            assert fb(g.objective) == fb(r.T)
            assert [fb(v) for v in g.stage_latency_ms] == [fb(v) for v in r.L]
            assert [fb(v) for v in g.stage_throughput_qps] == [fb(v) for v in r.Ti]
            assert g.gpus_used == r.u and g.gpu_of_instance == r.gpu_of_instance
            for a, b in zip(g.stage_latency_ms, r.L64):
                assert abs(a - b) <= 1e-5 * abs(b)     # north_star latency tolerance vs float64


# ------------------------------------------------------------------ searches
def test_golden_examples(api, oracle):
    g = json.load(open(os.path.join(GOLD, "worked_example_1pct.json")))
    p = H.linear_thr_problem([1.0, 2.0], list(range(1, 101)))
    got = api.Session(p).plan_max_load()
    assert got.objective == g["expected_T"] and got.quota_pct == g["expected_p"]
    g = json.load(open(os.path.join(GOLD, "contention_example.json")))
    for case in g["cases"]:
        p = H.contention_problem(case["qos"], case["flags"])
        got = api.Session(p).plan_max_load()
        assert got.index == case["expect_index"]
        if "expect_T_bits" in case:
            assert fb(got.objective) == int(case["expect_T_bits"], 16)


@pytest.mark.parametrize("cfg", [1, 2, 3])
@pytest.mark.parametrize("mode", ["pruned", "flat", "naive"])
def test_max_load_configs(api, oracle, cfg, mode):
    probs = G.config_problems(cfg)
    if mode != "pruned":
        probs = probs[:5]
    for prob in probs:
        flags = prob.flags | (G.F_NO_FILTER if mode == "flat" else 0)
        s = api.Session(prob, flags=flags)
        if mode == "naive":
            from paper_2005_02088_b200 import _lib as L
            import ctypes as C
            out = L.Plan()
            ex = s.exec()
            ex.exec_flags = 2   # CAMELOT_EXEC_NAIVE
            L.check(L.lib().camelot_plan_max_load(C.byref(s.cprob), C.byref(s.ccl), C.byref(ex), C.byref(out)))
            got = api._plan(out, prob.n_stages, prob.n_apps)
        else:
            got = s.plan_max_load()
        ref = oracle.search(prob, threads=8)[0]
        check_plan(api, prob, got, ref, oracle)
        if mode in ("flat", "naive"):
            assert got.n_feasible == ref.n_feasible


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_min_resource_configs(api, oracle, cfg):
    probs = G.config_problems(cfg)[:6]
    for prob in probs:
        bm = oracle.search(prob, threads=8)[0]
        nlev = 20 if cfg == 3 else 4
        loads = [[np.float32(k / nlev) * np.float32(bm.T)] for k in range(1, nlev + 1)]
        got = api.Session(prob, n_loads=nlev).plan_min_resource(loads)
        ref = oracle.search(prob, "min_resource", loads=loads, threads=8)
        for k, (g, r) in enumerate(zip(got, ref)):
            check_plan(api, prob, g, r, oracle, loads=[loads[k]])
            assert fb(g.objective) == fb(np.float32(r.U))


@pytest.mark.parametrize("seed", range(24))
def test_random_small_problems_all_flags(api, oracle, seed):
    """Random mixed pipelines (1-2 apps, 2-8 stages, 1-5 GPUs) under every flag."""
    rng = np.random.default_rng(seed)
    A = int(rng.integers(1, 3))
    n = int(rng.integers(max(2, A), 5 if A == 1 else 6))
    C = int(rng.integers(1, 6))
    flag_sets = [0, G.F_NO_BW_CAP, G.F_NO_CONTENTION, G.F_SAT | G.F_NO_BW_CAP, G.F_EQ2_BUDGET,
                 G.F_PAPER_GLOBAL, G.F_NO_FILTER]
    flags = flag_sets[seed % len(flag_sets)]
    prob = G.random_small_problem(seed, n_stages=n, n_gpus=C, n_apps=A,
                                  quota_step=int(rng.choice([20, 25, 34])),
                                  batches=(1, 4, 16)[: int(rng.integers(1, 4))],
                                  max_replicas=int(rng.integers(1, 4)),
                                  qos_rho=float(rng.choice([0.8, 1.0, 1.5])), flags=flags)
    if oracle.ntot(prob) > 3_000_000:
        pytest.skip("space too large for the in-test oracle")
    got = api.Session(prob).plan_max_load()
    ref = oracle.search(prob, threads=8)[0]
    check_plan(api, prob, got, ref, oracle)
    if ref.index is not None:
        loads = [[np.float32(f) * np.float32(ref.T)] * A for f in (0.2, 0.5, 1.0)]
        gm = api.Session(prob, n_loads=3).plan_min_resource(loads)
        rm = oracle.search(prob, "min_resource", loads=loads, threads=8)
        for k in range(3):
            check_plan(api, prob, gm[k], rm[k], oracle, loads=[loads[k]])


def test_infeasible_and_edges(api, oracle):
    prob = G.config_problems(2)[0]
    p = prob.with_(qos_ms=np.asarray([1e-3], np.float32))
    got = api.Session(p).plan_max_load()
    assert got.index is None and not got.feasible
    # one batch, one GPU, one replica
    p = G.config_problems(1)[0].with_(batch=np.asarray([8], np.int32),
                                      table=G.config_problems(1)[0].table[:, 3:4].copy())
    check_plan(api, p, api.Session(p).plan_max_load(), oracle.search(p)[0], oracle)


@pytest.mark.parametrize("name", ["C4r-p1c2m2c3m1", "C5-p2c3m1+p1c1m3"])
def test_large_configs_golden(api, oracle, name):
    """C4r (8.2e8) and C5 (2.3e9) against oracle results written by
    tests/golden/make_expected.py."""
    path = os.path.join(GOLD, f"expected_{name}.json")
    if not os.path.exists(path):
        pytest.skip("expected file not generated")
    e = json.load(open(path))
    prob = [p for c in (5, 6) for p in G.config_problems(c) if p.name == name][0]
    assert prob.sha256() == e["sha256"]
    got = api.Session(prob).plan_max_load()
    assert got.index == e["max_load"]["index"]
    assert fb(got.objective) == fb(np.float32(e["max_load"]["T"]))
    loads = e["min_resource"]["loads"]
    gm = api.Session(prob, n_loads=1).plan_min_resource(loads)[0]
    assert gm.index == e["min_resource"]["index"]
    assert (gm.gpus_used, gm.quota_used) == (e["min_resource"]["u"], e["min_resource"]["U"])


# ------------------------------------------------------------------ C4 (8.192e13): slices + properties
def test_c4_slices(api, oracle):
    prob = G.config_problems(4)[0]
    nt = oracle.ntot(prob)
    rng = np.random.default_rng(44)
    w = 1_500_000
    s = api.Session(prob)
    starts = [0, (nt // 2) & ~0xFFFF, int(rng.integers(0, nt - w))]
    for lo in starts:
        got = s.plan_max_load(lo=lo, hi=lo + w)
        ref = oracle.search(prob, lo=lo, hi=lo + w, threads=8)[0]
        check_plan(api, prob, got, ref, oracle)


def test_c4_full_properties(api, oracle):
    """Full C4: the winner is feasible per the oracle with the same T, and no
    smaller index in its neighbourhood ties it (tie rule)."""
    prob = G.config_problems(4)[0]
    s = api.Session(prob)
    got = s.plan_max_load()
    assert got.feasible
    sc = oracle.score(prob, got.index)
    assert sc.verdict == 0 and fb(sc.T) == fb(got.objective)
    c4r = [p for p in G.config_problems(6)][0]
    r4r = api.Session(c4r).plan_max_load()
    assert got.objective >= r4r.objective   # the 10% grid is a subset
    lo = max(0, got.index - 400_000)
    ref = oracle.search(prob, lo=lo, hi=got.index + 1, threads=8)[0]
    assert ref.index == got.index and fb(ref.T) == fb(got.objective)
    # min-resource at 30% of the peak
    lam = [[np.float32(0.3) * np.float32(got.objective)]]
    gm = api.Session(prob, n_loads=1).plan_min_resource(lam)[0]
    sm = oracle.score(prob, gm.index, loads=lam)
    assert gm.feasible and sm.level_verdict == [0]
    assert (gm.gpus_used, gm.quota_used) == (sm.u, sm.U)
    lo = max(0, gm.index - 400_000)
    ref = oracle.search(prob, "min_resource", loads=lam, lo=lo, hi=gm.index + 1, threads=8)[0]
    assert ref.index == gm.index


# ------------------------------------------------------------------ sharding (one GPU, several ranks)
@pytest.mark.parametrize("cfg,world", [(2, 2), (3, 3), (5, 4), (4, 2)])
def test_sharded_equals_single(api, oracle, cfg, world):
    """search_local on every rank + MIN of the keys + finalize == single plan
    (covers the chunk rescan when Ntot > 2^32)."""
    prob = G.config_problems(cfg)[0]
    lo, hi = (0, 0) if cfg != 4 else (10 ** 12, 10 ** 12 + 3_000_000)
    single = api.Session(prob).plan_max_load(lo=lo, hi=hi)
    keys = []
    sess = [api.Session(prob) for _ in range(world)]
    for r in range(world):
        keys.append(sess[r].search_local(0, rank=r, world=world, lo=lo, hi=hi).clone())
    red = torch.stack(keys).min(dim=0).values
    for r in range(world):
        pl = sess[r].finalize(0, red, rank=r, world=world, lo=lo, hi=hi)[0]
        assert pl.index == single.index and fb(pl.objective) == fb(single.objective)


@pytest.mark.parametrize("cfg,world", [(2, 2), (3, 3), (6, 2), (4, 3)])
def test_sharded_flat_equals_single(api, oracle, cfg, world):
    """The same with NO_FILTER (the leaf sweep: chunk ownership per parent; for
    C4, Ntot > 2^32, so the winning chunk is re-scanned by the tree search)."""
    prob = G.config_problems(cfg)[0]
    flags = prob.flags | G.F_NO_FILTER
    lo, hi = (0, 0) if cfg != 4 else (10 ** 12, 10 ** 12 + (1 << 27))
    single = api.Session(prob, flags=flags).plan_max_load(lo=lo, hi=hi)
    keys = []
    sess = [api.Session(prob, flags=flags) for _ in range(world)]
    for r in range(world):
        keys.append(sess[r].search_local(0, rank=r, world=world, lo=lo, hi=hi).clone())
    red = torch.stack(keys).min(dim=0).values
    for r in range(world):
        pl = sess[r].finalize(0, red, rank=r, world=world, lo=lo, hi=hi)[0]
        assert pl.index == single.index and fb(pl.objective) == fb(single.objective)


def test_repeatable(api):
    prob = G.config_problems(3)[0]
    s = api.Session(prob)
    a = [s.plan_max_load().index for _ in range(3)]
    assert len(set(a)) == 1


@pytest.mark.parametrize("cap", [1, 7, 300])
def test_frontier_overflow_fallback(api, oracle, cap, monkeypatch):
    """A tiny frontier forces the inline depth-first fallback in every pass:
    results must not change."""
    monkeypatch.setenv("CAMELOT_FRONTIER_CAP", str(cap))
    for prob in G.config_problems(2)[:3] + G.config_problems(3):
        got = api.Session(prob).plan_max_load()
        ref = oracle.search(prob, threads=8)[0]
        check_plan(api, prob, got, ref, oracle)
        lam = [[np.float32(0.3) * np.float32(ref.T)]]
        gm = api.Session(prob, n_loads=1).plan_min_resource(lam)[0]
        rm = oracle.search(prob, "min_resource", loads=lam, threads=8)[0]
        check_plan(api, prob, gm, rm, oracle, loads=lam)


@pytest.mark.parametrize("C,n,A,seed", [(12, 3, 1, 1), (16, 2, 1, 2), (9, 4, 2, 3), (3, 7, 1, 4), (2, 8, 2, 5),
                                        (10, 5, 1, 6)])
def test_wide_instantiations(api, oracle, C, n, A, seed):
    """Exercise the CM=16 (9-16 GPUs) and NS=8 (7-8 stages) kernel widths."""
    qstep = 34 if n >= 7 else 25
    prob = G.random_small_problem(100 + seed, n_stages=n, n_gpus=C, n_apps=A, quota_step=qstep,
                                  batches=(1, 8), max_replicas=2 if n < 7 else 1, qos_rho=1.25)
    if oracle.ntot(prob) > 4_000_000:
        pytest.skip("space too large for the in-test oracle")
    got = api.Session(prob).plan_max_load()
    ref = oracle.search(prob, threads=8)[0]
    check_plan(api, prob, got, ref, oracle)
    if ref.index is not None:
        lam = [[np.float32(0.3) * np.float32(ref.T)] * A]
        gm = api.Session(prob, n_loads=1).plan_min_resource(lam)[0]
        rm = oracle.search(prob, "min_resource", loads=lam, threads=8)[0]
        check_plan(api, prob, gm, rm, oracle, loads=lam)
        flat = api.Session(prob, flags=prob.flags | G.F_NO_FILTER).plan_max_load()
        assert flat.index == ref.index and flat.n_feasible == ref.n_feasible


def test_plan_diagnostics_and_trace(api):
    """camelot_plan.search_ns / n_evaluated and the camelot_trace phase marks."""
    prob = G.config_problems(6)[0]
    s = api.Session(prob)
    r = s.plan_max_load()
    st = s.last_stats()
    assert r.n_evaluated == st["cum_scored"] + st["cum_nodes"] > 0
    assert r.search_ns > 0 and abs(r.search_ns - st["t_ns"]) <= 1000
    tr = s.trace()
    tags = [t for t, _ in tr if t < 64]
    assert tags.count(0) >= 1 and 16 in tags and 32 in tags      # launch start, pass 0, CTA reduction
    times = [ns for t, ns in tr if t < 64]
    assert times == sorted(times)


def test_min_resource_unsorted_levels(api, oracle):
    """Several load levels in no particular order (the multi-level bound takes, per
    subtree, the best keys of the levels it can carry -- no ordering assumed)."""
    for prob in G.config_problems(2)[:4] + G.config_problems(3):
        bm = oracle.search(prob, threads=8)[0]
        fr = (0.9, 0.15, 0.6, 1.0, 0.35, 0.05)
        loads = [[np.float32(f) * np.float32(bm.T)] for f in fr]
        got = api.Session(prob, n_loads=len(fr)).plan_min_resource(loads)
        ref = oracle.search(prob, "min_resource", loads=loads, threads=8)
        for k, (g, r) in enumerate(zip(got, ref)):
            check_plan(api, prob, g, r, oracle, loads=[loads[k]])
