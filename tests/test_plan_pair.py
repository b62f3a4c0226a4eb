"""camelot_plan_max_then_min (-m gpu): both policies in one call, the low load
derived on the device from the max-load winner (low load = 30%
of the peak).  It must equal the two separate calls at the load a host caller
computes (float64 product, stored as binary32), and the oracle."""
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


def same(a, b):
    assert a.index == b.index
    assert a.status == b.status and a.violations == b.violations
    if a.index is not None:
        assert fb(a.objective) == fb(b.objective)
        assert (a.gpus_used, a.quota_used) == (b.gpus_used, b.quota_used)
        assert [fb(v) for v in a.stage_latency_ms] == [fb(v) for v in b.stage_latency_ms]


def cases():
    return (G.config_problems(1) + G.config_problems(2)[:4] + G.config_problems(3) + G.config_problems(5)
            + G.config_problems(6))


@pytest.mark.parametrize("frac", [0.3, 0.65, 1.0])
@pytest.mark.parametrize("k", range(len(cases())))
def test_pair_equals_separate_calls(api, k, frac):
    prob = cases()[k]
    s = api.Session(prob, n_loads=1)
    pm, pr = s.plan_max_then_min(frac)
    rm = s.plan_max_load()
    same(pm, rm)
    lam = [[float(np.float32(frac * rm.objective))] * prob.n_apps]
    rr = s.plan_min_resource(lam)[0]
    same(pr, rr)


@pytest.mark.parametrize("k", range(5))
def test_pair_equals_oracle(api, oracle, k):
    prob = (G.config_problems(1) + G.config_problems(2)[:1])[k]
    s = api.Session(prob, n_loads=1)
    pm, pr = s.plan_max_then_min(0.3)
    om = oracle.search(prob, threads=4)[0]
    assert pm.index == om.index and fb(pm.objective) == fb(om.T)
    orr = oracle.search(prob, "min_resource", loads=[[0.3 * om.T] * prob.n_apps], threads=4)[0]
    assert pr.index == orr.index


def test_pair_c4_golden(api):
    """The bench's step on BASELINE config C4 == the oracle's O7 goldens."""
    e = json.load(open(os.path.join(GOLD, "expected_C4-full.json")))
    prob = G.config_problems(4)[0]
    assert prob.sha256() == e["sha256"]
    s = api.Session(prob, n_loads=1)
    s.upload()
    for resident in (False, True):
        pm, pr = s.plan_max_then_min(0.3, resident=resident)
        assert pm.index == e["max_load"]["index"] and fb(pm.objective) == fb(e["max_load"]["T"])
        assert pr.index == e["min_resource"]["index"]
        assert (pr.gpus_used, pr.quota_used) == (e["min_resource"]["u"], e["min_resource"]["U"])
        assert pm.search_ns > 0 and pr.search_ns > 0


def test_pair_infeasible_peak(api):
    """No feasible peak: the min-resource plan is INFEASIBLE with V_LOAD (its load is +inf)."""
    prob = H.linear_thr_problem([1.0, 2.0], [10, 50, 100], qos=1e-6)
    s = api.Session(prob, n_loads=1)
    pm, pr = s.plan_max_then_min(0.3)
    assert pm.index is None and pr.index is None
    from paper_2005_02088_b200 import _lib as L
    assert pm.status == L.INFEASIBLE and pr.status == L.INFEASIBLE and pr.violations == L.V_LOAD


@pytest.mark.parametrize("frac", [0.0, -0.5, 1.5, float("nan")])
def test_pair_bad_fraction(api, frac):
    from paper_2005_02088_b200 import _lib as L
    prob = G.config_problems(1)[0]
    s = api.Session(prob, n_loads=1)
    with pytest.raises(L.CamelotError):
        s.plan_max_then_min(frac)


def test_resident_needs_upload(api):
    """CAMELOT_EXEC_RESIDENT reuses the workspace's problem image: a Session refuses it
    before anything uploaded the problem (the round-2 bench hang), and accepts it after."""
    from paper_2005_02088_b200 import _lib as L
    prob = G.config_problems(2)[0]
    s = api.Session(prob, n_loads=1)
    with pytest.raises(L.CamelotError):
        s.plan_max_then_min(0.3, resident=True)
    ref = s.plan_max_then_min(0.3)          # a non-resident call uploads the image
    got = s.plan_max_then_min(0.3, resident=True)
    assert got[0].index == ref[0].index and got[1].index == ref[1].index
