"""C-ABI checks that need no GPU (-m "not gpu"): the library loads, exports
every entry point include/camelot.h declares, validates arguments on the host
and refuses to compute without a device (no CPU fallback)."""
import ctypes as C
import re

import numpy as np
import pytest
import torch

from gen import problems as G
from paper_2005_02088_b200 import _lib as L


@pytest.fixture(scope="module")
def lib():
    L.build()
    return L.lib()


def header_functions():
    src = open(L.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(camelot_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 10
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(L.EXPORTS)
    assert lib.camelot_version().startswith(b"camelot-b200")


def test_struct_layouts_match_header():
    """sizeof of the ctypes mirrors == the C structs (compiled probe)."""
    import os
    import subprocess
    import tempfile
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "camelot.h"
int main(){printf("%zu %zu %zu %zu %zu\n", sizeof(camelot_cluster), sizeof(camelot_problem),
 sizeof(camelot_exec), sizeof(camelot_plan), offsetof(camelot_plan, objective)); return 0;}
'''
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "p.c")
        open(f, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.check_call(["gcc", "-I", os.path.dirname(L.HEADER), "-o", exe, f])
        out = subprocess.check_output([exe]).decode().split()
    got = [C.sizeof(L.Cluster), C.sizeof(L.Problem), C.sizeof(L.Exec), C.sizeof(L.Plan),
           L.Plan.objective.offset]
    assert [int(v) for v in out] == got


def _cstructs(prob, flags=None):
    keep = dict(app=np.ascontiguousarray(prob.app_of_stage, np.int32),
                qos=np.ascontiguousarray(prob.qos_ms, np.float32),
                Q=np.ascontiguousarray(prob.quota_pct, np.int32),
                S=np.ascontiguousarray(prob.batch, np.int32),
                tab=np.ascontiguousarray(prob.table, np.float32),
                W=np.ascontiguousarray(prob.weights_mib, np.uint32),
                Am=np.ascontiguousarray(prob.act_mib_per_item, np.uint32),
                cf=np.ascontiguousarray(prob.gflop_per_item, np.float32),
                gm=np.ascontiguousarray(prob.bw_sensitivity, np.float32))
    ptr = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    p = L.Problem(n_apps=prob.n_apps, n_stages=prob.n_stages, app_of_stage=ptr(keep["app"], C.c_int32),
                  qos_ms=ptr(keep["qos"], C.c_float), n_quota=len(keep["Q"]), quota_pct=ptr(keep["Q"], C.c_int32),
                  n_batch=len(keep["S"]), batch=ptr(keep["S"], C.c_int32), max_replicas=prob.max_replicas,
                  table=ptr(keep["tab"], C.c_float), weights_mib=ptr(keep["W"], C.c_uint32),
                  act_mib_per_item=ptr(keep["Am"], C.c_uint32), gflop_per_item=ptr(keep["cf"], C.c_float),
                  bw_sensitivity=ptr(keep["gm"], C.c_float), flags=prob.flags if flags is None else flags)
    c = prob.cluster
    cl = L.Cluster(n_gpus=c.n_gpus, quota_per_gpu=c.quota_per_gpu, max_instances=c.max_instances,
                   bw_gbs=c.bw_gbs, mem_mib=c.mem_mib, gflops=c.gflops)
    return p, cl, keep


def test_workspace_and_validation(lib):
    prob = G.config_problems(4)[0]
    p, cl, keep = _cstructs(prob)
    nb = lib.camelot_workspace_bytes(C.byref(p), C.byref(cl), 0)
    assert nb > 0
    nb20 = lib.camelot_workspace_bytes(C.byref(p), C.byref(cl), 20)
    assert nb20 > nb
    # invalid: quota grid not ascending
    keep["Q"][[0, 1]] = keep["Q"][[1, 0]]
    assert lib.camelot_workspace_bytes(C.byref(p), C.byref(cl), 0) == 0
    assert b"ascending" in lib.camelot_last_error()
    keep["Q"][[0, 1]] = keep["Q"][[1, 0]]
    # invalid: NaN in the table
    keep["tab"][0, 0, 0, 1] = np.nan
    assert lib.camelot_workspace_bytes(C.byref(p), C.byref(cl), 0) == 0
    assert b"non-finite" in lib.camelot_last_error()
    keep["tab"][0, 0, 0, 1] = 1.0
    # too many GPUs -> ERANGE message
    cl.n_gpus = 17
    assert lib.camelot_workspace_bytes(C.byref(p), C.byref(cl), 0) == 0
    assert b"n_gpus" in lib.camelot_last_error()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_cpu_fallback(lib):
    prob = G.config_problems(1)[0]
    p, cl, keep = _cstructs(prob)
    buf = (C.c_char * 64)()
    ex = L.Exec(device=0, stream=None, rank=0, world=1, index_lo=0, index_hi=0,
                workspace=C.cast(buf, C.c_void_p), workspace_bytes=64, exec_flags=0)
    out = L.Plan()
    rc = lib.camelot_plan_max_load(C.byref(p), C.byref(cl), C.byref(ex), C.byref(out))
    assert rc == L.ENODEV
    assert b"no CPU fallback" in lib.camelot_last_error()
    with pytest.raises(L.CamelotError):
        from paper_2005_02088_b200 import api
        api.Session(prob)
