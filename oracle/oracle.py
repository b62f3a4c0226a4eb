"""ctypes wrapper of the plain CPU oracle (oracle/camelot_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product path
(paper_2005_02088_b200/) never imports this module, and this module never
imports the product package.  It consumes problems from gen/problems.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "camelot_oracle.c")
LIB = os.path.join(HERE, "libcamelot_oracle.so")

MAX_STAGES, MAX_APPS, MAX_GPUS, MAX_REPL, MAX_LOADS = 8, 2, 16, 16, 64
V_QUOTA, V_INST, V_MEM, V_BW, V_QOS, V_LOAD, V_EQ2 = 1, 2, 4, 8, 16, 32, 64
NONE = (1 << 64) - 1


def build(force: bool = False) -> str:
    """Compile the oracle: plain C99, binary32 without FMA contraction."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-std=gnu99", "-O2", "-fPIC", "-shared", "-fopenmp",
               "-ffp-contract=off", "-fno-fast-math", "-fexcess-precision=standard",
               "-o", LIB, SRC, "-lm"]
        subprocess.check_call(cmd)
    return LIB


class OcProblem(C.Structure):
    _fields_ = [
        ("A", C.c_int32), ("n", C.c_int32),
        ("app", C.POINTER(C.c_int32)), ("qos", C.POINTER(C.c_float)),
        ("nQ", C.c_int32), ("Q", C.POINTER(C.c_int32)),
        ("nS", C.c_int32), ("S", C.POINTER(C.c_int32)),
        ("Rmax", C.c_int32),
        ("tab", C.POINTER(C.c_float)),
        ("W", C.POINTER(C.c_uint32)), ("Am", C.POINTER(C.c_uint32)),
        ("cflop", C.POINTER(C.c_float)), ("gamma", C.POINTER(C.c_float)),
        ("flags", C.c_uint32),
        ("C", C.c_int32), ("R", C.c_int32), ("I", C.c_int32),
        ("BW", C.c_float), ("FM", C.c_uint32), ("G", C.c_float),
        ("comm_mb", C.POINTER(C.c_float)), ("link_gbs", C.c_float), ("ipc_ms", C.c_float),
    ]


class OcScore(C.Structure):
    _fields_ = [
        ("verdict", C.c_uint32), ("place_viol", C.c_uint32),
        ("T", C.c_float), ("u", C.c_int32), ("U", C.c_int32),
        ("Tmin", C.c_float * MAX_APPS), ("Lsum", C.c_float * MAX_APPS),
        ("L", C.c_float * MAX_STAGES), ("Ti", C.c_float * MAX_STAGES),
        ("kappa", C.c_float * MAX_STAGES),
        ("L64", C.c_double * MAX_STAGES), ("T64", C.c_double * MAX_STAGES),
        ("Lsum64", C.c_double * MAX_APPS),
        ("gpu_of_instance", C.c_int8 * (MAX_STAGES * MAX_REPL)),
        ("dem", C.c_float * MAX_GPUS),
        ("comm", C.c_float * MAX_STAGES),
        ("level_verdict", C.c_uint32 * MAX_LOADS),
        ("eq2_y", C.c_int32 * MAX_LOADS),
    ]


class OcBest(C.Structure):
    _fields_ = [
        ("index", C.c_uint64), ("T", C.c_float), ("u", C.c_int32), ("U", C.c_int32),
        ("n_feasible", C.c_uint64), ("n_scanned", C.c_uint64),
        ("hist", C.c_uint64 * 7),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oc_ntot.restype = C.c_uint64
        _lib.oc_encode.restype = C.c_uint64
        assert _lib.oc_sizeof_score() == C.sizeof(OcScore), "oc_score_t layout"
        assert _lib.oc_sizeof_best() == C.sizeof(OcBest), "oc_best_t layout"
    return _lib


class Handle:
    """Keeps the numpy buffers of one problem alive while the oracle reads them."""

    def __init__(self, prob, flags: Optional[int] = None):
        p = prob
        self.keep = dict(
            app=np.ascontiguousarray(p.app_of_stage, np.int32),
            qos=np.ascontiguousarray(p.qos_ms, np.float32),
            Q=np.ascontiguousarray(p.quota_pct, np.int32),
            S=np.ascontiguousarray(p.batch, np.int32),
            tab=np.ascontiguousarray(p.table, np.float32),
            W=np.ascontiguousarray(p.weights_mib, np.uint32),
            Am=np.ascontiguousarray(p.act_mib_per_item, np.uint32),
            cflop=np.ascontiguousarray(p.gflop_per_item, np.float32),
            gamma=np.ascontiguousarray(p.bw_sensitivity, np.float32),
            comm=np.ascontiguousarray(p.comm_mb_per_item if p.comm_mb_per_item is not None
                                      else np.zeros(p.n_stages), np.float32),
        )
        k = self.keep
        ptr = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        c = p.cluster
        self.s = OcProblem(
            A=p.n_apps, n=p.n_stages, app=ptr(k["app"], C.c_int32),
            qos=ptr(k["qos"], C.c_float), nQ=len(k["Q"]), Q=ptr(k["Q"], C.c_int32),
            nS=len(k["S"]), S=ptr(k["S"], C.c_int32), Rmax=p.max_replicas,
            tab=ptr(k["tab"], C.c_float), W=ptr(k["W"], C.c_uint32),
            Am=ptr(k["Am"], C.c_uint32), cflop=ptr(k["cflop"], C.c_float),
            gamma=ptr(k["gamma"], C.c_float),
            flags=p.flags if flags is None else flags,
            C=c.n_gpus, R=c.quota_per_gpu, I=c.max_instances, BW=c.bw_gbs,
            FM=c.mem_mib, G=c.gflops,
            comm_mb=ptr(k["comm"], C.c_float), link_gbs=c.link_gbs, ipc_ms=c.ipc_ms)
        self.A, self.n = p.n_apps, p.n_stages
        self.Rmax = p.max_replicas

    @property
    def ref(self):
        return C.byref(self.s)


def validate(prob) -> int:
    h = Handle(prob)
    return lib().oc_validate(h.ref)


def ntot(prob) -> int:
    h = Handle(prob)
    return int(lib().oc_ntot(h.ref))


def decode(prob, x: int):
    h = Handle(prob)
    beta = (C.c_int32 * MAX_APPS)()
    rho = (C.c_int32 * MAX_STAGES)()
    theta = (C.c_int32 * MAX_STAGES)()
    lib().oc_decode(h.ref, C.c_uint64(x), beta, rho, theta)
    return list(beta[:h.A]), list(rho[:h.n]), list(theta[:h.n])


def encode(prob, beta, rho, theta) -> int:
    h = Handle(prob)
    b = (C.c_int32 * MAX_APPS)(*beta)
    r = (C.c_int32 * MAX_STAGES)(*rho)
    t = (C.c_int32 * MAX_STAGES)(*theta)
    return int(lib().oc_encode(h.ref, b, r, t))


@dataclass
class Score:
    verdict: int
    place_viol: int
    T: float
    u: int
    U: int
    Tmin: List[float]
    Lsum: List[float]
    L: List[float]
    Ti: List[float]
    kappa: List[float]
    L64: List[float]
    T64: List[float]
    Lsum64: List[float]
    gpu_of_instance: List[List[int]]
    dem: List[float]
    level_verdict: List[int]
    eq2_y: List[int]
    comm: List[float] = None   # COMM: hand-over time of edge i -> i+1 (ms)


def _loads_arr(loads, A):
    if loads is None:
        return None, 0
    arr = np.ascontiguousarray(np.asarray(loads, np.float32).reshape(-1, A))
    return arr, arr.shape[0]


def score(prob, x: int = None, digits=None, loads=None, flags=None) -> Score:
    """oracle_predict: score one candidate, by index or by (beta, rho, theta)."""
    h = Handle(prob, flags)
    out = OcScore()
    la, L = _loads_arr(loads, h.A)
    lp = la.ctypes.data_as(C.POINTER(C.c_float)) if la is not None else None
    if digits is not None:
        beta, rho, theta = digits
        b = (C.c_int32 * MAX_APPS)(*beta)
        r = (C.c_int32 * MAX_STAGES)(*rho)
        t = (C.c_int32 * MAX_STAGES)(*theta)
        lib().oc_score(h.ref, b, r, t, lp, L, C.byref(out))
    else:
        lib().oc_score_index(h.ref, C.c_uint64(x), lp, L, C.byref(out))
    n, A = h.n, h.A
    goi = [[g for g in out.gpu_of_instance[i * MAX_REPL:(i + 1) * MAX_REPL] if g >= 0]
           for i in range(n)]
    return Score(out.verdict, out.place_viol, out.T, out.u, out.U,
                 list(out.Tmin[:A]), list(out.Lsum[:A]), list(out.L[:n]),
                 list(out.Ti[:n]), list(out.kappa[:n]), list(out.L64[:n]),
                 list(out.T64[:n]), list(out.Lsum64[:A]), goi,
                 list(out.dem[:prob.cluster.n_gpus]), list(out.level_verdict[:L]),
                 list(out.eq2_y[:L]), list(out.comm[:n]))


def score_range(prob, lo: int, hi: int, flags=None):
    """Verdict / T / u / U vectors over candidate indices [lo, hi)."""
    h = Handle(prob, flags)
    m = hi - lo
    v = np.zeros(m, np.uint8)
    T = np.zeros(m, np.float32)
    u = np.zeros(m, np.int32)
    U = np.zeros(m, np.int32)
    lib().oc_score_range(h.ref, C.c_uint64(lo), C.c_uint64(hi),
                         v.ctypes.data_as(C.POINTER(C.c_uint8)),
                         T.ctypes.data_as(C.POINTER(C.c_float)),
                         u.ctypes.data_as(C.POINTER(C.c_int32)),
                         U.ctypes.data_as(C.POINTER(C.c_int32)))
    return v, T, u, U


@dataclass
class Best:
    index: Optional[int]   # None = infeasible
    T: float
    u: int
    U: int
    n_feasible: int
    n_scanned: int
    hist: List[int]


def search(prob, policy: str = "max_load", loads=None, lo: int = 0, hi: Optional[int] = None,
           threads: int = 1, flags=None) -> List[Best]:
    """oracle_search: exhaustive scan of [lo, hi) (default: the whole space).

    policy "max_load" returns [Best]; "min_resource" returns one Best per load
    level (loads: [L][A] QPS)."""
    h = Handle(prob, flags)
    pol = 0 if policy == "max_load" else 1
    la, L = _loads_arr(loads, h.A)
    if pol == 1 and L == 0:
        raise ValueError("min_resource needs loads")
    nb = 1 if pol == 0 else L
    out = (OcBest * nb)()
    if hi is None:
        hi = int(lib().oc_ntot(h.ref))
    lp = la.ctypes.data_as(C.POINTER(C.c_float)) if la is not None else None
    rc = lib().oc_search(h.ref, pol, lp, L, C.c_uint64(lo), C.c_uint64(hi), threads, out)
    if rc != 0:
        raise ValueError(f"oracle_search rc={rc}")
    res = []
    for b in out:
        res.append(Best(None if b.index == NONE else int(b.index), b.T, b.u, b.U,
                        int(b.n_feasible), int(b.n_scanned), list(b.hist)))
    return res


def eq2_y(prob, beta, lam) -> int:
    h = Handle(prob)
    b = (C.c_int32 * MAX_APPS)(*beta)
    l = (C.c_float * MAX_APPS)(*lam)
    return int(lib().oc_eq2_y(h.ref, b, l))


class OcSaChain(C.Structure):
    _fields_ = [("best_index", C.c_uint64), ("best_key", C.c_uint32), ("accepted", C.c_uint32),
                ("final_index", C.c_uint64)]


def sa(prob, policy: str = "max_load", load=None, seed: int = 1, chain_lo: int = 0, chain_hi: int = 64,
       iters: int = 300, p0: float = 0.3, cool: float = 0.995, flags=None):
    """oracle SA (the paper's algorithm): per-chain
    (best_index or None, best_key, accepted, final_index)."""
    h = Handle(prob, flags)
    assert lib().oc_sizeof_sa() == C.sizeof(OcSaChain)
    pol = 0 if policy == "max_load" else 1
    la = None
    if pol == 1:
        la = (C.c_float * MAX_APPS)(*[float(v) for v in np.asarray(load, np.float32).reshape(-1)])
    out = (OcSaChain * (chain_hi - chain_lo))()
    lib().oc_sa.argtypes = [C.POINTER(OcProblem), C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int,
                            C.c_float, C.c_float, C.c_void_p]
    rc = lib().oc_sa(h.ref, pol, C.cast(la, C.c_void_p) if la is not None else None, seed, chain_lo, chain_hi,
                     iters, p0, cool, C.cast(out, C.c_void_p))
    if rc != 0:
        raise ValueError(f"oracle sa rc={rc}")
    return [(None if r.best_index == NONE else int(r.best_index), int(r.best_key), int(r.accepted),
             int(r.final_index)) for r in out]


# ---------------------------------------------------------------------- NEXT-3
def tree_eval(tree, s: int, p: int) -> float:
    """oc_tree_eval: one decision-tree prediction at batch s, quota p."""
    f = lib().oc_tree_eval
    f.restype = C.c_float
    a = [np.ascontiguousarray(v) for v in (tree.feature, tree.threshold, tree.left, tree.right)]
    v = np.ascontiguousarray(tree.value, np.float32)
    ip = lambda x: x.ctypes.data_as(C.POINTER(C.c_int32))
    return float(f(ip(a[0]), ip(a[1]), ip(a[2]), ip(a[3]), v.ctypes.data_as(C.POINTER(C.c_float)),
                   C.c_int32(tree.n_nodes), C.c_int32(int(s)), C.c_int32(int(p))))


def tree_tables(trees, batch, quota) -> np.ndarray:
    """The predictor table [n][nS][nQ][4] = (dur, thr, bw, 0) from 3 trees per stage
    (component order), evaluated point by point."""
    n = len(trees) // 3
    tab = np.zeros((n, len(batch), len(quota), 4), np.float32)
    for t, tree in enumerate(trees):
        for b, s in enumerate(batch):
            for q, p in enumerate(quota):
                tab[t // 3, b, q, t % 3] = tree_eval(tree, s, p)
    return tab


# ---------------------------------------------------------------------- NEXT-4
def simulate(prob, x: int, loads, n_queries: int = 100000, warmup: int = 10000, seed: int = 1, sim: int = 0,
             flags=None):
    """oc_simulate: (p99[A], mean[A]) latency (ms) of candidate x at loads[A] QPS."""
    h = Handle(prob, flags)
    beta, rho, theta = decode(prob, x)
    b = (C.c_int32 * MAX_APPS)(*beta)
    r = (C.c_int32 * MAX_STAGES)(*rho)
    t = (C.c_int32 * MAX_STAGES)(*theta)
    lam = (C.c_float * MAX_APPS)(*[float(v) for v in loads])
    p99 = (C.c_double * MAX_APPS)()
    mean = (C.c_double * MAX_APPS)()
    f = lib().oc_simulate
    f.argtypes = [C.POINTER(OcProblem), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                  C.POINTER(C.c_float), C.c_int64, C.c_int64, C.c_uint64, C.c_uint64,
                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
    rc = f(h.ref, b, r, t, lam, n_queries, warmup, seed, sim, p99, mean)
    if rc != 0:
        raise ValueError(f"oc_simulate rc={rc}")
    A = prob.n_apps
    return list(p99[:A]), list(mean[:A])


# ---------------------------------------------------------------------- O7
def search_filtered(prob, policy: str = "max_load", load=None, T_inc: float = 0.0, u_inc: int = 0,
                    U_inc: int = 0, threads: int = 1, flags=None) -> Best:
    """O7: the exhaustive scan restricted to the candidates that
    survive the separable necessary-condition filters against an incumbent (a
    known feasible candidate's objective: T_inc for max-load; (u_inc, U_inc) for
    min-resource at ONE load level `load` [A]).  Same answer as search() over the
    whole space; n_scanned = candidates scored."""
    h = Handle(prob, flags)
    pol = 0 if policy == "max_load" else 1
    la = (C.c_float * MAX_APPS)()
    if pol == 1:
        vals = [float(v) for v in np.asarray(load, np.float32).reshape(-1)]
        for a, v in enumerate(vals):
            la[a] = v
    out = OcBest()
    f = lib().oc_search_filtered
    f.argtypes = [C.POINTER(OcProblem), C.c_int, C.POINTER(C.c_float), C.c_float, C.c_int32, C.c_int32,
                  C.c_int, C.POINTER(OcBest)]
    rc = f(h.ref, pol, la, float(np.float32(T_inc)), int(u_inc), int(U_inc), int(threads), C.byref(out))
    if rc != 0:
        raise ValueError(f"oc_search_filtered rc={rc}")
    return Best(None if out.index == NONE else int(out.index), out.T, out.u, out.U,
                int(out.n_feasible), int(out.n_scanned), list(out.hist))
