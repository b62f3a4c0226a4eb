"""Python API over the C ABI (include/camelot.h): argument marshalling only.

PyTorch provides the device workspace, the stream and (for N > 1 GPUs) the
process group; every step of the allocation search runs in libcamelot.so's
kernels.  A problem is any object with the attributes of gen.problems.Problem
(Table 2 variables of the paper).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Tuple, List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L


@dataclasses.dataclass
class PlanResult:
    """One optimal plan (camelot_plan)."""
    status: int
    index: Optional[int]
    batch: List[int]
    replicas: List[int]
    quota_pct: List[int]
    gpu_of_instance: List[List[int]]
    stage_latency_ms: List[float]
    stage_throughput_qps: List[float]
    kappa: List[float]
    e2e_latency_ms: List[float]
    throughput_qps: List[float]
    objective: float
    quota_used: int
    gpus_used: int
    eq2_gpus: int
    violations: int
    n_feasible: int
    n_scored: int
    n_covered: int
    comm_ms: List[float] = None   # COMM: hand-over time of edge i -> i+1 (ms)
    n_evaluated: int = 0          # leaves + inner nodes evaluated (cascade + main pass)
    search_ns: int = 0            # device time of the search (ns), 0 if unknown

    @property
    def feasible(self) -> bool:
        return self.status == L.OK


def _plan(p: L.Plan, n: int, A: int) -> PlanResult:
    none = p.index == (1 << 64) - 1
    goi = [[g for g in p.gpu_of_instance[i * L.MAX_REPLICAS:(i + 1) * L.MAX_REPLICAS] if g >= 0]
           for i in range(n)]
    return PlanResult(p.status, None if none else int(p.index), list(p.batch[:A]),
                      list(p.replicas[:n]), list(p.quota_pct[:n]), goi,
                      list(p.stage_latency_ms[:n]), list(p.stage_throughput_qps[:n]),
                      list(p.kappa[:n]), list(p.e2e_latency_ms[:A]), list(p.throughput_qps[:A]),
                      p.objective, p.quota_used, p.gpus_used, p.eq2_gpus, p.violations,
                      int(p.n_feasible), int(p.n_scored), int(p.n_covered), list(p.comm_ms[:n]),
                      int(p.n_evaluated), int(p.search_ns))


class Session:
    """One problem bound to a device workspace (torch uint8 tensor) and a stream."""

    def __init__(self, problem, device: Optional[int] = None, n_loads: int = 0,
                 flags: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None):
        L.lib()
        if not torch.cuda.is_available():
            raise L.CamelotError(L.ENODEV, "no CUDA device (there is no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else device
        self.stream = stream
        self.problem = problem
        self.n, self.A = int(problem.n_stages), int(problem.n_apps)
        pin = True
        self._keep = dict(
            app=np.ascontiguousarray(problem.app_of_stage, np.int32),
            qos=np.ascontiguousarray(problem.qos_ms, np.float32),
            Q=np.ascontiguousarray(problem.quota_pct, np.int32),
            S=np.ascontiguousarray(problem.batch, np.int32),
            W=np.ascontiguousarray(problem.weights_mib, np.uint32),
            Am=np.ascontiguousarray(problem.act_mib_per_item, np.uint32),
            cf=np.ascontiguousarray(problem.gflop_per_item, np.float32),
            gm=np.ascontiguousarray(problem.bw_sensitivity, np.float32),
            cm=np.ascontiguousarray(getattr(problem, "comm_mb_per_item", None)
                                    if getattr(problem, "comm_mb_per_item", None) is not None
                                    else np.zeros(self.n), np.float32),
        )
        tab = np.ascontiguousarray(problem.table, np.float32)
        # pinned host copy of the predictor tables (the only sizeable input)
        self._tab = torch.from_numpy(tab.copy()).pin_memory() if pin else torch.from_numpy(tab)
        k = self._keep
        ptr = lambda a, t: a.ctypes.data_as(C.POINTER(t))
        self.cprob = L.Problem(
            n_apps=self.A, n_stages=self.n, app_of_stage=ptr(k["app"], C.c_int32),
            qos_ms=ptr(k["qos"], C.c_float), n_quota=len(k["Q"]), quota_pct=ptr(k["Q"], C.c_int32),
            n_batch=len(k["S"]), batch=ptr(k["S"], C.c_int32), max_replicas=int(problem.max_replicas),
            table=C.cast(self._tab.data_ptr(), C.POINTER(C.c_float)),
            weights_mib=ptr(k["W"], C.c_uint32), act_mib_per_item=ptr(k["Am"], C.c_uint32),
            gflop_per_item=ptr(k["cf"], C.c_float), bw_sensitivity=ptr(k["gm"], C.c_float),
            flags=int(problem.flags if flags is None else flags), comm_mb_per_item=ptr(k["cm"], C.c_float))
        c = problem.cluster
        self.ccl = L.Cluster(n_gpus=int(c.n_gpus), quota_per_gpu=int(c.quota_per_gpu),
                             max_instances=int(c.max_instances), bw_gbs=float(c.bw_gbs),
                             mem_mib=int(c.mem_mib), gflops=float(c.gflops),
                             link_gbs=float(getattr(c, "link_gbs", 1.0)), ipc_ms=float(getattr(c, "ipc_ms", 0.0)))
        self.ws = None
        self._uploaded = False
        self._ensure(n_loads)

    # ------------------------------------------------------------------ plumbing
    def _ensure(self, n_loads: int):
        nb = L.lib().camelot_workspace_bytes(C.byref(self.cprob), C.byref(self.ccl), int(n_loads))
        if nb == 0:
            raise L.CamelotError(L.EINVAL, L.lib().camelot_last_error().decode())
        if self.ws is None or self.ws.numel() < nb:
            self.ws = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{self.device}")
            self._uploaded = False

    def _stream_ptr(self):
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        return s.cuda_stream

    def exec(self, rank: int = 0, world: int = 1, lo: int = 0, hi: int = 0, resident: bool = False) -> L.Exec:
        if resident and not self._uploaded:
            # CAMELOT_EXEC_RESIDENT reuses the problem image already in the workspace:
            # a workspace that never saw camelot_upload holds no problem
            raise L.CamelotError(L.EINVAL, "resident=True before upload() on this session")
        if not resident:
            self._uploaded = True   # a non-resident call uploads the problem image itself
        return L.Exec(device=self.device, stream=self._stream_ptr(), rank=rank, world=world,
                      index_lo=lo, index_hi=hi, workspace=self.ws.data_ptr(),
                      workspace_bytes=self.ws.numel(), exec_flags=L.EXEC_RESIDENT if resident else 0)

    def _loads(self, loads):
        arr = np.ascontiguousarray(np.asarray(loads, np.float32).reshape(-1, self.A))
        return arr, arr.shape[0]

    # ------------------------------------------------------------------ entry points
    def upload(self):
        ex = self.exec()
        L.check(L.lib().camelot_upload(C.byref(self.cprob), C.byref(self.ccl), C.byref(ex)), False)
        self._uploaded = True

    def plan_max_load(self, lo: int = 0, hi: int = 0, resident: bool = False) -> PlanResult:
        out = L.Plan()
        ex = self.exec(lo=lo, hi=hi, resident=resident)
        L.check(L.lib().camelot_plan_max_load(C.byref(self.cprob), C.byref(self.ccl), C.byref(ex), C.byref(out)))
        return _plan(out, self.n, self.A)

    def plan_min_resource(self, loads, lo: int = 0, hi: int = 0, resident: bool = False) -> List[PlanResult]:
        arr, nl = self._loads(loads)
        self._ensure(nl)
        out = (L.Plan * nl)()
        ex = self.exec(lo=lo, hi=hi, resident=resident)
        L.check(L.lib().camelot_plan_min_resource(C.byref(self.cprob), C.byref(self.ccl),
                                                  arr.ctypes.data_as(C.POINTER(C.c_float)), nl,
                                                  C.byref(ex), out))
        return [_plan(o, self.n, self.A) for o in out]

    def plan_max_then_min(self, low_load_frac: float = 0.3, lo: int = 0, hi: int = 0,
                          resident: bool = False) -> Tuple[PlanResult, PlanResult]:
        """Max-load plan, then the min-resource plan at low_load_frac x its T*
        (PAPER.md L1088), the load derived on the device: one call, one host
        synchronisation (camelot_plan_max_then_min)."""
        out = (L.Plan * 2)()
        ex = self.exec(lo=lo, hi=hi, resident=resident)
        L.check(L.lib().camelot_plan_max_then_min(C.byref(self.cprob), C.byref(self.ccl), float(low_load_frac),
                                                  C.byref(ex), out))
        return _plan(out[0], self.n, self.A), _plan(out[1], self.n, self.A)

    def predict(self, batch: Sequence[int], replicas: Sequence[int], quota_pct: Sequence[int],
                loads=None) -> PlanResult:
        b = (C.c_int32 * L.MAX_APPS)(*batch)
        r = (C.c_int32 * L.MAX_STAGES)(*replicas)
        q = (C.c_int32 * L.MAX_STAGES)(*quota_pct)
        out = L.Plan()
        if loads is not None:
            arr, nl = self._loads(loads)
            lp, nl = arr.ctypes.data_as(C.POINTER(C.c_float)), 1
        else:
            lp, nl = None, 0
        ex = self.exec()
        L.check(L.lib().camelot_predict(C.byref(self.cprob), C.byref(self.ccl), b, r, q, lp, nl,
                                        C.byref(ex), C.byref(out)))
        return _plan(out, self.n, self.A)

    def predict_index(self, x: int, loads=None) -> PlanResult:
        """camelot_predict_index: score the candidate with canonical index x (the
        library decodes the digits on the device)."""
        out = L.Plan()
        if loads is not None:
            arr, _ = self._loads(loads)
            lp, nl = arr.ctypes.data_as(C.POINTER(C.c_float)), 1
        else:
            lp, nl = None, 0
        ex = self.exec()
        L.check(L.lib().camelot_predict_index(C.byref(self.cprob), C.byref(self.ccl), int(x), lp, nl,
                                              C.byref(ex), C.byref(out)))
        return _plan(out, self.n, self.A)

    def score_range(self, lo: int, hi: int):
        """Device vectors (verdict u8, T f32, u i32, U i32) of every candidate in [lo, hi)."""
        m = hi - lo
        dev = f"cuda:{self.device}"
        v = torch.empty(m, dtype=torch.uint8, device=dev)
        T = torch.empty(m, dtype=torch.float32, device=dev)
        u = torch.empty(m, dtype=torch.int32, device=dev)
        U = torch.empty(m, dtype=torch.int32, device=dev)
        ex = self.exec()
        L.check(L.lib().camelot_score_range(C.byref(self.cprob), C.byref(self.ccl), lo, hi, C.byref(ex),
                                            v.data_ptr(), T.data_ptr(), u.data_ptr(), U.data_ptr()), False)
        return v, T, u, U

    def search_local(self, policy: int, loads=None, rank: int = 0, world: int = 1, lo: int = 0,
                     hi: int = 0, resident: bool = False, keys: Optional[torch.Tensor] = None) -> torch.Tensor:
        """This rank's shard -> device int64 keys (sign-mapped; all_reduce MIN them)."""
        if policy == L.POLICY_MIN_RESOURCE:
            arr, nl = self._loads(loads)
            lp = arr.ctypes.data_as(C.POINTER(C.c_float))
            self._ensure(nl)
        else:
            lp, nl = None, 0
        nk = max(1, nl)
        if keys is None:
            keys = torch.empty(nk, dtype=torch.int64, device=f"cuda:{self.device}")
        ex = self.exec(rank=rank, world=world, lo=lo, hi=hi, resident=resident)
        L.check(L.lib().camelot_search_local(C.byref(self.cprob), C.byref(self.ccl), policy, lp, nl,
                                             C.byref(ex), keys.data_ptr()), False)
        self._last_loads = (lp, nl, arr if policy else None)
        return keys

    def finalize(self, policy: int, keys: torch.Tensor, loads=None, rank: int = 0, world: int = 1,
                 lo: int = 0, hi: int = 0) -> List[PlanResult]:
        if policy == L.POLICY_MIN_RESOURCE:
            arr, nl = self._loads(loads)
            lp = arr.ctypes.data_as(C.POINTER(C.c_float))
        else:
            lp, nl = None, 0
        nk = max(1, nl)
        out = (L.Plan * nk)()
        ex = self.exec(rank=rank, world=world, lo=lo, hi=hi)
        L.check(L.lib().camelot_finalize(C.byref(self.cprob), C.byref(self.ccl), policy, lp, nl,
                                         keys.data_ptr(), C.byref(ex), out))
        return [_plan(o, self.n, self.A) for o in out]

    def sa(self, policy: int = 0, loads=None, seed: int = 1, chains: int = 4096, iters: int = 1000,
           p0: float = 0.3, cool: float = 0.995, per_chain: bool = False):
        """The paper's simulated annealing (NEXT-1) on the device.  Returns the best
        plan over all chains, plus (per_chain=True) the device tensors of each
        chain's best index and objective key."""
        if policy == L.POLICY_MIN_RESOURCE:
            arr, _ = self._loads(loads)
            lp = arr.ctypes.data_as(C.POINTER(C.c_float))
        else:
            lp = None
        dev = f"cuda:{self.device}"
        ci = torch.empty(chains, dtype=torch.int64, device=dev) if per_chain else None
        ck = torch.empty(chains, dtype=torch.int32, device=dev) if per_chain else None
        out = L.Plan()
        ex = self.exec()
        L.check(L.lib().camelot_sa(C.byref(self.cprob), C.byref(self.ccl), policy, lp, seed, chains, iters,
                                   p0, cool, C.byref(ex), C.byref(out),
                                   ci.data_ptr() if per_chain else None, ck.data_ptr() if per_chain else None))
        res = _plan(out, self.n, self.A)
        return (res, ci, ck) if per_chain else res

    def last_stats(self):
        out = (C.c_uint64 * 8)()
        ex = self.exec()
        L.check(L.lib().camelot_last_stats(C.byref(ex), out), False)
        return dict(n_scored=out[0], n_nodes=out[1], n_feasible=out[2], t_ns=out[3], items=out[4],
                    launches=out[5], cum_scored=out[6], cum_nodes=out[7])

    def simulate(self, batch, replicas, quota_pct, loads, n_queries: int = 100000, warmup: int = 10000,
                 seed: int = 1, n_sims: int = 1):
        """NEXT-4: simulated (p99, mean) latency in ms of an explicit plan at loads[A]
        QPS, for n_sims independent streams: two lists [n_sims][A]."""
        A = self.A
        nb = L.lib().camelot_simulate_workspace_bytes(C.byref(self.cprob), C.byref(self.ccl), int(n_queries),
                                                      int(n_sims))
        if nb == 0:
            raise L.CamelotError(L.EINVAL, L.lib().camelot_last_error().decode())
        ws = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{self.device}")
        ex = self.exec()
        ex.workspace, ex.workspace_bytes = ws.data_ptr(), nb
        ip = lambda v: (C.c_int32 * len(v))(*[int(a) for a in v])
        lam = (C.c_float * A)(*[float(v) for v in loads])
        p99 = (C.c_double * (A * n_sims))()
        mean = (C.c_double * (A * n_sims))()
        L.check(L.lib().camelot_simulate(C.byref(self.cprob), C.byref(self.ccl), ip(batch), ip(replicas),
                                         ip(quota_pct), lam, int(n_queries), int(warmup), int(seed), int(n_sims),
                                         C.byref(ex), p99, mean), False)
        return ([list(p99[k * A:(k + 1) * A]) for k in range(n_sims)],
                [list(mean[k * A:(k + 1) * A]) for k in range(n_sims)])

    def trace(self):
        """Phase timestamps of the last search: [(tag, ns since the first mark)]."""
        out = (C.c_uint64 * 256)()
        n = L.lib().camelot_trace(C.byref(self.exec()), out, 256)
        L.check(min(n, 0), False)
        if n == 0:
            return []
        m = (1 << 48) - 1
        t0 = next((out[i] & m for i in range(min(n, 256)) if (out[i] >> 48) < 64), 0)   # the first timestamp
        # tags < 64 are timestamps (ns since the first mark), tags >= 64 are values
        return [(out[i] >> 48, (out[i] & m) - (t0 if (out[i] >> 48) < 64 else 0)) for i in range(min(n, 256))]


# ---------------------------------------------------------------------- functional API
def tables_from_trees(trees, batch, quota_pct, device: Optional[int] = None) -> torch.Tensor:
    """NEXT-3: the predictor table [n][nS][nQ][4] of a problem built ON THE DEVICE
    from its decision-tree models (3 per stage: duration, throughput, bandwidth;
    gen.dt.Tree-like objects) evaluated at every (batch, quota) grid point."""
    L.lib()
    dev = torch.cuda.current_device() if device is None else device
    keep = []
    arr = (L.Tree * len(trees))()
    for t, tr in enumerate(trees):
        f, th, le, ri = (np.ascontiguousarray(a, np.int32) for a in (tr.feature, tr.threshold, tr.left, tr.right))
        v = np.ascontiguousarray(tr.value, np.float32)
        keep += [f, th, le, ri, v]
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
        arr[t] = L.Tree(int(f.shape[0]), ip(f), ip(th), ip(le), ip(ri), v.ctypes.data_as(C.POINTER(C.c_float)))
    S = np.ascontiguousarray(batch, np.int32)
    Q = np.ascontiguousarray(quota_pct, np.int32)
    nb = L.lib().camelot_trees_workspace_bytes(len(trees), arr, len(S), len(Q))
    if nb == 0:
        raise L.CamelotError(L.EINVAL, L.lib().camelot_last_error().decode())
    ws = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{dev}")
    out = torch.empty((len(trees) // 3, len(S), len(Q), 4), dtype=torch.float32, device=f"cuda:{dev}")
    ex = L.Exec(device=dev, stream=torch.cuda.current_stream(dev).cuda_stream, rank=0, world=1, index_lo=0,
                index_hi=0, workspace=ws.data_ptr(), workspace_bytes=nb, exec_flags=0)
    L.check(L.lib().camelot_tables_from_trees(len(trees) // 3, arr, len(S), S.ctypes.data_as(C.POINTER(C.c_int32)),
                                              len(Q), Q.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(ex),
                                              out.data_ptr()), False)
    return out


def plan_max_load(problem, **kw) -> PlanResult:
    return Session(problem, device=kw.pop("device", None)).plan_max_load(**kw)


def plan_min_resource(problem, loads, **kw) -> List[PlanResult]:
    s = Session(problem, device=kw.pop("device", None), n_loads=np.asarray(loads).reshape(-1, problem.n_apps).shape[0])
    return s.plan_min_resource(loads, **kw)


def predict(problem, batch, replicas, quota_pct, loads=None, device=None) -> PlanResult:
    return Session(problem, device=device).predict(batch, replicas, quota_pct, loads)


def plan_distributed(session: Session, policy: int, loads=None, group=None, lo: int = 0, hi: int = 0,
                     resident: bool = False) -> List[PlanResult]:
    """Multi-GPU plan: this rank searches chunks c = rank (mod world); ONE
    all_reduce(MIN) of the packed int64 keys over the process group (NCCL over
    NVLink); every rank then resolves and scores the winner locally."""
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    keys = session.search_local(policy, loads, rank=rank, world=world, lo=lo, hi=hi, resident=resident)
    if world > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    return session.finalize(policy, keys, loads, rank=rank, world=world, lo=lo, hi=hi)


# ---------------------------------------------------------------------- key helpers
SIGN = 1 << 63


def pack_key(objkey: int, low: int) -> int:
    """Packed 64-bit key as camelot_search_local writes it: (objective key << 32 |
    chunk-or-index), XOR 2^63 so that a signed int64 MIN equals the unsigned min
    (include/camelot.h).  objkey 0xFFFFFFFF with low 0xFFFFFFFF = no candidate."""
    u = ((objkey & 0xFFFFFFFF) << 32) | (low & 0xFFFFFFFF)
    v = u ^ SIGN
    return v - (1 << 64) if v >= SIGN else v


def unpack_key(k: int):
    u = (k + (1 << 64) if k < 0 else k) ^ SIGN
    return u >> 32, u & 0xFFFFFFFF
