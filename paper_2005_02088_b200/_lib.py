"""ctypes declarations of include/camelot.h and the loader of libcamelot.so.

Argument marshalling only: every step of the search runs in the CUDA kernels of
libcamelot.so.  If the library is missing the import of the compute entry
points raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("CAMELOT_LIB") or os.path.join(HERE, "libcamelot.so")   # override: experiments only
HEADER = os.path.join(ROOT, "include", "camelot.h")

MAX_STAGES, MAX_APPS, MAX_GPUS, MAX_REPLICAS, MAX_LOADS = 8, 2, 16, 16, 64
OK, INFEASIBLE, EINVAL, ERANGE, ECUDA, ENODEV, ENOMEM = 0, 1, -1, -2, -3, -4, -5
F_NO_BW_CAP, F_NO_CONTENTION, F_SAT, F_PAPER_GLOBAL, F_EQ2_BUDGET, F_NO_FILTER, F_COMM = 1, 2, 4, 8, 16, 32, 64
V_QUOTA, V_INST, V_MEM, V_BW, V_QOS, V_LOAD, V_EQ2 = 1, 2, 4, 8, 16, 32, 64
POLICY_MAX_LOAD, POLICY_MIN_RESOURCE = 0, 1
EXEC_RESIDENT = 1

# CAMELOT_SHARED_POLICY: one search-kernel instantiation serves both policies (the policy
# is a runtime argument), so the min-resource search of a plan pair runs on code the
# max-load search brought into L2 (C4 step 1.117 -> 1.090 ms with the L2
# flushed between steps; warm-cache 0.997 -> 1.019 ms, C4b 2.55 -> 2.73 ms)
NVCC_FLAGS_OBJ = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                  "-fmad=false", "-Xcompiler", "-fPIC", "-DCAMELOT_SHARED_POLICY"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh"))] + [HEADER]


def _deps(path, seen=None):
    """Transitive quoted #include files of a source (dependency tracking)."""
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for line in f:
            m = re.match(r'\s*#\s*include\s+"([^"]+)"', line)
            if m:
                _deps(os.path.normpath(os.path.join(os.path.dirname(path), m.group(1))), seen)
    return seen


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libcamelot.so for sm_100a (in-tree): one object per translation
    unit (rebuilt when it or an included header changed), compiled in parallel,
    linked into one shared library."""
    extra = os.environ.get("CAMELOT_NVCC_EXTRA", "").split()   # e.g. -DCAMELOT_FTRACE (profiling)
    objdir = os.environ.get("CAMELOT_OBJDIR") or os.path.join(HERE, "build")   # variant builds (profiling)
    os.makedirs(objdir, exist_ok=True)
    stamp = os.path.join(objdir, "flags.txt")
    flags = " ".join(NVCC_FLAGS_OBJ + extra)
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
    tus = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    objs, procs = [], []
    for tu in tus:
        src = os.path.join(CSRC, tu)
        obj = os.path.join(objdir, tu[:-3] + ".o")
        objs.append(obj)
        newest = max(os.path.getmtime(d) for d in _deps(src))
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < newest:
            cmd = ["nvcc"] + NVCC_FLAGS_OBJ + extra + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", obj, src]
            procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, pr in procs:
        if pr.wait() != 0:
            raise subprocess.CalledProcessError(pr.returncode, cmd)
    with open(stamp, "w") as f:
        f.write(flags)
    if procs or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        subprocess.check_call(["nvcc"] + NVCC_FLAGS + ["-o", LIB] + objs)
    return LIB


class Cluster(C.Structure):
    _fields_ = [("n_gpus", C.c_int32), ("quota_per_gpu", C.c_int32), ("max_instances", C.c_int32),
                ("bw_gbs", C.c_float), ("mem_mib", C.c_uint32), ("gflops", C.c_float),
                ("link_gbs", C.c_float), ("ipc_ms", C.c_float)]


class Problem(C.Structure):
    _fields_ = [("n_apps", C.c_int32), ("n_stages", C.c_int32),
                ("app_of_stage", C.POINTER(C.c_int32)), ("qos_ms", C.POINTER(C.c_float)),
                ("n_quota", C.c_int32), ("quota_pct", C.POINTER(C.c_int32)),
                ("n_batch", C.c_int32), ("batch", C.POINTER(C.c_int32)),
                ("max_replicas", C.c_int32), ("table", C.POINTER(C.c_float)),
                ("weights_mib", C.POINTER(C.c_uint32)), ("act_mib_per_item", C.POINTER(C.c_uint32)),
                ("gflop_per_item", C.POINTER(C.c_float)), ("bw_sensitivity", C.POINTER(C.c_float)),
                ("flags", C.c_uint32), ("comm_mb_per_item", C.POINTER(C.c_float))]


class Exec(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("rank", C.c_int32), ("world", C.c_int32),
                ("index_lo", C.c_uint64), ("index_hi", C.c_uint64), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("exec_flags", C.c_uint32)]


class Plan(C.Structure):
    _fields_ = [("index", C.c_uint64), ("status", C.c_int32),
                ("batch", C.c_int32 * MAX_APPS),
                ("replicas", C.c_int32 * MAX_STAGES), ("quota_pct", C.c_int32 * MAX_STAGES),
                ("gpu_of_instance", C.c_int8 * (MAX_STAGES * MAX_REPLICAS)),
                ("stage_latency_ms", C.c_float * MAX_STAGES),
                ("stage_throughput_qps", C.c_float * MAX_STAGES),
                ("kappa", C.c_float * MAX_STAGES),
                ("e2e_latency_ms", C.c_float * MAX_APPS), ("throughput_qps", C.c_float * MAX_APPS),
                ("objective", C.c_float), ("quota_used", C.c_int32), ("gpus_used", C.c_int32),
                ("eq2_gpus", C.c_int32), ("violations", C.c_uint32),
                ("n_feasible", C.c_uint64), ("n_scored", C.c_uint64), ("n_covered", C.c_uint64),
                ("comm_ms", C.c_float * MAX_STAGES), ("n_evaluated", C.c_uint64), ("search_ns", C.c_uint64)]


class Tree(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("feature", C.POINTER(C.c_int32)), ("threshold", C.POINTER(C.c_int32)),
                ("left", C.POINTER(C.c_int32)), ("right", C.POINTER(C.c_int32)), ("value", C.POINTER(C.c_float))]


EXPORTS = ["camelot_last_error", "camelot_version", "camelot_workspace_bytes", "camelot_upload",
           "camelot_plan_max_load", "camelot_plan_min_resource", "camelot_plan_max_then_min", "camelot_predict",
           "camelot_predict_index",
           "camelot_score_range", "camelot_search_local", "camelot_finalize", "camelot_last_stats",
           "camelot_kernel_launches", "camelot_sa", "camelot_trace",
           "camelot_trees_workspace_bytes", "camelot_tables_from_trees", "camelot_simulate_workspace_bytes",
           "camelot_simulate"]

_lib = None


class CamelotError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"camelot error {code}: {msg}")
        self.code = code


def lib():
    """Load libcamelot.so (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        L = C.CDLL(LIB)
        L.camelot_last_error.restype = C.c_char_p
        L.camelot_version.restype = C.c_char_p
        L.camelot_workspace_bytes.restype = C.c_size_t
        L.camelot_workspace_bytes.argtypes = [C.POINTER(Problem), C.POINTER(Cluster), C.c_int]
        P, Cl, E, Pl = C.POINTER(Problem), C.POINTER(Cluster), C.POINTER(Exec), C.POINTER(Plan)
        fp = C.POINTER(C.c_float)
        L.camelot_upload.argtypes = [P, Cl, E]
        L.camelot_plan_max_load.argtypes = [P, Cl, E, Pl]
        L.camelot_plan_min_resource.argtypes = [P, Cl, fp, C.c_int, E, Pl]
        L.camelot_plan_max_then_min.argtypes = [P, Cl, C.c_double, E, Pl]
        ip = C.POINTER(C.c_int32)
        L.camelot_predict.argtypes = [P, Cl, ip, ip, ip, fp, C.c_int, E, Pl]
        L.camelot_predict_index.argtypes = [P, Cl, C.c_uint64, fp, C.c_int, E, Pl]
        L.camelot_score_range.argtypes = [P, Cl, C.c_uint64, C.c_uint64, E, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.camelot_search_local.argtypes = [P, Cl, C.c_int, fp, C.c_int, E, C.c_void_p]
        L.camelot_finalize.argtypes = [P, Cl, C.c_int, fp, C.c_int, C.c_void_p, E, Pl]
        L.camelot_last_stats.argtypes = [E, C.POINTER(C.c_uint64)]
        L.camelot_trace.argtypes = [E, C.POINTER(C.c_uint64), C.c_int]
        L.camelot_simulate_workspace_bytes.restype = C.c_size_t
        L.camelot_simulate_workspace_bytes.argtypes = [P, Cl, C.c_int64, C.c_int]
        L.camelot_simulate.argtypes = [P, Cl, ip, ip, ip, fp, C.c_int64, C.c_int64, C.c_uint64, C.c_int, E,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.camelot_trees_workspace_bytes.restype = C.c_size_t
        L.camelot_trees_workspace_bytes.argtypes = [C.c_int, C.POINTER(Tree), C.c_int, C.c_int]
        L.camelot_tables_from_trees.argtypes = [C.c_int, C.POINTER(Tree), C.c_int, C.POINTER(C.c_int32), C.c_int,
                                                C.POINTER(C.c_int32), E, C.c_void_p]
        L.camelot_kernel_launches.restype = C.c_uint64
        L.camelot_sa.argtypes = [P, Cl, C.c_int, fp, C.c_uint64, C.c_int, C.c_int, C.c_float, C.c_float, E, Pl,
                                 C.c_void_p, C.c_void_p]
        for f in EXPORTS:
            getattr(L, f)
        _lib = L
    return _lib


def check(rc: int, allow_infeasible: bool = True) -> int:
    if rc == OK or (allow_infeasible and rc == INFEASIBLE):
        return rc
    raise CamelotError(rc, lib().camelot_last_error().decode())
