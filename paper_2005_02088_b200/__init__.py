"""B200-native contention-aware allocation search of Camelot (arXiv 2005.02088).

The compute path is libcamelot.so (hand-written sm_100a CUDA behind the C ABI
of include/camelot.h); this package only marshals arguments (see `api`).
See DESIGN.md.
"""
from ._lib import (F_EQ2_BUDGET, F_NO_BW_CAP, F_NO_CONTENTION, F_NO_FILTER, F_PAPER_GLOBAL, F_SAT,  # noqa: F401
                   POLICY_MAX_LOAD, POLICY_MIN_RESOURCE, CamelotError, build)
