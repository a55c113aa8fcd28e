"""GPU feature extraction: drop-in for `extract_features` (`src/features.py:420-425`)
plus the batched twin `extract_features_batch` the population scorer uses.

Host side encodes States (`encode.py`); the sm_100a kernel (`csrc/features.cu`)
computes every row.  No CPU fallback.
"""

from __future__ import annotations

import numpy as np

from . import runtime as rt
from .encode import encode_batch

N_FEATURES = 164


def extract_features_batch(programs, gpu_features: bool = False) -> list:
    """One (n_statements x 164) float64 matrix per program, in order.
    gpu_features: fill the 8 gpu_* slots (columns 51-58) with the statement's
    kernel binding instead of the reference's zeros (opt-in)."""
    lib = rt.load()
    words, stmt_off, prog_off = encode_batch(programs, gpu_features)
    n_stmt = len(stmt_off) - 1
    rows = np.empty((n_stmt, N_FEATURES), dtype=np.float64)
    if n_stmt:
        rt.check(lib.lt_features_batch(rt.ptr(words, rt.c_i32p), rt.ptr(stmt_off, rt.c_i64p), n_stmt,
                                       rt.ptr(rows, rt.c_f64p)), "lt_features_batch")
    return [rows[prog_off[i]:prog_off[i + 1]] for i in range(len(programs))]


def extract_features(program, gpu_features: bool = False) -> np.ndarray:
    return extract_features_batch([program], gpu_features)[0]
