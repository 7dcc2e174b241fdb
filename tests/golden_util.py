"""Shared helpers for parity tests: golden-buffer generation and oracle loading.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load oracle/.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
ORACLE_DIR = os.path.join(ROOT, "oracle", "_ref")


def cases(name: str):
    with open(os.path.join(GOLDEN, f"ref_{name}.json")) as f:
        return json.load(f)["cases"]


def buffer_values(kind: str, seed: int, gid: int, length: int) -> np.ndarray:
    """numpy mirror of buffer_value() in oracle/ref_driver.cpp (bit-identical doubles)."""
    e = np.arange(length, dtype=np.uint64)
    if kind == "cli":
        return 1.0 + 0.001 * gid + 1e-6 * e.astype(np.float64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
             + np.uint64(gid % (1 << 64)) * np.uint64(0xBF58476D1CE4E5B9)
             + e * np.uint64(0x94D049BB133111EB))
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 0.1 + 0.9 * u


def f64_digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def layout_arrays(mpl):
    counts = [len(l) for l in mpl]
    ids = [i for l in mpl for i in l]
    return counts, ids


_reduce_oracle = None


def reduce_oracle():
    global _reduce_oracle
    if _reduce_oracle is None:
        path = os.path.join(ORACLE_DIR, "libreduce_oracle.so")
        lib = C.CDLL(path)
        for name in ("oracle_execute_f32", "oracle_execute_f64"):
            fn = getattr(lib, name)
            fn.restype = C.c_int
            fn.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                           C.c_size_t, C.c_void_p]
        _reduce_oracle = lib
    return _reduce_oracle


def oracle_execute(algo: int, mpl, bufs: list[np.ndarray]) -> np.ndarray:
    counts, ids = layout_arrays(mpl)
    dtype = bufs[0].dtype
    length = bufs[0].shape[0]
    out = np.empty(length, dtype=dtype)
    arr = [np.ascontiguousarray(b) for b in bufs]
    ptrs = (C.c_void_p * len(arr))(*[a.ctypes.data for a in arr])
    fn = reduce_oracle().oracle_execute_f64 if dtype == np.float64 else reduce_oracle().oracle_execute_f32
    rc = fn(algo, len(mpl), (C.c_int * len(counts))(*counts), (C.c_int * len(ids))(*ids), ptrs, length,
            out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"oracle rejected layout (rc={rc})")
    return out
