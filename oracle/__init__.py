"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU reference for what the retrieval hot
path computes.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import it.  It shares no
code with paper_2505_12065_b200/ and never calls it.

  oracle.c      exact flat top-k in fp64 (plain C, OpenMP over queries)
  exact.py      an independent second oracle: exact rational arithmetic
                (fractions.Fraction) + sort, for tiny inputs (pin P9)
  ivf.py        IVF build + search, step by step

Functions below are thin ctypes wrappers over oracle.c; see that file for
the definitions and citations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc -O2 -fopenmp (no -ffast-math:
    the sequential fp64 sum must stay sequential)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", "-o", _SO, src, "-lm"]
        subprocess.check_call(cmd)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        L.oracle_bf16_round.argtypes = [P, P, i64]
        L.oracle_dot.argtypes = [P, P, i32]
        L.oracle_dot.restype = ctypes.c_double
        L.oracle_topk_init.argtypes = [i64, i32, P, P]
        L.oracle_topk_update.argtypes = [P, i64, i32, i64, P, i64, i32, P, P]
        L.oracle_flat_topk.argtypes = [P, i64, i32, P, i64, i32, P, P]
        L.oracle_pair_scores.argtypes = [P, i32, P, P, P, i64, P]
        L.oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits (uint16), round-to-nearest-even (reading R3)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.uint16)
    lib().oracle_bf16_round(_p(x), _p(out), x.size)
    return out


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


class TopK:
    """Running exact top-kk lists for nq queries, fed chunk by chunk."""

    def __init__(self, Q_bits: np.ndarray, kk: int):
        self.Q = np.ascontiguousarray(Q_bits, dtype=np.uint16)
        self.nq, self.d = self.Q.shape
        self.kk = int(kk)
        self.ids = np.empty((self.nq, self.kk), dtype=np.int64)
        self.scores = np.empty((self.nq, self.kk), dtype=np.float64)
        lib().oracle_topk_init(self.nq, self.kk, _p(self.ids), _p(self.scores))

    def update(self, X_bits: np.ndarray, id0: int = 0):
        X = np.ascontiguousarray(X_bits, dtype=np.uint16)
        assert X.shape[1] == self.d
        lib().oracle_topk_update(_p(X), X.shape[0], self.d, int(id0), _p(self.Q),
                                 self.nq, self.kk, _p(self.ids), _p(self.scores))
        return self


def flat_topk(X_bits: np.ndarray, Q_bits: np.ndarray, k: int):
    """Exact top-k (ids int64 [nq,k], scores f64 [nq,k]); pads (-1, -inf)."""
    t = TopK(Q_bits, k)
    t.update(X_bits, 0)
    return t.ids, t.scores


def pair_scores(X_bits: np.ndarray, Q_bits: np.ndarray, qidx, ridx) -> np.ndarray:
    X = np.ascontiguousarray(X_bits, dtype=np.uint16)
    Q = np.ascontiguousarray(Q_bits, dtype=np.uint16)
    qi = np.ascontiguousarray(qidx, dtype=np.int64)
    ri = np.ascontiguousarray(ridx, dtype=np.int64)
    out = np.empty(qi.shape[0], dtype=np.float64)
    lib().oracle_pair_scores(_p(X), X.shape[1], _p(Q), _p(qi), _p(ri), qi.shape[0], _p(out))
    return out


def num_threads() -> int:
    return int(lib().oracle_num_threads())
