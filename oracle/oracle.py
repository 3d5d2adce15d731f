"""ctypes front-end of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg, never by the product
package.  The oracle is a plain-C restatement of the reference's
``dmmv.solve`` path (see amvm_oracle.c for the function-by-function map to
/root/reference/pkg/src/dmmv) and takes the reference's row-major A.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")

PAIRS = ("random+random", "random+greedy", "worst+random", "worst+greedy")


class Params(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("sigma1", C.c_double), ("sigma2", C.c_double),
        ("sigma3", C.c_double), ("decay", C.c_double), ("accept_tie_tol", C.c_double),
        ("weight_floor", C.c_double), ("time_limit_s", C.c_double),
        ("r", C.c_int32), ("k_eps", C.c_int32), ("max_candidates", C.c_int32),
        ("max_iters", C.c_int32), ("l2_tiebreak", C.c_int32), ("refresh_period", C.c_int32),
        ("one_opt_max_sweeps", C.c_int32), ("ls_max_rounds", C.c_int32),
        ("n_segment", C.c_int32), ("threads", C.c_int32),
    ]


class PCG(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_uint32), ("uinteger", C.c_uint32)]


class Sol(C.Structure):
    _fields_ = [("idx", C.c_void_p), ("residual", C.c_void_p), ("objective", C.c_void_p),
                ("updates", C.c_void_p)]


class Result(C.Structure):
    _fields_ = [("best", Sol), ("initial_objective", C.c_void_p), ("iterations", C.c_void_p),
                ("operator_uses", C.c_void_p), ("trace_current_t", C.c_void_p),
                ("trace_best_t", C.c_void_p), ("trace_pair", C.c_void_p),
                ("trace_accepted", C.c_void_p), ("moves_scored", C.c_void_p),
                ("phase_cycles", C.c_void_p)]


class Problem(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nlev", C.c_int64), ("count", C.c_int64),
                ("A", C.c_void_p), ("B", C.c_void_p), ("levels", C.c_void_p),
                ("At", C.c_void_p)]  # optional column-major copy (speed only), NULL


def build() -> str:
    """Compile liboracle.so (make) if it is missing or stale."""
    src = os.path.join(_HERE, "amvm_oracle.c")
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _lib.orc_pairwise_sum.restype = C.c_double
        _lib.orc_norm.restype = C.c_double
        _lib.orc_random.restype = C.c_double
        _lib.orc_bounded.restype = C.c_int64
        _lib.orc_choice_p.restype = C.c_int64
        _lib.orc_pairwise_sum.argtypes = [C.c_void_p, C.c_int64]
        _lib.orc_norm.argtypes = [C.c_void_p, C.c_int64]
        _lib.orc_bounded.argtypes = [C.c_void_p, C.c_int64]
        _lib.orc_choice_noreplace.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        _lib.orc_choice_p.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    return _lib


def _p(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def make_params(n: int, *, destroy_rate=0.005, alpha=0.3, k_eps=100, max_iters=1000,
                time_limit=None, sigma1=3.0, sigma2=2.0, sigma3=1.0, decay=0.8,
                l2_tiebreak=True, max_candidates=5000, refresh_period=1000,
                one_opt_max_sweeps=10, ls_max_rounds=20, n_segment=50, r=None) -> Params:
    """Reference defaults (controller.py:35-50, core.py:18, localsearch.py:20-21)."""
    if r is None:
        r = max(1, int(round(destroy_rate * n)))
    return Params(alpha, sigma1, sigma2, sigma3, decay, 1e-12, 1e-3,
                  -1.0 if time_limit is None else float(time_limit), r, k_eps,
                  0 if max_candidates is None else max_candidates, max_iters, int(bool(l2_tiebreak)),
                  refresh_period, one_opt_max_sweeps, ls_max_rounds, n_segment, 0)


def pcg_from_seed(seed) -> PCG:
    return pcg_from_state(np.random.default_rng(seed).bit_generator.state)


def pcg_from_state(st: dict) -> PCG:
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return PCG(s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"]))


def pcg_to_state(g: PCG) -> dict:
    return {"bit_generator": "PCG64",
            "state": {"state": (g.state_hi << 64) | g.state_lo, "inc": (g.inc_hi << 64) | g.inc_lo},
            "has_uint32": int(g.has_uint32), "uinteger": int(g.uinteger)}


class _Batch:
    """Owns the numpy buffers behind one oracle call."""

    def __init__(self, A, B, L, colmajor: bool = False):
        self.A = np.ascontiguousarray(A, dtype=np.float64)
        self.B = np.ascontiguousarray(np.atleast_2d(B), dtype=np.float64)
        self.L = np.ascontiguousarray(np.atleast_2d(L), dtype=np.float64)
        m, n = self.A.shape
        # colmajor: also hand over A^T so column scans are contiguous (same
        # values in the same order; for full-size goldens, where the
        # reference's strided A[:, j] would take hours)
        self.At = np.ascontiguousarray(self.A.T) if colmajor else None
        self.prob = Problem(m, n, self.L.shape[1], self.B.shape[0], self.A.ctypes.data,
                            self.B.ctypes.data, self.L.ctypes.data,
                            self.At.ctypes.data if colmajor else None)


def _sol(idx, r, obj, cnt):
    idx = np.ascontiguousarray(np.atleast_2d(idx), dtype=np.int32).copy()
    r = np.ascontiguousarray(np.atleast_2d(r), dtype=np.float64).copy()
    obj = np.ascontiguousarray(np.atleast_1d(obj), dtype=np.float64).copy()
    cnt = np.ascontiguousarray(np.atleast_1d(cnt), dtype=np.int32).copy()
    return (idx, r, obj, cnt), Sol(idx.ctypes.data, r.ctypes.data, obj.ctypes.data, cnt.ctypes.data)


def solve(A, B, levels, idx0, r0, obj0, cnt0, prm: Params, states, threads: int = 1,
          colmajor: bool = False) -> dict:
    """Oracle counterpart of amvm_solve on HOST arrays.

    ``B``/``levels``/``idx0``/``r0`` may be 1-d (one instance) or stacked;
    ``states`` is one PCG (or numpy state dict) per instance.
    """
    bt = _Batch(A, B, levels, colmajor)
    count, m, n = bt.prob.count, bt.prob.m, bt.prob.n
    keep, start = _sol(idx0, r0, obj0, cnt0)
    if not isinstance(states, (list, tuple)):
        states = [states]
    rngs = (PCG * count)(*[s if isinstance(s, PCG) else pcg_from_state(s) for s in states])
    T = max(prm.max_iters, 1)
    out = {
        "best_idx": np.zeros((count, n), np.int32), "best_residual": np.zeros((count, m)),
        "best_objective": np.zeros(count), "best_updates": np.zeros(count, np.int32),
        "initial_objective": np.zeros(count), "iterations": np.zeros(count, np.int32),
        "operator_uses": np.zeros((count, 4), np.int64), "trace_current_t": np.zeros((count, T)),
        "trace_best_t": np.zeros((count, T)), "trace_pair": np.zeros((count, T), np.uint8),
        "trace_accepted": np.zeros((count, T), np.uint8), "moves_scored": np.zeros((count, 2), np.int64),
    }
    d = {k: v.ctypes.data for k, v in out.items()}
    res = Result(Sol(d["best_idx"], d["best_residual"], d["best_objective"], d["best_updates"]),
                 d["initial_objective"], d["iterations"], d["operator_uses"], d["trace_current_t"],
                 d["trace_best_t"], d["trace_pair"], d["trace_accepted"], d["moves_scored"])
    rc = lib().orc_solve(C.byref(bt.prob), C.byref(prm), C.byref(start), rngs, C.byref(res), int(threads))
    if rc != 0:
        raise RuntimeError(f"orc_solve failed: {rc}")
    out["rng_states"] = [pcg_to_state(rngs[k]) for k in range(count)]
    del keep
    return out


def _one(A, b, levels):
    return _Batch(A, b, levels)


def one_opt(A, b, levels, idx, r, obj, cnt, prm: Params):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, cnt)
    lib().orc_one_opt(C.byref(bt.prob), C.byref(prm), C.byref(s))
    return keep[0][0], keep[1][0], float(keep[2][0]), int(keep[3][0])


def local_search(A, b, levels, idx, r, obj, cnt, prm: Params):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, cnt)
    lib().orc_local_search(C.byref(bt.prob), C.byref(prm), C.byref(s))
    return keep[0][0], keep[1][0], float(keep[2][0]), int(keep[3][0])


def find_candidates(A, b, levels, idx, r, obj, prm: Params, cap: int = 1 << 22):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, 0)
    oi = np.zeros(cap, np.int32)
    oj = np.zeros(cap, np.int32)
    od = np.zeros(cap)
    cnt = np.zeros(1, np.int32)
    rc = lib().orc_find_candidates(C.byref(bt.prob), C.byref(prm), C.byref(s), _p(oi), _p(oj),
                                   _p(od), _p(cnt), C.c_int32(cap))
    if rc != 0:
        raise ValueError("candidate generation needs a positive objective")
    k = int(cnt[0])
    return oi[:k].copy(), oj[:k].copy(), od[:k].copy()


def best_swap(A, b, levels, idx, r, obj, prm: Params):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, 0)
    out = np.zeros(4)
    lib().orc_best_swap(C.byref(bt.prob), C.byref(prm), C.byref(s), _p(out))
    if out[0] < 0:
        return None
    return int(out[0]), int(out[1]), float(out[2]), float(out[3])


def impact_scores(A, b, levels, idx, r, obj, prm: Params):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, 0)
    d = np.zeros(bt.prob.n)
    rc = lib().orc_impact_scores(C.byref(bt.prob), C.byref(prm), C.byref(s), _p(d))
    if rc != 0:
        raise ValueError("impact scores are undefined at zero objective")
    return d


def destroy(kind, A, b, levels, idx, r, obj, prm: Params, state):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, 0)
    g = state if isinstance(state, PCG) else pcg_from_state(state)
    out = np.zeros(prm.r, np.int32)
    rc = lib().orc_destroy(C.byref(bt.prob), C.byref(prm), int(kind), C.byref(s), C.byref(g), _p(out))
    if rc != 0:
        raise ValueError("bad removal count")
    return out, pcg_to_state(g)


def repair(kind, A, b, levels, idx, r, obj, cnt, prm: Params, state, removed, saved):
    bt = _one(A, b, levels)
    keep, s = _sol(idx, r, obj, cnt)
    g = state if isinstance(state, PCG) else pcg_from_state(state)
    rem = np.ascontiguousarray(removed, np.int32)
    sv = np.ascontiguousarray(saved, np.int32)
    rc = lib().orc_repair(C.byref(bt.prob), C.byref(prm), int(kind), C.byref(s), C.byref(g), _p(rem),
                          _p(sv), C.c_int32(rem.size))
    if rc != 0:
        raise ValueError("two_nearest needs at least two levels")
    return (keep[0][0], keep[1][0], float(keep[2][0]), int(keep[3][0])), pcg_to_state(g)


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_pairwise_sum(_p(a), a.size))


def norm(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().orc_norm(_p(x), x.size))


def brute_force(A, b, levels, prune: bool = False, chunk: int = 1 << 15):
    """Exhaustive enumeration (dmmv.oracle.brute_force, oracle.py:38-111),
    numpy restatement: codes in lexicographic order (oracle.py:58-60), the
    first code attaining the minimum wins.  prune=False evaluates t as the
    reference's `assignments @ A.T - b` (oracle.py:62-64); prune=True in the
    pruned DFS's order, s = -b + levels[d_0] A[:,0] + ... unfused
    (oracle.py:95-111) — without pruning, which does not change the optimum.
    Returns (best_idx, best_t, enumerated = |V|^n)."""
    A = np.asarray(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    levels = np.asarray(levels, dtype=np.float64)
    m, n = A.shape
    nlev = levels.size
    total = nlev ** n
    place = nlev ** np.arange(n - 1, -1, -1, dtype=np.int64)
    best_t, best_idx = np.inf, None
    for lo in range(0, total, chunk):
        codes = np.arange(lo, min(lo + chunk, total), dtype=np.int64)
        digits = (codes[:, None] // place) % nlev
        X = levels[digits]
        if not prune:
            S = X @ A.T - b
        else:
            S = np.broadcast_to(-b, (codes.size, m)).copy()
            for j in range(n):
                S = S + X[:, j:j + 1] * A[:, j]
        t_all = np.max(np.abs(S), axis=1)
        k = int(np.argmin(t_all))
        if t_all[k] < best_t:
            best_t, best_idx = float(t_all[k]), digits[k].astype(np.intp)
    return best_idx, best_t, total


def score_moves(A, s, levels, idx, mode: str = "adjacent"):
    """numpy restatement of the one_opt candidate objective
    (/root/reference/pkg/src/dmmv/localsearch.py:76-78) for every column and
    candidate level: t[j, v] = max|s + (lv[l] - lv[idx_j]) * A[:, j]|, the
    same numpy expression per candidate.  Returns (t, best (j, level) | None,
    best_t) with best = the smallest (t, j, level) over level-changing moves."""
    A = np.asarray(A, dtype=np.float64)
    lv = np.asarray(levels, dtype=np.float64)
    m, n = A.shape
    nlev = lv.size
    nv = 2 if mode == "adjacent" else nlev
    t = np.full((n, nv), np.inf)
    best, best_t = None, np.inf
    for j in range(n):
        k = int(idx[j])
        col = A[:, j]
        cands = (k - 1, k + 1) if mode == "adjacent" else range(nlev)
        for v, c in enumerate(cands):
            if not 0 <= c < nlev:
                continue
            t[j, v] = float(np.max(np.abs(s + (lv[c] - lv[k]) * col)))
            if c != k and (best is None or t[j, v] < best_t):
                best, best_t = (j, c), t[j, v]
    return t, best, best_t
