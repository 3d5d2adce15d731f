"""The AMVM solve API (mirror of dmmv.controller + dmmv.localsearch/operators).

``solve(inst, cfg)`` keeps the reference's signature and semantics
(/root/reference/pkg/src/dmmv/controller.py:211-286): the host computes the
starting point with numpy exactly as the reference does (controller.py:
134-165), then ONE call into libamvm.so runs every ALNS iteration on the GPU
(device-resident state, no per-iteration host round trip) and the trace and
best solution come back once at the end.

The component functions (one_opt, local_search, find_candidates, best_swap,
impact_scores, random/worst-remove destroy, random/greedy repair) run the same
device code on a single instance; they exist so the reference's own test
strategy can be replayed against the GPU path.
"""

from __future__ import annotations

import os
import time
import warnings
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import _native as N
from .core import Instance, Solution

# destroy/repair pairs, in roulette-wheel slot order (controller.py:23-28)
PAIRS: tuple[tuple[str, str], ...] = (
    ("random", "random"),
    ("random", "greedy"),
    ("worst", "random"),
    ("worst", "greedy"),
)
N_SEGMENT = 50
WEIGHT_FLOOR = 1e-3
ACCEPT_TIE_TOL = 1e-12
ONE_OPT_MAX_SWEEPS = 10
LOCAL_SEARCH_MAX_ROUNDS = 20
REFRESH_PERIOD = 1000


@dataclass
class FilterConfig:
    """Candidate-generation knobs (localsearch.py:34-56)."""

    k_eps: int = 100
    max_candidates: int | None = 5000
    workers: int = 1
    l2_tiebreak: bool = False

    def __post_init__(self) -> None:
        if self.k_eps < 1:
            raise ValueError("k_eps must be at least 1")
        if self.max_candidates is not None and self.max_candidates < 1:
            raise ValueError("max_candidates must be positive or None")
        if self.workers < 1:
            raise ValueError("workers must be at least 1")


@dataclass
class SwapCandidate:
    """Ordered pair ``(i, j)`` with ``x_i > x_j`` (localsearch.py:24-31)."""

    i: int
    j: int
    delta: float
    predicted_t: float | None = None


@dataclass
class SolverConfig:
    """Tuning knobs for :func:`solve` (controller.py:35-68)."""

    destroy_rate: float = 0.005
    alpha: float = 0.3
    k_eps: int = 100
    max_iters: int = 1000
    time_limit: float | None = None
    seed: int = 0
    sigma1: float = 3.0
    sigma2: float = 2.0
    sigma3: float = 1.0
    decay: float = 0.8
    l2_tiebreak: bool = True
    max_candidates: int | None = 5000
    workers: int = 1

    def __post_init__(self) -> None:
        if not 0 < self.destroy_rate <= 1:
            raise ValueError("destroy_rate must lie in (0, 1]")
        if self.alpha < 0:
            raise ValueError("alpha must be non-negative")
        if self.max_iters < 0:
            raise ValueError("max_iters must be non-negative")
        if not self.sigma1 >= self.sigma2 >= self.sigma3 >= 0:
            raise ValueError("rewards must satisfy sigma1 >= sigma2 >= sigma3 >= 0")
        if not 0 < self.decay <= 1:
            raise ValueError("decay must lie in (0, 1]")

    def filter_config(self) -> FilterConfig:
        return FilterConfig(k_eps=self.k_eps, max_candidates=self.max_candidates, workers=self.workers)


class TraceEntry(NamedTuple):
    iteration: int
    current_t: float
    best_t: float
    op_pair: str
    accepted: bool


@dataclass
class SolveReport:
    """Everything a run produces (controller.py:194-203).  ``device`` adds the
    GPU-side counters (candidate moves scored, reference-equivalent and raw)."""

    best: Solution
    trace: list[TraceEntry]
    wall_time: float
    iterations: int
    initial_objective: float
    operator_uses: dict[str, int] = field(default_factory=dict)
    device: dict = field(default_factory=dict)


def removal_count(destroy_rate: float, n: int) -> int:
    """``max(1, round(rate*n))`` with Python's rounding (controller.py:206-208)."""
    return max(1, int(round(destroy_rate * n)))


def _nearest_level_indices(levels: np.ndarray, vec: np.ndarray) -> np.ndarray:
    vec = np.asarray(vec, dtype=float)
    dist = np.abs(vec[:, None] - levels[None, :])
    return np.argmin(dist, axis=1).astype(np.intp)


def initial_solution(inst: Instance, *, device: bool = False) -> Solution:
    """Rounded warm start or regularized least squares (controller.py:134-165).

    Host numpy by default: the starting residual is the one numpy's BLAS
    produces, bit for bit.  ``device=True`` solves the
    least-squares system on the GPU (``amvm_ls_start``: Gram matrix,
    Cholesky, substitution and rounding in CUDA); its target agrees with
    LAPACK's to rounding, so the rounded start matches unless a component
    sits within rounding of a midpoint between two levels."""
    if device and inst.continuous_init is None:
        return _initial_solution_device(inst)
    if inst.continuous_init is not None:
        target = inst.continuous_init
    else:
        gram = inst.A.T @ inst.A + 1e-8 * np.eye(inst.n)
        try:
            target = np.linalg.solve(gram, inst.A.T @ inst.b)
        except np.linalg.LinAlgError:
            warnings.warn("least-squares start failed; starting from zeros", stacklevel=2)
            target = np.zeros(inst.n)
        if not np.all(np.isfinite(target)):
            warnings.warn("least-squares start not finite; starting from zeros", stacklevel=2)
            target = np.zeros(inst.n)
    idx = _nearest_level_indices(inst.values.levels, target)
    return Solution.from_indices(inst, idx)


def _initial_solution_device(inst: Instance, return_target: bool = False):
    torch = N.torch_cuda()
    lib = N.load_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    At, b, lv = inst.device_arrays(dev)
    prob = N.Problem(inst.m, inst.n, len(inst.values), 1, At.data_ptr(), b.data_ptr(), lv.data_ptr())
    nbytes = lib.amvm_ls_start_workspace_bytes(inst.m, inst.n)
    ws = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
    idx = torch.empty(inst.n, dtype=torch.int32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    tgt = torch.empty(inst.n, dtype=torch.float64, device=dev) if return_target else None
    N.check(lib.amvm_ls_start(N.C.byref(prob), N.ptr(idx), N.ptr(tgt) if return_target else None, N.ptr(flag),
                              N.ptr(ws),
                              N.C.c_size_t(ws.numel()), N.stream_handle()), "amvm_ls_start")
    f = int(flag.item())
    if f == 1:
        warnings.warn("least-squares start failed; starting from zeros", stacklevel=3)
    elif f == 2:
        warnings.warn("least-squares start not finite; starting from zeros", stacklevel=3)
    sol = Solution.from_indices(inst, idx.cpu().numpy().astype(np.intp))
    return (sol, tgt.cpu().numpy(), f) if return_target else sol


# ----------------------------------------------------------------- plumbing
def make_params(cfg: SolverConfig | None, n: int, *, fcfg: FilterConfig | None = None,
                max_iters: int | None = None, time_budget: float | None = None,
                r: int | None = None) -> N.Params:
    cfg = cfg or SolverConfig()
    fcfg = fcfg or cfg.filter_config()
    return N.Params(
        float(cfg.alpha), float(cfg.sigma1), float(cfg.sigma2), float(cfg.sigma3), float(cfg.decay),
        ACCEPT_TIE_TOL, WEIGHT_FLOOR, -1.0 if time_budget is None else float(time_budget),
        removal_count(cfg.destroy_rate, n) if r is None else int(r), int(fcfg.k_eps),
        0 if fcfg.max_candidates is None else int(fcfg.max_candidates),
        int(cfg.max_iters if max_iters is None else max_iters), int(bool(cfg.l2_tiebreak)),
        REFRESH_PERIOD, ONE_OPT_MAX_SWEEPS, LOCAL_SEARCH_MAX_ROUNDS, N_SEGMENT, 0)


class _Dev:
    """Device mirror of one Instance + one Solution for a single call."""

    def __init__(self, inst: Instance, sol: Solution | None, device=None):
        torch = N.torch_cuda()
        self.torch = torch
        self.lib = N.load_library()
        self.device = (torch.device("cuda", torch.cuda.current_device()) if device is None
                       else torch.device(device))
        At, b, lv = inst.device_arrays(self.device)
        self.inst = inst
        self.prob = N.Problem(inst.m, inst.n, len(inst.values), 1, At.data_ptr(), b.data_ptr(), lv.data_ptr())
        self._keep = [At, b, lv]
        if sol is not None:
            self.idx = torch.from_numpy(np.asarray(sol.idx, dtype=np.int32)).to(self.device)
            self.r = torch.from_numpy(np.array(sol.residual, dtype=np.float64)).to(self.device)
            self.obj = torch.tensor([sol.objective], dtype=torch.float64, device=self.device)
            self.cnt = torch.tensor([sol.updates_since_refresh], dtype=torch.int32, device=self.device)
            self.sol = N.SolutionPtrs(self.idx.data_ptr(), self.r.data_ptr(), self.obj.data_ptr(),
                                      self.cnt.data_ptr())

    def ws(self, prm: N.Params):
        nbytes = self.lib.amvm_workspace_bytes(N.C.byref(self.prob), N.C.byref(prm))
        if nbytes == 0:
            raise ValueError("problem shape or parameters rejected by libamvm")
        buf = N.workspace(self.device, nbytes)
        return N.ptr(buf), N.C.c_size_t(buf.numel())

    def finish(self, rc: int, what: str, ws) -> None:
        N.check(rc, what)
        st = self.lib.amvm_status(ws, N.stream_handle())
        N.check(st, what)

    def write_back(self, sol: Solution) -> Solution:
        sol.idx = self.idx.cpu().numpy().astype(np.intp)
        sol.residual = self.r.cpu().numpy().copy()
        sol.objective = float(self.obj.item())
        sol.updates_since_refresh = int(self.cnt.item())
        return sol


def _rng_struct(rng: np.random.Generator, device=None):
    torch = N.torch_cuda()
    arr = N.pcg_array([rng.bit_generator.state])
    return torch.from_numpy(arr.view(np.uint8)).to(device or "cuda"), arr


def _rng_sync_back(rng: np.random.Generator, dev_buf) -> None:
    arr = dev_buf.cpu().numpy().view(N.PCG_DTYPE)
    rng.bit_generator.state = N.pcg_to_state(arr[0])


# --------------------------------------------------------------------- solve
def solve(inst: Instance, cfg: SolverConfig | None = None, *, device_warm_start: bool = False) -> SolveReport:
    """Run the adaptive destroy/repair/local-search loop on the GPU.

    Same semantics as dmmv.solve (controller.py:211-286): deterministic for a
    fixed seed, stops at ``max_iters``, ``time_limit`` or a zero objective.
    ``device_warm_start`` computes the least-squares start on the GPU
    (``initial_solution(device=True)``)."""
    cfg = cfg or SolverConfig()
    started = time.perf_counter()
    N.check_blas_order()
    rng = np.random.default_rng(cfg.seed)
    current = initial_solution(inst, device=device_warm_start)
    initial_objective = current.objective
    max_iters = cfg.max_iters
    budget = None
    if cfg.time_limit is not None:
        budget = cfg.time_limit - (time.perf_counter() - started)
        if budget <= 0:
            max_iters = 0
    will_iterate = max_iters > 0 and current.objective != 0.0
    if will_iterate and len(inst.values) < 2:
        raise ValueError("two_nearest needs at least two levels")
    if not will_iterate:
        return SolveReport(best=current.copy(), trace=[], wall_time=time.perf_counter() - started,
                           iterations=0, initial_objective=initial_objective,
                           operator_uses={f"{d}+{r_}": 0 for d, r_ in PAIRS})
    out = _solve_device(inst, cfg, current, rng, max_iters, budget)
    return _report(out, initial_objective, started)


def solve_from(inst: Instance, start: Solution, cfg: SolverConfig | None = None) -> SolveReport:
    """``solve`` from a given starting Solution instead of initial_solution
    (warm restart; also how the parity tests feed the reference's own start)."""
    cfg = cfg or SolverConfig()
    started = time.perf_counter()
    N.check_blas_order()
    rng = np.random.default_rng(cfg.seed)
    if cfg.max_iters == 0 or start.objective == 0.0:
        return SolveReport(best=start.copy(), trace=[], wall_time=0.0, iterations=0,
                           initial_objective=start.objective,
                           operator_uses={f"{d}+{r_}": 0 for d, r_ in PAIRS})
    if len(inst.values) < 2:
        raise ValueError("two_nearest needs at least two levels")
    out = _solve_device(inst, cfg, start, rng, cfg.max_iters, cfg.time_limit)
    return _report(out, start.objective, started)


def _report(out: dict, initial_objective: float, started: float) -> SolveReport:
    trace = [
        TraceEntry(k + 1, float(out["trace_current_t"][k]), float(out["trace_best_t"][k]),
                   "+".join(PAIRS[int(out["trace_pair"][k])]), bool(out["trace_accepted"][k]))
        for k in range(out["iterations"])
    ]
    best = Solution(out["best_idx"].astype(np.intp), out["best_residual"], out["best_objective"],
                    out["best_updates"])
    return SolveReport(
        best=best, trace=trace, wall_time=time.perf_counter() - started,
        iterations=out["iterations"], initial_objective=initial_objective,
        operator_uses={f"{d}+{r_}": int(out["operator_uses"][k]) for k, (d, r_) in enumerate(PAIRS)},
        device={"moves_scored_ref": int(out["moves_scored"][0]),
                "moves_scored_raw": int(out["moves_scored"][1])},
    )


def _sparse_view(D, inst):
    """A as CSC + CSR device arrays when it is sparse (density <= 1/8) and
    large (m*n >= 2^20), else None: solve() then runs the sparse engine
    (amvm_solve_sparse), whose results equal the dense engine's bit for bit
    (tests/test_sparse_gpu.py, tests/test_c3full_gpu.py).  AMVM_SPARSE_ROUTE=0
    keeps every solve on the dense engine."""
    if os.environ.get("AMVM_SPARSE_ROUTE", "1") == "0" or inst.m * inst.n < (1 << 20):
        return None
    key = f"{D.device}:sparse"
    if key in inst._device:  # built once per instance and device
        return inst._device[key]
    inst._device[key] = sp = _build_sparse_view(D, inst)
    return sp


def _build_sparse_view(D, inst):
    torch = D.torch
    At = D._keep[0]  # n x m, column-major A
    nnz = int(torch.count_nonzero(At).item())
    if nnz * 8 > inst.m * inst.n:
        return None
    m, n = inst.m, inst.n
    A = At.t()  # m x n view
    rc = torch.nonzero(A)  # row-major order: rows ascending, columns ascending within a row
    rows, cols = rc[:, 0], rc[:, 1]
    rval = A[rows, cols].contiguous()
    rptr = torch.zeros(m + 1, dtype=torch.int64, device=D.device)
    rptr[1:] = torch.cumsum(torch.bincount(rows, minlength=m), 0)
    order = torch.sort(cols * m + rows, stable=True).indices
    cptr = torch.zeros(n + 1, dtype=torch.int64, device=D.device)
    counts = torch.bincount(cols, minlength=n)
    cptr[1:] = torch.cumsum(counts, 0)
    keep = [rptr, cols.to(torch.int32).contiguous(), rval, cptr, rows[order].to(torch.int32).contiguous(),
            rval[order].contiguous()]
    max_row = int((rptr[1:] - rptr[:-1]).max().item())
    prob = N.SparseProblem(m, n, len(inst.values), 1, nnz, int(counts.max().item()),
                           keep[3].data_ptr(), keep[4].data_ptr(), keep[5].data_ptr(),
                           keep[0].data_ptr(), keep[1].data_ptr(), keep[2].data_ptr(),
                           D._keep[1].data_ptr(), D._keep[2].data_ptr(), max_row)
    return prob, keep


def _solve_device(inst, cfg, current, rng, max_iters, budget) -> dict:
    D = _Dev(inst, current)
    torch = D.torch
    prm = make_params(cfg, inst.n, max_iters=max_iters, time_budget=budget)
    T = max(int(max_iters), 1)
    dev = D.device
    rng_buf, _ = _rng_struct(rng, D.device)
    o = {
        "best_idx": torch.empty(inst.n, dtype=torch.int32, device=dev),
        "best_residual": torch.empty(inst.m, dtype=torch.float64, device=dev),
        "best_objective": torch.empty(1, dtype=torch.float64, device=dev),
        "best_updates": torch.empty(1, dtype=torch.int32, device=dev),
        "initial_objective": torch.empty(1, dtype=torch.float64, device=dev),
        "iterations": torch.empty(1, dtype=torch.int32, device=dev),
        "operator_uses": torch.empty(4, dtype=torch.int64, device=dev),
        "trace_current_t": torch.empty(T, dtype=torch.float64, device=dev),
        "trace_best_t": torch.empty(T, dtype=torch.float64, device=dev),
        "trace_pair": torch.empty(T, dtype=torch.uint8, device=dev),
        "trace_accepted": torch.empty(T, dtype=torch.uint8, device=dev),
        "moves_scored": torch.empty(2, dtype=torch.int64, device=dev),
    }
    res = N.ResultPtrs(
        N.SolutionPtrs(o["best_idx"].data_ptr(), o["best_residual"].data_ptr(),
                       o["best_objective"].data_ptr(), o["best_updates"].data_ptr()),
        o["initial_objective"].data_ptr(), o["iterations"].data_ptr(), o["operator_uses"].data_ptr(),
        o["trace_current_t"].data_ptr(), o["trace_best_t"].data_ptr(), o["trace_pair"].data_ptr(),
        o["trace_accepted"].data_ptr(), o["moves_scored"].data_ptr())
    sp = _sparse_view(D, inst)
    if sp is not None:  # sparse A: the sparse engine (same results)
        nbytes = D.lib.amvm_sparse_workspace_bytes(N.C.byref(sp[0]), N.C.byref(prm))
        if nbytes == 0:
            raise ValueError("problem shape or parameters rejected by libamvm")
        buf = N.workspace(D.device, nbytes)
        ws, wsb = N.ptr(buf), N.C.c_size_t(buf.numel())
        rc = D.lib.amvm_solve_sparse(N.C.byref(sp[0]), N.C.byref(prm), N.C.byref(D.sol), N.ptr(rng_buf),
                                     N.C.byref(res), ws, wsb, N.stream_handle())
        D.finish(rc, "amvm_solve_sparse", ws)
    else:
        ws, wsb = D.ws(prm)
        rc = D.lib.amvm_solve(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), N.ptr(rng_buf),
                              N.C.byref(res), ws, wsb, N.stream_handle())
        D.finish(rc, "amvm_solve", ws)
    host = {k: v.cpu().numpy() for k, v in o.items()}
    it = int(host["iterations"][0])
    return {
        "best_idx": host["best_idx"], "best_residual": host["best_residual"],
        "best_objective": float(host["best_objective"][0]), "best_updates": int(host["best_updates"][0]),
        "iterations": it, "operator_uses": host["operator_uses"],
        "trace_current_t": host["trace_current_t"][:it], "trace_best_t": host["trace_best_t"][:it],
        "trace_pair": host["trace_pair"][:it], "trace_accepted": host["trace_accepted"][:it],
        "moves_scored": host["moves_scored"],
    }


# --------------------------------------------- incremental residual algebra
def _device_update(inst: Instance, sol: Solution, kind: str, a: int, b: int) -> Solution:
    """apply_shift / apply_swap (core.py:208-245) on the GPU, in place."""
    D = _Dev(inst, sol)
    prm = make_params(None, inst.n)
    ws, wsb = D.ws(prm)
    if kind == "shift":
        rc = D.lib.amvm_apply_shift(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), a, b, ws, wsb,
                                    N.stream_handle())
    else:
        rc = D.lib.amvm_apply_swap(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), a, b, ws, wsb,
                                   N.stream_handle())
    D.finish(rc, f"amvm_apply_{kind}", ws)
    return D.write_back(sol)


# ------------------------------------------- operator bank and acceptance
OUTCOME_NEW_BEST = "new_best"
OUTCOME_IMPROVED = "improved"
OUTCOME_ACCEPTED = "accepted"
OUTCOME_REJECTED = "rejected"
_OUTCOMES = (OUTCOME_NEW_BEST, OUTCOME_IMPROVED, OUTCOME_ACCEPTED, OUTCOME_REJECTED)


class OperatorBank:
    """Adaptive weights, segment scores and usage counts per operator pair
    (controller.py:71-85).  The arrays live on the host like the reference's;
    ``select_operators`` / ``update_weights`` run the same arithmetic as the
    solve kernel's device bank (``amvm_select_operators`` /
    ``amvm_update_weights``)."""

    def __init__(self, decay: float = 0.8) -> None:
        if not 0 < decay <= 1:
            raise ValueError("decay must lie in (0, 1]")
        self.decay = float(decay)
        self.weights = np.ones(len(PAIRS))
        self.scores = np.zeros(len(PAIRS))
        self.segment_uses = np.zeros(len(PAIRS), dtype=int)
        self.lifetime_uses = np.zeros(len(PAIRS), dtype=int)
        self.iteration = 0

    def probabilities(self) -> np.ndarray:
        return self.weights / self.weights.sum()

    def _to_device(self, device):
        torch = N.torch_cuda()
        st = N.Bank((N.C.c_double * 4)(*self.weights), (N.C.c_double * 4)(*self.scores),
                    (N.C.c_int64 * 4)(*self.segment_uses), (N.C.c_int64 * 4)(*self.lifetime_uses),
                    int(self.iteration), float(self.decay))
        raw = np.frombuffer(bytes(st), dtype=np.uint8).copy()
        return torch.from_numpy(raw).to(device)

    def _from_device(self, buf) -> None:
        st = N.Bank.from_buffer_copy(buf.cpu().numpy().tobytes())
        self.weights = np.array(st.weights[:], dtype=float)
        self.scores = np.array(st.scores[:], dtype=float)
        self.segment_uses = np.array(st.segment_uses[:], dtype=int)
        self.lifetime_uses = np.array(st.lifetime_uses[:], dtype=int)
        self.iteration = int(st.iteration)


def select_operators(bank: OperatorBank, rng: np.random.Generator) -> int:
    """Roulette-wheel pick of a destroy/repair pair (controller.py:88-90); one
    ``random()`` of ``rng``'s PCG64 stream, drawn on the GPU (the generator's
    state is advanced exactly as numpy's ``rng.choice(4, p=...)``)."""
    torch = N.torch_cuda()
    lib = N.load_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    bb = bank._to_device(dev)
    rb, _ = _rng_struct(rng, dev)
    out = torch.empty(1, dtype=torch.int32, device=dev)
    N.check(lib.amvm_select_operators(N.ptr(bb), N.ptr(rb), N.ptr(out), N.stream_handle()),
            "amvm_select_operators")
    _rng_sync_back(rng, rb)
    return int(out.item())


def update_weights(bank: OperatorBank, pair_id: int, outcome: str,
                   cfg: SolverConfig | None = None) -> OperatorBank:
    """Score the pair for this iteration's outcome; decay at segment ends
    (controller.py:99-131), on the GPU.  Mutates and returns ``bank``."""
    cfg = cfg or SolverConfig()
    if outcome not in _OUTCOMES:
        raise KeyError(outcome)
    torch = N.torch_cuda()
    lib = N.load_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    bb = bank._to_device(dev)
    prm = make_params(cfg, 1)
    N.check(lib.amvm_update_weights(N.ptr(bb), N.C.byref(prm), int(pair_id), _OUTCOMES.index(outcome),
                                    N.stream_handle()), "amvm_update_weights")
    bank._from_device(bb)
    return bank


def accept(current: Solution, candidate: Solution, cfg: SolverConfig) -> bool:
    """Strict improvement, or with ``cfg.l2_tiebreak`` a tie within
    ACCEPT_TIE_TOL and a strictly smaller l2 residual (controller.py:168-183);
    the norms are the host BLAS ddot order, on the GPU (``amvm_accept``)."""
    torch = N.torch_cuda()
    lib = N.load_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    cur = np.ascontiguousarray(current.residual, dtype=np.float64)
    cand = np.ascontiguousarray(candidate.residual, dtype=np.float64)
    if cur.shape != cand.shape or cur.ndim != 1 or cur.size == 0:
        raise ValueError("current and candidate residuals must be non-empty vectors of equal length")
    t = torch.from_numpy(np.concatenate([cur, cand, [current.objective, candidate.objective]])).to(dev)
    m = cur.size
    out = torch.empty(1, dtype=torch.int32, device=dev)
    base = t.data_ptr()
    N.check(lib.amvm_accept(m, N.C.c_void_p(base), N.C.c_void_p(base + 8 * 2 * m), N.C.c_void_p(base + 8 * m),
                            N.C.c_void_p(base + 8 * (2 * m + 1)), int(bool(cfg.l2_tiebreak)), ACCEPT_TIE_TOL,
                            N.ptr(out), N.stream_handle()), "amvm_accept")
    return bool(out.item())


# ------------------------------------------------------ component functions
def one_opt(inst: Instance, sol: Solution, max_sweeps: int = ONE_OPT_MAX_SWEEPS) -> Solution:
    """Adjacent-level first-improvement sweeps on the GPU (localsearch.py:59-88)."""
    D = _Dev(inst, sol)
    prm = make_params(None, inst.n)
    prm.one_opt_max_sweeps = int(max_sweeps)
    ws, wsb = D.ws(prm)
    D.finish(D.lib.amvm_one_opt(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), ws, wsb,
                                N.stream_handle()), "amvm_one_opt", ws)
    return D.write_back(sol)


def local_search(inst: Instance, sol: Solution, cfg: FilterConfig | None = None,
                 max_rounds: int = LOCAL_SEARCH_MAX_ROUNDS) -> Solution:
    """one_opt + best filtered swaps on the GPU (localsearch.py:249-269)."""
    D = _Dev(inst, sol)
    prm = make_params(None, inst.n, fcfg=cfg or FilterConfig())
    prm.ls_max_rounds = int(max_rounds)
    ws, wsb = D.ws(prm)
    D.finish(D.lib.amvm_local_search(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), ws, wsb,
                                     N.stream_handle()), "amvm_local_search", ws)
    return D.write_back(sol)


def find_candidates(inst: Instance, sol: Solution, cfg: FilterConfig) -> list[SwapCandidate]:
    """Filtered swap candidates in (-delta, i, j) order (localsearch.py:128-169)."""
    if sol.objective <= 0:
        raise ValueError("candidate generation needs a positive objective")
    D = _Dev(inst, sol)
    torch = D.torch
    prm = make_params(None, inst.n, fcfg=cfg)
    cap = inst.n * (inst.n - 1) // 2 + 1
    if cfg.max_candidates is not None:
        cap = min(cap, cfg.max_candidates)
    oi = torch.empty(cap, dtype=torch.int32, device=D.device)
    oj = torch.empty(cap, dtype=torch.int32, device=D.device)
    od = torch.empty(cap, dtype=torch.float64, device=D.device)
    cnt = torch.zeros(1, dtype=torch.int32, device=D.device)
    ws, wsb = D.ws(prm)
    D.finish(D.lib.amvm_find_candidates(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), N.ptr(oi),
                                        N.ptr(oj), N.ptr(od), N.ptr(cnt), cap, ws, wsb, N.stream_handle()),
             "amvm_find_candidates", ws)
    k = int(cnt.item())
    i, j, d = oi[:k].cpu().numpy(), oj[:k].cpu().numpy(), od[:k].cpu().numpy()
    return [SwapCandidate(int(i[q]), int(j[q]), float(d[q])) for q in range(k)]


def best_swap(inst: Instance, sol: Solution, cfg: FilterConfig) -> SwapCandidate | None:
    """Best strictly improving filtered swap (localsearch.py:211-246).  With
    ``cfg.l2_tiebreak`` the candidates are chunked over ``cfg.workers`` and
    chunk winners merge by (t, l2, i, j) exactly as the reference's threads
    do (``amvm_best_swap_l2``); without it the merge key is (t, i, j) and the
    result does not depend on ``workers``."""
    if sol.objective <= 0:
        return None
    D = _Dev(inst, sol)
    torch = D.torch
    prm = make_params(None, inst.n, fcfg=cfg)
    out = torch.zeros(4, dtype=torch.float64, device=D.device)
    ws, wsb = D.ws(prm)
    if cfg.l2_tiebreak:
        rc = D.lib.amvm_best_swap_l2(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), int(cfg.workers),
                                     N.ptr(out), ws, wsb, N.stream_handle())
        D.finish(rc, "amvm_best_swap_l2", ws)
    else:
        D.finish(D.lib.amvm_best_swap(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), N.ptr(out), ws, wsb,
                                      N.stream_handle()), "amvm_best_swap", ws)
    v = out.cpu().numpy()
    if v[0] < 0:
        return None
    return SwapCandidate(int(v[0]), int(v[1]), float(v[2]), predicted_t=float(v[3]))


@dataclass
class ImpactScores:
    d: np.ndarray
    alpha: float


@dataclass
class DestroySet:
    removed: np.ndarray
    saved_idx: np.ndarray


def impact_scores(inst: Instance, sol: Solution, alpha: float) -> ImpactScores:
    """Per-variable blame scores (operators.py:54-74), computed on the GPU."""
    if alpha < 0:
        raise ValueError("alpha must be non-negative")
    if sol.objective <= 0:
        raise ValueError("impact scores are undefined at zero objective")
    D = _Dev(inst, sol)
    torch = D.torch
    cfg = SolverConfig(alpha=alpha)
    prm = make_params(cfg, inst.n)
    d = torch.empty(inst.n, dtype=torch.float64, device=D.device)
    ws, wsb = D.ws(prm)
    D.finish(D.lib.amvm_impact_scores(N.C.byref(D.prob), N.C.byref(prm), N.C.byref(D.sol), N.ptr(d), ws, wsb,
                                      N.stream_handle()), "amvm_impact_scores", ws)
    return ImpactScores(d=d.cpu().numpy(), alpha=float(alpha))


def _destroy(kind: int, inst: Instance, sol: Solution, r: int, alpha: float,
             rng: np.random.Generator) -> DestroySet:
    n = sol.idx.size
    if not 1 <= r <= n:
        raise ValueError(f"removal count r={r} must be in [1, n={n}]")
    D = _Dev(inst, sol)
    torch = D.torch
    prm = make_params(SolverConfig(alpha=alpha), inst.n, r=r)
    rb, _ = _rng_struct(rng, D.device)
    out = torch.empty(r, dtype=torch.int32, device=D.device)
    ws, wsb = D.ws(prm)
    D.finish(D.lib.amvm_destroy(N.C.byref(D.prob), N.C.byref(prm), kind, N.C.byref(D.sol), N.ptr(rb),
                                N.ptr(out), ws, wsb, N.stream_handle()), "amvm_destroy", ws)
    _rng_sync_back(rng, rb)
    removed = out.cpu().numpy().astype(np.intp)
    return DestroySet(removed=removed, saved_idx=sol.idx[removed].copy())


def random_destroy(sol: Solution, r: int, rng: np.random.Generator, inst: Instance | None = None) -> DestroySet:
    """Uniform pick of ``r`` variables (operators.py:34-39), drawn on the GPU
    from the same PCG64 stream (the generator's state is advanced)."""
    n = sol.idx.size
    if not 1 <= r <= n:
        raise ValueError(f"removal count r={r} must be in [1, n={n}]")
    if inst is None:
        # the draw needs no matrix; a 1-row stand-in instance carries n
        stand = Instance(np.zeros((1, n)), np.zeros(1), [0.0, 1.0])
        ds = _destroy(0, stand, Solution(np.zeros(n, dtype=np.intp), np.zeros(1), 0.0), r, 0.3, rng)
        return DestroySet(removed=ds.removed, saved_idx=sol.idx[ds.removed].copy())
    return _destroy(0, inst, sol, r, 0.3, rng)


def worst_remove_destroy(inst: Instance, sol: Solution, r: int, alpha: float,
                         rng: np.random.Generator) -> DestroySet:
    """Impact-proportional picks (operators.py:77-105), on the GPU."""
    return _destroy(1, inst, sol, r, alpha, rng)


def _repair(kind: int, inst: Instance, sol: Solution, destroyed: DestroySet, rng) -> Solution:
    if len(inst.values) < 2:
        raise ValueError("two_nearest needs at least two levels")
    D = _Dev(inst, sol)
    torch = D.torch
    prm = make_params(None, inst.n)
    rem = torch.from_numpy(np.asarray(destroyed.removed, dtype=np.int32)).to(D.device)
    sav = torch.from_numpy(np.asarray(destroyed.saved_idx, dtype=np.int32)).to(D.device)
    if rng is not None:
        rb, _ = _rng_struct(rng, D.device)
    else:
        rb = torch.zeros(N.PCG_DTYPE.itemsize, dtype=torch.uint8, device=D.device)
    ws, wsb = D.ws(prm)
    D.finish(D.lib.amvm_repair(N.C.byref(D.prob), N.C.byref(prm), kind, N.C.byref(D.sol), N.ptr(rb),
                               N.ptr(rem), N.ptr(sav), int(rem.numel()), ws, wsb, N.stream_handle()),
             "amvm_repair", ws)
    if rng is not None:
        _rng_sync_back(rng, rb)
    return D.write_back(sol)


def random_repair(inst: Instance, sol: Solution, destroyed: DestroySet, rng: np.random.Generator) -> Solution:
    """Coin-flip between the two nearest levels (operators.py:108-117), on the GPU."""
    return _repair(0, inst, sol, destroyed, rng)


def greedy_repair(inst: Instance, sol: Solution, destroyed: DestroySet) -> Solution:
    """Better of the two nearest levels, in place (operators.py:120-138), on the GPU."""
    return _repair(1, inst, sol, destroyed, None)
