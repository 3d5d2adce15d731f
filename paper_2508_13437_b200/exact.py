"""Exact solver for small instances: the reference's ``dmmv.oracle`` module
(/root/reference/pkg/src/dmmv/oracle.py:38-111), enumerated on the GPU.

``brute_force(inst, budget, prune)`` keeps the reference's signature, budget
check (``BudgetExceededError`` raised before any enumeration, same message)
and result type.  Every one of the |V|^n assignments is evaluated by
``amvm_brute_force`` (include/amvm.h, csrc/amvm_exact.cuh); the answer is the
lexicographically smallest index vector attaining the minimum, as the
reference's ordered scan returns.  ``prune=True`` selects the arithmetic order
of the reference's pruned DFS (oracle.py:95-111), so ``best_t`` is bitwise the
pruned result; the device does not prune, so ``enumerated`` is always the
full count |V|^n (the reference's pruned count is a property of its
sequential DFS and is documented as a deviation in DESIGN.md).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import Instance

DEFAULT_BUDGET = 10_000_000  # oracle.py:12


class BudgetExceededError(ValueError):
    """Raised before any enumeration when the search space exceeds the budget
    (oracle.py:19-28)."""

    def __init__(self, required: int, budget: int) -> None:
        self.required = required
        self.budget = budget
        super().__init__(
            f"enumeration needs {required} assignments but the budget is {budget}; "
            f"raise the budget to at least {required} to proceed"
        )


@dataclass
class OracleResult:
    best_idx: np.ndarray
    best_t: float
    enumerated: int


def brute_force(inst: Instance, budget: int = DEFAULT_BUDGET, prune: bool = False) -> OracleResult:
    """Exact optimum by enumerating every assignment (oracle.py:38-71)."""
    nlev = len(inst.values)
    total = nlev ** inst.n
    if total > budget:
        raise BudgetExceededError(total, budget)
    torch = N.torch_cuda()
    lib = N.load_library()
    dev = torch.device("cuda", torch.cuda.current_device())
    At, b, lv = inst.device_arrays(dev)
    prob = N.Problem(inst.m, inst.n, nlev, 1, At.data_ptr(), b.data_ptr(), lv.data_ptr())
    nbytes = lib.amvm_brute_force_workspace_bytes(N.C.byref(prob))
    if nbytes == 0:
        raise RuntimeError("amvm_brute_force: problem shape outside this build's limits (n <= 64)")
    ws = N.workspace(dev, nbytes)
    idx = torch.empty(inst.n, dtype=torch.int32, device=dev)
    t = torch.empty(1, dtype=torch.float64, device=dev)
    rc = lib.amvm_brute_force(N.C.byref(prob), int(bool(prune)), N.ptr(idx), N.ptr(t), None, N.ptr(ws),
                              N.C.c_size_t(ws.numel()), N.stream_handle())
    N.check(rc, "amvm_brute_force")
    return OracleResult(best_idx=idx.cpu().numpy().astype(np.intp), best_t=float(t.item()), enumerated=total)


MAX_SWAP_CHECK_N = 64  # oracle.py:16


def _device_problem(inst: Instance):
    torch = N.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    At, b, lv = inst.device_arrays(dev)
    return torch, dev, N.Problem(inst.m, inst.n, len(inst.values), 1, At.data_ptr(), b.data_ptr(), lv.data_ptr())


def is_improving(inst: Instance, sol, cand, use_screen: bool = True, check_screen: bool = False) -> bool:
    """Exact strict-improvement test for one swap candidate
    (localsearch.py:91-125) on the GPU (``amvm_is_improving``).  The row
    screen only skips rows that pass the test, so ``use_screen`` does not
    change the verdict and ``check_screen`` (which re-tests skipped rows)
    always holds; both are accepted for API parity."""
    if cand.delta <= 0:
        raise ValueError("swap candidates need delta = x_i - x_j > 0")
    return bool(is_improving_batch(inst, sol, [cand])[0])


def is_improving_batch(inst: Instance, sol, cands) -> np.ndarray:
    """Verdicts of many swap candidates in one launch (warp per candidate)."""
    torch, dev, prob = _device_problem(inst)
    lib = N.load_library()
    ci = torch.tensor([c.i for c in cands], dtype=torch.int32, device=dev)
    cj = torch.tensor([c.j for c in cands], dtype=torch.int32, device=dev)
    cd = torch.tensor([c.delta for c in cands], dtype=torch.float64, device=dev)
    if bool((cd <= 0).any()):
        raise ValueError("swap candidates need delta = x_i - x_j > 0")
    s = torch.from_numpy(np.asarray(sol.residual, dtype=np.float64)).to(dev)
    v = torch.empty(len(cands), dtype=torch.int32, device=dev)
    N.check(lib.amvm_is_improving(N.C.byref(prob), N.ptr(s), float(sol.objective), len(cands), N.ptr(ci), N.ptr(cj),
                                  N.ptr(cd), N.ptr(v), N.stream_handle()), "amvm_is_improving")
    return v.cpu().numpy().astype(bool)


@dataclass
class SwapCheckReport:
    """Disagreements between the swap test and recomputed objectives
    (oracle.py:114-127)."""

    discrepancies: list
    boundary: list
    pairs_checked: int


def exhaustive_swap_check(inst: Instance, sol, guard: float = 1e-12) -> SwapCheckReport:
    """Validate the strict-improvement swap test against full recomputes
    (oracle.py:130-161): every ordered pair with x_i > x_j, the post-swap
    objective recomputed from scratch in numpy's order and the test's
    verdict, all pairs in one launch (``amvm_swap_check``); records in the
    reference's (i, j) order."""
    if inst.n > MAX_SWAP_CHECK_N:
        raise ValueError(f"exhaustive swap check restricted to n <= {MAX_SWAP_CHECK_N}")
    torch, dev, prob = _device_problem(inst)
    lib = N.load_library()
    n = inst.n
    idx = torch.from_numpy(np.asarray(sol.idx, dtype=np.int32)).to(dev)
    s = torch.from_numpy(np.asarray(sol.residual, dtype=np.float64)).to(dev)
    out_t = torch.zeros(n * n, dtype=torch.float64, device=dev)
    out_v = torch.zeros(n * n, dtype=torch.int32, device=dev)
    N.check(lib.amvm_swap_check(N.C.byref(prob), N.ptr(idx), N.ptr(s), float(sol.objective), N.ptr(out_t),
                                N.ptr(out_v), N.stream_handle()), "amvm_swap_check")
    T = out_t.cpu().numpy().reshape(n, n)
    V = out_v.cpu().numpy().reshape(n, n).astype(bool)
    x = sol.values(inst)
    t = sol.objective
    discrepancies, boundary, pairs = [], [], 0
    for i in range(n):
        for j in range(n):
            if x[i] <= x[j] or i == j:
                continue
            pairs += 1
            t_after, verdict = float(T[i, j]), bool(V[i, j])
            if verdict != (t_after < t):
                record = ((i, j), t_after, verdict)
                (boundary if abs(t_after - t) <= guard else discrepancies).append(record)
    return SwapCheckReport(discrepancies=discrepancies, boundary=boundary, pairs_checked=pairs)
