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
