"""Batched candidate-move scoring on the GPU (``amvm_score_moves``).

The north-star scorer (BASELINE.json north_star (c)):
the one_opt candidate objective of ``localsearch.py:76-78``

    t(j, l) = max_k | s_k + (lv[l] - lv[idx_j]) * A[k, j] |

for every column j and candidate level l in one launch, each column of A
streamed once and amortised over all its candidates.  Bitwise numpy's value
for every entry (level difference, then unfused DMUL and DADD; the max of
absolute values is order-independent).  ``one_opt`` itself is a sequential
first-improvement sweep (it applies moves as it goes) and runs inside the
engine; this call scores a whole neighbourhood of one fixed solution -- the
primitive a best-improvement or batched caller builds on.

Modes: ``"adjacent"`` = the reference's candidate set {idx-1, idx+1}
(columns of the result: lower, upper; +inf where the level does not exist);
``"all"`` = every level (column l; l == idx_j holds the current objective).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import Instance

MODES = {"all": 0, "adjacent": 1}


@dataclass
class MoveScores:
    """Scores of one instance: ``t[j, v]``; ``best`` = (j, level) of the
    smallest (t, j, level) among moves that change a level (None if there
    are none) and ``best_t`` its objective; ``improving`` = best_t < the
    solution's objective (the reference's strict test, localsearch.py:79)."""

    t: np.ndarray
    best: tuple | None
    best_t: float
    improving: bool


def score_moves_device(prob: "N.Problem", idx, residual, mode: str = "adjacent", ws=None):
    """Device-tensor form for batches sharing A (``prob.count`` instances):
    idx int32 [count, n], residual float64 [count, m] -> (t [count, n, nv],
    best flat index int64 [count], best_t float64 [count]), all on device,
    asynchronous on the current stream.  ``ws``: optional uint8 device
    workspace of at least ``amvm_score_workspace_bytes``, zeroed before its
    first use (allocated zeroed if absent or short).  Inputs are validated
    (dtype, shape, contiguity, device, level range, finite residual; this
    costs a device sync -- keep ``ws`` and call the C-ABI directly to time
    the kernel alone)."""
    torch = N.torch_cuda()
    lib = N.load_library()
    if mode not in MODES:
        raise ValueError(f"mode must be one of {sorted(MODES)}, got {mode!r}")
    count, m, n = int(prob.count), int(prob.m), int(prob.n)
    dev = idx.device
    # the kernel reads raw pointers: check dtype, shape, layout and device first
    if idx.dtype != torch.int32 or tuple(idx.shape) != (count, n) or not idx.is_contiguous():
        raise ValueError(f"idx must be a contiguous int32 tensor of shape ({count}, {n}), got "
                         f"{idx.dtype} {tuple(idx.shape)}")
    if (residual.dtype != torch.float64 or tuple(residual.shape) != (count, m)
            or not residual.is_contiguous()):
        raise ValueError(f"residual must be a contiguous float64 tensor of shape ({count}, {m}), got "
                         f"{residual.dtype} {tuple(residual.shape)}")
    if dev.type != "cuda" or residual.device != dev:
        raise ValueError("idx and residual must be CUDA tensors on the same device")
    if count and (int(idx.min()) < 0 or int(idx.max()) >= int(prob.nlev)):
        raise ValueError(f"idx entries must lie in [0, {int(prob.nlev)})")
    if not bool(torch.isfinite(residual).all()):
        raise ValueError("residual must be finite")
    nv = 2 if mode == "adjacent" else int(prob.nlev)
    t = torch.empty((count, n, nv), dtype=torch.float64, device=dev)
    best = torch.empty(count, dtype=torch.int64, device=dev)
    best_t = torch.empty(count, dtype=torch.float64, device=dev)
    wsb = int(lib.amvm_score_workspace_bytes(N.C.byref(prob)))
    if ws is None or ws.numel() < wsb:
        ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)  # ticket counters start at zero
    elif ws.dtype != torch.uint8 or ws.device != dev:
        raise ValueError("ws must be a uint8 tensor on the same device (zeroed before its first use)")
    N.check(lib.amvm_score_moves(N.C.byref(prob), N.ptr(idx), N.ptr(residual), MODES[mode], N.ptr(t),
                                 N.ptr(best), N.ptr(best_t), N.ptr(ws), ws.numel(), N.stream_handle()),
            "amvm_score_moves")
    return t, best, best_t


def score_moves(inst: Instance, sol, mode: str = "adjacent") -> MoveScores:
    """Score every single-variable move of ``sol`` (see the module doc)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {sorted(MODES)}, got {mode!r}")
    idx_h = np.asarray(sol.idx)
    if idx_h.shape != (inst.n,):
        raise ValueError(f"solution has {idx_h.size} indices, instance has n={inst.n}")
    nlev = len(inst.values)
    if idx_h.size and (idx_h.min() < 0 or idx_h.max() >= nlev):
        raise ValueError(f"idx entries must lie in [0, {nlev})")
    res_h = np.asarray(sol.residual, dtype=np.float64)
    if res_h.shape != (inst.m,):
        raise ValueError(f"residual has {res_h.size} entries, instance has m={inst.m}")
    torch = N.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    At, b, lv = inst.device_arrays(dev)
    prob = N.Problem(inst.m, inst.n, len(inst.values), 1, At.data_ptr(), b.data_ptr(), lv.data_ptr())
    idx = torch.from_numpy(idx_h.astype(np.int32)).to(dev)
    s = torch.from_numpy(res_h).to(dev)
    t, best, best_t = score_moves_device(prob, idx[None], s[None], mode)
    t = t[0].cpu().numpy()
    flat = int(best.cpu()[0])
    bt = float(best_t.cpu()[0])
    if flat < 0:
        return MoveScores(t, None, float("inf"), False)
    j, v = divmod(flat, t.shape[1])
    level = int(idx_h[j]) + (-1 if v == 0 else 1) if mode == "adjacent" else v
    return MoveScores(t, (j, level), bt, bt < float(sol.objective))
