"""Shared-X batch front end: one quantized linear layer = many AMVM instances.

Post-training quantization of a layer row by row is the reference's
``build_quant`` problem (builders.py:355-372) with one
calibration matrix X shared by every output row r:
``min_{x in V_r^n} ||X x - X w_r||_inf``, V_r = linspace(min w_r, max w_r,
2^bits), warm start w_r, seed r.  The reference builds one Instance per row
(copying X each time) and loops; here the whole layer (or this rank's shard of
its rows) is ONE device pipeline:

  amvm_ptq_prepare      levels, nearest-level start, B = X W^T (BLAS order)
  amvm_compute_residual start residual and objective (BLAS order)
  amvm_solve            the ALNS loop, one CTA per row, persistent grid

Every stage reproduces numpy bit for bit, so each row's result equals
``dmmv.solve(Instance(X, X @ w_r, ValueSet(grid_r), continuous_init=w_r),
SolverConfig(seed=r, ...))`` on a single-threaded-BLAS host.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .controller import SolverConfig, make_params


@dataclass
class LayerReport:
    rows: np.ndarray               # global row ids solved here
    codes: np.ndarray              # rows x n int8 level indices of the best solutions
    levels: np.ndarray             # rows x 2^bits quantization grids
    objective: np.ndarray          # best l_inf per row
    initial_objective: np.ndarray  # rounded-warm-start l_inf per row
    iterations: np.ndarray
    moves_scored: np.ndarray       # rows x 2: reference-equivalent, raw
    seconds: dict = field(default_factory=dict)


class LayerBatch:
    """Device-resident state of one layer shard, reusable across solves."""

    def __init__(self, X, W, bits: int = 4, rows=None, device=None):
        torch = N.torch_cuda()
        N.check_blas_order()
        self.torch = torch
        self.lib = N.load_library()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        X_t = X if isinstance(X, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64))
        W_t = W if isinstance(W, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(W, dtype=np.float64))
        if X_t.dtype != torch.float64 or W_t.dtype != torch.float64:
            raise ValueError("X and W must be float64")
        if X_t.dim() != 2 or W_t.dim() != 2 or X_t.shape[1] != W_t.shape[1]:
            raise ValueError("X must be calib x d and W rows x d")
        self.m, self.n = int(X_t.shape[0]), int(X_t.shape[1])
        self.rows = np.arange(W_t.shape[0]) if rows is None else np.asarray(rows)
        self.count = int(self.rows.size)
        self.nlev = 2 ** int(bits)
        if not 1 <= bits <= 10:
            raise ValueError("bits must lie in [1, 10]")
        dev = self.device
        # column-major A: the transpose happens on the device
        self.At = X_t.to(dev, non_blocking=True).t().contiguous()
        Wsel = W_t if rows is None else W_t[torch.as_tensor(self.rows)]
        self.W = Wsel.to(dev, non_blocking=True).contiguous()
        # Instance validation (core.py:93-94), done on the device copies
        if not bool(torch.isfinite(self.At).all() & torch.isfinite(self.W).all()):
            raise ValueError("A and b must be finite")
        f64, i32 = torch.float64, torch.int32
        self.B = torch.empty((self.count, self.m), dtype=f64, device=dev)
        self.L = torch.empty((self.count, self.nlev), dtype=f64, device=dev)
        self.idx0 = torch.empty((self.count, self.n), dtype=i32, device=dev)
        self.r0 = torch.empty((self.count, self.m), dtype=f64, device=dev)
        self.obj0 = torch.empty(self.count, dtype=f64, device=dev)
        self.cnt0 = torch.empty(self.count, dtype=i32, device=dev)
        self.prepared = False

    def prepare(self) -> None:
        """levels, start assignment, targets and start residuals (device)."""
        st = N.stream_handle()
        N.check(self.lib.amvm_ptq_prepare(self.m, self.n, self.count, self.nlev, N.ptr(self.At), N.ptr(self.W),
                                          N.ptr(self.B), N.ptr(self.L), N.ptr(self.idx0), st),
                "amvm_ptq_prepare")
        prob = self.problem()
        sol = N.SolutionPtrs(self.idx0.data_ptr(), self.r0.data_ptr(), self.obj0.data_ptr(),
                             self.cnt0.data_ptr())
        N.check(self.lib.amvm_compute_residual(N.C.byref(prob), N.C.byref(sol), st), "amvm_compute_residual")
        self.prepared = True

    def problem(self) -> N.Problem:
        return N.Problem(self.m, self.n, self.nlev, self.count, self.At.data_ptr(), self.B.data_ptr(),
                         self.L.data_ptr())

    def solve(self, cfg: SolverConfig | None = None, seeds=None, trace: bool = False) -> dict:
        """Run amvm_solve over the shard; returns device tensors (no sync)."""
        torch = self.torch
        cfg = cfg or SolverConfig()
        if not self.prepared:
            self.prepare()
        dev = self.device
        seeds = self.rows if seeds is None else np.asarray(seeds)
        # pinned + non_blocking: the upload is stream-ordered and the host does
        # not wait for earlier work (back-to-back solves stay queued)
        self._rng_host = torch.from_numpy(N.seed_states(seeds).view(np.uint8)).pin_memory()
        self.rng = self._rng_host.to(dev, non_blocking=True)
        T = max(int(cfg.max_iters), 1)
        c, m, n = self.count, self.m, self.n
        o = {
            "best_idx": torch.empty((c, n), dtype=torch.int32, device=dev),
            "best_residual": torch.empty((c, m), dtype=torch.float64, device=dev),
            "best_objective": torch.empty(c, dtype=torch.float64, device=dev),
            "best_updates": torch.empty(c, dtype=torch.int32, device=dev),
            "initial_objective": torch.empty(c, dtype=torch.float64, device=dev),
            "iterations": torch.empty(c, dtype=torch.int32, device=dev),
            "operator_uses": torch.empty((c, 4), dtype=torch.int64, device=dev),
            "moves_scored": torch.empty((c, 2), dtype=torch.int64, device=dev),
            "phase_cycles": torch.empty((c, 16), dtype=torch.int64, device=dev),
        }
        tr = [None] * 4
        if trace:
            o["trace_current_t"] = torch.empty((c, T), dtype=torch.float64, device=dev)
            o["trace_best_t"] = torch.empty((c, T), dtype=torch.float64, device=dev)
            o["trace_pair"] = torch.empty((c, T), dtype=torch.uint8, device=dev)
            o["trace_accepted"] = torch.empty((c, T), dtype=torch.uint8, device=dev)
            tr = [o["trace_current_t"].data_ptr(), o["trace_best_t"].data_ptr(), o["trace_pair"].data_ptr(),
                  o["trace_accepted"].data_ptr()]
        res = N.ResultPtrs(
            N.SolutionPtrs(o["best_idx"].data_ptr(), o["best_residual"].data_ptr(),
                           o["best_objective"].data_ptr(), o["best_updates"].data_ptr()),
            o["initial_objective"].data_ptr(), o["iterations"].data_ptr(), o["operator_uses"].data_ptr(),
            *tr, o["moves_scored"].data_ptr(), o["phase_cycles"].data_ptr())
        prm = make_params(cfg, n, time_budget=cfg.time_limit)
        prob = self.problem()
        nbytes = self.lib.amvm_workspace_bytes(N.C.byref(prob), N.C.byref(prm))
        if nbytes == 0:
            raise ValueError("problem shape or parameters rejected by libamvm")
        ws = N.workspace(dev, nbytes)
        start = N.SolutionPtrs(self.idx0.data_ptr(), self.r0.data_ptr(), self.obj0.data_ptr(),
                               self.cnt0.data_ptr())
        rc = self.lib.amvm_solve(N.C.byref(prob), N.C.byref(prm), N.C.byref(start), N.ptr(self.rng),
                                 N.C.byref(res), N.ptr(ws), N.C.c_size_t(ws.numel()), N.stream_handle())
        N.check(rc, "amvm_solve")
        self._ws = ws
        return o

    def check_status(self) -> None:
        N.check(self.lib.amvm_status(N.ptr(self._ws), N.stream_handle()), "amvm_solve")


def layer_report(rows, host: dict, levels: np.ndarray, seconds: dict | None = None) -> LayerReport:
    """Assemble a LayerReport from per-row HOST arrays in the device result
    layout (best_idx, best_objective, initial_objective, iterations,
    moves_scored, optionally the trace_* arrays): codes narrowed to int8 for
    <= 128 levels (int16 otherwise)."""
    nlev = levels.shape[1]
    code_t = np.int8 if nlev <= 128 else np.int16
    rep = LayerReport(
        rows=np.asarray(rows), codes=np.asarray(host["best_idx"]).astype(code_t),
        levels=np.asarray(levels), objective=np.asarray(host["best_objective"]),
        initial_objective=np.asarray(host["initial_objective"]), iterations=np.asarray(host["iterations"]),
        moves_scored=np.asarray(host["moves_scored"]), seconds=dict(seconds or {}),
    )
    if "trace_current_t" in host:
        rep.seconds["trace"] = {k: host[k] for k in ("trace_current_t", "trace_best_t", "trace_pair",
                                                     "trace_accepted")}
    return rep


def solve_layer(X, W, bits: int = 4, cfg: SolverConfig | None = None, rows=None, seeds=None,
                device=None, trace: bool = False) -> LayerReport:
    """Quantize the rows of W (all, or ``rows``) against calibration X on the GPU."""
    torch = N.torch_cuda()
    t0 = time.perf_counter()
    lb = LayerBatch(X, W, bits=bits, rows=rows, device=device)
    lb.prepare()
    o = lb.solve(cfg, seeds=seeds, trace=trace)
    lb.check_status()
    t1 = time.perf_counter()
    # only what the report carries crosses PCIe; codes narrowed on the device
    keep = ("best_objective", "initial_objective", "iterations", "moves_scored")
    if trace:
        keep += ("trace_current_t", "trace_best_t", "trace_pair", "trace_accepted")
    host = {k: o[k].cpu().numpy() for k in keep}
    code_t = torch.int8 if lb.nlev <= 128 else torch.int16
    host["best_idx"] = o["best_idx"].to(code_t).cpu().numpy()
    return layer_report(lb.rows, host, lb.L.cpu().numpy(), {"device_pipeline": t1 - t0})


def shard_rows(total: int, rank: int, world: int) -> np.ndarray:
    """Contiguous row shard of ``rank``: rows [r*T/W, (r+1)*T/W)."""
    from .shard import shard_rows as _s

    return _s(total, rank, world)


def gather_layer(rep: LayerReport, total_rows: int, group=None) -> LayerReport:
    """All-gather every rank's shard results (the only inter-GPU traffic, one
    collective per field at the end; NCCL on GPUs, gloo on CPU)."""
    from .shard import gather_rows

    rows, f = gather_rows(rep.rows, {"codes": rep.codes, "levels": rep.levels, "objective": rep.objective,
                                     "initial_objective": rep.initial_objective, "iterations": rep.iterations,
                                     "moves_scored": rep.moves_scored}, total_rows, group)
    return LayerReport(rows=rows, codes=f["codes"], levels=f["levels"], objective=f["objective"],
                       initial_objective=f["initial_objective"], iterations=f["iterations"],
                       moves_scored=f["moves_scored"], seconds=dict(rep.seconds))
