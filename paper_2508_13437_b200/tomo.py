"""Discrete-tomography front end (C3 family).

Host-side instance construction for the tomography configs, restating the
reference builder's arithmetic so the projection matrix is bit-identical to
``dmmv.parallel_beam_matrix`` (builders.py:186-239) on the same numpy:

* the image is the square [-side/2, side/2]^2 of unit pixels; ray k of angle
  theta starts at offset o_k * (cos, sin) and runs along (-sin, cos);
* a ray's pixel weights are the lengths between consecutive sorted, distinct
  crossing parameters (the box entry/exit and every grid line strictly in
  between), each attributed to the pixel containing its midpoint;
* rows are ordered (angle, detector), columns row-major pixels.

Everything here is numpy on the host: it builds A once per instance family
(A is then shared by every slice of a batch).  The ALNS path itself runs on
the GPU through ``solve`` / ``solve_from``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

_EPS = 1e-12  # builders.py:195 — degenerate-direction and zero-length cut-off


def phantom(kind: str, side: int) -> np.ndarray:
    """Integer label image (builders.py:158-183 semantics)."""
    if side < 1:
        raise ValueError("side must be at least 1")
    if kind == "squares":
        img = np.zeros((side, side), dtype=np.int64)
        outer, inner = max(1, side // 8), max(2, (3 * side) // 8)
        for margin, label in ((outer, 1), (inner, 2)):
            if side > 2 * margin:
                img[margin:side - margin, margin:side - margin] = label
        return img
    if kind == "disk":
        c = (side - 1) / 2.0
        r, q = np.mgrid[0:side, 0:side]
        return ((r - c) ** 2 + (q - c) ** 2 <= (0.35 * side) ** 2).astype(np.int64)
    if kind == "checker":
        blk = max(1, side // 8)
        r, q = np.mgrid[0:side, 0:side]
        return ((r // blk + q // blk) % 2).astype(np.int64)
    raise ValueError(f"unknown phantom kind {kind!r}; pick disk, squares, or checker")


def _segments(side: int, origin, direction):
    """(pixel indices, lengths) of the ray origin + tau * direction."""
    half = side / 2.0
    enter, leave = -np.inf, np.inf
    steep = []  # axes the ray is not parallel to
    for ax in (0, 1):
        d, p = direction[ax], origin[ax]
        if abs(d) > _EPS:
            a, b = (-half - p) / d, (half - p) / d
            enter, leave = max(enter, min(a, b)), min(leave, max(a, b))
            steep.append(ax)
        elif not -half <= p <= half:
            return None
    if leave <= enter:
        return None
    parts = [np.array([enter, leave])]
    grid = -half + np.arange(side + 1)
    for ax in steep:
        cross = (grid - origin[ax]) / direction[ax]
        parts.append(cross[(cross > enter) & (cross < leave)])
    tau = np.unique(np.concatenate(parts))
    seg = np.diff(tau)
    mid = tau[:-1] + seg / 2
    col = np.clip(np.floor(origin[0] + mid * direction[0] + half).astype(np.intp), 0, side - 1)
    row = np.clip(np.floor(half - (origin[1] + mid * direction[1])).astype(np.intp), 0, side - 1)
    use = seg > _EPS
    return row[use] * side + col[use], seg[use]


def projection_csr(side: int, n_angles: int):
    """Parallel-beam projector as CSR (indptr, indices, values); rows =
    (angle, detector), one detector per image column at unit spacing."""
    thetas = np.arange(n_angles) * np.pi / n_angles
    offs = np.arange(side) - (side - 1) / 2.0
    indptr, idx, val = [0], [], []
    for th in thetas:
        c, s = np.cos(th), np.sin(th)
        for o in offs:
            hit = _segments(side, (o * c, o * s), (-s, c))
            if hit is not None and hit[0].size:
                # a convex cell is crossed once; keep builders.py's add.at
                # semantics anyway (duplicates summed in order)
                pix, w = hit
                if np.unique(pix).size != pix.size:
                    acc = {}
                    for p_, w_ in zip(pix.tolist(), w.tolist()):
                        acc[p_] = acc.get(p_, 0.0) + w_
                    pix = np.array(sorted(acc), dtype=np.intp)
                    w = np.array([acc[p_] for p_ in pix.tolist()])
                order = np.argsort(pix, kind="stable")
                idx.append(pix[order]); val.append(w[order])
                indptr.append(indptr[-1] + pix.size)
            else:
                indptr.append(indptr[-1])
    idx = np.concatenate(idx) if idx else np.zeros(0, np.intp)
    val = np.concatenate(val) if val else np.zeros(0)
    return np.asarray(indptr, dtype=np.int64), idx.astype(np.int64), val


def projection_matrix(side: int, n_angles: int) -> np.ndarray:
    """Dense projector (n_angles*side x side^2), bit-identical to the
    reference's ``parallel_beam_matrix(side, arange(n)*pi/n)``."""
    indptr, idx, val = projection_csr(side, n_angles)
    A = np.zeros((n_angles * side, side * side))
    for r in range(A.shape[0]):
        A[r, idx[indptr[r]:indptr[r + 1]]] = val[indptr[r]:indptr[r + 1]]
    return A


class SliceBatch:
    """Several tomography slices sharing one projector A as ONE device batch
    (slices shard like PTQ rows).  Slice k is the instance
    (A, B[k], levels) started from idx0[k] with seed seeds[k]; each slice's
    result equals ``solve_from`` on it alone (bitwise).

    ``solve`` returns the same device-tensor dict as ``ptq.LayerBatch.solve``.
    """

    def __init__(self, A, B, levels, idx0, device=None):
        from . import _native as N
        from .ptq import LayerBatch

        torch = N.torch_cuda()
        dev_in = isinstance(A, torch.Tensor)  # a device A (m x n, float64) is used in place
        if not dev_in:
            A = np.ascontiguousarray(A, dtype=np.float64)
        B = np.ascontiguousarray(np.atleast_2d(B), dtype=np.float64)
        idx0 = np.ascontiguousarray(np.atleast_2d(idx0), dtype=np.int32)
        levels = np.asarray(levels, dtype=np.float64)
        m, n = (int(v) for v in A.shape)
        if B.shape[1] != m or idx0.shape != (B.shape[0], n):
            raise ValueError("B must be slices x m and idx0 slices x n")
        if levels.ndim != 1 or np.any(np.diff(levels) <= 0) or not np.all(np.isfinite(levels)):
            raise ValueError("levels must be strictly increasing and finite")
        if idx0.min() < 0 or idx0.max() >= levels.size:
            raise ValueError("idx0 outside the level set")
        self._lb = lb = LayerBatch.__new__(LayerBatch)
        lb.torch, lb.lib = torch, N.load_library()
        lb.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        dev = lb.device
        lb.m, lb.n, lb.count, lb.nlev = m, n, B.shape[0], levels.size
        lb.rows = np.arange(lb.count)
        lb.At = (A.to(dev, torch.float64) if dev_in else torch.from_numpy(A).to(dev)).t().contiguous()
        lb.B = torch.from_numpy(B).to(dev)
        lb.L = torch.from_numpy(np.tile(levels, (lb.count, 1))).to(dev)
        lb.idx0 = torch.from_numpy(idx0).to(dev)
        lb.r0 = torch.empty((lb.count, m), dtype=torch.float64, device=dev)
        lb.obj0 = torch.empty(lb.count, dtype=torch.float64, device=dev)
        lb.cnt0 = torch.empty(lb.count, dtype=torch.int32, device=dev)
        prob = lb.problem()
        sol = N.SolutionPtrs(lb.idx0.data_ptr(), lb.r0.data_ptr(), lb.obj0.data_ptr(), lb.cnt0.data_ptr())
        # start residuals in numpy's BLAS order (core.py:183-197), on the device
        N.check(lb.lib.amvm_compute_residual(N.C.byref(prob), N.C.byref(sol), N.stream_handle()),
                "amvm_compute_residual")
        lb.prepared = True

    def solve(self, cfg=None, seeds=None, trace: bool = False) -> dict:
        return self._lb.solve(cfg, seeds=seeds, trace=trace)

    def check_status(self) -> None:
        self._lb.check_status()


class SparseSliceBatch:
    """Tomography slices sharing a SPARSE projector, solved by the sparse
    engine (``amvm_solve_sparse``): A stays CSC + CSR on the device (the
    full 256^2 x 180 slice: ~340 MB instead of 2 x 24 GB dense copies).
    Same results as :class:`SliceBatch` on the same inputs (bit for bit).

    ``csr`` = (indptr int64[m+1], indices int64[nnz], values f64[nnz]) device
    tensors with ascending columns per row (``projection_csr_device``); B is
    slices x m, idx0 slices x n (host or device).  The start residual
    A x0 - b is computed on the device in numpy's dense dgemv order."""

    def __init__(self, csr, m: int, n: int, B, levels, idx0, device=None, column_filter: bool = True):
        from . import _native as N

        torch = N.torch_cuda()
        self.torch, self.lib = torch, N.load_library()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        indptr, indices, values = (t.to(dev) for t in csr)
        levels = np.asarray(levels, dtype=np.float64)
        if levels.ndim != 1 or np.any(np.diff(levels) <= 0) or not np.all(np.isfinite(levels)):
            raise ValueError("levels must be strictly increasing and finite")
        B = torch.as_tensor(np.asarray(B) if not isinstance(B, torch.Tensor) else B, dtype=torch.float64).to(dev)
        idx0 = torch.as_tensor(np.asarray(idx0) if not isinstance(idx0, torch.Tensor) else idx0).to(dev)
        B = B.reshape(-1, m).contiguous()
        idx0 = idx0.reshape(B.shape[0], n).to(torch.int32).contiguous()
        if int(idx0.min()) < 0 or int(idx0.max()) >= levels.size:
            raise ValueError("idx0 outside the level set")
        self.m, self.n, self.count, self.nlev = m, n, B.shape[0], levels.size
        self.nnz = int(values.numel())
        # CSR with int32 columns; CSC (rows ascending per column) by a stable sort on the column
        self.rptr = indptr.contiguous()
        self.rcol = indices.to(torch.int32).contiguous()
        self.rval = values.contiguous()
        rows = torch.repeat_interleave(torch.arange(m, device=dev), indptr[1:] - indptr[:-1])
        order = torch.sort(indices * m + rows, stable=True).indices
        self.crow = rows[order].to(torch.int32).contiguous()
        self.cval = values[order].contiguous()
        counts = torch.bincount(indices, minlength=n)
        self.cptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        self.cptr[1:] = torch.cumsum(counts, 0)
        self.max_col_nnz = int(counts.max().item()) if n else 0
        # column_filter: the candidate filter indexes the filter rows' nonzeros
        # by column (same survivors; False runs the general staged-row filter)
        self.max_row_nnz = int((indptr[1:] - indptr[:-1]).max().item()) if m and column_filter else 0
        self.B = B
        self.L = torch.from_numpy(np.tile(levels, (self.count, 1))).to(dev)
        self.idx0 = idx0
        lvd = torch.from_numpy(levels).to(dev)
        X = lvd[idx0.long()].t().contiguous()                  # n x S level values of the start
        y = projections_device((self.rptr, indices, self.rval), m, n, X)  # A @ x in numpy's dgemv order
        self.r0 = (y - B).contiguous()
        self.obj0 = self.r0.abs().amax(dim=1).contiguous()
        self.cnt0 = torch.zeros(self.count, dtype=torch.int32, device=dev)

    def problem(self):
        from . import _native as N

        return N.SparseProblem(self.m, self.n, self.nlev, self.count, self.nnz, self.max_col_nnz,
                               self.cptr.data_ptr(), self.crow.data_ptr(), self.cval.data_ptr(),
                               self.rptr.data_ptr(), self.rcol.data_ptr(), self.rval.data_ptr(),
                               self.B.data_ptr(), self.L.data_ptr(), self.max_row_nnz)

    def workspace_bytes(self, cfg=None) -> int:
        from . import _native as N
        from .controller import SolverConfig, make_params

        cfg = cfg or SolverConfig()
        prm = make_params(cfg, self.n, time_budget=cfg.time_limit)
        prob = self.problem()
        return int(self.lib.amvm_sparse_workspace_bytes(N.C.byref(prob), N.C.byref(prm)))

    def solve(self, cfg=None, seeds=None, trace: bool = False) -> dict:
        """amvm_solve_sparse over the slices; returns device tensors (no sync),
        the same dict as ``ptq.LayerBatch.solve``."""
        from . import _native as N
        from .controller import SolverConfig, make_params

        torch = self.torch
        cfg = cfg or SolverConfig()
        dev = self.device
        seeds = np.arange(self.count) if seeds is None else np.asarray(seeds)
        # pinned + non_blocking: kept on self until the copy has run
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
            for k, dt in (("trace_current_t", torch.float64), ("trace_best_t", torch.float64),
                          ("trace_pair", torch.uint8), ("trace_accepted", torch.uint8)):
                o[k] = torch.empty((c, T), dtype=dt, device=dev)
            tr = [o[k].data_ptr() for k in ("trace_current_t", "trace_best_t", "trace_pair", "trace_accepted")]
        res = N.ResultPtrs(
            N.SolutionPtrs(o["best_idx"].data_ptr(), o["best_residual"].data_ptr(),
                           o["best_objective"].data_ptr(), o["best_updates"].data_ptr()),
            o["initial_objective"].data_ptr(), o["iterations"].data_ptr(), o["operator_uses"].data_ptr(),
            *tr, o["moves_scored"].data_ptr(), o["phase_cycles"].data_ptr())
        prm = make_params(cfg, n, time_budget=cfg.time_limit)
        prob = self.problem()
        nbytes = self.lib.amvm_sparse_workspace_bytes(N.C.byref(prob), N.C.byref(prm))
        if nbytes == 0:
            raise ValueError("problem shape or parameters rejected by libamvm")
        ws = N.workspace(dev, nbytes)
        start = N.SolutionPtrs(self.idx0.data_ptr(), self.r0.data_ptr(), self.obj0.data_ptr(),
                               self.cnt0.data_ptr())
        N.check(self.lib.amvm_solve_sparse(N.C.byref(prob), N.C.byref(prm), N.C.byref(start), N.ptr(self.rng),
                                           N.C.byref(res), N.ptr(ws), N.C.c_size_t(ws.numel()),
                                           N.stream_handle()), "amvm_solve_sparse")
        self._ws = ws
        return o

    def check_status(self) -> None:
        from . import _native as N

        N.check(self.lib.amvm_status(N.ptr(self._ws), N.stream_handle()), "amvm_solve_sparse")


def projection_csr_device(side: int, n_angles: int, device=None):
    """The projector built on the GPU (``amvm_projector_indptr`` /
    ``amvm_projector_fill``, csrc/amvm_tomo.cuh) as device CSR tensors
    (indptr, indices int64, values f64), bit-identical to
    :func:`projection_csr` and to the reference's ``parallel_beam_matrix``
    (builders.py:186-239).  The angle cosines/sines come from numpy, as in
    the reference (builders.py:234-235)."""
    from . import _native as N

    torch = N.torch_cuda()
    lib = N.load_library()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    th = np.arange(n_angles) * np.pi / n_angles
    c, s = np.cos(th), np.sin(th)
    dirs = torch.from_numpy(np.ascontiguousarray(np.stack([c, s, -s, c], axis=1))).to(dev)
    rows = side * n_angles
    ws = torch.empty(int(lib.amvm_projector_workspace_bytes(side, n_angles)), dtype=torch.uint8, device=dev)
    indptr = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    st = N.stream_handle()
    N.check(lib.amvm_projector_indptr(side, n_angles, N.ptr(dirs), N.ptr(indptr), N.ptr(ws),
                                      N.C.c_size_t(ws.numel()), st), "amvm_projector_indptr")
    nnz = int(indptr[-1].item())
    indices = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
    values = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    N.check(lib.amvm_projector_fill(side, n_angles, N.ptr(dirs), N.ptr(indptr), N.ptr(indices), N.ptr(values),
                                    st), "amvm_projector_fill")
    return indptr, indices[:nnz], values[:nnz]


def projections_device(csr, m: int, n: int, X, noise=None):
    """``A @ X[:, s] (+ noise[s])`` for each column s of X (n x S, device),
    in numpy's dense dgemv order (``amvm_csr_gemv``): bitwise the
    reference's ``A @ truth.ravel() + noise`` (builders.py:322).  Returns
    S x m."""
    from . import _native as N

    torch = N.torch_cuda()
    lib = N.load_library()
    indptr, indices, values = csr
    X = X.contiguous()
    S = X.shape[1]
    out = torch.empty((S, m), dtype=torch.float64, device=X.device)
    nz = noise.contiguous() if noise is not None else None
    N.check(lib.amvm_csr_gemv(m, n, S, N.ptr(indptr), N.ptr(indices), N.ptr(values), N.ptr(X),
                              N.ptr(nz) if nz is not None else None, N.ptr(out), N.stream_handle()),
            "amvm_csr_gemv")
    return out


def sirt_device(csr, m: int, n: int, B, iters: int, lo=None, hi=None):
    """Clamped SIRT (builders.py:242-274) for the S right-hand sides B (S x m,
    device) sharing the CSR A, on the GPU (``amvm_sirt``); returns X (n x S).
    Same validation as the reference; the sums run in sparse storage order,
    so X agrees with the reference to rounding."""
    from . import _native as N

    torch = N.torch_cuda()
    lib = N.load_library()
    indptr, indices, values = csr
    if iters < 0:
        raise ValueError("iters must be non-negative")
    if bool((values < 0).any()):
        raise ValueError("the projection matrix must be non-negative")
    if int(indptr[-1]) == 0:
        raise ValueError("every row of A is zero")
    B = B.contiguous()
    S = B.shape[0]
    nnz = int(values.numel())
    X = torch.empty((n, S), dtype=torch.float64, device=B.device)
    ws = torch.empty(int(lib.amvm_sirt_workspace_bytes(m, n, nnz, S)), dtype=torch.uint8, device=B.device)
    clamp = lo is not None or hi is not None
    lo_v = float(lo) if lo is not None else -np.inf
    hi_v = float(hi) if hi is not None else np.inf
    N.check(lib.amvm_sirt(m, n, nnz, S, N.ptr(indptr), N.ptr(indices), N.ptr(values), N.ptr(B), int(iters),
                          lo_v, hi_v, int(clamp), N.ptr(X), N.ptr(ws), N.C.c_size_t(ws.numel()),
                          N.stream_handle()), "amvm_sirt")
    return X


def build_tomo_device(side: int, gray_levels, n_angles: int, noise: float, seeds=(0,), phantom_kinds=("disk",),
                      sirt_iters: int = 500, device=None) -> dict:
    """The reference's ``build_tomo`` (builders.py:306-327) for several slices
    at once, front end on the GPU: projector (bitwise), noisy projections
    (bitwise; the uniform noise is drawn by numpy from each slice's seed, as
    the reference does), clamped SIRT warm start (to rounding) and its
    nearest-level start.  Slice k uses seeds[k] and phantom_kinds[k % len].
    Returns device tensors: csr, B (S x m), warm (S x n), idx0 (S x n int32),
    truth (S x n) and the host levels."""
    from . import _native as N

    torch = N.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    lv = np.asarray(gray_levels, dtype=np.float64)
    m, n = n_angles * side, side * side
    csr = projection_csr_device(side, n_angles, dev)
    truths, noises = [], []
    for k, seed in enumerate(seeds):
        labels = phantom(phantom_kinds[k % len(phantom_kinds)], side)
        truths.append(lv[np.minimum(labels, lv.size - 1)].ravel())
        noises.append(np.random.default_rng(seed).uniform(-noise, noise, m))
    truth = torch.from_numpy(np.stack(truths)).to(dev)
    B = projections_device(csr, m, n, truth.t().contiguous(), torch.from_numpy(np.stack(noises)).to(dev))
    X = sirt_device(csr, m, n, B, sirt_iters, lo=float(lv[0]), hi=float(lv[-1]))
    warm = X.t().contiguous()
    lvd = torch.from_numpy(lv).to(dev)
    idx0 = torch.argmin(torch.abs(warm[:, :, None] - lvd[None, None, :]), dim=2).to(torch.int32)
    return {"csr": csr, "B": B, "warm": warm, "idx0": idx0, "truth": truth, "levels": lv, "m": m, "n": n}


# ----------------------------------------------------------- many slices
@dataclass
class SliceReport:
    """Per-slice results of a tomography batch (one reference ``solve`` per
    slice, builders.py:302-318): slice ids, best level indices (int8), best
    and initial l_inf, iterations, candidate moves scored (reference-
    equivalent, raw)."""

    slices: np.ndarray
    codes: np.ndarray
    objective: np.ndarray
    initial_objective: np.ndarray
    iterations: np.ndarray
    moves_scored: np.ndarray
    seconds: dict = field(default_factory=dict)


def slice_report(slices, host: dict, seconds: dict | None = None) -> SliceReport:
    """Assemble a SliceReport from per-slice HOST arrays in the device result
    layout (best_idx, best_objective, initial_objective, iterations,
    moves_scored)."""
    return SliceReport(slices=np.asarray(slices), codes=np.asarray(host["best_idx"]).astype(np.int8),
                       objective=np.asarray(host["best_objective"]),
                       initial_objective=np.asarray(host["initial_objective"]),
                       iterations=np.asarray(host["iterations"]), moves_scored=np.asarray(host["moves_scored"]),
                       seconds=dict(seconds or {}))


def solve_slices(side: int, gray_levels, n_angles: int, noise: float, slices, phantom_kinds=("disk",),
                 cfg=None, sirt_iters: int = 500, device=None) -> SliceReport:
    """Solve the tomography slices ``slices`` (global ids: slice k uses
    phantom_kinds[k % len], noise seed k and ALNS seed k) of one projector
    geometry on this GPU: device front end (projector, projections, SIRT
    start), one batched ALNS solve, report.  Shard ``slices`` across ranks
    with ``shard.shard_rows`` and assemble with :func:`gather_slices`."""
    from . import _native as N
    from .controller import SolverConfig

    torch = N.torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    slices = np.asarray(slices, dtype=np.int64)
    kinds = tuple(phantom_kinds[int(k) % len(phantom_kinds)] for k in slices)
    t0 = time.perf_counter()
    fe = build_tomo_device(side, gray_levels, n_angles, noise, seeds=tuple(int(k) for k in slices),
                           phantom_kinds=kinds, sirt_iters=sirt_iters, device=dev)
    m, n = fe["m"], fe["n"]
    # the projector stays sparse: the sparse engine (same results as the dense
    # one, and the full 256^2 x 180 geometry fits in a few GB)
    sb = SparseSliceBatch(fe["csr"], m, n, fe["B"], fe["levels"], fe["idx0"], device=dev)
    o = sb.solve(cfg or SolverConfig(), seeds=slices)
    sb.check_status()
    t1 = time.perf_counter()
    host = {k: o[k].cpu().numpy() for k in ("best_objective", "initial_objective", "iterations", "moves_scored")}
    host["best_idx"] = o["best_idx"].to(torch.int8).cpu().numpy()
    return slice_report(slices, host, {"device_pipeline": t1 - t0})


def gather_slices(rep: SliceReport, total: int, group=None) -> SliceReport:
    """All-gather every rank's slice results (one collective per field; NCCL
    on GPUs, gloo on CPU) into one report ordered by slice id."""
    from .shard import gather_rows

    ids, f = gather_rows(rep.slices, {"codes": rep.codes, "objective": rep.objective,
                                      "initial_objective": rep.initial_objective, "iterations": rep.iterations,
                                      "moves_scored": rep.moves_scored}, total, group)
    return SliceReport(slices=ids, codes=f["codes"], objective=f["objective"],
                       initial_objective=f["initial_objective"], iterations=f["iterations"],
                       moves_scored=f["moves_scored"], seconds=dict(rep.seconds))
