"""ctypes binding of libamvm.so (include/amvm.h) and device-buffer plumbing.

PyTorch is used only for device memory and streams.  There is no CPU
fallback: if the library or a CUDA device is missing, every device-backed
call raises ``RuntimeError`` (``NativeUnavailable``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AMVM_LIBRARY") or os.path.join(HERE, "libamvm.so")  # override for A/B builds

AMVM_OK = 0
AMVM_ERR_INVALID = -1

EXPORTS = (
    "amvm_workspace_bytes", "amvm_solve", "amvm_one_opt", "amvm_local_search",
    "amvm_find_candidates", "amvm_best_swap", "amvm_impact_scores", "amvm_destroy",
    "amvm_repair", "amvm_compute_residual", "amvm_ptq_prepare", "amvm_seed_pcg64", "amvm_status",
    "amvm_strerror", "amvm_abi_version", "amvm_brute_force_workspace_bytes", "amvm_brute_force",
    "amvm_ls_start_workspace_bytes", "amvm_ls_start",
    "amvm_projector_workspace_bytes", "amvm_projector_indptr", "amvm_projector_fill",
    "amvm_csr_gemv", "amvm_sirt_workspace_bytes", "amvm_sirt", "amvm_is_improving", "amvm_swap_check",
    "amvm_score_moves", "amvm_score_workspace_bytes", "amvm_best_swap_l2", "amvm_apply_shift",
    "amvm_apply_swap", "amvm_accept", "amvm_select_operators", "amvm_update_weights",
    "amvm_sparse_workspace_bytes", "amvm_solve_sparse",
)


class NativeUnavailable(RuntimeError):
    pass


class Problem(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nlev", C.c_int64), ("count", C.c_int64),
                ("At", C.c_void_p), ("B", C.c_void_p), ("levels", C.c_void_p)]


class SparseProblem(C.Structure):
    """amvm_sparse_problem: A as CSC + CSR device arrays (include/amvm.h)."""
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nlev", C.c_int64), ("count", C.c_int64),
                ("nnz", C.c_int64), ("max_col_nnz", C.c_int64),
                ("cptr", C.c_void_p), ("crow", C.c_void_p), ("cval", C.c_void_p),
                ("rptr", C.c_void_p), ("rcol", C.c_void_p), ("rval", C.c_void_p),
                ("B", C.c_void_p), ("levels", C.c_void_p),
                ("max_row_nnz", C.c_int64)]  # > 0: the column-indexed candidate filter


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


class PCG64State(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64),
                ("inc_lo", C.c_uint64), ("has_uint32", C.c_uint32), ("uinteger", C.c_uint32)]


class Bank(C.Structure):
    """amvm_bank: OperatorBank (controller.py:71-85) as device data."""
    _fields_ = [("weights", C.c_double * 4), ("scores", C.c_double * 4), ("segment_uses", C.c_int64 * 4),
                ("lifetime_uses", C.c_int64 * 4), ("iteration", C.c_int64), ("decay", C.c_double)]


class SolutionPtrs(C.Structure):
    _fields_ = [("idx", C.c_void_p), ("residual", C.c_void_p), ("objective", C.c_void_p),
                ("updates", C.c_void_p)]


class ResultPtrs(C.Structure):
    _fields_ = [("best", SolutionPtrs), ("initial_objective", C.c_void_p),
                ("iterations", C.c_void_p), ("operator_uses", C.c_void_p),
                ("trace_current_t", C.c_void_p), ("trace_best_t", C.c_void_p),
                ("trace_pair", C.c_void_p), ("trace_accepted", C.c_void_p),
                ("moves_scored", C.c_void_p), ("phase_cycles", C.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libamvm.so (no GPU needed to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing; build it with `python -m paper_2508_13437_b200.build`")
    lib = C.CDLL(path)
    vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    lib.amvm_workspace_bytes.restype = sz
    lib.amvm_workspace_bytes.argtypes = [vp, vp]
    lib.amvm_solve.argtypes = [vp, vp, vp, vp, vp, vp, sz, vp]
    lib.amvm_one_opt.argtypes = [vp, vp, vp, vp, sz, vp]
    lib.amvm_local_search.argtypes = [vp, vp, vp, vp, sz, vp]
    lib.amvm_find_candidates.argtypes = [vp, vp, vp, vp, vp, vp, vp, i32, vp, sz, vp]
    lib.amvm_best_swap.argtypes = [vp, vp, vp, vp, vp, sz, vp]
    lib.amvm_impact_scores.argtypes = [vp, vp, vp, vp, vp, sz, vp]
    lib.amvm_destroy.argtypes = [vp, vp, C.c_int, vp, vp, vp, vp, sz, vp]
    lib.amvm_repair.argtypes = [vp, vp, C.c_int, vp, vp, vp, vp, i32, vp, sz, vp]
    lib.amvm_compute_residual.argtypes = [vp, vp, vp]
    lib.amvm_ptq_prepare.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp, vp]
    lib.amvm_seed_pcg64.argtypes = [vp, i64, vp]
    lib.amvm_status.argtypes = [vp, vp]
    lib.amvm_brute_force_workspace_bytes.restype = sz
    lib.amvm_brute_force_workspace_bytes.argtypes = [vp]
    lib.amvm_brute_force.argtypes = [vp, C.c_int, vp, vp, vp, vp, sz, vp]
    lib.amvm_ls_start_workspace_bytes.restype = sz
    lib.amvm_ls_start_workspace_bytes.argtypes = [i64, i64]
    lib.amvm_ls_start.argtypes = [vp, vp, vp, vp, vp, sz, vp]
    lib.amvm_projector_workspace_bytes.restype = sz
    lib.amvm_projector_workspace_bytes.argtypes = [i64, i64]
    lib.amvm_projector_indptr.argtypes = [i64, i64, vp, vp, vp, sz, vp]
    lib.amvm_projector_fill.argtypes = [i64, i64, vp, vp, vp, vp, vp]
    lib.amvm_is_improving.argtypes = [vp, vp, C.c_double, i64, vp, vp, vp, vp, vp]
    lib.amvm_swap_check.argtypes = [vp, vp, vp, C.c_double, vp, vp, vp]
    lib.amvm_score_moves.argtypes = [vp, vp, vp, C.c_int, vp, vp, vp, vp, sz, vp]
    lib.amvm_score_workspace_bytes.argtypes = [vp]
    lib.amvm_score_workspace_bytes.restype = sz
    lib.amvm_csr_gemv.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, vp, vp]
    lib.amvm_sirt_workspace_bytes.restype = sz
    lib.amvm_sirt_workspace_bytes.argtypes = [i64, i64, i64, i64]
    lib.amvm_sirt.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, i32, C.c_double, C.c_double, C.c_int, vp, vp,
                              sz, vp]
    lib.amvm_best_swap_l2.argtypes = [vp, vp, vp, i32, vp, vp, sz, vp]
    lib.amvm_apply_shift.argtypes = [vp, vp, vp, i64, i32, vp, sz, vp]
    lib.amvm_apply_swap.argtypes = [vp, vp, vp, i64, i64, vp, sz, vp]
    lib.amvm_accept.argtypes = [i64, vp, vp, vp, vp, i32, C.c_double, vp, vp]
    lib.amvm_select_operators.argtypes = [vp, vp, vp, vp]
    lib.amvm_update_weights.argtypes = [vp, vp, i32, i32, vp]
    lib.amvm_sparse_workspace_bytes.restype = sz
    lib.amvm_sparse_workspace_bytes.argtypes = [vp, vp]
    lib.amvm_solve_sparse.argtypes = [vp, vp, vp, vp, vp, vp, sz, vp]
    lib.amvm_strerror.restype = C.c_char_p
    lib.amvm_strerror.argtypes = [C.c_int]
    for name in EXPORTS:
        getattr(lib, name)
    _lib = lib
    return lib


# Host BLAS kernels whose ddot / dgemv order the device emulates bitwise
# (OpenBLAS 0.3.30 SkylakeX ddot + Haswell-microkernel dgemv_t; Cooperlake
# and SapphireRapids build on the SkylakeX kernel list).  np.linalg.norm and
# A @ x follow the host's kernel (controller.py:180, core.py:175,196).
BLAS_ORDERS = ("SkylakeX", "Cooperlake", "SapphireRapids")
_blas_checked: str | None = None


class BlasOrderMismatch(RuntimeError):
    pass


def host_blas() -> dict:
    """numpy's BLAS as threadpoolctl reports it (library, version, architecture)."""
    import numpy  # noqa: F401  (threadpoolctl only sees libraries already loaded)
    try:
        from threadpoolctl import threadpool_info
    except ImportError:
        return {}
    for info in threadpool_info():
        if info.get("user_api") == "blas":
            return {k: info.get(k) for k in ("internal_api", "version", "architecture", "num_threads")}
    return {}


def check_blas_order() -> str:
    """Fail loudly when the host BLAS is not one whose summation order the
    device reproduces: the reference's trajectory on such a host would differ
    from this build's at the first rounding-decided l2 tie.
    ``AMVM_ALLOW_BLAS_MISMATCH=1`` runs anyway (results stay valid solutions,
    just not bitwise equal to that host's reference run)."""
    global _blas_checked
    if _blas_checked is not None:
        return _blas_checked
    info = host_blas()
    arch = info.get("architecture") or "unknown"
    ok = info.get("internal_api") == "openblas" and arch in BLAS_ORDERS
    if not ok and os.environ.get("AMVM_ALLOW_BLAS_MISMATCH") != "1":
        raise BlasOrderMismatch(
            f"host BLAS is {info.get('internal_api')} {info.get('version')} ({arch}); the device reproduces the "
            f"ddot/dgemv summation order of OpenBLAS {'/'.join(BLAS_ORDERS)} only, so this host's reference "
            "trajectory would not be matched bit for bit (set AMVM_ALLOW_BLAS_MISMATCH=1 to run anyway)")
    _blas_checked = arch
    return arch


def torch_cuda():
    """torch with a usable CUDA device, else NativeUnavailable (no fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("the AMVM path needs a CUDA (sm_100) device; none is visible")
    return torch


def check(rc: int, what: str) -> None:
    if rc == AMVM_OK:
        return
    msg = load_library().amvm_strerror(rc).decode()
    if rc == AMVM_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed: {msg} ({rc})")


def stream_handle():
    torch = torch_cuda()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def pcg_from_state(st: dict) -> PCG64State:
    """numpy ``Generator.bit_generator.state`` (PCG64) -> ABI struct."""
    if st.get("bit_generator") != "PCG64":
        raise ValueError("only numpy's default PCG64 bit generator is supported")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return PCG64State(s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"]))


def pcg_to_state(g) -> dict:
    hi, lo = int(g["state_hi"]), int(g["state_lo"])
    ihi, ilo = int(g["inc_hi"]), int(g["inc_lo"])
    return {"bit_generator": "PCG64", "state": {"state": (hi << 64) | lo, "inc": (ihi << 64) | ilo},
            "has_uint32": int(g["has_uint32"]), "uinteger": int(g["uinteger"])}


PCG_DTYPE = np.dtype([("state_hi", "<u8"), ("state_lo", "<u8"), ("inc_hi", "<u8"),
                      ("inc_lo", "<u8"), ("has_uint32", "<u4"), ("uinteger", "<u4")])


def seed_states(seeds) -> np.ndarray:
    """numpy default_rng(seed) PCG64 states for many int seeds (host, in libamvm)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.zeros(seeds.size, PCG_DTYPE)
    rc = load_library().amvm_seed_pcg64(C.c_void_p(seeds.ctypes.data), seeds.size,
                                        C.c_void_p(out.ctypes.data))
    check(rc, "amvm_seed_pcg64")
    return out


def pcg_array(states: list[dict]) -> np.ndarray:
    out = np.zeros(len(states), PCG_DTYPE)
    for k, st in enumerate(states):
        g = pcg_from_state(st)
        out[k] = (g.state_hi, g.state_lo, g.inc_hi, g.inc_lo, g.has_uint32, g.uinteger)
    return out


class Workspace:
    """Caller-owned scratch (amvm_workspace_bytes), kept across calls."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device):
        torch = torch_cuda()
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        return self.buf


_WS: dict = {}


def workspace(device, nbytes: int):
    key = str(device)
    ws = _WS.setdefault(key, Workspace())
    return ws.get(nbytes, device)
