"""CPU-side checks of the boundary: libamvm.so builds/loads, exports every
symbol include/amvm.h declares, and the host mirror validates like the
reference (no GPU calls)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "amvm.h")).read()
    return sorted(set(re.findall(r"AMVM_API\s+[\w\s\*]*?\b(amvm_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2508_13437_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libamvm.so not built (run __graft_entry__.build())")
    lib = _native.load_library()
    declared = _declared()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.EXPORTS)
    assert lib.amvm_abi_version() == 1
    assert lib.amvm_strerror(-3).decode().startswith("workspace")


def test_no_cuda_means_loud_failure(monkeypatch):
    import torch

    import paper_2508_13437_b200 as P
    from paper_2508_13437_b200 import _native

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    inst = P.Instance(np.eye(2), np.ones(2) * 0.4, P.ValueSet([0.0, 1.0]))
    with pytest.raises(_native.NativeUnavailable):
        P.solve(inst, P.SolverConfig(max_iters=3))


def test_host_validation_messages_match_reference():
    import paper_2508_13437_b200 as P

    with pytest.raises(ValueError, match="strictly increasing"):
        P.ValueSet([1.0, 1.0])
    with pytest.raises(ValueError, match="b has length 2, expected m=3"):
        P.Instance(np.zeros((3, 2)), np.zeros(2), P.ValueSet([0, 1]))
    with pytest.raises(ValueError, match="decay"):
        P.SolverConfig(decay=0.0)
    with pytest.raises(ValueError, match="sigma1 >= sigma2"):
        P.SolverConfig(sigma1=1.0, sigma2=2.0)
    with pytest.raises(ValueError, match="k_eps"):
        P.FilterConfig(k_eps=0)
    assert P.removal_count(0.005, 100) == 1 and P.removal_count(0.005, 300) == 2  # banker's rounding
    assert P.removal_count(0.005, 4096) == 20 and P.removal_count(0.005, 768) == 4


def test_trivial_solves_need_no_device(monkeypatch):
    """max_iters=0 / zero objective return the initial solution (controller.py:233-235)."""
    import paper_2508_13437_b200 as P

    inst = P.Instance(np.eye(2), np.array([1.0, 0.0]), P.ValueSet([0.0, 1.0]))
    rep = P.solve(inst, P.SolverConfig(max_iters=5))
    assert rep.iterations == 0 and rep.best.objective == 0.0
    rep = P.solve(P.Instance(np.eye(2), np.array([0.3, 0.2]), P.ValueSet([0.0, 1.0])),
                  P.SolverConfig(max_iters=0))
    assert rep.iterations == 0 and rep.initial_objective == rep.best.objective


def test_seed_states_match_numpy_seedsequence():
    from paper_2508_13437_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libamvm.so not built")
    seeds = np.array([0, 1, 7, 14335, 2**32 + 5, 2**63 + 1], dtype=np.uint64)
    st = _native.seed_states(seeds)
    for k, s in enumerate(seeds):
        assert _native.pcg_to_state(st[k]) == np.random.default_rng(int(s)).bit_generator.state


def test_blas_order_guard(monkeypatch):
    """solve() refuses a host BLAS whose ddot/dgemv order the device does not
    reproduce (the reference's trajectory there would differ), unless the
    caller opts out."""
    import paper_2508_13437_b200 as P
    from paper_2508_13437_b200 import _native

    inst = P.Instance(np.eye(2), np.array([0.3, 0.2]), P.ValueSet([0.0, 1.0]))
    monkeypatch.setattr(_native, "_blas_checked", None)
    monkeypatch.setattr(_native, "host_blas", lambda: {"internal_api": "openblas", "version": "0.3.30",
                                                       "architecture": "Zen", "num_threads": 8})
    monkeypatch.delenv("AMVM_ALLOW_BLAS_MISMATCH", raising=False)
    with pytest.raises(_native.BlasOrderMismatch, match="Zen"):
        P.solve(inst, P.SolverConfig(max_iters=0))
    monkeypatch.setattr(_native, "host_blas", lambda: {"internal_api": "mkl", "architecture": None})
    with pytest.raises(_native.BlasOrderMismatch):
        P.solve(inst, P.SolverConfig(max_iters=0))
    monkeypatch.setenv("AMVM_ALLOW_BLAS_MISMATCH", "1")
    assert P.solve(inst, P.SolverConfig(max_iters=0)).iterations == 0
    monkeypatch.setattr(_native, "_blas_checked", None)
    monkeypatch.delenv("AMVM_ALLOW_BLAS_MISMATCH")
    monkeypatch.setattr(_native, "host_blas", lambda: {"internal_api": "openblas", "architecture": "SkylakeX"})
    assert _native.check_blas_order() == "SkylakeX"


def test_api_validation_matches_reference():
    """apply_shift / apply_swap / OperatorBank / update_weights reject bad
    arguments with the reference's messages before touching the device
    (core.py:215-238, controller.py:74-76, 115-120)."""
    import paper_2508_13437_b200 as P

    inst = P.Instance(np.eye(3), np.zeros(3), P.ValueSet([0.0, 1.0, 2.0]))
    sol = P.Solution.from_indices(inst, np.array([0, 1, 1]))
    with pytest.raises(ValueError, match="variable index 3 out of range for n=3"):
        P.apply_shift(inst, sol, 3, 0)
    with pytest.raises(ValueError, match="level index 3 out of range for 3 levels"):
        P.apply_shift(inst, sol, 0, 3)
    assert P.apply_shift(inst, sol, 1, 1) is sol and sol.updates_since_refresh == 0  # no-op, no device
    with pytest.raises(ValueError, match="two distinct variables"):
        P.apply_swap(inst, sol, 1, 1)
    with pytest.raises(ValueError, match=r"swap indices \(0, 5\) out of range for n=3"):
        P.apply_swap(inst, sol, 0, 5)
    with pytest.raises(ValueError, match="swap of equal values"):
        P.apply_swap(inst, sol, 1, 2)
    with pytest.raises(ValueError, match="decay"):
        P.OperatorBank(0.0)
    bank = P.OperatorBank()
    np.testing.assert_array_equal(bank.probabilities(), [0.25] * 4)
    with pytest.raises(KeyError):
        P.update_weights(bank, 0, "bogus")


def test_ctypes_structs_match_the_c_header(tmp_path):
    """Every struct the Python side hands to libamvm has the C header's size
    and field offsets (gcc on include/amvm.h): the ABI cannot drift silently."""
    import ctypes as C
    import shutil
    import subprocess

    from paper_2508_13437_b200 import _native as N

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    pairs = {"amvm_problem": N.Problem, "amvm_sparse_problem": N.SparseProblem, "amvm_params": N.Params,
             "amvm_pcg64": N.PCG64State, "amvm_bank": N.Bank, "amvm_solution": N.SolutionPtrs,
             "amvm_result": N.ResultPtrs}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "amvm.h"', "int main(void) {"]
    for cname, py in pairs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in pairs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, f"{cname}.{fname}"
