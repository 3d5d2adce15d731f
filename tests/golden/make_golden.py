"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the dev container (the reference lives at /root/reference and does not
travel to the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Every fixture stores the inputs the reference saw (or the recipe that
regenerates them plus a sha256 of the regenerated array) and what the
reference returned.  OPENBLAS_NUM_THREADS=1 pins the BLAS order the
reference's residuals are computed in.
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import dmmv  # noqa: E402
from dmmv import controller as ctl  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden import recipes  # noqa: E402

PAIR_IDS = {f"{d}+{r}": k for k, (d, r) in enumerate(ctl.PAIRS)}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_fields(cfg: dmmv.SolverConfig) -> dict:
    return {
        "destroy_rate": cfg.destroy_rate, "alpha": cfg.alpha, "k_eps": cfg.k_eps,
        "max_iters": cfg.max_iters, "seed": cfg.seed, "sigma1": cfg.sigma1,
        "sigma2": cfg.sigma2, "sigma3": cfg.sigma3, "decay": cfg.decay,
        "l2_tiebreak": int(cfg.l2_tiebreak),
        "max_candidates": -1 if cfg.max_candidates is None else cfg.max_candidates,
    }


def solve_record(inst: dmmv.Instance, cfg: dmmv.SolverConfig, store_A: bool) -> dict:
    s0 = dmmv.initial_solution(inst)
    rep = dmmv.solve(inst, cfg)
    rec = {
        "m": inst.m, "n": inst.n, "b": inst.b, "levels": inst.values.levels,
        "idx0": s0.idx.astype(np.int32), "r0": s0.residual, "obj0": s0.objective,
        "A_sha": sha(inst.A),
        "iterations": rep.iterations, "initial_objective": rep.initial_objective,
        "best_idx": rep.best.idx.astype(np.int32), "best_residual": rep.best.residual,
        "best_objective": rep.best.objective, "best_updates": rep.best.updates_since_refresh,
        "operator_uses": np.array([rep.operator_uses[f"{d}+{r}"] for d, r in ctl.PAIRS]),
        "trace_current_t": np.array([e.current_t for e in rep.trace]),
        "trace_best_t": np.array([e.best_t for e in rep.trace]),
        "trace_pair": np.array([PAIR_IDS[e.op_pair] for e in rep.trace], dtype=np.uint8),
        "trace_accepted": np.array([e.accepted for e in rep.trace], dtype=np.uint8),
    }
    if inst.continuous_init is not None:
        rec["continuous_init"] = inst.continuous_init
    if store_A:
        rec["A"] = inst.A
    rec.update({f"cfg_{k}": v for k, v in cfg_fields(cfg).items()})
    return rec


def save(name: str, records: list[dict]) -> None:
    flat = {"count": len(records)}
    for k, rec in enumerate(records):
        for key, val in rec.items():
            flat[f"{k}/{key}"] = np.asarray(val)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **flat)
    print(f"{name}: {len(records)} records, {os.path.getsize(path) / 1024:.0f} KiB")


def mk(data: dict, cfg: dict):
    inst = dmmv.Instance(data["A"], data["b"], dmmv.ValueSet(data["levels"]),
                         continuous_init=data["continuous_init"])
    return inst, dmmv.SolverConfig(**cfg)


def small_solves() -> list[dict]:
    return [solve_record(*mk(*recipes.small_case(k)), store_A=True) for k in range(48)]


def refresh_solves() -> list[dict]:
    return [solve_record(*mk(*recipes.refresh_case(k)), store_A=True) for k in range(3)]


def named_solves() -> dict[str, list[dict]]:
    return {name: [solve_record(*mk(*recipes.named_case(name)), store_A=False)]
            for name in recipes.NAMED}


def sol_fields(prefix: str, sol: dmmv.Solution) -> dict:
    return {f"{prefix}idx": sol.idx.astype(np.int32), f"{prefix}residual": sol.residual,
            f"{prefix}objective": sol.objective, f"{prefix}updates": sol.updates_since_refresh}


def component_cases() -> list[dict]:
    """one_opt / local_search / find_candidates / best_swap / impact_scores /
    destroy / repair on random (instance, solution) pairs."""
    out = []
    for k in range(60):
        data, idx, filt, alpha, seed = recipes.component_case(k)
        inst, _ = mk(data, {})
        sol = dmmv.Solution.from_indices(inst, idx)
        fc = dmmv.FilterConfig(**filt)
        rec = {"A": inst.A, "b": inst.b, "levels": inst.values.levels, "k_eps": fc.k_eps,
               "max_candidates": -1 if fc.max_candidates is None else fc.max_candidates,
               "alpha": alpha, "seed": seed}
        rec.update(sol_fields("in_", sol))
        s = sol.copy(); dmmv.one_opt(inst, s); rec.update(sol_fields("oneopt_", s))
        s = sol.copy(); dmmv.local_search(inst, s, fc); rec.update(sol_fields("ls_", s))
        if sol.objective > 0:
            cands = dmmv.find_candidates(inst, sol, fc)
            rec["fc_i"] = np.array([c.i for c in cands], np.int32)
            rec["fc_j"] = np.array([c.j for c in cands], np.int32)
            rec["fc_delta"] = np.array([c.delta for c in cands])
            bs = dmmv.best_swap(inst, sol, fc)
            rec["bs"] = np.array([-1, -1, 0, 0] if bs is None else [bs.i, bs.j, bs.delta, bs.predicted_t])
            rec["impact"] = dmmv.impact_scores(inst, sol, alpha).d
        r = max(1, min(inst.n, 1 + k % 4))
        rec["r"] = r
        rng = np.random.default_rng(seed)
        ds = dmmv.random_destroy(sol.copy(), r, rng)
        rec["rd_removed"] = ds.removed.astype(np.int32)
        rng = np.random.default_rng(seed)
        ds = dmmv.worst_remove_destroy(inst, sol.copy(), r, alpha, rng)
        rec["wd_removed"] = ds.removed.astype(np.int32)
        if len(inst.values) >= 2:
            rng = np.random.default_rng(seed + 1)
            s = sol.copy(); dmmv.random_repair(inst, s, ds, rng); rec.update(sol_fields("rr_", s))
            s = sol.copy(); dmmv.greedy_repair(inst, s, ds); rec.update(sol_fields("gr_", s))
            rec["saved"] = ds.saved_idx.astype(np.int32)
        out.append(rec)
    return out


def c3_scaled() -> None:
    """Tomography (C3 family) at 64^2 x 45 angles, 3 grey levels: A stored as
    CSR in the fixture (the GPU box has no reference builder)."""
    angles = np.arange(45) * np.pi / 45
    A = dmmv.parallel_beam_matrix(64, angles)
    eta = 0.05 * float(A.sum(axis=1).max())
    spec = dmmv.TomoSpec(side=64, gray_levels=(0.0, 1.0, 2.0), n_angles=45, noise=eta, phantom="squares",
                         sirt_iters=100, seed=0)
    inst, _ = dmmv.build_tomo(spec)
    rec = solve_record(inst, dmmv.SolverConfig(max_iters=4, seed=0), store_A=False)
    Ac = inst.A
    nz = np.nonzero(Ac)
    rec["A_shape"] = np.array(Ac.shape)
    rec["A_rows"] = nz[0].astype(np.int32)
    rec["A_cols"] = nz[1].astype(np.int32)
    rec["A_vals"] = Ac[nz]
    save("solve_c3s", [rec])


def c3_medium() -> None:
    """Tomography at 128^2 x 64 angles (8192 x 16384: 48 s per
    reference iteration).  A is NOT stored: the package's own projector
    (paper_2508_13437_b200.tomo) regenerates it bit-identically (sha checked)."""
    side, n_angles = 128, 64
    A = dmmv.parallel_beam_matrix(side, np.arange(n_angles) * np.pi / n_angles)
    eta = 0.05 * float(A.sum(axis=1).max())
    spec = dmmv.TomoSpec(side=side, gray_levels=(0.0, 1.0, 2.0), n_angles=n_angles, noise=eta,
                         phantom="squares", sirt_iters=100, seed=0)
    inst, _ = dmmv.build_tomo(spec)
    rec = solve_record(inst, dmmv.SolverConfig(max_iters=3, seed=0), store_A=False)
    rec.pop("continuous_init", None)
    rec["A_recipe"] = np.array([side, n_angles])
    save("solve_c3m", [rec])


def main() -> None:
    assert os.environ.get("OPENBLAS_NUM_THREADS") == "1"
    if "--c3s" in sys.argv:
        c3_scaled()
        return
    if "--c3m" in sys.argv:
        c3_medium()
        return
    save("components", component_cases())
    save("small_solves", small_solves())
    save("refresh_solves", refresh_solves())
    for name, recs in named_solves().items():
        save(f"solve_{name}", recs)
    c3_scaled()


if __name__ == "__main__":
    main()
