"""Goldens for the reference's remaining public API on the path, made by
running the UNMODIFIED reference (dev container only):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_api.py

* apply_shift / apply_swap sequences (core.py:208-245), including runs that
  cross REFRESH_PERIOD (the dgemv recompute of core.py:173-177) and no-op
  shifts (core.py:219-220);
* accept verdicts (controller.py:168-183) on tie cases whose residuals differ
  only by rounding (the l2 branch decides);
* OperatorBank / select_operators / update_weights trajectories
  (controller.py:71-131): picks, final weights/scores/uses, RNG state;
* best_swap with the l2 tie-break (localsearch.py:181-246) for several worker
  counts (chunk winners merged by (t, l2, i, j)), including the reference's
  own tie instance (tests/test_localsearch.py:304-332).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import dmmv  # noqa: E402
from dmmv import controller as ctl  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden import make_golden as mg  # noqa: E402
from tests.golden import recipes  # noqa: E402

OUTCOMES = (ctl.OUTCOME_NEW_BEST, ctl.OUTCOME_IMPROVED, ctl.OUTCOME_ACCEPTED, ctl.OUTCOME_REJECTED)


def rand_inst(rng, m=None, n=None, nlev=None, integer=False):
    m = int(rng.integers(1, 60)) if m is None else m
    n = int(rng.integers(2, 12)) if n is None else n
    nlev = int(rng.integers(2, 7)) if nlev is None else nlev
    if integer:
        A = rng.integers(-5, 6, (m, n)).astype(float)
        b = rng.integers(-9, 10, m).astype(float)
        lv = np.arange(nlev, dtype=float) - 1.0
    else:
        A = rng.uniform(-1.0, 1.0, (m, n))
        b = rng.uniform(-1.0, 1.0, m)
        lv = recipes._levels(rng, nlev)
    return dmmv.Instance(A, b, dmmv.ValueSet(lv))


def base(inst, sol):
    return {"A": inst.A, "b": inst.b, "levels": inst.values.levels,
            "idx0": sol.idx.astype(np.int32), "r0": sol.residual.copy(), "obj0": sol.objective,
            "cnt0": sol.updates_since_refresh}


def shift_cases():
    out = []
    for k in range(24):
        rng = np.random.default_rng(5000 + k)
        inst = rand_inst(rng, integer=(k % 4 == 1))
        sol = dmmv.Solution.from_indices(inst, rng.integers(0, len(inst.values), inst.n))
        # k % 3 == 2: start just below REFRESH_PERIOD so the sequence refreshes
        sol.updates_since_refresh = [0, 400, 990][k % 3]
        rec = base(inst, sol)
        steps = 40
        js = rng.integers(0, inst.n, steps).astype(np.int32)
        ls = rng.integers(0, len(inst.values), steps).astype(np.int32)
        ls[::7] = sol.idx[js[::7]]  # some no-op shifts (current level)
        objs, cnts = [], []
        for j, lvl in zip(js, ls):
            lvl = int(sol.idx[j]) if lvl < 0 else int(lvl)
            dmmv.apply_shift(inst, sol, int(j), lvl)
            objs.append(sol.objective)
            cnts.append(sol.updates_since_refresh)
        rec.update({"js": js, "ls": ls, "objs": np.array(objs), "cnts": np.array(cnts, np.int32),
                    "idx1": sol.idx.astype(np.int32), "r1": sol.residual, "obj1": sol.objective,
                    "cnt1": sol.updates_since_refresh})
        out.append(rec)
    return out


def swap_cases():
    out = []
    for k in range(24):
        rng = np.random.default_rng(6000 + k)
        inst = rand_inst(rng, integer=(k % 4 == 1))
        sol = dmmv.Solution.from_indices(inst, rng.integers(0, len(inst.values), inst.n))
        sol.updates_since_refresh = [0, 500, 985][k % 3]
        rec = base(inst, sol)
        pis, pjs, objs, cnts = [], [], [], []
        for _ in range(30):
            lv = sol.idx
            pairs = [(i, j) for i in range(inst.n) for j in range(inst.n)
                     if i != j and inst.values[int(lv[i])] != inst.values[int(lv[j])]]
            if not pairs:
                break
            i, j = pairs[int(rng.integers(0, len(pairs)))]
            dmmv.apply_swap(inst, sol, i, j)
            pis.append(i); pjs.append(j); objs.append(sol.objective); cnts.append(sol.updates_since_refresh)
        rec.update({"is": np.array(pis, np.int32), "js": np.array(pjs, np.int32), "objs": np.array(objs),
                    "cnts": np.array(cnts, np.int32), "idx1": sol.idx.astype(np.int32), "r1": sol.residual,
                    "obj1": sol.objective, "cnt1": sol.updates_since_refresh})
        out.append(rec)
    return out


def accept_cases():
    """(current, candidate) residual pairs: strict wins, tie-tolerance cases
    whose residuals differ by revert round-off, and clear losses."""
    out = []
    for k in range(40):
        rng = np.random.default_rng(7000 + k)
        m = [1, 2, 3, 15, 16, 17, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 255, 256, 300, 1024][k % 20]
        cur = rng.uniform(-1.0, 1.0, m)
        kind = k % 4
        if kind == 0:     # candidate = current after a shift and its revert (round-off only)
            a = rng.uniform(-1.0, 1.0, m)
            d = float(rng.uniform(-2.0, 2.0))
            cand = (cur + d * a) + (-d) * a
        elif kind == 1:   # strictly smaller objective
            cand = cur * 0.5
        elif kind == 2:   # tie within ACCEPT_TIE_TOL: same max, different bulk
            cand = rng.uniform(-1.0, 1.0, m) * 0.99
            j = int(np.argmax(np.abs(cur)))
            cand[j % m] = cur[j]
        else:             # worse
            cand = cur * 1.01
        co, ca = float(np.max(np.abs(cur))), float(np.max(np.abs(cand)))
        if kind == 0 and k % 8 == 4:
            ca = co + 5e-13  # inside the tolerance band, not strictly smaller
        rec = {"cur_r": cur, "cur_obj": co, "cand_r": cand, "cand_obj": ca}
        for l2 in (0, 1):
            cfg = dmmv.SolverConfig(l2_tiebreak=bool(l2))
            c = dmmv.Solution(np.zeros(1, np.intp), cur, co)
            d_ = dmmv.Solution(np.zeros(1, np.intp), cand, ca)
            rec[f"verdict_l2_{l2}"] = int(dmmv.accept(c, d_, cfg))
        out.append(rec)
    return out


def bank_cases():
    out = []
    for k in range(12):
        rng_o = np.random.default_rng(8000 + k)
        decay = [0.8, 0.5, 1.0, 0.95][k % 4]
        cfg = dmmv.SolverConfig(decay=decay, sigma1=[3.0, 5.0, 1.0][k % 3], sigma2=[2.0, 2.0, 0.5][k % 3],
                                sigma3=[1.0, 0.0, 0.25][k % 3])
        bank = ctl.OperatorBank(decay)
        rng = np.random.default_rng(k)
        seed_state = rng.bit_generator.state
        picks, outs = [], []
        for it in range(230):
            p = ctl.select_operators(bank, rng)
            o = int(rng_o.integers(0, 4))
            ctl.update_weights(bank, p, OUTCOMES[o], cfg)
            picks.append(p); outs.append(o)
        st = rng.bit_generator.state
        out.append({"seed": k, "decay": decay, "sigma": np.array([cfg.sigma1, cfg.sigma2, cfg.sigma3]),
                    "outcomes": np.array(outs, np.int32), "picks": np.array(picks, np.int32),
                    "weights": bank.weights.copy(), "scores": bank.scores.copy(),
                    "segment_uses": bank.segment_uses.copy(), "lifetime_uses": bank.lifetime_uses.copy(),
                    "iteration": bank.iteration,
                    "state_after": np.array([st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1),
                                             st["state"]["inc"] >> 64, st["state"]["inc"] & (2**64 - 1),
                                             st["has_uint32"], st["uinteger"]], dtype=np.uint64),
                    "state_before_ok": int(seed_state["bit_generator"] == "PCG64")})
    return out


def tie_instance():
    A = np.column_stack([[0.4, 0.0, 0.0, 0.5], [-0.4, 0.0, 0.0, 0.5],
                         [0.4, 0.0, -0.45, -0.5], [-0.4, 0.0, 0.45, -0.5]])
    b = np.array([-0.1, -0.5, 0.05, 0.0])
    inst = dmmv.Instance(A=A, b=b, values=dmmv.ValueSet(np.array([0.0, 1.0])))
    return inst, dmmv.Solution.from_indices(inst, np.array([1, 0, 1, 0]))


def swap_l2_cases():
    out = []
    cases = [tie_instance()]
    for k in range(40):
        rng = np.random.default_rng(9000 + k)
        # integer instances make exact t' ties (and so the l2 branch) common
        inst = rand_inst(rng, m=int(rng.integers(1, 40)), n=int(rng.integers(3, 14)),
                         nlev=int(rng.integers(2, 5)), integer=(k % 2 == 0))
        cases.append((inst, dmmv.Solution.from_indices(inst, rng.integers(0, len(inst.values), inst.n))))
    for inst, sol in cases:
        rec = base(inst, sol)
        res = []
        for workers in (1, 2, 3, 5):
            for k_eps, mc in ((100, None), (2, 7)):
                fc = dmmv.FilterConfig(k_eps=k_eps, max_candidates=mc, workers=workers, l2_tiebreak=True)
                got = dmmv.best_swap(inst, sol, fc)
                res.append([workers, k_eps, -1 if mc is None else mc,
                            -1 if got is None else got.i, -1 if got is None else got.j,
                            0.0 if got is None else got.delta, 0.0 if got is None else got.predicted_t])
        rec["runs"] = np.array(res, dtype=float)
        out.append(rec)
    return out


def main() -> None:
    assert os.environ.get("OPENBLAS_NUM_THREADS") == "1"
    mg.save("api_shift", shift_cases())
    mg.save("api_swap", swap_cases())
    mg.save("api_accept", accept_cases())
    mg.save("api_bank", bank_cases())
    mg.save("api_swap_l2", swap_l2_cases())


if __name__ == "__main__":
    main()
