"""Loading the committed golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str) -> list[dict]:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    count = int(z["count"])
    recs = [dict() for _ in range(count)]
    for key in z.files:
        if key == "count":
            continue
        k, field = key.split("/", 1)
        v = z[key]
        recs[int(k)][field] = v.item() if v.ndim == 0 else v
    return recs


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_kwargs(rec: dict) -> dict:
    out = {k[4:]: rec[k] for k in rec if k.startswith("cfg_")}
    out["l2_tiebreak"] = bool(out["l2_tiebreak"])
    out["max_candidates"] = None if out["max_candidates"] < 0 else int(out["max_candidates"])
    for key in ("k_eps", "max_iters", "seed"):
        out[key] = int(out[key])
    return out


def named_A(name: str, rec: dict):
    """Regenerate a named config's A from its recipe; None if the host's numpy
    does not reproduce the reference bits (sha mismatch)."""
    from tests.golden import recipes
    data, _ = recipes.named_case(name)
    if sha(data["A"]) != rec["A_sha"]:
        return None
    return data["A"]


def stored_A(rec: dict) -> np.ndarray:
    """Dense A of a fixture that stores it sparsely (A_shape/A_rows/A_cols/A_vals)."""
    A = np.zeros(tuple(int(x) for x in rec["A_shape"]))
    A[rec["A_rows"], rec["A_cols"]] = rec["A_vals"]
    return A
