"""Deterministic instance recipes shared by the golden generator and tests.

Pure numpy (no reference import), so the GPU box can regenerate the named
configs' matrices from their seeds; fixtures carry a sha256 of each A so a
host whose numpy produces different bits is detected instead of trusted.
Recipes follow SURVEY.md §8(d) (C1, C1x, C2, C4/C5 rows) and the reference's
own random test helpers (/root/reference/pkg/tests/helpers.py:10-34).
"""

from __future__ import annotations

import numpy as np


def _levels(rng, count):
    while True:
        lv = np.sort(rng.uniform(-1.0, 1.0, count))
        if count == 1 or np.all(np.diff(lv) > 0):
            return lv


def small_case(k: int):
    """48 varied small instances + configs exercising every solve branch."""
    rng = np.random.default_rng(1000 + k)
    m = int(rng.integers(2, 41))
    n = int(rng.integers(2, 25))
    nlev = int(rng.integers(2, 9))
    kind = k % 6
    cont = None
    if kind == 1:  # exact-integer twin
        A = rng.integers(-8, 8, (m, n)).astype(float)
        b = rng.integers(-20, 20, m).astype(float)
        lv = np.arange(nlev, dtype=float) - nlev // 2
    else:
        A = rng.uniform(-1.0, 1.0, (m, n))
        lv = _levels(rng, nlev)
        b = rng.uniform(-1.0, 1.0, m)
        if kind == 2:  # sparse columns: exercises zero entries in impact scores
            A[rng.random((m, n)) < 0.4] = 0.0
        elif kind == 3:  # planted: objective can reach 0 -> early stop
            x = lv[rng.integers(0, nlev, n)]
            b = A @ x
            if k % 12 == 3:
                b = b + rng.uniform(-1e-3, 1e-3, m)
        elif kind == 4:
            cont = rng.uniform(lv[0], lv[-1], n)
        elif kind == 5:
            A[0, :] = 0.0
    cfg = dict(
        max_iters=[60, 150, 300][k % 3], seed=k,
        destroy_rate=[0.005, 0.1, 0.3, 0.5][k % 4],
        l2_tiebreak=(k % 5 != 0), k_eps=[100, 1, 3, 7][(k // 3) % 4],
        max_candidates=[5000, 1, 4, None][(k // 2) % 4],
        alpha=[0.3, 0.0, 1.5][(k // 4) % 3], decay=[0.8, 0.5, 1.0][(k // 5) % 3],
        sigma1=3.0, sigma2=2.0, sigma3=[1.0, 0.0][k % 2],
    )
    return dict(A=A, b=b, levels=lv, continuous_init=cont), cfg


def refresh_case(k: int):
    """Long lineages that cross REFRESH_PERIOD many times (core.py:18,200-205)."""
    rng = np.random.default_rng(2000 + k)
    m, n = [(92, 50), (38, 51), (61, 40)][k]
    nlev = [6, 5, 8][k]
    A = rng.uniform(-1.0, 1.0, (m, n))
    b = rng.uniform(-1.0, 1.0, m)
    lv = _levels(rng, nlev)
    cfg = dict(max_iters=1500, seed=7 + k, destroy_rate=0.2)
    return dict(A=A, b=b, levels=lv, continuous_init=None), cfg


def c1(exact: bool = False):
    """C1 / C1x: m=1024, n=256, V={-8..7}."""
    rng = np.random.default_rng(0)
    if exact:
        A = rng.integers(-8, 8, (1024, 256)).astype(float)
        b = rng.integers(-64, 64, 1024).astype(float)
    else:
        A = rng.uniform(-1.0, 1.0, (1024, 256))
        b = A @ rng.uniform(-8.0, 7.0, 256)
    return dict(A=A, b=b, levels=np.arange(-8, 8, dtype=float), continuous_init=None)


def fir_c2(order: int = 126, bits: int = 10, points: int = 8192):
    """C2: tap-quantised lowpass (tests/test_acceptance.py:103-116 semantics,
    builders.py:88-111) on an 8192-point grid; levels k/2^(bits-1)."""
    bands = [(0.0, 2 * np.pi / 5, 1.0, 1.0), (4 * np.pi / 7, np.pi, 0.0, 1.0)]
    lengths = np.array([hi - lo for lo, hi, _, _ in bands])
    raw = points * lengths / lengths.sum()
    counts = np.maximum(2, np.floor(raw).astype(int))
    short = points - int(counts.sum())
    by_frac = np.argsort(-(raw - np.floor(raw)), kind="stable")
    for q in range(short):
        counts[by_frac[q % len(counts)]] += 1
    omega = np.concatenate([np.linspace(lo, hi, c) for (lo, hi, _, _), c in zip(bands, counts)])
    b = np.concatenate([np.full(c, d) for (_, _, d, _), c in zip(bands, counts)])
    A = np.cos(np.outer(omega, np.arange(order + 1)))
    A[:, 1:] *= 2.0
    coef, *_ = np.linalg.lstsq(A, b, rcond=None)
    half = 2 ** (bits - 1)
    lv = np.arange(-half, half) / half
    return dict(A=A, b=b, levels=lv, continuous_init=coef)


def ptq_layer(d: int, rows: int, calib: int = 2048, scale: float = 0.02):
    """Shared calibration X and weights W (builders.py:355-372
    semantics with one X for the whole layer)."""
    X = np.random.default_rng(0).standard_normal((calib, d))
    W = np.random.default_rng(1).standard_normal((rows, d)) * scale
    return X, W


def ptq_row(X: np.ndarray, w: np.ndarray, bits: int = 4):
    lo, hi = float(w.min()), float(w.max())
    if hi - lo < 1e-12:
        lo, hi = lo - 0.5, hi + 0.5
    lv = np.linspace(lo, hi, 2**bits)
    return dict(A=X, b=X @ w, levels=lv, continuous_init=w)


NAMED = {
    # name: (builder, SolverConfig kwargs)
    "c1": (lambda: c1(False), dict(max_iters=1000, seed=0)),
    "c1x": (lambda: c1(True), dict(max_iters=1000, seed=0)),
    "c2": (lambda: fir_c2(), dict(max_iters=60, seed=0)),
    "c4row": (lambda: ptq_row(*_row(768, 3072, 0)), dict(max_iters=30, seed=0)),
    "c5row": (lambda: ptq_row(*_row(4096, 14336, 0)), dict(max_iters=4, seed=0)),
}


def _row(d, rows, r):
    X, W = ptq_layer(d, rows)
    return X, W[r]


def named_case(name: str):
    build, cfg = NAMED[name]
    return build(), dict(cfg)


def component_case(k: int):
    """Random (instance, solution) pair for the component goldens."""
    rng = np.random.default_rng(3000 + k)
    m = int(rng.integers(2, 31))
    n = int(rng.integers(2, 17))
    nlev = int(rng.integers(2, 7))
    if k % 5 == 1:
        A = rng.integers(-4, 5, (m, n)).astype(float)
        b = rng.integers(-6, 7, m).astype(float)
        lv = np.arange(nlev, dtype=float) - 1.0
    else:
        A = rng.uniform(-1.0, 1.0, (m, n))
        b = rng.uniform(-1.0, 1.0, m)
        lv = _levels(rng, nlev)
        if k % 5 == 2:
            A[rng.random((m, n)) < 0.5] = 0.0
    idx = rng.integers(0, nlev, n)
    filt = dict(k_eps=[100, 1, 2, 5][k % 4], max_candidates=[5000, 1, 3, None][(k // 4) % 4])
    alpha = [0.3, 0.0, 2.0][k % 3]
    return dict(A=A, b=b, levels=lv, continuous_init=None), idx, filt, alpha, 40 + k
