"""Scorer streaming sweep (diagnostic): per-launch time of amvm_score_moves
(adjacent, one instance, m=2048) vs n, back-to-back launches cycling over
copies of A so every launch reads from HBM; fits t = t0 + bytes / BW."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13437_b200 import _native as N  # noqa: E402
from paper_2508_13437_b200.scoring import score_moves_device  # noqa: E402

lib = N.load_library()
dev = torch.device("cuda", 0)
m, nlev = 2048, 16
res = []
for n in [1024, 4096, 8192, 16384, 32768]:
    copies = max(2, -(-(256 << 20) // (8 * m * n)) + 1)
    Ats = [torch.randn((n, m), dtype=torch.float64, device=dev) for _ in range(copies)]
    lv = torch.linspace(-1, 1, nlev, dtype=torch.float64)[None].to(dev)
    idx = torch.randint(0, nlev, (1, n), dtype=torch.int32, device=dev)
    s = torch.randn((1, m), dtype=torch.float64, device=dev) * 0.1
    B = torch.zeros((1, m), dtype=torch.float64, device=dev)
    probs = [N.Problem(m, n, nlev, 1, a.data_ptr(), B.data_ptr(), lv.data_ptr()) for a in Ats]
    ws = torch.zeros(int(lib.amvm_score_workspace_bytes(N.C.byref(probs[0]))), dtype=torch.uint8, device=dev)
    t, best, bt = score_moves_device(probs[0], idx, s, "adjacent", ws)
    calls = [(N.C.byref(p), N.ptr(idx), N.ptr(s), 1, N.ptr(t), *((N.ptr(best), N.ptr(bt)) if os.environ.get("BEST", "1") == "1" else (None, None)), N.ptr(ws), ws.numel(),
              N.stream_handle()) for p in probs]
    L = 12
    per = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(L):
            lib.amvm_score_moves(*calls[k % copies])
        b.record()
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b) / L)
    ms = float(np.median(per))
    byt = 8 * m * n
    res.append((n, byt, ms))
    print(f"n={n} MB={byt / 1e6:.1f} us={ms * 1e3:.2f} GB/s={byt / ms / 1e6:.0f}", flush=True)
    del Ats
x = np.array([r[1] for r in res]); y = np.array([r[2] for r in res]) * 1e-3
A_ = np.vstack([np.ones_like(x), x]).T
t0, inv = np.linalg.lstsq(A_, y, rcond=None)[0]
print(f"fit: t0 = {t0 * 1e6:.2f} us, asymptotic BW = {1 / inv / 1e9:.0f} GB/s")
