"""Per-CTA timeline of one k_score_adj launch (diagnostic build with
-DAMVM_SCORE_TIMELINE): stamps 0 start, 1 init done, 2 first stage landed,
3 last stage done, 4 columns final, 5 ticket, 6 best written (last CTA)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13437_b200 import _native as N  # noqa: E402
from paper_2508_13437_b200.scoring import score_moves_device  # noqa: E402

lib = N.load_library()
dev = torch.device("cuda", 0)
m, n, nlev = 2048, int(os.environ.get("NCOLS", "4096")), 16
At = torch.randn((n, m), dtype=torch.float64, device=dev)
lv = torch.linspace(-1, 1, nlev, dtype=torch.float64)[None].to(dev)
idx = torch.randint(0, nlev, (1, n), dtype=torch.int32, device=dev)
s = torch.randn((1, m), dtype=torch.float64, device=dev) * 0.1
B = torch.zeros((1, m), dtype=torch.float64, device=dev)
prob = N.Problem(m, n, nlev, 1, At.data_ptr(), B.data_ptr(), lv.data_ptr())
ws = torch.zeros(int(lib.amvm_score_workspace_bytes(N.C.byref(prob))), dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
t, best, bt = score_moves_device(prob, idx, s, "adjacent", ws)
args = (N.C.byref(prob), N.ptr(idx), N.ptr(s), 1, N.ptr(t), *((N.ptr(best), N.ptr(bt)) if os.environ.get("BEST", "1") == "1" else (None, None)), N.ptr(ws), ws.numel(),
        N.stream_handle())
out = np.zeros((148, 8), dtype=np.uint64)
lib.amvm_debug_score_timeline.argtypes = [C.c_void_p, C.c_int]
for rep in range(3):
    flush.zero_()
    torch.cuda.synchronize()
    lib.amvm_score_moves(*args)
    torch.cuda.synchronize()
    lib.amvm_debug_score_timeline(out.ctypes.data, 148)
    t0 = out[:, 0].min()
    rel = (out.astype(np.int64) - int(t0)) / 1e3
    names = ["start", "init", "first", "laststage", "preticket", "ticket", "best", "atomic"]
    print(f"rep {rep}: " + "  ".join(
        f"{nm}: med {np.median(rel[:, k]):.2f} max {rel[:, k].max():.2f}" for k, nm in enumerate(names) if nm != "best"))
    lastcta = np.argmax(out[:, 6])
    print("   best written at", (int(out[lastcta, 6]) - int(t0)) / 1e3, "us by CTA", lastcta,
          "start spread", rel[:, 0].max())

st = np.zeros((148, 2, 16), dtype=np.uint64)
lib.amvm_debug_score_stages.argtypes = [C.c_void_p, C.c_int]
lib.amvm_debug_score_stages(st.ctypes.data, 148)
rel = (st.astype(np.int64) - int(t0)) / 1e3
for b in (0, 50, 100):
    print(f"CTA {b} issue:", " ".join(f"{x:.2f}" for x in rel[b, 0, :8]))
    print(f"CTA {b} ready:", " ".join(f"{x:.2f}" for x in rel[b, 1, :8]))
print("median ready per stage:", " ".join(f"{np.median(rel[:, 1, k]):.2f}" for k in range(8)))
print("median issue per stage:", " ".join(f"{np.median(rel[:, 0, k]):.2f}" for k in range(8)))
