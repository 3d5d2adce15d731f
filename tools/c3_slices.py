"""C3 family throughput: S tomography slices sharing one projector, one
device batch (tomo.SliceBatch).  Front end on the device with torch
(projector CSR -> dense A, noisy projections, clamped SIRT warm start);
the ALNS path is libamvm.  Prints one JSON line.

usage: python tools/c3_slices.py SIDE N_ANGLES SLICES ITERS [SIRT_ITERS]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402

side, n_ang, S, iters = (int(v) for v in sys.argv[1:5])
sirt_iters = int(sys.argv[5]) if len(sys.argv) > 5 else 100
dev = torch.device("cuda")
t0 = time.perf_counter()
indptr, idx, val = tomo.projection_csr(side, n_ang)
m, n = n_ang * side, side * side
t1 = time.perf_counter()
import warnings  # noqa: E402
warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")
A = torch.sparse_csr_tensor(torch.from_numpy(indptr), torch.from_numpy(idx), torch.from_numpy(val),
                            size=(m, n), dtype=torch.float64).to(dev).to_dense()
lv = np.array([0.0, 1.0, 2.0])
kinds = ("squares", "disk", "checker")
truth = torch.stack([torch.from_numpy(lv[np.minimum(tomo.phantom(kinds[k % 3], side), 2)].ravel())
                     for k in range(S)]).to(dev).t()  # n x S
eta = 0.05 * float(A.sum(dim=1).max())
g = torch.Generator(device=dev).manual_seed(0)
Bm = A @ truth + (torch.rand((m, S), generator=g, device=dev, dtype=torch.float64) * 2 - 1) * eta
# SIRT (builders.py:242-274 semantics), batched over slices, clamped
rs, cs = A.sum(dim=1), A.sum(dim=0)
R = torch.where(rs > 0, 1.0 / rs, torch.zeros_like(rs))[:, None]
C = torch.where(cs > 0, 1.0 / cs, torch.zeros_like(cs))[:, None]
X = torch.zeros((n, S), dtype=torch.float64, device=dev)
for _ in range(sirt_iters):
    X = (X + C * (A.t() @ (R * (Bm - A @ X)))).clamp(lv[0], lv[-1])
idx0 = torch.argmin((X[:, :, None] - torch.from_numpy(lv).to(dev)).abs(), dim=2).t().to(torch.int32)
torch.cuda.synchronize()
t2 = time.perf_counter()
sb = tomo.SliceBatch(A, Bm.t().contiguous().cpu().numpy(), lv, idx0.cpu().numpy())
del A, truth, X
torch.cuda.synchronize()
cfg = SolverConfig(max_iters=iters)
o = sb.solve(cfg)  # warm-up
sb.check_status()
s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s_.record()
o = sb.solve(cfg)
e_.record()
torch.cuda.synchronize()
sb.check_status()
ms = s_.elapsed_time(e_)
pc = o["phase_cycles"].cpu().numpy().sum(axis=0)
names = ["select+copy", "rand-destroy", "worst-destroy", "repair", "one_opt", "find_candidates", "swap_eval", "accept"]
mv = int(o["moves_scored"][:, 0].sum().item())
print(json.dumps({
    "config": f"C3 slices {side}^2 x {n_ang} angles", "m": m, "n": n, "nnz": int(indptr[-1]), "slices": S,
    "iters": iters, "device_ms": round(ms, 2), "slice_iters_per_s": S * iters / (ms / 1e3),
    "moves_scored_per_s": mv / (ms / 1e3),
    "initial_obj_mean": float(o["initial_objective"].mean()), "best_obj_mean": float(o["best_objective"].mean()),
    "phase_share": {k: round(float(v / pc[:8].sum()), 3) for k, v in zip(names, pc[:8])},
    "events_per_slice": {k: round(float(v / S), 1) for k, v in zip(
        ["fc_calls", "fc_survivors", "swaps", "oo_exact_scans", "oo_moves", "oo_windows", "impact_calls",
         "refreshes"], pc[8:16])},
    "front_end_s": {"projector_csr": round(t1 - t0, 2), "device_build_sirt": round(t2 - t1, 2)}}))
