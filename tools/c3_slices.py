"""C3 family throughput: S tomography slices sharing one projector, one
device batch (tomo.SliceBatch).  Front end on the device through libamvm
(tomo.build_tomo_device: projector CSR, noisy projections, clamped SIRT warm
start); the ALNS path is libamvm.  Prints one JSON line.

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
m, n = n_ang * side, side * side
lv = np.array([0.0, 1.0, 2.0])
kinds = ("squares", "disk", "checker")
# eta = 5% of the max row sum (make_golden.py), from the device projector
csr = tomo.projection_csr_device(side, n_ang, dev)
rows = torch.repeat_interleave(torch.arange(m, device=dev), csr[0][1:] - csr[0][:-1])
eta = 0.05 * float(torch.zeros(m, dtype=torch.float64, device=dev).index_add_(0, rows, csr[2]).max())
torch.cuda.synchronize()
t1 = time.perf_counter()
# build_tomo (builders.py:306-327) for S slices on the device: projector,
# noisy projections (bitwise), clamped SIRT, rounded start
fe = tomo.build_tomo_device(side, lv, n_ang, eta, seeds=tuple(range(S)), phantom_kinds=kinds,
                            sirt_iters=sirt_iters, device=dev)
torch.cuda.synchronize()
t2 = time.perf_counter()
indptr = fe["csr"][0].cpu().numpy()
import warnings  # noqa: E402
warnings.filterwarnings("ignore", message="Sparse CSR tensor support is in beta")
A = torch.sparse_csr_tensor(*fe["csr"], size=(m, n), dtype=torch.float64).to_dense()
Bm, idx0 = fe["B"], fe["idx0"]
sb = tomo.SliceBatch(A, Bm.cpu().numpy(), lv, idx0.cpu().numpy())
del A, fe
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
    "front_end_s": {"projector_csr_eta": round(t1 - t0, 2),
                    f"build_tomo_device (projector, projections, {sirt_iters} SIRT iterations)": round(t2 - t1, 2)}}))
