"""C3 slices on the sparse engine (tomo.SparseSliceBatch): device front end
(projector CSR, projections, SIRT start), one batched amvm_solve_sparse.
usage: python tools/c3_sparse.py SIDE N_ANGLES SLICES ITERS [SIRT_ITERS] [--dense]"""
import json
import os
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402

side, n_ang, S, iters = (int(v) for v in sys.argv[1:5])
sirt = int(sys.argv[5]) if len(sys.argv) > 5 and not sys.argv[5].startswith("--") else 100
dense = "--dense" in sys.argv
dev = torch.device("cuda")
m, n = n_ang * side, side * side
t0 = time.perf_counter()
csr = tomo.projection_csr_device(side, n_ang, dev)
rows = torch.repeat_interleave(torch.arange(m, device=dev), csr[0][1:] - csr[0][:-1])
eta = 0.05 * float(torch.zeros(m, dtype=torch.float64, device=dev).index_add_(0, rows, csr[2]).max())
fe = tomo.build_tomo_device(side, (0.0, 1.0, 2.0), n_ang, eta, seeds=tuple(range(S)),
                            phantom_kinds=("squares", "disk", "checker"), sirt_iters=sirt, device=dev)
if dense:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        A = torch.sparse_csr_tensor(*fe["csr"], size=(m, n), dtype=torch.float64).to_dense()
    sb = tomo.SliceBatch(A, fe["B"].cpu().numpy(), fe["levels"], fe["idx0"].cpu().numpy())
    del A
else:
    sb = tomo.SparseSliceBatch(fe["csr"], m, n, fe["B"], fe["levels"], fe["idx0"])
torch.cuda.synchronize()
t1 = time.perf_counter()
cfg = SolverConfig(max_iters=iters)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.reset_peak_memory_stats()
a.record()
o = sb.solve(cfg, seeds=np.arange(S))
b.record()
torch.cuda.synchronize()
sb.check_status()
ms = a.elapsed_time(b)
pc = o["phase_cycles"].cpu().numpy().sum(axis=0)
names = ["select+copy", "rand-destroy", "worst-destroy", "repair", "one_opt", "find_candidates", "swap_eval", "accept"]
print(json.dumps({"engine": "dense" if dense else "sparse", "config": f"{side}^2 x {n_ang}", "m": m, "n": n,
                  "nnz": int(csr[2].numel()), "slices": S, "iters": iters, "device_ms": round(ms, 1),
                  "slice_iters_per_s": S * iters / (ms / 1e3),
                  "moves_per_s": float(o["moves_scored"][:, 0].sum()) / (ms / 1e3),
                  "peak_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                  "workspace_GB": round((sb.workspace_bytes(cfg) if not dense else 0) / 1e9, 2),
                  "setup_s": round(t1 - t0, 2),
                  "best_mean": float(o["best_objective"].mean()), "init_mean": float(o["initial_objective"].mean()),
                  "phase_share": {k: round(float(v / pc[:8].sum()), 3) for k, v in zip(names, pc[:8])},
                  "events_per_slice_it": {k: round(float(v / S / iters), 1) for k, v in zip(
                      ["fc_calls", "fc_survivors", "swaps", "oo_exact", "oo_moves", "oo_windows", "impact",
                       "refresh"], pc[8:16])}}), flush=True)
