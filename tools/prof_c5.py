"""Short C5-row run for ncu (one amvm_solve launch)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2508_13437_b200 import ptq, SolverConfig
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 148
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((rows, 4096)) * 0.02
lb = ptq.LayerBatch(X, W)
lb.prepare()
o = lb.solve(SolverConfig(max_iters=iters)); lb.check_status()
pc = o["phase_cycles"].cpu().numpy().sum(axis=0)
names = ["select+copy","rand-destroy","worst-destroy","repair","one_opt","find_cand","swap_eval","accept"]
print("phase Gcycles", {k: round(v/1e9, 2) for k, v in zip(names, pc[:8])})
ev = ["fc_calls","fc_survivors","swaps","oo_rechecks","oo_moves","oo_windows","impact_calls","refreshes"]
print("events per row", {k: round(v/rows, 1) for k, v in zip(ev, pc[8:])}, "moves", o["moves_scored"].cpu().numpy().sum(axis=0))
