"""find_candidates work counters (needs a -DAMVM_FC_STATS build via AMVM_LIBRARY)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2508_13437_b200 import ptq, SolverConfig
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 296
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((rows, 4096)) * 0.02
lb = ptq.LayerBatch(X, W)
lb.prepare()
o = lb.solve(SolverConfig(max_iters=iters)); lb.check_status()
pc = o["phase_cycles"].cpu().numpy().sum(axis=0)
calls = pc[8]
print("fc_calls/row", calls / rows, "survivors/call", pc[9] / calls)
print("warp-positions/call", pc[14] / calls, "useful pair-lanes/call", pc[15] / calls,
      "lane efficiency", pc[15] / (32 * pc[14]))
print("queued pairs/call", pc[11] / calls, "after row passes/call", pc[12] / calls)
