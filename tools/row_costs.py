"""Per-row cost distribution of the C5 bench batch (load-balance diagnostics).

usage: python tools/row_costs.py ROWS ITERS [ITERS ...]
"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2508_13437_b200 import ptq, SolverConfig
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1792
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((rows, 4096)) * 0.02
lb = ptq.LayerBatch(X, W)
lb.prepare()
for iters in [int(v) for v in sys.argv[2:]] or [2]:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); o = lb.solve(SolverConfig(max_iters=iters)); e.record(); torch.cuda.synchronize()
    pc = o["phase_cycles"].cpu().numpy()
    c = pc[:, :8].sum(axis=1) / 1.965e6  # ms at 1965 MHz
    mv = o["moves_scored"][:, 0].sum().item()
    print(f"iters {iters}: {s.elapsed_time(e):.1f} ms (ideal {c.sum() / 296:.1f}); per-row ms mean {c.mean():.2f} "
          f"p50 {np.median(c):.2f} p99 {np.percentile(c, 99):.2f} max {c.max():.2f}; moves/row {mv / rows:.3g}; "
          f"fc calls/row {pc[:, 8].mean():.1f}", flush=True)
