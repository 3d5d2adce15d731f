"""Per-row cost distribution of the C5 bench batch (load-balance diagnostics)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2508_13437_b200 import ptq, SolverConfig
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((rows, 4096)) * 0.02
lb = ptq.LayerBatch(X, W)
lb.prepare()
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); o = lb.solve(SolverConfig(max_iters=iters)); e.record(); torch.cuda.synchronize()
    pc = o["phase_cycles"].cpu().numpy()
    c = pc[:, :8].sum(axis=1) / 1.965e6  # ms at 1965 MHz
    print(f"rep {rep}: {s.elapsed_time(e):.1f} ms; per-row ms mean {c.mean():.2f} p50 {np.median(c):.2f} p90 {np.percentile(c, 90):.2f} "
          f"p99 {np.percentile(c, 99):.2f} max {c.max():.2f}; ideal {c.sum() / 296:.1f} ms; fc calls max {pc[:, 8].max()} mean {pc[:, 8].mean():.1f}")
    top = np.argsort(-c)[:8]
    print("  slowest rows", top.tolist(), np.round(c[top], 1).tolist(), "fc calls", pc[top, 8].tolist())
