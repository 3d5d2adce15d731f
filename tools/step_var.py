"""Step-time variance diagnostics for the C5 bench batch: per launch, device
time vs the busy-cycle ideal, and the finish-time spread of the CTAs."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2508_13437_b200 import ptq, SolverConfig
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1792
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((rows, 4096)) * 0.02
lb = ptq.LayerBatch(X, W)
lb.prepare()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for r in range(reps):
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); o = lb.solve(SolverConfig(max_iters=iters)); e.record(); torch.cuda.synchronize()
    pc = o["phase_cycles"].cpu().numpy()
    busy = pc[:, :8].sum() / 296 / 1.965e6
    print(f"rep {r}: {s.elapsed_time(e):.1f} ms, busy-ideal {busy:.1f} ms", flush=True)
