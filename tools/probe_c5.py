import time, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2508_13437_b200 import ptq, SolverConfig
rng = np.random.default_rng(0)
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((1184, 4096)) * 0.02
for rows, iters in [(148, 2), (148, 10), (1184, 2)]:
    lb = ptq.LayerBatch(X, W[:rows])
    torch.cuda.synchronize(); t0 = time.perf_counter(); lb.prepare(); torch.cuda.synchronize(); t1 = time.perf_counter()
    o = lb.solve(SolverConfig(max_iters=iters)); lb.check_status(); t2 = time.perf_counter()
    mv = o["moves_scored"].cpu().numpy(); it = o["iterations"].cpu().numpy()
    pc = o["phase_cycles"].cpu().numpy().sum(axis=0); names = ["select+copy","rand-destroy","worst-destroy","repair","one_opt","find_cand","swap_eval","accept"]
    print("  phases %:", {nm: round(100*v/pc[:8].sum(),1) for nm, v in zip(names, pc[:8])}, "total Gcycles", pc[:8].sum()/1e9, flush=True)
    ev = ["fc_calls","fc_survivors","swaps","oo_rechecks","oo_moves","oo_windows","impact_calls","refreshes"]
    print("  events per row-iter", {k: round(v/rows/iters, 1) for k, v in zip(ev, pc[8:])}, flush=True)
    print(f"rows {rows} iters {iters}: prepare {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, moves ref {mv[:,0].sum()} raw {mv[:,1].sum()}, "
          f"ref moves/s {mv[:,0].sum()/(t2-t1):.3e}, iters {it.min()}-{it.max()}, obj0 {o['initial_objective'][:3].cpu().numpy()} best {o['best_objective'][:3].cpu().numpy()}", flush=True)
