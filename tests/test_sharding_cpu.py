"""Multi-instance sharding across ranks on CPU with gloo:
contiguous shards, the per-rank report assembly and the single end-of-solve
gather, for both sharded workloads (PTQ layer rows, tomography slices).

There is no GPU here, so each rank solves its shard with the CPU oracle
(test infrastructure; bit-identical trajectories to the device path) and
hands the results, in the device result layout, to the SAME report
assembly (ptq.layer_report / tomo.slice_report) and gather
(ptq.gather_layer / tomo.gather_slices) the GPU path uses.  The gathered
reports must equal a single-process solve of every instance."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------ PTQ rows
D, CALIB, ITERS = 24, 40, 6


def _layer():
    X = np.random.default_rng(0).standard_normal((CALIB, D))
    W = np.random.default_rng(1).standard_normal((11, D)) * 0.02
    return X, W


def _oracle_rows(rows):
    """The oracle solving PTQ rows `rows` exactly as ptq.LayerBatch sets them
    up (builders.py:355-372: linspace grid, nearest-level start, seed = row)."""
    from oracle import oracle as O

    X, W = _layer()
    L, B, I0, R0, OB = [], [], [], [], []
    for r in rows:
        w = W[r]
        lv = np.linspace(w.min(), w.max(), 16)
        b = X @ w
        idx = np.argmin(np.abs(w[:, None] - lv[None, :]), axis=1)
        res = X @ lv[idx] - b
        L.append(lv); B.append(b); I0.append(idx); R0.append(res); OB.append(float(np.max(np.abs(res))))
    if not len(rows):
        return {"best_idx": np.zeros((0, D), np.int32), "best_objective": np.zeros(0),
                "initial_objective": np.zeros(0), "iterations": np.zeros(0, np.int32),
                "moves_scored": np.zeros((0, 2), np.int64)}, np.zeros((0, 16))
    prm = O.make_params(D, max_iters=ITERS)
    out = O.solve(X, np.stack(B), np.stack(L), np.stack(I0), np.stack(R0), np.array(OB), np.zeros(len(rows)), prm,
                  [O.pcg_from_seed(int(r)) for r in rows])
    return out, np.stack(L)


def _ptq_worker(rank, world, port, total, out):
    import torch.distributed as dist

    from paper_2508_13437_b200 import ptq

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = ptq.shard_rows(total, rank, world)
    host, levels = _oracle_rows(rows)
    full = ptq.gather_layer(ptq.layer_report(rows, host, levels), total)
    if rank == 0:
        np.savez(out, rows=full.rows, codes=full.codes, levels=full.levels, objective=full.objective,
                 initial=full.initial_objective, iterations=full.iterations, moves=full.moves_scored)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(11, 2), (8, 2), (3, 3)])
def test_layer_shards_gather_to_the_single_process_solve(tmp_path, total, world):
    import torch.multiprocessing as mp

    from paper_2508_13437_b200 import ptq

    out = str(tmp_path / "g.npz")
    mp.spawn(_ptq_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    z = np.load(out)
    host, levels = _oracle_rows(np.arange(total))
    want = ptq.layer_report(np.arange(total), host, levels)
    np.testing.assert_array_equal(z["rows"], np.arange(total))
    np.testing.assert_array_equal(z["codes"], want.codes)
    np.testing.assert_array_equal(z["levels"], want.levels)
    np.testing.assert_array_equal(z["objective"], want.objective)
    np.testing.assert_array_equal(z["initial"], want.initial_objective)
    np.testing.assert_array_equal(z["iterations"], want.iterations)
    np.testing.assert_array_equal(z["moves"], want.moves_scored)


# ------------------------------------------------------ tomography slices
SIDE, ANGLES, LV = 8, 6, np.array([0.0, 1.0, 2.0])
KINDS = ("squares", "disk", "checker")


def _oracle_slices(slices):
    """The oracle solving tomography slices (shared projector, the package's
    host projector = the reference's parallel_beam_matrix bit for bit;
    slice k: phantom KINDS[k % 3], noise seed k, ALNS seed k)."""
    from oracle import oracle as O
    from paper_2508_13437_b200 import tomo

    A = tomo.projection_matrix(SIDE, ANGLES)
    m, n = A.shape
    B, I0, R0, OB = [], [], [], []
    for k in slices:
        truth = LV[np.minimum(tomo.phantom(KINDS[k % 3], SIDE), 2)].ravel()
        b = A @ truth + np.random.default_rng(int(k)).uniform(-0.05, 0.05, m)
        idx = np.argmin(np.abs((0.6 * truth)[:, None] - LV[None, :]), axis=1)
        res = A @ LV[idx] - b
        B.append(b); I0.append(idx); R0.append(res); OB.append(float(np.max(np.abs(res))))
    if not len(slices):
        return {"best_idx": np.zeros((0, n), np.int32), "best_objective": np.zeros(0),
                "initial_objective": np.zeros(0), "iterations": np.zeros(0, np.int32),
                "moves_scored": np.zeros((0, 2), np.int64)}
    prm = O.make_params(n, max_iters=ITERS, destroy_rate=0.05)
    return O.solve(A, np.stack(B), np.tile(LV, (len(slices), 1)), np.stack(I0), np.stack(R0), np.array(OB),
                   np.zeros(len(slices)), prm, [O.pcg_from_seed(int(k)) for k in slices])


def _tomo_worker(rank, world, port, total, out):
    import torch.distributed as dist

    from paper_2508_13437_b200 import shard, tomo

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    slices = shard.shard_rows(total, rank, world)
    full = tomo.gather_slices(tomo.slice_report(slices, _oracle_slices(slices)), total)
    if rank == 0:
        np.savez(out, slices=full.slices, codes=full.codes, objective=full.objective,
                 initial=full.initial_objective, iterations=full.iterations, moves=full.moves_scored)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(5, 2), (4, 2), (2, 3)])
def test_tomography_slice_shards_gather_to_the_single_process_solve(tmp_path, total, world):
    import torch.multiprocessing as mp

    from paper_2508_13437_b200 import tomo

    out = str(tmp_path / "t.npz")
    mp.spawn(_tomo_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    z = np.load(out)
    want = tomo.slice_report(np.arange(total), _oracle_slices(np.arange(total)))
    np.testing.assert_array_equal(z["slices"], np.arange(total))
    np.testing.assert_array_equal(z["codes"], want.codes)
    np.testing.assert_array_equal(z["objective"], want.objective)
    np.testing.assert_array_equal(z["initial"], want.initial_objective)
    np.testing.assert_array_equal(z["iterations"], want.iterations)
    np.testing.assert_array_equal(z["moves"], want.moves_scored)
    assert (z["objective"] <= z["initial"]).all()


def test_shard_rows_partition():
    from paper_2508_13437_b200 import ptq, shard

    for total in (1, 7, 14336):
        for world in (1, 2, 4, 8):
            parts = [shard.shard_rows(total, r, world) for r in range(world)]
            np.testing.assert_array_equal(np.concatenate(parts), np.arange(total))
            sizes = [p.size for p in parts]
            assert max(sizes) - min(sizes) <= 1
            np.testing.assert_array_equal(ptq.shard_rows(total, 0, world), parts[0])
