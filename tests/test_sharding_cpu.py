"""Multi-instance sharding across ranks on CPU with gloo,
world_size 2: contiguous row shards and the single end-of-solve all_gather."""

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


def _fake_report(rows, n=12, nlev=16):
    from paper_2508_13437_b200.ptq import LayerReport

    k = rows.size
    return LayerReport(
        rows=rows, codes=((rows[:, None] * 7 + np.arange(n)[None, :]) % nlev).astype(np.int8),
        levels=np.stack([np.linspace(-r, r + 1, nlev) for r in rows]) if k else np.zeros((0, nlev)),
        objective=rows * 0.5 + 0.25, initial_objective=rows + 1.0, iterations=rows % 5 + 1,
        moves_scored=np.stack([rows * 3, rows * 4], axis=1) if k else np.zeros((0, 2), np.int64))


def _worker(rank, world, port, total, out):
    import torch.distributed as dist

    from paper_2508_13437_b200 import ptq

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = ptq.shard_rows(total, rank, world)
    full = ptq.gather_layer(_fake_report(rows), total)
    if rank == 0:
        np.savez(out, rows=full.rows, codes=full.codes, levels=full.levels, objective=full.objective,
                 iterations=full.iterations, moves=full.moves_scored)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(11, 2), (8, 2), (3, 3)])
def test_gather_layer_reassembles_every_row(tmp_path, total, world):
    import torch.multiprocessing as mp

    out = str(tmp_path / "g.npz")
    mp.spawn(_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    z = np.load(out)
    want = _fake_report(np.arange(total))
    np.testing.assert_array_equal(z["rows"], np.arange(total))
    np.testing.assert_array_equal(z["codes"], want.codes)
    np.testing.assert_array_equal(z["levels"], want.levels)
    np.testing.assert_array_equal(z["objective"], want.objective)
    np.testing.assert_array_equal(z["iterations"], want.iterations)
    np.testing.assert_array_equal(z["moves"], want.moves_scored)


def test_shard_rows_partition():
    from paper_2508_13437_b200 import ptq

    for total in (1, 7, 14336):
        for world in (1, 2, 4, 8):
            parts = [ptq.shard_rows(total, r, world) for r in range(world)]
            np.testing.assert_array_equal(np.concatenate(parts), np.arange(total))
            sizes = [p.size for p in parts]
            assert max(sizes) - min(sizes) <= 1
