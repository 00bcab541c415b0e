"""The benchmark's synthetic problem (bench.make_problem) must be the SAME matrix
and right-hand side for any GPU count (strong scaling compares equal work):
rows generated per global chunk, the Gram / norm reductions through
torch.distributed.  Checked here on CPU with world sizes 2 and 3 (gloo)
against the single-rank result."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M, N, COND, RHO = 9_000, 12, 1e6, 0.5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bounds(world):
    return [M * k // world for k in range(world + 1)]


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = _bounds(world)
    Abuf, ld, xs = bench.make_problem(torch, M, N, COND, RHO, b[rank], b[rank + 1], torch.device("cpu"), dist,
                                      chunk=1000)
    np.save(os.path.join(out_dir, f"A{rank}.npy"), Abuf.numpy())
    np.save(os.path.join(out_dir, f"x{rank}.npy"), xs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_make_problem_partition_independent(world, tmp_path):
    sys.path.insert(0, ROOT)
    import bench

    A1, ld, x1 = bench.make_problem(torch, M, N, COND, RHO, 0, M, torch.device("cpu"), None, chunk=1000)
    A1 = A1.numpy()
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"A{r}.npy") for r in range(world)]
    Aw = np.concatenate(parts, axis=0)
    assert Aw.shape == A1.shape
    # the reductions are summed in a different grouping across ranks: equal to rounding
    scale = np.abs(A1).max()
    assert np.abs(Aw - A1).max() <= 1e-12 * scale
    for r in range(world):
        assert np.allclose(np.load(tmp_path / f"x{r}.npy"), x1, rtol=1e-12, atol=0)
    # the matrix the bench claims: cond(A) = COND, ||b|| = 1, ||b - A x*|| = RHO
    A, bb = A1[:, :N], A1[:, N]
    s = np.linalg.svd(A, compute_uv=False)
    assert abs(s[0] / s[-1] / COND - 1) < 1e-6
    assert abs(np.linalg.norm(bb) - 1) < 1e-12
    assert abs(np.linalg.norm(bb - A @ x1) - RHO) < 1e-10
