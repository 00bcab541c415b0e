"""Multi-process (world_size 2 and 7, gloo, CPU) test of the row-partitioned path's
host logic -- the same decomposition the NCCL path runs on B200s:

  * rows partitioned by partition_rows (distsim.hpp:31-42, via the C-ABI);
  * each rank generates ONLY its sketch columns, keyed by global row id
    (distsim.hpp:346-361), applies them to its rows, and one sum-reduction of
    the d x (n+1) partials gives S [A b] (distsim.hpp:383-409);
  * QR / M / x0 on rank 0, broadcast (status first);
  * LSQR with ONE allreduce of n+1 doubles per iteration (distsim.hpp:312-331),
    in the device algorithm's algebra: u is never rescaled in memory (u_true =
    su * u_hat folded into the next pass's coefficient), M v computed once.

Per-rank arithmetic uses the CPU oracle; the collectives are torch.distributed
(gloo).  Results must match the serial oracle (test_distsim.cpp:151-255 bars).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _bcast(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    dist.broadcast(t, 0)
    return t.numpy()


def device_algorithm_lsqr(Ak, bk, M, x0, maxit, counter):
    """Mirror of csrc/lsqr.cu (fused pass + reduce + mtz + mv_update)."""
    n = M.shape[1]
    # init pass: u_hat = A x0 - b, z = A^T u_hat, ||u_hat||^2  (1 allreduce)
    uh = Ak @ x0 - bk
    red = _allreduce(np.concatenate([Ak.T @ uh, [uh @ uh]]))
    counter[0] += 1
    beta1 = np.sqrt(red[n])
    vhat = M.T @ (red[:n] * (-1.0 / beta1))
    alpha = np.linalg.norm(vhat)
    v = vhat * (1.0 / alpha)
    p = M @ v
    w = p.copy()
    x = x0.copy()
    phi_bar, rho_bar = beta1, alpha
    c = -alpha * (-1.0 / beta1)
    hist = []
    for _ in range(maxit):
        uh = Ak @ p + c * uh
        red = _allreduce(np.concatenate([Ak.T @ uh, [uh @ uh]]))
        counter[0] += 1
        beta = np.sqrt(red[n])
        vhat = M.T @ (red[:n] * (1.0 / beta)) + (-beta) * v
        alpha_n = np.linalg.norm(vhat)
        rho = np.hypot(rho_bar, beta)
        cs, sn = rho_bar / rho, beta / rho
        theta = sn * alpha_n
        rho_bar = -cs * alpha_n
        phi = cs * phi_bar
        phi_bar = sn * phi_bar
        v = vhat * (1.0 / alpha_n)
        p = M @ v
        x = x + (phi / rho) * w
        w = p + (-theta / rho) * w
        c = -alpha_n * (1.0 / beta)
        hist.append(phi_bar)
    return x, hist


def device_algorithm_hbm(Ak, bk, M, x0, alpha, beta, maxit, counter):
    """Mirror of gd_dev (csrc/lsqr.cu): one pass per iteration gives
    u_hat = A x - b and z = A^T u_hat (one allreduce of n values)."""
    x, xp = x0.copy(), x0.copy()
    hist = []
    for _ in range(maxit):
        uh = Ak @ x - bk
        z = _allreduce(Ak.T @ uh)
        counter[0] += 1
        h = M.T @ (-z)
        hist.append(np.linalg.norm(h))
        g = M @ h
        xn = x * (1.0 + beta) + (-beta) * xp + alpha * g
        xp, x = x, xn
    return x, hist


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2506_03070_b200 as slq

        C = oracle.C()
        m, n, d, zeta, seed = 600, 24, 192, 6, 93
        A = C.gen_dense(m, n, 50.0, 91)
        b, _ = C.gen_rhs(A, 0.5, 92)
        part = slq.partition_rows(m, world)
        r0, r1 = part.begin(rank), part.end(rank)
        Ak, bk = np.asfortranarray(A[r0:r1]), b[r0:r1].copy()

        # sketch: local columns keyed by global row id, one reduction
        rows, vals, colptr, _ = C.generate_sparse_sign(d, r1 - r0, zeta, seed, col_begin=r0)
        Yk = C.spmm(d, rows, vals, colptr, Ak)
        Sbk = C.csc_matvec(d, rows, vals, colptr, bk)
        tot = _allreduce(np.concatenate([Yk.ravel(order="F"), Sbk]))
        Y = tot[: d * n].reshape((d, n), order="F")
        Sb = tot[d * n:]

        # preconditioner on rank 0, status then M / x0 broadcast
        if rank == 0:
            M, Q = C.build_preconditioner(Y)
            x0 = C.initial_guess(M, Q, Sb)
            status = np.zeros(1)
        else:
            M, x0, status = np.zeros((n, n)), np.zeros(n), np.zeros(1)
        status = _bcast(status)
        assert status[0] == 0
        M = _bcast(np.asfortranarray(M).ravel(order="F")).reshape((n, n), order="F")
        x0 = _bcast(x0)

        counter = [0]
        x, hist = device_algorithm_lsqr(Ak, bk, M, x0, 10, counter)
        gcount = [0]
        alpha, beta = C.gradient_params(float(np.sqrt(n / d)), True)
        xg, ghist = device_algorithm_hbm(Ak, bk, M, x0, alpha, beta, 12, gcount)
        results[rank] = {"Y": Y, "Sb": Sb, "x": x, "hist": np.array(hist), "allreduces": counter[0],
                         "M": M, "x0": x0, "xg": xg, "ghist": np.array(ghist), "g_allreduces": gcount[0]}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 7])  # 7: 600 rows -> 6 blocks of 85 + a last block of 90 (partition_rows)
def test_row_partitioned_pipeline_gloo(world):
    import oracle

    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    C = oracle.C()
    m, n, d, zeta, seed = 600, 24, 192, 6, 93
    A = C.gen_dense(m, n, 50.0, 91)
    b, _ = C.gen_rhs(A, 0.5, 92)
    Ys, Sbs = C.sketch_apply(d, zeta, seed, A, b)
    M, Q = C.build_preconditioner(Ys)
    x0 = C.initial_guess(M, Q, Sbs)
    xs, rep = C.lsqr(A, M, b, x0, eps=0.0, maxit=10, one_sync=True)
    for r in range(world):
        res = results[r]
        # partial sums in a different order: test_distsim.cpp:169 bar
        assert np.abs(res["Y"] - Ys).max() <= 1e-12 * max(1.0, np.abs(Ys).max())
        assert np.abs(res["Sb"] - Sbs).max() <= 1e-12 * max(1.0, np.abs(Sbs).max())
        assert np.linalg.norm(res["x"] - xs) <= 1e-8 * max(1.0, np.linalg.norm(xs))  # test_distsim.cpp:243
        assert np.allclose(res["hist"], rep.residual_estimate, rtol=1e-8)
        # one reduction per iteration + one at init (the reference's one-sync count)
        assert res["allreduces"] == 10 + 1
    # heavy ball over the same decomposition: one allreduce per iteration
    # (the reference's dist HBM counts one reduction per iteration, test_distsim.cpp:282)
    a, bb = C.gradient_params(float(np.sqrt(n / d)), True)
    xgs, greps = C.gd_hbm(A, M, b, x0, a, bb, eps=0.0, maxit=12)
    for r in range(world):
        res = results[r]
        assert np.linalg.norm(res["xg"] - xgs) <= 1e-10 * max(1.0, np.linalg.norm(xgs))
        assert np.allclose(res["ghist"], greps.residual_estimate, rtol=1e-9)
        assert res["g_allreduces"] == 12
    # replicated state is bitwise identical on every rank (allreduce/broadcast semantics)
    for r in range(1, world):
        assert np.array_equal(results[0]["xg"], results[r]["xg"])
        assert np.array_equal(results[0]["x"], results[r]["x"])
        assert np.array_equal(results[0]["M"], results[r]["M"])
