"""Benchmark: end-to-end sketch-and-precondition LSQ solve on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

Workload (BASELINE.json configs[2], the metric's headline config, fits one
B200): dense A m=4,000,000 x n=1000, cond(A)=1e8 (singular values log-spaced
in [1e-8, 1], A = U diag(s) V^T with U, V orthonormal, problems.hpp:45-66),
b with ||b|| = 1 and ||b - A x*|| = 0.5 (x* the LS solution), sparse-sign
sketch d = 4n, zeta = 8, LSQR to relative backward error
||A^T r|| / (||A|| ||r||) <= 1e-10 (T iterations, calibrated in warm-up and
verified after the timed steps).  A is row-partitioned over N GPUs
(partition_rows, distsim.hpp:31-42); strong scaling (total work fixed).

A "step" is one full solve (sketch generation + S[A b] + reduce + QR / R^-1 /
x0 + T LSQR iterations) with A resident in HBM.  `value` = seconds per solve
(max over ranks, CUDA events); `e2e` = the same solve through the C-ABI from
pinned HOST buffers (column-major A, as the reference's DenseMatrix), H2D and
layout conversion inside the timed region.

`cpu_baseline` / `--impl reference`: the reference itself (oracle/_ref, the
unmodified sketchlsq headers compiled -O3 -march=native) on the SAME A and b
bytes, full size, all T iterations, on every host thread -- not
extrapolated.  `parity_vs_reference` compares the two solutions in
backward-error / residual space.
"""
from __future__ import annotations

import argparse
import ctypes as ct
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LSQ solve time (s) & LSQR GB/s vs HBM peak, 4M×1000 cond1e8, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=4_000_000)
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--cond", type=float, default=1e8)
    ap.add_argument("--dfac", type=int, default=4)
    ap.add_argument("--zeta", type=int, default=8)
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--iters", type=int, default=0, help="LSQR iterations (0 = calibrate to eta <= 1e-10)")
    ap.add_argument("--eta", type=float, default=1e-10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="seconds of full-size reference solves per run (at least one)")
    ap.add_argument("--config", default="c3", choices=["c3", "c4"],
                    help="c3: dense 4M x 1000 cond 1e8 (headline); c4: sparse CSR 2^24 x 2000, 50 nnz/row, cond 1e6")
    return ap.parse_args()


# ------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm = float(s[1])
                mx = float(s[2])
                pw = float(s[3])
            except Exception:
                continue
            if pw > 200:  # under load
                sms.append(sm)
            for k, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(k)
        if not sms:
            sms = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------ problem

def make_problem(torch, m, n, cond, rho, row_begin, row_end, dev, dist=None, seed=1, chunk=4000):
    """A = U diag(s) V^T (U: CholeskyQR2 of a Gaussian, row-keyed chunks so
    the matrix is identical for any row partition), b = A w s + rho r_perp.
    Returns the device buffer in the solver layout (row-major [A | b | 0],
    ld = round_up(n+1, 4)) and x_star."""
    f64 = torch.float64
    ml = row_end - row_begin
    ld = ((n + 1 + 3) // 4) * 4

    def allreduce(t):
        if dist is not None:
            dist.all_reduce(t)
        return t

    def gauss_rows(r0, r1):
        # rows [r0, r1) of G, generated per global chunk (partition independent)
        out = torch.empty((r1 - r0, n), dtype=f64, device=dev)
        c0, c1 = r0 // chunk, (r1 - 1) // chunk
        for c in range(c0, c1 + 1):
            g = torch.Generator(device=dev)
            g.manual_seed(seed * 1_000_003 + c)
            blk = torch.randn((chunk, n), dtype=f64, device=dev, generator=g)
            a, b = max(r0, c * chunk), min(r1, (c + 1) * chunk)
            out[a - r0:b - r0] = blk[a - c * chunk:b - c * chunk]
        return out

    step = 256_000
    gram = torch.zeros((n, n), dtype=f64, device=dev)
    for r in range(row_begin, row_end, step):
        G = gauss_rows(r, min(row_end, r + step))
        gram += G.T @ G
    allreduce(gram)
    R1 = torch.linalg.cholesky(gram).T
    U = torch.empty((ml, n), dtype=f64, device=dev)
    gram2 = torch.zeros((n, n), dtype=f64, device=dev)
    for r in range(row_begin, row_end, step):
        r1 = min(row_end, r + step)
        Uc = torch.linalg.solve_triangular(R1, gauss_rows(r, r1), upper=True, left=False)
        U[r - row_begin:r1 - row_begin] = Uc
        gram2 += Uc.T @ Uc
    allreduce(gram2)
    R2 = torch.linalg.cholesky(gram2).T
    for r in range(0, ml, step):
        U[r:r + step] = torch.linalg.solve_triangular(R2, U[r:r + step], upper=True, left=False)
    gV = torch.Generator(device=dev)
    gV.manual_seed(seed * 7 + 1)
    V, _ = torch.linalg.qr(torch.randn((n, n), dtype=f64, device=dev, generator=gV))
    s = torch.pow(10.0, -math.log10(cond) * torch.arange(n, dtype=f64, device=dev) / max(n - 1, 1))
    B = (s[:, None] * V.T).contiguous()  # diag(s) V^T
    Abuf = torch.zeros((ml, ld), dtype=f64, device=dev)
    for r in range(0, ml, step):
        Abuf[r:r + step, :n] = U[r:r + step] @ B
    # right-hand side (problems.hpp:137-167 semantics, stable projection with U)
    gw = torch.Generator(device=dev)
    gw.manual_seed(seed * 11 + 2)
    w = torch.rand(n, dtype=f64, device=dev, generator=gw) * 2 - 1
    p = torch.empty(ml, dtype=f64, device=dev)
    for r in range(0, ml, step):
        p[r:r + step] = Abuf[r:r + step, :n] @ w
    pn2 = allreduce((p * p).sum().reshape(1))
    pn = float(pn2.sqrt())
    # residual direction, drawn per GLOBAL chunk (like G) so b is the same for any row partition
    z = torch.empty(ml, dtype=f64, device=dev)
    for c in range(row_begin // chunk, (row_end - 1) // chunk + 1):
        g = torch.Generator(device=dev)
        g.manual_seed(seed * 13 + 3 + c)
        blk = torch.rand(chunk, dtype=f64, device=dev, generator=g) * 2 - 1
        a, b_ = max(row_begin, c * chunk), min(row_end, (c + 1) * chunk)
        z[a - row_begin:b_ - row_begin] = blk[a - c * chunk:b_ - c * chunk]
    for _ in range(2):
        c = allreduce(U.T @ z)
        z -= U @ c
    zn = float(allreduce((z * z).sum().reshape(1)).sqrt())
    range_norm = math.sqrt(1.0 - rho * rho)
    Abuf[:, n] = p * (range_norm / pn) + z * (rho / zn)
    x_star = (w * (range_norm / pn)).cpu().numpy()
    del U, z, p
    if dev.type == "cuda":
        torch.cuda.synchronize()
    return Abuf, ld, x_star


# ------------------------------------------------------------ reference (CPU)

def cpu_info():
    """Host CPU model, logical CPUs and NUMA layout (recorded with every CPU timing)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        fam = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith(("cpu family", "model\t"))][:2]
        model += f" (family {fam[0]} model {fam[1]})" if len(fam) == 2 else ""
    except Exception:
        pass
    numa = []
    try:
        base = "/sys/devices/system/node"
        for nd in sorted(x for x in os.listdir(base) if x.startswith("node") and x[4:].isdigit()):
            numa.append({"node": int(nd[4:]), "cpus": open(os.path.join(base, nd, "cpulist")).read().strip()})
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count(), "numa": numa}


def host_copy(torch, Abuf, n, ml, pinned=True):
    """Column-major host copy of the device block's A (an (n, ml) row-major
    tensor == column-major A) and b, filled in 256K-row slabs."""
    Ah = torch.empty((n, ml), dtype=torch.float64, pin_memory=pinned)
    bh = torch.empty(ml, dtype=torch.float64, pin_memory=pinned)
    for r in range(0, ml, 256_000):
        Ah[:, r:r + 256_000].copy_(Abuf[r:r + 256_000, :n].T)
    bh.copy_(Abuf[:, n])
    return Ah, bh


def reference_full(args, Ah, bh, T):
    """The reference (oracle/_ref: the unmodified sketchlsq headers, g++ -O3
    -march=native) on the SAME A and b bytes as the GPU, full size, not
    extrapolated: distribute (untimed in `value`, reported) + the reference's
    threaded backend on every host thread (WorkerPool(nproc):
    dist_generate_sparse_sign + dist_sketch_apply + sketch_vector, serial
    build_preconditioner + initial_guess, lsqr_one_sync over dist_operator for
    T iterations, eps = 0).  Returns (solve seconds, phases, x, cores)."""
    import oracle

    R = oracle.REF()
    n, d, zeta = args.n, args.dfac * args.n, args.zeta
    cores = os.cpu_count() or 1
    A = Ah.numpy().T  # (ml, n) column-major view, no copy
    x, rep, ph = R.solve_timed(A, bh.numpy(), d, zeta, 3, 0.0, T, cores)
    assert rep.iterations == T, (rep.iterations, T)
    solve_s = ph["generate"] + ph["apply"] + ph["precond"] + ph["x0"] + ph["lsqr"]
    return solve_s, {k: float(v) for k, v in ph.items()}, x, cores


def reference_desc(m, n, d, zeta, T, cores):
    return (f"reference sketchlsq (oracle/_ref: unmodified headers, g++ -O3 -march=sapphirerapids -ffp-contract=off) "
            f"on the full {m}x{n} A and b (the GPU's bytes, column-major host copy), WorkerPool({cores}): "
            f"dist_generate_sparse_sign + dist_sketch_apply + sketch_vector, serial build_preconditioner + "
            f"initial_guess on the {d}x{n} sketch, lsqr_one_sync(dist_operator) x{T} iterations (zeta={zeta}); "
            f"value = the solve without distribute (reported as phases.distribute); not extrapolated")


def eta_and_parity(torch, Abuf, n, x_gpu, x_ref, dist=None):
    """eta(x) = ||A^T r|| / (||A||_2 ||r||) (||A||_2 = 1 by construction) for both
    solutions and their distance in residual space, on the device-resident A."""
    dev = Abuf.device
    A = Abuf[:, :n]
    b = Abuf[:, n]

    def red(t):
        if dist is not None:
            dist.all_reduce(t)
        return t

    def eta(x):
        r = b - A @ torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        atr = red((A.T @ r).reshape(-1))
        rn2 = red((r * r).sum().reshape(1))
        return float(torch.linalg.norm(atr) / torch.sqrt(rn2))

    out = {"eta_gpu": eta(x_gpu)}
    if x_ref is not None:
        dxr = A @ torch.from_numpy(np.ascontiguousarray(x_gpu - x_ref)).to(dev)
        num = float(torch.sqrt(red((dxr * dxr).sum().reshape(1))))
        bn = float(torch.sqrt(red((b * b).sum().reshape(1))))
        out.update({"eta_ref": eta(x_ref), "res_delta": num / bn,
                    "x_rel_delta": float(np.linalg.norm(x_gpu - x_ref) / np.linalg.norm(x_ref)),
                    "bar": "eta_gpu <= max(2 eta_ref, 1e-14) and res_delta <= 1e-12 cond(A) (SURVEY 8(c)(iv))"})
        out["pass"] = bool(out["eta_gpu"] <= max(2 * out["eta_ref"], 1e-14) and out["res_delta"] <= 1e-12 * 1e8)
    return out


# ------------------------------------------------------------ config C4 (sparse)

def run_sparse(args, world, rank, local_rank):
    """BASELINE configs[3]: sparse CSR A, m=2^24, n=2000, exactly 50 distinct
    random columns per row (the reference rejection sampler, seed 4), values
    +-sigma_j with sigma log-spaced in [1e-6, 1] (cond ~1e6), b uniform(-1,1);
    d = 4n, zeta = 8; one line like the dense one (value = seconds per solve)."""
    import ctypes as ct

    import torch

    import paper_2506_03070_b200 as slq

    m = args.m if args.m != 4_000_000 else 1 << 24
    n = args.n if args.n != 1000 else 2000
    nnz_row, d, zeta = 50, args.dfac * n, args.zeta
    cond = 1e6
    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    part = slq.partition_rows(m, world)
    r0, r1 = part.begin(rank), part.end(rank)
    ml = r1 - r0
    ctx = slq.Context(local_rank)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [slq.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(uid[0], rank, world)
    sigma = np.power(10.0, -np.log10(cond) * np.arange(n) / max(n - 1, 1))
    t_gen = time.perf_counter()
    A, _ = slq.SparseDeviceMatrix.create_csr(ml, n, ml * nnz_row, row_begin=r0, with_b=True, ctx=ctx)
    A.fill_random(nnz_row, 4, sigma)
    b = np.random.default_rng(1000 + rank).uniform(-1.0, 1.0, ml)
    A.set_rhs(b)
    t_gen = time.perf_counter() - t_gen
    # the row-blocked CSC copy the two-pass LSQR operator streams for A^T u_hat is built once per
    # matrix (a layout conversion, like the CSC -> CSR of an upload): the first solve builds it on a
    # side stream, overlapped with its sketch and QR (first_solve_s); an explicit rebuild is timed
    # alone (transposed_copy_build_s).  The timed solves reuse it.
    def solve0():
        return slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=args.iters or 30), ctx=ctx)

    torch.cuda.synchronize()
    t_first = time.perf_counter()
    solve0()
    t_first = time.perf_counter() - t_first
    t_prep = time.perf_counter()
    A.prepare()
    t_prep = time.perf_counter() - t_prep
    a_norm_f = float(np.sqrt(m * nnz_row * np.mean(sigma ** 2)))  # E||A||_F (an upper bound for ||A||_2)
    # ||A||_2 >= ||A e_0|| = sigma_0 sqrt(nnz of column 0) ~ sqrt(m nnz_row / n): with 1% margin a lower
    # bound, so eta computed with it over-estimates the true backward error (conservative stopping rule)
    a_norm_lb = 0.99 * float(sigma[0]) * math.sqrt(m * nnz_row / n)

    def solve(eta=False, norm=None):
        return slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=T, a_norm_est=(norm or a_norm_lb) if eta else 0.0),
                         ctx=ctx)

    # calibration of T to eta <= target (as for C3), then the warm-up solves
    T = args.iters or 16
    while True:
        _, rep_w, _ = solve(eta=True)
        eta_w = rep_w.backward_error
        if args.iters or eta_w <= args.eta or T >= 80:
            break
        T = min(80, T + max(1, int(math.ceil(T * (math.log(eta_w / args.eta) / max(math.log(eta_w / 1e-16), 1.0))))))
    for _ in range(max(args.warmup, 3)):
        solve()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(1.5)
    solve()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.kernel_launches
    ev0.record(stream)
    phases = []
    for _ in range(args.steps):
        _, rep, ph = solve()
        phases.append(ph)
    ev1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    sec = ev0.elapsed_time(ev1) * 1e-3 / args.steps
    if dist is not None:
        t = torch.tensor([sec], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    ph = {k: float(np.mean([p[k] for p in phases])) for k in phases[0]}
    _, rep_eta, _ = solve(eta=True)
    _, rep_etaf, _ = solve(eta=True, norm=a_norm_f)
    nnz = ml * nnz_row
    pass_bytes = 12.0 * nnz + 8.0 * (ml + 1) + 16.0 * ml
    # bytes the two-pass operator streams: the CSR pass (values + u16 columns + row pointers, u in,
    # u_hat out), then the row-blocked CSC copy (u16 row + value per entry), u_hat once more and the
    # per-block column starts
    moved_bytes = (10.0 * nnz + 8.0 * (ml + 1) + 16.0 * ml) + (10.0 * nnz + 8.0 * ml + 4.0 * math.ceil(ml / 16384) * (n + 1))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    it_s = ph["lsqr_per_iteration"]
    kt = ct.c_double(0.0)  # K4s alone: average launch time over 10 launches on the library stream
    slq._capi.lib.slq_time_sparse_pass(ctx.handle, A.handle, 10, ct.byref(kt))
    k_s = kt.value
    if rank == 0:
        print(json.dumps({
            "metric": METRIC + " [config C4 sparse]", "value": sec, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": sec * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device generator: 50 distinct random columns/row, seed 4; b uniform)",
            "config": {"workload": f"C4: sparse CSR m={m} n={n} nnz/row={nnz_row} cond~1e6, d={d} zeta={zeta}, "
                                   f"LSQR to eta<={args.eta:g} (||A||_2 bounded below by column 0's norm)",
                       "m": m, "n": n, "nnz": m * nnz_row, "d": d, "zeta": zeta,
                       "lsqr_iterations": T, "parallelism": f"rows/{world}" if world > 1 else "1 GPU"},
            "eta_final": rep_eta.backward_error, "eta_F_final": rep_etaf.backward_error, "phases_s": ph,
            "roofline": {"bound": "hbm", "kernel": "K4s two-pass operator (sparse_upass: u_hat = A p + c u, "
                                                   "||u_hat||^2 over the CSR, TMA-staged; sparse_tpass: z = A^T u_hat "
                                                   "over the row-blocked CSC copy)",
                         "moved_bytes_per_launch": moved_bytes,
                         "moved_gbs": moved_bytes / k_s / 1e9 if k_s else None,
                         "moved_frac": moved_bytes / k_s / 1e9 / peak if k_s else None,
                         "achieved": pass_bytes / k_s / 1e9 if k_s else None, "peak": peak, "unit": "GB/s",
                         "frac": pass_bytes / k_s / 1e9 / peak if k_s else None, "traffic": _sparse_traffic(m, n, world),
                         "algorithmic_bytes_per_launch": pass_bytes, "seconds_per_launch": k_s,
                         "lsqr_iteration_gbs": pass_bytes / it_s / 1e9 if it_s else None},
            "gpu_launches": int(ctx.kernel_launches - launches0), "clocks": ck, "generation_s": t_gen,
            "transposed_copy_build_s": t_prep, "first_solve_s": t_first}))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------ main

def _sparse_traffic(m, n, world):
    """DRAM bytes per launch of the two-pass sparse operator (u_hat pass + A^T u_hat
    pass) from the committed ncu capture (profiles/ncu_summary.json), scaled to
    this rank's rows; None if absent."""
    try:
        sp = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get("sparse_two_pass", {})
        if sp.get("n") != n or not sp.get("m"):
            return None
        return sp["dram_bytes_per_operator_launch"] * (m / world) / sp["m"]
    except Exception:
        return None


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # NCCL's init lines (communicator size, rank, transport) document the N-rank run
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.config == "c4" and args.impl == "ours":
        return run_sparse(args, world, rank, local_rank)
    n, d, zeta = args.n, args.dfac * args.n, args.zeta
    config = {"workload": f"C3: dense m={args.m} n={n} cond={args.cond:g} rho={args.rho}, sparse-sign d={d} "
                          f"zeta={zeta}, LSQR to eta<={args.eta:g}",
              "m": args.m, "n": n, "d": d, "zeta": zeta, "cond": args.cond,
              "parallelism": f"rows/{world}" if world > 1 else "1 GPU",
              "l2": "A is 32 GB >> 126 MB L2: inputs larger than L2, no flush needed"}

    import torch

    if args.impl == "reference":
        if rank != 0:
            return
        # same A / b bytes as the GPU arm (device generator, untimed harness), copied to the host
        T = args.iters or 30
        dev = torch.device("cuda", 0)
        Abuf, ld, _ = make_problem(torch, args.m, n, args.cond, args.rho, 0, args.m, dev)
        Ah, bh = host_copy(torch, Abuf, n, args.m, pinned=False)
        vals, phs, x_ref, cores = [], [], None, os.cpu_count()
        t_start = time.perf_counter()
        for k in range(max(1, args.steps)):
            v, ph, x_ref, cores = reference_full(args, Ah, bh, T)
            vals.append(v)
            phs.append(ph)
            el = time.perf_counter() - t_start
            if el + el / (k + 1) > args.ref_budget:  # the next full solve would exceed the budget
                break
        v = float(np.mean(vals))
        ph = {k: float(np.mean([p[k] for p in phs])) for k in phs[0]}
        par = eta_and_parity(torch, Abuf, n, x_ref, None)
        desc = reference_desc(args.m, n, d, zeta, T, cores)
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
                          "steps": len(vals), "steps_requested": args.steps, "warmup": 0, "ms_per_step": v * 1e3,
                          "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic (the GPU arm's device generator, seed 1, copied to the host)",
                          "config": dict(config, lsqr_iterations=T),
                          "eta_final": par["eta_gpu"],
                          "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "reference",
                                           "sample": desc, "phases": ph, "cpu": cpu_info()},
                          "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import paper_2506_03070_b200 as slq

    dist = None
    if world > 1:
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)

    part = slq.partition_rows(args.m, world)
    r0, r1 = part.begin(rank), part.end(rank)
    t_gen = time.perf_counter()
    Abuf, ld, x_star = make_problem(torch, args.m, n, args.cond, args.rho, r0, r1, dev, dist)
    t_gen = time.perf_counter() - t_gen

    ctx = slq.Context(local_rank)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [slq.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(uid[0], rank, world)
    A = slq.DeviceMatrix.wrap(Abuf.data_ptr(), r1 - r0, n, ld, row_begin=r0, ctx=ctx, owner=Abuf)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def solve(T, eta=False):
        # eta=True adds one direct ||A^T r|| pass (backward error); never inside the timed steps
        return slq.solve(A, d, zeta, 3, slq.SolveOptions(eps=0.0, maxit=T, a_norm_est=1.0 if eta else 0.0), ctx=ctx)

    # calibration of T (iterations to eta <= target), then the warm-up solves
    T = args.iters or 24
    eta = None
    while True:
        x, rep, ph = solve(T, eta=True)
        eta = rep.backward_error
        if args.iters or eta <= args.eta or T >= 80:
            break
        T = min(80, T + max(1, int(math.ceil(T * (math.log(eta / args.eta) / max(math.log(eta / 1e-16), 1.0))))))
    for _ in range(max(args.warmup, 3)):
        solve(T)
    # timed region: K solves, CUDA events on the solver stream, max over ranks
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(1.5)  # let nvidia-smi/NVML initialise outside the timed region
    solve(T)         # keep the GPU busy while the sampler settles
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches0 = ctx.kernel_launches
    phases = []
    host_s = []
    for _ in range(args.steps):
        h0 = time.perf_counter()
        x, rep, ph = solve(T)
        host_s.append(time.perf_counter() - h0)
        phases.append(ph)
    ev1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    launches = ctx.kernel_launches - launches0
    sec = ev0.elapsed_time(ev1) * 1e-3 / args.steps
    if dist is not None:
        t = torch.tensor([sec], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    ph = {k: float(np.mean([p[k] for p in phases])) for k in phases[0]}
    _, rep_eta, _ = solve(T, eta=True)  # untimed: verify the backward error of the timed configuration
    eta = rep_eta.backward_error

    # kernel-level timing for the roofline (dominant kernel: K4 fused LSQR pass)
    kt = np.zeros(4)
    slq._capi.lib.slq_time_kernels(ctx.handle, A.handle, d, zeta, 3, 10, kt.ctypes.data_as(ct.POINTER(ct.c_double)))
    ml = r1 - r0
    pass_bytes = 8.0 * ml * n + 16.0 * ml
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak = json.load(open(peaks_path))["hbm_gbs"]
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    achieved = pass_bytes / kt[0] / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            fp = json.load(open(prof)).get("fused_pass", {})
            traffic = fp.get("dram_bytes_per_launch")
            if fp.get("n") != n or not fp.get("m"):
                traffic = None  # the capture is for another shape
            elif traffic is not None and fp["m"] != ml:
                traffic = traffic * ml / fp["m"]  # per-row traffic is size-independent; this rank's rows
        except Exception:
            traffic = None
    iter_bytes = 8.0 * ml * n + 16.0 * ml + 8.0 * n * n
    in_solve = ph["lsqr"] / (T + 1)  # init pass + T iterations, K5 kernels included (conservative)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "fused_pass (K4: u_hat = A p + c u, z = A^T u_hat, ||u_hat||^2)",
                "algorithmic_bytes_per_launch": pass_bytes, "seconds_per_launch": float(kt[0]),
                "timing": "10 launches on the library stream (CUDA events) with the live u, p, c of the last solve",
                "in_solve_seconds_per_iteration": in_solve, "in_solve_gbs": pass_bytes / in_solve / 1e9,
                "in_solve_frac": pass_bytes / in_solve / 1e9 / peak,
                "peak_source": peak_src,
                "lsqr_iteration_gbs": iter_bytes / ph["lsqr_per_iteration"] / 1e9 if ph["lsqr_per_iteration"] else None,
                "sketch_seconds": float(kt[1]), "sketch_gbs": (8.0 * ml * (ld) + 4.0 * ml * zeta) / kt[1] / 1e9,
                # SURVEY 8(d)'s second bound for S.[A b]: 16 zeta m n B of shared-memory read-modify-write at the
                # 37.2 TB/s aggregate shared-memory rate (the scatter formulation; HBM alone would allow 4.98 ms at C3)
                "sketch_smem_bound_seconds": 16.0 * zeta * ml * (n + 1) / 37.2e12,
                "sketch_frac_of_smem_bound": (16.0 * zeta * ml * (n + 1) / 37.2e12) / float(kt[1]) if kt[1] else None,
                "precond_seconds": float(kt[3])}

    # e2e through the C-ABI from pinned host buffers (column-major A as the reference's DenseMatrix)
    e2e = None
    Ah = bh = None
    want_cpu = rank == 0 and world == 1 and not args.no_cpu
    if not args.no_e2e or want_cpu:
        Ah, bh = host_copy(torch, Abuf, n, ml, pinned=True)
    if not args.no_e2e:
        try:
            xh = np.zeros(n)
            rep_h = slq._capi.Report()
            pt = slq._capi.PhaseTimes()
            co = slq._capi.SolveOpts()
            slq._capi.lib.slq_solve_opts_default(ct.byref(co))
            co.eps, co.maxit, co.one_sync = 0.0, T, 1

            def e2e_step():
                st = slq._capi.lib.slq_solve_host(ctx.handle, ct.cast(Ah.data_ptr(), slq._capi.dp), ml, n, ml,
                                                  ct.cast(bh.data_ptr(), slq._capi.dp), r0, d, zeta, 3, ct.byref(co),
                                                  xh.ctypes.data_as(slq._capi.dp), ct.byref(rep_h), ct.byref(pt), None)
                if st != 0:
                    raise RuntimeError(slq._capi.lib.slq_last_error().decode())

            e2e_step()  # warm
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ke = max(1, min(args.steps, 3))
            for _ in range(ke):
                e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            es = e0.elapsed_time(e1) * 1e-3 / ke
            if dist is not None:
                t = torch.tensor([es], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                es = float(t.item())
            e2e = {"value": es, "unit": "s", "h2d_bytes_per_step": int(8 * ml * n + 8 * ml),
                   "d2h_bytes_per_step": int(8 * n), "steps": ke,
                   "path": "slq_solve_host (C-ABI, pinned column-major host A)",
                   # the host path sketches each block as it lands (register gather): rounding-level difference
                   "x_rel_delta_vs_device_path": float(np.linalg.norm(xh - x) / np.linalg.norm(x))}
        except Exception as ex:  # report, never hide
            e2e = {"value": None, "unit": "s", "error": str(ex)[:300]}

    # multi-GPU consistency: every rank must hold the same x, bit for bit (replicated n-vector work)
    ranks_agree = None
    if dist is not None:
        xt = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        xs = [torch.empty_like(xt) for _ in range(world)]
        dist.all_gather(xs, xt)
        ranks_agree = bool(all(torch.equal(xs[0], y) for y in xs))

    cpu = None
    x_ref = None
    if want_cpu:
        try:
            v, cph, x_ref, cores = reference_full(args, Ah, bh, T)
            cpu = {"value": v, "unit": "s", "cores": cores, "kind": "reference",
                   "sample": reference_desc(args.m, n, d, zeta, T, cores), "phases": cph, "cpu": cpu_info()}
        except Exception as ex:
            cpu = {"value": None, "unit": "s", "error": str(ex)[:300]}
    parity = eta_and_parity(torch, Abuf, n, x, x_ref, dist)
    del Ah, bh

    if rank == 0:
        line = {
            "metric": METRIC, "value": sec, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": sec * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (device generator, seed 1)",
            "config": dict(config, lsqr_iterations=T),
            "eta_final": eta, "iterations": rep.iterations, "parity_vs_reference": parity,
            "multi_gpu": {"ranks": world, "x_bitwise_equal_across_ranks": ranks_agree,
                          "nccl_calls_per_solve": ph["nccl_calls"],
                          "nccl_calls_per_iteration": 1 if world > 1 else 0,
                          "collectives": "ncclReduce S[A b] + ncclBroadcast status/M/M^T/x0 + one ncclAllReduce "
                                         "of n+1 doubles per LSQR iteration" if world > 1 else None},
            "phases_s": ph, "host_s_per_step": float(np.mean(host_s)), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": ck, "generation_s": t_gen,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
