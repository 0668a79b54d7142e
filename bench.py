#!/usr/bin/env python
"""BTA solver benchmark (BASELINE.json configs[1], SURVEY.md §8(d) "C2").

One step = one pass of the reference's structured-solver hot path over the
C2 matrix (n=48 time blocks, block size b=2048, arrowhead a=6, FP64):

    restore the input matrix (POBTAF works in place, bta.py:177)
    POBTAF + fused log-determinant      (bta.factorize / bta.logdet)
    POBTAS, one right-hand side         (bta.solve)
    POBTASI                             (bta.selected_invert)

value  = algorithmic FLOPs of the three routines (SURVEY.md §8(d) formulas,
         paper_2507_06938_b200/perf.py) / device time, summed over ranks.
e2e    = the same metric through the reference-facing Python API with HOST
         buffers: pinned matrix upload, factorize, logdet read-back, solve
         of a host RHS, selected inverse copied back to pinned host memory.
roofline: the dominant routine (the longest of POBTAF / POBTASI, each a short
         chain of launches on one stream) against the FP64 DMMA peak measured live on the box with a
         register-resident DMMA.8x8x4 loop (MEASURED_PEAKS.json has no FP64
         entry).
cpu_baseline: the oracle port of the reference algorithm (numpy/OpenBLAS,
         oracle/bta_np.py) on a bounded sample, rank 0 at N=1 only.

Multi-GPU (torchrun): every rank factorizes its own C2 replica (the C2
microbench is one matrix per GPU), so scaling is "weak" and there is no
collective on the data path; only the timing max-reduction uses NCCL.  The
time-partitioned distributed solver (S3, NCCL point-to-point reduced system)
is measured with `--config c5` (SURVEY §8(d) C5, 96 time blocks per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BTA Cholesky/selinv FP64 TFLOP/s"
UNIT = "TFLOP/s"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--n", type=int, default=48)
    p.add_argument("--b", type=int, default=2048)
    p.add_argument("--a", type=int, default=6)
    p.add_argument("--cpu-sample-blocks", type=int, default=6)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--config", default="c2", choices=["c2", "c5"],
                   help="c2: BTA microbench (default); c5: distributed POBTAF weak scaling, "
                        "96 time blocks per GPU, one partition per rank over NCCL")
    p.add_argument("--lb", type=float, default=1.6, help="C5 load-balance factor (plan_partitions lb; 1.6 measured best at 2 and 4 GPUs)")
    p.add_argument("--no-inla", action="store_true",
                   help="skip the C3 f_obj measurement (north-star model, rank 0 at N=1)")
    return p.parse_args()


def workload(args):
    return {
        "workload": f"C2 BTA microbench: POBTAF+POBTAS(1 rhs)+POBTASI, n={args.n} time blocks, "
        f"b={args.b}, a={args.a}, FP64",
        "n_blocks": args.n,
        "block_size": args.b,
        "arrow_size": args.a,
        "l2_policy": "inputs larger than L2 (matrix %.2f GB restored from a pristine copy each step)"
        % (8e-9 * (args.n * args.b**2 + (args.n - 1) * args.b**2 + args.n * args.a * args.b + args.a**2)),
    }


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- CPU legs
def cpu_sample(args, blocks, reps=1):
    """Time the oracle port (reference algorithm on numpy/OpenBLAS) on a
    bounded sample of the workload: the first `blocks` time blocks."""
    import numpy as np

    from oracle import bta_np
    from paper_2507_06938_b200 import perf

    n, b, a = blocks, args.b, args.a
    rng = np.random.default_rng(0)
    data0 = bta_np.random_spd_bta(rng, n, b, a)
    rhs = rng.normal(size=n * b + a)
    flops = (perf.flops_pobtaf(n, b, a) + perf.flops_pobtasi(n, b, a)
             + perf.flops_pobtas(n, b, a))
    times = []
    for _ in range(reps):
        data = data0.copy()
        t0 = time.perf_counter()
        has = bta_np.factorize(data, n, b, a)
        bta_np.logdet(data, n, b, a)
        bta_np.solve(data, n, b, a, has, rhs)
        bta_np.selected_invert(data, n, b, a, has)
        times.append(time.perf_counter() - t0)
    try:
        from threadpoolctl import threadpool_info

        cores = max([int(i.get("num_threads", 1)) for i in threadpool_info()] or [1])
    except Exception:  # noqa: BLE001
        cores = os.cpu_count() or 1
    sample = (f"oracle port (numpy/scipy OpenBLAS, reference bta.py algorithm): POBTAF+POBTAS+POBTASI "
              f"on the first {n} of {args.n} time blocks, b={b}, a={a}")
    return flops, times, cores, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.warmup > 0:  # one untimed pass (BLAS thread pool, page faults)
        cpu_sample(args, args.cpu_sample_blocks, reps=1)
    flops, times, cores, sample = cpu_sample(args, args.cpu_sample_blocks, reps=args.steps)
    tot = sum(times)
    value = flops * len(times) / tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator law, seeded)", "config": workload(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- C3 f_obj
def measure_c3(dev):
    """One trivariate (n_v=3, n_s=1675, n_t=48) f_obj at theta0 on this GPU --
    the north-star model (BASELINE configs[2]); reported beside the C2 line with
    the per-iteration estimate for a full 8-GPU box (1 line-search + 31
    gradient evaluations, round-robin)."""
    import numpy as np
    import torch

    from paper_2507_06938_b200 import inla
    from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic

    th0 = np.array([-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05,
                    0.05, 0.65, -0.35, 0.35])
    true = [-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00, 0.00, 0.60,
            -0.40, 0.30]
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), true, seed=2, device=dev)
    ev = inla.ObjectiveEvaluator(data.spec, prior=inla.ThetaPrior.for_dim(15, mean=th0, sd=2.0),
                                 device=dev)
    ev.objective(th0)
    torch.cuda.synchronize()
    ts, tc = [], []
    for _ in range(2):
        inla.prior_cache_clear()  # a full f_obj: both factorizations
        t0 = time.perf_counter()
        f = ev.objective(th0)
        ts.append(time.perf_counter() - t0)
    for _ in range(2):  # Q_p already factorized for these prior coefficients (noise-only moves)
        t0 = time.perf_counter()
        ev.objective(th0)
        tc.append(time.perf_counter() - t0)
    ev.release_workspaces()
    t = min(ts)
    return {"model": "C3 trivariate n_v=3 n_s=1675 n_t=48 n_r=1 (b=5025, N=241203), theta0",
            "f_obj_s": t, "f_obj_s_prior_cached": min(tc), "f_obj": f,
            "oracle_f_obj": -193110.15144130366,
            "iteration_s_est_8gpu": t * (1 + -(-31 // 8)),
            # near the mode: 1 line-search try (split over a GPU pair) + the 30
            # new gradient points through the cost-ordered queue on 8 GPUs (24
            # full f_obj, 3 per GPU, then the 6 prior-cached ones)
            "iteration_s_est_8gpu_near_mode": max(min(tc), t / 2) + 3 * t + min(tc),
            "iteration_s_est_1gpu": t * 32,
            "iteration_s_measured_4gpu": "12.0-13.2 (profiles/r01_c3_lbfgs_iterations_4gpu_v3.json)",
            "cpu_reference_f_obj_s_survey": 67.7}


def measure_c3_iteration(n_gpus, max_iter=2):
    """Measured north-star number at N GPUs: C3 L-BFGS iterations from theta0
    (Armijo line search split over a GPU pair + the 31-point central-difference
    gradient round-robin over the N GPUs, inla.py:535-605 / sched.py:99), one
    ObjectiveEvaluator per GPU driven by sched.GpuRunner from this process."""
    import warnings

    import numpy as np
    import torch

    from paper_2507_06938_b200 import inla, sched
    from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic

    th0 = np.array([-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05,
                    0.05, 0.65, -0.35, 0.35])
    true = [-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00, 0.00, 0.60,
            -0.40, 0.30]
    t0 = time.perf_counter()
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), true, seed=2,
                              device=torch.device("cuda", 0))
    prior = inla.ThetaPrior.for_dim(15, mean=th0, sd=2.0)
    evs = [inla.ObjectiveEvaluator(data.spec, prior=prior, device=torch.device("cuda", g))
           for g in range(n_gpus)]
    runner = sched.GpuRunner(evs)
    runner.evaluate_points([th0] * n_gpus)  # warm every device
    setup = time.perf_counter() - t0
    inla.prior_cache_clear()
    recs = []
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = inla.minimize(evs[0], th0, gtol=1e-3, ftol=1e-12, max_iter=max_iter, runner=runner,
                            on_iteration=recs.append)
    total = time.perf_counter() - t0
    for ev in evs:
        ev.release_workspaces()
    return {"model": "C3 trivariate n_v=3 n_s=1675 n_t=48 n_r=1 (b=5025, N=241203), "
                     "L-BFGS from theta0",
            "n_gpus": n_gpus, "iteration_s_measured": [r.seconds for r in recs],
            "f_evals_per_iteration": [r.f_evals for r in recs],
            "total_s_incl_first_gradient": total, "setup_s": setup, "f": res.f,
            "timing": "host wall clock (perf_counter) around minimize; each f_obj synchronises"}


# --------------------------------------------------------------- GPU leg
def run_c5(args):
    """random SPD BTA (96*N, b, a), plan_partitions(96*N, N, lb),
    PPOBTAF with one partition per GPU over NCCL; value = the sequential
    POBTAF's algorithmic FLOPs / time (useful throughput, weak scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2507_06938_b200 import bta, bta_dist, perf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, b, a = 96 * world, args.b, args.a
    plan = bta_dist.plan_partitions(n, world, args.lb)
    m = bta.BTAMatrix(n, b, a, perf.device_random_spd_bta(n, b, a, seed=7, device=dev)) \
        if rank == 0 else None

    def step():
        if world > 1:
            return bta_dist.d_factorize_nccl(m, plan)[0]
        return bta.logdet(bta.factorize(m.copy()))

    for _ in range(args.warmup):
        ld = step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ld = step()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    fl = perf.flops_pobtaf(n, b, a)
    if rank == 0:
        print(json.dumps({
            "metric": "distributed POBTAF useful FP64 TFLOP/s (C5)",
            "value": fl * args.steps / el / 1e12, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic SPD BTA (reference generator law), seeded",
            "config": {"workload": f"C5 d_factorize n={n} (96 per GPU), b={b}, a={a}, "
                                   f"P={world}, lb={args.lb}", "boundaries": list(plan.boundaries)},
            "logdet": ld,
            "timing": "host wall clock around the synchronous call, max over ranks",
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    # stdout carries exactly one JSON line: native libraries (NCCL's version
    # banner, ...) write to fd 1, so fd 1 becomes stderr and Python's stdout
    # keeps the original descriptor
    out_fd = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(out_fd, "w", buffering=1)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c5":
        return run_c5(args)

    import torch
    import torch.distributed as dist

    from paper_2507_06938_b200 import _lib, bta, perf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    n, b, a = args.n, args.b, args.a
    stream = torch.cuda.current_stream()
    sp = _lib.stream_ptr(stream)

    # live FP64 DMMA peak (roofline denominator)
    scratch = torch.zeros(16, dtype=torch.float64, device=dev)
    peak = 0.0
    for _ in range(3):
        iters = 20000
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        _lib.check(lib.stbta_probe_dmma(148 * 2, iters, _lib.ptr(scratch), sp), "probe")
        s1.record()
        torch.cuda.synchronize()
        peak = max(peak, 148 * 2 * 8 * iters * 16 * 512 / (s0.elapsed_time(s1) * 1e-3) / 1e12)

    pristine = perf.device_random_spd_bta(n, b, a, seed=1234 + rank, device=dev)
    mat = bta.BTAMatrix(n, b, a, torch.empty_like(pristine))
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    rhs0 = torch.randn(mat.dim, dtype=torch.float64, device=dev, generator=g)
    x = torch.empty_like(rhs0)
    inv = bta.BTAMatrix(n, b, a, torch.empty_like(pristine))
    ws_f = torch.empty(lib.stbta_pobtaf_workspace_bytes(n, b, a), dtype=torch.uint8, device=dev)
    ws_s = torch.empty(lib.stbta_pobtas_workspace_bytes(n, b, a, 1), dtype=torch.uint8, device=dev)
    ws_i = torch.empty(lib.stbta_pobtasi_workspace_bytes(n, b, a), dtype=torch.uint8, device=dev)
    ld = torch.zeros(2, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)

    f_f = perf.flops_pobtaf(n, b, a)
    f_s = perf.flops_pobtas(n, b, a)
    f_i = perf.flops_pobtasi(n, b, a)
    step_flops = f_f + f_s + f_i

    def step(evs=None):
        mat.data.copy_(pristine)
        if evs:
            evs[0].record(stream)
        _lib.check(lib.stbta_pobtaf(_lib.ptr(mat.data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info),
                                    _lib.ptr(ws_f), ws_f.numel(), sp), "pobtaf")
        if evs:
            evs[1].record(stream)
        x.copy_(rhs0)
        _lib.check(lib.stbta_pobtas(_lib.ptr(mat.data), n, b, a, 1, _lib.ptr(x), 1, 0,
                                    _lib.ptr(ws_s), ws_s.numel(), sp), "pobtas")
        if evs:
            evs[2].record(stream)
        _lib.check(lib.stbta_pobtasi(_lib.ptr(mat.data), _lib.ptr(inv.data), n, b, a, 1,
                                     _lib.ptr(ws_i), ws_i.numel(), sp), "pobtasi")
        if evs:
            evs[3].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(info.item()) != 0:
        raise RuntimeError(f"POBTAF reported a non-SPD pivot (info={int(info.item())})")
    logdet_dev = float(ld[0].item())

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.stbta_launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = lib.stbta_launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = t_start.elapsed_time(t_end) * 1e-3
    t_f = sum(e[0].elapsed_time(e[1]) for e in evs) * 1e-3 / args.steps
    t_s = sum(e[1].elapsed_time(e[2]) for e in evs) * 1e-3 / args.steps
    t_i = sum(e[2].elapsed_time(e[3]) for e in evs) * 1e-3 / args.steps
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    ms_step = 1e3 * elapsed / args.steps
    value = world * step_flops * args.steps / elapsed / 1e12

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        host_in = pristine.cpu().pin_memory()
        host_rhs = rhs0.cpu().numpy()
        host_out = torch.empty(inv.data.numel(), dtype=torch.float64).pin_memory()
        del mat, inv
        torch.cuda.empty_cache()

        def e2e_step():
            m = bta.BTAMatrix(n, b, a, host_in)                  # pinned H2D upload
            fac = bta.factorize(m, use_arrow=True)                 # bta.py:177
            bta.logdet(fac)                                        # bta.py:238
            xs = bta.solve(fac, host_rhs)                          # bta.py:305 (host in/out)
            sel = bta.selected_invert(fac, out=host_out)           # bta.py:310, streamed to host
            sel.numpy(out=host_out)                                # waits for the D2H stream
            return xs

        e2e_step()
        torch.cuda.synchronize()
        e2e_steps = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([t_e2e], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        nbytes = 8 * perf.storage_elems(n, b, a)
        e2e = {"value": world * step_flops * e2e_steps / t_e2e / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": nbytes + 8 * (n * b + a),
               "d2h_bytes_per_step": nbytes + 8 * (n * b + a) + 8 + 4,
               "steps": e2e_steps, "timing": "host wall clock around synchronous API calls",
               "overlap": "H2D in time-block chunks overlapped with POBTAF (per-block ready flags); "
                          "inverse D2H block by block overlapped with POBTASI (completion counters)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        flops_c, times_c, cores, sample = cpu_sample(args, args.cpu_sample_blocks, reps=1)
        cpu = {"value": flops_c / min(times_c) / 1e12, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": sample, "seconds": min(times_c)}

    inla_obj = None
    if rank == 0 and world == 1 and not args.no_inla:
        inla_obj = measure_c3(dev)
    if world > 1:
        # every rank's timed work is done; the C3 north-star iteration then
        # runs from rank 0 over all N GPUs of the run (ranks > 0 leave first)
        dist.barrier()
        dist.destroy_process_group()
        if rank != 0:
            return 0
        if not args.no_inla:
            del pristine, ws_f, ws_s, ws_i
            torch.cuda.empty_cache()
            try:
                inla_obj = measure_c3_iteration(world)
            except Exception as exc:  # the C2 line must still print
                inla_obj = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        # roofline of the dominant routine (the longest launch chain of the step)
        dom = "pobtasi" if t_i > t_f else "pobtaf"
        achieved = (f_i / t_i if dom == "pobtasi" else f_f / t_f) / 1e12
        traffic = None
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")
        if os.path.exists(tpath) and (n, b, a) == (48, 2048, 6):
            with open(tpath) as fh:
                traffic = json.load(fh).get(f"c2_{dom}", {}).get("dram_bytes")
        kname = ("POBTASI (stbta_pobtasi launch chain: W pre-pass + persistent TMA recursion)"
                 if dom == "pobtasi" else "POBTAF (stbta_pobtaf launch chain: persistent TMA task graph)")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator law: SPD L L^T, seeded, drawn on device)",
            "config": workload(args),
            "roofline": {"bound": "tensor", "kernel": kname,
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per call (ncu, profiles/r01_traffic.json)",
                         "peak_source": "FP64 DMMA.8x8x4 register-loop probe measured live "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            "routines": {
                "pobtaf": {"ms": 1e3 * t_f, "tflops": f_f / t_f / 1e12},
                "pobtas": {"ms": 1e3 * t_s, "gbs": perf.bytes_pobtas(n, b, a) / t_s / 1e9},
                "pobtasi": {"ms": 1e3 * t_i, "tflops": f_i / t_i / 1e12},
            },
            "logdet": logdet_dev,
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "inla": inla_obj,
        }
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
