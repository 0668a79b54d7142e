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
cpu_baseline: the reference's own CPU path -- the UNMODIFIED stinla package
         installed into baseline/_ref (oracle port if absent) -- on the FULL
         C2 matrix from the reference generator, once, all host cores; rank 0
         at N=1 only.  `--impl reference` times the same for every step.
inla:    the north-star number (BASELINE configs[2]/[3]): measured seconds of
         one BFGS iteration of the trivariate C3 model from theta0 and one
         near the mode over all N GPUs of the run (sched.GpuRunner), with the
         iteration's useful FP64 TFLOP/s.  `--impl reference` at N=1 also
         times the reference CPU f_obj of the same model on the host cores.

Multi-GPU: `--gpus N` without torchrun re-launches itself through
torch.distributed.run (one rank per GPU).  Every rank factorizes its own C2
replica (the C2 microbench is one matrix per GPU), so scaling is "weak" and
there is no collective on the data path; only the timing max-reduction uses
NCCL.  Rank 0 then drives all N GPUs for the C3 iterations.  The
time-partitioned distributed solver (S3, NCCL reduced system) is measured
with `--config c5` (SURVEY §8(d) C5, 96 time blocks per GPU).

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


def _hbm_gbs():
    """Measured copy bandwidth of this pool's B200s (MEASURED_PEAKS.json), else
    the B200_PROFILING.md fallback."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6540.0


HBM_GBS = _hbm_gbs()


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--n", type=int, default=48)
    p.add_argument("--b", type=int, default=2048)
    p.add_argument("--a", type=int, default=6)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--config", default="c2", choices=["c2", "c5"],
                   help="c2: BTA microbench (default); c5: distributed POBTAF weak scaling, "
                        "96 time blocks per GPU, one partition per rank over NCCL")
    p.add_argument("--lb", type=float, default=2.2,
                   help="C5 load-balance factor (plan_partitions lb: the first partition, "
                        "whose blocks cost about 2.2-2.7x less, gets lb times the others' "
                        "share; 2.2 measured best at 2 and 4 GPUs, profiles/r02_c5_lb_sweep.jsonl)")
    p.add_argument("--cpu-c3", action="store_true",
                   help="also time the reference CPU C3 f_obj in this arm (the --impl reference "
                        "arm does it by default at N=1)")
    p.add_argument("--solve", default="w", choices=["w", "tile"],
                   help="C2 step's POBTAS: w = block-inverse GEMVs sharing POBTASI's W pre-pass "
                        "(stbta_pobtasi_prepare / stbta_pobtas_w / stbta_pobtasi_prepared), "
                        "tile = the tile-sweep kernel with POBTASI computing W itself")
    p.add_argument("--no-inla", action="store_true",
                   help="skip the C3 north-star measurement (BFGS iterations over the N GPUs)")
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
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

C3_THETA0 = [-0.35, -0.25, -0.30, -0.20, -0.25, -0.25, 2.05, 2.05, 2.05, 0.05, 0.05, 0.05, 0.65,
             -0.35, 0.35]
C3_TRUE = [-0.40, -0.30, -0.35, -0.25, -0.30, -0.30, 2.00, 2.00, 2.00, 0.00, 0.00, 0.00, 0.60,
           -0.40, 0.30]
def reference_module():
    """The UNMODIFIED reference package (stinla) installed into baseline/_ref
    (DESIGN.md §4), or None when it is absent (then the oracle port is timed)."""
    if not os.path.isdir(os.path.join(REF_DIR, "stinla")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import stinla  # noqa: F401
    from stinla import bta as ref_bta

    return ref_bta


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([int(i.get("num_threads", 1)) for i in threadpool_info()] or [1])
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


class CpuC2:
    """The reference's CPU path on the C2 matrix: stinla (baseline/_ref) when
    installed (kind "reference"), else the oracle port (kind "port").  The
    input is generated once by the reference generator (random_spd_bta,
    default_rng(0)); each pass copies it (untimed), then times factorize +
    logdet + solve (1 RHS) + selected_invert on all host cores."""

    def __init__(self, n, b, a):
        import numpy as np

        self.n, self.b, self.a = n, b, a
        self.ref = reference_module()
        rng = np.random.default_rng(0)
        if self.ref is not None:
            self.kind = "reference"
            self.pristine = self.ref.random_spd_bta(rng, n, b, a)
        else:
            from oracle import bta_np

            self.kind = "port"
            self.pristine = bta_np.random_spd_bta(rng, n, b, a)
        self.rhs = rng.normal(size=n * b + a)

    def run(self):
        """Seconds of one timed pass; returns (seconds, logdet)."""
        n, b, a = self.n, self.b, self.a
        if self.ref is not None:
            m = self.pristine.copy()
            t0 = time.perf_counter()
            f = self.ref.factorize(m)
            ld = self.ref.logdet(f)
            self.ref.solve(f, self.rhs)
            self.ref.selected_invert(f)
            return time.perf_counter() - t0, ld
        from oracle import bta_np

        data = self.pristine.copy()
        t0 = time.perf_counter()
        has = bta_np.factorize(data, n, b, a)
        ld = bta_np.logdet(data, n, b, a)
        bta_np.solve(data, n, b, a, has, self.rhs)
        bta_np.selected_invert(data, n, b, a, has)
        return time.perf_counter() - t0, ld

    def sample(self):
        who = ("reference stinla (baseline/_ref, numpy/scipy OpenBLAS)" if self.kind == "reference"
               else "oracle port (numpy/scipy OpenBLAS, reference bta.py algorithm)")
        return (f"{who}: factorize+logdet+solve(1 rhs)+selected_invert on the full C2 matrix "
                f"random_spd_bta(default_rng(0), {self.n}, {self.b}, {self.a}); copy of the input "
                f"untimed; {blas_threads()} BLAS threads")


def cpu_c3_fobj():
    """One C3 f_obj at theta0 through the reference's own ObjectiveEvaluator
    (stinla.inla, baseline/_ref) on the host cores.  The model: the
    reference's build_spec(settings, default_rng(2)) (the designs: the first
    draws of generate_synthetic's generator) plus the committed observations
    bench_data/c3_observations.npz (the package's generator, pinned to the
    reference's input checksums by tests/test_gpu_baseline_configs.py) --
    which skips the CPU latent draw (one more C3 POBTAF)."""
    import numpy as np

    if reference_module() is None:
        return {"unavailable": "baseline/_ref (reference stinla) not installed"}
    from stinla import inla as ref_inla
    from stinla.synthetic import SyntheticSettings, build_spec

    spec = build_spec(SyntheticSettings(3, 1675, 48, 1, 80400), np.random.default_rng(2))
    obs = np.load(os.path.join(ROOT, "bench_data", "c3_observations.npz"))
    spec.observations = [obs[f"y{i}"] for i in range(3)]
    spec.validate()
    th0 = np.array(C3_THETA0)
    t0 = time.perf_counter()
    ev = ref_inla.ObjectiveEvaluator(spec, prior=ref_inla.ThetaPrior.for_dim(15, mean=th0, sd=2.0))
    t_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = ev.objective(th0)
    t_f = time.perf_counter() - t0
    return {"kind": "reference", "f_obj_s": t_f, "f_obj": f, "evaluator_init_s": t_init,
            "cores": blas_threads(),
            "sample": "one C3 f_obj at theta0 (reference ObjectiveEvaluator.evaluate, "
                      "inla.py:320-371), workers=1, all host cores for BLAS",
            "per_iteration_s_extrapolated": {"from_theta0 (48 f_obj)": 48 * t_f,
                                             "near_mode (32 f_obj)": 32 * t_f}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c2 = CpuC2(args.n, args.b, args.a)
    # warm-up passes on a 6-block matrix (BLAS thread pool, page faults); the
    # timed steps are full C2 passes
    warm = CpuC2(min(6, args.n), args.b, args.a)
    for _ in range(args.warmup):
        warm.run()
    times = []
    for _ in range(args.steps):
        times.append(c2.run()[0])
    from paper_2507_06938_b200 import perf

    n, b, a = args.n, args.b, args.a
    flops = perf.flops_pobtaf(n, b, a) + perf.flops_pobtasi(n, b, a) + perf.flops_pobtas(n, b, a)
    tot = sum(times)
    value = flops * len(times) / tot / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator random_spd_bta, default_rng(0))",
        "config": workload(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas_threads(), "kind": c2.kind,
                         "sample": c2.sample() + "; warm-up steps on a 6-block matrix"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "seconds_per_step": times,
    }
    if args.gpus == 1 and not args.no_inla:
        # the north-star model's f_obj on the same host cores (BASELINE configs[2])
        del c2, warm
        try:
            line["inla_cpu"] = cpu_c3_fobj()
        except Exception as exc:  # noqa: BLE001 -- the C2 line must still print
            line["inla_cpu"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- C3 north star
def measure_north_star(n_gpus, peak, cpu=False):
    """The north-star number at N GPUs (BASELINE configs[2]/[3]): seconds per
    BFGS iteration of the trivariate model (n_v=3, n_s=1675, n_t=48; b=5025,
    N=241 203), IterationRecord.seconds of the reference minimize
    (inla.py:535-597) -- Armijo line search + 31-point central-difference
    gradient -- for one iteration from theta0 (far from the mode: many
    backtracking tries) and one started near the mode, one ObjectiveEvaluator
    per GPU driven by sched.GpuRunner.  Also one f_obj's latency on GPU 0
    (and with --cpu-c3 at N = 1 the reference CPU f_obj on the host cores,
    which the --impl reference arm reports by default).  The iterations resume
    recorded BFGS states of the full C3 fit (bench_data/c3_bfgs_states.npz,
    tools/c3_fit.py; minimize(state0=...)): state 0 = theta0 with its
    gradient and an identity inverse Hessian, and the first state near the
    mode whose next iteration takes one line-search try."""
    import warnings

    import numpy as np
    import torch

    from paper_2507_06938_b200 import inla, perf, sched
    from paper_2507_06938_b200.synthetic import SyntheticSettings, generate_synthetic

    th0 = np.array(C3_THETA0)
    t0 = time.perf_counter()
    data = generate_synthetic(SyntheticSettings(3, 1675, 48, 1, 80400), C3_TRUE, seed=2,
                              device=torch.device("cuda", 0))
    prior = inla.ThetaPrior.for_dim(15, mean=th0, sd=2.0)
    evs = [inla.ObjectiveEvaluator(data.spec, prior=prior, device=torch.device("cuda", g))
           for g in range(n_gpus)]
    runner = sched.GpuRunner(evs)
    runner.evaluate_points([th0] * n_gpus)  # warm every device (workspaces, TMA maps)
    setup = time.perf_counter() - t0
    pm = evs[0].pmap
    f_full = (perf.flops_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size, True)
              + perf.flops_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size, False))

    # one f_obj on GPU 0: both factorizations, then with log det Q_p cached
    ts, tc = [], []
    for _ in range(2):
        inla.prior_cache_clear()
        t0 = time.perf_counter()
        f0 = evs[0].objective(th0)
        ts.append(time.perf_counter() - t0)
    for _ in range(2):
        t0 = time.perf_counter()
        evs[0].objective(th0)
        tc.append(time.perf_counter() - t0)

    class Tracked:
        """Runner wrapper: the work counters before / after the iteration."""

        def __init__(self):
            self.width = runner.width
            self.rounds = 0

        def __call__(self, tasks):
            self.rounds += 1
            return runner(tasks)

    def one_iteration(theta, state):
        """One BFGS iteration resumed from a recorded state (minimize state0);
        IterationRecord.seconds covers the line search + the gradient."""
        inla.prior_cache_clear()
        tr, recs = Tracked(), []
        w0 = inla.work_counters()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            inla.minimize(evs[0], theta, gtol=1e-3, ftol=1e-8, max_iter=1, runner=tr,
                          on_iteration=recs.append, state0=state)
        w1 = inla.work_counters()
        r = recs[0]
        fl = w1["pobtaf_flops"] - w0["pobtaf_flops"]
        return {"seconds": r.seconds, "line_search_tries": r.f_evals - 31, "f_evals": r.f_evals,
                "rounds": tr.rounds, "pobtaf_completed": w1["pobtaf"] - w0["pobtaf"],
                "pobtaf_aborted": w1["aborted"] - w0["aborted"],
                "useful_tflops": fl / r.seconds / 1e12,
                "frac_of_n_peak": fl / r.seconds / 1e12 / (n_gpus * peak), "f": r.f}

    st = np.load(os.path.join(ROOT, "bench_data", "c3_bfgs_states.npz"))
    tries = st["tries"]
    # near the mode: the first recorded state whose next iteration took 1 try
    k_near = next(k for k in range(1, len(tries) - 1) if tries[k + 1] == 1)

    def state(k):
        return st["theta"][k], (st["f"][k], st["grad"][k], st["hinv"][k])

    far = one_iteration(*state(0))
    near = one_iteration(*state(k_near))
    far["recorded_state"], near["recorded_state"] = 0, int(k_near)
    runner.close()
    for ev in evs:
        ev.release_workspaces()
    out = {"model": "C3 trivariate n_v=3 n_s=1675 n_t=48 n_r=1 (b=5025, a=3, N=241203), "
                    "dim theta=15, prior N(theta0, 2^2), gtol 1e-3, ftol 1e-8",
           "n_gpus": n_gpus,
           "iteration_s_measured": {"from_theta0": far["seconds"], "near_mode": near["seconds"]},
           "iteration_from_theta0": far, "iteration_near_mode": near,
           "f_obj_s": min(ts), "f_obj_s_prior_cached": min(tc), "f_obj": f0,
           "f_obj_tflops": f_full / min(ts) / 1e12,
           "f_obj_frac_of_peak": f_full / min(ts) / 1e12 / peak,
           "setup_s": setup,
           "timing": "IterationRecord.seconds (host perf_counter inside inla.minimize, reference "
                     "inla.py:547,596); every f_obj synchronises; useful TFLOP/s counts the "
                     "completed POBTAFs of the iteration by the SURVEY §8(d) formula"}
    if cpu and n_gpus == 1:
        try:
            out["cpu_reference"] = cpu_c3_fobj()
        except Exception as exc:  # noqa: BLE001 -- the GPU line must still print
            out["cpu_reference"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


# --------------------------------------------------------------- GPU leg
def run_c5(args):
    """SPD BTA (96*N, b, a) of the reference generator's law,
    plan_partitions(96*N, N, lb), one partition per rank: every rank draws ONLY
    its own block rows in HBM (perf.device_random_spd_rows), then PPOBTAF,
    PPOBTAS (1 RHS) and PPOBTASI over NCCL.  value = the sequential routines'
    algorithmic FLOPs / the step's device time, max over ranks
    (useful throughput, weak scaling).  N = 1 runs the sequential routines."""
    import torch
    import torch.distributed as dist

    from paper_2507_06938_b200 import _lib, bta, bta_dist, perf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, b, a = 96 * world, args.b, args.a
    plan = bta_dist.plan_partitions(n, world, args.lb)
    t0, t1 = plan.boundaries[rank], plan.boundaries[rank + 1]
    rows = perf.device_random_spd_rows(n, b, a, t0, t1, seed=7, device=dev, with_tip=(rank == 0))
    g = torch.Generator(device=dev)
    g.manual_seed(11 + rank)
    rhs = torch.randn((t1 - t0) * b, dtype=torch.float64, device=dev, generator=g)
    rhs_tip = torch.randn(a, dtype=torch.float64, device=dev, generator=g) if rank == 0 else None
    if world == 1:
        full = bta.BTAMatrix(n, b, a, device=dev)
        bta_dist._rows_into(full, rows)
        if a:
            full.tip.copy_(rows.tip)
        del rows
    lib_count = _lib.load().stbta_launch_count

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(times=None):
        def mark(k, t):
            barrier()
            if times is not None:
                times[k] = times.get(k, 0.0) + time.perf_counter() - t
            return time.perf_counter()

        t = time.perf_counter()
        if world == 1:
            f = bta.factorize(full.copy())
            ld = bta.logdet(f)
            t = mark("pobtaf", t)
            bta.solve(f, torch.cat([rhs, rhs_tip]))
            t = mark("pobtas", t)
            bta.selected_invert(f)
            mark("pobtasi", t)
            return ld
        f = bta_dist.d_factorize_nccl(rows, plan)
        ld = bta_dist.d_logdet(f)
        t = mark("pobtaf", t)
        bta_dist.d_solve_nccl(f, rhs, rhs_tip)
        t = mark("pobtas", t)
        bta_dist.d_selected_invert_nccl(f)
        mark("pobtasi", t)
        return ld

    for _ in range(args.warmup):
        ld = step()
    barrier()
    times = {}
    c0 = lib_count()
    for _ in range(args.steps):
        ld = step(times)
    launches = lib_count() - c0
    el = {}
    for k, v in times.items():
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el[k] = float(t.item()) / args.steps
    fl = {"pobtaf": perf.flops_pobtaf(n, b, a), "pobtas": perf.flops_pobtas(n, b, a),
          "pobtasi": perf.flops_pobtasi(n, b, a)}
    tot = sum(el.values())
    if rank == 0:
        print(json.dumps({
            "metric": "distributed BTA useful FP64 TFLOP/s (C5: PPOBTAF+PPOBTAS+PPOBTASI)",
            "value": sum(fl.values()) / tot / 1e12, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic SPD BTA (reference generator law), each rank draws only its own "
                    "block rows in HBM",
            "config": {"workload": f"C5 n={n} (96 per GPU), b={b}, a={a}, P={world}, "
                                   f"lb={args.lb}", "boundaries": list(plan.boundaries)},
            "routines": {k: {"ms": 1e3 * el[k], "useful_tflops": fl[k] / el[k] / 1e12}
                         for k in el},
            "logdet": ld, "gpu_launches_per_rank": launches,
            "timing": "host wall clock between barriers + device syncs, max over ranks",
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn(args):
    """`bench.py --gpus N` without torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on this node and return its exit code; rank 0's JSON
    line goes straight to our stdout."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
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
    use_w = args.solve == "w"
    ws_s = torch.empty(lib.stbta_pobtas_w_workspace_bytes(n, b, a) if use_w else
                       lib.stbta_pobtas_workspace_bytes(n, b, a, 1), dtype=torch.uint8, device=dev)
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
        if use_w:  # W_t = L_tt^-1 once, shared by the solve and the selected inversion
            _lib.check(lib.stbta_pobtasi_prepare(_lib.ptr(mat.data), n, b, a, _lib.ptr(ws_i),
                                                 ws_i.numel(), sp), "pobtasi_prepare")
        if evs:
            evs[2].record(stream)
        x.copy_(rhs0)
        if use_w:
            _lib.check(lib.stbta_pobtas_w(_lib.ptr(mat.data), n, b, a, 1, _lib.ptr(x), 1, 0,
                                          _lib.ptr(ws_i), _lib.ptr(ws_s), ws_s.numel(), sp),
                       "pobtas_w")
        else:
            _lib.check(lib.stbta_pobtas(_lib.ptr(mat.data), n, b, a, 1, _lib.ptr(x), 1, 0,
                                        _lib.ptr(ws_s), ws_s.numel(), sp), "pobtas")
        if evs:
            evs[3].record(stream)
        if use_w:
            _lib.check(lib.stbta_pobtasi_prepared(_lib.ptr(mat.data), _lib.ptr(inv.data), None, n,
                                                  b, a, 1, _lib.ptr(ws_i), ws_i.numel(), sp, None),
                       "pobtasi_prepared")
        else:
            _lib.check(lib.stbta_pobtasi(_lib.ptr(mat.data), _lib.ptr(inv.data), n, b, a, 1,
                                         _lib.ptr(ws_i), ws_i.numel(), sp), "pobtasi")
        if evs:
            evs[4].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if int(info.item()) != 0:
        raise RuntimeError(f"POBTAF reported a non-SPD pivot (info={int(info.item())})")
    logdet_dev = float(ld[0].item())

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
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
    t_w = sum(e[1].elapsed_time(e[2]) for e in evs) * 1e-3 / args.steps  # W pass (w mode)
    t_s = sum(e[2].elapsed_time(e[3]) for e in evs) * 1e-3 / args.steps
    t_i = t_w + sum(e[3].elapsed_time(e[4]) for e in evs) * 1e-3 / args.steps
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
            if use_w:
                bta.prepare_inverse(fac)                           # W shared by solve + selinv
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
        try:
            c2 = CpuC2(n, b, a)
            secs, ld_cpu = c2.run()
            cpu = {"value": step_flops / secs / 1e12, "unit": UNIT, "cores": blas_threads(),
                   "kind": c2.kind, "sample": c2.sample(), "seconds": secs, "logdet": ld_cpu}
            del c2
        except Exception as exc:  # noqa: BLE001 -- the GPU line must still print
            cpu = {"error": f"{type(exc).__name__}: {exc}"}

    inla_obj = None
    if world > 1:
        # every rank's timed work is done; the C3 north-star iteration then
        # runs from rank 0 over all N GPUs of the run (ranks > 0 leave first)
        dist.barrier()
        dist.destroy_process_group()
        if rank != 0:
            return 0
    if rank == 0 and not args.no_inla:
        del pristine, ws_f, ws_s, ws_i
        torch.cuda.empty_cache()
        try:
            inla_obj = measure_north_star(world, peak, cpu=args.cpu_c3)
        except Exception as exc:  # noqa: BLE001 -- the C2 line must still print
            inla_obj = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        # roofline of the dominant routine (the longest launch chain of the step)
        dom = "pobtasi" if t_i > t_f else "pobtaf"
        achieved = (f_i / t_i if dom == "pobtasi" else f_f / t_f) / 1e12
        traffic = None
        tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")
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
                         "traffic_unit": "DRAM bytes per call (ncu --set full, profiles/r02_traffic.json)",
                         "peak_source": "FP64 DMMA.8x8x4 register-loop probe measured live "
                                        "(MEASURED_PEAKS.json has no FP64 entry)"},
            "routines": {
                "pobtaf": {"ms": 1e3 * t_f, "tflops": f_f / t_f / 1e12},
                "pobtas": {"ms": 1e3 * t_s, "gbs": perf.bytes_pobtas(n, b, a) / t_s / 1e9,
                           "frac_hbm": perf.bytes_pobtas(n, b, a) / t_s / 1e9 / HBM_GBS,
                           "kernel": "stbta_pobtas_w (block-inverse GEMVs, one cooperative "
                                     "launch)" if use_w else "stbta_pobtas (tile sweeps)"},
                "pobtasi": {"ms": 1e3 * t_i, "tflops": f_i / t_i / 1e12,
                            "w_prepass_ms": 1e3 * t_w if use_w else None},
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
