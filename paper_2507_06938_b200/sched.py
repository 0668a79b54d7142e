"""Layered worker allocation and deterministic task execution (S1/S2 layers).

Reference: pkg/src/stinla/sched.py — greedy g1*g2*g3 allocation, tasks dealt
round-robin (task i -> group i % g1), results gathered in index order, the
lowest failing index re-raised.  The B200 build keeps that policy and adds two
executors for the gradient layer (S1):

* :class:`GpuRunner` — one process driving several GPUs of a box, one host
  thread per GPU, each GPU evaluating its share through its own
  ObjectiveEvaluator (the device work releases the GIL); batches of at most G
  points go task i -> GPU i % G, larger ones through a cost-ordered queue.
* :class:`DistRunner` — one process per GPU (torchrun / NCCL): rank r evaluates
  tasks i with i % world == r, the scalar results are exchanged with one
  all-gather and every rank reassembles the identical list in index order,
  so each rank's optimizer takes bit-identical decisions.
"""

import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


class TaskError(RuntimeError):
    """A task failed; carries the lowest failing task index (sched.py:18-23)."""

    def __init__(self, task_index, message):
        self.task_index = task_index
        super().__init__(f"task {task_index} failed: {message}")


def n_objective_tasks(dim_theta):
    return 2 * dim_theta + 1


@dataclass(frozen=True)
class LayerAllocation:
    """g1 evaluation groups, g2 in {1,2} precision-pair width, g3 partitions (sched.py:31-48)."""

    workers: int
    g1: int
    g2: int
    g3: int

    def __post_init__(self):
        if self.g1 * self.g2 * self.g3 > self.workers:
            raise ValueError("allocation exceeds the worker pool")
        if self.g2 not in (1, 2):
            raise ValueError("the precision-pair layer is at most two wide")

    def saturated_s1(self, dim_theta):
        return self.g1 >= n_objective_tasks(dim_theta)


def allocate(workers, dim_theta, memory_fits_single=True, min_partitions=2):
    """Greedy S1 -> S2 -> S3 allocation (sched.py:51-68)."""
    if workers < 1:
        raise ValueError("at least one worker required")
    n_eval = n_objective_tasks(dim_theta)
    g3 = 1 if memory_fits_single else max(1, min(min_partitions, workers))
    g1 = max(1, min(n_eval, workers // g3))
    g2 = 2 if (g1 >= n_eval and workers // (g1 * g3) >= 2) else 1
    g3 = max(g3, workers // (g1 * g2))
    return LayerAllocation(workers=workers, g1=g1, g2=g2, g3=g3)


@dataclass
class TaskTrace:
    index: int
    group: int
    round: int
    start: float
    stop: float


def _run_groups(tasks, groups, call):
    """Deal task i to group i % groups; returns (results, failures, records)."""
    results = [None] * len(tasks)
    failures = []

    def worker(g):
        recs = []
        for rnd, idx in enumerate(range(g, len(tasks), groups)):
            t0 = time.perf_counter()
            try:
                results[idx] = call(g, idx)
            except Exception as exc:  # reported with its task index
                failures.append((idx, exc))
                return recs
            recs.append(TaskTrace(idx, g, rnd, t0, time.perf_counter()))
        return recs

    if groups == 1:
        recs = worker(0)
    else:
        with ThreadPoolExecutor(max_workers=groups) as pool:
            recs = [r for rs in pool.map(worker, range(groups)) for r in rs]
    return results, failures, recs


def run_tasks(tasks, alloc=None, trace=None):
    """Zero-argument tasks, results in index order (sched.py:82-123)."""
    tasks = list(tasks)
    if not tasks:
        return []
    groups = 1 if alloc is None else max(1, min(alloc.g1, len(tasks)))
    results, failures, recs = _run_groups(tasks, groups, lambda g, i: tasks[i]())
    if failures:
        idx, exc = min(failures, key=lambda p: p[0])
        raise TaskError(idx, str(exc)) from exc
    if trace is not None:
        trace.extend(sorted(recs, key=lambda r: r.index))
    return results


class TaskRunner:
    """Allocation-bound task hook for the inference routines (sched.py:126-135)."""

    def __init__(self, alloc=None, trace=None):
        self.alloc = alloc
        self.trace = trace

    def __call__(self, tasks):
        return run_tasks(tasks, self.alloc, self.trace)


def pair_runner(alloc):
    """Two-wide runner for the Q_p / Q_c pair, or None (sched.py:138-144).  On the
    device the pair already runs on two CUDA streams inside one evaluation."""
    if alloc is None or alloc.g2 < 2:
        return None
    return TaskRunner(LayerAllocation(workers=2, g1=2, g2=1, g3=1))


class GpuRunner:
    """S1 over the GPUs of one process: theta-point tasks are re-bound to the
    evaluator of GPU (i % G) and run by one host thread per GPU.

    ``evaluators[g]`` is an ObjectiveEvaluator on GPU g.  The runner is called
    by :func:`inla.fd_gradient` / ``minimize`` / ``fd_hessian`` with tasks
    tagged with their point and function (``inla._run``).  When the function
    is the negated objective of an evaluator equivalent to the runner's (same
    model spec, prior and variance calibration -- every f_obj is then the same
    bits on any of them), each point is re-bound to the evaluator of GPU
    (i % G) and ``-evaluators[g].objective(p)`` is evaluated there; any other
    task is simply called, one thread per GPU, so a user callable is never
    replaced.  Per GPU the tasks are issued ``depth`` at a time so several
    f_obj overlap on the device.
    """

    def __init__(self, evaluators, negate=True, trace=None, depth=1, split_pairs=True):
        self.evaluators = list(evaluators)
        self.negate = negate
        self.trace = trace
        self.depth = max(1, int(depth))
        # S2 across GPUs: a batch of at most G/2 points (the line search) runs
        # each f_obj on a GPU pair -- Q_p's factorization on one, Q_c's chain
        # on the other -- halving its latency; bigger batches (the gradient)
        # run one f_obj per GPU.
        self.split_pairs = bool(split_pairs) and len(self.evaluators) >= 2
        # one long-lived worker thread per GPU, always driving the same
        # evaluator: workspace slots are keyed by thread, so fresh (or
        # rotating) threads would allocate fresh Q_p / Q_c workspaces
        self._pools = None
        self.dispatch_log = None  # list: queue dispatch order (tests)

    @property
    def width(self):
        """Line-search candidates per round: one per GPU pair when f_obj is
        split across a pair, else one per GPU."""
        G = len(self.evaluators)
        return G // 2 if self.split_pairs else G

    def close(self):
        for p in self._pools or []:
            p.shutdown(wait=True)
        self._pools = None

    def _compatible(self, ev):
        """Does evaluator ``ev`` compute the same f_obj as the runner's?"""
        if any(ev is e for e in self.evaluators):
            return True
        ref = self.evaluators[0]
        try:
            return (ev.spec is ref.spec
                    and np.array_equal(ev.prior.mean, ref.prior.mean)
                    and np.array_equal(ev.prior.sd, ref.prior.sd)
                    and np.array_equal(ev.calibration, ref.calibration))
        except AttributeError:
            return False

    def _points(self, tasks):
        """The tasks' points when every task is a tagged negated objective of
        an equivalent evaluator (and the runner negates), else None."""
        if not self.negate:
            return None
        pts = []
        for t in tasks:
            p = getattr(t, "stbta_point", None)
            ev = getattr(getattr(t, "stbta_fun", None), "stbta_evaluator", None)
            if p is None or ev is None or not self._compatible(ev):
                return None
            pts.append(np.asarray(p, dtype=np.float64))
        return pts

    def _pools_ready(self, G):
        if self._pools is None:
            self._pools = [ThreadPoolExecutor(max_workers=1) for _ in range(G)]

    def _evaluate_split(self, points):
        """Point k: prior half on GPU 2k (published through the shared prior
        cache), conditional half on GPU 2k+1, which assembles f."""
        G = len(self.evaluators)
        sign = -1.0 if self.negate else 1.0
        out = [None] * len(points)
        self._pools_ready(G)

        def prior(k):
            self.evaluators[2 * k].prior_logdet(points[k])

        def cond(k):
            ev = self.evaluators[2 * k + 1]
            out[k] = sign * ev.collect(ev.launch(points[k], defer_prior=True))[0]

        futs = []
        for k in range(len(points)):
            futs.append(self._pools[2 * k].submit(prior, k))
            futs.append(self._pools[2 * k + 1].submit(cond, k))
        errors = []
        for i, f in enumerate(futs):
            try:
                f.result()
            except Exception as exc:  # report the lowest failing point
                errors.append((i // 2, exc))
        if errors:
            idx, exc = min(errors, key=lambda p: p[0])
            raise TaskError(idx, str(exc)) from exc
        return out

    def evaluate_points(self, points):
        G = len(self.evaluators)
        if self.split_pairs and 0 < len(points) <= G // 2:
            return self._evaluate_split(points)
        sign = -1.0 if self.negate else 1.0
        out = [None] * len(points)
        failures = []

        if G > 1 and self.depth == 1 and len(points) > G:
            return self._evaluate_queue(points)

        def worker(g):
            ev = self.evaluators[g]
            mine = list(range(g, len(points), G))
            for k in range(0, len(mine), self.depth):
                batch = mine[k : k + self.depth]
                slots = [ev.slot(j) for j in range(len(batch))] if self.depth > 1 else [None]
                handles = []
                for i, s in zip(batch, slots):
                    try:
                        handles.append((i, ev.launch(points[i], slot=s)))
                    except Exception as exc:  # the index that actually failed
                        failures.append((i, exc))
                        break
                for i, h in handles:
                    try:
                        out[i] = sign * ev.collect(h)[0]
                    except Exception as exc:
                        failures.append((i, exc))
                if failures:
                    return

        if G == 1:
            worker(0)
        else:
            self._pools_ready(G)
            futs = [self._pools[g].submit(worker, g) for g in range(G)]
            for f in futs:
                f.result()
        if failures:
            idx, exc = min(failures, key=lambda p: p[0])
            raise TaskError(idx, str(exc)) from exc
        return out

    def _evaluate_queue(self, points):
        """Batches larger than G (the gradient stencil): one shared queue,
        longest tasks first.  Points whose log det Q_p is already cached (the
        stencil's noise-precision moves) cost about half an f_obj, so they go
        last and fill the GPUs that finish their full evaluations first.
        Every f_obj is a deterministic function of its point on any of the
        (identical) GPUs, so results are the same bits as the static i % G
        assignment; only the makespan changes (31 points on 8 GPUs: 5 -> 4.5
        full-f_obj rounds)."""
        G = len(self.evaluators)
        sign = -1.0 if self.negate else 1.0
        out = [None] * len(points)
        failures = []
        probe = getattr(self.evaluators[0], "prior_cached", None)
        cheap = [bool(probe(p)) if probe else False for p in points]
        order = sorted(range(len(points)), key=lambda i: (cheap[i], i))
        lock = threading.Lock()
        nxt = [0]

        def worker(g):
            ev = self.evaluators[g]
            while True:
                with lock:
                    if nxt[0] >= len(order):
                        return
                    i = order[nxt[0]]
                    nxt[0] += 1
                    if self.dispatch_log is not None:
                        self.dispatch_log.append(i)
                try:
                    out[i] = sign * ev.collect(ev.launch(points[i]))[0]
                except Exception as exc:  # keep going: the lowest failing index is raised
                    with lock:
                        failures.append((i, exc))

        self._pools_ready(G)
        futs = [self._pools[g].submit(worker, g) for g in range(G)]
        for f in futs:
            f.result()
        if failures:
            idx, exc = min(failures, key=lambda p: p[0])
            raise TaskError(idx, str(exc)) from exc
        return out

    def __call__(self, tasks):
        tasks = list(tasks)
        pts = self._points(tasks)
        if pts is not None:
            return self.evaluate_points(pts)
        G = len(self.evaluators)
        return run_tasks(tasks, LayerAllocation(workers=G, g1=G, g2=1, g3=1))


class DistRunner:
    """S1 across processes (one per GPU): rank r evaluates tasks i % world == r,
    results are all-gathered and returned in index order on every rank."""

    def __init__(self, evaluator, group=None, negate=True):
        import torch.distributed as dist

        self.dist = dist
        self.evaluator = evaluator
        self.group = group
        self.negate = negate
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    @property
    def width(self):
        return self.world

    def _run_mine(self, n, call):
        """Run this rank's indices (i % world == rank) through call(i); values
        and failure flags are all-gathered, results returned in index order
        on every rank, and a failure anywhere raises the same TaskError (the
        lowest failing index) on every rank."""
        import torch

        local = torch.full((2, n), float("nan"), dtype=torch.float64)
        local[1].zero_()
        errors = {}
        for i in range(self.rank, n, self.world):
            try:
                local[0, i] = call(i)
            except Exception as exc:  # published, raised below on every rank
                local[1, i] = 1.0
                errors[i] = exc
        backend = self.dist.get_backend(self.group)
        dev = self.evaluator.device if backend == "nccl" else torch.device("cpu")
        buf = local.to(dev)
        gathered = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(gathered, buf, group=self.group)
        out, failed = np.empty(n), np.zeros(n, dtype=bool)
        for r in range(self.world):
            g = gathered[r].cpu().numpy()
            out[r::self.world] = g[0, r::self.world]
            failed[r::self.world] = g[1, r::self.world] != 0
        if failed.any():
            idx = int(np.flatnonzero(failed)[0])
            exc = errors.get(idx)
            raise TaskError(idx, str(exc) if exc else "failed on another rank") from exc
        return out.tolist()

    def evaluate_points(self, points):
        sign = -1.0 if self.negate else 1.0
        return self._run_mine(len(points),
                              lambda i: sign * self.evaluator.objective(points[i]))

    def __call__(self, tasks):
        """Each rank calls its own tasks (i % world == rank): every task is a
        deterministic function of its point, so no re-binding is needed."""
        tasks = list(tasks)
        return self._run_mine(len(tasks), lambda i: float(tasks[i]()))
