"""Time-partitioned BTA solver (S3): PPOBTAF / PPOBTAS / PPOBTASI on B200.

Mirror of the reference ``stinla.bta_dist`` (pkg/src/stinla/bta_dist.py):
same plan (``plan_partitions``, bta_dist.py:65-112), separators
(bta_dist.py:257-265), error tagging and results, re-designed around the
device kernels:

* A partition's interior is eliminated by ONE partial POBTAF
  (``stbta_pobtaf_ex`` with ``nfact``) on an *extended chain*: the interior
  blocks, then the right separator as a last ordinary block, and an arrowhead
  made of the left separator's rows stacked on the true arrow rows.  The
  elimination leaves exactly the reference's Schur contributions in the
  unfactored parts (bta_dist.py:174-254): d_right/f_right in the last block,
  fill in its left-separator arrow rows, d_left/f_left/d_tip in the extended
  tip.
* The reduced 2(P-1)-block BTA (bta_dist.py:322-350) is assembled in
  partition order on the root device and factorized by POBTAF.
* ``d_solve`` is a Schur-complement solve: two interior solves per partition
  (POBTAS on the interior view of the chain factor) around one reduced solve.
* ``d_selected_invert`` seeds each chain's inverse with the reduced selected
  inverse (separator, fill and tip entries) and continues the POBTASI
  recursion over the interior (``stbta_pobtasi_ex`` with ``nstart``), which is
  the reference's three-term interior recursion (bta_dist.py:508-602).

Partitions may live on different GPUs of one process (``devices``; a mapper
runs them concurrently), or one per rank under torchrun:
``d_factorize_nccl`` ships the chains and Schur pieces point-to-point over
NCCL (NVLink) and factorizes the reduced system on the root.
"""

import time
import warnings
from concurrent.futures import ThreadPoolExecutor
from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import bta
from .bta import BTAMatrix, FactorizationError


class PlanError(ValueError):
    """The requested (n, P) partitioning is infeasible (bta_dist.py:41-42)."""


@dataclass(frozen=True)
class PartitionPlan:
    """Deterministic slicing of the time-block chain (bta_dist.py:45-62)."""

    n_blocks: int
    boundaries: tuple
    lb: float

    @property
    def n_partitions(self):
        return len(self.boundaries) - 1

    @property
    def sizes(self):
        return tuple(self.boundaries[p + 1] - self.boundaries[p] for p in range(self.n_partitions))


def plan_partitions(n_blocks, n_partitions, lb=1.0):
    """Near-even split (remainder from the front); ``lb > 1`` enlarges the first
    partition to floor(lb*n/(P-1+lb)), clamped to keep >= 2 blocks per partition
    (bta_dist.py:65-98)."""
    if n_partitions < 1:
        raise PlanError("at least one partition required")
    if lb < 1.0:
        raise PlanError("load-balance factor must be >= 1")
    if n_partitions == 1:
        if n_blocks < 1:
            raise PlanError("empty matrix")
        return PartitionPlan(n_blocks, (0, n_blocks), lb)
    if n_blocks < 2 * n_partitions:
        raise PlanError(
            f"{n_partitions} partitions require at least {2 * n_partitions} time blocks, "
            f"got {n_blocks}"
        )
    if lb == 1.0:
        q, r = divmod(n_blocks, n_partitions)
        sizes = [q + 1] * r + [q] * (n_partitions - r)
    else:
        first = int(np.floor(lb * n_blocks / (n_partitions - 1 + lb)))
        first = max(2, min(first, n_blocks - 2 * (n_partitions - 1)))
        q, r = divmod(n_blocks - first, n_partitions - 1)
        sizes = [first] + [q + 1] * r + [q] * (n_partitions - 1 - r)
    bounds = [0]
    for s in sizes:
        bounds.append(bounds[-1] + s)
    return PartitionPlan(n_blocks, tuple(bounds), lb)


def plan_partitions_with_fallback(n_blocks, n_partitions, lb=1.0):
    """Reduce the partition count (with a warning) when infeasible (bta_dist.py:101-112)."""
    feasible = max(1, min(n_partitions, n_blocks // 2))
    if feasible != n_partitions:
        warnings.warn(
            f"reducing partitions from {n_partitions} to {feasible} ({n_blocks} time blocks)",
            stacklevel=2,
        )
    return plan_partitions(n_blocks, feasible, lb)


@contextmanager
def _phase(phase_times, name):
    """Wall-time accumulator (bta_dist.py:28-38); synchronises the device."""
    if phase_times is None:
        yield
        return
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        yield
    finally:
        torch.cuda.synchronize()
        phase_times[name] = phase_times.get(name, 0.0) + time.perf_counter() - t0


def _separators(plan):
    seps = []
    for p in range(plan.n_partitions):
        if p > 0:
            seps.append(plan.boundaries[p])
        if p < plan.n_partitions - 1:
            seps.append(plan.boundaries[p + 1] - 1)
    return seps


def _partition_ranges(plan):
    """(lo, hi, left, right) of each partition's interior (bta_dist.py:268-279)."""
    out = []
    P = plan.n_partitions
    for p in range(P):
        start, end = plan.boundaries[p], plan.boundaries[p + 1]
        lo = start + 1 if p > 0 else start
        hi = end - 1 if p < P - 1 else end
        out.append((lo, hi, start if p > 0 else None, end - 1 if p < P - 1 else None))
    return out


class _Chain:
    """Extended chain of one partition on its device: interior blocks
    [lo, hi), then the right separator block (if any); arrowhead rows =
    [left separator (b rows, if any); true arrow (a rows)]."""

    def __init__(self, index, lo, hi, left, right, b, a, use_arrow, device):
        self.index, self.lo, self.hi, self.left, self.right = index, lo, hi, left, right
        self.b, self.a = b, a
        self.n_int = hi - lo
        self.n_ext = self.n_int + (1 if right is not None else 0)
        self.off = b if left is not None else 0  # first true-arrow row in the arrowhead
        self.ap = self.off + a
        self.use_arrow = use_arrow
        self.chain_arrow = (left is not None) or use_arrow
        self.device = device
        f64 = dict(dtype=torch.float64, device=device)
        n = max(self.n_ext, 1)
        self.diag = torch.empty(n, b, b, **f64)
        self.lower = torch.empty(max(self.n_ext - 1, 1), b, b, **f64)
        self.arrow = torch.zeros(n, max(self.ap, 1), b, **f64)
        self.tip = torch.zeros(max(self.ap, 1), max(self.ap, 1), **f64)
        self.logdet_dev = torch.zeros(1, dtype=torch.float64, device=device)
        self.info = torch.zeros(1, dtype=torch.int32, device=device)
        self.logdet = 0.0

    @property
    def interior_count(self):
        return self.n_int

    def load(self, M):
        """Copy this partition's blocks out of the global matrix M (any device)."""
        lo, hi, ni = self.lo, self.hi, self.n_int
        dev = self.device
        self.diag[:ni].copy_(M.diag[lo:hi].to(dev, non_blocking=True))
        if ni > 1:
            self.lower[: ni - 1].copy_(M.lower[lo : hi - 1].to(dev, non_blocking=True))
        if self.right is not None:
            self.diag[ni].copy_(M.diag[hi].to(dev, non_blocking=True))
            if ni > 0:
                self.lower[ni - 1].copy_(M.lower[hi - 1].to(dev, non_blocking=True))
        if self.left is not None and ni > 0:
            self.arrow[0, : self.b].copy_(M.lower[lo - 1].to(dev, non_blocking=True).T)
        if self.a > 0 and self.use_arrow:
            self.arrow[:ni, self.off :].copy_(M.arrow[lo:hi].to(dev, non_blocking=True))
            if self.right is not None:
                self.arrow[ni, self.off :].copy_(M.arrow[hi].to(dev, non_blocking=True))

    def regions(self):
        return [_lib.ptr(self.diag), _lib.ptr(self.lower), _lib.ptr(self.arrow), _lib.ptr(self.tip)]

    def last_diag(self):
        """Right separator block after the elimination (its reduced diagonal)."""
        return self.diag[self.n_int]

    def last_arrow(self):
        """Arrowhead rows of the right separator block ([fill; f_right])."""
        return self.arrow[self.n_int]

    def eliminate(self):
        """Partial POBTAF: factor the interior, leave the Schur pieces."""
        if self.n_int == 0:
            return
        lib = _lib.load()
        with torch.cuda.device(self.device):
            ws = torch.empty(lib.stbta_pobtaf_workspace_bytes(self.n_ext, self.b, self.ap),
                             dtype=torch.uint8, device=self.device)
            d, l, ar, tp = self.regions()
            _lib.check(
                lib.stbta_pobtaf_ex(d, l, ar, tp, self.n_ext, self.b, self.ap, self.b,
                                    int(self.chain_arrow), self.n_int, _lib.ptr(self.logdet_dev),
                                    _lib.ptr(self.info), _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr()),
                "stbta_pobtaf_ex",
            )
            code = int(self.info.item())
            if code:
                raise FactorizationError(self.lo + code - 1, partition=self.index)
            self.logdet = float(self.logdet_dev.item())

    def interior_solve(self, rhs):
        """In place: rhs (n_int*b, k) := A_int^{-1} rhs with the interior factor."""
        lib = _lib.load()
        n, b = self.n_int, self.b
        k = rhs.shape[1]
        with torch.cuda.device(self.device):
            ws = torch.empty(lib.stbta_pobtas_workspace_bytes(n, b, 0, k), dtype=torch.uint8,
                             device=self.device)
            _lib.check(
                lib.stbta_pobtas_ex(_lib.ptr(self.diag), _lib.ptr(self.lower), None, None, n, b, 0,
                                    b, 0, _lib.ptr(rhs), k, 0, _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr()),
                "stbta_pobtas_ex",
            )
        return rhs


def _sym_lower(x):
    """Full symmetric matrix from the lower triangle of x."""
    return torch.tril(x) + torch.tril(x, -1).T


class DistBTAFactor:
    """Partition chains plus the factorized reduced system (bta_dist.py:143-166)."""

    def __init__(self, plan, matrix, partitions, reduced_factor, separators, use_arrow=False):
        self.plan = plan
        self.n_blocks, self.block_size, self.arrow_size = (
            plan.n_blocks, matrix.block_size, matrix.arrow_size)
        self.matrix = matrix  # the (unmodified) input, used by d_solve's couplings
        self.partitions = partitions
        self.reduced_factor = reduced_factor
        self.separators = separators
        self.sep_pos = {t: k for k, t in enumerate(separators)}
        self._use_arrow = use_arrow
        self.sequential = None

    @property
    def dim(self):
        return self.n_blocks * self.block_size + self.arrow_size

    @property
    def has_arrow(self):
        if self.sequential is not None:
            return self.sequential.has_arrow
        return self._use_arrow


def _default_mapper(devices):
    if devices is None or len(set(str(d) for d in devices)) <= 1:
        return None

    def mapper(fn, items):
        with ThreadPoolExecutor(max_workers=len(items)) as pool:
            return list(pool.map(fn, items))

    return mapper


def _charge(counter, units, times=1):
    if counter is not None:
        for _ in range(times):
            counter.charge(units)


def d_factorize(matrix, plan, counter=None, mapper=None, phase_times=None, devices=None):
    """Partitioned block Cholesky (bta_dist.py:282-359).

    ``matrix`` is read only for P > 1 (factorized in place for P == 1, like the
    reference).  ``devices[p % len(devices)]`` hosts partition p; the reduced
    system lives on the matrix's device.  Results are combined in partition
    order, independent of the mapper.
    """
    if plan.n_blocks != matrix.n_blocks:
        raise PlanError("plan does not match the matrix block count")
    if plan.n_partitions == 1:
        with _phase(phase_times, "total"):
            factor = bta.factorize(matrix, counter=counter)
        dist = DistBTAFactor(plan, matrix, [], None, [])
        dist.sequential = factor
        return dist

    b, a = matrix.block_size, matrix.arrow_size
    use_arrow = bta._arrow_nonzero(matrix)
    devices = list(devices) if devices else [matrix.device]
    chains = [
        _Chain(p, lo, hi, left, right, b, a, use_arrow, torch.device(devices[p % len(devices)]))
        for p, (lo, hi, left, right) in enumerate(_partition_ranges(plan))
    ]
    mapper = mapper or _default_mapper(devices)

    def job(ch):
        with torch.cuda.device(ch.device):
            ch.load(matrix)
            ch.eliminate()
        return ch

    with _phase(phase_times, "eliminate"):
        chains = [job(c) for c in chains] if mapper is None else list(mapper(job, chains))
    for ch in chains:  # modeled cost units, as the reference (bta_dist.py:220-225)
        _charge(counter, b**3, ch.n_int * (2 if ch.left is not None else 1))
        if use_arrow:
            _charge(counter, a**3, ch.n_int)

    seps = _separators(plan)
    with _phase(phase_times, "reduced"):
        reduced_factor = _reduce_and_factorize(matrix, plan, chains, use_arrow, counter)
    return DistBTAFactor(plan, matrix, chains, reduced_factor, seps, use_arrow)


def _reduce_and_factorize(matrix, plan, pieces, use_arrow, counter=None):
    """Reduced 2(P-1)-block BTA over the separators from the original blocks
    plus each partition's Schur pieces, summed in partition order
    (bta_dist.py:322-350), factorized on the matrix's device.  ``pieces`` are
    chains (or received copies) exposing n_int, off, left, right, tip, and the
    last block's diag / arrow."""
    b, a = matrix.block_size, matrix.arrow_size
    seps = _separators(plan)
    dev = matrix.device
    n_red = len(seps)
    with torch.cuda.device(dev):
        red = BTAMatrix(n_red, b, a, device=dev)
        for k, t in enumerate(seps):
            red.diag[k].copy_(matrix.diag[t])
            if use_arrow:
                red.arrow[k].copy_(matrix.arrow[t])
        for k in range(n_red - 1):
            if seps[k + 1] == seps[k] + 1:
                red.lower[k].copy_(matrix.lower[seps[k]])
        if a > 0:
            red.tip.copy_(matrix.tip)
        sp = {t: k for k, t in enumerate(seps)}
        for ch in pieces:  # partition order
            if ch.n_int == 0:
                continue
            o = ch.off
            if ch.left is not None:
                pos = sp[ch.left]
                red.diag[pos] += _sym_lower(ch.tip[:b, :b]).to(dev)
                if use_arrow:
                    red.arrow[pos] += ch.tip[o:, :b].to(dev)
            if ch.right is not None:
                pos = sp[ch.right]
                red.diag[pos].copy_(_sym_lower(ch.last_diag()).to(dev))
                if use_arrow:
                    red.arrow[pos].copy_(ch.last_arrow()[o:].to(dev))
                if ch.left is not None:
                    red.lower[sp[ch.left]].copy_(ch.last_arrow()[:b].T.to(dev))
            if use_arrow:
                red.tip += _sym_lower(ch.tip[o:, o:]).to(dev)
        try:
            return bta.factorize(red, counter=counter, use_arrow=use_arrow)
        except FactorizationError as err:
            raise FactorizationError(seps[min(err.block_index, n_red - 1)], partition=-1) from None


class _Pieces:
    """Schur pieces of a remote partition, received by the root."""

    def __init__(self, ch, device):
        self.index, self.left, self.right = ch.index, ch.left, ch.right
        self.n_int, self.off, self.b = ch.n_int, ch.off, ch.b
        f64 = dict(dtype=torch.float64, device=device)
        self.tip = torch.empty_like(ch.tip, device=device)
        self._diag = torch.empty(ch.b, ch.b, **f64) if ch.right is not None else None
        self._arrow = torch.empty(ch.arrow.shape[1], ch.b, **f64) if ch.right is not None else None
        self.logdet = 0.0

    def last_diag(self):
        return self._diag

    def last_arrow(self):
        return self._arrow


def d_factorize_nccl(matrix, plan, group=None, root=0):
    """PPOBTAF with one partition per rank (torchrun, NCCL over NVLink).

    ``matrix`` (a BTAMatrix) is needed on ``root`` only; the other ranks pass
    None.  The root ships each partition's extended chain to its rank
    (point-to-point), every rank eliminates its interior concurrently, the
    Schur pieces come back to the root, which assembles and factorizes the
    reduced system in partition order.  Returns ``(logdet, chain)`` on every
    rank (logdet broadcast from the root); a non-SPD pivot raises the same
    FactorizationError on every rank.
    """
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if plan.n_partitions != world:
        raise PlanError(f"plan has {plan.n_partitions} partitions for {world} ranks")
    dev = torch.device("cuda", torch.cuda.current_device())
    if world == 1:  # sequential delegation on a copy (the input stays read-only)
        f = bta.factorize(matrix.copy())
        return bta.logdet(f), None
    meta = torch.zeros(4, dtype=torch.int64, device=dev)
    if rank == root:
        meta[:] = torch.tensor([matrix.n_blocks, matrix.block_size, matrix.arrow_size,
                                int(bta._arrow_nonzero(matrix))], device=dev)
    dist.broadcast(meta, root, group=group)
    n, b, a, use_arrow = (int(x) for x in meta.tolist())
    if plan.n_blocks != n:
        raise PlanError("plan does not match the matrix block count")
    ranges = _partition_ranges(plan)
    chains = {}
    if rank == root:  # build and ship every chain, keep our own
        for p, (lo, hi, left, right) in enumerate(ranges):
            ch = _Chain(p, lo, hi, left, right, b, a, bool(use_arrow), dev)
            ch.load(matrix)
            if p == rank:
                chains[p] = ch
            else:
                for t in (ch.diag, ch.lower, ch.arrow):
                    dist.send(t, p, group=group)
                del ch
    else:
        lo, hi, left, right = ranges[rank]
        ch = _Chain(rank, lo, hi, left, right, b, a, bool(use_arrow), dev)
        for t in (ch.diag, ch.lower, ch.arrow):
            dist.recv(t, root, group=group)
        chains[rank] = ch
    mine = chains[rank]
    err = torch.zeros(2, dtype=torch.int64, device=dev)
    try:
        mine.eliminate()
    except FactorizationError as e:
        err[:] = torch.tensor([1, e.block_index], device=dev)
    errs = [torch.zeros_like(err) for _ in range(world)]
    dist.all_gather(errs, err, group=group)
    for p, e in enumerate(errs):
        if int(e[0]):
            raise FactorizationError(int(e[1]), partition=p)
    # Schur pieces to the root
    ld = torch.tensor([mine.logdet], dtype=torch.float64, device=dev)
    if rank != root:
        dist.send(ld, root, group=group)
        dist.send(mine.tip, root, group=group)
        if mine.right is not None:
            dist.send(mine.last_diag().contiguous(), root, group=group)
            dist.send(mine.last_arrow().contiguous(), root, group=group)
        total = torch.zeros(1, dtype=torch.float64, device=dev)
        dist.broadcast(total, root, group=group)
        return float(total.item()), mine
    pieces = []
    interior = 0.0
    for p, (lo, hi, left, right) in enumerate(ranges):
        if p == rank:
            pieces.append(mine)
            interior += mine.logdet
            continue
        stub = _Chain.__new__(_Chain)
        stub.index, stub.lo, stub.hi, stub.left, stub.right = p, lo, hi, left, right
        stub.b, stub.n_int = b, hi - lo
        stub.off = b if left is not None else 0
        stub.tip = mine.tip.new_empty((max(stub.off + a, 1), max(stub.off + a, 1)))
        stub.arrow = mine.arrow.new_empty((1, max(stub.off + a, 1), b))
        pc = _Pieces(stub, dev)
        buf = torch.zeros(1, dtype=torch.float64, device=dev)
        dist.recv(buf, p, group=group)
        pc.logdet = float(buf.item())
        interior += pc.logdet
        dist.recv(pc.tip, p, group=group)
        if right is not None:
            dist.recv(pc._diag, p, group=group)
            dist.recv(pc._arrow, p, group=group)
        pieces.append(pc)
    reduced = _reduce_and_factorize(matrix, plan, pieces, bool(use_arrow))
    total = torch.tensor([interior + bta.logdet(reduced)], dtype=torch.float64, device=dev)
    dist.broadcast(total, root, group=group)
    return float(total.item()), mine


def d_logdet(factor):
    """Interior log-dets plus the reduced system's (bta_dist.py:362-367)."""
    if factor.sequential is not None:
        return bta.logdet(factor.sequential)
    return sum(ch.logdet for ch in factor.partitions) + bta.logdet(factor.reduced_factor)


def d_solve(factor, rhs, counter=None, phase_times=None):
    """Partitioned solve (bta_dist.py:370-458) as a Schur-complement solve."""
    if factor.sequential is not None:
        with _phase(phase_times, "total"):
            return bta.solve(factor.sequential, rhs, counter=counter)
    M = factor.matrix
    b, a, n = factor.block_size, factor.arrow_size, factor.n_blocks
    dev = M.device
    host = not isinstance(rhs, torch.Tensor)
    if host:
        x = torch.from_numpy(np.array(rhs, dtype=np.float64, copy=True)).to(dev)
    else:
        x = rhs.detach().to(device=dev, dtype=torch.float64).clone()
    if x.dim() == 0 or x.shape[0] != factor.dim:
        raise ValueError(f"rhs has length {x.shape[0] if x.dim() else 0}, expected {factor.dim}")
    squeeze = x.dim() == 1
    X = x.reshape(factor.dim, -1)
    k = X.shape[1]
    use_arrow = factor.has_arrow
    seps, sp = factor.separators, factor.sep_pos
    n_red = len(seps)

    def blk(t):
        return slice(t * b, (t + 1) * b)

    red_rhs = torch.zeros(n_red * b + a, k, dtype=torch.float64, device=dev)
    for kk, t in enumerate(seps):
        red_rhs[kk * b : (kk + 1) * b] = X[blk(t)]
    if a > 0:
        red_rhs[n_red * b :] = X[n * b :]

    zs = []
    with _phase(phase_times, "forward"):
        for ch in factor.partitions:
            if ch.n_int == 0:
                zs.append(None)
                continue
            z = X[ch.lo * b : ch.hi * b].to(ch.device).contiguous()
            ch.interior_solve(z)
            zd = z.to(dev)
            zs.append(zd)
            if ch.left is not None:  # A(left, lo) = lower[lo-1]^T
                red_rhs[blk(sp[ch.left])] -= M.lower[ch.lo - 1].T @ zd[:b]
            if ch.right is not None:  # A(right, hi-1) = lower[hi-1]
                red_rhs[blk(sp[ch.right])] -= M.lower[ch.hi - 1] @ zd[-b:]
            if use_arrow:
                ar = M.arrow[ch.lo : ch.hi]  # (n_int, a, b)
                red_rhs[n_red * b :] -= torch.einsum("jtb,jbk->tk", ar, zd.view(ch.n_int, b, k))
            _charge(counter, b**2, ch.n_int)

    with _phase(phase_times, "reduced"):
        red_x = bta.solve(factor.reduced_factor, red_rhs, counter=counter)
    for kk, t in enumerate(seps):
        X[blk(t)] = red_x[kk * b : (kk + 1) * b]
    if a > 0:
        X[n * b :] = red_x[n_red * b :]
    x_tip = X[n * b :]

    with _phase(phase_times, "backward"):
        for ch, zd in zip(factor.partitions, zs):
            if zd is None:
                continue
            w = torch.zeros(ch.n_int * b, k, dtype=torch.float64, device=dev)
            if ch.left is not None:
                w[:b] += M.lower[ch.lo - 1] @ X[blk(ch.left)]
            if ch.right is not None:
                w[-b:] += M.lower[ch.hi - 1].T @ X[blk(ch.right)]
            if use_arrow:
                w += torch.einsum("jtb,tk->jbk", M.arrow[ch.lo : ch.hi], x_tip).reshape(-1, k)
            wd = w.to(ch.device).contiguous()
            ch.interior_solve(wd)
            X[ch.lo * b : ch.hi * b] = zd - wd.to(dev)
            _charge(counter, b**2, ch.n_int)
    out = x if not squeeze else X.reshape(-1)
    return out.cpu().numpy() if host else out


def d_selected_invert(factor, counter=None, mapper=None, phase_times=None):
    """Pattern entries of the inverse (bta_dist.py:461-505): reduced selected
    inverse, then each chain's POBTASI recursion seeded with it."""
    if factor.sequential is not None:
        with _phase(phase_times, "total"):
            return bta.selected_invert(factor.sequential, counter=counter)
    lib = _lib.load()
    M = factor.matrix
    n, b, a = factor.n_blocks, factor.block_size, factor.arrow_size
    dev = M.device
    use_arrow = factor.has_arrow
    seps, sp = factor.separators, factor.sep_pos
    with torch.cuda.device(dev):
        inv = BTAMatrix(n, b, a, device=dev)
        with _phase(phase_times, "reduced"):
            red = bta.selected_invert(factor.reduced_factor, counter=counter)
        for kk, t in enumerate(seps):
            inv.diag[t].copy_(red.diag[kk])
            if use_arrow:
                inv.arrow[t].copy_(red.arrow[kk])
            if kk + 1 < len(seps) and seps[kk + 1] == t + 1:
                inv.lower[t].copy_(red.lower[kk])
        if a > 0:
            inv.tip.copy_(red.tip)

    def job(ch):
        o = ch.off
        with torch.cuda.device(ch.device):
            f64 = dict(dtype=torch.float64, device=ch.device)
            Xd = torch.zeros(ch.n_ext, b, b, **f64)
            Xl = torch.zeros(max(ch.n_ext - 1, 1), b, b, **f64)
            Xa = torch.zeros(ch.n_ext, max(ch.ap, 1), b, **f64)
            Xt = torch.zeros(max(ch.ap, 1), max(ch.ap, 1), **f64)
            if ch.left is not None:
                pl = sp[ch.left]
                Xt[:b, :b] = red.diag[pl].to(ch.device)
                if use_arrow:
                    Xt[o:, :b] = red.arrow[pl].to(ch.device)
                    Xt[:b, o:] = red.arrow[pl].T.to(ch.device)
            if a > 0 and use_arrow:
                Xt[o:, o:] = red.tip.to(ch.device)
            elif a > 0:
                Xt[o:, o:] = red.tip.to(ch.device)
            if ch.right is not None:
                pr = sp[ch.right]
                Xd[ch.n_int] = red.diag[pr].to(ch.device)
                if use_arrow:
                    Xa[ch.n_int, o:] = red.arrow[pr].to(ch.device)
                if ch.left is not None:
                    Xa[ch.n_int, :b] = red.lower[sp[ch.left]].T.to(ch.device)
            ws = torch.empty(lib.stbta_pobtasi_workspace_bytes(ch.n_ext, b, ch.ap),
                             dtype=torch.uint8, device=ch.device)
            _lib.check(
                lib.stbta_pobtasi_ex(*ch.regions(), _lib.ptr(Xd), _lib.ptr(Xl), _lib.ptr(Xa),
                                     _lib.ptr(Xt), ch.n_ext, b, ch.ap, int(ch.chain_arrow),
                                     ch.n_int, _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
                "stbta_pobtasi_ex",
            )
            torch.cuda.current_stream().synchronize()
        return Xd, Xl, Xa

    parts = [ch for ch in factor.partitions if ch.n_int > 0]
    devices = list({str(ch.device): ch.device for ch in parts}.values())
    mapper = mapper or _default_mapper(devices)
    with _phase(phase_times, "recover"):
        results = [job(c) for c in parts] if mapper is None else list(mapper(job, parts))
    with torch.cuda.device(dev):
        for ch, (Xd, Xl, Xa) in zip(parts, results):
            ni, lo, hi = ch.n_int, ch.lo, ch.hi
            inv.diag[lo:hi].copy_(Xd[:ni].to(dev))
            if ni > 1:
                inv.lower[lo : hi - 1].copy_(Xl[: ni - 1].to(dev))
            if ch.right is not None:
                inv.lower[hi - 1].copy_(Xl[ni - 1].to(dev))
            if ch.left is not None:
                inv.lower[lo - 1].copy_(Xa[0, :b].T.to(dev))
            if use_arrow:
                inv.arrow[lo:hi].copy_(Xa[:ni, ch.off :].to(dev))
            _charge(counter, b**3, ni * (2 if ch.left is not None else 1))
            if use_arrow:  # reference bta_dist.py:584-589: a^3 per interior block
                _charge(counter, a**3, ni)
    return inv
