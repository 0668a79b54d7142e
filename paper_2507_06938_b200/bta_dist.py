"""Time-partitioned BTA solver (S3): PPOBTAF / PPOBTAS / PPOBTASI on B200.

Mirror of the reference ``stinla.bta_dist`` (pkg/src/stinla/bta_dist.py):
same plan (``plan_partitions``, bta_dist.py:65-112), separators
(bta_dist.py:257-265), error tagging and results, re-designed around the
device kernels:

* A partition owns its block rows [start, end) (:class:`BTARows`) and never
  reads another partition's data.  Its interior is eliminated by ONE partial
  POBTAF (``stbta_pobtaf_ex`` with ``nfact``) on an *extended chain*: the
  interior blocks, then the right separator as a last ordinary block, and an
  arrowhead made of the left separator's rows stacked on the true arrow rows.
  The elimination leaves exactly the reference's Schur contributions in the
  unfactored parts (bta_dist.py:174-254).
* The Schur pieces plus the separator rows (a few b x b blocks per
  partition) are packed into one flat buffer; the root assembles the reduced
  2(P-1)-block BTA in partition order (bta_dist.py:322-350) and factorizes it
  by POBTAF.
* ``d_solve`` runs through the chain factor: one forward and one backward
  interior POBTAS sweep per partition around one reduced solve, joined by
  the factor's right-separator link and arrowhead rows in ``stbta_couple``
  (device kernels, fixed summation order).
* ``d_selected_invert`` seeds each chain's inverse with the reduced selected
  inverse (separator, fill and tip entries) and continues the POBTASI
  recursion over the interior (``stbta_pobtasi_ex`` with ``nstart``), which is
  the reference's three-term interior recursion (bta_dist.py:508-602).

Partitions live on the GPUs of one process (``devices``; a mapper runs them
concurrently: :func:`d_factorize` / :func:`d_solve` / :func:`d_selected_invert`,
the reference's API), or one per rank under torchrun
(:func:`d_factorize_nccl` / :func:`d_solve_nccl` /
:func:`d_selected_invert_nccl`): each rank holds only its own rows, and only
the packed pieces, reduced right-hand sides, separator solutions and inverse
seeds cross NCCL (grouped point-to-point over NVLink).
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



def _rows_of(plan, p):
    """Block rows [start, end) owned by partition p (its separators included)."""
    return plan.boundaries[p], plan.boundaries[p + 1]


# ---------------------------------------------------------------- coupling kernel
def _couple(trans, A, X, Y, alpha=1.0, reduce=False):
    """Y (+)= alpha * op(A_j) X_j on the device (``stbta_couple``; the `@` /
    einsum couplings of the reference d_solve, bta_dist.py:370-458).

    A: (nb, m, n) or (m, n); X: (nb, rows, k) or (rows, k) (batch stride 0
    broadcasts); Y: (nb, rows, k), or (rows, k) when reduced over the batch.
    Rows of every operand must be contiguous (stride(-1) == 1)."""
    lib = _lib.load()
    if A.dim() == 2:
        A = A.unsqueeze(0)
    if X.dim() == 2:
        X = X.unsqueeze(0)
    Y3 = Y.unsqueeze(0) if Y.dim() == 2 else Y
    nb, m, n = A.shape
    k = X.shape[-1]
    for t in (A, X, Y3):
        if t.stride(-1) != 1 or t.dtype != torch.float64:
            raise ValueError("coupling operands must be float64 with contiguous rows")
    ws = bta._workspace(lib.stbta_couple_workspace_bytes(int(trans), nb, m, n, int(reduce)),
                        A.device)
    _lib.check(
        lib.stbta_couple(int(trans), nb, m, n, k, float(alpha), _lib.ptr(A), A.stride(1),
                         A.stride(0), _lib.ptr(X), X.stride(1), X.stride(0) if X.shape[0] > 1 else 0,
                         _lib.ptr(Y3), Y3.stride(1), Y3.stride(0), int(reduce), _lib.ptr(ws),
                         ws.numel(), _lib.stream_ptr()),
        "stbta_couple",
    )
    return Y


def _sym_lower(x):
    """Full symmetric matrix from the lower triangle of x."""
    return torch.tril(x) + torch.tril(x, -1).T


# ---------------------------------------------------------------- row slices
class BTARows:
    """Block rows [t0, t1) of an n-block BTA matrix: one partition's share of
    the data, the unit a rank owns (it never sees the other partitions' rows).

    ``diag[j]`` = A(t0+j, t0+j), ``lower[j]`` = A(t0+j, t0+j-1) (zero for the
    first block row of the matrix), ``arrow[j]`` = A(arrow, t0+j); ``tip`` =
    A(arrow, arrow) on the rank that owns the reduced system (None elsewhere).
    Same row-major block layout as :class:`~.bta.BTAMatrix`."""

    def __init__(self, n_blocks, t0, t1, block_size, arrow_size=0, device=None, with_tip=True,
                 data=None):
        self.n_blocks, self.t0, self.t1 = n_blocks, t0, t1
        self.block_size, self.arrow_size = block_size, arrow_size
        dev = torch.device(device) if device is not None else bta.default_device()
        m, b, a = t1 - t0, block_size, arrow_size
        size = 2 * m * b * b + m * a * b + (a * a if with_tip else 0)
        if data is None:
            data = torch.zeros(size, dtype=torch.float64, device=dev)
        elif data.numel() != size:
            raise ValueError(f"rows buffer has {data.numel()} elements, expected {size}")
        self.data = data  # flat: diag (m,b,b) | lower (m,b,b) | arrow (m,a,b) [| tip (a,a)]
        e0, e1 = m * b * b, 2 * m * b * b
        e2 = e1 + m * a * b
        self.diag = data[:e0].view(m, b, b)
        self.lower = data[e0:e1].view(m, b, b)
        self.arrow = data[e1:e2].view(m, a, b)
        self.tip = data[e2:].view(a, a) if with_tip else None

    @property
    def device(self):
        return self.diag.device

    @classmethod
    def from_matrix(cls, matrix, t0, t1, device=None, with_tip=True):
        """Copy block rows [t0, t1) out of a global BTAMatrix (any device)."""
        dev = torch.device(device) if device is not None else matrix.device
        r = cls(matrix.n_blocks, t0, t1, matrix.block_size, matrix.arrow_size, dev, with_tip)
        r.diag.copy_(matrix.diag[t0:t1])
        lo = max(t0, 1)
        if t1 > lo:
            r.lower[lo - t0 :].copy_(matrix.lower[lo - 1 : t1 - 1])
        r.arrow.copy_(matrix.arrow[t0:t1])
        if with_tip and matrix.arrow_size:
            r.tip.copy_(matrix.tip)
        return r

    # accessors by global block row
    def d(self, t):
        return self.diag[t - self.t0]

    def low(self, t):
        return self.lower[t - self.t0]

    def arw(self, t):
        return self.arrow[t - self.t0]


class _MatrixRows:
    """Global BTAMatrix seen through the BTARows accessors."""

    def __init__(self, m):
        self.m, self.t0, self.t1 = m, 0, m.n_blocks
        self.tip = m.tip if m.arrow_size else None

    def d(self, t):
        return self.m.diag[t]

    def low(self, t):
        return self.m.lower[t - 1]

    def arw(self, t):
        return self.m.arrow[t]

    @property
    def diag(self):
        return self.m.diag

    @property
    def arrow(self):
        return self.m.arrow


def _rows_arrow_nonzero(rows):
    return rows.arrow.numel() > 0 and bool(torch.any(rows.arrow != 0).item())


# ---------------------------------------------------------------- partitions
class _Chain:
    """One partition on its device.

    The *extended chain* (what the partial POBTAF eliminates): interior blocks
    [lo, hi), then the right separator block (if any); arrowhead rows = [left
    separator (b rows, if any); true arrow (a rows)].  The elimination leaves
    exactly the reference's Schur contributions in the unfactored parts
    (bta_dist.py:174-254): d_right / f_right in the last block, the fill in its
    left-separator arrowhead rows, d_left / f_left / d_tip in the chain's tip.

    Next to it, the original separator-row data the reduced system needs (the
    left separator's diagonal, arrow and coupling to the previous partition).
    The partitioned solve runs through the chain factor itself: one forward
    and one backward interior sweep, joined to the reduced system by the
    factor's right-separator link and arrowhead rows."""

    def __init__(self, index, lo, hi, left, right, b, a, use_arrow, device):
        self.index, self.lo, self.hi, self.left, self.right = index, lo, hi, left, right
        self.b, self.a = b, a
        self.n_int = hi - lo
        self.n_ext = self.n_int + (1 if right is not None else 0)
        self.off = b if left is not None else 0  # first true-arrow row in the arrowhead
        self.ap = self.off + a
        self.use_arrow = use_arrow
        self.chain_arrow = (left is not None) or use_arrow
        self.device = torch.device(device)
        self.start = left if left is not None else lo
        self.end = right + 1 if right is not None else hi
        f64 = dict(dtype=torch.float64, device=self.device)
        n = max(self.n_ext, 1)
        self.diag = torch.empty(n, b, b, **f64)
        self.lower = torch.empty(max(self.n_ext - 1, 1), b, b, **f64)
        self.arrow = torch.zeros(n, max(self.ap, 1), b, **f64)
        self.tip = torch.zeros(max(self.ap, 1), max(self.ap, 1), **f64)
        self.logdet_dev = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.info = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.logdet = 0.0
        self.sep_diag = self.sep_lower = self.sep_arrow = None

    def load(self, rows):
        """Fill the chain from block rows [start, end) (BTARows or a global
        matrix view, any device) and keep the originals it needs later."""
        lo, hi, ni, b = self.lo, self.hi, self.n_int, self.b

        def g(x):
            return x.to(self.device, non_blocking=True)

        if ni > 0:
            self.diag[:ni].copy_(g(rows.diag[lo - rows.t0 : hi - rows.t0]))
            for j in range(ni - 1):  # chain lower[j] = A(lo+j+1, lo+j)
                self.lower[j].copy_(g(rows.low(lo + j + 1)))
        if self.right is not None:
            self.diag[ni].copy_(g(rows.d(hi)))
            if ni > 0:
                self.lower[ni - 1].copy_(g(rows.low(hi)))
        if self.left is not None:
            # A(left, lo) = A(lo, left)^T; with an empty interior this is the
            # original A(left, right)^T -- the fill the reduced system reads
            self.arrow[0, :b].copy_(g(rows.low(lo)).T)
            t = self.left
            self.sep_diag = g(rows.d(t)).clone()
            self.sep_lower = g(rows.low(t)).clone() if t > 0 else None
            if self.a > 0 and self.use_arrow:
                self.sep_arrow = g(rows.arw(t)).clone()
        if self.a > 0 and self.use_arrow:
            if ni > 0:
                self.arrow[:ni, self.off :].copy_(g(rows.arrow[lo - rows.t0 : hi - rows.t0]))
            if self.right is not None:
                self.arrow[ni, self.off :].copy_(g(rows.arw(hi)))
        return self

    def regions(self):
        return [_lib.ptr(self.diag), _lib.ptr(self.lower), _lib.ptr(self.arrow), _lib.ptr(self.tip)]

    def last_diag(self):
        return self.diag[self.n_int]

    def last_arrow(self):
        return self.arrow[self.n_int]

    def eliminate_async(self):
        """Issue the partial POBTAF (interior only) on the current stream."""
        if self.n_int == 0:
            return
        lib = _lib.load()
        with torch.cuda.device(self.device):
            ws = bta._workspace(lib.stbta_pobtaf_workspace_bytes(self.n_ext, self.b, self.ap),
                                self.device)
            d, l, ar, tp = self.regions()
            _lib.check(
                lib.stbta_pobtaf_ex(d, l, ar, tp, self.n_ext, self.b, self.ap, self.b,
                                    int(self.chain_arrow), self.n_int, _lib.ptr(self.logdet_dev),
                                    _lib.ptr(self.info), _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr()),
                "stbta_pobtaf_ex",
            )

    def eliminate(self):
        """Partial POBTAF; returns the failing global block index or None."""
        if self.n_int == 0:
            return None
        self.eliminate_async()
        with torch.cuda.device(self.device):
            code = int(self.info.item())
            self.logdet = float(self.logdet_dev.item())
        return self.lo + code - 1 if code else None

    # -- Schur pieces for the reduced system ---------------------------------
    def piece_layout(self):
        return _piece_layout(self.left is not None, self.right is not None, self.b, self.a,
                             self.use_arrow)

    def pack_pieces(self):
        """Flat FP64 buffer of this partition's contribution to the reduced
        system (layout: :func:`_piece_layout`), on this device."""
        b, o = self.b, self.off
        parts = {"logdet": self.logdet_dev}
        if self.left is not None:
            parts["sep_diag"] = self.sep_diag
            parts["sep_lower"] = self.sep_lower if self.sep_lower is not None else \
                torch.zeros_like(self.sep_diag)
            parts["d_left"] = _sym_lower(self.tip[:b, :b]) if self.n_int else \
                torch.zeros_like(self.sep_diag)
            if self.use_arrow and self.a:
                parts["sep_arrow"] = self.sep_arrow
                parts["f_left"] = self.tip[o:, :b]
        if self.right is not None:
            parts["d_right"] = _sym_lower(self.last_diag()) if self.n_int else self.last_diag()
            if self.left is not None:
                parts["fill"] = self.last_arrow()[:b]
            if self.use_arrow and self.a:
                parts["f_right"] = self.last_arrow()[o:]
        if self.use_arrow and self.a:
            parts["d_tip"] = _sym_lower(self.tip[o:, o:])
        layout = self.piece_layout()
        return torch.cat([parts[name].reshape(-1) for name, _ in layout])

    # -- partitioned solve -----------------------------------------------------
    def interior_sweep(self, rhs, mode):
        """In place on rhs (n_int*b, k) with the interior factor L_int:
        mode 1: L_int y = rhs (forward), mode 2: L_int^T x = rhs (backward)."""
        lib = _lib.load()
        n, b = self.n_int, self.b
        k = rhs.shape[1]
        with torch.cuda.device(self.device):
            ws = bta._workspace(lib.stbta_pobtas_workspace_bytes(n, b, 0, k), self.device)
            _lib.check(
                lib.stbta_pobtas_ex(_lib.ptr(self.diag), _lib.ptr(self.lower), None, None, n, b, 0,
                                    b, 0, _lib.ptr(rhs), k, mode, _lib.ptr(ws), ws.numel(),
                                    _lib.stream_ptr()),
                "stbta_pobtas_ex",
            )
        return rhs

    def solve_forward(self, xr):
        """Forward half of the partitioned solve through the chain factor
        (bta_dist.py:370-420): y_int = L_int^-1 x_int, then the extended rows'
        reduced right-hand sides r_ext - L_ext,int y_int, with L_ext,int the
        right separator's link L(hi, hi-1) and the arrowhead rows (left
        separator + arrow) of the factor.  xr: this partition's rows [start,
        end) (rows*b, k) on this device.  Returns (y_int, flat [c_left |
        c_right | c_tip]) (the parts that exist)."""
        b = self.b
        k = xr.shape[1]
        i0 = (self.lo - self.start) * b
        y = xr[i0 : i0 + self.n_int * b].clone()
        out = []
        with torch.cuda.device(self.device):
            s_ah = None
            if self.n_int:
                self.interior_sweep(y, 1)
                if self.chain_arrow:  # sum_j L(arrowhead, j) y_j, j over the interior
                    s_ah = torch.zeros(self.ap, k, dtype=torch.float64, device=self.device)
                    _couple(0, self.arrow[: self.n_int, : self.ap], y.view(self.n_int, b, k),
                            s_ah, 1.0, reduce=True)
            if self.left is not None:
                c = xr[:b].clone()
                if s_ah is not None:
                    c -= s_ah[:b]
                out.append(c)
            if self.right is not None:
                c = xr[(self.end - 1 - self.start) * b :].clone()
                if self.n_int:
                    _couple(0, self.lower[self.n_int - 1], y[-b:], c, -1.0)
                out.append(c)
            if self.use_arrow and self.a:
                out.append(-s_ah[self.off :] if s_ah is not None else
                           torch.zeros(self.a, k, dtype=torch.float64, device=self.device))
        flat = torch.cat([c.reshape(-1) for c in out]) if out else \
            torch.zeros(0, dtype=torch.float64, device=self.device)
        return y, flat

    def solve_backward(self, y, x_left, x_right, x_tip):
        """x_int = L_int^-T (y_int - L_ext,int^T x_ext); returns this
        partition's solution rows [start, end)."""
        b = self.b
        k = y.shape[1]
        with torch.cuda.device(self.device):
            rows = torch.empty((self.end - self.start) * b, k, dtype=torch.float64,
                               device=self.device)
            if self.left is not None:
                rows[:b] = x_left
            if self.right is not None:
                rows[(self.end - 1 - self.start) * b :] = x_right
            if self.n_int:
                w = y.clone()
                if self.right is not None:
                    _couple(1, self.lower[self.n_int - 1], x_right, w[-b:], -1.0)
                if self.chain_arrow:
                    x_ah = torch.zeros(self.ap, k, dtype=torch.float64, device=self.device)
                    if self.left is not None:
                        x_ah[:b] = x_left
                    if self.a > 0 and x_tip is not None:
                        x_ah[self.off :] = x_tip
                    _couple(1, self.arrow[: self.n_int, : self.ap],
                            x_ah.expand(self.n_int, self.ap, k), w.view(self.n_int, b, k), -1.0)
                self.interior_sweep(w, 2)
                i0 = (self.lo - self.start) * b
                rows[i0 : i0 + self.n_int * b] = w
        return rows

    # -- partitioned selected inversion ------------------------------------
    def invert(self, seeds):
        """Continue the POBTASI recursion over the interior from the reduced
        inverse's entries (``seeds``: dict of Xd_left, Xa_left, Xd_right,
        Xa_right, X_fill, X_tip, X_prev on this device); returns the inverse's
        block rows [start, end) as BTARows (tip not included)."""
        lib = _lib.load()
        b, o, ni = self.b, self.off, self.n_int
        dev = self.device
        out = BTARows(0, self.start, self.end, b, self.a, dev, with_tip=False)
        with torch.cuda.device(dev):
            if self.left is not None:
                out.d(self.left).copy_(seeds["Xd_left"])
                if "X_prev" in seeds:
                    out.low(self.left).copy_(seeds["X_prev"])
                if self.use_arrow and self.a:
                    out.arw(self.left).copy_(seeds["Xa_left"])
            if self.right is not None:
                out.d(self.right).copy_(seeds["Xd_right"])
                if self.use_arrow and self.a:
                    out.arw(self.right).copy_(seeds["Xa_right"])
                if self.left is not None and ni == 0:
                    out.low(self.right).copy_(seeds["X_fill"])
            if ni == 0:
                return out
            f64 = dict(dtype=torch.float64, device=dev)
            Xd = torch.zeros(self.n_ext, b, b, **f64)
            Xl = torch.zeros(max(self.n_ext - 1, 1), b, b, **f64)
            Xa = torch.zeros(self.n_ext, max(self.ap, 1), b, **f64)
            Xt = torch.zeros(max(self.ap, 1), max(self.ap, 1), **f64)
            if self.left is not None:
                Xt[:b, :b] = seeds["Xd_left"]
                if self.use_arrow and self.a:
                    Xt[o:, :b] = seeds["Xa_left"]
                    Xt[:b, o:] = seeds["Xa_left"].T
            if self.a > 0:
                Xt[o:, o:] = seeds["X_tip"]
            if self.right is not None:
                Xd[ni] = seeds["Xd_right"]
                if self.use_arrow and self.a:
                    Xa[ni, o:] = seeds["Xa_right"]
                if self.left is not None:
                    Xa[ni, :b] = seeds["X_fill"].T
            ws = bta._workspace(lib.stbta_pobtasi_workspace_bytes(self.n_ext, b, self.ap), dev)
            _lib.check(
                lib.stbta_pobtasi_ex(*self.regions(), _lib.ptr(Xd), _lib.ptr(Xl), _lib.ptr(Xa),
                                     _lib.ptr(Xt), self.n_ext, b, self.ap, int(self.chain_arrow),
                                     ni, _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
                "stbta_pobtasi_ex",
            )
            out.diag[self.lo - self.start : self.hi - self.start].copy_(Xd[:ni])
            for j in range(ni - 1):  # X(lo+j+1, lo+j)
                out.low(self.lo + j + 1).copy_(Xl[j])
            if self.right is not None:
                out.low(self.hi).copy_(Xl[ni - 1])
            if self.left is not None:
                out.low(self.lo).copy_(Xa[0, :b].T)
            if self.use_arrow and self.a:
                out.arrow[self.lo - self.start : self.hi - self.start].copy_(Xa[:ni, o:])
        return out


def _piece_layout(left, right, b, a, use_arrow):
    """Ordered (name, numel) of one partition's packed reduced-system pieces."""
    arrow = use_arrow and a > 0
    lay = [("logdet", 1)]
    if left:
        lay += [("sep_diag", b * b), ("sep_lower", b * b), ("d_left", b * b)]
        if arrow:
            lay += [("sep_arrow", a * b), ("f_left", a * b)]
    if right:
        lay += [("d_right", b * b)]
        if left:
            lay += [("fill", b * b)]
        if arrow:
            lay += [("f_right", a * b)]
    if arrow:
        lay += [("d_tip", a * a)]
    return lay


def _unpack(flat, layout, b, a):
    shapes = {"logdet": (1,), "sep_arrow": (a, b), "f_left": (a, b), "f_right": (a, b),
              "d_tip": (a, a)}
    out, o = {}, 0
    for name, size in layout:
        out[name] = flat[o : o + size].view(*shapes.get(name, (b, b)))
        o += size
    return out


def _reduce_and_factorize(plan, pieces, tip, b, a, use_arrow, device, counter=None):
    """Reduced 2(P-1)-block BTA over the separators (bta_dist.py:322-350) from
    the partitions' packed pieces, summed in partition order, factorized by
    POBTAF on ``device``.  Returns (factor, failing separator or None)."""
    seps = _separators(plan)
    sp = {t: k for k, t in enumerate(seps)}
    n_red = len(seps)
    with torch.cuda.device(device):
        red = BTAMatrix(n_red, b, a, device=device)
        if a > 0 and tip is not None:
            red.tip.copy_(tip)
        for p, (lo, hi, left, right) in enumerate(_partition_ranges(plan)):
            pc = _unpack(pieces[p], _piece_layout(left is not None, right is not None, b, a,
                                                  use_arrow), b, a)
            if left is not None:
                pos = sp[left]
                red.diag[pos] = pc["sep_diag"] + pc["d_left"]
                if pos > 0:
                    red.lower[pos - 1].copy_(pc["sep_lower"])
                if "sep_arrow" in pc:
                    red.arrow[pos] = pc["sep_arrow"] + pc["f_left"]
            if right is not None:
                pos = sp[right]
                red.diag[pos].copy_(pc["d_right"])
                if left is not None:
                    red.lower[sp[left]].copy_(pc["fill"].T)
                if "f_right" in pc:
                    red.arrow[pos].copy_(pc["f_right"])
            if "d_tip" in pc:
                red.tip += pc["d_tip"]
        try:
            return bta.factorize(red, counter=counter, use_arrow=use_arrow), None
        except FactorizationError as err:
            return None, seps[min(err.block_index, n_red - 1)]


def _interior_logdet(pieces):
    """Sum of the partition log-dets in partition order (host)."""
    return sum(float(pc[0].item()) for pc in pieces)


# ---------------------------------------------------------------- factor object
class DistBTAFactor:
    """Partition chains plus the factorized reduced system (bta_dist.py:143-166).

    Single process: ``partitions`` holds every chain (possibly on several
    GPUs), ``reduced_factor`` lives on the root device.  One partition per
    rank (:func:`d_factorize_nccl`): ``partitions`` holds this rank's chain
    only, ``reduced_factor`` is set on the root rank only, ``group`` / ``root``
    name the process group."""

    def __init__(self, plan, matrix_shape, partitions, reduced_factor, separators,
                 use_arrow=False):
        self.plan = plan
        self.n_blocks, self.block_size, self.arrow_size = matrix_shape
        self.partitions = partitions
        self.reduced_factor = reduced_factor
        self.separators = separators
        self.sep_pos = {t: k for k, t in enumerate(separators)}
        self._use_arrow = use_arrow
        self.sequential = None
        self.interior_logdet = 0.0
        self.total_logdet = None
        self.group = None
        self.root = 0
        self.device = None

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


def _make_chains(plan, b, a, use_arrow, devices):
    return [
        _Chain(p, lo, hi, left, right, b, a, use_arrow, torch.device(devices[p % len(devices)]))
        for p, (lo, hi, left, right) in enumerate(_partition_ranges(plan))
    ]


def _charge_eliminate(counter, chains, b, a, use_arrow):
    for ch in chains:  # modeled cost units, as the reference (bta_dist.py:220-225)
        _charge(counter, b**3, ch.n_int * (2 if ch.left is not None else 1))
        if use_arrow:
            _charge(counter, a**3, ch.n_int)


def d_factorize(matrix, plan, counter=None, mapper=None, phase_times=None, devices=None):
    """Partitioned block Cholesky (bta_dist.py:282-359).

    ``matrix`` is read only for P > 1 (factorized in place for P == 1, like the
    reference).  ``devices[p % len(devices)]`` hosts partition p (each chain
    is loaded from its own block rows only); the reduced system lives on the
    matrix's device.  Results are combined in partition order, independent of
    the mapper.
    """
    if plan.n_blocks != matrix.n_blocks:
        raise PlanError("plan does not match the matrix block count")
    shape = (matrix.n_blocks, matrix.block_size, matrix.arrow_size)
    if plan.n_partitions == 1:
        with _phase(phase_times, "total"):
            factor = bta.factorize(matrix, counter=counter)
        dist = DistBTAFactor(plan, shape, [], None, [])
        dist.sequential = factor
        return dist
    b, a = matrix.block_size, matrix.arrow_size
    use_arrow = bta._arrow_nonzero(matrix)
    devices = list(devices) if devices else [matrix.device]
    chains = _make_chains(plan, b, a, use_arrow, devices)
    view = _MatrixRows(matrix)
    return _factorize_chains(plan, shape, chains, lambda ch: ch.load(view), matrix.tip if a else
                             None, use_arrow, matrix.device, counter, mapper or
                             _default_mapper(devices), phase_times)


def _factorize_chains(plan, shape, chains, fill, tip, use_arrow, root_device, counter=None,
                      mapper=None, phase_times=None):
    """Load (``fill(chain)``) and eliminate every chain, then reduce and
    factorize on ``root_device`` (the single-process S3 driver)."""
    n, b, a = shape

    def job(ch):
        with torch.cuda.device(ch.device):
            fill(ch)
            bad = ch.eliminate()
            return ch, bad, ch.pack_pieces().to(root_device)

    with _phase(phase_times, "eliminate"):
        res = [job(c) for c in chains] if mapper is None else list(mapper(job, chains))
    for ch, bad, _ in res:  # lowest partition first
        if bad is not None:
            raise FactorizationError(bad, partition=ch.index)
    _charge_eliminate(counter, chains, b, a, use_arrow)
    pieces = [pc for _, _, pc in res]
    with _phase(phase_times, "reduced"):
        red, bad = _reduce_and_factorize(plan, pieces, tip, b, a, use_arrow, root_device, counter)
    if bad is not None:
        raise FactorizationError(bad, partition=-1)
    f = DistBTAFactor(plan, shape, chains, red, _separators(plan), use_arrow)
    f.interior_logdet = _interior_logdet(pieces)
    f.device = torch.device(root_device)
    return f


def d_logdet(factor):
    """Interior log-dets plus the reduced system's (bta_dist.py:362-367)."""
    if factor.sequential is not None:
        return bta.logdet(factor.sequential)
    if factor.total_logdet is not None:  # one partition per rank: broadcast by the root
        return factor.total_logdet
    return factor.interior_logdet + bta.logdet(factor.reduced_factor)


def _reduced_rhs(factor, contribs, x_tip, k):
    """Reduced right-hand side from the partitions' flat contributions
    (partition order) and the tip right-hand side, on the root device."""
    b, a = factor.block_size, factor.arrow_size
    seps, sp = factor.separators, factor.sep_pos
    n_red = len(seps)
    dev = factor.device
    red = torch.zeros(n_red * b + a, k, dtype=torch.float64, device=dev)
    if a > 0 and x_tip is not None:
        red[n_red * b :] = x_tip
    for p, (lo, hi, left, right) in enumerate(_partition_ranges(factor.plan)):
        c, o = contribs[p].view(-1, k), 0
        if left is not None:
            red[sp[left] * b : (sp[left] + 1) * b] = c[o : o + b]
            o += b
        if right is not None:
            red[sp[right] * b : (sp[right] + 1) * b] = c[o : o + b]
            o += b
        if factor.has_arrow and a > 0:
            red[n_red * b :] += c[o : o + a]
    return red


def _sep_solution(factor, red_x, p):
    """(x_left, x_right) of partition p from the reduced solution."""
    b = factor.block_size
    lo, hi, left, right = _partition_ranges(factor.plan)[p]
    sp = factor.sep_pos
    xl = red_x[sp[left] * b : (sp[left] + 1) * b] if left is not None else None
    xr = red_x[sp[right] * b : (sp[right] + 1) * b] if right is not None else None
    return xl, xr


def d_solve(factor, rhs, counter=None, phase_times=None):
    """Partitioned solve (bta_dist.py:370-458) through the chain factors: a
    forward interior sweep per partition, the reduced separator solve, a
    backward interior sweep; the factor's link / arrowhead couplings run in
    ``stbta_couple``."""
    if factor.sequential is not None:
        with _phase(phase_times, "total"):
            return bta.solve(factor.sequential, rhs, counter=counter)
    b, a, n = factor.block_size, factor.arrow_size, factor.n_blocks
    dev = factor.device
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
    zs, contribs = [], []
    with _phase(phase_times, "forward"):
        for ch in factor.partitions:
            xr = X[ch.start * b : ch.end * b].to(ch.device)
            z, c = ch.solve_forward(xr)
            zs.append(z)
            contribs.append(c.to(dev))
            _charge(counter, b**2, ch.n_int)
    with _phase(phase_times, "reduced"):
        red_rhs = _reduced_rhs(factor, contribs, X[n * b :] if a else None, k)
        red_x = bta.solve(factor.reduced_factor, red_rhs, counter=counter)
    x_tip = red_x[len(factor.separators) * b :]
    with _phase(phase_times, "backward"):
        for ch, z in zip(factor.partitions, zs):
            xl, xr = _sep_solution(factor, red_x, ch.index)
            g = (lambda t: None if t is None else t.to(ch.device))
            rows = ch.solve_backward(z, g(xl), g(xr), x_tip.to(ch.device))
            X[ch.start * b : ch.end * b] = rows.to(dev)
            _charge(counter, b**2, ch.n_int)
    if a > 0:
        X[n * b :] = x_tip
    out = x if not squeeze else X.reshape(-1)
    return out.cpu().numpy() if host else out


def _seeds(factor, red, p):
    """Reduced-inverse entries partition p's interior recursion starts from."""
    lo, hi, left, right = _partition_ranges(factor.plan)[p]
    sp = factor.sep_pos
    s = {}
    if factor.arrow_size > 0:
        s["X_tip"] = red.tip
    if left is not None:
        pl = sp[left]
        s["Xd_left"] = red.diag[pl]
        s["Xa_left"] = red.arrow[pl]
        if pl > 0:
            s["X_prev"] = red.lower[pl - 1]  # X(left, previous partition's right separator)
    if right is not None:
        pr = sp[right]
        s["Xd_right"] = red.diag[pr]
        s["Xa_right"] = red.arrow[pr]
        if left is not None:
            s["X_fill"] = red.lower[sp[left]]  # X(right, left)
    return s


_SEED_ORDER = ("X_tip", "Xd_left", "Xa_left", "X_prev", "Xd_right", "Xa_right", "X_fill")


def d_selected_invert(factor, counter=None, mapper=None, phase_times=None):
    """Pattern entries of the inverse (bta_dist.py:461-505): reduced selected
    inverse, then each chain's POBTASI recursion seeded with it."""
    if factor.sequential is not None:
        with _phase(phase_times, "total"):
            return bta.selected_invert(factor.sequential, counter=counter)
    n, b, a = factor.n_blocks, factor.block_size, factor.arrow_size
    dev = factor.device
    with torch.cuda.device(dev):
        with _phase(phase_times, "reduced"):
            red = bta.selected_invert(factor.reduced_factor, counter=counter)
        inv = BTAMatrix(n, b, a, device=dev)
        if a > 0:
            inv.tip.copy_(red.tip)

    def job(ch):
        seeds = {k: v.to(ch.device) for k, v in _seeds(factor, red, ch.index).items()}
        with torch.cuda.device(ch.device):
            rows = ch.invert(seeds)
            torch.cuda.current_stream().synchronize()
        return rows

    parts = factor.partitions
    devices = list({str(ch.device): ch.device for ch in parts}.values())
    mapper = mapper or _default_mapper(devices)
    with _phase(phase_times, "recover"):
        results = [job(c) for c in parts] if mapper is None else list(mapper(job, parts))
    with torch.cuda.device(dev):
        for ch, rows in zip(parts, results):
            _rows_into(inv, rows)
            _charge(counter, b**3, ch.n_int * (2 if ch.left is not None else 1))
            if factor.has_arrow:  # reference bta_dist.py:584-589: a^3 per interior block
                _charge(counter, a**3, ch.n_int)
    return inv


def _rows_into(inv, rows):
    """Write BTARows [t0, t1) into a global BTAMatrix (the inverse)."""
    t0, t1, dev = rows.t0, rows.t1, inv.device
    inv.diag[t0:t1].copy_(rows.diag.to(dev))
    lo = max(t0, 1)
    if t1 > lo:
        inv.lower[lo - 1 : t1 - 1].copy_(rows.lower[lo - t0 :].to(dev))
    if inv.arrow_size:
        inv.arrow[t0:t1].copy_(rows.arrow.to(dev))


# ---------------------------------------------------------------- one partition per rank
def _dist():
    import torch.distributed as dist

    return dist


def _gather_flat(local, sizes, root, group):
    """Root receives every rank's flat buffer (sizes known to all); grouped
    point-to-point over NCCL.  Returns the list on root, None elsewhere."""
    dist = _dist()
    rank = dist.get_rank(group)
    if rank != root:
        op = dist.P2POp(dist.isend, local.contiguous(),
                        dist.get_global_rank(group, root) if group else root, group=group)
        for req in dist.batch_isend_irecv([op]):
            req.wait()
        return None
    out, ops = [], []
    for r, size in enumerate(sizes):
        if r == root:
            out.append(local)
            continue
        buf = torch.empty(size, dtype=torch.float64, device=local.device)
        out.append(buf)
        ops.append(dist.P2POp(dist.irecv, buf, dist.get_global_rank(group, r) if group else r,
                              group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return out


def _scatter_flat(parts, size, root, group, device):
    """Root sends parts[r] to every rank r; returns this rank's buffer."""
    dist = _dist()
    rank = dist.get_rank(group)
    if rank != root:
        buf = torch.empty(size, dtype=torch.float64, device=device)
        op = dist.P2POp(dist.irecv, buf, dist.get_global_rank(group, root) if group else root,
                        group=group)
        for req in dist.batch_isend_irecv([op]):
            req.wait()
        return buf
    ops = []
    for r, part in enumerate(parts):
        if r != root:
            ops.append(dist.P2POp(dist.isend, part.contiguous(),
                                  dist.get_global_rank(group, r) if group else r, group=group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return parts[root]


def _bcast_status(status, root, group, device):
    """Broadcast a small float64 vector from root; returns it on every rank."""
    dist = _dist()
    t = torch.as_tensor(status, dtype=torch.float64, device=device).clone()
    dist.broadcast(t, dist.get_global_rank(group, root) if group else root, group=group)
    return t.cpu().numpy()


def local_rows(matrix, plan, rank, device=None):
    """Block rows a rank owns under ``plan`` (tip only on rank 0) -- for
    callers that hold the whole matrix; the distributed routines themselves
    only ever touch a rank's own rows."""
    start, end = _rows_of(plan, rank)
    return BTARows.from_matrix(matrix, start, end, device=device, with_tip=(rank == 0))


def d_factorize_nccl(rows, plan, group=None, root=0):
    """PPOBTAF with one partition per rank (torchrun, NCCL over NVLink).

    ``rows``: this rank's :class:`BTARows` -- block rows [start, end) of its
    partition (``plan.boundaries[rank:rank+2]``), plus the tip on ``root``.
    Every rank eliminates its own interior; only the Schur pieces and the
    separator rows (a few b x b blocks) travel to the root, which assembles
    and factorizes the reduced system in partition order.  Returns a
    :class:`DistBTAFactor` on every rank (``d_logdet`` = the broadcast total);
    a non-SPD pivot anywhere raises the same FactorizationError on every rank.
    """
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if plan.n_partitions != world:
        raise PlanError(f"plan has {plan.n_partitions} partitions for {world} ranks")
    if (rows.t0, rows.t1) != _rows_of(plan, rank) or rows.n_blocks not in (0, plan.n_blocks):
        raise PlanError(f"rank {rank} holds block rows [{rows.t0}, {rows.t1}), the plan gives "
                        f"{_rows_of(plan, rank)}")
    dev = rows.device
    b, a = rows.block_size, rows.arrow_size
    flag = torch.tensor([float(a > 0 and _rows_arrow_nonzero(rows))], dtype=torch.float64,
                        device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    use_arrow = bool(flag.item() > 0)
    lo, hi, left, right = _partition_ranges(plan)[rank]
    ch = _Chain(rank, lo, hi, left, right, b, a, use_arrow, dev)
    # every failure (pivot, launch) is published, so no rank is left waiting
    err = torch.zeros(2, dtype=torch.float64, device=dev)
    try:
        with torch.cuda.device(dev):
            ch.load(rows)
            bad = ch.eliminate()
        if bad is not None:
            err[0], err[1] = 1.0, float(bad)
    except Exception:  # noqa: BLE001 -- re-raised below on every rank
        err[0] = 2.0
    errs = [torch.zeros_like(err) for _ in range(world)]
    dist.all_gather(errs, err, group=group)
    for p, e in enumerate(errs):
        if e[0].item() == 1.0:
            raise FactorizationError(int(e[1].item()), partition=p)
        if e[0].item() == 2.0:
            raise _lib.StbtaError(f"partition {p} failed to eliminate its interior")
    ranges = _partition_ranges(plan)
    sizes = [sum(s for _, s in _piece_layout(l is not None, r is not None, b, a, use_arrow))
             for (_, _, l, r) in ranges]
    pieces = _gather_flat(ch.pack_pieces(), sizes, root, group)
    shape = (plan.n_blocks, b, a)
    f = DistBTAFactor(plan, shape, [ch], None, _separators(plan), use_arrow)
    f.group, f.root, f.device = group, root, dev
    status = [0.0, 0.0, 0.0]
    if rank == root:
        try:
            red, bad = _reduce_and_factorize(plan, pieces, rows.tip, b, a, use_arrow, dev)
            if bad is None:
                f.reduced_factor = red
                status = [0.0, 0.0, _interior_logdet(pieces) + bta.logdet(red)]
            else:
                status = [1.0, float(bad), 0.0]
        except Exception:  # noqa: BLE001
            status = [2.0, 0.0, 0.0]
    st = _bcast_status(status, root, group, dev)
    if st[0] == 1.0:
        raise FactorizationError(int(st[1]), partition=-1)
    if st[0] == 2.0:
        raise _lib.StbtaError("reduced system factorization failed on the root")
    f.total_logdet = float(st[2])
    return f


def d_solve_nccl(factor, rhs_rows, rhs_tip=None):
    """PPOBTAS with one partition per rank.  ``rhs_rows``: this rank's rows
    ((end-start)*b, k) or ((end-start)*b,) of the right-hand side; ``rhs_tip``
    its arrow part (a, k) on the root.  Only the per-partition reduced
    right-hand sides (<= 2b+a rows) go to the root and the separator
    solutions come back.  Returns (x_rows, x_tip) with x_tip on every rank."""
    dist = _dist()
    group, root = factor.group, factor.root
    rank = dist.get_rank(group)
    ch = factor.partitions[0]
    b, a = factor.block_size, factor.arrow_size
    squeeze = rhs_rows.dim() == 1
    xr = rhs_rows.reshape(rhs_rows.shape[0], -1).to(ch.device, torch.float64)
    if xr.shape[0] != (ch.end - ch.start) * b:
        raise ValueError(f"rank {rank} rhs has {xr.shape[0]} rows, expected "
                         f"{(ch.end - ch.start) * b}")
    k = xr.shape[1]
    z, contrib = ch.solve_forward(xr)
    ranges = _partition_ranges(factor.plan)
    arrow = factor.has_arrow and a > 0
    sizes = [k * (b * ((l is not None) + (r is not None)) + (a if arrow else 0))
             for (_, _, l, r) in ranges]
    contribs = _gather_flat(contrib, sizes, root, group)
    out_sizes = [k * (b * ((l is not None) + (r is not None)) + a) for (_, _, l, r) in ranges]
    parts = None
    if rank == root:
        tip = rhs_tip.reshape(a, k).to(ch.device, torch.float64) if a else None
        red_rhs = _reduced_rhs(factor, contribs, tip, k)
        red_x = bta.solve(factor.reduced_factor, red_rhs)
        x_tip = red_x[len(factor.separators) * b :]
        parts = []
        for p in range(len(ranges)):
            xl, xr_ = _sep_solution(factor, red_x, p)
            parts.append(torch.cat([t.reshape(-1) for t in (xl, xr_, x_tip) if t is not None]))
    mine = _scatter_flat(parts, out_sizes[rank], root, group, ch.device).view(-1, k)
    o = 0
    xl = xr_ = None
    if ch.left is not None:
        xl, o = mine[o : o + b], o + b
    if ch.right is not None:
        xr_, o = mine[o : o + b], o + b
    x_tip = mine[o : o + a]
    rows = ch.solve_backward(z, xl, xr_, x_tip)
    if squeeze:
        return rows.reshape(-1), x_tip.reshape(-1)
    return rows, x_tip


def d_selected_invert_nccl(factor):
    """PPOBTASI with one partition per rank: the root's reduced selected
    inverse sends each rank the separator / fill / tip entries its interior
    recursion starts from; returns this rank's inverse rows (BTARows, tip on
    the root)."""
    dist = _dist()
    group, root = factor.group, factor.root
    rank = dist.get_rank(group)
    ch = factor.partitions[0]
    b, a = factor.block_size, factor.arrow_size
    ranges = _partition_ranges(factor.plan)

    def seed_sizes(p):
        lo, hi, left, right = ranges[p]
        sz = {"X_tip": a * a, "Xd_left": b * b, "Xa_left": a * b, "X_prev": b * b,
              "Xd_right": b * b, "Xa_right": a * b, "X_fill": b * b}
        have = set()
        if a > 0:
            have.add("X_tip")
        if left is not None:
            have |= {"Xd_left", "Xa_left"}
            if factor.sep_pos[left] > 0:
                have.add("X_prev")
        if right is not None:
            have |= {"Xd_right", "Xa_right"}
            if left is not None:
                have.add("X_fill")
        return [(k, sz[k]) for k in _SEED_ORDER if k in have]

    parts = None
    red_tip = None
    if rank == root:
        red = bta.selected_invert(factor.reduced_factor)
        red_tip = red.tip.clone() if a else None
        parts = []
        for p in range(len(ranges)):
            s = _seeds(factor, red, p)
            parts.append(torch.cat([s[k].reshape(-1) for k, _ in seed_sizes(p)]) if s else
                         torch.zeros(0, dtype=torch.float64, device=ch.device))
    lay = seed_sizes(rank)
    mine = _scatter_flat(parts, sum(s for _, s in lay), root, group, ch.device)
    seeds, o = {}, 0
    shapes = {"X_tip": (a, a), "Xa_left": (a, b), "Xa_right": (a, b)}
    for k, s in lay:
        seeds[k] = mine[o : o + s].view(*shapes.get(k, (b, b)))
        o += s
    rows = ch.invert(seeds)
    rows.n_blocks = factor.n_blocks
    if rank == root and a:
        rows.tip = red_tip
    return rows
