"""Coregionalization, the time-major permutation and the sparse -> BTA scatter.

Mirrors the reference (pkg/src/stinla/coreg.py) on the host side — mixing
algebra, ``PermutationMap`` and its per-nonzero storage offsets — and moves
the per-evaluation work to the device:

* :func:`map_to_bta` uploads the values of an assembled CSR matrix and
  scatters them with the tiled zero-fill + scatter kernel (``stbta_assemble``).
* :class:`AssemblyPlan` is the hot path used by the objective evaluator: the
  theta -> Q value map is frozen at construction as (offset, pair, source)
  triplets over a fixed basis table, so an evaluation uploads only a
  ``pairs x terms`` coefficient table and the kernel writes Q_p / Q_c straight
  into BTA storage (reference coreg.py:80-121 + model.py:196-248 +
  inla.py:264-283 + coreg.py:250-276 fused into one HBM pass).
"""

from dataclasses import dataclass

import ctypes

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .model import ST_TERMS, TIP_TERM, DimensionError, st_basis


class EnvelopeError(ValueError):
    """A structural nonzero falls outside the BTA envelope (coreg.py:12-14)."""


def coupling_positions(n_processes):
    """Strictly-lower (row, col) slots of the couplings, nearest predecessor
    first (coreg.py:17-28)."""
    return [(i, j) for i in range(1, n_processes) for j in range(i - 1, -1, -1)]


@dataclass
class Coregionalization:
    """Linear mixing of unit-variance processes (coreg.py:31-77)."""

    scales: np.ndarray
    couplings: np.ndarray

    def __post_init__(self):
        self.scales = np.asarray(self.scales, dtype=np.float64).ravel()
        self.couplings = np.asarray(self.couplings, dtype=np.float64).ravel()
        nv = self.scales.size
        if self.couplings.size != nv * (nv - 1) // 2:
            raise DimensionError(
                f"{nv} processes require {nv * (nv - 1) // 2} couplings, "
                f"got {self.couplings.size}"
            )
        if np.any(self.scales <= 0):
            raise ValueError("coregionalization scales must be strictly positive")

    @property
    def n_processes(self):
        return self.scales.size

    def _lam(self):
        nv = self.n_processes
        lam = np.zeros((nv, nv))
        for value, (i, j) in zip(self.couplings, coupling_positions(nv)):
            lam[i, j] = value
        return lam

    def mixing(self):
        nv = self.n_processes
        return np.linalg.solve(np.eye(nv) - self._lam(), np.eye(nv)) @ np.diag(self.scales)

    def mixing_inverse(self):
        nv = self.n_processes
        return np.diag(1.0 / self.scales) @ (np.eye(nv) - self._lam())


def pair_weights(linv):
    """w[k, i, j] = Linv[k, i] * Linv[k, j] for k >= max(i, j), else 0 — the
    scalar weight of process k's precision in joint block (i, j)
    (coreg.py:104-107)."""
    nv = linv.shape[0]
    w = np.zeros((nv, nv, nv))
    for i in range(nv):
        for j in range(i + 1):
            for k in range(i, nv):
                w[k, i, j] = w[k, j, i] = linv[k, i] * linv[k, j]
    return w


def assemble_joint_precision(precisions, coreg):
    """Host joint precision (coreg.py:80-121): block (i, j) =
    sum_{k >= max(i,j)} Linv[k,i] Linv[k,j] Q_k, all structural terms kept."""
    nv = len(precisions)
    if coreg.n_processes != nv:
        raise DimensionError(
            f"coregionalization has {coreg.n_processes} processes, got {nv} precisions"
        )
    dim = precisions[0].shape[0]
    if any(q.shape != (dim, dim) for q in precisions):
        raise DimensionError("all univariate precisions must share their dimension")
    w = pair_weights(coreg.mixing_inverse())
    coo = [sp.coo_matrix(q) for q in precisions]
    rows, cols, vals = [], [], []
    for i in range(nv):
        for j in range(nv):
            for k in range(max(i, j), nv):
                rows.append(coo[k].row + i * dim)
                cols.append(coo[k].col + j * dim)
                vals.append(w[k, i, j] * coo[k].data)
    out = sp.coo_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(nv * dim, nv * dim),
    ).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


@dataclass
class _BoundScatter:
    """Per-nonzero storage offsets of one bound CSR pattern (coreg.py:124-130)."""

    kept: np.ndarray
    offsets: np.ndarray
    nnz: int
    _device: dict = None

    def device_tables(self, device, nstore):
        """(sorted offsets, permutation into kept order, tile starts) on device."""
        if self._device is None:
            self._device = {}
        key = (str(device), nstore)
        if key not in self._device:
            order = np.argsort(self.offsets, kind="stable")
            off = self.offsets[order]
            tile = _lib.ASM_TILE
            starts = np.searchsorted(off, np.arange(0, nstore + tile, tile, dtype=np.int64)[
                : (nstore + tile - 1) // tile + 1])
            self._device[key] = (
                torch.from_numpy(off).to(device),
                torch.from_numpy(self.kept[order].astype(np.int32)).to(device),
                torch.from_numpy(starts.astype(np.int64)).to(device),
            )
        return self._device[key]


class PermutationMap:
    """Variable-major -> time-major (BTA) reordering (coreg.py:133-241).

    ``forward[old] = new``; :meth:`bind` precomputes one flat storage offset
    per nonzero of a CSR pattern that lands in the lower BTA envelope.
    """

    def __init__(self, n_processes, n_spatial, n_time, n_fixed):
        self.n_processes, self.n_spatial = n_processes, n_spatial
        self.n_time, self.n_fixed = n_time, n_fixed
        self.n_blocks = n_time
        self.block_size = n_processes * n_spatial
        self.arrow_size = n_processes * n_fixed
        self.dim = self.n_blocks * self.block_size + self.arrow_size
        per = n_spatial * n_time + n_fixed
        v, local = np.divmod(np.arange(n_processes * per, dtype=np.int64), per)
        t, s = np.divmod(local, n_spatial)
        st_part = local < n_spatial * n_time
        fwd = np.where(
            st_part,
            t * self.block_size + v * n_spatial + s,
            n_processes * n_spatial * n_time + v * n_fixed + (local - n_spatial * n_time),
        )
        self.forward = fwd.astype(np.int64)
        self.backward = np.argsort(self.forward)
        self._bound = None

    def permute_vector(self, x):
        x = np.asarray(x)
        out = np.empty_like(x)
        out[self.forward] = x
        return out

    def restore_vector(self, x):
        return np.asarray(x)[self.forward]

    def permuted_matrix(self, matrix):
        m = sp.csr_matrix(matrix)
        return m[self.backward][:, self.backward].tocsr()

    def offsets_of(self, rows, cols):
        """Storage offsets of (row, col) pairs in variable-major indices;
        -1 for strictly-upper blocks.  Raises EnvelopeError outside the band."""
        n, b, a = self.n_blocks, self.block_size, self.arrow_size
        pr, pc = self.forward[rows], self.forward[cols]
        split = n * b
        st_r, st_c = pr < split, pc < split
        tr, tc = pr // b, pc // b
        both = st_r & st_c
        bad = both & (np.abs(tr - tc) >= 2)
        if np.any(bad):
            k = int(np.flatnonzero(bad)[0])
            raise EnvelopeError(
                f"nonzero at ({rows[k]}, {cols[k]}) maps to time blocks "
                f"({tr[k]}, {tc[k]}), outside the block-tridiagonal envelope"
            )
        off = np.full(pr.shape[0], -1, dtype=np.int64)
        base_lo = n * b * b
        base_ar = base_lo + (n - 1) * b * b
        base_tip = base_ar + n * a * b
        m = both & (tr == tc)
        off[m] = tr[m] * b * b + (pr[m] % b) * b + pc[m] % b
        m = both & (tr == tc + 1)
        off[m] = base_lo + tc[m] * b * b + (pr[m] % b) * b + pc[m] % b
        m = ~st_r & st_c
        off[m] = base_ar + tc[m] * a * b + (pr[m] - split) * b + pc[m] % b
        m = ~st_r & ~st_c
        off[m] = base_tip + (pr[m] - split) * a + (pc[m] - split)
        return off

    def bind(self, pattern):
        pattern = sp.csr_matrix(pattern)
        if pattern.shape != (self.dim, self.dim):
            raise DimensionError(f"pattern is {pattern.shape}, expected ({self.dim}, {self.dim})")
        rows = np.repeat(np.arange(self.dim, dtype=np.int64), np.diff(pattern.indptr))
        off = self.offsets_of(rows, pattern.indices.astype(np.int64))
        kept = np.flatnonzero(off >= 0)
        return _BoundScatter(kept=kept, offsets=off[kept], nnz=pattern.nnz)


def build_permutation(spec):
    return PermutationMap(spec.n_processes, spec.n_spatial, spec.n_time, spec.n_fixed)


def map_to_bta(matrix, pmap, workspace, bound=None, stream=None):
    """Scatter an assembled symmetric CSR matrix into a device BTA workspace
    (coreg.py:250-276).  Values are uploaded once and written by the tiled
    zero-fill + scatter kernel; positions outside the pattern become zero."""
    matrix = sp.csr_matrix(matrix)
    if (workspace.n_blocks, workspace.block_size, workspace.arrow_size) != (
        pmap.n_blocks, pmap.block_size, pmap.arrow_size,
    ):
        raise DimensionError("workspace envelope does not match the permutation map")
    if bound is None:
        if pmap._bound is None or pmap._bound.nnz != matrix.nnz:
            pmap._bound = pmap.bind(matrix)
        bound = pmap._bound
    elif bound.nnz != matrix.nnz:
        raise DimensionError("bound scatter was built for a different pattern")
    dev = workspace.device
    nstore = workspace.data.numel()
    off_d, kept_d, starts_d = bound.device_tables(dev, nstore)
    lib = _lib.load()
    with torch.cuda.device(dev):
        vals = torch.from_numpy(np.ascontiguousarray(matrix.data, dtype=np.float64)).to(dev)
        one = torch.ones(1, dtype=torch.float64, device=dev)
        zero_pairs = torch.zeros(kept_d.numel(), dtype=torch.int32, device=dev)
        # value(e) = coef[0][0] * basis[kept[e]][0]: the uploaded CSR values act
        # as a one-term basis table indexed by the kept nonzero positions
        _lib.check(
            lib.stbta_assemble(
                _lib.ptr(workspace.data), nstore, _lib.ptr(starts_d), _lib.ptr(off_d),
                _lib.ptr(zero_pairs), _lib.ptr(kept_d), _lib.ptr(vals), _lib.ptr(one), 1,
                _lib.stream_ptr(stream),
            ),
            "stbta_assemble",
        )
    workspace._scatter_source = bound
    return workspace


def _pair_index(i, j):
    i, j = max(i, j), min(i, j)
    return i * (i + 1) // 2 + j


def _same_discretization(spec):
    ref_s, ref_t = spec.spatial[0], spec.temporal[0]
    for sd, td in zip(spec.spatial[1:], spec.temporal[1:]):
        for x, y in (
            (sd.mass, ref_s.mass), (sd.stiffness, ref_s.stiffness), (td.mass, ref_t.mass),
            (td.coupling, ref_t.coupling), (td.stiffness, ref_t.stiffness),
        ):
            if x.shape != y.shape or abs(x - y).sum() != 0:
                return False
    return True


def padded_storage_elems(n, b, a, ldb):
    """diag | lower | arrow with row stride ldb, then the a x a tip."""
    return ((2 * n - 1) * b + n * a) * ldb + a * a


def pad_offsets(off, n, b, a, ldb):
    """Map flat reference-layout offsets (coreg.py:219-241 / BTAMatrix) to the
    row-padded layout: every diag / lower / arrow row is one storage row of
    length b; the tip is stored unchanged after them."""
    if ldb == b:
        return off
    off = np.asarray(off, dtype=np.int64)
    rows_total = (2 * n - 1) * b + n * a
    split = rows_total * b
    out = np.empty_like(off)
    blk = off < split
    r, c = np.divmod(off[blk], b)
    out[blk] = r * ldb + c
    out[~blk] = rows_total * ldb + (off[~blk] - split)
    return out


class AssemblyPlan:
    """theta -> (Q_p, Q_c) values in BTA storage, as one device kernel.

    Construction (host, once per model): the local basis of every process —
    9 SPDE Kronecker terms (:func:`model.st_basis`), the fixed-effect identity
    and the per-response Gram matrix A_i^T A_i (inla.py:195-203) — is laid out
    as a table ``basis[src][term]`` over the union of their local patterns;
    every nonzero of the joint conditional pattern that lands in the lower BTA
    envelope becomes an entry (storage offset, process pair, src), sorted by
    offset.  Q_p uses the same entries with zero Gram coefficients (its
    pattern is a subset of Q_c's, the extra slots are zero in the reference's
    workspace too).

    Per evaluation the host builds the ``pairs x terms`` coefficient tables
    (:meth:`coefficients`), and :meth:`assemble` launches ``stbta_assemble``.
    """

    def __init__(self, spec, pmap, grams, device):
        self.spec, self.pmap, self.device = spec, pmap, torch.device(device)
        nv, nl = spec.n_processes, spec.latent_per_process
        nst, nf = spec.n_spatial * spec.n_time, spec.n_fixed
        self.shared = _same_discretization(spec)
        nbases = 1 if self.shared else nv
        self.n_pairs = nv * (nv + 1) // 2
        self.gram_col0 = 10 * nbases
        self.n_terms = self.gram_col0 + (nv if grams else 0)

        def pad(m):
            m = sp.coo_matrix(m)
            return sp.csr_matrix((m.data, (m.row, m.col)), shape=(nl, nl))

        # local basis matrices per column of the basis table
        cols = []
        for k in range(nbases):
            for bmat in st_basis(spec.spatial[k], spec.temporal[k]):
                cols.append(pad(bmat))
            tip = sp.csr_matrix(
                (np.ones(nf), (np.arange(nst, nl), np.arange(nst, nl))), shape=(nl, nl)
            )
            cols.append(tip)
        for g in grams:
            cols.append(sp.csr_matrix(g, shape=(nl, nl)))
        assert len(cols) == self.n_terms

        # union local pattern and its sorted keys
        union = None
        for m in cols:
            s = abs(m).astype(bool).astype(np.float64)
            union = s if union is None else union + s
        union = sp.csr_matrix(union)
        union.sum_duplicates()
        union.sort_indices()
        urow = np.repeat(np.arange(nl, dtype=np.int64), np.diff(union.indptr))
        ukeys = urow * nl + union.indices.astype(np.int64)
        table = np.zeros((ukeys.size, self.n_terms))
        for t, m in enumerate(cols):
            m = sp.coo_matrix(m)
            keys = m.row.astype(np.int64) * nl + m.col.astype(np.int64)
            np.add.at(table[:, t], np.searchsorted(ukeys, keys), m.data)

        # structural pattern of each ordered process pair (i, j): the union of
        # the local patterns of the terms that feed joint block (i, j)
        member = []
        for m in cols:
            m = sp.coo_matrix(m)
            keys = m.row.astype(np.int64) * nl + m.col.astype(np.int64)
            member.append(np.unique(np.searchsorted(ukeys, keys)))
        offs, pairs, srcs = [], [], []
        for i in range(nv):
            for j in range(nv):
                terms = []
                for k in range(max(i, j), nv):
                    kk = 0 if self.shared else k
                    terms += list(range(10 * kk, 10 * kk + 10))
                if i == j and grams:
                    terms.append(self.gram_col0 + i)
                s_idx = np.unique(np.concatenate([member[t] for t in sorted(set(terms))]))
                r_loc, c_loc = np.divmod(ukeys[s_idx], nl)
                off = pmap.offsets_of(r_loc + i * nl, c_loc + j * nl)
                keep = off >= 0
                offs.append(off[keep])
                srcs.append(s_idx[keep].astype(np.int32))
                pairs.append(np.full(int(keep.sum()), _pair_index(i, j), dtype=np.int32))
        off = np.concatenate(offs)
        order = np.argsort(off, kind="stable")
        off = off[order]
        if off.size > 1 and np.any(off[1:] == off[:-1]):
            raise EnvelopeError("two structural nonzeros map to the same storage slot")
        self.n_entries = int(off.size)
        n, b, a = pmap.n_blocks, pmap.block_size, pmap.arrow_size
        self.nstore_flat = n * b * b + (n - 1) * b * b + n * a * b + a * a
        # device workspaces pad odd block rows to an even stride, so every row
        # of diag / lower / arrow is 16-byte aligned for the kernels' vector
        # copies (C3: b = 5025); the padding column stays zero.
        self.ldb = b + (b % 2)
        self.nstore = padded_storage_elems(n, b, a, self.ldb)
        poff = pad_offsets(off, n, b, a, self.ldb)
        tile = _lib.ASM_TILE
        ntiles = (self.nstore + tile - 1) // tile
        starts = np.searchsorted(poff, np.arange(ntiles + 1, dtype=np.int64) * tile)
        # does any entry of the conditional pattern sit in an arrow block?
        base_ar = n * b * b + (n - 1) * b * b
        self.cond_has_arrow = bool(a > 0 and np.any((off >= base_ar) & (off < base_ar + n * a * b)))
        dev = self.device
        self.h_offsets = off
        self.h_pair = np.concatenate(pairs)[order]
        self.h_src = np.concatenate(srcs)[order]
        self.h_basis = table
        self.d_offsets = torch.from_numpy(off).to(dev)  # flat layout (quadform)
        self.d_poffsets = torch.from_numpy(poff).to(dev) if self.ldb != b else self.d_offsets
        self.d_pair = torch.from_numpy(self.h_pair).to(dev)
        self.d_src = torch.from_numpy(self.h_src).to(dev)
        self.d_basis = torch.from_numpy(np.ascontiguousarray(table)).to(dev)
        self.d_starts = torch.from_numpy(starts.astype(np.int64)).to(dev)
        self.table_bytes = int(
            off.nbytes + 8 * off.size + table.nbytes + starts.nbytes
        )

    def coefficients(self, process_hypers, linv, taus):
        """(coef_p, coef_c) host tables of shape (pairs, terms)."""
        spec = self.spec
        nv = spec.n_processes
        from .model import st_coefficients

        cp = np.zeros((self.n_pairs, self.n_terms))
        w = pair_weights(linv) if nv > 1 else np.ones((1, 1, 1))
        for i in range(nv):
            for j in range(i + 1):
                p = _pair_index(i, j)
                for k in range(i, nv):
                    c = st_coefficients(process_hypers[k])
                    col = 0 if self.shared else 10 * k
                    with np.errstate(over="ignore", invalid="ignore"):
                        cp[p, col : col + ST_TERMS] += w[k, i, j] * c
                        cp[p, col + TIP_TERM] += w[k, i, j] * spec.fixed_effect_precision
        cc = cp.copy()
        if self.n_terms > self.gram_col0:
            for i in range(nv):
                cc[_pair_index(i, i), self.gram_col0 + i] = taus[i]
        return cp, cc

    def rows_plan(self, t0, t1, with_tip, device):
        """Assembly of block rows [t0, t1) only (one time partition, S3): the
        entries whose storage slots fall in those rows (plus the tip when
        ``with_tip``), re-addressed into a :class:`~.bta_dist.BTARows` flat
        buffer ``diag (m,b,b) | lower (m,b,b) | arrow (m,a,b) [| tip (a,a)]``
        with ``lower[j] = A(t0+j, t0+j-1)``; same basis table and coefficients."""
        return _RowsAssembly(self, t0, t1, with_tip, device)

    def assemble_host(self, coef):
        """numpy evaluation of what :meth:`assemble` writes, in the flat
        reference layout (host checks)."""
        out = np.zeros(self.nstore_flat)
        vals = np.einsum("et,et->e", coef[self.h_pair], self.h_basis[self.h_src])
        out[self.h_offsets] = vals
        return out

    def regions(self, data):
        """(diag, lower, arrow, tip) device pointers of a padded workspace."""
        n, b, a, ld = self.pmap.n_blocks, self.pmap.block_size, self.pmap.arrow_size, self.ldb
        base = data.data_ptr()
        lo = base + 8 * n * b * ld
        ar = lo + 8 * (n - 1) * b * ld
        tp = ar + 8 * n * a * ld
        return [ctypes.c_void_p(p) for p in (base, lo, ar, tp)]

    def unpad(self, data):
        """Flat reference-layout copy of a padded workspace (tests / views)."""
        n, b, a, ld = self.pmap.n_blocks, self.pmap.block_size, self.pmap.arrow_size, self.ldb
        if ld == b:
            return data
        rows = (2 * n - 1) * b + n * a
        blocks = data[: rows * ld].view(rows, ld)[:, :b].reshape(-1)
        return torch.cat([blocks, data[rows * ld : rows * ld + a * a]])

    def assemble(self, data, coef_dev, stream=None):
        lib = _lib.load()
        _lib.check(
            lib.stbta_assemble(
                _lib.ptr(data), self.nstore, _lib.ptr(self.d_starts), _lib.ptr(self.d_poffsets),
                _lib.ptr(self.d_pair), _lib.ptr(self.d_src), _lib.ptr(self.d_basis),
                _lib.ptr(coef_dev), self.n_terms, _lib.stream_ptr(stream),
            ),
            "stbta_assemble",
        )

    def quadform(self, coef_dev, x, partial, out, stream=None):
        lib = _lib.load()
        pm = self.pmap
        _lib.check(
            lib.stbta_quadform(
                _lib.ptr(self.d_offsets), _lib.ptr(self.d_pair), _lib.ptr(self.d_src),
                _lib.ptr(self.d_basis), _lib.ptr(coef_dev), self.n_terms, self.n_entries,
                pm.n_blocks, pm.block_size, pm.arrow_size, _lib.ptr(x), _lib.ptr(partial),
                partial.numel(), _lib.ptr(out), _lib.stream_ptr(stream),
            ),
            "stbta_quadform",
        )


class _RowsAssembly:
    """Per-partition slice of an :class:`AssemblyPlan` (see ``rows_plan``)."""

    def __init__(self, plan, t0, t1, with_tip, device):
        pm = plan.pmap
        n, b, a = pm.n_blocks, pm.block_size, pm.arrow_size
        self.t0, self.t1, self.with_tip = t0, t1, with_tip
        self.n, self.b, self.a = n, b, a
        self.device = torch.device(device)
        m, bb, ab = t1 - t0, b * b, a * b
        e0 = n * bb
        e1 = e0 + (n - 1) * bb
        e2 = e1 + n * ab
        off = plan.h_offsets
        new = np.full(off.shape, -1, dtype=np.int64)
        sel = (off >= t0 * bb) & (off < t1 * bb)  # diag rows
        new[sel] = off[sel] - t0 * bb
        lo_end = e0 + (t1 - 1) * bb  # lower blocks g = t-1 for rows t in [max(t0,1), t1)
        lo_beg = e0 + (max(t0, 1) - 1) * bb
        sel = (off >= lo_beg) & (off < lo_end)
        new[sel] = m * bb + (off[sel] - e0) - (t0 - 1) * bb
        sel = (off >= e1 + t0 * ab) & (off < e1 + t1 * ab)
        new[sel] = 2 * m * bb + (off[sel] - e1 - t0 * ab)
        if with_tip:
            sel = off >= e2
            new[sel] = 2 * m * bb + m * ab + (off[sel] - e2)
        keep = new >= 0
        self.nstore = 2 * m * bb + m * ab + (a * a if with_tip else 0)
        order = np.argsort(new[keep], kind="stable")
        offs = new[keep][order]
        tile = _lib.ASM_TILE
        ntiles = (self.nstore + tile - 1) // tile
        starts = np.searchsorted(offs, np.arange(ntiles + 1, dtype=np.int64) * tile)
        dev = self.device
        self.n_terms = plan.n_terms
        self.d_offsets = torch.from_numpy(offs).to(dev)
        self.d_pair = torch.from_numpy(plan.h_pair[keep][order]).to(dev)
        self.d_src = torch.from_numpy(plan.h_src[keep][order]).to(dev)
        self.d_basis = plan.d_basis.to(dev)
        self.d_starts = torch.from_numpy(starts.astype(np.int64)).to(dev)

    def new_rows(self):
        """A BTARows over a fresh flat buffer of this slice's layout."""
        from .bta_dist import BTARows

        buf = torch.empty(self.nstore, dtype=torch.float64, device=self.device)
        return BTARows(self.n, self.t0, self.t1, self.b, self.a, self.device,
                       with_tip=self.with_tip, data=buf)

    def assemble(self, rows, coef_dev, stream=None):
        """Zero-fill + scatter the slice's values into ``rows.data``."""
        lib = _lib.load()
        _lib.check(
            lib.stbta_assemble(
                _lib.ptr(rows.data), self.nstore, _lib.ptr(self.d_starts),
                _lib.ptr(self.d_offsets), _lib.ptr(self.d_pair), _lib.ptr(self.d_src),
                _lib.ptr(self.d_basis), _lib.ptr(coef_dev), self.n_terms,
                _lib.stream_ptr(stream)),
            "stbta_assemble",
        )
        return rows
