"""Device-resident BTA matrices and the sequential structured solver.

Drop-in mirror of the reference solver API (``stinla.bta``,
pkg/src/stinla/bta.py): same class / function names, argument meaning and
exceptions, but the flat block buffer lives in HBM (a float64 torch tensor)
and every operation is one call into the sm_100a library ``libstbta.so``:

=================  =========================  ==============================
reference           here                       C ABI (include/stbta.h)
=================  =========================  ==============================
bta.py:177-235      :func:`factorize`          ``stbta_pobtaf`` (+ fused logdet)
bta.py:238-246      :func:`logdet`             value produced by ``stbta_pobtaf``
bta.py:249-307      :func:`solve` & co.        ``stbta_pobtas``
bta.py:310-359      :func:`selected_invert`    ``stbta_pobtasi``
=================  =========================  ==============================

There is no CPU fallback: without the library or a CUDA device every call
raises :class:`~paper_2507_06938_b200._lib.StbtaError`.
"""

import os

import numpy as np
import torch

from . import _lib


class FactorizationError(RuntimeError):
    """A pivot block was not positive definite (reference bta.py:17-31).

    ``block_index`` is the time block (``n_blocks`` for the arrow tip) and
    ``partition`` the partition of a partitioned factorization (-1 for the
    reduced system), exactly as in the reference.
    """

    def __init__(self, block_index, partition=None):
        self.block_index = block_index
        self.partition = partition
        where = f"block {block_index}"
        if partition is not None:
            where += f" (partition {partition})"
        super().__init__(f"non-positive-definite pivot at {where}")


class OpCounter:
    """Modeled elimination cost in cubic block units (reference bta.py:34-47)."""

    def __init__(self):
        self.flops = 0.0

    def charge(self, units):
        self.flops += float(units)


_SIDE_STREAMS = {}


def _side_stream(dev, role):
    """One cached side stream per (device, role) for the pipelined copies."""
    dev = torch.device(dev)
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), role)
    st = _SIDE_STREAMS.get(key)
    if st is None:
        st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=key[0])
    return st


_MEMOPS = None


def _memops_supported():
    global _MEMOPS
    if _MEMOPS is None:
        try:
            _MEMOPS = bool(torch.cuda.is_available() and _lib.load().stbta_stream_memops_supported())
        except Exception:
            _MEMOPS = False
    return _MEMOPS


def default_device():
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def _storage_elems(n, b, a):
    return n * b * b + (n - 1) * b * b + n * a * b + a * a


class BTAMatrix:
    """Lower-triangle block storage of a symmetric BTA matrix, in HBM.

    The flat ``data`` tensor is ordered ``diag (n,b,b) | lower (n-1,b,b) |
    arrow (n,a,b) | tip (a,a)``, row-major, identical to the reference
    (bta.py:50-89); ``diag``/``lower``/``arrow``/``tip`` are views of it.
    ``data`` may be given as a numpy array (copied to the device) or as a
    CUDA float64 tensor (aliased).
    """

    def __init__(self, n_blocks, block_size, arrow_size=0, data=None, device=None):
        if n_blocks < 1 or block_size < 1 or arrow_size < 0:
            raise ValueError(
                f"invalid BTA shape (n_blocks={n_blocks}, block_size={block_size}, "
                f"arrow_size={arrow_size})"
            )
        self.n_blocks, self.block_size, self.arrow_size = n_blocks, block_size, arrow_size
        total = _storage_elems(n_blocks, block_size, arrow_size)
        self._upload = None      # (ready flags, done event, host source) of a pipelined upload
        self._host_copy = None   # (pinned host tensor, done event) of a streamed-out result
        if data is None:
            dev = torch.device(device) if device is not None else default_device()
            data = torch.zeros(total, dtype=torch.float64, device=dev)
        elif isinstance(data, torch.Tensor):
            if data.dtype != torch.float64:
                raise ValueError("data must be a float64 tensor")
            if data.numel() != total or data.dim() != 1 or not data.is_contiguous():
                raise ValueError(f"data buffer must have {total} entries")
            if not data.is_cuda:  # host tensor: copied (pipelined per time block when pinned)
                dev = torch.device(device) if device is not None else default_device()
                if data.is_pinned() and _memops_supported():
                    data = self._start_upload(data, dev)
                else:
                    data = data.to(dev, non_blocking=data.is_pinned())
        else:
            arr = np.asarray(data, dtype=np.float64)
            if arr.shape != (total,):
                raise ValueError(f"data buffer must have {total} entries")
            dev = torch.device(device) if device is not None else default_device()
            data = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        self._data = data
        self._scatter_source = None

    def _start_upload(self, host, dev):
        """Chunked H2D copy on a side stream; per-block flags let POBTAF start
        before the upload has finished (stbta_upload_blocks / stbta_pobtaf_ready)."""
        lib = _lib.load()
        n, b, a = self.n_blocks, self.block_size, self.arrow_size
        with torch.cuda.device(dev):
            cur = torch.cuda.current_stream()
            dst = torch.empty(host.numel(), dtype=torch.float64, device=dev)
            flags = torch.zeros(n, dtype=torch.int32, device=dev)
            up = _side_stream(dev, "upload")
            up.wait_stream(cur)  # allocation + flag zeroing precede the copies
            _lib.check(
                lib.stbta_upload_blocks(_lib.ptr(dst), host.data_ptr(), n, b, a, _lib.ptr(flags), 1,
                                        up.cuda_stream),
                "stbta_upload_blocks",
            )
            done = torch.cuda.Event()
            done.record(up)
            dst.record_stream(up)
            flags.record_stream(up)
        self._upload = (flags, done, host)
        return dst

    @property
    def data(self):
        """The flat device buffer; waits (stream-ordered) for a pending upload."""
        if self._upload is not None:
            torch.cuda.current_stream(self._data.device).wait_event(self._upload[1])
        return self._data

    @property
    def diag(self):
        n, b = self.n_blocks, self.block_size
        return self.data[: n * b * b].view(n, b, b)

    @diag.setter
    def diag(self, value):  # `m.diag += x` / `m.diag = x` write through to the buffer
        view = self.diag
        if value is not view:
            view.copy_(value)

    @property
    def lower(self):
        n, b = self.n_blocks, self.block_size
        e0 = n * b * b
        return self.data[e0 : e0 + (n - 1) * b * b].view(n - 1, b, b)

    @lower.setter
    def lower(self, value):  # `m.lower += x` / `m.lower = x` write through to the buffer
        view = self.lower
        if value is not view:
            view.copy_(value)

    @property
    def arrow(self):
        n, b, a = self.n_blocks, self.block_size, self.arrow_size
        e1 = (2 * n - 1) * b * b
        return self.data[e1 : e1 + n * a * b].view(n, a, b)

    @arrow.setter
    def arrow(self, value):  # `m.arrow += x` / `m.arrow = x` write through to the buffer
        view = self.arrow
        if value is not view:
            view.copy_(value)

    @property
    def tip(self):
        n, b, a = self.n_blocks, self.block_size, self.arrow_size
        e2 = (2 * n - 1) * b * b + n * a * b
        return self.data[e2:].view(a, a)

    @tip.setter
    def tip(self, value):  # `m.tip += x` / `m.tip = x` write through to the buffer
        view = self.tip
        if value is not view:
            view.copy_(value)

    @property
    def dim(self):
        return self.n_blocks * self.block_size + self.arrow_size

    @property
    def device(self):
        return self._data.device

    def copy(self):
        return BTAMatrix(self.n_blocks, self.block_size, self.arrow_size, self.data.clone())

    def zero(self):
        self.data.zero_()
        self._scatter_source = None
        return self

    def numpy(self, out=None):
        """Host copy of the flat buffer; ``out`` may be a (pinned) CPU float64
        tensor of the same size that receives the copy (when it is the buffer
        this matrix was already streamed into, only the copy is awaited)."""
        if self._host_copy is not None and out is self._host_copy[0]:
            self._host_copy[1].synchronize()
            return out.numpy()
        if out is not None:
            out.copy_(self.data)
            return out.numpy()
        return self.data.detach().cpu().numpy()

    def to_dense(self):
        """Densified host matrix (oracles / debugging only)."""
        n, b, a = self.n_blocks, self.block_size, self.arrow_size
        d = self.numpy()
        out = np.zeros((self.dim, self.dim))
        e0 = n * b * b
        e1 = e0 + (n - 1) * b * b
        e2 = e1 + n * a * b
        diag = d[:e0].reshape(n, b, b)
        lower = d[e0:e1].reshape(n - 1, b, b)
        arrow = d[e1:e2].reshape(n, a, b)
        for i in range(n):
            s = slice(i * b, (i + 1) * b)
            out[s, s] = diag[i]
            if i + 1 < n:
                t = slice((i + 1) * b, (i + 2) * b)
                out[t, s] = lower[i]
                out[s, t] = lower[i].T
            if a:
                out[n * b :, s] = arrow[i]
                out[s, n * b :] = arrow[i].T
        if a:
            out[n * b :, n * b :] = d[e2:].reshape(a, a)
        return out

    @classmethod
    def from_dense(cls, dense, n_blocks, block_size, arrow_size=0, device=None):
        dense = np.asarray(dense, dtype=np.float64)
        n, b, a = n_blocks, block_size, arrow_size
        if dense.shape != (n * b + a, n * b + a):
            raise ValueError("dense matrix does not match the BTA envelope")
        flat = np.zeros(_storage_elems(n, b, a))
        e0 = n * b * b
        e1 = e0 + (n - 1) * b * b
        e2 = e1 + n * a * b
        diag = flat[:e0].reshape(n, b, b)
        lower = flat[e0:e1].reshape(n - 1, b, b)
        arrow = flat[e1:e2].reshape(n, a, b)
        for i in range(n):
            diag[i] = dense[i * b : (i + 1) * b, i * b : (i + 1) * b]
            if i + 1 < n:
                lower[i] = dense[(i + 1) * b : (i + 2) * b, i * b : (i + 1) * b]
            if a:
                arrow[i] = dense[n * b :, i * b : (i + 1) * b]
        if a:
            flat[e2:] = dense[n * b :, n * b :].ravel()
        return cls(n, b, a, flat, device=device)


class BTAFactor:
    """Cholesky factor stored in the matrix's own blocks (reference bta.py:165-174).

    ``logdet_dev`` / ``info_dev`` are the device scalars written by the
    factorization kernel chain.
    """

    def __init__(self, matrix, has_arrow, logdet_dev=None, info_dev=None):
        self.matrix = matrix
        self.has_arrow = has_arrow
        self.logdet_dev = logdet_dev
        self.info_dev = info_dev
        self._logdet = None
        self._si_ws = None  # POBTASI workspace holding W_t = L_tt^-1 (prepare_inverse)

    @property
    def dim(self):
        return self.matrix.dim


def _workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _arrow_nonzero(matrix):
    """The reference's `a > 0 and np.any(arrow)` test (bta.py:202), on device."""
    if matrix.arrow_size == 0:
        return False
    return bool(torch.any(matrix.arrow != 0).item())


def factorize_async(matrix, use_arrow, stream=None):
    """Issue POBTAF on `stream` without synchronising.

    Returns ``(logdet_dev, info_dev)``; ``info_dev`` holds 1 + failing block.
    """
    lib = _lib.load()
    n, b, a = matrix.n_blocks, matrix.block_size, matrix.arrow_size
    dev = matrix.device
    ws = _workspace(lib.stbta_pobtaf_workspace_bytes(n, b, a), dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    matrix._scatter_source = None
    if matrix._upload is not None and not matrix._upload[1].query() and stream is None:
        # the upload is still in flight: the task graph waits per time block
        flags = matrix._upload[0]
        _lib.check(
            lib.stbta_pobtaf_ready(
                _lib.ptr(matrix._data), n, b, a, int(bool(use_arrow)), _lib.ptr(out),
                _lib.ptr(info), _lib.ptr(flags), 1, _lib.ptr(ws), ws.numel(), _lib.stream_ptr(None),
            ),
            "stbta_pobtaf_ready",
        )
        return out, info
    _lib.check(
        lib.stbta_pobtaf(
            _lib.ptr(matrix.data), n, b, a, int(bool(use_arrow)), _lib.ptr(out), _lib.ptr(info),
            _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream),
        ),
        "stbta_pobtaf",
    )
    return out, info


def _charge_factorize(counter, n, b, a, use_arrow):
    if counter is None:
        return
    for _ in range(n):
        counter.charge(b**3)
        if use_arrow:
            counter.charge(a**3)
    if a > 0:
        counter.charge(a**3)


def factorize(matrix, counter=None, use_arrow=None):
    """Block Cholesky in place (reference bta.py:177-235).

    ``use_arrow`` defaults to the reference's data-dependent test; callers
    that know the structure (the objective evaluator) pass it to skip the
    device scan.  Raises :class:`FactorizationError` on an indefinite pivot.
    """
    if use_arrow is None:
        use_arrow = _arrow_nonzero(matrix)
    use_arrow = bool(use_arrow) and matrix.arrow_size > 0
    with torch.cuda.device(matrix.device):
        ld, info = factorize_async(matrix, use_arrow)
        code = int(info.item())
    if code:
        raise FactorizationError(code - 1)
    _charge_factorize(counter, matrix.n_blocks, matrix.block_size, matrix.arrow_size, use_arrow)
    return BTAFactor(matrix, use_arrow, ld, info)


def logdet(factor):
    """2 * sum(log diag L) (reference bta.py:238-246), computed on device."""
    if factor._logdet is None:
        if factor.logdet_dev is None:
            raise ValueError("factor carries no device log-determinant")
        factor._logdet = float(factor.logdet_dev[0].item())
    return factor._logdet


def _as_device_rhs(factor, rhs):
    m = factor.matrix
    host = not isinstance(rhs, torch.Tensor)
    if host:
        x = torch.from_numpy(np.array(rhs, dtype=np.float64, copy=True)).to(m.device)
    else:
        x = rhs.detach().to(device=m.device, dtype=torch.float64).clone()
    if x.dim() == 0 or x.shape[0] != m.dim:
        raise ValueError(f"rhs has length {x.shape[0] if x.dim() else 0}, expected {m.dim}")
    return x.contiguous(), host


def _solve_policy():
    """STBTA_SOLVE: "tile" (POBTAS tile sweeps), "w" (block-inverse GEMVs,
    preparing W when the factor has none) or "auto" (default: W when the
    factor already holds it, tile sweeps otherwise)."""
    v = os.environ.get("STBTA_SOLVE", "auto")
    if v not in ("auto", "tile", "w"):
        raise ValueError(f"STBTA_SOLVE={v!r}: expected auto, tile or w")
    return v


def prepare_inverse(factor, stream=None):
    """Compute the block inverses W_t = L_tt^-1 (and W_tip) of `factor` once
    (the first step of POBTASI) and keep them with the factor: later solves
    then run as block GEMVs (``stbta_pobtas_w``) and :func:`selected_invert`
    skips its own W pass.  Returns the workspace holding them."""
    if factor._si_ws is None:
        lib = _lib.load()
        m = factor.matrix
        n, b, a = m.n_blocks, m.block_size, m.arrow_size
        with torch.cuda.device(m.device):
            ws = _workspace(lib.stbta_pobtasi_workspace_bytes(n, b, a), m.device)
            _lib.check(
                lib.stbta_pobtasi_prepare(_lib.ptr(m.data), n, b, a, _lib.ptr(ws), ws.numel(),
                                          _lib.stream_ptr(stream)),
                "stbta_pobtasi_prepare",
            )
        factor._si_ws = ws
    return factor._si_ws


def _pobtas(factor, x, mode, counter=None, stream=None, policy=None):
    lib = _lib.load()
    m = factor.matrix
    n, b, a = m.n_blocks, m.block_size, m.arrow_size
    nrhs = 1 if x.dim() == 1 else int(x.shape[1])
    policy = policy or _solve_policy()
    if policy == "w" or (policy == "auto" and factor._si_ws is not None):
        si = prepare_inverse(factor, stream)
        ws = _workspace(lib.stbta_pobtas_w_workspace_bytes(n, b, a), m.device)
        _lib.check(
            lib.stbta_pobtas_w(
                _lib.ptr(m.data), n, b, a, int(bool(factor.has_arrow)), _lib.ptr(x), nrhs, mode,
                _lib.ptr(si), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream),
            ),
            "stbta_pobtas_w",
        )
    else:
        ws = _workspace(lib.stbta_pobtas_workspace_bytes(n, b, a, nrhs), m.device)
        _lib.check(
            lib.stbta_pobtas(
                _lib.ptr(m.data), n, b, a, int(bool(factor.has_arrow)), _lib.ptr(x), nrhs, mode,
                _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream),
            ),
            "stbta_pobtas",
        )
    if counter is not None:  # reference charges: b^2 per block and sweep, a^2 for the forward tip
        if mode in (0, 1):
            for _ in range(n):
                counter.charge(b**2)
            if a > 0:
                counter.charge(a**2)
        if mode in (0, 2):
            for _ in range(n):
                counter.charge(b**2)
    return x


def _solve_api(factor, rhs, mode, counter):
    with torch.cuda.device(factor.matrix.device):
        x, host = _as_device_rhs(factor, rhs)
        _pobtas(factor, x, mode, counter)
        return x.cpu().numpy() if host else x


def forward_substitute(factor, rhs, counter=None):
    """Solve L y = rhs (reference bta.py:249-275).  numpy in -> numpy out."""
    return _solve_api(factor, rhs, 1, counter)


def backward_substitute(factor, rhs, counter=None):
    """Solve L^T x = rhs (reference bta.py:278-302)."""
    return _solve_api(factor, rhs, 2, counter)


def solve(factor, rhs, counter=None):
    """Solve M x = rhs (reference bta.py:305-307)."""
    return _solve_api(factor, rhs, 0, counter)


def selected_invert(factor, counter=None, stream=None, out=None):
    """Pattern entries of M^-1 as a new BTAMatrix (reference bta.py:310-359).

    ``out``: optional pinned CPU float64 tensor of the storage size; the
    inverse then also streams into it block by block while the recursion
    runs (``inv.numpy(out=out)`` waits for the copy only).
    """
    lib = _lib.load()
    m = factor.matrix
    n, b, a = m.n_blocks, m.block_size, m.arrow_size
    with torch.cuda.device(m.device):
        inv = BTAMatrix(n, b, a, torch.empty_like(m.data))
        prepared = factor._si_ws is not None
        ws = factor._si_ws if prepared else _workspace(lib.stbta_pobtasi_workspace_bytes(n, b, a), m.device)
        if (out is not None and isinstance(out, torch.Tensor) and not out.is_cuda and out.is_pinned()
                and out.dtype == torch.float64 and out.numel() == inv._data.numel()
                and out.is_contiguous() and stream is None):
            cs = _side_stream(m.device, "download")
            fn = lib.stbta_pobtasi_prepared if prepared else lib.stbta_pobtasi_stream_out
            _lib.check(
                fn(
                    _lib.ptr(m.data), _lib.ptr(inv.data), out.data_ptr(), n, b, a,
                    int(bool(factor.has_arrow)), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(None),
                    cs.cuda_stream,
                ),
                "stbta_pobtasi_prepared" if prepared else "stbta_pobtasi_stream_out",
            )
            done = torch.cuda.Event()
            done.record(cs)
            inv._data.record_stream(cs)
            ws.record_stream(cs)
            inv._host_copy = (out, done)
        elif prepared:
            _lib.check(
                lib.stbta_pobtasi_prepared(
                    _lib.ptr(m.data), _lib.ptr(inv.data), None, n, b, a,
                    int(bool(factor.has_arrow)), _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream),
                    None,
                ),
                "stbta_pobtasi_prepared",
            )
        else:
            _lib.check(
                lib.stbta_pobtasi(
                    _lib.ptr(m.data), _lib.ptr(inv.data), n, b, a, int(bool(factor.has_arrow)),
                    _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream),
                ),
                "stbta_pobtasi",
            )
    if counter is not None:
        for _ in range(n):
            counter.charge(b**3)
            if factor.has_arrow:
                counter.charge(a**3)
    return inv


def random_spd_bta(rng, n_blocks, block_size, arrow_size=0, device=None):
    """Random SPD BTA matrix L L^T, same draws as the reference generator
    (bta.py:362-394): built on the host from the numpy Generator so CPU and
    GPU runs see identical bytes, then moved to the device."""
    n, b, a = n_blocks, block_size, arrow_size
    sd = 0.3 / np.sqrt(b)
    fac_d = rng.normal(scale=sd, size=(n, b, b))
    for i in range(n):
        fac_d[i] = np.tril(fac_d[i], -1) + np.diag(1.0 + rng.uniform(0.0, 1.0, size=b))
    fac_s = rng.normal(scale=sd, size=(n - 1, b, b)) if n > 1 else np.zeros((0, b, b))
    fac_a = rng.normal(scale=sd, size=(n, a, b))
    fac_t = rng.normal(scale=sd, size=(a, a))
    fac_t = np.tril(fac_t, -1) + np.diag(1.0 + rng.uniform(0.0, 1.0, size=a))
    flat = np.zeros(_storage_elems(n, b, a))
    e0 = n * b * b
    e1 = e0 + (n - 1) * b * b
    e2 = e1 + n * a * b
    D = flat[:e0].reshape(n, b, b)
    S = flat[e0:e1].reshape(n - 1, b, b)
    A = flat[e1:e2].reshape(n, a, b)
    for i in range(n):
        D[i] = fac_d[i] @ fac_d[i].T
        if i > 0:
            D[i] += fac_s[i - 1] @ fac_s[i - 1].T
            S[i - 1] = fac_s[i - 1] @ fac_d[i - 1].T
    if a:
        for i in range(n):
            A[i] = fac_a[i] @ fac_d[i].T
            if i > 0:
                A[i] += fac_a[i - 1] @ fac_s[i - 1].T
        tip = fac_t @ fac_t.T
        for i in range(n):
            tip += fac_a[i] @ fac_a[i].T
        flat[e2:] = tip.ravel()
    return BTAMatrix(n, b, a, flat, device=device)
