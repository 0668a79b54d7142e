"""INLA objective on the device and the quasi-Newton mode search around it.

Mirror of the reference inference driver (pkg/src/stinla/inla.py): same
hyperparameter layout, prior, objective formula, finite-difference gradient /
Hessian and inverse-Hessian BFGS line search, so optimizer decisions are taken
on the same numbers.  What changes is :class:`ObjectiveEvaluator`:

* construction freezes the model into an :class:`~.coreg.AssemblyPlan`
  (device tables) plus the design in BTA column order;
* one evaluation uploads two small coefficient tables, assembles Q_p and Q_c
  straight into HBM, factorizes them concurrently on two CUDA streams (the
  paper's S2 layer), solves for the conditional mean, reduces the quadratic
  form and residuals on the device, and reads back one small scalar block —
  a single host synchronisation per f_obj.
"""

import itertools
import threading
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from . import bta
from .coreg import AssemblyPlan, Coregionalization, PermutationMap, build_permutation
from .model import DimensionError, UnivariateHypers, build_univariate_prior

LOG_2PI = np.log(2.0 * np.pi)


def load_balance_ratio(block_size, arrow_size):
    """(arrow/block)^3, the conditional factorization's extra work (inla.py:34-37)."""
    return float(arrow_size) ** 3 / float(block_size) ** 3


class HyperParams:
    """Hyperparameter vector and its layout (inla.py:40-108).

    Univariate: (log spatial scale, log temporal scale, log variance scale,
    log noise precision).  n_v > 1: two SPDE scales per process, one log noise
    precision per response, one log mixing scale per process, then couplings.
    """

    def __init__(self, values, n_processes):
        values = np.asarray(values, dtype=np.float64).ravel()
        need = self.dim_for(n_processes)
        if values.size != need:
            raise DimensionError(
                f"{n_processes}-process model needs {need} hyperparameters, got {values.size}"
            )
        self.values = values
        self.n_processes = n_processes

    @staticmethod
    def dim_for(n_processes):
        return 4 if n_processes == 1 else 4 * n_processes + n_processes * (n_processes - 1) // 2

    @property
    def dim(self):
        return self.values.size

    def process_hypers(self, i):
        v, nv = self.values, self.n_processes
        if nv == 1:
            return UnivariateHypers(v[0], v[1], v[2], v[3])
        return UnivariateHypers(v[2 * i], v[2 * i + 1], 0.0, v[2 * nv + i])

    def noise_precisions(self):
        nv = self.n_processes
        return np.exp(self.values[3:4]) if nv == 1 else np.exp(self.values[2 * nv : 3 * nv])

    def coregionalization(self):
        nv = self.n_processes
        if nv == 1:
            return None
        return Coregionalization(np.exp(self.values[3 * nv : 4 * nv]), self.values[4 * nv :])

    def names(self):
        nv = self.n_processes
        if nv == 1:
            return ["log_spatial_scale", "log_temporal_scale", "log_variance_scale",
                    "log_noise_precision"]
        out = []
        for i in range(nv):
            out += [f"log_spatial_scale_{i}", f"log_temporal_scale_{i}"]
        out += [f"log_noise_precision_{i}" for i in range(nv)]
        out += [f"log_scale_{i}" for i in range(nv)]
        out += [f"coupling_{k}" for k in range(nv * (nv - 1) // 2)]
        return out


@dataclass
class ThetaPrior:
    """Independent Gaussian priors on theta (inla.py:111-135)."""

    mean: np.ndarray
    sd: np.ndarray

    def __post_init__(self):
        self.mean = np.atleast_1d(np.asarray(self.mean, dtype=np.float64))
        self.sd = np.broadcast_to(np.asarray(self.sd, dtype=np.float64), self.mean.shape).copy()
        if np.any(self.sd <= 0):
            raise ValueError("prior standard deviations must be positive")

    @classmethod
    def for_dim(cls, dim, mean=None, sd=10.0):
        mean = np.zeros(dim) if mean is None else np.asarray(mean, dtype=np.float64)
        return cls(mean=mean, sd=np.full(dim, float(sd)))

    def log_density(self, theta):
        z = (np.asarray(theta) - self.mean) / self.sd
        return float(
            -0.5 * np.sum(z**2) - np.sum(np.log(self.sd)) - 0.5 * self.mean.size * LOG_2PI
        )


# log det Q_p and pivot flag per (spec, prior coefficients), shared by the
# evaluators of all GPUs of the process (small LRU).
_PRIOR_CACHE = {}
_PRIOR_ORDER = []
_PRIOR_LOCK = threading.Lock()
_PRIOR_MAX = 32
_SPEC_TOKENS = itertools.count(1)


def _prior_cache_get(key):
    with _PRIOR_LOCK:
        return _PRIOR_CACHE.get(key)


def _prior_cache_wait(key, timeout=600.0):
    """Block until `key` is in the prior cache (published by prior_logdet)."""
    t0 = time.perf_counter()
    while True:
        hit = _prior_cache_get(key)
        if hit is not None:
            return hit
        if time.perf_counter() - t0 > timeout:
            raise TimeoutError("prior log-determinant was never published")
        time.sleep(0.0005)


def prior_cache_clear():
    """Drop the shared log det Q_p cache (benchmarks timing full evaluations)."""
    with _PRIOR_LOCK:
        _PRIOR_CACHE.clear()
        _PRIOR_ORDER.clear()


# completed (non-aborted) factorizations of every evaluator of the process:
# the numerator of the INLA-level useful TFLOP/s (bench.py)
_WORK = {"pobtaf": 0, "pobtaf_flops": 0.0, "aborted": 0}
_WORK_LOCK = threading.Lock()


def work_counters():
    """Snapshot of the completed-factorization counters."""
    with _WORK_LOCK:
        return dict(_WORK)


def _count_pobtaf(n, b, a, arrow, ok):
    from .perf import flops_pobtaf

    with _WORK_LOCK:
        if ok:
            _WORK["pobtaf"] += 1
            _WORK["pobtaf_flops"] += flops_pobtaf(n, b, a, arrow)
        else:
            _WORK["aborted"] += 1


def _prior_cache_put(key, logdet, info):
    with _PRIOR_LOCK:
        if key in _PRIOR_CACHE:
            return
        _PRIOR_CACHE[key] = (logdet, info)
        _PRIOR_ORDER.append(key)
        while len(_PRIOR_ORDER) > _PRIOR_MAX:
            _PRIOR_CACHE.pop(_PRIOR_ORDER.pop(0), None)


class _Scratch:
    """Per-(thread, device) workspaces and streams of one evaluation slot."""

    def __init__(self, device, nstore, N, nobs, nv, npartial):
        self.device = device
        self.s_prior = torch.cuda.Stream(device=device)
        self.s_cond = torch.cuda.Stream(device=device)
        self.ws_p = torch.empty(nstore, dtype=torch.float64, device=device)
        self.ws_c = torch.empty(nstore, dtype=torch.float64, device=device)
        self.rhs = torch.empty(N, dtype=torch.float64, device=device)
        self.sq = torch.empty(max(nobs, 1), dtype=torch.float64, device=device)
        self.partial = torch.empty(npartial, dtype=torch.float64, device=device)
        # scalars: [logdet_p, logdet_c, quad, resid_0..resid_{nv-1}]
        self.scal = torch.zeros(3 + nv, dtype=torch.float64, device=device)
        self.info = torch.zeros(2, dtype=torch.int32, device=device)
        self.host_scal = torch.zeros(3 + nv, dtype=torch.float64).pin_memory()
        self.host_info = torch.zeros(2, dtype=torch.int32).pin_memory()
        self.host_coef = None
        self.done = torch.cuda.Event()


class ObjectiveEvaluator:
    """Precompiled model for repeated f_obj evaluations on one GPU (inla.py:138-395).

    ``device`` selects the GPU; evaluations from different threads get their
    own workspaces and stream pair, so concurrent calls (the gradient layer)
    are safe, as in the reference.
    """

    def __init__(self, spec, prior=None, partitions=1, lb=1.0, pair_runner=None,
                 calibrate_variance=False, device=None, devices=None):
        spec.validate()
        _lib.load()
        self.spec = spec
        self.n_processes = spec.n_processes
        self.theta_dim = HyperParams.dim_for(spec.n_processes)
        self.prior = prior if prior is not None else ThetaPrior.for_dim(self.theta_dim)
        if self.prior.mean.size != self.theta_dim:
            raise DimensionError("prior dimension does not match the hyperparameter layout")
        self.pair_runner = pair_runner  # streams replace the reference's 2-thread pair layer
        self.device = torch.device(device) if device is not None else bta.default_device()
        self.pmap = build_permutation(spec)
        nv, nl, N = spec.n_processes, spec.latent_per_process, spec.joint_dim

        if spec.design:
            self.design = sp.block_diag(spec.design, format="csr")
            self.observations = np.concatenate(
                [np.asarray(y, dtype=np.float64) for y in spec.observations]
            )
            self.obs_counts = np.array([a.shape[0] for a in spec.design])
        else:
            self.design = sp.csr_matrix((0, N))
            self.observations = np.zeros(0)
            self.obs_counts = np.zeros(nv, dtype=int)
        self.n_observations = int(self.obs_counts.sum())
        if partitions > 1:
            from . import bta_dist

            self.plan = bta_dist.plan_partitions_with_fallback(spec.n_time, partitions, lb)
        else:
            self.plan = None

        self.calibration = np.zeros(nv)
        grams = []
        if self.n_observations:
            for a in spec.design:
                g = (a.T @ a).tocsr()
                grams.append(((g + g.T) * 0.5).tocsr())
        self._grams = grams
        self.assembly = AssemblyPlan(spec, self.pmap, grams, self.device)
        if calibrate_variance:
            self.calibration = np.array([self._calibration_offset(i) for i in range(nv)])

        dev = self.device
        if self.n_observations:
            # design with columns in BTA order; per-process A_i^T y_i in BTA order
            coo = self.design.tocoo()
            perm_cols = self.pmap.forward[coo.col]
            dperm = sp.csr_matrix((coo.data, (coo.row, perm_cols)), shape=self.design.shape)
            dperm.sort_indices()
            self.d_indptr = torch.from_numpy(dperm.indptr.astype(np.int64)).to(dev)
            self.d_indices = torch.from_numpy(dperm.indices.astype(np.int32)).to(dev)
            self.d_vals = torch.from_numpy(dperm.data.astype(np.float64)).to(dev)
            self.d_y = torch.from_numpy(self.observations).to(dev)
            seg = np.concatenate([[0], np.cumsum(self.obs_counts)]).astype(np.int64)
            self.d_seg = torch.from_numpy(seg).to(dev)
            U = np.zeros((nv, N))
            for i in range(nv):
                yi = np.zeros(self.n_observations)
                yi[seg[i] : seg[i + 1]] = self.observations[seg[i] : seg[i + 1]]
                U[i] = self.pmap.permute_vector(self.design.T @ yi)
            self.d_U = torch.from_numpy(U).to(dev)
        self._npartial = 148 * 4
        self._slots = {}
        self._lock = threading.Lock()
        # S3 (reference inla.py:287-308): with a multi-partition plan both
        # factorizations of an f_obj run as PPOBTAF over time partitions, each
        # assembled straight into its own block rows on devices[p % D]
        self._dist = None
        if self.plan is not None and self.plan.n_partitions > 1:
            self._dist = _DistState(self, devices or [self.device])

    # -------------------------------------------------------------- helpers

    def _hypers(self, theta):
        return theta if isinstance(theta, HyperParams) else HyperParams(theta, self.n_processes)

    def _process_hypers(self, hp, i):
        base = hp.process_hypers(i)
        if self.calibration[i] == 0.0:
            return base
        return UnivariateHypers(
            base.log_spatial_scale, base.log_temporal_scale,
            base.log_variance_scale + self.calibration[i], base.log_noise_precision,
        )

    def _calibration_offset(self, i):
        """log multiplier making the unit-hyper prior marginal variance one
        (inla.py:239-249), through the device factorization + selected inverse."""
        from .coreg import map_to_bta

        spec = self.spec
        q = build_univariate_prior(spec, UnivariateHypers(0.0, 0.0, 0.0, 0.0), i)
        pm = PermutationMap(1, spec.n_spatial, spec.n_time, spec.n_fixed)
        ws = bta.BTAMatrix(pm.n_blocks, pm.block_size, pm.arrow_size, device=self.device)
        map_to_bta(q, pm, ws)
        inv = bta.selected_invert(bta.factorize(ws))
        var = torch.diagonal(inv.diag, dim1=1, dim2=2).reshape(-1).cpu().numpy()
        return float(np.log(np.mean(var)))

    def _prior_matrix(self, hp):
        """Host CSR joint prior (oracle / API use; not on the evaluation path)."""
        from .coreg import assemble_joint_precision

        qs = [build_univariate_prior(self.spec, self._process_hypers(hp, i), i)
              for i in range(self.n_processes)]
        if self.n_processes == 1:
            return qs[0]
        return assemble_joint_precision(qs, hp.coregionalization())

    def _noise_diag(self, hp):
        return np.repeat(hp.noise_precisions(), self.obs_counts)

    def _conditional_matrix(self, hp, prior_matrix):
        if not self._grams:
            return prior_matrix.copy()
        nl = self.spec.latent_per_process
        out = prior_matrix.tocsr(copy=True)
        taus = hp.noise_precisions()
        for i, g in enumerate(self._grams):
            gc = g.tocoo()
            out = out + sp.csr_matrix(
                (taus[i] * gc.data, (gc.row + i * nl, gc.col + i * nl)), shape=out.shape
            )
        out = out.tocsr()
        out.sum_duplicates()
        out.sort_indices()
        return out

    def slot(self, index=0):
        """Workspace slot `index` of the calling thread (several slots let one
        thread keep several evaluations in flight)."""
        key = (threading.get_ident(), index)
        with self._lock:
            s = self._slots.get(key)
            if s is None:
                s = _Scratch(self.device, self.assembly.nstore, self.spec.joint_dim,
                             self.n_observations, self.n_processes, self._npartial)
                self._slots[key] = s
        return s

    def release_workspaces(self):
        with self._lock:
            self._slots.clear()
        torch.cuda.empty_cache()

    # ------------------------------------------------------------ objective

    def _coefficients(self, hp):
        nv = self.n_processes
        ph = [self._process_hypers(hp, k) for k in range(nv)]
        linv = hp.coregionalization().mixing_inverse() if nv > 1 else np.ones((1, 1))
        taus = hp.noise_precisions()
        cp, cc = self.assembly.coefficients(ph, linv, taus)
        return cp, cc, taus

    def _spec_token(self):
        """Identity of the model spec for the shared prior cache (a counter
        stamped on the spec object; evaluators of the same spec share it)."""
        tok = getattr(self.spec, "_stbta_token", None)
        if tok is None:
            with _PRIOR_LOCK:
                tok = getattr(self.spec, "_stbta_token", None)
                if tok is None:
                    tok = next(_SPEC_TOKENS)
                    try:
                        setattr(self.spec, "_stbta_token", tok)
                    except (AttributeError, TypeError):
                        tok = ("evaluator", id(self))
        pm = self.pmap
        return (tok, pm.n_blocks, pm.block_size, pm.arrow_size, self.assembly.nstore)

    def prior_logdet(self, theta, slot=None):
        """(log det Q_p, pivot flag) at theta -- the prior half of an f_obj,
        published to the shared prior cache (so an evaluation of the same theta
        on another GPU launched with ``defer_prior=True`` picks it up).  Returns
        None for an invalid theta."""
        hp = self._hypers(theta)
        if not np.all(np.isfinite(hp.values)) or self.n_observations == 0:
            return None
        try:
            cp, _, _ = self._coefficients(hp)
        except ValueError:
            return None
        pkey = (self._spec_token(), cp.tobytes())
        hit = _prior_cache_get(pkey)
        if hit is not None:
            return hit
        dev = self.device
        try:
            if self._dist is not None:
                val = self._dist.prior_logdet(cp)
                _prior_cache_put(pkey, *val)
                return val
            s = slot or self.slot()
            s.done.synchronize()
            with torch.cuda.device(dev):
                coef_p = torch.from_numpy(np.ascontiguousarray(cp.ravel())).to(dev)
                s.s_prior.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.stream(s.s_prior):
                    self.assembly.assemble(s.ws_p, coef_p, s.s_prior)
                    self._pobtaf(s.ws_p, False, s.scal[0:1], s.info[0:1], s.s_prior)
                    s.host_scal.copy_(s.scal, non_blocking=True)
                    s.host_info.copy_(s.info, non_blocking=True)
                    s.done.record(s.s_prior)
            s.done.synchronize()
            val = (float(s.host_scal.numpy()[0]), int(s.host_info.numpy()[0]))
            pm = self.pmap
            _count_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size, False, val[1] == 0)
        except Exception:
            val = (float("nan"), -1)  # unblocks a deferred consumer, which then fails cleanly
            _prior_cache_put(pkey, *val)
            raise
        _prior_cache_put(pkey, *val)
        return val

    def prior_cached(self, theta):
        """True when log det Q_p of ``theta`` is already in the shared prior
        cache, i.e. an evaluation of it skips the prior POBTAF (about half
        the cost of an f_obj).  Used by the runners to order work."""
        if self.n_observations == 0:
            return False
        hp = self._hypers(theta)
        if not np.all(np.isfinite(hp.values)):
            return False
        try:
            cp, _, _ = self._coefficients(hp)
        except ValueError:
            return False
        return _prior_cache_get((self._spec_token(), cp.tobytes())) is not None

    def launch(self, theta, slot=None, defer_prior=False):
        """Issue one f_obj on the device without waiting.  Returns a handle
        for :meth:`collect`, or None for a non-finite / invalid theta.
        ``defer_prior``: skip the prior factorization here; :meth:`collect`
        takes log det Q_p from the shared cache (filled by
        :meth:`prior_logdet` on another GPU)."""
        hp = self._hypers(theta)
        if not np.all(np.isfinite(hp.values)):
            return None
        try:
            cp, cc, taus = self._coefficients(hp)
        except ValueError:
            return None
        if self._dist is not None:
            return ("dist",) + self._dist.evaluate(hp, cp, cc, taus, defer_prior)
        s = slot or self.slot()
        dev = self.device
        P, T = cp.shape
        nv = self.n_processes
        host = np.concatenate([cp.ravel(), cc.ravel(), taus]).astype(np.float64)
        if s.host_coef is None or s.host_coef.numel() != host.size:
            s.host_coef = torch.zeros(host.size, dtype=torch.float64).pin_memory()
            s.dev_coef = torch.zeros(host.size, dtype=torch.float64, device=dev)
        cur = torch.cuda.current_stream(dev)
        # the previous evaluation on this slot must have released the buffers
        s.done.synchronize()
        s.host_coef.numpy()[:] = host
        s.s_cond.wait_stream(cur)
        s.s_prior.wait_stream(cur)
        lib = _lib.load()
        with torch.cuda.device(dev):
            s.dev_coef.copy_(s.host_coef, non_blocking=True)
            coef_p = s.dev_coef[: P * T]
            coef_c = s.dev_coef[P * T : 2 * P * T]
            tau_d = s.dev_coef[2 * P * T :]
            s.s_cond.wait_stream(cur)
            s.s_prior.wait_stream(cur)
            same = self.n_observations == 0
            # prior chain (S2 layer: concurrent with the conditional chain).  Its
            # only outputs are log det Q_p and the pivot flag, a pure function of
            # the prior coefficients: reuse them when another evaluation of the
            # same spec already factorized this exact Q_p (e.g. the gradient
            # stencil points that only move the noise precisions) -- the same
            # bits, one POBTAF fewer.
            pkey = (self._spec_token(), cp.tobytes()) if not same else None
            cached = _prior_cache_get(pkey) if pkey is not None else None
            deferred = defer_prior and pkey is not None and cached is None
            with torch.cuda.stream(s.s_prior):
                if deferred:
                    pass  # log det Q_p arrives through the cache (prior_logdet elsewhere)
                elif cached is not None:
                    s.scal[0:1].fill_(cached[0])
                    s.info[0:1].fill_(cached[1])
                else:
                    self.assembly.assemble(s.ws_p, coef_p, s.s_prior)
                    self._pobtaf(s.ws_p, False, s.scal[0:1], s.info[0:1], s.s_prior)
            with torch.cuda.stream(s.s_cond):
                if not same:
                    self.assembly.assemble(s.ws_c, coef_c, s.s_cond)
                    self._pobtaf(s.ws_c, self.assembly.cond_has_arrow, s.scal[1:2],
                                 s.info[1:2], s.s_cond)
                    _lib.check(lib.stbta_rhs_combine(
                        _lib.ptr(s.rhs), _lib.ptr(self.d_U), _lib.ptr(tau_d), nv,
                        self.spec.joint_dim, _lib.stream_ptr(s.s_cond)), "rhs_combine")
                    self._pobtas(s.ws_c, self.assembly.cond_has_arrow, s.rhs, s.s_cond)
                    self.assembly.quadform(coef_p, s.rhs, s.partial, s.scal[2:3], s.s_cond)
                    _lib.check(lib.stbta_residual(
                        _lib.ptr(self.d_indptr), _lib.ptr(self.d_indices), _lib.ptr(self.d_vals),
                        self.n_observations, _lib.ptr(self.d_y), _lib.ptr(s.rhs),
                        _lib.ptr(self.d_seg), nv, _lib.ptr(s.sq), _lib.ptr(s.scal[3:]),
                        _lib.stream_ptr(s.s_cond)), "residual")
            s.s_cond.wait_stream(s.s_prior)
            with torch.cuda.stream(s.s_cond):
                s.host_scal.copy_(s.scal, non_blocking=True)
                s.host_info.copy_(s.info, non_blocking=True)
                s.done.record(s.s_cond)
        return (s, hp, taus, same, pkey if cached is None else None, deferred)

    def collect(self, handle, want_mu=False):
        """Wait for a launched evaluation; returns (f, mu_perm_device or None)."""
        if handle is None:
            return -np.inf, None
        if handle[0] == "dist":
            value, mu = handle[1], handle[2]
            return value, (mu if want_mu else None)
        s, hp, taus, same, pkey, deferred = handle
        s.done.synchronize()
        info = s.host_info.numpy().copy()
        sc = s.host_scal.numpy().copy()
        if deferred:
            got = _prior_cache_wait(pkey)
            sc[0], info[0] = got[0], (got[1] if np.isfinite(got[0]) else 1)
        elif pkey is not None:
            _prior_cache_put(pkey, float(sc[0]), int(info[0]))
        pm = self.pmap
        if same or (pkey is not None and not deferred):
            _count_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size, False, info[0] == 0)
        if not same:
            _count_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size,
                          self.assembly.cond_has_arrow, info[1] == 0)
        if info[0] != 0 or (not same and info[1] != 0):
            return -np.inf, None
        ld_p = float(sc[0])
        ld_c = ld_p if same else float(sc[1])
        value = self._combine(hp, taus, ld_p, ld_c, sc)
        mu = None
        if want_mu:
            if self.n_observations:
                mu = s.rhs.clone()
            else:
                mu = torch.zeros(self.spec.joint_dim, dtype=torch.float64, device=self.device)
        return value, mu

    def _combine(self, hp, taus, ld_p, ld_c, sc):
        """f_obj from the log-dets and the device scalars [.., .., quad,
        rss_0..rss_{nv-1}] (reference inla.py:360-371)."""
        value = self.prior.log_density(hp.values)
        if self.n_observations:
            active = taus > 0
            counts = self.obs_counts
            logsum = float(np.sum(counts[active] * np.log(taus[active])))
            rss = float(np.sum(taus[active] * sc[3:][active]))
            value += 0.5 * (logsum - rss)
            value -= 0.5 * int(np.sum(counts[active])) * LOG_2PI
            quad = float(sc[2])
        else:
            quad = 0.0
        value += 0.5 * ld_p - 0.5 * quad
        value -= 0.5 * ld_c
        return value

    def _pobtaf(self, buf, use_arrow, logdet_out, info_out, stream):
        """POBTAF on a (row-padded) scratch workspace."""
        lib = _lib.load()
        pm = self.pmap
        n, b, a = pm.n_blocks, pm.block_size, pm.arrow_size
        nbytes = lib.stbta_pobtaf_workspace_bytes(n, b, a)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        _lib.check(lib.stbta_pobtaf_ex(
            *self.assembly.regions(buf), n, b, a, self.assembly.ldb,
            int(bool(use_arrow) and a > 0), -1, _lib.ptr(logdet_out), _lib.ptr(info_out),
            _lib.ptr(ws), nbytes, _lib.stream_ptr(stream)), "stbta_pobtaf_ex")

    def _pobtas(self, buf, has_arrow, rhs, stream):
        """In-place L L^T x = rhs against a (row-padded) scratch factor."""
        lib = _lib.load()
        pm = self.pmap
        n, b, a = pm.n_blocks, pm.block_size, pm.arrow_size
        nbytes = lib.stbta_pobtas_workspace_bytes(n, b, a, 1)
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        _lib.check(lib.stbta_pobtas_ex(
            *self.assembly.regions(buf), n, b, a, self.assembly.ldb, int(bool(has_arrow)),
            _lib.ptr(rhs), 1, 0, _lib.ptr(ws), nbytes, _lib.stream_ptr(stream)), "stbta_pobtas_ex")

    def evaluate(self, theta, counters=None):
        """(f_obj, conditional mean in variable-major order) (inla.py:320-371).

        Returns ``(-inf, None)`` when a factorization meets an indefinite pivot.
        """
        h = self.launch(theta)
        f, mu = self.collect(h, want_mu=True)
        if mu is None:
            return f, None
        if counters:
            hp = self._hypers(theta)
            pm = self.pmap
            if "prior" in counters:
                bta._charge_factorize(counters["prior"], pm.n_blocks, pm.block_size,
                                      pm.arrow_size, False)
            if "conditional" in counters:
                bta._charge_factorize(counters["conditional"], pm.n_blocks, pm.block_size,
                                      pm.arrow_size, self.assembly.cond_has_arrow)
            del hp
        return f, self.pmap.restore_vector(mu.cpu().numpy())

    def objective(self, theta):
        return self.collect(self.launch(theta))[0]

    def latent_marginals(self, theta):
        """Conditional mean and marginal sd at theta via POBTAF + POBTAS +
        POBTASI on the device (inla.py:376-395)."""
        hp = self._hypers(theta)
        cp, cc, taus = self._coefficients(hp)
        if self._dist is not None:
            return self._dist.latent_marginals(cc, taus)
        dev = self.device
        with torch.cuda.device(dev):
            ws = bta.BTAMatrix(self.pmap.n_blocks, self.pmap.block_size, self.pmap.arrow_size,
                               device=dev)
            coef = torch.from_numpy(np.ascontiguousarray(cc.ravel())).to(dev)
            padded = torch.empty(self.assembly.nstore, dtype=torch.float64, device=dev)
            self.assembly.assemble(padded, coef)
            ws.data.copy_(self.assembly.unpad(padded))
            del padded
            factor = bta.factorize(ws, use_arrow=self.assembly.cond_has_arrow)
            bta.prepare_inverse(factor)  # W shared by the mean solve and the selected inversion
            if self.n_observations:
                rhs = torch.empty(self.spec.joint_dim, dtype=torch.float64, device=dev)
                tau_d = torch.from_numpy(np.asarray(taus, dtype=np.float64)).to(dev)
                _lib.check(_lib.load().stbta_rhs_combine(
                    _lib.ptr(rhs), _lib.ptr(self.d_U), _lib.ptr(tau_d), self.n_processes,
                    self.spec.joint_dim, _lib.stream_ptr()), "rhs_combine")
                bta._pobtas(factor, rhs, 0)
                mu = self.pmap.restore_vector(rhs.cpu().numpy())
            else:
                mu = np.zeros(self.spec.joint_dim)
            inv = bta.selected_invert(factor)
            var = torch.diagonal(inv.diag, dim1=1, dim2=2).reshape(-1)
            if self.pmap.arrow_size:
                var = torch.cat([var, torch.diagonal(inv.tip)])
            var = self.pmap.restore_vector(var.cpu().numpy())
        return mu, np.sqrt(var)


class _DistState:
    """f_obj over time partitions (S3, reference inla.py:287-308 dispatching
    to bta_dist): partition p's block rows of Q_p / Q_c are assembled on
    devices[p % D] by a row-sliced assembly plan (no global workspace), its
    interior eliminated there, the reduced system factorized on the
    evaluator's device; the conditional mean comes from the partitioned
    solve, the quadratic form and residuals from the same device kernels as
    the one-GPU path."""

    def __init__(self, ev, devices):
        from . import bta_dist

        self.ev = ev
        self.bd = bta_dist
        self.plan = ev.plan
        self.devices = [torch.device(d) for d in devices]
        P = self.plan.n_partitions
        self.parts = [ev.assembly.rows_plan(self.plan.boundaries[p], self.plan.boundaries[p + 1],
                                            p == 0, self.devices[p % len(self.devices)])
                      for p in range(P)]
        self.mapper = bta_dist._default_mapper(self.devices)
        self.lock = threading.Lock()

    def factorize(self, coef, use_arrow):
        """PPOBTAF of the matrix with coefficient table ``coef``; raises
        FactorizationError on a non-SPD pivot."""
        pm = self.ev.pmap
        n, b, a = pm.n_blocks, pm.block_size, pm.arrow_size
        flat = np.ascontiguousarray(coef.ravel())
        coefs = {}
        for d in self.devices:
            coefs.setdefault(str(d), torch.from_numpy(flat).to(d))
        rows = [ra.assemble(ra.new_rows(), coefs[str(ra.device)]) for ra in self.parts]
        chains = self.bd._make_chains(self.plan, b, a, use_arrow, self.devices)
        tip = rows[0].tip.to(self.ev.device) if a else None
        return self.bd._factorize_chains(self.plan, (n, b, a), chains,
                                         lambda ch: ch.load(rows[ch.index]), tip, use_arrow,
                                         self.ev.device, mapper=self.mapper)

    def _logdet(self, coef, use_arrow):
        pm = self.ev.pmap
        try:
            f = self.factorize(coef, use_arrow)
        except bta.FactorizationError:
            _count_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size, use_arrow, False)
            return None, float("nan"), 1
        _count_pobtaf(pm.n_blocks, pm.block_size, pm.arrow_size, use_arrow, True)
        return f, self.bd.d_logdet(f), 0

    def prior_logdet(self, cp):
        with self.lock:
            _, ld, info = self._logdet(cp, False)
        return ld, info

    def evaluate(self, hp, cp, cc, taus, defer_prior=False):
        """(f, mu in BTA order on the evaluator's device or None)."""
        ev = self.ev
        lib = _lib.load()
        same = ev.n_observations == 0
        pkey = (ev._spec_token(), cp.tobytes()) if not same else None
        with self.lock, torch.cuda.device(ev.device):
            cached = _prior_cache_get(pkey) if pkey is not None else None
            if cached is None and defer_prior and pkey is not None:
                cached = _prior_cache_wait(pkey)
            if cached is not None:
                ld_p, info_p = cached[0], (cached[1] if np.isfinite(cached[0]) else 1)
            else:
                _, ld_p, info_p = self._logdet(cp, False)
                if pkey is not None:
                    _prior_cache_put(pkey, ld_p, info_p)
            if info_p != 0:
                return -np.inf, None
            s = ev.slot()
            s.scal.zero_()
            if same:
                ld_c = ld_p
                mu = torch.zeros(ev.spec.joint_dim, dtype=torch.float64, device=ev.device)
            else:
                fc, ld_c, info_c = self._logdet(cc, ev.assembly.cond_has_arrow)
                if info_c != 0:
                    return -np.inf, None
                coef = torch.from_numpy(np.concatenate([cp.ravel(), taus]).astype(np.float64)
                                        ).to(ev.device)
                coef_p, tau_d = coef[: cp.size], coef[cp.size :]
                _lib.check(lib.stbta_rhs_combine(
                    _lib.ptr(s.rhs), _lib.ptr(ev.d_U), _lib.ptr(tau_d), ev.n_processes,
                    ev.spec.joint_dim, _lib.stream_ptr()), "rhs_combine")
                mu = self.bd.d_solve(fc, s.rhs)
                ev.assembly.quadform(coef_p, mu, s.partial, s.scal[2:3])
                _lib.check(lib.stbta_residual(
                    _lib.ptr(ev.d_indptr), _lib.ptr(ev.d_indices), _lib.ptr(ev.d_vals),
                    ev.n_observations, _lib.ptr(ev.d_y), _lib.ptr(mu), _lib.ptr(ev.d_seg),
                    ev.n_processes, _lib.ptr(s.sq), _lib.ptr(s.scal[3:]), _lib.stream_ptr()),
                    "residual")
            sc = s.scal.cpu().numpy()
        return ev._combine(hp, taus, ld_p, ld_c, sc), mu

    def latent_marginals(self, cc, taus):
        """(mu, sd) via PPOBTAF + PPOBTAS + PPOBTASI of Q_c (inla.py:376-395)."""
        ev = self.ev
        dev = ev.device
        with self.lock, torch.cuda.device(dev):
            f = self.factorize(cc, ev.assembly.cond_has_arrow)
            if ev.n_observations:
                rhs = torch.empty(ev.spec.joint_dim, dtype=torch.float64, device=dev)
                tau_d = torch.from_numpy(np.asarray(taus, dtype=np.float64)).to(dev)
                _lib.check(_lib.load().stbta_rhs_combine(
                    _lib.ptr(rhs), _lib.ptr(ev.d_U), _lib.ptr(tau_d), ev.n_processes,
                    ev.spec.joint_dim, _lib.stream_ptr()), "rhs_combine")
                mu = ev.pmap.restore_vector(self.bd.d_solve(f, rhs).cpu().numpy())
            else:
                mu = np.zeros(ev.spec.joint_dim)
            inv = self.bd.d_selected_invert(f)
            var = torch.diagonal(inv.diag, dim1=1, dim2=2).reshape(-1)
            if ev.pmap.arrow_size:
                var = torch.cat([var, torch.diagonal(inv.tip)])
            var = ev.pmap.restore_vector(var.cpu().numpy())
        return mu, np.sqrt(var)


def eval_objective(theta, model):
    ev = model if isinstance(model, ObjectiveEvaluator) else ObjectiveEvaluator(model)
    return ev.evaluate(theta)


def _scalar_function(objective):
    """Callables pass through; evaluators and model specs become the negated
    objective (inla.py:405-415).  The closure is tagged with its evaluator so
    the GPU runners can re-bind a task to an identical evaluator on another
    device (sched.GpuRunner); untagged tasks are simply called."""
    if callable(objective) and not isinstance(objective, ObjectiveEvaluator):
        return objective
    if hasattr(objective, "objective"):  # an evaluator (or evaluator-like object)
        ev = objective
    else:  # a model spec
        ev = ObjectiveEvaluator(objective)

    def neg_objective(theta):
        return -ev.objective(theta)

    neg_objective.stbta_evaluator = ev
    return neg_objective


def _stencil(theta, step, cross):
    """Central-difference points: centre, then (+h, -h) per coordinate, then
    (if cross) the four-point cross stencil per pair i < j (inla.py:428-462)."""
    pts = [theta.copy()]
    d = theta.size
    for i in range(d):
        for sign in (1.0, -1.0):
            p = theta.copy()
            p[i] += sign * step
            pts.append(p)
    pairs = []
    if cross:
        for i in range(d):
            for j in range(i + 1, d):
                for si, sj in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
                    p = theta.copy()
                    p[i] += si * step
                    p[j] += sj * step
                    pts.append(p)
                    pairs.append((i, j))
    return pts, pairs


def _run(fun, points, runner):
    tasks = []
    for p in points:
        def task(p=p):
            return fun(p)

        task.stbta_point, task.stbta_fun = p, fun  # lets a GPU runner re-bind the task
        tasks.append(task)
    if runner is None:
        return np.asarray([t() for t in tasks])
    return np.asarray(runner(tasks))


def fd_gradient(fun, theta, step=1e-3, runner=None):
    """(f(theta), central-difference gradient) from 2*dim+1 independent tasks
    reduced in coordinate order (inla.py:418-437)."""
    if step <= 0:
        raise ValueError("finite-difference step must be positive")
    f = _scalar_function(fun)
    theta = np.asarray(theta, dtype=np.float64)
    pts, _ = _stencil(theta, step, cross=False)
    vals = _run(f, pts, runner)
    return float(vals[0]), (vals[1::2] - vals[2::2]) / (2.0 * step)


def fd_hessian(fun, theta, step=1e-2, runner=None):
    """Second-order central-difference Hessian, symmetrized (inla.py:440-476)."""
    if step <= 0:
        raise ValueError("finite-difference step must be positive")
    f = _scalar_function(fun)
    theta = np.asarray(theta, dtype=np.float64)
    d = theta.size
    pts, pairs = _stencil(theta, step, cross=True)
    vals = _run(f, pts, runner)
    f0 = vals[0]
    hess = np.zeros((d, d))
    for i in range(d):
        hess[i, i] = (vals[1 + 2 * i] - 2.0 * f0 + vals[2 + 2 * i]) / step**2
    base = 1 + 2 * d
    for k in range(0, len(pairs), 4):
        i, j = pairs[k]
        fpp, fpm, fmp, fmm = vals[base + k : base + k + 4]
        hess[i, j] = hess[j, i] = (fpp - fpm - fmp + fmm) / (4.0 * step**2)
    return 0.5 * (hess + hess.T)


@dataclass
class IterationRecord:
    iteration: int
    f: float
    grad_norm: float
    step: float
    f_evals: int
    seconds: float


@dataclass
class MinimizeResult:
    theta: np.ndarray
    f: float
    grad: np.ndarray
    iterations: int
    f_evals: int
    status: str
    trace: list = field(default_factory=list)

    @property
    def converged(self):
        return self.status.startswith("converged")


def _bfgs_inverse_update(hinv, delta, gamma):
    """Dense inverse-Hessian BFGS update, skipped on non-positive curvature
    (inla.py:575-586)."""
    curv = float(gamma @ delta)
    if not (np.isfinite(curv) and curv > 1e-10 * (np.linalg.norm(delta) * np.linalg.norm(gamma) + 1e-300)):
        return hinv
    rho = 1.0 / curv
    eye = np.eye(delta.size)
    outer = np.outer(delta, gamma)
    return (eye - rho * outer) @ hinv @ (eye - rho * outer.T) + rho * np.outer(delta, delta)


def minimize(objective, theta0, gtol=1e-3, ftol=1e-6, max_iter=100, grad_step=1e-3, runner=None,
             c1=1e-4, shrink=0.5, max_backtracks=20, on_iteration=None, state0=None):
    """Quasi-Newton minimization with Armijo backtracking and central-difference
    gradients — the reference algorithm (inla.py:504-613).  Extensions:
    ``on_iteration`` is called with each IterationRecord; ``state0`` =
    (f, grad, hinv) resumes a run at theta0 from a recorded BFGS state
    (MinimizeResult.hinv) instead of the starting gradient and identity."""
    fun = _scalar_function(objective)
    theta = np.asarray(theta0, dtype=np.float64).copy()
    d = theta.size
    if state0 is None:
        f, grad = fd_gradient(fun, theta, grad_step, runner)
        n_eval = 2 * d + 1
        hinv = np.eye(d)
    else:
        f, grad, hinv = float(state0[0]), np.array(state0[1], dtype=np.float64), \
            np.array(state0[2], dtype=np.float64)
        n_eval = 0
    if not np.isfinite(f):
        raise ValueError("objective is not finite at the starting point")
    trace = []
    status = "max_iterations"
    for it in range(1, max_iter + 1):
        if not np.all(np.isfinite(grad)):
            status = "invalid_gradient"
            break
        if float(np.max(np.abs(grad))) <= gtol:
            status = "converged"
            break
        tic = time.perf_counter()
        direction = -(hinv @ grad)
        slope = float(grad @ direction)
        if slope >= 0:
            hinv = np.eye(d)
            direction = -grad
            slope = -float(grad @ grad)
        step, accepted, tries = 1.0, False, 0
        width = max(1, int(getattr(runner, "width", 1))) if runner is not None else 1
        if runner is not None:
            # Armijo backtracking with the next `width` step sizes evaluated
            # concurrently through the runner (one per GPU or GPU pair; width
            # 1 still lets the runner split an f_obj over a GPU pair); the
            # first acceptable one in backtracking order is taken, so the
            # accepted step, theta and the sequential try count are exactly
            # those of the loop below.
            k, st = 0, 1.0
            while k <= max_backtracks and not accepted:
                ks = list(range(k, min(k + width, max_backtracks + 1)))
                steps = []
                for _ in ks:  # the same repeated products as the sequential loop
                    steps.append(st)
                    st *= shrink
                vals = _run(fun, [theta + sj * direction for sj in steps], runner)
                for j, sj, fv in zip(ks, steps, vals):
                    if np.isfinite(fv) and fv <= f + c1 * sj * slope:
                        step, accepted, tries = sj, True, j + 1
                        break
                k = ks[-1] + 1
            if not accepted:
                tries = max_backtracks + 1
            cand = theta + step * direction
        else:
            for _ in range(max_backtracks + 1):
                cand = theta + step * direction
                f_cand = fun(cand)
                tries += 1
                if np.isfinite(f_cand) and f_cand <= f + c1 * step * slope:
                    accepted = True
                    break
                step *= shrink
        n_eval += tries
        if not accepted:
            status = "line_search_failed"
            warnings.warn("line search failed to find sufficient decrease", stacklevel=2)
            break
        f_new, g_new = fd_gradient(fun, cand, grad_step, runner)
        n_eval += 2 * d + 1
        hinv = _bfgs_inverse_update(hinv, cand - theta, g_new - grad)
        f_prev = f
        theta, f, grad = cand, f_new, g_new
        rec = IterationRecord(it, f, float(np.max(np.abs(grad))), step, tries + 2 * d + 1,
                              time.perf_counter() - tic)
        trace.append(rec)
        if on_iteration is not None:
            on_iteration(rec)
        if abs(f_prev - f) <= ftol * max(1.0, abs(f_prev)):
            status = "converged_ftol"
            break
    if status == "max_iterations":
        warnings.warn("maximum iterations reached without convergence", stacklevel=2)
    res = MinimizeResult(theta, f, grad, len(trace), n_eval, status, trace)
    res.hinv = hinv
    return res


def latent_marginals(theta, model):
    ev = model if isinstance(model, ObjectiveEvaluator) else ObjectiveEvaluator(model)
    return ev.latent_marginals(theta)


def predict(design_pred, latent_mean):
    """Posterior predictive mean design_pred @ latent_mean (inla.py:622-632)."""
    design_pred = sp.csr_matrix(design_pred)
    latent_mean = np.asarray(latent_mean, dtype=np.float64)
    if design_pred.shape[1] != latent_mean.size:
        raise DimensionError(
            f"prediction design has {design_pred.shape[1]} columns, expected {latent_mean.size}"
        )
    return design_pred @ latent_mean


@dataclass
class PosteriorSummary:
    theta_mode: HyperParams
    theta_sd: np.ndarray
    latent_mean: np.ndarray
    latent_sd: np.ndarray
    logpost_at_mode: float
    iterations: int
    f_evals: int
    status: str
    theta_hessian: np.ndarray


@dataclass
class FitOptions:
    grad_step: float = 1e-3
    hess_step: float = 1e-2
    gtol: float = 1e-3
    ftol: float = 1e-6
    max_iter: int = 100
    prior_sd: float = 10.0
    prior_mean: np.ndarray = None


def fit(model, theta0, options=None, runner=None, partitions=1, lb=1.0, pair_runner=None,
        calibrate_variance=False):
    """Mode search, Hessian at the mode, latent marginals (inla.py:661-729)."""
    options = options or FitOptions()
    theta0 = np.asarray(theta0, dtype=np.float64)
    if isinstance(model, ObjectiveEvaluator):
        ev = model
    else:
        mean = options.prior_mean if options.prior_mean is not None else theta0
        ev = ObjectiveEvaluator(
            model, prior=ThetaPrior.for_dim(theta0.size, mean=mean, sd=options.prior_sd),
            partitions=partitions, lb=lb, pair_runner=pair_runner,
            calibrate_variance=calibrate_variance,
        )
    res = minimize(ev, theta0, gtol=options.gtol, ftol=options.ftol, max_iter=options.max_iter,
                   grad_step=options.grad_step, runner=runner)
    hess = fd_hessian(ev, res.theta, options.hess_step, runner)
    d = res.theta.size
    try:
        np.linalg.cholesky(hess)
        theta_sd = np.sqrt(np.diagonal(np.linalg.inv(hess)))
    except np.linalg.LinAlgError:
        warnings.warn("Hessian at the mode is not positive definite; "
                      "hyperparameter uncertainties unavailable", stacklevel=2)
        theta_sd = np.full(d, np.nan)
    mean, sd = ev.latent_marginals(res.theta)
    summary = PosteriorSummary(
        theta_mode=HyperParams(res.theta, ev.n_processes), theta_sd=theta_sd,
        latent_mean=mean, latent_sd=sd, logpost_at_mode=-res.f, iterations=res.iterations,
        f_evals=res.f_evals + 1 + 2 * d + 2 * d * (d - 1), status=res.status,
        theta_hessian=hess,
    )
    return summary, res
