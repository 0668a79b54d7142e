"""numpy/scipy restatement of the objective path — TEST INFRASTRUCTURE ONLY.

Follows the reference operation by operation on the CPU:
  * SPDE precision in product form q1 -> q2 -> q3   (model.py:196-248)
  * coregional joint assembly                        (coreg.py:80-121)
  * conditional precision from per-response Grams    (inla.py:195-203, 264-283)
  * permutation bind + scatter                       (coreg.py:133-276)
  * f_obj                                            (inla.py:320-371)
  * latent marginals via selected inversion          (inla.py:376-395)
Model *inputs* (ModelSpec, discretizations, designs) are taken from the object
passed in, so the oracle and the device path see identical bytes.
"""

import numpy as np
import scipy.sparse as sp

from . import bta_np

LOG_2PI = np.log(2.0 * np.pi)


def theta_layout(theta, nv):
    """(per-process (ls, lt, lv, ln), taus, mixing scales, couplings) — inla.py:40-91."""
    v = np.asarray(theta, dtype=np.float64)
    if nv == 1:
        return [(v[0], v[1], v[2], v[3])], np.exp(v[3:4]), None, None
    procs = [(v[2 * i], v[2 * i + 1], 0.0, v[2 * nv + i]) for i in range(nv)]
    return procs, np.exp(v[2 * nv : 3 * nv]), np.exp(v[3 * nv : 4 * nv]), v[4 * nv :]


def st_precision(spatial, temporal, ls, lt, lv):
    """model.py:196-228, product form."""
    gs, gt, ge = np.exp(ls), np.exp(lt), np.exp(lv)
    minv = sp.diags(1.0 / spatial.mass.diagonal())
    q1 = (gs**2) * spatial.mass + spatial.stiffness
    q1 = ((q1 + q1.T) * 0.5).tocsr()
    q2 = q1 @ minv @ q1
    q2 = ((q2 + q2.T) * 0.5).tocsr()
    q3 = q1 @ minv @ q2
    q3 = ((q3 + q3.T) * 0.5).tocsr()
    out = ge * (
        sp.kron(temporal.mass, q3, format="csr")
        + gt * sp.kron(temporal.coupling, q2, format="csr")
        + gt**2 * sp.kron(temporal.stiffness, q1, format="csr")
    )
    out.sum_duplicates()
    out.sort_indices()
    return out


def univariate_prior(spec, i, hyp):
    """model.py:231-248."""
    st = st_precision(spec.spatial[i], spec.temporal[i], *hyp[:3])
    if spec.n_fixed == 0:
        return st
    out = sp.block_diag(
        [st, spec.fixed_effect_precision * sp.identity(spec.n_fixed, format="csr")], format="csr"
    )
    out.sort_indices()
    return out


def mixing_inverse(scales, couplings):
    """coreg.py:59-77."""
    nv = scales.size
    lam = np.zeros((nv, nv))
    k = 0
    for i in range(1, nv):
        for j in range(i - 1, -1, -1):
            lam[i, j] = couplings[k]
            k += 1
    return np.diag(1.0 / scales) @ (np.eye(nv) - lam)


def joint_prior(spec, theta):
    """inla.py:251-258 + coreg.py:80-121."""
    nv = spec.n_processes
    procs, _, scales, couplings = theta_layout(theta, nv)
    qs = [univariate_prior(spec, i, procs[i]) for i in range(nv)]
    if nv == 1:
        return qs[0]
    linv = mixing_inverse(scales, couplings)
    dim = qs[0].shape[0]
    coos = [sp.coo_matrix(q) for q in qs]
    rows, cols, data = [], [], []
    for i in range(nv):
        for j in range(i + 1):
            for k in range(i, nv):
                c = linv[k, i] * linv[k, j]
                rows.append(coos[k].row + i * dim)
                cols.append(coos[k].col + j * dim)
                data.append(c * coos[k].data)
                if i != j:
                    rows.append(coos[k].row + j * dim)
                    cols.append(coos[k].col + i * dim)
                    data.append(c * coos[k].data)
    out = sp.coo_matrix(
        (np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
        shape=(nv * dim, nv * dim),
    ).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


def conditional(spec, prior, taus):
    """inla.py:195-203 + 264-283."""
    if not spec.design:
        return prior.copy()
    per = spec.latent_per_process
    coo = prior.tocoo()
    rows, cols, data = [coo.row], [coo.col], [coo.data]
    for i, a in enumerate(spec.design):
        g = (a.T @ a).tocsr()
        g = ((g + g.T) * 0.5).tocoo()
        rows.append(g.row + i * per)
        cols.append(g.col + i * per)
        data.append(taus[i] * g.data)
    out = sp.coo_matrix(
        (np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))), shape=prior.shape
    ).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


def forward_perm(spec):
    """coreg.py:153-164."""
    nv, ns, nt, nf = spec.n_processes, spec.n_spatial, spec.n_time, spec.n_fixed
    b = nv * ns
    per = ns * nt + nf
    fwd = np.empty(nv * per, dtype=np.int64)
    for v in range(nv):
        st = np.arange(ns * nt)
        t, s = np.divmod(st, ns)
        fwd[v * per + st] = t * b + v * ns + s
        if nf:
            e = np.arange(nf)
            fwd[v * per + ns * nt + e] = nv * ns * nt + v * nf + e
    return fwd


def to_bta(spec, mat):
    """Scatter of a symmetric CSR matrix into BTA storage (coreg.py:186-276):
    entries of the diagonal and first sub-diagonal blocks, the arrow rows
    and the tip, in the permuted order; vectorised (C3: ~10^7 entries)."""
    nv, ns, nt, nf = spec.n_processes, spec.n_spatial, spec.n_time, spec.n_fixed
    n, b, a = nt, nv * ns, nv * nf
    fwd = forward_perm(spec)
    coo = sp.coo_matrix(mat)
    pr, pc, v = fwd[coo.row], fwd[coo.col], coo.data
    split = n * b
    data = np.zeros(bta_np.storage_elems(n, b, a))
    e0 = n * b * b
    e1 = e0 + (n - 1) * b * b
    e2 = e1 + n * a * b
    lat = (pr < split) & (pc < split)
    ti, tj = pr // b, pc // b
    m = lat & (ti == tj)
    data[ti[m] * b * b + (pr[m] % b) * b + pc[m] % b] = v[m]
    m = lat & (ti == tj + 1)
    data[e0 + tj[m] * b * b + (pr[m] % b) * b + pc[m] % b] = v[m]
    m = (pr >= split) & (pc < split)
    data[e1 + tj[m] * a * b + (pr[m] - split) * b + pc[m] % b] = v[m]
    m = (pr >= split) & (pc >= split)
    data[e2 + (pr[m] - split) * a + (pc[m] - split)] = v[m]
    return data, (n, b, a)


def evaluate(spec, theta, prior_mean, prior_sd):
    """f_obj and mu (inla.py:320-371) with the sequential BTA oracle.
    Returns (-inf, None) on an indefinite pivot."""
    theta = np.asarray(theta, dtype=np.float64)
    if not np.all(np.isfinite(theta)):
        return -np.inf, None
    nv = spec.n_processes
    _, taus, _, _ = theta_layout(theta, nv)
    qp = joint_prior(spec, theta)
    qc = conditional(spec, qp, taus)
    fwd = forward_perm(spec)
    try:
        dp, (n, b, a) = to_bta(spec, qp)
        bta_np.factorize(dp, n, b, a)
        ld_p = bta_np.logdet(dp, n, b, a)
        dc, _ = to_bta(spec, qc)
        has = bta_np.factorize(dc, n, b, a)
        ld_c = bta_np.logdet(dc, n, b, a)
    except bta_np.OracleFactorizationError:
        return -np.inf, None
    z = (theta - prior_mean) / prior_sd
    value = float(-0.5 * np.sum(z**2) - np.sum(np.log(prior_sd)) - 0.5 * theta.size * LOG_2PI)
    if spec.design:
        design = sp.block_diag(spec.design, format="csr")
        y = np.concatenate([np.asarray(o, dtype=np.float64) for o in spec.observations])
        noise = np.repeat(taus, [d_.shape[0] for d_ in spec.design])
        rhs = design.T @ (noise * y)
        rp = np.empty_like(rhs)
        rp[fwd] = rhs
        mu = bta_np.solve(dc, n, b, a, has, rp)[fwd]
        resid = y - design @ mu
        act = noise > 0
        value += 0.5 * (np.sum(np.log(noise[act])) - np.sum(noise[act] * resid[act] ** 2))
        value -= 0.5 * np.count_nonzero(act) * LOG_2PI
    else:
        mu = np.zeros(spec.joint_dim)
    value += 0.5 * ld_p - 0.5 * float(mu @ (qp @ mu))
    value -= 0.5 * ld_c
    return value, mu


def marginal_sd(spec, theta):
    """inla.py:376-395: sqrt(diag(Q_c^-1)) via the selected-inversion oracle."""
    nv = spec.n_processes
    _, taus, _, _ = theta_layout(theta, nv)
    qc = conditional(spec, joint_prior(spec, theta), taus)
    dc, (n, b, a) = to_bta(spec, qc)
    has = bta_np.factorize(dc, n, b, a)
    inv = bta_np.selected_invert(dc, n, b, a, has)
    d, _, _, tp = bta_np.views(inv, n, b, a)
    var = np.concatenate([np.diagonal(d[t]) for t in range(n)] + ([np.diagonal(tp)] if a else []))
    return np.sqrt(var[forward_perm(spec)])
