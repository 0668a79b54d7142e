"""numpy restatement of the sequential BTA solver — TEST INFRASTRUCTURE ONLY.

Follows pkg/src/stinla/bta.py of the reference operation by operation
(same LAPACK calls through numpy/scipy, same update order), on a flat FP64
buffer with the reference layout diag | lower | arrow | tip.
"""

import numpy as np
from scipy.linalg import solve_triangular


class OracleFactorizationError(RuntimeError):
    """Mirror of stinla.bta.FactorizationError (bta.py:17-31)."""

    def __init__(self, block_index, partition=None):
        self.block_index = block_index
        self.partition = partition
        super().__init__(f"non-positive-definite pivot at block {block_index}")


def storage_elems(n, b, a):
    """bta.py:69-72."""
    return n * b * b + (n - 1) * b * b + n * a * b + a * a


def views(data, n, b, a):
    """(diag, lower, arrow, tip) views of the flat buffer (bta.py:80-84)."""
    e0 = n * b * b
    e1 = e0 + (n - 1) * b * b
    e2 = e1 + n * a * b
    return (
        data[:e0].reshape(n, b, b),
        data[e0:e1].reshape(n - 1, b, b),
        data[e1:e2].reshape(n, a, b),
        data[e2 : e2 + a * a].reshape(a, a),
    )


def to_dense(data, n, b, a):
    """bta.py:105-120."""
    d, lo, ar, tp = views(data, n, b, a)
    N = n * b + a
    out = np.zeros((N, N))
    for i in range(n):
        out[i * b : (i + 1) * b, i * b : (i + 1) * b] = d[i]
        if i + 1 < n:
            out[(i + 1) * b : (i + 2) * b, i * b : (i + 1) * b] = lo[i]
            out[i * b : (i + 1) * b, (i + 1) * b : (i + 2) * b] = lo[i].T
        if a:
            out[n * b :, i * b : (i + 1) * b] = ar[i]
            out[i * b : (i + 1) * b, n * b :] = ar[i].T
    if a:
        out[n * b :, n * b :] = tp
    return out


def from_dense(dense, n, b, a):
    """bta.py:122-139."""
    data = np.zeros(storage_elems(n, b, a))
    d, lo, ar, tp = views(data, n, b, a)
    for i in range(n):
        d[i] = dense[i * b : (i + 1) * b, i * b : (i + 1) * b]
        if i + 1 < n:
            lo[i] = dense[(i + 1) * b : (i + 2) * b, i * b : (i + 1) * b]
        if a:
            ar[i] = dense[n * b :, i * b : (i + 1) * b]
    if a:
        tp[...] = dense[n * b :, n * b :]
    return data


def random_spd_bta(rng, n, b, a):
    """Same generator and draw order as bta.random_spd_bta (bta.py:362-394)."""
    sd = 0.3 / np.sqrt(b)
    l_d = rng.normal(scale=sd, size=(n, b, b))
    for i in range(n):
        l_d[i] = np.tril(l_d[i], -1) + np.diag(1.0 + rng.uniform(0.0, 1.0, size=b))
    l_s = rng.normal(scale=sd, size=(n - 1, b, b)) if n > 1 else np.zeros((0, b, b))
    l_a = rng.normal(scale=sd, size=(n, a, b))
    l_t = rng.normal(scale=sd, size=(a, a))
    l_t = np.tril(l_t, -1) + np.diag(1.0 + rng.uniform(0.0, 1.0, size=a))

    data = np.zeros(storage_elems(n, b, a))
    d, lo, ar, tp = views(data, n, b, a)
    for i in range(n):
        d[i] = l_d[i] @ l_d[i].T
        if i:
            d[i] += l_s[i - 1] @ l_s[i - 1].T
    for i in range(n - 1):
        lo[i] = l_s[i] @ l_d[i].T
    if a:
        for i in range(n):
            ar[i] = l_a[i] @ l_d[i].T
            if i:
                ar[i] += l_a[i - 1] @ l_s[i - 1].T
        t = l_t @ l_t.T
        for i in range(n):
            t += l_a[i] @ l_a[i].T
        tp[...] = t
    return data


def factorize(data, n, b, a, use_arrow=None):
    """In-place POBTAF (bta.py:177-235).  Returns has_arrow."""
    d, lo, ar, tp = views(data, n, b, a)
    if use_arrow is None:
        use_arrow = a > 0 and bool(np.any(ar))
    for i in range(n):
        try:
            d[i] = np.linalg.cholesky(d[i])
        except np.linalg.LinAlgError:
            raise OracleFactorizationError(i) from None
        piv = d[i]
        if i < n - 1:
            lo[i] = solve_triangular(piv, lo[i].T, lower=True, check_finite=False).T
        if use_arrow:
            ar[i] = solve_triangular(piv, ar[i].T, lower=True, check_finite=False).T
        if i < n - 1:
            d[i + 1] -= lo[i] @ lo[i].T
            if use_arrow:
                ar[i + 1] -= ar[i] @ lo[i].T
        if use_arrow:
            tp -= ar[i] @ ar[i].T
    if a:
        try:
            tp[...] = np.linalg.cholesky(tp)
        except np.linalg.LinAlgError:
            raise OracleFactorizationError(n) from None
    return use_arrow


def logdet(data, n, b, a):
    """bta.py:238-246."""
    d, _, _, tp = views(data, n, b, a)
    s = 0.0
    for i in range(n):
        s += np.sum(np.log(np.diagonal(d[i])))
    if a:
        s += np.sum(np.log(np.diagonal(tp)))
    return 2.0 * s


def forward(data, n, b, a, has_arrow, rhs):
    """L y = r (bta.py:249-275)."""
    d, lo, ar, tp = views(data, n, b, a)
    x = np.array(rhs, dtype=np.float64, copy=True)
    X = x.reshape(n * b + a, -1)
    for i in range(n):
        seg = X[i * b : (i + 1) * b]
        if i:
            seg -= lo[i - 1] @ X[(i - 1) * b : i * b]
        X[i * b : (i + 1) * b] = solve_triangular(d[i], seg, lower=True, check_finite=False)
    if a:
        seg = X[n * b :]
        if has_arrow:
            for i in range(n):
                seg -= ar[i] @ X[i * b : (i + 1) * b]
        X[n * b :] = solve_triangular(tp, seg, lower=True, check_finite=False)
    return x


def backward(data, n, b, a, has_arrow, rhs):
    """L^T x = r (bta.py:278-302)."""
    d, lo, ar, tp = views(data, n, b, a)
    x = np.array(rhs, dtype=np.float64, copy=True)
    X = x.reshape(n * b + a, -1)
    if a:
        X[n * b :] = solve_triangular(tp, X[n * b :], lower=True, trans="T", check_finite=False)
    for i in range(n - 1, -1, -1):
        seg = X[i * b : (i + 1) * b]
        if i < n - 1:
            seg -= lo[i].T @ X[(i + 1) * b : (i + 2) * b]
        if a and has_arrow:
            seg -= ar[i].T @ X[n * b :]
        X[i * b : (i + 1) * b] = solve_triangular(
            d[i], seg, lower=True, trans="T", check_finite=False
        )
    return x


def solve(data, n, b, a, has_arrow, rhs):
    """bta.py:305-307."""
    return backward(data, n, b, a, has_arrow, forward(data, n, b, a, has_arrow, rhs))


def selected_invert(data, n, b, a, has_arrow):
    """POBTASI (bta.py:310-359); returns a new flat buffer."""
    d, lo, ar, tp = views(data, n, b, a)
    out = np.zeros_like(data)
    Xd, Xl, Xa, Xt = views(out, n, b, a)
    eye = np.eye(b)
    if a:
        ti = solve_triangular(tp, np.eye(a), lower=True, check_finite=False)
        Xt[...] = ti.T @ ti
    for i in range(n - 1, -1, -1):
        winv = solve_triangular(d[i], eye, lower=True, check_finite=False)
        sub = lo[i] if i < n - 1 else None
        arr = ar[i] if has_arrow else None
        xn = None
        if sub is not None:
            acc = Xd[i + 1] @ sub
            if has_arrow:
                acc += Xa[i + 1].T @ arr
            xn = -(acc @ winv)
            Xl[i] = xn
        xa = None
        if has_arrow:
            acc = Xt @ arr
            if sub is not None:
                acc += Xa[i + 1] @ sub
            xa = -(acc @ winv)
            Xa[i] = xa
        acc = winv.T
        if xn is not None:
            acc = acc - xn.T @ sub
        if xa is not None:
            acc = acc - xa.T @ arr
        Xd[i] = acc @ winv
    return out


def flops_pobtaf(n, b, a, arrow=True):
    """Algorithmic FLOPs of POBTAF."""
    f = n * b**3 / 3 + (n - 1) * 2 * b**3 + a**3 / 3
    if arrow:
        f += n * a * b**2 + (n - 1) * 2 * a * b**2 + n * a * a * b
    return float(f)


def flops_pobtasi(n, b, a, arrow=True):
    """Algorithmic FLOPs of POBTASI."""
    f = n * (b**3 / 3 + b**3) + (n - 1) * 5 * b**3 + 2 * a**3 / 3
    if arrow:
        f += n * (3 * a * b * b + 2 * a * a * b) + (n - 1) * 4 * a * b * b
    return float(f)


def bytes_pobtas(n, b, a):
    """Factor bytes read by one POBTAS sweep pair."""
    return 16.0 * (n * b * (b + 1) / 2 + (n - 1) * b * b + n * a * b + a * (a + 1) / 2)
