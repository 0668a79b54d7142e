"""Algorithmic work formulas and device-side synthetic BTA inputs.

The FLOP / byte counts are the fixed, LAPACK-standard counts of SURVEY.md
§8(d), following the reference's operation sequence (bta.py:177-235,
249-307, 310-359); they are the numerators of every TFLOP/s and GB/s figure
this package reports, independent of how many operations the kernels actually
execute.
"""

import torch


def flops_pobtaf(n, b, a, arrow=True):
    """POBTAF(n,b,a) = n b^3/3 + (n-1) 2b^3 + a^3/3 [+ n a b^2 + (n-1) 2 a b^2 + n a^2 b]."""
    f = n * b**3 / 3 + (n - 1) * 2 * b**3 + a**3 / 3
    if arrow:
        f += n * a * b**2 + (n - 1) * 2 * a * b**2 + n * a * a * b
    return float(f)


def flops_pobtasi(n, b, a, arrow=True):
    """POBTASI(n,b,a) = n (b^3/3 + b^3) + (n-1) 5b^3 + 2a^3/3 [+ n (3ab^2 + 2a^2 b) + (n-1) 4ab^2]."""
    f = n * (b**3 / 3 + b**3) + (n - 1) * 5 * b**3 + 2 * a**3 / 3
    if arrow:
        f += n * (3 * a * b * b + 2 * a * a * b) + (n - 1) * 4 * a * b * b
    return float(f)


def flops_pobtas(n, b, a, nrhs=1):
    """POBTAS, forward + backward sweep: 2 (n b^2 + (n-1) 2b^2 + 2nab + a^2) per RHS."""
    return float(2 * (n * b * b + (n - 1) * 2 * b * b + 2 * n * a * b + a * a) * nrhs)


def bytes_pobtas(n, b, a):
    """Factor bytes read by one forward + backward sweep pair (each reads the factor once)."""
    return 16.0 * (n * b * (b + 1) / 2 + (n - 1) * b * b + n * a * b + a * (a + 1) / 2)


def storage_elems(n, b, a):
    return n * b * b + (n - 1) * b * b + n * a * b + a * a


@torch.no_grad()
def device_random_spd_bta(n, b, a, seed=0, device="cuda"):
    """SPD BTA matrix L L^T with the reference generator's distribution
    (bta.py:362-394: diag of L ~ 1 + U(0,1), off-diagonals ~ N(0, (0.3/sqrt b)^2)),
    drawn with torch's generator directly in HBM.  Same law as the reference,
    not the same bytes: used for the large benchmark inputs, where a host
    numpy draw of several GB would dominate the run; parity tests use the
    byte-identical host generator instead."""
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    sd = 0.3 / b**0.5
    f64 = torch.float64
    data = torch.zeros(storage_elems(n, b, a), dtype=f64, device=dev)
    e0 = n * b * b
    e1 = e0 + (n - 1) * b * b
    e2 = e1 + n * a * b
    D = data[:e0].view(n, b, b)
    S = data[e0:e1].view(n - 1, b, b)
    A = data[e1:e2].view(n, a, b)
    T = data[e2:].view(a, a)

    def lower_factor(m):
        x = torch.randn(m, m, dtype=f64, device=dev, generator=g) * sd
        x = torch.tril(x, -1)
        x.diagonal().copy_(1.0 + torch.rand(m, dtype=f64, device=dev, generator=g))
        return x

    fac_d = [lower_factor(b) for _ in range(n)]
    fac_s = [torch.randn(b, b, dtype=f64, device=dev, generator=g) * sd for _ in range(n - 1)]
    fac_a = [torch.randn(a, b, dtype=f64, device=dev, generator=g) * sd for _ in range(n)]
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
        ft = lower_factor(a)
        tip = ft @ ft.T
        for i in range(n):
            tip += fac_a[i] @ fac_a[i].T
        T.copy_(tip)
    return data


@torch.no_grad()
def device_random_spd_rows(n, b, a, t0, t1, seed=0, device="cuda", with_tip=True):
    """Block rows [t0, t1) of an SPD BTA matrix L L^T of the reference
    generator's law (bta.py:362-394), drawn in HBM by the rank that owns them:
    every factor block of L is drawn from its own generator seeded by (seed,
    block, kind), so any rank can produce its rows without the rest of the
    matrix (the partitioned benchmark).  Rows t need the
    factor blocks of t and t-1.  The tip (sum over ALL arrow factor blocks)
    is built when ``with_tip`` (the root)."""
    from .bta_dist import BTARows

    dev = torch.device(device)
    sd = 0.3 / b**0.5
    f64 = torch.float64

    def gen(i, kind):
        g = torch.Generator(device=dev)
        g.manual_seed(int(seed) * 1_000_003 + 4 * i + kind)
        return g

    def ld(i):  # lower factor of diagonal block i
        g = gen(i, 0)
        x = torch.tril(torch.randn(b, b, dtype=f64, device=dev, generator=g) * sd, -1)
        x.diagonal().copy_(1.0 + torch.rand(b, dtype=f64, device=dev, generator=g))
        return x

    def ls(i):  # factor block (i, i-1), i >= 1
        return torch.randn(b, b, dtype=f64, device=dev, generator=gen(i, 1)) * sd

    def la(i):  # arrow factor block of column block i
        return torch.randn(a, b, dtype=f64, device=dev, generator=gen(i, 2)) * sd

    rows = BTARows(n, t0, t1, b, a, dev, with_tip=with_tip)
    prev_d = ld(t0 - 1) if t0 > 0 else None
    prev_a = la(t0 - 1) if t0 > 0 and a else None
    for t in range(t0, t1):
        d = ld(t)
        rows.d(t).copy_(d @ d.T)
        if a:
            at = la(t)
            rows.arw(t).copy_(at @ d.T)
        if t > 0:
            s = ls(t)
            rows.d(t).add_(s @ s.T)
            rows.low(t).copy_(s @ prev_d.T)
            if a:
                rows.arw(t).add_(prev_a @ s.T)
        prev_d = d
        if a:
            prev_a = at
    if with_tip and a:
        g = gen(n, 3)
        ft = torch.tril(torch.randn(a, a, dtype=f64, device=dev, generator=g) * sd, -1)
        ft.diagonal().copy_(1.0 + torch.rand(a, dtype=f64, device=dev, generator=g))
        tip = ft @ ft.T
        for i in range(n):
            x = la(i)
            tip += x @ x.T
        rows.tip.copy_(tip)
    return rows
