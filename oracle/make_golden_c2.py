"""Golden vectors for the BTA microbench configuration itself (SURVEY.md §8(d)
C2, BASELINE configs[1]): random_spd_bta(default_rng(0), 48, 2048, 6)
(bta.py:362-394), rhs = rng.normal(size=N) from the same generator, then the
UNMODIFIED reference factorize / logdet / solve / selected_invert
(bta.py:177-359).  The full arrays are 3.2 GB each, so the fixture keeps the
log-determinant, input checksums and a few thousand seeded sample entries of
the input, the factor, the solution and the selected inverse from every
storage region (diag / lower / arrow / tip).  Test infrastructure only:

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_c2.py

Output: tests/golden/c2.npz.
"""

import os
import sys
import time

import numpy as np

from make_golden import OUT, REF

N_BLOCKS, BLOCK, ARROW = 48, 2048, 6


def sample_index(n, b, a, count=2500, seed=11):
    """Flat storage offsets: `count` entries from each of diag (lower triangle
    incl. the diagonal), lower and arrow, plus the whole tip; sorted."""
    rng = np.random.default_rng(seed)
    e0 = n * b * b
    e1 = e0 + (n - 1) * b * b
    e2 = e1 + n * a * b
    t = rng.integers(0, n, count)
    r = rng.integers(0, b, count)
    c = (rng.random(count) * (r + 1)).astype(np.int64)
    d = t * b * b + r * b + c
    dd = np.arange(n) * b * b + rng.integers(0, b, n) * (b + 1)  # diagonal entries
    lo = e0 + rng.integers(0, (n - 1) * b * b, count)
    ar = e1 + rng.integers(0, n * a * b, count)
    tip = e2 + np.arange(a * a)
    return np.unique(np.concatenate([d, dd, lo, ar, tip]).astype(np.int64))


def checksums(x):
    w = np.arange(1, x.size + 1, dtype=np.float64) / x.size
    return np.array([np.sum(x), np.sum(x * w), np.sum(np.abs(x))])


def main():
    sys.path.insert(0, REF)
    from stinla import bta

    n, b, a = N_BLOCKS, BLOCK, ARROW
    rng = np.random.default_rng(0)
    t0 = time.perf_counter()
    m = bta.random_spd_bta(rng, n, b, a)
    rhs = rng.normal(size=m.dim)
    t_gen = time.perf_counter() - t0
    idx = sample_index(n, b, a)
    out = {"shape": np.array([n, b, a]), "index": idx, "input": m.data[idx],
           "input_checksums": checksums(m.data), "rhs_checksums": checksums(rhs)}
    t0 = time.perf_counter()
    f = bta.factorize(m)
    t_f = time.perf_counter() - t0
    out["logdet"] = np.array([bta.logdet(f)])
    out["factor"] = f.matrix.data[idx]
    out["has_arrow"] = np.array([int(f.has_arrow)])
    t0 = time.perf_counter()
    x = bta.solve(f, rhs)
    t_s = time.perf_counter() - t0
    sidx = np.unique(np.concatenate([np.arange(0, m.dim, 37), np.arange(m.dim - a, m.dim)]))
    out["solve_index"] = sidx
    out["solve"] = x[sidx]
    out["solve_checksums"] = checksums(x)
    t0 = time.perf_counter()
    inv = bta.selected_invert(f)
    t_i = time.perf_counter() - t0
    out["sinv"] = inv.data[idx]
    # the inverse's diagonal (the marginal variances a caller reads)
    dg = np.concatenate([np.diagonal(inv.diag[i]) for i in range(n)] + [np.diagonal(inv.tip)])
    out["sinv_diag"] = dg[sidx]
    out["sinv_diag_checksums"] = checksums(dg)
    out["seconds"] = np.array([t_gen, t_f, t_s, t_i])
    np.savez_compressed(os.path.join(OUT, "c2.npz"), **out)
    print(f"c2 golden: logdet {out['logdet'][0]!r}; gen {t_gen:.1f} s, POBTAF {t_f:.1f} s, "
          f"POBTAS {t_s:.2f} s, POBTASI {t_i:.1f} s")


if __name__ == "__main__":
    main()
