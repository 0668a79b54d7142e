"""Host model of the POBTAF task graph's enumeration (csrc/pobtaf.cu:
band_rows / band_row / chunking / group_size /
decode), used by tests/test_host_logic.py to check on the CPU that the ticket
order covers every block-tile update exactly once, in panel order, and is a
topological order of the task dependencies (deadlock freedom of the
persistent kernel).  Test infrastructure; must mirror the device code."""

NSTRIP = 4
NGRP = 8


class Band:
    def __init__(self, n, b, a, use_arrow=True, nfact=-1):
        self.n, self.b, self.a = n, b, a
        self.nbt = (b + 127) // 128
        self.nat = (a + 127) // 128 if a > 0 else 0
        self.S = n * self.nbt + self.nat
        self.SP = self.S if nfact < 0 else nfact * self.nbt
        self.use_arrow = bool(use_arrow and a > 0)
        self.NB = n * self.nbt


def band_rows(g, s):
    if s >= g.NB:
        return g.S - s - 1, g.S - s - 1
    t = s // g.nbt
    end = min(t + 2, g.n) * g.nbt
    mb = end - s - 1
    return mb + (g.nat if g.use_arrow else 0), mb


def band_row(g, s, i, mb):
    return s + 1 + i if i < mb else g.NB + (i - mb)


def look(g):
    return 2 if g.nbt >= 24 else 3


def chunk_k(g):
    return 8 if g.nbt >= 24 else 4


def chunk_first(g, p):
    t, j = divmod(p, g.nbt)
    return t * g.nbt + (j // chunk_k(g)) * chunk_k(g)


def chunk_end(g, p):
    return min(chunk_first(g, p) + chunk_k(g) - 1, (p // g.nbt + 1) * g.nbt - 1)


def chunk_last(g, p):
    return p == chunk_end(g, p)


def cross_col(g, p, C):
    if p >= g.NB:
        return False
    return C >= chunk_end(g, p) + 1 + look(g)


def col_mode(g, p, c):
    """1 per panel, 2 chunk task at this panel, 0 elsewhere (pobtaf.cu col_mode)."""
    if p >= g.NB:
        return 1
    if cross_col(g, p, c):
        return 2 if chunk_last(g, p) else 0
    if c <= p + look(g) or g.nbt < 24:
        return 1
    return 2 if p == c - look(g) - 1 else 0


def g1_active(g, s):
    if s < 1:
        return False
    mp, mb = band_rows(g, s - 1)
    return mp >= 2 and band_row(g, s - 1, 1, mb) == s + 1


def g4_prev(g, s):
    if s < 1 or s >= g.SP:
        return False
    m, mb = band_rows(g, s)
    if m < 2:
        return False
    mp, mbp = band_rows(g, s - 1)
    return mp >= 3 and band_row(g, s - 1, 1, mbp) == s + 1 and \
        band_row(g, s - 1, 2, mbp) == band_row(g, s, 1, mb)


def group_size(g, kind, s):
    if s >= g.SP and kind not in (1, 5):
        return 0
    m = band_rows(g, s)[0] if s < g.S else 0
    if kind == 0:
        return NSTRIP if m >= 1 else 0
    if kind == 1:
        return NSTRIP if g1_active(g, s) else 0
    if kind == 2:
        return NSTRIP if m >= 1 else 0
    if kind == 3:
        return NSTRIP if m >= 2 else 0
    if kind == 4:
        return (1 if m >= 2 else 0) + (1 if g4_prev(g, s) else 0)
    if kind == 5:
        if s < 1:
            return 0
        p = s - 1
        mp, mb = band_rows(g, p)
        e = 0
        for j in range(1, mp):
            if col_mode(g, p, band_row(g, p, j, mb)) == 0:
                continue
            e += NSTRIP + (mp - 1 - j)
        return e - (NSTRIP if g1_active(g, s) else 0) - (1 if g4_prev(g, s) else 0)
    if kind == 6:
        return NSTRIP * (m - 2) if m >= 3 else 0
    return m - 2 if m >= 3 else 0


def decode(g, kind, s, local):
    """(type, s0, s, R, C, q); type 'T' TRSM, 'S' STRIP, 'U' UPDATE."""
    if kind == 0:
        return ("T", s, s, s + 1, s, local)
    if kind == 1:
        return ("S", s - 1, s - 1, s + 1, s + 1, local)
    if kind == 2:
        return ("S", s, s, s + 1, s + 1, local)
    if kind in (3, 6):
        _, mb = band_rows(g, s)
        off = 1 if kind == 3 else 2
        return ("T", s, s, band_row(g, s, off + local // NSTRIP, mb), s, local % NSTRIP)
    if kind == 4:
        _, mb = band_rows(g, s)
        ss = s - 1 if (local == 0 and g4_prev(g, s)) else s
        return ("U", ss, ss, band_row(g, s, 1, mb), s + 1, 0)
    if kind == 7:
        _, mb = band_rows(g, s)
        return ("U", s, s, band_row(g, s, 2 + local, mb), s + 1, 0)
    p = s - 1
    mp, mb = band_rows(g, p)
    skip = g1_active(g, s)
    hoist = 1 if g4_prev(g, s) else 0
    for j in range(1, mp):
        c = band_row(g, p, j, mb)
        mode = col_mode(g, p, c)
        if mode == 0:
            continue
        s0 = chunk_first(g, p) if mode == 2 else p
        ns = 0 if (j == 1 and skip) else NSTRIP
        hj = hoist if j == 1 else 0
        cnt = ns + (mp - 1 - j) - hj
        if local < cnt:
            if local < ns:
                return ("S", s0, p, c, c, local)
            return ("U", s0, p, band_row(g, p, j + 1 + hj + (local - ns), mb), c, 0)
        local -= cnt
    raise AssertionError("unreachable")


def tickets(g):
    """Every ticketed task in ticket order."""
    out = []
    for gi in range(NGRP * g.SP + 6):
        kind, s = gi % NGRP, gi // NGRP
        for local in range(group_size(g, kind, s)):
            out.append(decode(g, kind, s, local))
    return out


def check(g):
    """Raises AssertionError on a coverage / order violation; returns the
    number of UPDATE tasks."""
    tk = tickets(g)
    pos = {}
    upd = {}  # (R, C) -> list of (ticket, s0, s) for UPDATE / STRIP (per strip q for STRIP)
    for t, (typ, s0, s, R, C, q) in enumerate(tk):
        if typ == "T":
            assert (s, R, q) not in pos, ("dup trsm", s, R, q)
            pos[(s, R, q)] = t
        else:
            key = (R, C, q) if typ == "S" else (R, C)
            upd.setdefault(key, []).append((t, s0, s))
    # every tile of the band below / on the diagonal gets each panel exactly once, in order
    for s in range(g.SP):
        m, mb = band_rows(g, s)
        rows = [band_row(g, s, i, mb) for i in range(m)]
        for c in rows:
            for R in rows:
                if R < c:
                    continue
                keys = [(R, c, q) for q in range(NSTRIP)] if R == c else [(R, c)]
                for key in keys:
                    assert key in upd, ("missing tile", key, s)
    nupd = 0
    for key, lst in upd.items():
        R, C = key[0], key[1]
        panels = []
        for t, s0, s in lst:
            panels += list(range(s0, s + 1))
        want = [s for s in range(min(C, g.SP)) if R in
                [band_row(g, s, i, band_rows(g, s)[1]) for i in range(band_rows(g, s)[0])] and
                C in [band_row(g, s, i, band_rows(g, s)[1]) for i in range(band_rows(g, s)[0])]]
        assert panels == want, ("panel set/order", key, panels, want)
        # panel order of the tile's tasks follows ticket order
        ts = [t for t, _, _ in lst]
        assert ts == sorted(ts), ("tile update order", key)
        # dependencies: TRSM strips of every panel of the task come earlier
        for t, s0, s in lst:
            for sp in range(s0, s + 1):
                for q in range(NSTRIP):
                    for X in ((R, C) if R != C else (R,)):
                        if X < g.NB * 0 + g.S and (sp, X, q) in pos:
                            assert pos[(sp, X, q)] < t, ("dep after task", key, sp, X, q)
            if len(key) == 2:
                nupd += 1
    # a TRSM of panel s needs POTRF(s), i.e. every update of tile (s, s): all earlier
    for (s, R, q), t in pos.items():
        for qq in range(NSTRIP):
            for t2, _, _ in upd.get((s, s, qq), []):
                assert t2 < t, ("potrf dep", s, R, q)
        # and every update of its own tile (R, s)
        for t2, _, _ in upd.get((R, s), []):
            assert t2 < t, ("trsm tile dep", s, R)
    return nupd
