"""CPU: lane-exact emulation of the warp-chunk slot->row resolution and row segmentation
(paper_2404_17101_b200/csrc/wchunk.cuh), checked against brute force on the golden graphs
plus CSRs dominated by empty rows (isolated vertices, as in RMAT), and of the blocked
chunk protocol of k_tags_blk (row starts, sequential lane reduce, segmented scan, writes).  Catches index
arithmetic bugs without a GPU; the GPU parity tests check the kernels themselves."""

import numpy as np

from tests import golden_io

WCH = 256


def chunk_row(off, n, s):
    lo, hi = 0, n - 1
    while lo < hi:
        mid = (lo + hi + 1) >> 1
        if off[mid] <= s:
            lo = mid
        else:
            hi = mid - 1
    return lo


def resolve(off, n, cur, sb, valid):
    rows = [0] * 32
    done = [not v for v in valid]
    c = cur
    while True:
        d = []
        for lane in range(32):
            e = c + 1 + lane
            dd = int(off[e]) - sb if e <= n else 64
            d.append(0 if dd < 0 else (33 if dd > 33 else dd))
        for lane in range(32):
            pos = 0
            for step in (16, 8, 4, 2, 1):
                if d[pos + step - 1] <= lane:
                    pos += step
            if d[pos] <= lane:
                pos += 1
            if not done[lane] and pos < 32:
                rows[lane] = c + pos
                done[lane] = True
        if all(done):
            return rows
        c += 32


def segments(rows, valid):
    """(lo, hi, cut_left, cut_right) per valid lane, as wc_segment computes them."""
    heads = 0
    for lane in range(32):
        if valid[lane] and (lane == 0 or rows[lane - 1] != rows[lane]):
            heads |= 1 << lane
    last_valid = max(i for i in range(32) if valid[i])
    out = []
    for lane in range(32):
        le = (1 << (lane + 1)) - 1
        lo = (heads & le).bit_length() - 1
        after = heads & ~le & 0xFFFFFFFF
        hi = ((after & -after).bit_length() - 2) if after else last_valid
        out.append((lo, hi, lo == 0, not after))
    return out


def check_csr(off):
    n = off.shape[0] - 1
    m = int(off[-1])
    src = np.repeat(np.arange(n), np.diff(off))
    for c in range((m + WCH - 1) // WCH):
        s0, s1 = c * WCH, min(c * WCH + WCH, m)
        cur = chunk_row(off, n, s0)
        for sb in range(s0, s1, 32):
            valid = [sb + lane < s1 for lane in range(32)]
            rows = resolve(off, n, cur, sb, valid)
            cur = rows[31]
            segs = segments(rows, valid)
            for lane in range(32):
                if not valid[lane]:
                    continue
                assert rows[lane] == src[sb + lane]
                lo, hi, _, _ = segs[lane]
                assert all(rows[i] == rows[lane] for i in range(lo, hi + 1))
                assert lo == 0 or rows[lo - 1] != rows[lane]
                assert hi == 31 or not valid[hi + 1] or rows[hi + 1] != rows[lane]


def test_golden_graphs():
    for case in golden_io.kats() + golden_io.corpus()[:80] + [golden_io.single("rmat_s12_d16_seed7.npz")]:
        if case.m:
            check_csr(case.offsets)


def test_mostly_empty_rows():
    rng = np.random.default_rng(1)
    for trial in range(20):
        n = int(rng.integers(50, 3000))
        deg = np.where(rng.random(n) < 0.8, 0, rng.integers(1, 40, n))
        if trial % 4 == 0:
            deg[: n // 2] = 0                      # long run of isolated vertices
        if trial % 5 == 0:
            deg[int(rng.integers(0, n))] = 700     # a hub spanning several chunks
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        if off[-1]:
            check_csr(off)


def blk_rows(off, n, s0, s1, base):
    """Lane-exact emulation of wchunk.cuh blk_rows: per-lane start bytes, row of each
    lane's first slot, the row id at every start, and whether the chunk's last row
    continues past s1."""
    mask, rowat, last_open = 0, {}, False
    v0 = base
    while True:
        a = [int(off[v]) if v < n else int(off[n]) for v in range(v0, v0 + 32)]
        b = [int(off[v + 1]) if v + 1 <= n else int(off[n]) for v in range(v0, v0 + 32)]
        for lane in range(32):
            p = a[lane] - s0
            if b[lane] > a[lane] and 0 <= p < s1 - s0:
                rowat[p] = v0 + lane
                mask |= 1 << p
        hl = [lane for lane in range(32) if b[lane] > a[lane] and a[lane] < s1 and b[lane] >= s1]
        if hl:
            last_open = b[hl[0]] > s1
        if b[31] >= s1 or v0 + 32 >= n:
            break
        v0 += 32
    mb, rfirst = [], []
    for lane in range(32):
        p0 = 8 * lane
        mb.append((mask >> p0) & 0xFF)
        below = mask & ((2 << p0) - 1)
        rfirst.append(rowat[below.bit_length() - 1] if below else base)
    return mb, rfirst, rowat, last_open


def emulate_tags_blk(off, vals, first):
    """Lane-exact emulation of k_tags_blk (sequential lane reduce, segmented warp scan,
    boundary writes).  Returns W (min, max) per row; W starts at (first, first) like the
    preorder pass."""
    n = off.shape[0] - 1
    m = int(off[-1])
    INV = 0xFFFFFFFF
    W = [[int(first[r]), int(first[r])] for r in range(n)]
    stores = {}

    def write(row, mn, mx, atomic):
        f = int(first[row])
        if atomic:
            W[row][0] = min(W[row][0], mn)
            W[row][1] = max(W[row][1], mx)
        else:
            assert row not in stores, "non-atomic store twice"
            stores[row] = True
            W[row] = [min(mn, f), max(mx, f)]

    for c in range((m + WCH - 1) // WCH):
        s0, s1 = c * WCH, min(c * WCH + WCH, m)
        base = chunk_row(off, n, s0)
        if int(off[base + 1]) >= s1:        # one row over the whole chunk: warp min/max
            seg = [int(vals[s]) for s in range(s0, s1)]
            write(base, min(seg), max(seg), int(off[base]) < s0 or int(off[base + 1]) > s1)
            continue
        mb, rfirst, rowat, last_open = blk_rows(off, n, s0, s1, base)
        T, H, R, head, hst, inner = [], [], [], [], [], []
        for lane in range(32):
            sl = s0 + 8 * lane
            r, mn, mx, hmn, hmx, in_head = rfirst[lane], INV, 0, INV, 0, True
            hstart = bool(mb[lane] & 1)
            for i in range(8):
                if i > 0 and (mb[lane] >> i) & 1:
                    if in_head:
                        hmn, hmx, in_head = mn, mx, False
                        if hstart:
                            write(r, mn, mx, False)
                    else:
                        write(r, mn, mx, False)
                    r, mn, mx = rowat[8 * lane + i], INV, 0
                if sl + i < s1:
                    mn, mx = min(mn, int(vals[sl + i])), max(mx, int(vals[sl + i]))
            T.append((mn, mx))
            H.append((hmn, hmx))
            R.append(r)
            hst.append(hstart)
            inner.append((mb[lane] & 0xFE) != 0)
            head.append(hstart or inner[-1])
        # segmented inclusive scan (sequential equivalent of blk_seg_scan)
        C, started = [], []
        for lane in range(32):
            if head[lane] or lane == 0:
                C.append(T[lane])
                started.append(head[lane])
            else:
                C.append((min(C[-1][0], T[lane][0]), max(C[-1][1], T[lane][1])))
                started.append(started[-1])
        for lane in range(32):
            if inner[lane] and not hst[lane]:
                tmn, tmx = H[lane]
                pst = False
                if lane > 0:
                    tmn, tmx = min(tmn, C[lane - 1][0]), max(tmx, C[lane - 1][1])
                    pst = started[lane - 1]
                write(rfirst[lane], tmn, tmx, not pst)
            if lane < 31 and hst[lane + 1]:
                write(R[lane], C[lane][0], C[lane][1], not started[lane])
            if lane == 31:
                write(R[lane], C[lane][0], C[lane][1], (not started[lane]) or last_open)
    return W


def _random_csrs(seed, trials):
    rng = np.random.default_rng(seed)
    for trial in range(trials):
        n = int(rng.integers(20, 400))
        deg = np.where(rng.random(n) < 0.5, 0, rng.integers(1, 12, n))
        if trial % 3 == 0:
            deg[int(rng.integers(0, n))] = int(rng.integers(200, 900))   # hub spanning chunks
        if trial % 4 == 0:
            deg[rng.integers(0, n, 5)] = 32                              # exact window sizes
        if trial % 5 == 0:
            deg[rng.integers(0, n, 5)] = 8                               # exact lane sizes
        if trial % 7 == 0:
            deg[:] = np.where(rng.random(n) < 0.9, 0, 1)                 # mostly empty rows
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        if off[-1] == 0:
            continue
        yield trial, n, off, rng.integers(0, 10 * n, int(off[-1])), rng.permutation(n)


def test_tags_blk_write_protocol():
    for trial, n, off, vals, first in _random_csrs(5, 60):
        W = emulate_tags_blk(off, vals, first)
        for r in range(n):
            seg = vals[off[r]:off[r + 1]]
            want = [int(first[r]), int(first[r])] if seg.shape[0] == 0 else \
                [min(int(first[r]), int(seg.min())), max(int(first[r]), int(seg.max()))]
            assert W[r] == want, (trial, r)


def _validator_rule(off, tgt):
    """Slot-level restatement of k_validate_slots: checker iff (deg w, w) < (deg u, u);
    a checker finds its own copy of u in row w; checker and non-checker counts balance."""
    import bisect

    n = off.shape[0] - 1
    up = down = 0
    for u in range(n):
        for s in range(off[u], off[u + 1]):
            w = int(tgt[s])
            if w == u:
                continue
            du, dw = off[u + 1] - off[u], off[w + 1] - off[w]
            if not (dw < du or (dw == du and w < u)):
                down += 1
                continue
            up += 1
            k = 0
            while s - k - 1 >= off[u] and tgt[s - k - 1] == w:
                k += 1
            row = tgt[off[w]:off[w + 1]].tolist()
            q = bisect.bisect_left(row, u) + k
            if q >= len(row) or row[q] != u:
                return False
    return up == down


def test_validator_checker_rule_equals_oracle_is_symmetric():
    import oracle
    from tests import multigraph

    rng = np.random.default_rng(7)
    for trial in range(600):
        _, off, tgt = multigraph.perturbed(rng, trial)
        assert _validator_rule(off, tgt) == oracle.is_symmetric(off, tgt), trial


# --------------------------------------------------------------------------
# Two-level tags (k_tags2_blk): every slot carries a monotone 4-bit code of its value; the
# exact value is used only where the code equals the row's minimum or maximum code.
# --------------------------------------------------------------------------
NEUT = 0xFFFFFFFF
TAG_NB = 15


def _vminu2(a, b):
    return min(a & 0xFFFF, b & 0xFFFF) | (min(a >> 16, b >> 16) << 16)


def _pair(c):
    return c | ((TAG_NB - c) << 16)


def tags2_candidates(mb, codes, nvalid):
    """Lane-exact emulation of the candidate selection of k_tags2_blk's blocked path for one
    chunk: the lane's own pass, the forward / backward segmented scans over the lanes
    (Hillis-Steele steps with the segment bounds from one ballot), the second lane pass and
    the backward sweep.  mb[lane] = start bits, codes[p] for p < nvalid.  Returns the set of
    candidate positions."""
    ci = [[codes[8 * l + i] if 8 * l + i < nvalid else 0 for i in range(8)] for l in range(32)]
    val = [[8 * l + i < nvalid for i in range(8)] for l in range(32)]
    head, tail = [], []
    for l in range(32):
        acc, seen, h = NEUT, False, NEUT
        for i in range(8):
            if (mb[l] >> i) & 1:
                if not seen:
                    h = acc
                seen, acc = True, NEUT
            if val[l][i]:
                acc = _vminu2(acc, _pair(ci[l][i]))
        if not seen:
            h = acc
        head.append(h)
        tail.append(acc)
    hb = sum(1 << l for l in range(32) if mb[l])
    F, Bk = list(tail), list(head)
    lo, hi = [], []
    for l in range(32):
        le = hb & ((2 << l) - 1)
        lo.append(le.bit_length() - 1 if le else 0)
        ge = hb >> l
        hi.append(l + ((ge & -ge).bit_length() - 1) if ge else 31)
    o = 1
    while o < 32:
        Fn, Bn = list(F), list(Bk)
        for l in range(32):
            if l - o >= lo[l]:
                Fn[l] = _vminu2(F[l], F[l - o])
            if l + o <= hi[l]:
                Bn[l] = _vminu2(Bk[l], Bk[l + o])
        F, Bk = Fn, Bn
        o <<= 1
    cand = set()
    for l in range(32):
        fprev = F[l - 1] if l > 0 else NEUT
        bnext = Bk[l + 1] if l < 31 else NEUT
        fw, acc = [], fprev
        for i in range(8):
            if (mb[l] >> i) & 1:
                acc = NEUT
            if val[l][i]:
                acc = _vminu2(acc, _pair(ci[l][i]))
            fw.append(acc)
        full = _vminu2(fw[7], bnext)
        for i in range(7, -1, -1):
            if i < 7 and (mb[l] >> (i + 1)) & 1:
                full = fw[i]
            if val[l][i] and (ci[l][i] == (full & 0xFFFF) or TAG_NB - ci[l][i] == (full >> 16)):
                cand.add(8 * l + i)
    return cand


def emulate_tags2(off, vals, first, bounds):
    """k_tags2_blk: W (min, max) per row from the exact values of the candidate slots only."""
    n = off.shape[0] - 1
    m = int(off[-1])
    code = lambda x: int(np.searchsorted(bounds, x, side="right"))
    W = [[int(first[r]), int(first[r])] for r in range(n)]
    ncand = 0
    for c in range((m + WCH - 1) // WCH):
        s0, s1 = c * WCH, min(c * WCH + WCH, m)
        base = chunk_row(off, n, s0)
        codes = [code(int(vals[s])) for s in range(s0, s1)]
        if int(off[base + 1]) >= s1:        # one row over the whole chunk
            cb = code(int(first[base]))
            cmn, cmx = min(codes), max(codes)
            cmn = None if cmn > cb else cmn
            cmx = None if cmx < cb else cmx
            cand = [s for s in range(s0, s1) if codes[s - s0] in (cmn, cmx)]
            rows = {s: base for s in cand}
        else:
            mb, rfirst, rowat, _ = blk_rows(off, n, s0, s1, base)
            cset = tags2_candidates(mb, codes, s1 - s0)
            # candidates = exactly the slots at the extreme codes of their row within the chunk
            rowof, r = [], base
            for p in range(s1 - s0):
                r = rowat.get(p, r)
                rowof.append(r)
            for rr in set(rowof):
                ps = [p for p in range(s1 - s0) if rowof[p] == rr]
                lo, hi = min(codes[p] for p in ps), max(codes[p] for p in ps)
                assert {p for p in ps if p in cset} == {p for p in ps if codes[p] in (lo, hi)}, (c, rr)
            cand = [s0 + p for p in sorted(cset)]
            rows = {s0 + p: rowof[p] for p in cset}
        ncand += len(cand)
        for s in cand:
            r = rows[s]
            W[r][0] = min(W[r][0], int(vals[s]))
            W[r][1] = max(W[r][1], int(vals[s]))
    return W, ncand


def test_tags2_candidates_give_exact_tags():
    """For any monotone code, the candidate slots alone reproduce every row's min / max, and
    the candidate set is exactly the slots at their row's extreme codes (per chunk)."""
    rng = np.random.default_rng(11)
    for trial, n, off, vals, first in _random_csrs(9, 40):
        hi = 10 * n
        kinds = [np.sort(rng.integers(0, hi, TAG_NB)),                 # arbitrary boundaries
                 np.full(TAG_NB, hi + 1),                               # one code for everything
                 np.quantile(vals, np.linspace(0, 1, TAG_NB + 2)[1:-1]).astype(np.int64)]
        bounds = kinds[trial % 3]
        W, ncand = emulate_tags2(off, vals, first, bounds)
        for r in range(n):
            seg = vals[off[r]:off[r + 1]]
            want = [int(first[r]), int(first[r])] if seg.shape[0] == 0 else \
                [min(int(first[r]), int(seg.min())), max(int(first[r]), int(seg.max()))]
            assert W[r] == want, (trial, r)
        assert ncand <= int(off[-1])
