"""CPU: lane-exact emulation of the warp-chunk slot->row resolution and row segmentation
(paper_2404_17101_b200/csrc/wchunk.cuh), checked against brute force on the golden graphs
plus CSRs dominated by empty rows (isolated vertices, as in RMAT).  Catches index
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


def emulate_tags(off, vals, first):
    """Lane-exact emulation of k_tags' segment reduce + carry/flush/atomic write protocol.
    Returns W (min, max) per row; W starts at (first, first) like the preorder pass."""
    n = off.shape[0] - 1
    m = int(off[-1])
    W = [[int(first[r]), int(first[r])] for r in range(n)]
    stores = {}                     # rows written without atomics (must be written once)

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
        cur = chunk_row(off, n, s0)
        crw, cmn, cmx, cbefore = None, None, None, False
        for k in range(8):
            sb = s0 + 32 * k
            if sb >= s1:
                break
            valid = [sb + lane < s1 for lane in range(32)]
            rows = resolve(off, n, cur, sb, valid)
            cur = rows[31]
            segs = segments(rows, valid)
            mn = [None] * 32
            mx = [None] * 32
            for lane in range(32):
                if valid[lane]:
                    lo, hi, _, _ = segs[lane]
                    seg_vals = [vals[sb + i] for i in range(lo, hi + 1)]
                    mn[lane], mx[lane] = min(seg_vals), max(seg_vals)
            row0 = rows[0]
            if crw is not None and crw != row0:
                write(crw, cmn, cmx, cbefore)
                crw = None
            merged = crw is not None
            before = [False] * 32
            for lane in range(32):
                lo = segs[lane][0]
                if merged and lo == 0 and valid[lane]:
                    mn[lane], mx[lane] = min(mn[lane], cmn), max(mx[lane], cmx)
                before[lane] = lo == 0 and (cbefore if merged else k == 0)
            has_next = sb + 32 < s1
            for lane in range(32):
                lo, hi, _, cut_right = segs[lane]
                if valid[lane] and lane == lo and not (cut_right and has_next):
                    write(rows[lane], mn[lane], mx[lane], before[lane] or cut_right)
            if has_next:
                crw, cmn, cmx, cbefore = rows[31], mn[31], mx[31], before[31]
            else:
                crw = None
    return W


def test_tags_write_protocol():
    rng = np.random.default_rng(3)
    for trial in range(25):
        n = int(rng.integers(20, 400))
        deg = np.where(rng.random(n) < 0.5, 0, rng.integers(1, 12, n))
        if trial % 3 == 0:
            deg[int(rng.integers(0, n))] = int(rng.integers(200, 900))   # hub spanning chunks
        if trial % 4 == 0:
            deg[rng.integers(0, n, 5)] = 32                              # exact window sizes
        off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
        m = int(off[-1])
        if m == 0:
            continue
        vals = rng.integers(0, 10 * n, m)
        first = rng.permutation(n)
        W = emulate_tags(off, vals, first)
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
