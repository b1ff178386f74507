"""Generate tests/golden/adj_cases.json and grid10x10_ref.adj from the REAL reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_adj_golden.py

Each case is a byte string fed to the reference's own ``pasgal.graph.load_adj``
(graph.py:250-318); the fixture records what it returned (n, m, offsets, targets) or the
exception type and message it raised, with the file path replaced by ``{path}``.  The
device loader (paper_2404_17101_b200.io.load_adj) must reproduce every one.
/root/reference does not exist on the GPU box, so the fixtures are committed.
"""

import base64
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from pasgal.graph import from_edges, gen_grid, load_adj, save_adj, symmetrize  # noqa: E402

A = b"AdjacencyGraph"
W = b"WeightedAdjacencyGraph"


def j(*toks, sep=b"\n"):
    return sep.join(t if isinstance(t, bytes) else str(t).encode() for t in toks) + b"\n"


def cases():
    c = []
    add = lambda name, data, weighted=None: c.append((name, data, weighted))  # noqa: E731
    ok3 = [A, 3, 4, 0, 2, 3, 1, 2, 0, 0]
    add("ok_small", j(*ok3))
    add("ok_spaces_tabs_crlf", b"  " + j(*ok3, sep=b" \t\r\n\x0b\x0c"))
    add("ok_no_trailing_newline", j(*ok3)[:-1])
    add("ok_underscore_plus_zeros", j(A, 3, 4, b"+0", b"0_2", b"003", b"1", b"+2", b"0", b"-0"))
    add("ok_empty_graph", j(A, 0, 0))
    add("ok_isolated", j(A, 4, 2, 0, 0, 1, 2, 2, 1))
    add("ok_weighted", j(W, 2, 2, 0, 1, 1, 0, b"1.5", b"2e0"))
    add("ok_weighted_forms", j(W, 2, 2, 0, 1, 1, 0, b"inf", b"-1e-400"))
    add("ok_weighted_more", j(W, 3, 4, 0, 2, 3, 1, 2, 0, 0, b".5", b"5.", b"1_0.2_5", b"+1E-3"))
    add("empty_file", b"")
    add("whitespace_only", b"  \n\t\n\r\n")
    add("malformed_header", j(b"AdjGraph", 1, 0, 0))
    add("malformed_header_leading_ws", b"\n\n  " + j(b"Adjacency", 1, 0, 0))
    add("header_long", j(b"X" * 100, 1, 0, 0))
    add("weighted_mismatch_true", j(*ok3), True)
    add("weighted_mismatch_false", j(W, 2, 2, 0, 1, 1, 0, 1, 1), False)
    add("missing_counts_1", j(A))
    add("missing_counts_2", j(A, 5))
    add("missing_counts_trailing_ws", j(A, 5) + b"\n\n  ")
    add("invalid_count", j(A, b"x", 0))
    add("invalid_count_m", j(A, 1, b"2.0", 0))
    add("count_overflow", j(A, b"99999999999999999999", 0))
    add("negative_n", j(A, -1, 0))
    add("negative_m", j(A, 1, -3, 0))
    add("token_count_short", j(A, 2, 1, 0, 1))
    add("token_count_long", j(A, 2, 1, 0, 1, 0, 7, 8))
    add("invalid_offset", j(A, 2, 2, 0, b"1x", 1, 0))
    add("invalid_offset_underscore", j(A, 2, 2, 0, b"1__0", 1, 0))
    add("offset_overflow", j(A, 2, 2, 0, b"99999999999999999999", 1, 0))
    add("offset_overflow_then_invalid", j(A, 3, 2, 0, b"99999999999999999999", b"z", 1, 0))
    add("first_offset_nonzero", j(A, 2, 2, 1, 1, 1, 0))
    add("offset_gt_m", j(A, 3, 2, 0, 5, 1, 1, 0))
    add("offset_negative", j(A, 3, 2, 0, -1, 1, 1, 0))
    add("offsets_decrease", j(A, 4, 3, 0, 2, 1, 3, 1, 0, 0))
    add("invalid_target", j(A, 2, 2, 0, 1, b"1.0", 0))
    add("invalid_target_ctrl", j(A, 2, 2, 0, 1, b"1\x1c", 0))
    add("target_out_of_range", j(A, 2, 2, 0, 1, 1, 2))
    add("target_negative", j(A, 2, 2, 0, 1, -1, 0))
    add("target_overflow", j(A, 2, 2, 0, 1, 1, b"-99999999999999999999"))
    add("target_range_after_offset_error", j(A, 2, 2, 0, 3, 9, 0))
    add("invalid_target_after_offset_error", j(A, 2, 2, 0, 3, b"q", 0))
    add("n0_m1", j(A, 0, 1, 0))
    add("invalid_weight", j(W, 2, 2, 0, 1, 1, 0, b"1.5f", 1))
    add("weight_hex", j(W, 2, 2, 0, 1, 1, 0, b"0x1p3", 1))
    add("weight_negative", j(W, 2, 2, 0, 1, 1, 0, 1, b"-2"))
    add("weight_nan", j(W, 2, 2, 0, 1, 1, 0, b"nan", 1))
    add("weight_neg_inf", j(W, 2, 2, 0, 1, 1, 0, 1, b"-inf"))
    add("weight_negative_small", j(W, 2, 2, 0, 1, 1, 0, 1, b"-1e-300"))
    add("weight_subnormal_neg", j(W, 2, 2, 0, 1, 1, 0, 1, b"-1e-320"))
    add("weight_subnormal_neg_rounds_to_zero", j(W, 2, 2, 0, 1, 1, 0, b"-2e-324", b"-1e-330"))
    add("weight_subnormal_neg_min", j(W, 2, 2, 0, 1, 1, 0, b"-2e-324", b"-3e-324"))
    add("weight_subnormal_neg_frac", j(W, 2, 2, 0, 1, 1, 0, b"-0.000_3e-320", b"1"))
    add("weight_after_target_error", j(W, 2, 2, 0, 1, 1, 5, b"-1", 1))
    # a random symmetric multigraph-free graph written by the reference's own save_adj
    rng = np.random.default_rng(31)
    n = 500
    g = symmetrize(from_edges(n, rng.integers(0, n, 1500), rng.integers(0, n, 1500)))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.adj")
        save_adj(g, p)
        add("save_adj_random500", open(p, "rb").read())
    return c


POOL = [b"0", b"1", b"2", b"-0", b"+1", b"00", b"1_0", b"_1", b"1_", b"1__2", b"+-1", b"--1", b"1e5", b"1.",
        b".", b".5", b"inf", b"-inf", b"nan", b"NaN", b"Infinity", b"-1e-400", b"1e-320", b"-1e-320",
        b"-2e-324", b"-3e-324", b"-1e-310", b"9" * 25, b"-" + b"9" * 19, b"9223372036854775807",
        b"9223372036854775808", b"-9223372036854775808", b"x", b"1\x1c", b"\xff", b"0x1", b"1e1_0", b"1e_1",
        b"1_.5", b"1._5", b"+.5e-3", b"-0.0", b"-0e5", b"3", b"5", b"-1", b"-2"]


def fuzz(seed=4321, count=160):
    """Single-token mutations (replace / delete / duplicate) of small valid files."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        weighted = bool(i % 2)
        toks = [W if weighted else A, b"3", b"4", b"0", b"2", b"3", b"1", b"2", b"0", b"0"]
        if weighted:
            toks += [b"1.5", b"0", b"2e1", b"7"]
        k = int(rng.integers(0, len(toks)))
        op = int(rng.integers(0, 6))
        if op <= 3:
            toks[k] = POOL[int(rng.integers(0, len(POOL)))]
        elif op == 4:
            del toks[k]
        else:
            toks.insert(k, POOL[int(rng.integers(0, len(POOL)))])
        seps = [b"\n", b" ", b"\t", b"\r\n", b"\x0b", b"\x0c"]
        data = b"".join(t + seps[int(rng.integers(0, len(seps)))] for t in toks)
        out.append((f"fuzz{i:03d}", data, None if i % 3 else weighted))
    return out


def run(name, data, weighted):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "case.adj")
        with open(p, "wb") as f:
            f.write(data)
        try:
            g = load_adj(p, weighted)
        except Exception as e:  # noqa: BLE001 -- record exactly what the reference raised
            return {"error": type(e).__name__, "message": str(e).replace(p, "{path}")}
        return {"n": int(g.n), "m": int(g.m), "offsets": [int(x) for x in g.offsets],
                "targets": [int(x) for x in g.targets]}


def main():
    out = []
    for name, data, weighted in cases() + fuzz():
        out.append({"name": name, "data_b64": base64.b64encode(data).decode(), "weighted": weighted,
                    "expect": run(name, data, weighted)})
    with open(os.path.join(HERE, "adj_cases.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("adj cases", len(out), "errors", sum("error" in c["expect"] for c in out))
    save_adj(gen_grid(10, 10), os.path.join(HERE, "grid10x10_ref.adj"))
    print("grid10x10_ref.adj written by pasgal.graph.save_adj")


if __name__ == "__main__":
    main()
