"""Per-instruction stall samples of one kernel from `ncu -i X --page source --csv
--kernel-name regex:K --print-source sass`: totals per stall reason, and the top
instructions with their dominant reasons (the dependent load a stall waits on sits just
before the stalled instruction)."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    ri = [h.index(x) for x in reasons]
    seen, data = set(), []
    for r in rows[2:]:
        if len(r) <= si or not r[si].isdigit() or r[0] in seen:
            continue
        seen.add(r[0])
        data.append((int(r[si]), r[0], r[1].strip(), [int(r[i] or 0) for i in ri]))
    tot = sum(d[0] for d in data) or 1
    agg = [sum(d[3][k] for d in data) for k in range(len(reasons))]
    print("reasons:", " ".join(f"{reasons[k][6:]}={100 * agg[k] / tot:.0f}%" for k in
                               sorted(range(len(reasons)), key=lambda k: -agg[k]) if agg[k] * 50 > tot))
    order = {a: i for i, (_, a, _, _) in enumerate(data)}
    for s, a, src, rs in sorted(data, reverse=True)[:top]:
        why = " ".join(f"{reasons[k][6:]}:{100 * rs[k] / s:.0f}" for k in sorted(range(len(rs)), key=lambda k: -rs[k])[:2])
        print(f"{100 * s / tot:5.1f}% #{order[a]:5d} {src[:70]:70s} {why}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
