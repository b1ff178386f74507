"""Summarise ncu CSV exports: per-kernel launch table (from --metrics ... --csv) or the
key metrics of a --set full report (ncu -i X --page raw --csv)."""
import collections
import csv
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        key = (d.get("ID"), name)
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(unit, 1.0)
        agg.setdefault(key, {})[d["Metric Name"]] = v * scale
    per = collections.OrderedDict()
    for (i, name), m in agg.items():
        a = per.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in per.values())
    print(f"{'kernel':28s} {'n':>4s} {'ms':>9s} {'share':>6s} {'rd GB':>8s} {'wr GB':>8s} {'GB/s':>7s}")
    for k, v in sorted(per.items(), key=lambda x: -x[1][1]):
        gbs = (v[2] + v[3]) / (v[1] / 1e3) if v[1] else 0
        print(f"{k:28s} {v[0]:4d} {v[1]:9.3f} {100 * v[1] / tot:5.1f}% {v[2]:8.2f} {v[3]:8.2f} {gbs:7.0f}")
    print(f"total {tot:.3f} ms")


def full(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        print("-----", name)
        for w in want:
            if w in idx:
                print(f"  {w:58s} {r[idx[w]]:>14s} {units[idx[w]]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s[0] for s in st) or 1
        print("  stalls:", " ".join(f"{n}={100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:7]))


if __name__ == "__main__":
    (launches if sys.argv[1] == "launches" else full)(sys.argv[2])
