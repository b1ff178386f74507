"""Per-kernel roofline table of one BCC call from an ncu launch list (--metrics
gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv): DRAM GB/s against
the measured copy peak and DRAM 128-byte lines/s against the measured random-line rate
(profiles/random_access_peak.json).  A kernel near neither ceiling is latency-bound.

    python tools/kernel_rooflines.py profiles/r01_launches_c5a_v20.csv
"""
import collections
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        sc = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1, "byte": 1e-9,
              "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1, "Tbyte": 1e3}.get(d["Metric Unit"], 1)
        agg.setdefault((d["ID"], name), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * sc
    keys = list(agg)
    start = [i for i, k in enumerate(keys) if k[1] == "k_cc_local"][-1]   # the last BCC call
    peak = 6545.6
    try:
        peak = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    lines_peak = json.load(open(os.path.join(REPO, "profiles", "random_access_peak.json")))["hbm_random_lines_per_s"]
    per = collections.OrderedDict()
    for k in keys[start:]:
        nm = "k_scan (preorder)" if k[1] == "k_scan" else k[1]
        m = agg[k]
        a = per.setdefault(nm, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    print(f"| kernel | launches | ms | DRAM GB | GB/s | % of {peak:.0f} GB/s | G lines/s | % of {lines_peak / 1e9:.1f} G lines/s |")
    print("|---|---|---|---|---|---|---|---|")
    tot = 0.0
    for k, v in sorted(per.items(), key=lambda x: -x[1][1]):
        if v[1] < 0.05:
            continue
        tot += v[1]
        gbs = v[2] / (v[1] / 1e3)
        lps = v[2] / 128 / (v[1] / 1e3)
        print(f"| `{k}` | {v[0]} | {v[1]:.2f} | {v[2]:.1f} | {gbs:.0f} | {100 * gbs / peak:.0f} | {lps:.1f} | {100 * lps * 1e9 / lines_peak:.0f} |")
    print(f"\nsum of kernel times {tot:.2f} ms (serialised, cold-cache ncu replay)")


if __name__ == "__main__":
    main(sys.argv[1])
