"""Stage times of one config under several environment settings, in ONE process (the
library reads its PASGAL_* knobs per call), L2 flushed between calls:
    python tools/env_sweep.py --config c5a --sets "PASGAL_TAGS_POL=0;PASGAL_TAGS_POL=1,PASGAL_TAGS_HOTDEG=64"
Sets are separated by ';', assignments inside a set by ','.  Each set runs twice
(interleaved) so drift between boxes/clocks shows.
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402
from paper_2404_17101_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5a")
    ap.add_argument("--sets", required=True)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--check", action="store_true", help="run checksum per set (canonical), must agree")
    ap.add_argument("--scale", type=int, default=0, help="RMAT configs: scale override (draws scaled along)")
    a = ap.parse_args()
    dg = pg.make_config(a.config, scale_override=a.scale or None)
    if a.scale:
        a.config += f"@{a.scale}"
    torch.cuda.synchronize()
    n, m = dg.n, dg.m
    ws = torch.empty(pg.workspace_bytes(n, m), dtype=torch.uint8, device="cuda")
    out = pg.DeviceBcc(edge_label=torch.empty(m, dtype=torch.int32, device="cuda"),
                       artic_bits=torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda"),
                       bcc_count=torch.empty(1, dtype=torch.int64, device="cuda"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sets = [s for s in a.sets.split(";") if s.strip()]
    base_env = {k: v for k, v in os.environ.items() if k.startswith("PASGAL_")}
    S = _lib.NSTAGES
    ref_sum = None
    for rnd in range(a.rounds):
        for s in sets:
            for k in [k for k in os.environ if k.startswith("PASGAL_") and k not in base_env]:
                del os.environ[k]
            for kv in s.split(","):
                if "=" in kv:
                    k, v = kv.split("=", 1)
                    os.environ[k.strip()] = v.strip()
            pg.bcc_device(dg.offsets, dg.targets, out=out, workspace=ws, graph=False)
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(S)] for _ in range(a.steps)]
            for k in range(a.steps):
                flush.zero_()
                pg.bcc_device(dg.offsets, dg.targets, out=out, workspace=ws, events=evs[k], graph=False)
            torch.cuda.synchronize()
            st = {}
            for si in range(1, S - 1):
                st[_lib.STAGES[si]] = sum(evs[k][si - 1].elapsed_time(evs[k][si]) for k in range(a.steps)) / a.steps
            tot = sum(evs[k][0].elapsed_time(evs[k][S - 2]) for k in range(a.steps)) / a.steps
            line = f"{a.config} [{s}] total {tot:.2f} " + " ".join(f"{k}={v:.2f}" for k, v in st.items())
            if a.check:
                r = pg.bcc_device(dg.offsets, dg.targets, workspace=ws, canonical=True, graph=False)
                cs = pg.canonical_checksum_device(r.edge_label, r.artic_bits, r.bcc_count)
                line += f" checksum {cs}"
                if ref_sum is None:
                    ref_sum = cs
                elif cs != ref_sum:
                    line += " MISMATCH"
            print(line, flush=True)


if __name__ == "__main__":
    main()
