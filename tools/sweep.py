"""Run bench.py for several library variants x configs; print ms/step and stage times.
    python tools/sweep.py --variants default,u4,u16 --configs c5a,c3,c4
"""
import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="default")
    ap.add_argument("--configs", default="c5a")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    for cfg in a.configs.split(","):
        for var in a.variants.split(","):
            env = dict(os.environ)
            if var != "default":
                env["PASGAL_BCC_LIB"] = os.path.join(REPO, "paper_2404_17101_b200", "lib", "variants", f"lib_{var}.so")
            r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--config", cfg, "--steps", str(a.steps),
                                "--warmup", "2", "--no-e2e", "--no-cpu-baseline"], env=env, capture_output=True, text=True)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                st = d["pipeline"]["stage_ms"]
                print(f"{cfg:4s} {var:8s} {d['ms_per_step']:9.3f} ms  " + " ".join(f"{k}={v:.2f}" for k, v in st.items()),
                      flush=True)
            except Exception:
                print(f"{cfg} {var} FAILED rc={r.returncode}: {r.stderr[-500:]}", flush=True)


if __name__ == "__main__":
    main()
