"""Run FAST-BCC on RMAT / kNN / grid at increasing sizes in subprocesses; report failures."""
import subprocess
import sys

CASES = sys.argv[1:] or ["rmat:21", "rmat:22", "rmat:23", "rmat:24", "rmat:25", "knn:21", "knn:23", "knn:24", "knn:25"]
CODE = """
import sys; sys.path.insert(0, '.')
import torch, paper_2404_17101_b200 as pg
kind, s = '{k}', int('{s}')
dg = pg.gen_rmat(s, 8 << s, seed=1) if kind == 'rmat' else (pg.gen_knn(1 << s, 5, seed=1) if kind == 'knn' else pg.gen_grid(1 << (s // 2), 1 << (s - s // 2), 0.6, 1))
r = pg.bcc_device(dg.offsets, dg.targets)
torch.cuda.synchronize()
print('ok', kind, s, dg.n, dg.m, int(r.bcc_count.item()))
"""
for c in CASES:
    k, s = c.split(":")
    r = subprocess.run([sys.executable, "-c", CODE.format(k=k, s=s)], capture_output=True, text=True, timeout=600)
    print(c, "rc", r.returncode, (r.stdout.strip().splitlines() or [""])[-1], r.stderr.strip().splitlines()[-1:] if r.returncode else "",
          flush=True)
