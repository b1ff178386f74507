"""Degree skew of the spanning forest FAST-BCC builds (children per parent)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_17101_b200 as pg

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5a"
dg = pg.make_config(cfg)
r = pg.bcc_device(dg.offsets, dg.targets, forest=True)
par = r.parent.long()
n = dg.n
v = torch.arange(n, device=par.device)
nonroot = par != v
cnt = torch.bincount(par[nonroot], minlength=n)
top = torch.topk(cnt, 10)
print("n", n, "tree edges", int(nonroot.sum()), "max children", top.values.tolist(), "at", top.indices.tolist())
for k in [1, 10, 100, 1000, 10000]:
    print(f"vertices with >= {k} children: {int((cnt >= k).sum())}, holding {int(cnt[cnt >= k].sum())} children")
