"""Timeline of BccPipeline over K copies of a config graph (device events per stream)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_17101_b200 as pg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5a"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dg = pg.make_config(cfg)
n, m = dg.n, dg.m
off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
tgt_h = torch.empty(m, dtype=torch.int32, pin_memory=True)
off_h.copy_(dg.offsets)
tgt_h.copy_(dg.targets)
del dg
torch.cuda.empty_cache()
g = pg.Graph(off_h.numpy(), tgt_h.numpy())
for _ in pg.BccPipeline().run([g, g]):
    pass
trace = []
pipe = pg.BccPipeline(trace=trace)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in pipe.run([g] * K):
    pass
torch.cuda.synchronize()
print(f"{cfg}: {K} graphs in {(time.perf_counter() - t0) * 1e3:.0f} ms")
e0 = trace[0][2]
for i, what, e in trace:
    print(f"  g{i} {what:14s} {e0.elapsed_time(e):9.1f} ms")
