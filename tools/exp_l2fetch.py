import ctypes, os, sys, time, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2404_17101_b200 as pg
from paper_2404_17101_b200 import _lib
cudart = None
for name in ["libcudart.so.12", "libcudart.so"]:
    try:
        cudart = ctypes.CDLL(name); break
    except OSError:
        pass
if cudart is None:
    import glob
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    cudart = ctypes.CDLL(cands[0])
torch.cuda.init(); torch.zeros(1, device='cuda')
dg = pg.make_config('c5a'); torch.cuda.synchronize(); torch.cuda.empty_cache()
n, m = dg.n, dg.m
ws = torch.empty(pg.workspace_bytes(n, m), dtype=torch.uint8, device='cuda')
out = pg.DeviceBcc(edge_label=torch.empty(m, dtype=torch.int32, device='cuda'),
                   artic_bits=torch.empty((n+31)//32, dtype=torch.int32, device='cuda'),
                   bcc_count=torch.empty(1, dtype=torch.int64, device='cuda'))
cudaLimitMaxL2FetchGranularity = 0x05
for gran in [None, 32, 64, 128, 32]:
    if gran is not None:
        r = cudart.cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, ctypes.c_size_t(gran))
        v = ctypes.c_size_t(0); cudart.cudaDeviceGetLimit(ctypes.byref(v), cudaLimitMaxL2FetchGranularity)
        print('set', gran, 'rc', r, 'now', v.value)
    for _ in range(2): pg.bcc_device(dg.offsets, dg.targets, out=out, workspace=ws)
    torch.cuda.synchronize()
    S = _lib.NSTAGES
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(S)] for _ in range(3)]
    for k in range(3): pg.bcc_device(dg.offsets, dg.targets, out=out, workspace=ws, events=evs[k])
    torch.cuda.synchronize()
    st = {}
    for si in range(1, 10):
        st[_lib.STAGES[si]] = round(sum(evs[k][si-1].elapsed_time(evs[k][si]) for k in range(3)) / 3, 2)
    tot = sum(evs[k][0].elapsed_time(evs[k][9]) for k in range(3)) / 3
    print(gran, round(tot, 2), st, flush=True)
