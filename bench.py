#!/usr/bin/env python
"""bench.py -- FAST-BCC on B200: BASELINE.json's metric on its headline config.

Metric: "BCC edges/sec per B200 (device-timed); achieved HBM GB/s vs ~8 TB/s peak".
Default workload: BASELINE configs[4](a), RMAT scale 28 / 2^31 draws (avg degree 16), the
graph the north-star target (>= 30% of HBM peak) is stated on.  One step = one FAST-BCC
call (S2-S6: spanning forest, rooting, tags, skeleton, labels + articulation + count) over
the device-resident CSR.  value = undirected edges processed by all ranks / max-over-ranks
device time (CUDA events on the launching stream).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5a|c1|c2|c3|c4]
  python bench.py --impl reference ...   # the reference CPU path (oracle port) on host cores

Multi-GPU: BCC of one graph does not shard, so N>1 runs N independent
replicas (config 5b style: each rank its own seeded instance), no collective on the data
path; torch.distributed is used only for the barrier and the max/sum of the timings.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "BCC edges/sec per B200 (device-timed); achieved HBM GB/s vs ~8 TB/s peak"
UNIT = "edges/s"
L2_BYTES = 126 * 2**20

# algorithmic bytes: counted once per pass that needs
# the field, at element width, random gathers at 4 B, no credit for sector over-fetch
def b_alg_pipeline(n, m):
    return 56 * m + 180 * n


KERNEL_BYTES = {
    # k_tags: per slot target 4 + first[w] 4; per vertex offsets 8 + first[u] 4 + w1/w2 write 8
    "tags": lambda n, m: 8 * m + 20 * n,
    # k_labels: per slot target 4 + CID[w] 4 (one gather; the giant bitmap only avoids some of
    # them) + label write 4; per vertex offsets 8 + CID[u] 4
    "labels": lambda n, m: 12 * m + 12 * n,
}
KERNEL_NAMES = {"tags": "k_tags_blk", "labels": "k_labels"}


def assign_instances(n_instances, rank, world):
    """Config 5b: instances dealt round-robin to ranks (no data exchange between ranks)."""
    return list(range(rank, n_instances, world))


def reduce_over_ranks(total_ms, edges, device):
    """Max of the device times and sum of the work over all ranks (timing plumbing only;
    nothing on the data path is exchanged)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(total_ms), float(edges)
    t = torch.tensor([float(total_ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e = torch.tensor([float(edges)], dtype=torch.float64, device=device)
    dist.all_reduce(e, op=dist.ReduceOp.SUM)
    return float(t.item()), float(e.item())


def _sync():
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def _allreduce(vals, op, device):
    """Element-wise all-reduce of a list of floats (identity on one rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in vals]
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return [float(v) for v in t.tolist()]


def e2e_ranks(n, m, world, device):
    """How many ranks run the e2e legs at once: each needs its pinned host CSR and pinned
    output buffers (C5a: 19.2 + 17.3 GB), and N ranks on one node must not exhaust its
    memory.  Ranks 0..k-1 run them concurrently, the rest wait at the same barriers; k is
    the minimum over ranks so every rank takes the same decision."""
    import torch.distributed as dist

    need = (8 * (n + 1) + 4 * m) + (4 * m + n + 8)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    try:
        import psutil

        k = int(0.7 * psutil.virtual_memory().available // max(need, 1))
    except Exception:
        k = local_world
    k = max(0, min(k, local_world)) * max(1, world // max(local_world, 1))
    return int(_allreduce([k], dist.ReduceOp.MIN, device)[0]) if world > 1 else min(k, 1)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


def traffic_from_profiles(config, kernel):
    """ncu dram bytes per launch for `kernel` on `config`, from the committed summary
    (profiles/traffic.json, written from an `ncu --set full` capture), else None."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d[config][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def random_access_roofline(traffic, kernel_ms):
    """The dominant kernels are random-gather bound, and on this part every HBM miss moves
    a whole 128-byte line, so their ceiling is lines/s, not bytes/s: DRAM lines fetched per
    launch (ncu traffic / 128) over the live kernel time, against the measured random-line
    rate of tools/probes/gather_probe.cu (profiles/random_access_peak.json)."""
    try:
        with open(os.path.join(REPO, "profiles", "random_access_peak.json")) as f:
            pk = json.load(f)
    except Exception:
        return None
    if not traffic:
        return None
    lines = traffic / pk["bytes_per_miss"]
    ach = lines / (kernel_ms / 1e3)
    return {"achieved_lines_per_s": ach, "peak_lines_per_s": pk["hbm_random_lines_per_s"],
            "frac": ach / pk["hbm_random_lines_per_s"], "lines_per_launch": lines,
            "peak_source": "profiles/random_access_peak.json (measured, tools/probes/gather_probe.cu)"}


# --------------------------------------------------------------------------------------
# reference arm: the reference's CPU BCC (Hopcroft-Tarjan, oracles.py:119-201) restated in
# C (oracle/), on all host cores, on a bounded sample of the same workload
# --------------------------------------------------------------------------------------

SAMPLE_DESC = ("RMAT scale 20, 2^24 draws, (a,b,c)=(.57,.19,.19), seed 1 -- the same generator "
               "rules as the bench workload at 1/256 of its size (= BASELINE configs[1])")
SAMPLE_CONFIG = "c2"


def cpu_sample_graph():
    """The bounded CPU sample (BASELINE configs[1]), built on the host by the generator twin
    (oracle/gen_host.c; equal to the device generator's output, tests/test_oracle.py), so the
    reference arm never loads libpasgal_bcc.so."""
    import oracle

    return oracle.rmat(20, 1 << 24, seed=1)


def oracle_rate(off, tgt, threads=1):
    """Run `threads` concurrent oracle instances; returns (seconds, undirected edges done)."""
    import oracle

    mu = (tgt.shape[0]) // 2
    res = [None] * threads

    def work(i):
        t0 = time.perf_counter()
        oracle.bcc_hopcroft_tarjan(off, tgt)
        res[i] = time.perf_counter() - t0

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return time.perf_counter() - t0, mu * threads


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def _python_reference_worker(args):
    """One process: the UNMODIFIED reference (baseline/_ref, pip-installed from the
    reference package) -- pasgal.oracles.bcc_hopcroft_tarjan (oracles.py:119-201) -- on C1."""
    off, tgt, reps = args
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from pasgal.graph import Graph
    from pasgal.oracles import bcc_hopcroft_tarjan

    g = Graph(off, tgt)
    bcc_hopcroft_tarjan(g)                      # warm-up (imports, numba-free path)
    t0 = time.perf_counter()
    for _ in range(reps):
        r = bcc_hopcroft_tarjan(g)
    return time.perf_counter() - t0, int(r.bcc_count)


def python_reference_rate(procs, reps=3):
    """The reference's own Python CPU path on BASELINE configs[0] (C1, grid 256^2 p=0.6,
    the reference's CPU-runnable case), `procs` concurrent processes, or None when
    baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "pasgal")):
        return None
    import multiprocessing as mp

    import oracle

    off, tgt = oracle.gen_grid(256, 256, 0.6, 1)
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_python_reference_worker, [(off, tgt, reps)] * procs)
    wall = time.perf_counter() - t0
    per = max(r[0] for r in res)
    mu = tgt.shape[0] // 2
    return {"value": mu * reps * procs / per, "unit": UNIT, "cores": procs, "kind": "reference",
            "config": "c1: grid 256x256, p=0.6, seed 1 (BASELINE configs[0])",
            "bcc_count": res[0][1], "seconds_per_call": per / reps, "wall_s": round(wall, 1),
            "path": "pasgal.oracles.bcc_hopcroft_tarjan from baseline/_ref (pip install --no-deps of "
                    "/root/reference/pkg), unmodified; one instance per process"}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    off, tgt = cpu_sample_graph()
    for _ in range(args.warmup):
        oracle_rate(off, tgt, cores)
    times, edges = [], 0
    for _ in range(args.steps):
        dt, e = oracle_rate(off, tgt, cores)
        times.append(dt)
        edges += e
    total = sum(times)
    value = edges / total
    pyref = None
    try:
        pyref = python_reference_rate(cores)
    except Exception as e:  # noqa: BLE001 -- reported, the C-port line stands
        pyref = {"unavailable": f"{type(e).__name__}: {e}"}
    cfg = workload_config(SAMPLE_CONFIG)
    cfg.update(n=int(off.shape[0] - 1), m_slots=int(tgt.shape[0]),
               sample_of=workload_config(args.config)["workload"],
               note=f"a bounded sample of the GPU arm's workload: the same generator rules at 1/256 of its size")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{SAMPLE_DESC}; {cores} concurrent instances per step (one per host thread) "
                                   "of oracle/bcc_oracle.c, the C restatement of bcc_hopcroft_tarjan"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "python_reference": pyref,
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name):
    import importlib

    g = importlib.import_module("paper_2404_17101_b200.graph")
    return {"workload": f"{name}: {g.CONFIGS[name]['desc']}", "ids": "int32", "offsets": "int64"}


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------

def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    import paper_2404_17101_b200 as pg
    from paper_2404_17101_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    cfg_seed = pg.CONFIGS[args.config]["seed"] + rank   # independent replica per rank
    t0 = time.perf_counter()
    dg = pg.make_config(args.config, device=dev, seed=cfg_seed)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    torch.cuda.empty_cache()
    n, m = dg.n, dg.m
    mu = m // 2
    ws = torch.empty(pg.workspace_bytes(n, m), dtype=torch.uint8, device=dev)
    out = pg.DeviceBcc(edge_label=torch.empty(m, dtype=torch.int32, device=dev),
                       artic_bits=torch.empty((n + 31) // 32, dtype=torch.int32, device=dev),
                       bcc_count=torch.empty(1, dtype=torch.int64, device=dev))
    working_set = 8 * (n + 1) + 4 * m + 4 * m + ws.numel()
    flush = None
    if working_set < 4 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)

    def step(events=None):
        return pg.bcc_device(dg.offsets, dg.targets, seed=args.seed, out=out, workspace=ws, events=events)

    for _ in range(args.warmup):
        if flush is not None:
            flush.fill_(1)
        step()
    torch.cuda.synchronize()
    S = _lib.NSTAGES
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(S)] for _ in range(args.steps)]
    launches = 0
    sampler = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    win0 = torch.cuda.Event(enable_timing=True)
    win1 = torch.cuda.Event(enable_timing=True)
    win0.record()
    for k in range(args.steps):
        if flush is not None:
            flush.fill_(k)
        r = step(evs[k])
        launches += r.launches
    win1.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    LAB = _lib.STAGES.index("labels")
    step_ms = [evs[k][0].elapsed_time(evs[k][LAB]) for k in range(args.steps)]
    stage_ms = {}
    for si in range(1, LAB + 1):
        stage_ms[_lib.STAGES[si]] = statistics.mean(evs[k][si - 1].elapsed_time(evs[k][si]) for k in range(args.steps))
    total_ms = sum(step_ms)
    window_ms = win0.elapsed_time(win1)
    total_ms, edges = reduce_over_ranks(total_ms, mu * args.steps, dev)
    value = edges / (total_ms / 1e3)

    peak, peak_src = measured_peak()
    # dominant kernel among the single-kernel stages
    dom = max(KERNEL_BYTES, key=lambda s: stage_ms[s])
    kb = KERNEL_BYTES[dom](n, m)
    achieved = kb / (stage_ms[dom] / 1e3) / 1e9
    pipe_bytes = b_alg_pipeline(n, m)
    pipe_gbs = pipe_bytes / (statistics.mean(step_ms) / 1e3) / 1e9
    kname = KERNEL_NAMES[dom]
    if dom == "tags" and _lib.load().pasgal_bcc_two_level_tags(n, m):
        # two-level tags: the stage is k_tag_bounds + k_tag_codes (~1 % of it) + k_tags2_blk
        kname = "k_tags2_blk"
    traffic = traffic_from_profiles(args.config, kname)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname,
                "algorithmic_bytes_per_launch": kb, "kernel_ms": stage_ms[dom], "peak_source": peak_src,
                "random_access": random_access_roofline(traffic, stage_ms[dom])}
    pipeline = {"algorithmic_bytes": pipe_bytes, "model": "56*M + 180*n (SURVEY 8(d))",
                "achieved_gbs": pipe_gbs, "frac": pipe_gbs / peak,
                "stage_ms": {k: round(v, 4) for k, v in stage_ms.items()},
                "stage_share": {k: round(v / statistics.mean(step_ms), 4) for k, v in stage_ms.items()}}

    # ---- run checksum of the LAST TIMED step's output (outside the timed region): its raw
    # labels canonicalised on the device, checksummed, and compared with the value pinned
    # from the oracle-verified output of the same CSR (tests/golden/c5a_oracle_hashes.json)
    run_checksum = None
    if not args.no_checksum:
        canon = pg.canonicalize_device(dg.offsets, dg.targets, out.edge_label, label_bound=max(n, 1))
        cs = pg.canonical_checksum_device(canon, out.artic_bits, out.bcc_count)
        del canon
        torch.cuda.empty_cache()
        pinned = pinned_checksum(args.config, cfg_seed, n, m)
        run_checksum = {"value": [str(x) for x in cs], "pinned": pinned,
                        "match": (None if pinned is None else [str(x) for x in cs] == pinned),
                        "rule": "(bcc_count, articulation points, sum canon[s]*(((s*0x9E3779B1) mod 2^32)|1) "
                                "mod 2^64) of the last timed step's labels, canonicalised after the timing"}

    # ---- e2e through the public drop-in call with host buffers (pinned), H2D + D2H timed
    e2e = None
    if not args.no_e2e:
        k = e2e_ranks(n, m, world, dev)
        if k == 0:
            e2e = {"unavailable": "host memory cannot hold one rank's pinned CSR and output buffers"}
        else:
            # host copy of the CSR (pinned), then free every device buffer of the device-timed
            # arm: the e2e arms allocate their own (the pipelined one keeps two graphs in flight)
            off_h = tgt_h = None
            if rank < k:
                off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
                tgt_h = torch.empty(m, dtype=torch.int32, pin_memory=True)
                off_h.copy_(dg.offsets)
                tgt_h.copy_(dg.targets)
            del dg, ws, out, r
            torch.cuda.empty_cache()
            e2e = run_e2e(args, off_h, tgt_h, dev, n, m, rank < k, k, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        oracle.build()
        off_s, tgt_s = cpu_sample_graph()
        dt, e = oracle_rate(off_s, tgt_s, 1)
        cpu = {"value": e / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{SAMPLE_DESC}; one run of the C restatement of bcc_hopcroft_tarjan "
                         f"(incl. its is_symmetric + twin passes), {dt:.2f} s"}

    # ---- the other BASELINE configs, device-timed (L2 flushed between steps), and the CPU
    # sample config through bcc(g) end to end: a like-for-like pair for the reference arm
    per_config = same_config = None
    if not args.no_per_config and args.config == "c5a":
        per_config, same_config = run_per_config(args, dev, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": dict(workload_config(args.config), n=n, m_slots=m, m_undirected=mu, seed=cfg_seed,
                           replicas=world,
                           l2=("L2 flushed between steps (256 MB write)" if flush is not None else
                               f"inputs larger than L2 (CSR {(8 * (n + 1) + 4 * m) / 1e9:.1f} GB)"),
                           generation_s=round(gen_s, 2)),
            "roofline": roofline,
            "pipeline": pipeline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "window_ms": window_ms,
            "run_checksum": run_checksum,
            "per_config": per_config,
            "same_config": same_config,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def pinned_checksum(config, seed, n, m):
    """The canonical checksum pinned for (config, seed) in tests/golden/*_oracle_hashes.json
    (written from an output whose full labels hashed equal to the oracle's), else None."""
    try:
        with open(os.path.join(REPO, "tests", "golden", f"{config}_oracle_hashes.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    if d.get("n") != n or d.get("m_slots") != m or "checksum" not in d or d.get("seed", 1) != seed:
        return None
    return [str(x) for x in d["checksum"]]


def time_device(pg, torch, dg, steps, warmup, seed=0):
    """Mean device ms of one pasgal_bcc call on a resident CSR, L2 flushed between steps."""
    n, m = dg.n, dg.m
    ws = torch.empty(pg.workspace_bytes(n, m), dtype=torch.uint8, device=dg.offsets.device)
    out = pg.DeviceBcc(edge_label=torch.empty(max(m, 1), dtype=torch.int32, device=ws.device),
                       artic_bits=torch.empty(max((n + 31) // 32, 1), dtype=torch.int32, device=ws.device),
                       bcc_count=torch.empty(1, dtype=torch.int64, device=ws.device))
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=ws.device)
    for _ in range(warmup):
        flush.fill_(1)
        pg.bcc_device(dg.offsets, dg.targets, seed=seed, out=out, workspace=ws)
    torch.cuda.synchronize()
    tot = 0.0
    launches = 0
    for k in range(steps):
        flush.fill_(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launches += pg.bcc_device(dg.offsets, dg.targets, seed=seed, out=out, workspace=ws).launches
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / steps, launches // steps


def run_per_config(args, dev, world):
    """Device time of C1-C4 (each: generate, warm up, time, free) and the CPU sample config
    (C2) through the public bcc(g) with pinned host buffers -- the reference arm's config."""
    import torch

    import paper_2404_17101_b200 as pg

    per = {}
    same = None
    for name in ("c1", "c2", "c3", "c4"):
        dg = pg.make_config(name, device=dev)
        torch.cuda.synchronize()
        ms, nl = time_device(pg, torch, dg, steps=10, warmup=3)
        if world > 1:
            import torch.distributed as dist

            ms = _allreduce([ms], dist.ReduceOp.MAX, dev)[0]
        per[name] = {"ms": round(ms, 4), "edges_per_s": (dg.m // 2) / (ms / 1e3), "n": dg.n, "m_slots": dg.m,
                     "launches": nl}
        if name == SAMPLE_CONFIG:
            off_h = torch.empty(dg.n + 1, dtype=torch.int64, pin_memory=True)
            tgt_h = torch.empty(dg.m, dtype=torch.int32, pin_memory=True)
            off_h.copy_(dg.offsets)
            tgt_h.copy_(dg.targets)
            g = pg.Graph(off_h.numpy(), tgt_h.numpy())
            hb = pg.HostBuffers.allocate(dg.n, dg.m)
            for _ in range(3):
                pg.bcc(g, device=dev, host_out=hb)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 10
            for _ in range(reps):
                r = pg.bcc(g, device=dev, host_out=hb)
            e2e_s = (time.perf_counter() - t0) / reps
            same = {"config": workload_config(name)["workload"],
                    "device": {"value": (dg.m // 2) / (ms / 1e3), "unit": UNIT, "ms_per_step": round(ms, 4)},
                    "e2e": {"value": (dg.m // 2) / e2e_s, "unit": UNIT, "ms_per_step": round(e2e_s * 1e3, 3),
                            "h2d_bytes_per_step": 8 * (dg.n + 1) + 4 * dg.m,
                            "d2h_bytes_per_step": 4 * dg.m + dg.n + 8, "bcc_count": int(r.bcc_count),
                            "path": "paper_2404_17101_b200.bcc(g): H2D, validate, FAST-BCC, D2H (pinned)"},
                    "note": "the reference arm's config (bench.py --impl reference times its CPU path on it)"}
            del hb, g, off_h, tgt_h, r
        del dg
        pg.release_workspace()
        torch.cuda.empty_cache()
    return per, same


def run_batch(args, rank, world, local):
    """Config 5b: a batch of `--instances` independent 4096x4096 p=0.6 grids (seeds 1..64),
    dealt round-robin to the ranks, each generated on its GPU and kept resident; one step =
    FAST-BCC over all of the rank's instances.  Reports edges/s and instances/s."""
    import torch

    import paper_2404_17101_b200 as pg

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    mine = assign_instances(args.instances, rank, world)
    graphs = [pg.gen_grid(4096, 4096, 0.6, 1 + i, device=dev) for i in mine]
    torch.cuda.synchronize()
    nmax = max((g.n for g in graphs), default=1)
    mmax = max((g.m for g in graphs), default=1)
    # independent instances run concurrently on S streams (each with its own workspace and
    # outputs): a single 4096^2 grid is latency-bound and leaves the GPU partly idle
    S = max(1, min(args.streams, len(graphs)))
    streams = [torch.cuda.Stream(device=dev) for _ in range(S)]
    wss = [torch.empty(pg.workspace_bytes(nmax, mmax), dtype=torch.uint8, device=dev) for _ in range(S)]
    # one output per instance (a workspace per stream): the outputs of the last timed step
    # are the ones checksummed and verified below
    outs = [pg.DeviceBcc(edge_label=torch.empty(g.m, dtype=torch.int32, device=dev),
                         artic_bits=torch.empty((g.n + 31) // 32, dtype=torch.int32, device=dev),
                         bcc_count=torch.empty(1, dtype=torch.int64, device=dev)) for g in graphs]
    launches = 0
    main_stream = torch.cuda.current_stream(dev)

    def step():
        nl = 0
        ev = torch.cuda.Event()
        ev.record(main_stream)
        for st in streams:
            st.wait_event(ev)
        for i, g in enumerate(graphs):
            k = i % S
            with torch.cuda.stream(streams[k]):
                nl += pg.bcc_device(g.offsets, g.targets, out=outs[i], workspace=wss[k]).launches
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            main_stream.wait_event(e)
        return nl

    for _ in range(args.warmup):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        launches += step()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    total_ms = e0.elapsed_time(e1)
    mu = sum(g.m // 2 for g in graphs) * args.steps
    total_ms, edges = reduce_over_ranks(total_ms, mu, dev)
    # per-instance canonical checksums of the outputs the LAST TIMED step wrote (
    # canonicalised after the timing), and on rank 0 the first --verify instances re-run by
    # the C oracle on the host threads
    sums = []
    for i, g in enumerate(graphs):
        canon = pg.canonicalize_device(g.offsets, g.targets, outs[i].edge_label, label_bound=max(g.n, 1))
        sums.append(pg.canonical_checksum_device(canon, outs[i].artic_bits, outs[i].bcc_count))
        del canon
    verified = None
    if rank == 0 and args.verify > 0:
        verified = verify_instances([graphs[i] for i in range(min(args.verify, len(graphs)))],
                                    sums[:args.verify])
    if rank == 0:
        line = {
            "metric": METRIC, "value": edges / (total_ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"c5b: batch of {args.instances} grid 4096x4096 p=0.6 instances, seeds 1..{args.instances}",
                       "streams_per_gpu": S,
                       "instances_per_s": args.instances * args.steps / (total_ms / 1e3),
                       "l2": "inputs larger than L2 (batch of 64 x 295 MB CSR)"},
            "gpu_launches": launches, "clocks": clocks,
            "checksums": {"instances": [mine[i] + 1 for i in range(len(sums))],
                          "bcc_count_art_hash": [list(map(str, c)) for c in sums],
                          "of": "the outputs of the last timed concurrent step (one output buffer per instance)",
                          "rule": "(bcc_count, articulation points, sum canon[s]*(((s*0x9E3779B1) mod 2^32)|1) mod 2^64)"},
            "verified": verified,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def verify_instances(graphs, sums):
    """Re-run the first instances with the C oracle (one host thread each) and compare the
    canonical checksums (per-instance checksums against the oracle)."""
    import numpy as np

    import oracle
    import paper_2404_17101_b200 as pg

    oracle.build()
    host = [(g.offsets.cpu().numpy(), g.targets.cpu().numpy().view(np.uint32)) for g in graphs]
    got = [None] * len(host)

    def work(i):
        off, tgt = host[i]
        r = oracle.bcc_hopcroft_tarjan(off, tgt)
        canon = oracle.canonical_min_eid(off, tgt, r.edge_label)
        got[i] = pg.canonical_checksum(canon, r.articulation, r.bcc_count)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(host))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return {"instances": len(host), "match": all(a == tuple(b) for a, b in zip(got, sums)),
            "host_threads": len(host), "seconds": round(time.perf_counter() - t0, 1),
            "checker": "oracle/bcc_oracle.c (C restatement of bcc_hopcroft_tarjan) + canonical_min_eid"}


def run_e2e(args, off_h, tgt_h, dev, n, m, participate=True, k=1, world=1):
    """The same metric through pg.bcc(g): H2D of the CSR from pinned host memory, device
    validation (the reference's is_symmetric), FAST-BCC, D2H of labels + articulation bytes
    + count into pinned host buffers -- all inside the timed region, one call at a time.
    Also reported (not the headline): the same steps through pg.BccPipeline, which overlaps
    one graph's H2D with the previous graph's D2H and BCC.
    With N ranks, ranks 0..k-1 (k from e2e_ranks) run each leg concurrently between
    barriers; the value is their summed edges over the slowest participant's time."""
    import torch
    import torch.distributed as dist

    import paper_2404_17101_b200 as pg

    steps = max(1, min(args.steps, args.e2e_steps))
    h2d = 8 * (n + 1) + 4 * m
    d2h = 4 * m + n + 8
    dt = h2d_s = val_s = 0.0
    if participate:
        g = pg.Graph(off_h.numpy(), tgt_h.numpy())
        hb = pg.HostBuffers.allocate(n, m)
        res = pg.bcc(g, device=dev, host_out=hb)         # warm-up
        torch.cuda.synchronize()
        # split-out components (diagnostic only): H2D copy and device validation alone
        t0 = time.perf_counter()
        off_d = off_h.to(dev, non_blocking=True)
        tgt_d = tgt_h.to(dev, non_blocking=True)
        torch.cuda.synchronize()
        h2d_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        pg.validate_device(off_d, tgt_d)
        val_s = time.perf_counter() - t0
        del off_d, tgt_d
    _sync()
    if participate:
        t0 = time.perf_counter()
        for _ in range(steps):
            res = pg.bcc(g, device=dev, host_out=hb)
        dt = (time.perf_counter() - t0) / steps
        del res, hb
    _sync()
    edges, = _allreduce([(m // 2) if participate else 0], dist.ReduceOp.SUM, dev) if world > 1 else [m // 2]
    dt, = _allreduce([dt], dist.ReduceOp.MAX, dev) if world > 1 else [dt]
    out = {"value": edges / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": dt * 1e3, "steps": steps,
           "h2d_ms": round(h2d_s * 1e3, 1), "validate_ms": round(val_s * 1e3, 1),
           "path": "paper_2404_17101_b200.bcc(g) with host numpy CSR (pinned) -> H2D, validate, FAST-BCC, "
                   "D2H labels+articulation bytes+count (pinned)"}
    if world > 1:
        out["ranks"] = k
        out["bytes_per_step_note"] = "h2d/d2h bytes are per participating rank"
    # vertex mode: the same call returning the reference's O(n) parallel-mode BccLabels
    # (comp/parent/first, results.py:49-52): no per-slot labelling pass, 13 B/vertex back
    vdt = 0.0
    if participate:
        hbv = pg.HostBuffers.allocate(n, m, edge_labels=False)
        res = pg.bcc(g, device=dev, host_out=hbv, edge_labels=False)     # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            res = pg.bcc(g, device=dev, host_out=hbv, edge_labels=False)
        vdt = (time.perf_counter() - t0) / steps
        del res, hbv
    _sync()
    vdt, = _allreduce([vdt], dist.ReduceOp.MAX, dev) if world > 1 else [vdt]
    out["vertex_mode"] = {"value": edges / vdt, "unit": UNIT, "ms_per_step": vdt * 1e3, "steps": steps,
                          "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 13 * n + 8,
                          "path": "paper_2404_17101_b200.bcc(g, edge_labels=False): H2D, validate, FAST-BCC "
                                  "without the per-slot pass, D2H articulation bytes + comp/parent/first + count "
                                  "(the reference's O(n) BccLabels mode, results.py:49-52)"}
    # pipelined: the same per-step copies and work, consecutive steps overlapped
    pg.release_workspace()
    torch.cuda.empty_cache()
    need = 2 * (4 * m + n + 8)                          # two pinned output slots per rank
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = None
    ok = avail is None or avail >= 1.5 * k * need      # k participants on this node
    if world > 1:
        ok = _allreduce([1.0 if ok else 0.0], dist.ReduceOp.MIN, dev)[0] > 0
    if not ok:
        out["pipelined"] = {"unavailable": f"host memory: {k} ranks x {need / 1e9:.1f} GB of pinned output "
                                           f"slots exceed 2/3 of the {(avail or 0) / 1e9:.0f} GB available"}
        return out
    psteps = max(6, steps + 1)
    pdt, oom = 0.0, 0.0
    pipe = None
    if participate:
        try:
            pipe = pg.BccPipeline(device=dev)
            for _ in pipe.run([g, g]):                     # warm-up: rings and workspaces
                pass
            torch.cuda.synchronize()
        except torch.cuda.OutOfMemoryError:
            oom, pipe = 1.0, None
    if world > 1:
        oom = _allreduce([oom], dist.ReduceOp.MAX, dev)[0]
    if oom:
        del pipe
        pg.release_workspace()
        torch.cuda.empty_cache()
        out["pipelined"] = {"unavailable": "out of device memory for two graphs in flight"}
        return out
    _sync()
    if participate:
        t0 = time.perf_counter()
        for _ in pipe.run([g] * psteps):
            pass
        pdt = (time.perf_counter() - t0) / psteps
    _sync()
    if world > 1:
        pdt = _allreduce([pdt], dist.ReduceOp.MAX, dev)[0]
    out["pipelined"] = {"value": edges / pdt, "unit": UNIT, "ms_per_step": pdt * 1e3, "steps": psteps,
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "path": "paper_2404_17101_b200.BccPipeline.run(graphs): H2D of step i+1 overlaps "
                                "BCC + D2H of step i (two-slot device rings, three streams); "
                                "fill and drain included"}
    del pipe
    pg.release_workspace()
    torch.cuda.empty_cache()
    return out


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 with the same arguments; rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """The launch path without a GPU (gloo): every rank reports the replica seed and the
    c5b instances it would run; rank 0 prints them.  Used by tests/test_replicas.py."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    import paper_2404_17101_b200.graph as gmod

    seed = gmod.CONFIGS[args.config]["seed"] + rank if args.config in gmod.CONFIGS else 1 + rank
    mine = assign_instances(args.instances, rank, world)
    rec = torch.tensor([rank, seed, len(mine), sum(mine)], dtype=torch.int64)
    allr = [torch.zeros_like(rec) for _ in range(world)]
    if world > 1:
        dist.all_gather(allr, rec)
    else:
        allr = [rec]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "gpus_arg": args.gpus,
                          "ranks": [r.tolist() for r in allr], "config": args.config}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5a", choices=["c1", "c2", "c3", "c4", "c5a", "c5b"])
    ap.add_argument("--instances", type=int, default=64, help="c5b: batch size (grid instances)")
    ap.add_argument("--streams", type=int, default=4, help="c5b: concurrent instances per GPU")
    ap.add_argument("--verify", type=int, default=8, help="c5b: instances re-checked by the C oracle on rank 0")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0, help="sampling seed of the BCC call")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-checksum", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launch path only (gloo, no GPU)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return run_dry(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.config == "c5b":
        return run_batch(args, rank, world, local)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
