"""CPU: the multi-GPU plumbing of bench.py (replicas only -- BCC of one graph does not
shard) on a world-size-2 gloo group: instance dealing for config 5b
and the max-time / summed-work reduction the whole-job value is built from."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    mine = bench.assign_instances(64, rank, world)
    t, e = bench.reduce_over_ranks(10.0 + 5 * rank, 1000 * (rank + 1), "cpu")
    q.put((rank, mine, t, e))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_reduction_and_dealing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    (r0, m0, t0, e0), (r1, m1, t1, e1) = res
    assert sorted(m0 + m1) == list(range(64)) and not set(m0) & set(m1)
    assert len(m0) == len(m1) == 32
    assert t0 == t1 == 15.0           # max over ranks
    assert e0 == e1 == 3000.0         # whole-job work


def test_single_process_passthrough():
    import bench

    assert bench.reduce_over_ranks(7.5, 42, "cpu") == (7.5, 42.0)
    assert bench.assign_instances(5, 0, 1) == [0, 1, 2, 3, 4]


def _e2e_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    small = bench.e2e_ranks(1000, 10000, world, "cpu")            # fits: every rank runs the e2e legs
    huge = bench.e2e_ranks(1 << 40, 1 << 44, world, "cpu")        # does not fit anywhere
    mx = bench._allreduce([rank + 1.0, -rank], dist.ReduceOp.MAX, "cpu")
    q.put((rank, small, huge, mx))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_e2e_participants_agree_across_ranks():
    """bench.py's e2e legs at N ranks: the number of concurrently participating ranks is
    bounded by host memory (pinned CSR + outputs per rank) and identical on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_e2e_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
    assert [r[1] for r in res] == [2, 2]
    assert [r[2] for r in res] == [0, 0]
    assert res[0][3] == res[1][3] == [2.0, 0.0]


def _bench_json(args, env_extra=None):
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), *args], capture_output=True, text=True,
                       env=env, timeout=150)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.timeout(180)
def test_bench_gpus_2_spawns_two_ranks():
    """`python bench.py --gpus 2` outside torchrun launches two ranks itself (the driver's
    command form); each rank gets its own replica seed and its own c5b instances."""
    d = _bench_json(["--gpus", "2", "--dry-run"])
    assert d["n_gpus"] == 2 and d["gpus_arg"] == 2
    seeds = [r[1] for r in d["ranks"]]
    assert sorted(r[0] for r in d["ranks"]) == [0, 1] and len(set(seeds)) == 2
    d = _bench_json(["--gpus", "2", "--dry-run", "--config", "c5b"])
    assert sum(r[2] for r in d["ranks"]) == 64 and sum(r[3] for r in d["ranks"]) == sum(range(64))


def test_bench_rejects_world_mismatch():
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
