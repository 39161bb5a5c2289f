"""N>1 host logic on CPU (gloo, world_size 2): every rank runs its own
independent channel (no data-path collective) and the timing is the max over
ranks, exactly as bench.py does under torchrun with NCCL."""
from __future__ import annotations

import os
import socket

import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import bench
    from paper_2411_03357_b200 import workload
    from paper_2411_03357_b200.replay import ReplayConfig, run_engine

    dist = bench.init_dist(world, "gloo")
    # each rank: its own channel seed and its own trace, dry data plane
    tr = workload.gen_offload_trace(4, [1, 2, 3, 4], 2, layer_bytes=4096, seed=rank)
    res = run_engine(tr, ReplayConfig(seed=rank, plane="dry"))
    nat = run_engine(tr, ReplayConfig(seed=rank, plane="dry", native_dispatch="python"))  # per-event calls
    assert nat.engine.report() == res.engine.report()
    key = res.engine.cpu.key.key_bytes
    local = float(10 + rank)
    bench.barrier(dist)
    mx = bench.reduce_max(dist, local)
    out.put((rank, mx, key.hex(), res.engine.report()["data_msgs"]))
    dist.destroy_process_group()


def test_two_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    assert all(mx == 11.0 for _, mx, _, _ in got)       # max over ranks
    assert got[0][2] != got[1][2]                         # independent channel keys
    assert all(n > 0 for *_, n in got)
