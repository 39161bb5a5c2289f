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


def test_affinity_sysfs_parsing_and_binding(tmp_path, monkeypatch):
    """affinity.bind_to_gpu: the GPU's local CPUs come from sysfs
    (numa_node, local_cpulist) and the process is restricted to them when
    they are a proper subset of what it may use."""
    from paper_2411_03357_b200 import affinity

    assert affinity.parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert affinity._fmt([0, 1, 2, 3, 8, 10, 11]) == "0-3,8,10-11"
    allowed = sorted(os.sched_getaffinity(0))
    dev = tmp_path / "0000:1b:00.0"
    dev.mkdir()
    (dev / "numa_node").write_text("1\n")
    local = allowed[: max(1, len(allowed) // 2)]
    (dev / "local_cpulist").write_text(affinity._fmt(local) + "\n")
    info = affinity.gpu_locality("0000:1b:00.0", str(tmp_path))
    assert info["numa_node"] == 1 and info["cpus"] == local
    monkeypatch.setattr(affinity, "pci_bus_id", lambda d: "0000:1b:00.0")
    try:
        got = affinity.bind_to_gpu(0, str(tmp_path))
        if len(allowed) > 1:
            assert got["bound"] and sorted(os.sched_getaffinity(0)) == local
        else:
            assert not got["bound"]
    finally:
        os.sched_setaffinity(0, allowed)
    assert affinity.bind_to_gpu(0, str(tmp_path / "missing"))["bound"] is False


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_two_ranks_same_device_gpu():
    """The bench's multi-rank flow on a 1-GPU box: torchrun, 2 ranks on
    cuda:0 (gloo for the barrier / max-over-ranks), each with its own
    channel and traces through the offload and KV legs (--quick)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--same-device", "--dist-backend", "gloo", "--quick", "--no-cpu-baseline", "--steps", "3"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 prints, once
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["offload"]["n_gpus"] == 2 and d["offload"]["tokens_per_s_ratio"] > 0
    assert d["workloads"]["kv_swap_opt30b"]["swap_only"]["arms"]["specpipe"]["gbs"] > 0
    assert "host_placement" in d["config"]
