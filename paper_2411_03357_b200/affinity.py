"""Host placement for one process per GPU (shared host
resources — PCIe switches, pinned DRAM bandwidth, NUMA — are the multi-GPU
scaling risk, not GPU-GPU links).

`bind_to_gpu(i)` pins the calling process (and every thread it starts
later, including libsppipe's issuing thread, which inherits the mask) to
the CPUs local to GPU i's PCIe root, read from sysfs.  Pinned host memory
allocated afterwards (the swap slabs of memory.host_buffer, the staging
ring, cudaHostAlloc) is first touched on those CPUs, so the kernel's
default local-allocation policy places it on the GPU's NUMA node: each
rank's swaps cross only its own socket's memory controller and PCIe root.
"""
from __future__ import annotations

import os

SYSFS_PCI = "/sys/bus/pci/devices"


def parse_cpulist(text: str) -> set[int]:
    """'0-3,8,10-11' -> {0,1,2,3,8,10,11} (the sysfs cpulist format)."""
    out: set[int] = set()
    for part in text.strip().split(","):
        part = part.strip()
        if not part:
            continue
        if "-" in part:
            lo, hi = part.split("-", 1)
            out.update(range(int(lo), int(hi) + 1))
        else:
            out.add(int(part))
    return out


def pci_bus_id(device: int) -> str | None:
    """'0000:1b:00.0' for a torch CUDA device index (None without CUDA)."""
    try:
        import torch

        p = torch.cuda.get_device_properties(device)
        return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:  # noqa: BLE001 - no CUDA / older torch
        return None


def gpu_locality(bus_id: str, sysfs: str = SYSFS_PCI) -> dict:
    """NUMA node and local CPUs of a PCI device ({} when sysfs lacks them)."""
    base = os.path.join(sysfs, bus_id.lower())
    info: dict = {"pci_bus_id": bus_id}
    try:
        node = int(open(os.path.join(base, "numa_node")).read().strip())
        info["numa_node"] = node
    except (OSError, ValueError):
        pass
    try:
        info["cpus"] = sorted(parse_cpulist(open(os.path.join(base, "local_cpulist")).read()))
    except (OSError, ValueError):
        pass
    return info


def bind_to_gpu(device: int, sysfs: str = SYSFS_PCI) -> dict:
    """Restrict this process to GPU `device`'s local CPUs (intersected with
    the CPUs it may use); returns what was done, for the bench's config."""
    bus = pci_bus_id(device)
    if bus is None:
        return {"bound": False, "why": "no CUDA device"}
    info = gpu_locality(bus, sysfs)
    cpus = set(info.get("cpus", ()))
    try:
        allowed = os.sched_getaffinity(0)
    except AttributeError:  # pragma: no cover - non-Linux
        return {"bound": False, "why": "no sched_setaffinity", **info}
    use = cpus & allowed
    if not use or use == allowed:
        info.update(bound=False, why="GPU-local CPUs are all the allowed CPUs" if use else "no locality in sysfs")
        info["cpus"] = _fmt(sorted(allowed))
        return info
    os.sched_setaffinity(0, use)
    info.update(bound=True, cpus=_fmt(sorted(use)))
    return info


def _fmt(cpus: list[int]) -> str:
    """[0,1,2,3,8] -> '0-3,8'."""
    out, i = [], 0
    while i < len(cpus):
        j = i
        while j + 1 < len(cpus) and cpus[j + 1] == cpus[j] + 1:
            j += 1
        out.append(str(cpus[i]) if i == j else f"{cpus[i]}-{cpus[j]}")
        i = j + 1
    return ",".join(out)
