"""Host NUMA placement for per-GPU replicas.

A replica's expert fetches read its pinned host mirror over PCIe; when the
mirror's pages sit on the other socket every byte also crosses the socket
link. This module finds the NUMA node of a GPU (its PCI device's
``numa_node`` in sysfs) and the CPUs of a node, so a rank can bind itself to
its GPU's node and the first writer of a node-shared mirror places the pages
there (Linux first-touch). Missing sysfs entries (containers, single-socket
hosts) read as node -1 / "no binding"; nothing here is needed for
correctness.
"""

from __future__ import annotations

import os


def _parse_cpulist(text: str) -> set:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        else:
            cpus.add(int(part))
    return cpus


def node_cpus(node: int) -> set:
    """CPUs of NUMA node ``node`` (empty when unknown)."""
    if node < 0:
        return set()
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            return _parse_cpulist(f.read())
    except OSError:
        return set()


def num_nodes() -> int:
    try:
        return len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit()])
    except OSError:
        return 1


def gpu_pci_bus_id(index: int) -> str | None:
    """PCI address of CUDA device ``index`` (as torch numbers it, i.e. after
    CUDA_VISIBLE_DEVICES) in sysfs form dddd:bb:dd.0."""
    try:
        import torch
        p = torch.cuda.get_device_properties(index)
        return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:
        return None


def gpu_numa_node(index: int) -> int:
    """NUMA node of CUDA device ``index`` (-1 when unknown)."""
    bus = gpu_pci_bus_id(index)
    if bus is None:
        return -1
    try:
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            return int(f.read().strip())
    except (OSError, ValueError):
        return -1


def bind_to_node(node: int) -> bool:
    """Restrict this process to the CPUs of ``node`` it may use; False if nothing changed."""
    cpus = node_cpus(node) & set(os.sched_getaffinity(0))
    if not cpus:
        return False
    os.sched_setaffinity(0, cpus)
    return True
