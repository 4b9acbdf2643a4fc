"""NUMA placement of one rank: a GPU's PCIe function sits on one NUMA
node; the CPU thread that issues its I/O and the host tier its kernels read over that GPU's own link
belong on the same node, or every byte also crosses the socket interconnect.

Plumbing only (sysfs reads, sched_setaffinity, mbind): no part of the I/O path's arithmetic.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional

_SYS_MBIND = 237        # x86_64
_MPOL_BIND = 2


def gpu_bus_id(device: int) -> Optional[str]:
    """sysfs PCI address (dddd:bb:dd.0) of a CUDA device, or None."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:
        return None


def _sysfs(bus: Optional[str], leaf: str) -> Optional[str]:
    if not bus:
        return None
    try:
        with open(f"/sys/bus/pci/devices/{bus}/{leaf}") as f:
            return f.read().strip()
    except OSError:
        return None


def parse_cpulist(text: str) -> List[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11]."""
    out: List[int] = []
    for part in (text or "").split(","):
        part = part.strip()
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_numa_node(device: int) -> int:
    v = _sysfs(gpu_bus_id(device), "numa_node")
    try:
        return int(v) if v is not None else -1
    except ValueError:
        return -1


def gpu_local_cpus(device: int) -> List[int]:
    return parse_cpulist(_sysfs(gpu_bus_id(device), "local_cpulist") or "")


def bind_to_gpu(device: int) -> dict:
    """Pin this process to the CPUs local to `device` (intersected with those it may use).  Returns
    what was done, for the bench record."""
    node = gpu_numa_node(device)
    allowed = sorted(os.sched_getaffinity(0))
    local = [c for c in gpu_local_cpus(device) if c in set(allowed)]
    if local and len(local) < len(allowed):
        os.sched_setaffinity(0, local)
    return {"numa_node": node, "cpus": len(local) if local else len(allowed),
            "affinity": "gpu-local cpus" if local and len(local) < len(allowed) else "all (one node or unknown)"}


def mbind(addr: int, nbytes: int, node: int) -> bool:
    """Bind [addr, addr+nbytes) (page aligned) to NUMA node `node` before its pages are first touched;
    best effort (False when unsupported)."""
    if node < 0 or node >= 64 or nbytes <= 0:
        return False
    libc = ctypes.CDLL(None, use_errno=True)
    mask = ctypes.c_ulong(1 << node)
    rc = libc.syscall(ctypes.c_long(_SYS_MBIND), ctypes.c_void_p(addr), ctypes.c_ulong(nbytes),
                      ctypes.c_int(_MPOL_BIND), ctypes.byref(mask), ctypes.c_ulong(64), ctypes.c_uint(0))
    return rc == 0
