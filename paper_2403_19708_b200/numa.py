"""Host memory on a chosen NUMA node (one process per GPU,
each with its pinned KV arena on its own GPU's NUMA node, so the pre-loader's
H2D DMAs never cross the socket interconnect).

The arena is an anonymous mapping given the node as its preferred node with
mbind(MPOL_PREFERRED) before any page is touched; page-locking it with
cudaHostRegister then faults every page in on that node (falling back to
another node only if that one is full -- MPOL_BIND would have the kernel
kill the process instead) and makes it DMA-able like cudaHostAlloc memory.
No libnuma is needed (raw syscall through libc)."""

from __future__ import annotations

import ctypes
import mmap
import os
import platform

_MPOL_PREFERRED = 1
_SYS_MBIND = {"x86_64": 237, "aarch64": 235}


def node_count() -> int:
    try:
        return sum(1 for d in os.listdir("/sys/devices/system/node")
                   if d.startswith("node") and d[4:].isdigit())
    except OSError:
        return 1


def gpu_numa_node(device_index: int) -> int | None:
    """NUMA node of a CUDA device from its PCI address (sysfs), None if the
    platform does not report one (single-node hosts report -1)."""
    import torch

    p = torch.cuda.get_device_properties(device_index)
    bus = "%04x:%02x:%02x.0" % (getattr(p, "pci_domain_id", 0), p.pci_bus_id, p.pci_device_id)
    try:
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
    except (OSError, ValueError):
        return None
    return node if node >= 0 else None


def _mbind(addr: int, length: int, node: int) -> None:
    nr = _SYS_MBIND.get(platform.machine())
    if nr is None:
        raise OSError(f"mbind: unsupported machine {platform.machine()}")
    maxnode = max(64, node + 1)
    mask = (ctypes.c_ulong * (maxnode // 64 + 1))()
    mask[node // 64] = 1 << (node % 64)
    libc = ctypes.CDLL(None, use_errno=True)
    libc.syscall.restype = ctypes.c_long
    rc = libc.syscall(ctypes.c_long(nr), ctypes.c_void_p(addr), ctypes.c_ulong(length),
                      ctypes.c_int(_MPOL_PREFERRED), mask, ctypes.c_ulong(maxnode + 1),
                      ctypes.c_uint(0))
    if rc != 0:
        e = ctypes.get_errno()
        raise OSError(e, f"mbind(node {node}): {os.strerror(e)}")


class _Region:
    """An mbind'ed anonymous mapping, registered with CUDA while alive: the
    registration is dropped before the mapping goes (a later mapping at the
    same address could not be registered otherwise)."""

    def __init__(self, nbytes: int, node: int, pin: bool):
        import torch

        self.mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        self.addr = ctypes.addressof(ctypes.c_char.from_buffer(self.mm))
        self.registered = False
        _mbind(self.addr, nbytes, node)
        if pin:
            err = torch.cuda.cudart().cudaHostRegister(self.addr, nbytes, 0)
            if int(err) != 0:
                raise RuntimeError(f"cudaHostRegister of {nbytes} B failed: {err}")
            self.registered = True

    def __del__(self):
        if self.registered:
            try:
                import torch

                torch.cuda.synchronize()
                torch.cuda.cudart().cudaHostUnregister(self.addr)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass
            self.registered = False


def host_buffer(nbytes: int, node: int, *, pin: bool = True):
    """(uint8 tensor of `nbytes` on NUMA node `node`, node).  pin=True
    page-locks and registers it with CUDA (cudaHostRegister); the
    registration lives as long as the returned tensor object (keep it, e.g.
    as HostArena.buffer, for as long as views of it are in use)."""
    import torch

    if node < 0 or node >= max(1, node_count()):
        raise ValueError(f"no NUMA node {node} (host has {node_count()})")
    region = _Region(nbytes, node, pin)
    buf = torch.frombuffer(region.mm, dtype=torch.uint8)
    buf._askv_region = region
    return buf, node
