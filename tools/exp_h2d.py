"""Pinned host <-> HBM copy bandwidth vs the process's CPU placement (experiment).

    python tools/exp_h2d.py [GB]

Prints the GPU's PCI NUMA node, the process affinity, and H2D / D2H GB/s of
a pinned buffer allocated (first-touched) before and after binding the
process to the GPU-local cores that NVML reports.
"""
import json
import os
import sys
import time

import torch


def bw(host, dev, reps=3):
    out = {}
    for name, (dst, src) in {"h2d": (dev, host), "d2h": (host, dev)}.items():
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, host.numel() / (time.perf_counter() - t0) / 1e9)
        out[name] = round(best, 2)
    return out


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
    n = int(gb * 1e9)
    torch.cuda.set_device(0)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    info = {"affinity_before": len(os.sched_getaffinity(0))}
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        node_path = f"/sys/bus/pci/devices/{bus.lower()[4:] if len(bus) > 12 else bus.lower()}/numa_node"
        info["pci"] = bus
        if os.path.exists(node_path):
            info["gpu_numa_node"] = open(node_path).read().strip()
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = [w * 64 + b for w, word in enumerate(words) for b in range(64) if word >> b & 1]
        info["gpu_local_cpus"] = len(cpus)
    except Exception as e:  # noqa: BLE001
        info["nvml_error"] = repr(e)
        cpus = []
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host.fill_(1)
    info["unbound"] = bw(host, dev)
    del host
    if cpus:
        os.sched_setaffinity(0, cpus)
        host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        host.fill_(1)
        info["bound"] = bw(host, dev)
    print(json.dumps(info))


if __name__ == "__main__":
    main()
