"""Pinned D2H bandwidth vs the NUMA node the pinned pages live on.

The e2e leg (lf_assemble -> host CSR) is bounded by PCIe D2H; boxes measured
41-56 GB/s.  This probe places the pinned buffer on each NUMA node in turn
(thread affinity set to the node's CPUs before cudaHostAlloc, so first-touch
puts the pages there) and times a 4 GB D2H, best of 3.
    python tools/numa_d2h_probe.py
"""
import glob
import os
import time

import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_numa_node(dev=0):
    props = torch.cuda.get_device_properties(dev)
    bus = "%04x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
    path = f"/sys/bus/pci/devices/{bus}/numa_node"
    try:
        return bus, int(open(path).read())
    except OSError:
        return bus, None


def main():
    bus, node = gpu_numa_node()
    nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
    print(f"gpu {bus} numa_node={node}; nodes={[os.path.basename(n) for n in nodes]}; "
          f"affinity={len(os.sched_getaffinity(0))} cpus")
    n = (4 << 30) // 8
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    full = os.sched_getaffinity(0)
    cases = [("default", full)]
    for nd in nodes:
        cpus = set(cpulist(open(os.path.join(nd, "cpulist")).read())) & full
        if cpus:
            cases.append((os.path.basename(nd), cpus))
    for name, cpus in cases:
        os.sched_setaffinity(0, cpus)
        host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        host.zero_()
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            host.copy_(dev)
            torch.cuda.synchronize()
            best = max(best, n * 8 / (time.perf_counter() - t0) / 1e9)
        print(f"pinned pages on {name:8s} ({len(cpus)} cpus): D2H {best:.1f} GB/s")
        del host
        os.sched_setaffinity(0, full)


if __name__ == "__main__":
    main()
