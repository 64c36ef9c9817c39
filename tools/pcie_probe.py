"""Host<->device copy bandwidth on this box (the bench's e2e leg is PCIe-bound).

    python tools/pcie_probe.py

Prints the GPU's PCI / NUMA placement and pinned-memory H2D, D2H and
simultaneous (both directions, two streams) bandwidth for 153.6 MB copies,
with the pinned buffers allocated (first-touched) by a thread bound to the
GPU's NUMA node and, for contrast, to the other node(s).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gpu_numa(dev=0):
    import torch
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    try:
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            return bus, int(f.read().strip())
    except OSError:
        return bus, -1


def node_cpus(node):
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
    except OSError:
        return None
    cpus = set()
    for part in spec.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def measure(torch, nbytes, reps=8):
    dev = torch.device("cuda", 0)
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_in.fill_(1)
    h_out.fill_(2)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    extra = []

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        for st in [s1, s2] + extra:
            torch.cuda.current_stream().wait_stream(st)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    s3, s4 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    extra += [s3, s4]
    half = nbytes // 2

    def h2d_split():  # the same upload as two halves on two streams (two DMA queues)
        with torch.cuda.stream(s1):
            d_a[:half].copy_(h_in[:half], non_blocking=True)
        with torch.cuda.stream(s3):
            d_a[half:].copy_(h_in[half:], non_blocking=True)

    def d2h_split():
        with torch.cuda.stream(s2):
            h_out[:half].copy_(d_b[:half], non_blocking=True)
        with torch.cuda.stream(s4):
            h_out[half:].copy_(d_b[half:], non_blocking=True)

    def both_split():
        h2d_split()
        d2h_split()

    res = {}
    for name, fn, mult in (("h2d", h2d, 1), ("d2h", d2h, 1), ("bidir", both, 2), ("h2d_2q", h2d_split, 1),
                           ("d2h_2q", d2h_split, 1), ("bidir_2q", both_split, 2)):
        ms = timed(fn)
        res[name + "_gbs"] = round(mult * nbytes / ms / 1e6, 1)
    return res


def main():
    import torch
    bus, node = gpu_numa()
    nodes = sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit()) \
        if os.path.isdir("/sys/devices/system/node") else []
    out = {"gpu_pci": bus, "gpu_numa_node": node, "numa_nodes": nodes, "cpus": os.cpu_count(),
           "affinity": len(os.sched_getaffinity(0))}
    nbytes = 153_600_000
    orig = os.sched_getaffinity(0)
    out["default"] = measure(torch, nbytes)
    for n in nodes:
        cpus = node_cpus(n)
        if not cpus or not (cpus & orig):
            continue
        os.sched_setaffinity(0, cpus & orig)
        out[f"bound_node{n}"] = measure(torch, nbytes)
        os.sched_setaffinity(0, orig)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
