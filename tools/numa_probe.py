"""Host NUMA placement vs device->host copy bandwidth (measurement scaffolding):
the GPU's NUMA node, then D2H / H2D GB/s into 4 GiB of pinned memory
allocated while the process runs on each node's CPUs (first-touch placement)."""
import glob
import os
import time

import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


props = torch.cuda.get_device_properties(0)
bus = getattr(props, "pci_bus_id", None)
print("device", props.name, "pci", bus)
gpu_node = None
for d in glob.glob("/sys/bus/pci/devices/*"):
    try:
        if bus is not None and os.path.basename(d).lower().endswith(f"{bus:02x}:00.0"):
            gpu_node = int(open(d + "/numa_node").read())
    except OSError:
        pass
nodes = {}
for nd in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
    nodes[int(nd.rsplit("node", 1)[1])] = cpulist(open(nd + "/cpulist").read())
print("gpu numa node", gpu_node, "nodes", {k: (v[0], v[-1], len(v)) for k, v in nodes.items()})
print("process affinity", len(os.sched_getaffinity(0)), "cpus")
n = 4 << 30
src = torch.empty(n, dtype=torch.uint8, device="cuda")
full = os.sched_getaffinity(0)
for node, cpus in list(nodes.items()) + [(-1, sorted(full))]:
    cpus = [c for c in cpus if c in full]
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst[::4096] = 1  # touch (first-touch placement if not already placed)
    res = []
    for direction in ("d2h", "h2d"):
        best = 0
        for rep in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            if direction == "d2h":
                dst.copy_(src, non_blocking=True)
            else:
                src.copy_(dst, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, n / (time.perf_counter() - t) / 1e9)
        res.append(f"{direction} {best:.1f} GB/s")
    print(f"alloc on node {node} ({len(cpus)} cpus):", ", ".join(res), flush=True)
    del dst
os.sched_setaffinity(0, full)
