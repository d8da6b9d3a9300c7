"""H2D / D2H bandwidth of pinned host buffers allocated from each NUMA node's cores (first-touch
placement), vs the GPU's own NUMA node (/sys/bus/pci/devices/<bus id>/numa_node)."""
import glob
import os
import subprocess

import numpy as np
import torch

print(subprocess.run(["bash", "-c", "lscpu | grep -i 'numa\\|^CPU(s)\\|Model name'; nvidia-smi topo -m | head -4"],
                     capture_output=True, text=True).stdout)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
props = torch.cuda.get_device_properties(0)
busid = "%04x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
for f in glob.glob(f"/sys/bus/pci/devices/{busid.lower()}/numa_node"):
    print("GPU", busid, "numa_node", open(f).read().strip())
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
all_cpus = os.sched_getaffinity(0)


def cpus_of(node):
    s = open(f"{node}/cpulist").read().strip()
    out = set()
    for part in s.split(","):
        a, _, b = part.partition("-")
        out |= set(range(int(a), int(b or a) + 1))
    return out & all_cpus


d = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")


def tm(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for node in nodes:
    c = cpus_of(node)
    if not c:
        continue
    os.sched_setaffinity(0, c)
    h = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    os.sched_setaffinity(0, all_cpus)
    gbs_in = (16 << 20) / tm(lambda: d.copy_(h, non_blocking=True)) / 1e6
    gbs_out = (16 << 20) / tm(lambda: h.copy_(d, non_blocking=True)) / 1e6
    print(f"{os.path.basename(node)} ({len(c)} cpus): H2D {gbs_in:.1f} GB/s  D2H {gbs_out:.1f} GB/s")
