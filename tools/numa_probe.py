"""Host-link probe (tools only): the GPU's NUMA node and local CPUs, and the
pinned H2D / D2H rate with the pinned buffer first touched from CPUs local
to the GPU vs from the other socket's CPUs."""
import os
import sys

import torch


def pci_info(dev=0):
    import subprocess
    bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i",
                          str(dev)], capture_output=True, text=True).stdout.strip().lower()
    tail = bus.split(":", 1)[1] if bus.count(":") == 2 else bus  # drop the domain
    cands = [p for p in os.listdir("/sys/bus/pci/devices") if p.lower().endswith(tail)]
    path = "/sys/bus/pci/devices/" + cands[0] if cands else None
    node = open(path + "/numa_node").read().strip() if path else "?"
    cpus = open(path + "/local_cpulist").read().strip() if path else "?"
    return bus, path, node, cpus


def parse_list(s):
    out = set()
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def rate(n_bytes=1 << 30, reps=3):
    h = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)  # touch from the current affinity
    d = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    best_up = best_dn = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best_up = max(best_up, n_bytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        e0.record()
        h.copy_(d, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best_dn = max(best_dn, n_bytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best_up, best_dn


def main():
    torch.cuda.init()
    bus, path, node, cpus = pci_info(0)
    allc = os.sched_getaffinity(0)
    print(f"gpu0 bus {bus} numa_node {node} local_cpus {cpus}; process affinity {len(allc)} cpus")
    try:
        nodes = sorted(os.listdir("/sys/devices/system/node"))
        for nd in nodes:
            if nd.startswith("node"):
                print(nd, open(f"/sys/devices/system/node/{nd}/cpulist").read().strip())
    except OSError:
        pass
    print("default affinity:", rate())
    local = parse_list(cpus) & allc if cpus != "?" else set()
    remote = allc - local
    if local:
        os.sched_setaffinity(0, local)
        print("local cpus:", rate())
    if remote:
        os.sched_setaffinity(0, remote)
        print("remote cpus:", rate())
    os.sched_setaffinity(0, allc)


if __name__ == "__main__":
    main()
