"""Probe the GPU box's host: cores, RAM, pinned-allocation cost and PCIe
H2D bandwidth for the miss path (256 KiB rows from a pinned host dataset)."""
import json
import os
import subprocess
import time

import torch

out = {"nproc": os.cpu_count()}
try:
    out["lscpu"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                    if l.split(":")[0].strip() in ("Model name", "Socket(s)", "Core(s) per socket",
                                                   "Thread(s) per core", "NUMA node(s)", "CPU(s)")]
except Exception as e:  # noqa: BLE001
    out["lscpu"] = str(e)
out["meminfo"] = [l for l in open("/proc/meminfo").read().splitlines()[:3]]
out["shm"] = subprocess.run(["df", "-h", "/dev/shm", "/tmp"], capture_output=True, text=True).stdout
try:
    out["affinity"] = len(os.sched_getaffinity(0))
except Exception:  # noqa: BLE001
    pass
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
for gib in (8, 64):
    t0 = time.time()
    h = torch.empty(gib << 30, dtype=torch.uint8, pin_memory=True)
    out[f"pin_alloc_{gib}gib_s"] = time.time() - t0
    d = torch.empty(8 << 30, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            d.copy_(h[: 8 << 30], non_blocking=True)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        d.copy_(h[: 8 << 30], non_blocking=True)
        e1.record(s)
        s.synchronize()
        out[f"h2d_8gib_GBps_from_{gib}gib"] = (8 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9
        # 256 KiB rows, scattered sources
        rows = 4096
        SB = 262144
        import random
        ids = [random.randrange((gib << 30) // SB) for _ in range(rows)]
        e0.record(s)
        for i, r in enumerate(ids):
            d[i * SB:(i + 1) * SB].copy_(h[r * SB:(r + 1) * SB], non_blocking=True)
        e1.record(s)
        s.synchronize()
        out[f"h2d_rows256k_GBps_{gib}"] = rows * SB / (e0.elapsed_time(e1) * 1e-3) / 1e9
        e0.record(s)
        d[: 8 << 30].copy_(d[: 8 << 30].flip(0)[:0].new_empty(0)) if False else None
        # D2H
        e0.record(s)
        h[: 8 << 30].copy_(d, non_blocking=True)
        e1.record(s)
        s.synchronize()
        out[f"d2h_8gib_GBps_{gib}"] = (8 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9
    del h, d
    torch.cuda.empty_cache()
out["free_mem_gpu"] = torch.cuda.mem_get_info()
print(json.dumps(out, indent=1))
