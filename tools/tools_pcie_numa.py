"""Diagnostic: pinned copy bandwidth with and without binding the process to
the GPU's NUMA-local CPUs (NVML ideal affinity), and the topology."""
import os
import subprocess
import sys

mode = sys.argv[1] if len(sys.argv) > 1 else "none"
if mode == "bind":
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    pynvml.nvmlDeviceSetCpuAffinity(hd)
print("mode", mode, "cpus", len(os.sched_getaffinity(0)), sorted(os.sched_getaffinity(0))[:4])
import torch  # noqa: E402

n = 90000
for label, elems in [("pos+q 2.88MB h2d", 4 * n), ("F 2.16MB d2h", -3 * n)]:
    e = abs(elems)
    h = torch.zeros(e, dtype=torch.float64).pin_memory()
    d = torch.zeros(e, dtype=torch.float64, device="cuda")
    fn = (lambda: h.copy_(d, non_blocking=True)) if elems < 0 else \
         (lambda: d.copy_(h, non_blocking=True))
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{label}: median {ts[25]:.1f} us ({e * 8 / ts[25] / 1e3:.1f} GB/s)")
