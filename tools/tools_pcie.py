"""Diagnostic: pinned host <-> device copy times by size (CUDA events)."""
import torch

n = 90000
res = {}
for label, elems in [("q 0.72MB", n), ("pos 2.16MB", 3 * n), ("pos+q 2.88MB", 4 * n),
                     ("F 2.16MB d2h", -3 * n)]:
    e = abs(elems)
    h = torch.zeros(e, dtype=torch.float64).pin_memory()
    d = torch.zeros(e, dtype=torch.float64, device="cuda")
    fn = (lambda: h.copy_(d, non_blocking=True)) if elems < 0 else \
         (lambda: d.copy_(h, non_blocking=True))
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{label}: median {ts[15]:.1f} us  min {ts[0]:.1f} us  "
          f"({e * 8 / ts[15] / 1e3:.1f} GB/s)")
