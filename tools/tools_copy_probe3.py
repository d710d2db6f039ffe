"""Diagnostic: H2D speed before / after building a KSpaceSolver and with a
host stepper alive."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, _lib, workloads  # noqa: E402

L = _lib.lib()
n = 360000
dev = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
buf = _lib.HostBuffer((n,))
buf.tensor.zero_()


def t(src, k=30):
    for _ in range(3):
        L.esp_copy_async(C.c_void_p(dev.data_ptr()), C.c_void_p(src.data_ptr()), n * 8,
                         C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(k):
        L.esp_copy_async(C.c_void_p(dev.data_ptr()), C.c_void_p(src.data_ptr()), n * 8,
                         C.c_void_p(s.cuda_stream))
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / k * 1e3, 1)


print("start               ", t(buf.tensor))
w, pos_np, q_np = workloads.generate(1)
print("after generate      ", t(buf.tensor))
solver = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                           cell_type=w.cell_type), capacity=w.n)
print("after solver        ", t(buf.tensor))
time.sleep(2)
print("after sleep 2s      ", t(buf.tensor))
pos = torch.as_tensor(pos_np, device="cuda")
q = torch.as_tensor(q_np, device="cuda")
g, out7, F = solver.graphed(pos, q, True)
print("after graph         ", t(buf.tensor))
for _ in range(20):
    g.replay()
torch.cuda.synchronize()
print("after replays       ", t(buf.tensor))
hs = solver.host_stepper(w.n, True)
print("after host_stepper  ", t(buf.tensor))
print("hs.positions        ", t(hs.positions.view(-1)[:n] if hs.positions.numel() >= n else buf.tensor))
