"""Diagnostic: where the e2e time goes (graph replays, CUDA events)."""
import os
import sys

import torch
from threadpoolctl import threadpool_limits
threadpool_limits(1)
torch.set_num_threads(1)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads  # noqa: E402

w, pos_np, q_np = workloads.generate(1)
solver = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                           cell_type=w.cell_type), capacity=w.n)
hs = solver.host_stepper(w.n, True)
hs.positions.copy_(torch.as_tensor(pos_np))
hs.charges.copy_(torch.as_tensor(q_np))
pos = torch.as_tensor(pos_np, device="cuda")
q = torch.as_tensor(q_np, device="cuda")
g, out7, F = solver.graphed(pos, q, True)
# copies only
cg = torch.cuda.CUDAGraph()
dpos, dq = torch.empty_like(pos), torch.empty_like(q)
hF = torch.empty((w.n, 3), dtype=torch.float64).pin_memory()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2):
        dpos.copy_(hs.positions, non_blocking=True)
        dq.copy_(hs.charges, non_blocking=True)
        hF.copy_(F, non_blocking=True)
torch.cuda.synchronize()
with torch.cuda.graph(cg):
    dpos.copy_(hs.positions, non_blocking=True)
    dq.copy_(hs.charges, non_blocking=True)
    hF.copy_(F, non_blocking=True)


def t(fn, k=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3


import time
time.sleep(0.5)
print("device step graph  us", round(t(g.replay), 1))
print("host_stepper graph us", round(t(hs.launch), 1))
print("copies-only graph  us", round(t(cg.replay), 1))

import ctypes as C  # noqa: E402

from paper_2601_00161_b200 import _lib  # noqa: E402

L = _lib.lib()


def cp(dst, src):
    L.esp_copy_async(C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()),
                     src.numel() * src.element_size(),
                     C.c_void_p(torch.cuda.current_stream().cuda_stream))


def ours():
    cp(dpos, hs.positions)
    cp(dq, hs.charges)
    cp(hs.forces, F)


print("esp copies eager   us", round(t(ours), 1))
og = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    ours()
torch.cuda.synchronize()
with torch.cuda.graph(og):
    ours()
print("esp copies graph   us", round(t(og.replay), 1))
print("h2d pos only eager us", round(t(lambda: cp(dpos, hs.positions)), 1))
print("d2h F only eager   us", round(t(lambda: cp(hs.forces, F)), 1))
