"""Diagnostic: H2D from library-allocated page-locked memory, untouched vs
written by the CPU (numpy / torch)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import _lib  # noqa: E402

L = _lib.lib()
n = 360000
dev = torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()


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


b1 = _lib.HostBuffer((n,))
print("untouched         ", t(b1.tensor))
b1.tensor.zero_()
print("after torch zero_ ", t(b1.tensor))
b2 = _lib.HostBuffer((n,))
b2.tensor.numpy()[:] = np.random.default_rng(0).normal(size=n)
print("after numpy write ", t(b2.tensor))
b3 = _lib.HostBuffer((n,))
b3.tensor.copy_(torch.ones(n, dtype=torch.float64))
print("after torch copy_ ", t(b3.tensor))
print("again b1          ", t(b1.tensor))
print("threads", torch.get_num_threads())
