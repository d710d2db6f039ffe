"""Diagnostic: H2D/D2H copy time from torch-pinned vs cudaMallocHost memory."""
import ctypes as C
import glob
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import _lib  # noqa: E402

L = _lib.lib()
nb = 2880000
dev = torch.empty(nb // 8, dtype=torch.float64, device="cuda")
tp = torch.zeros(nb // 8, dtype=torch.float64).pin_memory()
print("torch pinned?", tp.is_pinned())
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime",
                               "lib", "libcudart.so*"))
rt = C.CDLL(cands[0])
hp = C.c_void_p()
print("cudaMallocHost", rt.cudaMallocHost(C.byref(hp), C.c_size_t(nb)))
s = torch.cuda.current_stream()


def t(dst, src, k=30):
    for _ in range(3):
        L.esp_copy_async(C.c_void_p(dst), C.c_void_p(src), nb, C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(k):
        L.esp_copy_async(C.c_void_p(dst), C.c_void_p(src), nb, C.c_void_p(s.cuda_stream))
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3


print("H2D torch-pinned  us", round(t(dev.data_ptr(), tp.data_ptr()), 1))
print("H2D cudaMallocHost us", round(t(dev.data_ptr(), hp.value), 1))
print("D2H torch-pinned  us", round(t(tp.data_ptr(), dev.data_ptr()), 1))
print("D2H cudaMallocHost us", round(t(hp.value, dev.data_ptr()), 1))
x = torch.empty(nb // 8, dtype=torch.float64)
print("H2D pageable      us", round(t(dev.data_ptr(), x.data_ptr(), 5), 1))
