"""Analytic-force steps of config N (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w, pos, q = workloads.generate(c)
s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                      force_mode="analytic"), capacity=w.n)
P, Q = torch.as_tensor(pos, device="cuda"), torch.as_tensor(q, device="cuda")
for _ in range(3):
    s.evaluate_device(P, Q)
torch.cuda.synchronize()
print("ok")
