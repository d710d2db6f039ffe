"""Per-kernel times (CUDA events) of the analytic-force step at a config."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w, pos, q = workloads.generate(c)
for mode in ("ik", "analytic"):
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          force_mode=mode), capacity=w.n)
    P = torch.as_tensor(pos, device="cuda")
    Q = torch.as_tensor(q, device="cuda")
    for _ in range(3):
        s.evaluate_device(P, Q)
    s.plan.set_profiling(True)
    prof = {}
    for _ in range(5):
        s.evaluate_device(P, Q)
        for name, t in s.plan.profile():
            prof[name] = prof.get(name, 0.0) + t / 5
    s.plan.set_profiling(False)
    print(mode, {k: round(v * 1e3, 1) for k, v in prof.items()}, "us")
