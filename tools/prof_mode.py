"""Per-kernel times of one config-4 step in a given force mode / precision."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads
mode = sys.argv[1] if len(sys.argv) > 1 else "ik"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 4
w, pos, q = workloads.generate(cfg)
s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                      precision=prec, cell_type=w.cell_type, force_mode=mode),
                 capacity=w.n)
P_, Q_ = torch.as_tensor(pos, device="cuda"), torch.as_tensor(q, device="cuda")
for _ in range(3):
    s.evaluate_device(P_, Q_)
s.plan.set_profiling(True)
acc = {}
for _ in range(5):
    s.evaluate_device(P_, Q_)
    for k, v in s.plan.profile():
        acc[k] = acc.get(k, 0) + v / 5
s.plan.set_profiling(False)
print(mode, prec, round(sum(acc.values()), 3), {k: round(v, 3) for k, v in acc.items()})
