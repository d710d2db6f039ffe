"""Small non-plane grid through the TMA gather path vs the oracle (debug aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import esp_oracle as O
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads

L, M, n = 40.0, (96, 96, 96), 3000
rng = np.random.default_rng(5)
pos = workloads.wrap_positions(np.diag([L] * 3), rng.uniform(0, L, (n, 3)))
q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
s = KSpaceSolver(np.diag([L] * 3), EwaldParameters(r_c=10.0, delta_split=1e-7, P=8, fixed_M=M,
                                                  precision=prec))
r = s.evaluate(pos, q)
torch.cuda.synchronize()
print("fields layout padded:", s.plan.fields_view().stride())
plan = O.make_plan(np.diag([L] * 3), M, 8, 1e-7, 10.0)
E, Pt, F = O.kspace(plan, pos, q)
print("relE", O.rel_scalar(r.energy, E), "relF", O.rms_rel_forces(r.forces, F))
