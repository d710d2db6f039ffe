"""One near-field evaluation of config N (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_00161_b200 import SplitKernel, build_pswf, solve_bandwidth, workloads
from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table
c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
div = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w, pos, q = workloads.generate(c)
kern = SplitKernel(basis=build_pswf(solve_bandwidth(w.delta)), r_c=w.r_c)
plan = NearFieldPlan(kern, build_pair_table(kern), capacity=w.n, cell_div=div)
plan.set_cell(w.h)
P, Q = torch.as_tensor(pos, device="cuda"), torch.as_tensor(q, device="cuda")
for _ in range(2):
    plan.evaluate(P, Q)
torch.cuda.synchronize()
print("ok")
