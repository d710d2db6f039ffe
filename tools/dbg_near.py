import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd()+"/tests")
import numpy as np, torch
from conftest import golden
from oracle import esp_oracle as O
from paper_2601_00161_b200 import SplitKernel, build_pswf, solve_bandwidth
from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table, out7_to_pressure
g = golden("near_brick")
kern = SplitKernel(basis=build_pswf(solve_bandwidth(float(g["delta"]))), r_c=float(g["r_c"]))
t = build_pair_table(kern)
for div in (1, 2):
    plan = NearFieldPlan(kern, t, cell_div=div); plan.set_cell(g["h"])
    P = torch.as_tensor(g["pos"], device="cuda"); Q = torch.as_tensor(g["q"], device="cuda")
    o, F, st = plan.evaluate(P, Q)
    print("cell div", div, plan.info(), st.cpu().numpy(), o.cpu().numpy()[:2], g["E_tab"], g["count"])
    F = F.cpu().numpy()
    bad = np.nonzero(np.abs(F - g["F_tab"]).max(1) > 1e-8)[0]
    print("bad particles", bad[:20], len(bad))
    print(g["pos"][bad[:5]])
o, F, st = plan.evaluate_pairs(P, Q, torch.as_tensor(g["pi"], device="cuda"), torch.as_tensor(g["pj"], device="cuda"))
print("list", st.cpu().numpy(), o.cpu().numpy()[:2], np.abs(F.cpu().numpy()-g["F_tab"]).max())
# single pair values
from paper_2601_00161_b200 import Cell
for d in (0.05, 0.1, 0.14, 0.2, 0.5, 1.0, 1.3):
    pos = np.array([[1.0, 1.0, 1.0], [1.0 + d, 1.0, 1.0]])
    o, F, st = plan.evaluate(torch.as_tensor(pos, device="cuda"), torch.as_tensor(np.array([1.0, 1.0]), device="cuda"))
    print(d, o[0].item(), t.near_field(np.array([d]))[0], F[0,0].item(), -t.fn_weight(np.array([d]))[0]/d**2)
