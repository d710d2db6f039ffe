import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2601_00161_b200 import EspPlan, build_pswf, solve_bandwidth, tabulate_window
g = np.load("tests/golden/small_cube_p5.npz")
for thr in ("0", None):
    if thr is None:
        os.environ.pop("ESP_SORT_THRESHOLD", None)
    else:
        os.environ["ESP_SORT_THRESHOLD"] = thr
    b = build_pswf(solve_bandwidth(float(g["delta"])))
    plan = EspPlan(tuple(g["M"]), int(g["P"]), tabulate_window(b, int(g["P"])), b, float(g["r_c"]), capacity=1 << 12)
    plan.set_cell(g["h"])
    P_ = torch.as_tensor(g["pos"], device="cuda"); Q_ = torch.as_tensor(g["q"], device="cuda")
    grid = plan.spread(P_, Q_).clone()
    out7, F = plan.evaluate(P_, Q_, True)
    torch.cuda.synchronize()
    print(thr, "radix", plan.radix_binning(len(g["q"])), "gridsum", grid.sum().item(), "ref", g["grid"].sum(), "E", out7[0].item(), g["E"])
