"""Time the device near-field pair sum (cell list + fused pass) per config
and cells-per-reach setting.  Usage: python tools/tools_near_time.py [cfg ...]"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_00161_b200 import SplitKernel, build_pswf, solve_bandwidth, workloads  # noqa
from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table  # noqa


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1]
    for c in cfgs:
        w, pos, q = workloads.generate(c)
        kern = SplitKernel(basis=build_pswf(solve_bandwidth(w.delta)), r_c=w.r_c)
        table = build_pair_table(kern)
        P = torch.as_tensor(pos, device="cuda")
        Q = torch.as_tensor(q, device="cuda")
        for div in (0, 2, 3):
            plan = NearFieldPlan(kern, table, capacity=w.n, cell_div=div)
            plan.set_cell(w.h)
            for _ in range(3):
                out7, F, st = plan.evaluate(P, Q)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            reps = 10
            e0.record()
            for _ in range(reps):
                plan.evaluate(P, Q, forces=F, out7=out7, stats=st)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            pairs = int(st[0])
            inf = plan.info()
            print(f"cfg{c} N={w.n} div={div} cells={inf['cells']} stencil={inf['stencil']} "
                  f"pairs={pairs} ms={ms:.3f} pair-evals/s={2 * pairs / ms * 1e3:.3e} "
                  f"E={out7[0].item():.10g}", flush=True)


if __name__ == "__main__":
    main()
