"""Diagnostic: per-stage CUDA-graph replay times (median of 30, L2 flushed)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
w, pos, q = workloads.generate(cfg)
s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                      precision=prec), capacity=w.n)
P_ = torch.as_tensor(pos, device='cuda'); Q_ = torch.as_tensor(q, device='cuda')
plan = s.plan
out7 = torch.empty(7, dtype=torch.float64, device='cuda')
F = torch.empty((w.n, 3), dtype=torch.float64, device='cuda')
plan.evaluate(P_, Q_, True, out7, F)
torch.cuda.synchronize()
flush = torch.empty(64 * 1024 * 1024, device='cuda')

def graph_of(fn):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    return g

def t(g):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(30):
        flush.zero_(); e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)) * 1e3

stages = {
    "full F+P": lambda: plan.evaluate(P_, Q_, True, out7, F),
    "pressure-only": lambda: plan.evaluate(P_, Q_, False, out7, None),
    "bin+spread+combine": lambda: plan.spread(P_, Q_),
    "forward fft": lambda: plan.forward(),
    "scale/reduce (E,P)": lambda: plan.scale_reduce(False, out7),
    "scale/reduce + ik": lambda: plan.scale_reduce(True, out7),
}
res = {}
for k, fn in stages.items():
    res[k] = t(graph_of(fn))
g_ik = graph_of(lambda: (plan.scale_reduce(True, out7), plan.forces_ik(w.n, F)))
res["ik spectra + C2R x3 + gather"] = t(g_ik)
for k, v in res.items():
    print(f"{k:32s} {v:9.1f} us")
