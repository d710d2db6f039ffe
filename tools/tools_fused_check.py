"""Diagnostic: fused band-pruned transforms vs the cuFFT path (same plan
inputs), relative differences and CUDA-graph step times (L2 flushed)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads

flush = torch.empty(64 * 1024 * 1024, device='cuda')


def run(cfg, prec, mode, forces=True):
    os.environ["ESP_FFT"] = mode
    w, pos, q = workloads.generate(cfg)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          precision=prec), capacity=w.n)
    P_ = torch.as_tensor(pos, device='cuda')
    Q_ = torch.as_tensor(q, device='cuda')
    out7 = torch.empty(7, dtype=torch.float64, device='cuda')
    F = torch.zeros((w.n, 3), dtype=torch.float64, device='cuda')
    plan = s.plan

    def fn():
        plan.evaluate(P_, Q_, forces, out7, F)
    fn()
    torch.cuda.synchronize()
    res = (out7.cpu().numpy().copy(), F.cpu().numpy().copy())
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        flush.zero_()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del g, s, plan
    torch.cuda.synchronize()
    return res, float(np.median(ts))


cfgs = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 2]
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fp64"]
if len(sys.argv) > 3 and sys.argv[3] == "fusedonly":
    for cfg in cfgs:
        for prec in precs:
            print(cfg, prec, run(cfg, prec, "fused", True)[1], flush=True)
    sys.exit(0)
for cfg in cfgs:
    for prec in precs:
        for forces in (True, False):
            (a7, aF), ta = run(cfg, prec, "fused", forces)
            (b7, bF), tb = run(cfg, prec, "cufft", forces)
            dE = abs(a7[0] - b7[0]) / abs(b7[0])
            dP = np.linalg.norm(a7[1:] - b7[1:]) / np.linalg.norm(b7[1:])
            dF = (np.sqrt(np.mean((aF - bF) ** 2)) / np.sqrt(np.mean(bF ** 2))) if forces else 0.0
            print(f"cfg{cfg} {prec} forces={forces}: fused {ta:.4f} ms  cufft {tb:.4f} ms  "
                  f"dE {dE:.2e} dP {dP:.2e} dF {dF:.2e}", flush=True)
