"""Tile-shape sweep (diagnostic): graph-replay step time for (TZ gather, TZS spread)."""
import os, sys, json, subprocess
cfg = sys.argv[1] if len(sys.argv) > 1 else "1"
for tz, tzs in [(8, 8), (4, 4), (8, 4), (4, 8), (8, 16), (16, 16), (6, 6)]:
    code = f"""
import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads
from paper_2601_00161_b200.plan import EspPlan
w, pos, q = workloads.generate({cfg})
s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M), capacity=w.n)
s.plan = EspPlan(w.M, w.P, s.spec.window, s.kern.basis, w.r_c, capacity=w.n, tile=(0, 0, {tz}))
s.plan.set_cell(w.h)
P_ = torch.as_tensor(pos, device='cuda'); Q_ = torch.as_tensor(q, device='cuda')
res = []
for wf in (True, False):
    g, o7, F = s.graphed(P_, Q_, wf)
    for _ in range(5): g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64*1024*1024, device='cuda')
    ts = []
    for _ in range(20):
        flush.zero_(); e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    res.append(float(np.median(ts)))
print({tz}, {tzs}, res)
"""
    env = dict(os.environ, ESP_TILE_ZS=str(tzs))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    print(r.stdout.strip() or r.stderr[-500:], flush=True)
