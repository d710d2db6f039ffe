#!/usr/bin/env python
"""Benchmark: ESP long-range (k-space) atom-steps/s on B200.

Workload (BASELINE.json metric config): config 1 — 90,000
charges (30,000 rigid 3-site waters), 67x67x67.5 A semi-isotropic cell,
grid 64^3, P=8, Delta=1e-7, r_c=10, fp64, seeded synthetic inputs.  One step
= bin -> spread -> 1 forward FFT -> fused scale/reduce (E + 6 pressure
components) -> 3 ik inverse FFTs -> force gather.  ``value`` is whole-job
force+pressure atom-steps/s with inputs resident in HBM; ``pressure_only``
is the same for the pressure-only path; ``e2e`` goes through the public API
with pinned host buffers and the H2D/D2H copies inside the timed region.
L2 (126 MB) is flushed between timed steps by writing a 256 MB buffer.

--impl reference times the CPU oracle port of the reference algorithm
(oracle/esp_oracle.py; the reference is pure numpy, nothing to compile) on
all host cores: particle chunks of spread/gather in a process pool (exact by
linearity), numpy pocketfft transforms.

Multi-GPU (torchrun, N>1): config 1 does not shard (G = 2.6e5 is
latency-bound on one GPU), so N ranks run N independent
replicas ("scaling": "weak"); timings are max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIG = 1
METRIC = "ESP long-range atom-steps/s (force+pressure)"
UNIT = "atom-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-near", dest="near", action="store_false",
                    help="skip the near-field / whole-Coulomb-step leg")
    ap.add_argument("--profile-only", action="store_true",
                    help="run a few steps for ncu (no JSON contract line)")
    ap.add_argument("--slab", action="store_true",
                    help="multi-GPU z-slab decomposition of one system (strong "
                         "scaling; default workload config 4)")
    return ap.parse_args()


# --------------------------------------------------------------------------
# distributed plumbing


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, local, backend="nccl"):
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return dist if world > 1 else None


def max_over_ranks(x, dist, device=None):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md recipe)


class ClockSampler:
    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        # NVML polls every ESP_BENCH_CLOCK_MS ms (default 2; the timed regions
        # are tens of ms); nvidia-smi every 200 ms when NVML is unavailable
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                    "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                act = ["Active" if r & b else "Not Active" for b in
                       (bits["hw_slowdown"], bits["hw_thermal_slowdown"],
                        bits["sw_thermal_slowdown"], bits["sw_power_cap"])]
                self.samples.append([str(sm), str(mx), hex(r)] + act)
                self._stop.wait(float(os.environ.get("ESP_BENCH_CLOCK_MS", "2")) * 1e-3)
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, nm in enumerate(names):
                if len(s) > 3 + i and s[3 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------
# algorithmic bytes / flops (stated in DESIGN.md)


def box_counts(M, band):
    """In-band box of the half spectrum: nbx (kx >= 0), nby, nbz (esp_api.cu
    set_cell), and the fused path's padded kx pitch."""
    nbx = min(band[0], M[0] // 2) + 1
    nb = [M[d] if 2 * band[d] + 1 >= M[d] else 2 * band[d] + 1 for d in (1, 2)]
    return nbx, nb[0], nb[1], (nbx + 7) // 8 * 8


def scratch_elems(w):
    """Spread scratch blocks (esp_api.cu plan create): tiles of TX = TY = 17-P
    anchors, TZS planes (4 on grids with Mz <= 128, else 32), padded 16 x 16
    x (TZS + P - 1)."""
    Mx, My, Mz = w.M
    T = 17 - w.P
    tzs = min(4 if Mz <= 128 else 32, Mz)
    ntx, nty, ntz = -(-Mx // T), -(-My // T), -(-Mz // tzs)
    return ntx * nty * ntz * (tzs + w.P - 1) * 256


def algorithmic(w, n, band, real_bytes=8, n_scratch=None):
    """Compulsory HBM bytes and flops per launch of each stage kernel."""
    Mx, My, Mz = w.M
    G = Mx * My * Mz
    H = (Mx // 2 + 1) * My * Mz
    r, c, pb = real_bytes, 2 * real_bytes, 32
    P, D = w.P, 18
    nbx, nby, nbz, _ = box_counts(w.M, band)
    nbox = nbx * nby * nbz
    scratch = n_scratch if n_scratch is not None else G
    lg = np.log2
    return {
        "spread": dict(bytes=pb * n + r * G, flops=2 * (3 * P * D + P * P + P + P ** 3) * n),
        "combine": dict(bytes=r * (scratch + G), flops=0),   # tile blocks in, grid out
        # cuFFT path
        "fft_forward": dict(bytes=r * G + c * H, flops=2.5 * G * lg(G)),
        "scale_reduce": dict(bytes=c * H, flops=40 * H),
        "fft_inverse_x3": dict(bytes=3 * (c * H + r * G), flops=3 * 2.5 * G * lg(G)),
        # band-pruned fused path (esp_fft.cu)
        "fft_x": dict(bytes=r * G + c * My * Mz * nbx, flops=2.5 * G * lg(Mx)),
        "fft_y": dict(bytes=c * Mz * nbx * (My + nby), flops=5 * Mz * nbx * My * lg(My)),
        "fft_z_scale_reduce": dict(bytes=c * Mz * nby * nbx + (c + 16) * nbox,
                                   flops=5 * nby * nbx * Mz * lg(Mz) + 40 * nbox),
        "ifft_z_ik": dict(bytes=(c + 8) * nbox + 3 * c * Mz * nby * nbx,
                          flops=3 * 5 * nby * nbx * Mz * lg(Mz)),
        "ifft_y": dict(bytes=3 * c * Mz * nbx * (nby + My), flops=3 * 5 * Mz * nbx * My * lg(My)),
        "ifft_x": dict(bytes=3 * (c * My * Mz * nbx + r * G), flops=3 * 2.5 * G * lg(Mx)),
        "gather": dict(bytes=pb * n + 3 * r * G + 3 * r * n,
                       flops=2 * (3 * P * D + P * P + 3 * P ** 3) * n),
    }


def dram_traffic(workload, precision):
    """Per-launch DRAM bytes (read + write) of each stage kernel, from the
    ncu capture summarised by profiles/traffic.py."""
    try:
        with open(os.path.join(REPO, "profiles", "dram_traffic.json")) as f:
            return json.load(f).get(f"{workload}/{precision}", {})
    except Exception:
        return {}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------------------
# our arm


def quiet_host_pools():
    """Host thread pools (OpenBLAS / OpenMP / torch intra-op) busy-wait after
    parallel CPU work; on the B200 box that slows pinned H2D DMA ~3x
    (tools/tools_copy_probe3.py).  The timed path does no CPU math, so pin
    the pools to one thread and let spinning threads park before timing."""
    import torch
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    torch.set_num_threads(1)
    time.sleep(0.3)


def run_ours(args):
    import torch

    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads
    from paper_2601_00161_b200.plan import probe_fp64_tflops

    rank, world, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w, pos_np, q_np = workloads.generate(args.config)
    n = w.n
    solver = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                               fixed_M=w.M, precision=args.precision,
                                               cell_type=w.cell_type), capacity=n)
    pos = torch.as_tensor(pos_np, device=dev)
    q = torch.as_tensor(q_np, device=dev)
    out7 = torch.empty(7, dtype=torch.float64, device=dev)
    F = torch.empty((n, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step(want_forces=True):
        solver.evaluate_device(pos, q, want_forces, out7, F if want_forces else None)

    if args.profile_only:
        for _ in range(max(args.warmup, 1) + args.steps):
            step()
        torch.cuda.synchronize()
        return None

    def timed(fn, K, W):
        for _ in range(W):
            fn()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        total = 0.0
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        for i in range(K):
            flush.zero_()                      # evict L2 between timed steps
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        total = sum(a.elapsed_time(b) for a, b in ev)
        return max_over_ranks(total / K, dist, dev)

    K, W = args.steps, args.warmup
    # The whole step is captured once as a CUDA graph (bin, spread, combine,
    # cuFFT, scale/reduce, cuFFT x3, gather) and replayed per timed step.
    out7_po = torch.empty(7, dtype=torch.float64, device=dev)
    g_fp, _, _ = solver.graphed(pos, q, True, out7, F)
    launches = solver.plan.launches_last_step()
    g_po, _, _ = solver.graphed(pos, q, False, out7_po, None)
    launches_po = solver.plan.launches_last_step()
    # analytic-differentiation forces (the paper's production mode, SURVEY
    # §8(f) f1): 1 inverse transform + window-gradient gather
    an = None
    if w.cell_type != "triclinic":
        solver_an = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                                      fixed_M=w.M, precision=args.precision,
                                                      cell_type=w.cell_type,
                                                      force_mode="analytic"), capacity=n)
        F_an = torch.empty((n, 3), dtype=torch.float64, device=dev)
        o7_an = torch.empty(7, dtype=torch.float64, device=dev)
        g_an, _, _ = solver_an.graphed(pos, q, True, o7_an, F_an)
    # fp32 mode (BASELINE config 1 lists fp64 and fp32; fp64 positions/anchors,
    # fp32 grid / transforms / fields, fp64 reductions; tolerance 1e-5)
    f32 = None
    if args.precision == "fp64":
        solver32 = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                                     fixed_M=w.M, precision="fp32",
                                                     cell_type=w.cell_type), capacity=n)
        F32 = torch.empty((n, 3), dtype=torch.float64, device=dev)
        o7_32 = torch.empty(7, dtype=torch.float64, device=dev)
        g_32, _, _ = solver32.graphed(pos, q, True, o7_32, F32)
    hs = solver.host_stepper(n, True)            # public host-buffer API
    hs.positions.copy_(torch.as_tensor(pos_np))
    hs.charges.copy_(torch.as_tensor(q_np))
    quiet_host_pools()
    with ClockSampler(local) as clk:
        ms_fp = timed(g_fp.replay, K, W)
        ms_po = timed(g_po.replay, K, W)
        ms_e2e = timed(hs.launch, K, W)
        ms_eager = timed(lambda: step(True), K, W)
        if args.precision == "fp64":
            ms_32 = timed(g_32.replay, K, W)
            f32 = {"ms_per_step": ms_32, "value": world * n / (ms_32 * 1e-3), "unit": UNIT,
                   "what": "force+pressure, precision='fp32' (fp32 grid, transforms and "
                           "fields; fp64 coordinates and reductions)"}
        if w.cell_type != "triclinic":
            ms_an = timed(g_an.replay, K, W)
            an = {"ms_per_step": ms_an, "value": world * n / (ms_an * 1e-3), "unit": UNIT,
                  "what": "force+pressure with analytic-differentiation forces "
                          "(force_mode='analytic'; the headline uses ik, the reference default)"}
        near = near_field_leg(w, pos, q, solver, timed, K, W) if args.near else None
    clocks = clk.summary()
    torch.cuda.synchronize()
    assert np.isfinite(hs.forces.numpy()).all() and np.isfinite(hs.out7.numpy()).all()

    # per-kernel profile (separate, untimed pass): dominant kernel roofline
    solver.plan.set_profiling(True)
    prof = {}
    reps = 5
    for _ in range(reps):
        flush.zero_()
        step(True)
        for name, t in solver.plan.profile():
            prof[name] = prof.get(name, 0.0) + t / reps
    solver.plan.set_profiling(False)
    torch.cuda.synchronize()
    fp64_tflops = probe_fp64_tflops()
    hbm_peak, peak_kind = measured_peaks()
    real_b = 8 if args.precision == "fp64" else 4
    alg = algorithmic(w, n, solver.plan.tables.band, real_b, n_scratch=scratch_elems(w))
    kern = {k: v for k, v in prof.items() if k in alg}
    dom = max(kern, key=kern.get) if kern else None
    roof = None
    roof_fp = None
    line_smem = None
    if dom:
        t = kern[dom] * 1e-3
        ach = alg[dom]["bytes"] / t / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 2), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(ach / hbm_peak, 4), "traffic": None,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                "avg_launch_ms": round(kern[dom], 5)}
        if alg[dom]["flops"]:
            fl = alg[dom]["flops"] / t / 1e12
            roof_fp = {"kernel": dom, "bound": "fp64" if real_b == 8 else "fp32",
                       "achieved": round(fl, 3), "peak": round(fp64_tflops, 2),
                       "unit": "TFLOP/s", "frac": round(fl / fp64_tflops, 4),
                       "peak_source": "measured DFMA-chain probe (esp_probe_fp64)"}

        # measured DRAM bytes of the same kernel from the committed ncu capture
        tr = dram_traffic(w.name, args.precision).get(dom)
        if tr is not None:
            roof["traffic"] = tr
            roof["traffic_source"] = "profiles/dram_traffic.json (ncu --set full)"
        if dom == "gather" and clocks.get("sm_mhz"):
            # the gather is bound by shared-memory reads of the field tile:
            # 3 fields x P^3 points x real bytes per charge
            sm_bytes = 3 * w.P ** 3 * real_b * n
            peak_sm = 148 * 128 * clocks["sm_mhz"] * 1e6 / 1e9
            ach_sm = sm_bytes / t / 1e9
            line_smem = {"kernel": dom, "bound": "smem", "achieved": round(ach_sm, 1),
                         "peak": round(peak_sm, 1), "unit": "GB/s",
                         "frac": round(ach_sm / peak_sm, 4),
                         "peak_source": "148 SMs x 128 B/clk x median SM clock"}
        else:
            line_smem = None

    # stage-wise roofline of the whole step: per stage
    # max(compulsory bytes / HBM, flops / FP peak), binning excluded
    stages = ["spread", "fft_forward", "scale_reduce", "fft_inverse_x3", "gather"]
    fp_peak = fp64_tflops if real_b == 8 else 2 * fp64_tflops
    t_roof = sum(max(alg[k]["bytes"] / (hbm_peak * 1e9), alg[k]["flops"] / (fp_peak * 1e12))
                 for k in stages) * 1e3
    step_roof = {"model": "SURVEY §8(d) stage-wise: spread, forward FFT, scale/reduce, "
                          "3 inverse FFTs, gather; max(bytes/HBM, flops/FP peak) per stage, "
                          "binning not counted",
                 "t_roof_ms": round(t_roof, 5), "frac": round(t_roof / ms_fp, 4),
                 "hbm_gbs": hbm_peak, "fp_peak_tflops": round(fp_peak, 2)}
    value = world * n / (ms_fp * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_fp, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if real_b == 8 else "f32",
        "data": "synthetic (seeded config recipe, SURVEY §8(d.1))",
        "config": {"workload": w.name, "n_charges": n, "grid": list(w.M), "P": w.P,
                   "delta": w.delta, "r_c": w.r_c, "cell_type": w.cell_type,
                   "precision": args.precision,
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "flushed between timed steps (256 MB write)"},
        "pressure_only": {"value": world * n / (ms_po * 1e-3), "unit": UNIT,
                          "ms_per_step": ms_po, "gpu_launches_per_step": launches_po},
        "e2e": {"value": world * n / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": int(hs.h2d_bytes), "d2h_bytes_per_step": int(hs.d2h_bytes),
                "api": "KSpaceSolver.host_stepper (pinned host in/out, one CUDA graph)"},
        "eager_ms_per_step": ms_eager,
        "gpu_launches": int(launches * K),
        "gpu_launches_per_step": launches,
        "clocks": clocks,
        "roofline": roof,
        "roofline_fp": roof_fp,
        "roofline_smem": line_smem,
        "step_roofline": step_roof,
        "kernel_ms": {k: round(v, 5) for k, v in prof.items()},
        "fp64_peak_tflops_measured": round(fp64_tflops, 2),
    }
    if an is not None:
        line["analytic_forces"] = an
    if f32 is not None:
        line["fp32_mode"] = f32
    if near is not None:
        near["fp64_frac_est"] = round(near["fp64_tflops_est"] / fp64_tflops, 4)
        line["near_field"] = near
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_port(args.config)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


NEAR_FLOPS_PER_DIRECTED_PAIR = 55   # table path, DESIGN.md §9
NEAR_FLOPS_PER_CANDIDATE = 8


def near_field_leg(w, pos, q, kspace, timed, K, W):
    """Near field on the same particles: the device cell
    list + fused pair pass alone, and the whole Coulomb step (near + far +
    forces summed) as CoulombSolver.evaluate_device runs it (eager launches).
    Reported beside the headline, which stays the k-space metric."""
    import torch

    from paper_2601_00161_b200 import SplitKernel
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table

    kern = SplitKernel(basis=kspace.kern.basis, r_c=w.r_c)
    table = build_pair_table(kern)
    plan = NearFieldPlan(kern, table, capacity=w.n)
    plan.set_cell(w.h)
    o7 = torch.empty(7, dtype=torch.float64, device=pos.device)
    st = torch.empty(4, dtype=torch.int64, device=pos.device)
    Fn = torch.empty((w.n, 3), dtype=torch.float64, device=pos.device)
    o7f = torch.empty(7, dtype=torch.float64, device=pos.device)

    def near():
        plan.evaluate(pos, q, forces=Fn, out7=o7, stats=st)

    def coulomb():
        kspace.evaluate_device(pos, q, True, o7f, Fn)
        plan.evaluate(pos, q, forces=Fn, accumulate=True, out7=o7, stats=st)

    from paper_2601_00161_b200 import CoulombSolver, EwaldParameters
    cs = CoulombSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                            fixed_M=w.M, cell_type=w.cell_type))
    g_all, _ = cs.graphed(pos, q, True)
    kn, wn = max(3, min(K, 20)), max(W, 3)
    ms_near = timed(near, kn, wn)
    ms_all = timed(coulomb, kn, wn)
    ms_graph = timed(g_all.replay, kn, wn)
    pairs = int(st[0].item())
    directed = 2.0 * pairs
    tfl = directed * NEAR_FLOPS_PER_DIRECTED_PAIR / (ms_near * 1e-3) / 1e12
    info = plan.info()
    return {"ms_per_step": ms_near, "pairs_within_rc": pairs,
            "directed_pair_evals_per_s": directed / (ms_near * 1e-3),
            "fp64_tflops_est": round(tfl, 3),
            "flops_model": f"{NEAR_FLOPS_PER_DIRECTED_PAIR} flop per directed pair (table path)",
            "cells": list(info["cells"]), "launches_per_step": info["launches"],
            "coulomb_step": {"ms_per_step": ms_all, "value": w.n / (ms_all * 1e-3),
                             "unit": UNIT,
                             "what": "far (k-space, eager) + near (cell list) + summed forces"},
            "coulomb_step_graphed": {
                "ms_per_step": ms_graph, "value": w.n / (ms_graph * 1e-3), "unit": UNIT,
                "what": "CoulombSolver.graphed: near and far on two streams of one CUDA graph"},
            "steps": kn}


# --------------------------------------------------------------------------
# CPU legs


def cpu_baseline_port(config):
    """Oracle port, 1 thread, one full step of the workload (bounded sample)."""
    from oracle import esp_oracle as O
    from paper_2601_00161_b200 import workloads
    w, pos, q = workloads.generate(config)
    plan = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    modes = O.Modes(plan)
    t0 = time.perf_counter()
    rh = O.forward_density(plan, pos, q)
    O.energy(modes, rh)
    O.pressure(modes, rh)
    t1 = time.perf_counter()
    O.forces_ik(plan, modes, rh, pos, q)
    t2 = time.perf_counter()
    return {"value": w.n / (t2 - t0), "unit": UNIT, "cores": 1, "kind": "port",
            "pressure_only_value": w.n / (t1 - t0),
            "sample": f"1 full {w.name} force+pressure step ({w.n} charges, grid "
                      f"{'x'.join(map(str, w.M))}, P={w.P}), numpy oracle port "
                      f"(oracle/esp_oracle.py), single thread; ModeWorkspace setup excluded",
            "seconds": round(t2 - t0, 3)}


_POOL_STATE = {}


def _spread_chunk(args):
    lo, hi = args
    st = _POOL_STATE
    from oracle import esp_oracle as O
    return O.spread(st["plan"], st["pos"][lo:hi], st["q"][lo:hi])


def _gather_chunk(args):
    lo, hi, fields = args
    st = _POOL_STATE
    from oracle import esp_oracle as O
    out = np.empty((hi - lo, 3))
    for d in range(3):
        out[:, d] = O.gather(st["plan"], fields[d], st["pos"][lo:hi])
    return out


def run_reference(args):
    """Reference arm: the oracle port of the reference CPU path on all host
    cores, same config/metric as our arm.  Rank 0 only."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp

    from oracle import esp_oracle as O
    from paper_2601_00161_b200 import workloads
    w, pos, q = workloads.generate(args.config)
    plan = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    modes = O.Modes(plan)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    _POOL_STATE.update(plan=plan, pos=pos, q=q)
    ctx = mp.get_context("fork")
    chunks = np.linspace(0, w.n, cores + 1).astype(int)
    spans = [(int(a), int(b)) for a, b in zip(chunks[:-1], chunks[1:]) if b > a]
    h3 = plan.volume_element
    with ctx.Pool(cores) as pool:
        def one_step():
            grid = sum(pool.map(_spread_chunk, spans))
            rh = np.fft.fftn(grid) * h3
            O.energy(modes, rh)
            O.pressure(modes, rh)
            scale = modes.fhat * modes.w_inv2 * rh[modes.mask]
            fields = []
            for d in range(3):
                spec = np.zeros(plan.M, dtype=complex)
                spec[modes.mask] = 1j * modes.kvec[d] * scale
                fields.append(np.fft.ifftn(spec).real / h3)
            parts = pool.map(_gather_chunk, [(a, b, fields) for a, b in spans])
            return -q[:, None] * h3 * np.concatenate(parts)

        budget = 150.0
        t_start = time.perf_counter()
        for _ in range(args.warmup):
            one_step()
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one_step()
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > budget:
                break
    ms = 1e3 * float(np.mean(times))
    v = w.n / (ms * 1e-3)
    sample = (f"{len(times)} of {args.steps} requested full {w.name} force+pressure steps "
              f"({w.n} charges); spread/gather in {cores} processes, numpy FFT")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": len(times),
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config recipe, SURVEY §8(d.1))",
            "config": {"workload": w.name, "n_charges": w.n, "grid": list(w.M), "P": w.P,
                       "delta": w.delta, "r_c": w.r_c, "parallelism": "cpu"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_slab(args):
    """Strong scaling: one config-4 system decomposed into z-slabs over the
    ranks (NCCL halo send/recv, transposes stored over peer memory by the
    band-pruned transform kernels, 7-double all-gather)."""
    import torch

    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads
    from paper_2601_00161_b200.pswf import build_pswf, solve_bandwidth, tabulate_window
    from paper_2601_00161_b200.slab import SlabKSpaceSolver

    rank, world, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config if args.config != CONFIG else 4
    w, pos_np, q_np = workloads.generate(cfg)
    basis = build_pswf(solve_bandwidth(w.delta))
    window = tabulate_window(basis, w.P)
    s = SlabKSpaceSolver(w.h, w.M, w.P, basis, window, w.r_c, precision=args.precision,
                         capacity=w.n // max(world, 1) + w.n // 8)
    mine = s.owned(pos_np)
    pos = torch.as_tensor(pos_np[mine], device=dev)
    q = torch.as_tensor(q_np[mine], device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def timed(want_forces, K, W):
        for _ in range(W):
            s.evaluate(pos, q, want_forces)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        for i in range(K):
            flush.zero_()
            ev[i][0].record(stream)
            s.evaluate(pos, q, want_forces)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / K, dist, dev)

    near = None
    if args.near:
        from paper_2601_00161_b200 import Cell, SplitKernel
        from paper_2601_00161_b200.realspace import build_pair_table
        from paper_2601_00161_b200.slab_near import CudaNearOps, SlabNearField
        kern = SplitKernel(basis=basis, r_c=w.r_c)
        sn = SlabNearField.from_kspace(s, w.r_c, CudaNearOps(kern, build_pair_table(kern),
                                                             Cell(np.asarray(w.h, float))))
        sn.ops.plan.reserve(pos.shape[0] + pos.shape[0] // 2)

    def timed_near(K, W):
        for _ in range(W):
            sn.evaluate(pos, q)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)]
        for i in range(K):
            flush.zero_()
            ev[i][0].record(stream)
            sn.evaluate(pos, q)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / K, dist, dev)

    with ClockSampler(local) as clk:
        ms_fp = timed(True, args.steps, args.warmup)
        ms_po = timed(False, args.steps, args.warmup)
        if args.near:
            ms_near = timed_near(max(3, min(args.steps, 5)), 2)
            near = {"ms_per_step": ms_near, "value": w.n / (ms_near * 1e-3), "unit": UNIT,
                    "what": "slab near field (ghost all-to-all, slab-local pair sums, "
                            "rank-ordered reduction), slab_near.SlabNearField"}
    line = {"metric": METRIC, "value": w.n / (ms_fp * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_fp,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (seeded config recipe, SURVEY §8(d.1))",
            "config": {"workload": w.name, "n_charges": w.n, "grid": list(w.M), "P": w.P,
                       "parallelism": f"zslab{world}", "precision": args.precision,
                       "l2": "flushed between timed steps (256 MB write)"},
            "pressure_only": {"value": w.n / (ms_po * 1e-3), "unit": UNIT,
                              "ms_per_step": ms_po},
            "clocks": clk.summary()}
    if near is not None:
        line["near_field"] = near
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.slab:
        run_slab(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
