#!/usr/bin/env python
"""Benchmark: ESP long-range (k-space) atom-steps/s on B200.

Workload: config 4 (BASELINE.json ``configs[4]``), the largest configuration
and the one the metric is quoted on at N=1 — 8,100,000 charges (2.7M rigid
3-site waters), cubic 300 A cell, grid 384^3, P=8, Delta=1e-7, r_c=10, fp64,
seeded synthetic inputs.  One step = bin -> spread -> 1
forward FFT -> fused scale/reduce (E + 6 pressure components) -> 3 ik
inverse FFTs -> force gather, replayed as one CUDA graph.  ``value`` is
whole-job force+pressure atom-steps/s with inputs resident in HBM, from the
MEDIAN of the K CUDA-event-timed steps; ``pressure_only`` is
the same for the pressure-only path; ``e2e`` goes through the public API
(``KSpaceSolver.host_stepper``) with pinned host buffers and the H2D/D2H
copies inside the timed region.  L2 (126 MB) is flushed between timed steps
by writing a 256 MB buffer (the config-4 grids are 0.45 GB each anyway).
``--config i`` selects another BASELINE config (0-3 are parity cases).

--impl reference times the CPU port of the reference algorithm
(oracle/esp_oracle.py; the reference is pure numpy, nothing to compile) on
all host cores: particle chunks of spread/gather in a fork process pool over
shared-memory buffers (exact by linearity), numpy pocketfft transforms as the
reference calls them.  Each step is a full config-4 step; the run is bounded
by a time budget (``--ref-budget`` seconds of timed steps, at least one).

Multi-GPU (torchrun, N>1): config 4 is decomposed into z-slabs over the N
ranks (``slab.SlabKSpaceSolver``: NCCL halo send/recv, band-pruned transforms
whose transposes are stored into the peer ranks' buffers, rank-ordered
7-double reduction) — strong scaling, ``"scaling": "strong"``; timings are
the max over ranks.  ``--replicas`` runs N independent single-GPU copies
instead (weak scaling, the small configs).
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

CONFIG = 4
METRIC = "ESP long-range atom-steps/s (force+pressure)"
UNIT = "atom-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
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
                    help="z-slab decomposition of one system even at N=1 (strong "
                         "scaling; the default whenever WORLD_SIZE > 1)")
    ap.add_argument("--replicas", action="store_true",
                    help="with N>1: N independent single-GPU replicas (weak scaling)")
    ap.add_argument("--ref-budget", type=float, default=300.0,
                    help="--impl reference: seconds of timed CPU steps (at least one)")
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
    if Mz >= 256 and (-(-Mx // T)) * (-(-My // T)) * (Mz // 64) >= 148 * 8 * 4:
        tzs = min(64, Mz)
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
# timing


def timed_steps(fn, K, W, flush, stream, dist, dev, stats=None, tag=None):
    """W untimed warm-up steps, then K steps each bracketed by CUDA events on
    the launching stream, L2 flushed (256 MB write) before each; a barrier +
    synchronize on both sides.  Returns the MEDIAN step time in ms (SURVEY
    §8(d)), max over ranks; mean / min / max go into ``stats[tag]``."""
    import torch
    for _ in range(W):
        fn()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
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
    ts = [a.elapsed_time(b) for a, b in ev]
    med = max_over_ranks(statistics.median(ts), dist, dev)
    if stats is not None and tag:
        stats[tag] = {"median_ms": round(med, 5),
                      "mean_ms": round(max_over_ranks(sum(ts) / K, dist, dev), 5),
                      "min_ms": round(min(ts), 5), "max_ms": round(max(ts), 5), "steps": K}
    return med


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

    stats = {}

    def timed(fn, K, W, tag=None):
        return timed_steps(fn, K, W, flush, stream, dist, dev, stats, tag)

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
        ms_fp = timed(g_fp.replay, K, W, "force_pressure")
        ms_po = timed(g_po.replay, K, W, "pressure_only")
        ms_e2e = timed(hs.launch, K, W, "e2e")
        ms_eager = timed(lambda: step(True), K, W, "eager")
        if args.precision == "fp64":
            ms_32 = timed(g_32.replay, K, W, "fp32")
            f32 = {"ms_per_step": ms_32, "value": world * n / (ms_32 * 1e-3), "unit": UNIT,
                   "what": "force+pressure, precision='fp32' (fp32 grid, transforms and "
                           "fields; fp64 coordinates and reductions)"}
        if w.cell_type != "triclinic":
            ms_an = timed(g_an.replay, K, W, "analytic")
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
    if "combine" not in prof and "fft_x" in prof:
        # the forward x pass summed the spread's tile blocks itself
        # (k_x_comb_r2c): it reads the scratch instead of a combined grid
        Mx, My, Mz = w.M
        nbx = box_counts(w.M, solver.plan.tables.band)[0]
        alg["fft_x"] = dict(bytes=real_b * scratch_elems(w) + 2 * real_b * My * Mz * nbx,
                            flops=alg["fft_x"]["flops"])
    kern = {k: v for k, v in prof.items() if k in alg}
    dom = max(kern, key=kern.get) if kern else None
    # every stage kernel against both ceilings (algorithmic bytes and flops
    # per launch over its event-timed duration)
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

    fp_pk = fp64_tflops if real_b == 8 else 2 * fp64_tflops
    kernel_roofline = {
        k: {"ms": round(v, 5),
            "hbm_gbs": round(alg[k]["bytes"] / (v * 1e-3) / 1e9, 1),
            "hbm_frac": round(alg[k]["bytes"] / (v * 1e-3) / 1e9 / hbm_peak, 4),
            "tflops": round(alg[k]["flops"] / (v * 1e-3) / 1e12, 3),
            "fp_frac": round(alg[k]["flops"] / (v * 1e-3) / 1e12 / fp_pk, 4)}
        for k, v in kern.items() if v > 0}
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
        "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
        "dtype": "f64" if real_b == 8 else "f32",
        "data": "synthetic (seeded config recipe, SURVEY §8(d.1))",
        "config": {"workload": w.name, "n_charges": n, "grid": list(w.M), "P": w.P,
                   "delta": w.delta, "r_c": w.r_c, "cell_type": w.cell_type,
                   "precision": args.precision,
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "flushed between timed steps (256 MB write)",
                   "statistic": "median step time"},
        "pressure_only": {"value": world * n / (ms_po * 1e-3), "unit": UNIT,
                          "ms_per_step": ms_po, "gpu_launches_per_step": launches_po},
        "e2e": {"value": world * n / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": int(hs.h2d_bytes), "d2h_bytes_per_step": int(hs.d2h_bytes),
                "api": "KSpaceSolver.host_stepper (pinned host in/out, one CUDA graph)"},
        "eager_ms_per_step": ms_eager,
        "timing": dict(stats, statistic="median over the K timed steps (CUDA events, "
                                         "L2 flushed before each)"),
        "gpu_launches": int(launches * K),
        "gpu_launches_per_step": launches,
        "clocks": clocks,
        "roofline": roof,
        "roofline_fp": roof_fp,
        "roofline_smem": line_smem,
        "step_roofline": step_roof,
        "kernel_ms": {k: round(v, 5) for k, v in prof.items()},
        "kernel_roofline": kernel_roofline,
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
    kn, wn = max(3, min(K, 20 if w.n < 2_000_000 else 5)), max(min(W, 5), 3)
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


CPU_SAMPLE_CHARGES = 100_000


def cpu_baseline_port(config):
    """Oracle port (the reference's numpy algorithm), 1 thread, bounded
    sample of one step.  Small configs: one full step.  Large configs (config
    4 would take ~11 min on one core): every mesh stage once at full size
    (spread grid -> fftn -> energy + pressure; one ik spectrum + ifftn, x3),
    plus spread and the 3-field gather of the first CPU_SAMPLE_CHARGES
    charges, scaled to N (both are per-charge linear, mesh.py:204-218)."""
    from oracle import esp_oracle as O
    from paper_2601_00161_b200 import workloads
    w, pos, q = workloads.generate(config)
    plan = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    modes = O.Modes(plan)
    ns = min(w.n, CPU_SAMPLE_CHARGES) if w.n > 3 * CPU_SAMPLE_CHARGES else w.n
    h3 = plan.volume_element
    t0 = time.perf_counter()
    grid = O.spread(plan, pos[:ns], q[:ns])
    t1 = time.perf_counter()
    rh = np.fft.fftn(grid) * h3
    O.energy(modes, rh)
    O.pressure(modes, rh)
    t2 = time.perf_counter()
    scale = modes.fhat * modes.w_inv2 * rh[modes.mask]
    n_inv = 3 if ns == w.n else 1
    fields = []
    for d in range(n_inv):
        spec = np.zeros(plan.M, dtype=complex)
        spec[modes.mask] = 1j * modes.kvec[d] * scale
        fields.append(np.fft.ifftn(spec).real / h3)
    t3 = time.perf_counter()
    for d in range(3):
        O.gather(plan, fields[d % n_inv], pos[:ns])
    t4 = time.perf_counter()
    per_charge = ((t1 - t0) + (t4 - t3)) / ns
    mesh_fwd = t2 - t1
    mesh_inv = (t3 - t2) * (3 / n_inv)
    step = mesh_fwd + mesh_inv + per_charge * w.n
    step_po = mesh_fwd + (t1 - t0) / ns * w.n
    if ns == w.n:
        sample = (f"1 full {w.name} force+pressure step ({w.n} charges, grid "
                  f"{'x'.join(map(str, w.M))}, P={w.P}), numpy oracle port "
                  f"(oracle/esp_oracle.py), single thread; ModeWorkspace setup excluded")
    else:
        sample = (f"{w.name}: full-size mesh stages timed once (fftn + energy/pressure "
                  f"{mesh_fwd:.1f} s; one ik spectrum + ifftn {mesh_inv / 3:.1f} s, x3) plus "
                  f"spread and 3-field gather of {ns} of {w.n} charges "
                  f"({((t1 - t0) + (t4 - t3)):.1f} s), scaled linearly to N; numpy oracle "
                  f"port, single thread; ModeWorkspace setup excluded")
    return {"value": w.n / step, "unit": UNIT, "cores": 1, "kind": "port",
            "pressure_only_value": w.n / step_po, "sample": sample,
            "seconds": round(t4 - t0, 3), "step_seconds_est": round(step, 3)}


_POOL_STATE = {}


def _shared_array(shape):
    """Zero-filled float64 array in an anonymous MAP_SHARED mapping: fork
    children inherit it, so pool workers read and write it without pickling."""
    import mmap
    n = int(np.prod(shape))
    buf = mmap.mmap(-1, max(8 * n, 8))
    return np.frombuffer(buf, dtype=np.float64, count=n).reshape(shape)


def _spread_chunk(args):
    i, lo, hi = args
    st = _POOL_STATE
    from oracle import esp_oracle as O
    st["parts"][i] = O.spread(st["plan"], st["pos"][lo:hi], st["q"][lo:hi],
                              chunk=st["chunk"]).reshape(-1)
    return i


def _gather_chunk(args):
    lo, hi = args
    st = _POOL_STATE
    from oracle import esp_oracle as O
    M = st["plan"].M
    for d in range(3):
        st["F"][lo:hi, d] = O.gather(st["plan"], st["fields"][d].reshape(M),
                                     st["pos"][lo:hi], chunk=st["chunk"])
    return lo


def run_reference(args):
    """Reference arm: the oracle port of the reference CPU path (the same
    numpy operations as mesh.py:204-342) on all host cores, same config and
    metric as our arm.  Spread and gather run over particle chunks in a fork
    process pool writing into shared-memory buffers (exact by linearity; the
    per-chunk grids are summed in chunk order); the FFTs are numpy's, called
    as the reference calls them.  Rank 0 only; other ranks exit 0."""
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
    G = int(np.prod(w.M))
    chunks = np.linspace(0, w.n, cores + 1).astype(int)
    spans = [(int(a), int(b)) for a, b in zip(chunks[:-1], chunks[1:]) if b > a]
    parts = _shared_array((len(spans), G))
    fields = _shared_array((3, G))
    F = _shared_array((w.n, 3))
    _POOL_STATE.update(plan=plan, pos=pos, q=q, parts=parts, fields=fields, F=F,
                       chunk=50_000)
    h3 = plan.volume_element
    ctx = mp.get_context("fork")
    with ctx.Pool(len(spans)) as pool:
        def one_step():
            pool.map(_spread_chunk, [(i, a, b) for i, (a, b) in enumerate(spans)])
            grid = parts[0].copy()
            for i in range(1, len(spans)):
                grid += parts[i]
            rh = np.fft.fftn(grid.reshape(w.M)) * h3
            O.energy(modes, rh)
            O.pressure(modes, rh)
            scale = modes.fhat * modes.w_inv2 * rh[modes.mask]
            for d in range(3):
                spec = np.zeros(plan.M, dtype=complex)
                spec[modes.mask] = 1j * modes.kvec[d] * scale
                fields[d] = (np.fft.ifftn(spec).real / h3).reshape(-1)
            pool.map(_gather_chunk, spans)
            return -q[:, None] * h3 * F

        t_start = time.perf_counter()
        warm = 0
        for _ in range(args.warmup):
            one_step()
            warm += 1
            if time.perf_counter() - t_start > 0.25 * args.ref_budget:
                break
        times = []
        t_timed = time.perf_counter()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            Fr = one_step()
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_timed > args.ref_budget:
                break
    assert np.isfinite(Fr).all()
    ms = 1e3 * float(statistics.median(times))
    v = w.n / (ms * 1e-3)
    sample = (f"{len(times)} of {args.steps} requested full {w.name} force+pressure steps "
              f"({w.n} charges, grid {'x'.join(map(str, w.M))}) after {warm} warm-up; "
              f"spread/gather in {len(spans)} processes over shared memory, numpy FFT "
              f"(single-threaded, as the reference); median step; time budget "
              f"{args.ref_budget:.0f} s of timed steps; ModeWorkspace setup excluded")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": len(times),
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config recipe, SURVEY §8(d.1))",
            "config": {"workload": w.name, "n_charges": w.n, "grid": list(w.M), "P": w.P,
                       "delta": w.delta, "r_c": w.r_c, "cell_type": w.cell_type,
                       "precision": "fp64", "parallelism": "cpu"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": len(spans), "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_slab(args):
    """Strong scaling (the default under torchrun): one config-4 system
    decomposed into z-slabs over the ranks — spread on a z-slab plan, ghost
    planes by NCCL send/recv, band-pruned transforms whose transposes are
    stored into the peer ranks' buffers (symmetric memory over NVLink),
    7-double all-gather summed in rank order on the device, gather.  The
    step (SlabKSpaceSolver.evaluate_device) has no host synchronisation and
    is replayed as one CUDA graph per rank when NCCL capture is available."""
    import torch

    from paper_2601_00161_b200 import workloads
    from paper_2601_00161_b200.plan import probe_fp64_tflops
    from paper_2601_00161_b200.pswf import build_pswf, solve_bandwidth, tabulate_window
    from paper_2601_00161_b200.slab import SlabKSpaceSolver

    rank, world, local = dist_env()
    dist = init_dist(world, local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = args.config
    w, pos_np, q_np = workloads.generate(cfg)
    basis = build_pswf(solve_bandwidth(w.delta))
    window = tabulate_window(basis, w.P)
    s = SlabKSpaceSolver(w.h, w.M, w.P, basis, window, w.r_c, precision=args.precision,
                         capacity=w.n // max(world, 1) + w.n // 8)
    mine = s.owned(pos_np)
    pos = torch.as_tensor(pos_np[mine], device=dev)
    q = torch.as_tensor(q_np[mine], device=dev)
    n_mine = int(mine.sum())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    K, W = args.steps, args.warmup
    stats = {}

    # one CUDA graph per rank and path; eager stream-ordered steps otherwise
    capture = "cuda_graph"
    try:
        g_fp, o7, F = s.graphed(pos, q, True)
        g_po, o7_po, _ = s.graphed(pos, q, False)
        step_fp, step_po = g_fp.replay, g_po.replay
    except Exception as exc:   # NCCL capture unavailable: keep the eager step
        capture = f"eager ({type(exc).__name__})"
        o7 = torch.empty(7, dtype=torch.float64, device=dev)
        F = torch.empty((n_mine, 3), dtype=torch.float64, device=dev)
        step_fp = lambda: s.evaluate_device(pos, q, True, o7, F)         # noqa: E731
        step_po = lambda: s.evaluate_device(pos, q, False, o7, None)     # noqa: E731

    # public-API end to end: this rank's charges from pinned host buffers,
    # the step, forces and the 7 sums back to pinned host memory
    h_pos = torch.empty((n_mine, 3), dtype=torch.float64).pin_memory()
    h_q = torch.empty(n_mine, dtype=torch.float64).pin_memory()
    h_F = torch.empty((n_mine, 3), dtype=torch.float64).pin_memory()
    h_7 = torch.empty(7, dtype=torch.float64).pin_memory()
    h_pos.copy_(torch.as_tensor(pos_np[mine]))
    h_q.copy_(torch.as_tensor(q_np[mine]))

    def step_e2e():
        pos.copy_(h_pos, non_blocking=True)
        q.copy_(h_q, non_blocking=True)
        step_fp()
        h_F.copy_(F, non_blocking=True)
        h_7.copy_(o7, non_blocking=True)

    def timed(fn, tag, k=K, wu=W):
        return timed_steps(fn, k, wu, flush, stream, dist, dev, stats, tag)

    near = None
    if args.near:
        from paper_2601_00161_b200 import Cell, SplitKernel
        from paper_2601_00161_b200.realspace import build_pair_table
        from paper_2601_00161_b200.slab_near import CudaNearOps, SlabNearField
        kern = SplitKernel(basis=basis, r_c=w.r_c)
        sn = SlabNearField.from_kspace(s, w.r_c, CudaNearOps(kern, build_pair_table(kern),
                                                             Cell(np.asarray(w.h, float))))
        sn.ops.plan.reserve(pos.shape[0] + pos.shape[0] // 2)

    quiet_host_pools()
    with ClockSampler(local) as clk:
        ms_fp = timed(step_fp, "force_pressure")
        ms_po = timed(step_po, "pressure_only")
        ms_e2e = timed(step_e2e, "e2e")
        if args.near:
            ms_near = timed(lambda: sn.evaluate(pos, q), "near_field", max(3, min(K, 5)), 2)
            near = {"ms_per_step": ms_near, "value": w.n / (ms_near * 1e-3), "unit": UNIT,
                    "what": "slab near field (ghost all-to-all, slab-local pair sums, "
                            "rank-ordered reduction), slab_near.SlabNearField"}
    clocks = clk.summary()
    assert np.isfinite(h_F.numpy()).all() and np.isfinite(h_7.numpy()).all()

    # per-kernel profile of this rank's slab plan (bin, spread, combine, gather)
    plan, spectral = s.ops.plan, s.ops.spectral
    prof = {}
    for _ in range(3):
        flush.zero_()
        plan.set_profiling(True)           # resets the event list and launch count
        spectral.set_profiling(True)
        s.evaluate_device(pos, q, True)
        for name, t in plan.profile():
            prof[name] = prof.get(name, 0.0) + t / 3
        launches = plan.launches_last_step() + spectral.launches_last_step()
    plan.set_profiling(False)
    spectral.set_profiling(False)
    hbm_peak, peak_kind = measured_peaks()
    real_b = 8 if args.precision == "fp64" else 4
    alg = algorithmic(w, n_mine, plan.tables.band, real_b)
    roof = None
    kern_t = {k: v for k, v in prof.items() if k in ("gather", "spread")}
    if kern_t:
        dom = max(kern_t, key=kern_t.get)
        t = kern_t[dom] * 1e-3
        ach = alg[dom]["bytes"] / t / 1e9
        fp64 = probe_fp64_tflops()
        roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 2), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(ach / hbm_peak, 4), "traffic": None,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs",
                "avg_launch_ms": round(kern_t[dom], 5),
                "fp64": {"achieved_tflops": round(alg[dom]["flops"] / t / 1e12, 3),
                         "peak_tflops": round(fp64, 2)},
                "scope": f"rank {rank}'s slab plan ({n_mine} charges)"}
    h2d = int((h_pos.numel() + h_q.numel()) * 8)
    d2h = int((h_F.numel() + h_7.numel()) * 8)
    line = {"metric": METRIC, "value": w.n / (ms_fp * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms_fp,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (seeded config recipe, SURVEY §8(d.1))",
            "config": {"workload": w.name, "n_charges": w.n, "grid": list(w.M), "P": w.P,
                       "delta": w.delta, "r_c": w.r_c, "cell_type": w.cell_type,
                       "parallelism": f"zslab{world}", "precision": args.precision,
                       "l2": "flushed between timed steps (256 MB write)",
                       "statistic": "median step time, max over ranks",
                       "capture": capture},
            "pressure_only": {"value": w.n / (ms_po * 1e-3), "unit": UNIT,
                              "ms_per_step": ms_po},
            "e2e": {"value": w.n / (ms_e2e * 1e-3), "unit": UNIT, "ms_per_step": ms_e2e,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "SlabKSpaceSolver step per rank from pinned host buffers "
                           "(bytes are rank 0's share)"},
            "gpu_launches": int(launches * K), "gpu_launches_per_step": launches,
            "timing": dict(stats, statistic="median over the K timed steps, max over ranks"),
            "clocks": clocks, "roofline": roof,
            "kernel_ms": {k: round(v, 5) for k, v in prof.items()}}
    if near is not None:
        line["near_field"] = near
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_port(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    _, world, _ = dist_env()
    if args.impl == "reference":
        run_reference(args)
    elif args.slab or (world > 1 and not args.replicas):
        run_slab(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
