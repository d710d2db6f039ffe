"""Solver composition on the B200 (reference: prolate_ewald/evaluate.py).

:class:`KSpaceSolver` is the fused product entry point: positions and charges
(CUDA tensors, or host arrays that are copied in) -> far-field energy, the
full 3x3 pressure tensor and ik forces in one device pipeline (bin, spread,
1 forward FFT, fused scale/reduce, and for forces 3 inverse FFTs + gather).
:class:`CoulombSolver` mirrors ``evaluate.CoulombSolver`` (evaluate.py:81-152):
near field (realspace.py, on the device), far field, self energy and the
uniform background.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import ctypes as C
import os

from . import _lib
from .cells import CellType, infer_cell_type
from .errors import ParameterError
from .kernel import SplitKernel, background_correction, self_energy
from .mesh import ModeWorkspace, TransformProvider, plan_grid
from .plan import EspPlan, PlanGraph, out7_to_tensor
from .realspace import NearFieldPlan, build_pair_table, out7_to_pressure
from .pswf import build_pswf, solve_bandwidth
from .system import Cell, check_cutoff


@dataclass(frozen=True)
class EwaldParameters:
    """Accuracy knobs (evaluate.py:29-57) plus the B200 execution options."""

    r_c: float
    delta_split: float = 1e-6
    delta_spread: float | None = None
    P: int | None = None
    oversampling: float = 1.0
    prefactor: float = 1.0
    force_mode: str = "ik"
    fixed_M: tuple | None = None
    precision: str = "fp64"
    deterministic: bool = True
    cell_type: str | None = None

    def resolved(self):
        if self.r_c <= 0:
            raise ParameterError("cutoff r_c must be positive")
        if self.force_mode not in ("ik", "analytic"):
            raise ParameterError(f"unknown force mode {self.force_mode!r}")
        if self.precision not in ("fp64", "fp32"):
            raise ParameterError(f"unknown precision {self.precision!r}")
        d_split = float(self.delta_split)
        d_spread = d_split if self.delta_spread is None else float(self.delta_spread)
        P = self.P if self.P is not None else int(np.ceil(-np.log10(d_split))) + 1
        return d_split, d_spread, int(P)


@dataclass
class KSpaceResult:
    energy: float
    pressure: np.ndarray            # (3,3)
    forces: object = None           # (N,3) tensor/array or None
    cell_type: CellType | None = None

    @property
    def reported_pressure(self):
        """The pressure quantities the cell type couples to."""
        ct = self.cell_type or CellType.TRICLINIC
        return ct.reduce(self.pressure)


def _to_device(x, dtype=torch.float64):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    npd = np.int64 if dtype == torch.int64 else np.float64
    return torch.as_tensor(np.ascontiguousarray(x, dtype=npd), device="cuda").to(dtype)


class KSpaceSolver:
    """Far-field solver bound to one cell (M pinned by ``fixed_M`` or planned)."""

    def __init__(self, cell, params: EwaldParameters, capacity: int = 1 << 16):
        d_split, d_spread, P = params.resolved()
        self.params = params
        h = np.asarray(cell.h if hasattr(cell, "h") else cell, dtype=float)
        self.cell = Cell(h)
        self.cell_type = CellType(params.cell_type) if params.cell_type else \
            infer_cell_type(self.cell.h)
        self.cell_type.validate(self.cell.h)
        check_cutoff(self.cell, params.r_c)
        basis = build_pswf(solve_bandwidth(d_split))
        spread = basis if abs(d_spread - d_split) <= 1e-300 else build_pswf(solve_bandwidth(d_spread))
        self.kern = SplitKernel(basis=basis, r_c=params.r_c)
        self.spec = plan_grid(self.cell, self.kern, delta_spread=d_spread, P=P,
                              oversampling=params.oversampling, spread_basis=spread,
                              fixed_M=params.fixed_M,
                              allow_triclinic=self.cell_type is CellType.TRICLINIC)
        self.plan = EspPlan(self.spec.M, P, self.spec.window, basis, params.r_c,
                            spread=spread, precision=params.precision,
                            deterministic=params.deterministic, capacity=capacity)
        self.plan.set_cell(self.cell.h)

    @property
    def M(self):
        return self.spec.M

    def rebind_cell(self, cell, fixed_M=None):
        """Re-plan the mesh for a new cell (evaluate.py:99-112).

        ``fixed_M`` pins the grid counts (the barostat's cheap rebind: the
        per-cell tables are re-uploaded, no host re-plan).  Without it the
        grid is re-planned like the reference: ``params.fixed_M`` if the
        solver was built with one, else the automatic plan from the
        oversampling factor.  When the counts change the device plan is
        rebuilt.  The window table and bases persist.  CUDA graphs captured
        before a rebind refuse to replay (``PlanGraph``)."""
        h = np.asarray(cell.h if hasattr(cell, "h") else cell, dtype=float)
        new = Cell(h)
        self.cell_type.validate(new.h)
        check_cutoff(new, self.params.r_c)
        target = fixed_M if fixed_M is not None else self.params.fixed_M
        spec = plan_grid(new, self.kern, delta_spread=self.spec.delta_spread,
                         P=self.spec.P, oversampling=self.params.oversampling,
                         spread_basis=self.spec.spread_basis,
                         fixed_M=tuple(target) if target is not None else None,
                         window=self.spec.window,
                         allow_triclinic=self.cell_type is CellType.TRICLINIC)
        if tuple(spec.M) != tuple(self.spec.M):
            old = self.plan
            self.plan = EspPlan(spec.M, spec.P, spec.window, self.kern.basis, self.params.r_c,
                                spread=spec.spread_basis, precision=self.params.precision,
                                deterministic=self.params.deterministic,
                                capacity=old.capacity)
            self.plan.generation = old.generation + 1
            old.generation += 1          # graphs on the old plan are stale
            old.close()
        self.spec = spec
        self.cell = new
        self.plan.set_cell(new.h)

    def evaluate_device(self, positions: torch.Tensor, charges: torch.Tensor,
                        want_forces: bool = True, out7=None, forces=None, stream=None):
        """Device-only step: returns (out7 tensor, forces tensor|None) without
        synchronising.  out7 = [E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz] (prefactor 1)."""
        return self.plan.evaluate(positions, charges, want_forces, out7, forces, stream,
                                  analytic=self.params.force_mode == "analytic")

    def graphed(self, positions: torch.Tensor, charges: torch.Tensor,
                want_forces: bool = True, out7=None, forces=None):
        """Capture the device step on fixed buffers into a CUDA graph.
        Returns (graph, out7, forces); ``graph.replay()`` recomputes them after
        the caller updates ``positions`` / ``charges`` in place."""
        n = positions.shape[0]
        out7 = out7 if out7 is not None else torch.empty(7, dtype=torch.float64,
                                                         device=positions.device)
        if want_forces and forces is None:
            forces = torch.empty((n, 3), dtype=torch.float64, device=positions.device)
        g = self.plan.graph(positions, charges, want_forces, out7, forces,
                            analytic=self.params.force_mode == "analytic")
        return g, out7, forces

    def host_stepper(self, n: int, want_forces: bool = True):
        """Public host-buffer path: pinned host inputs -> device step ->
        pinned host outputs, captured as one CUDA graph (H2D copies, the
        k-space step and D2H copies).  Returns an object with pinned
        ``positions`` (N,3), ``charges`` (N,), ``forces`` (N,3), ``out7`` (7,)
        and ``step()`` (replay + synchronise)."""
        return _HostStepper(self, n, want_forces)

    def evaluate(self, positions, charges, want_forces: bool = True,
                 want_pressure: bool = True) -> KSpaceResult:
        host = not isinstance(positions, torch.Tensor)
        pos = _to_device(positions)
        q = _to_device(charges)
        out7, F = self.plan.evaluate(pos, q, want_forces,
                                     analytic=self.params.force_mode == "analytic")
        E, Pt = out7_to_tensor(out7)
        pref = self.params.prefactor
        if want_forces:
            F = F * pref
            if host:
                F = F.cpu().numpy()
        return KSpaceResult(energy=pref * E, pressure=pref * Pt if want_pressure else None,
                            forces=F if want_forces else None, cell_type=self.cell_type)

    def local_pressure(self, positions, charges):
        """Per-particle far-field pressure tensors (N,3,3), prefactored
        (evaluate.py:147-152, mesh.py:353-379)."""
        host = not isinstance(positions, torch.Tensor)
        pos, q = _to_device(positions), _to_device(charges)
        self.plan.evaluate(pos, q, want_forces=False)
        out = self.plan.local_pressure(pos.shape[0]) * self.params.prefactor
        return out.cpu().numpy() if host else out

    def pressure_only(self, positions, charges):
        r = self.evaluate(positions, charges, want_forces=False)
        return r.energy, r.pressure


def host_force_chunks() -> int:
    """Original-index ranges the host-buffer step gathers and copies out in
    (ESP_HOST_CHUNKS, default 2; 1 = one copy after the gather)."""
    return max(1, min(8, int(os.environ.get("ESP_HOST_CHUNKS", "2"))))


class _HostStepper:
    def __init__(self, solver: "KSpaceSolver", n: int, want_forces: bool):
        f64 = torch.float64
        # page-locked buffers from the library's cudaHostAlloc (H2D from
        # torch's pinned allocator measured ~4x slower on the B200 box);
        # zero-initialised: the graph warm-up runs before the caller fills them
        self._bufs = [_lib.HostBuffer(sh) for sh in ((n, 3), (n,), (n, 3), (7,))]
        self.positions, self.charges, self.forces, self.out7 = (b.tensor for b in self._bufs)
        self.positions.zero_()
        self.charges.zero_()
        self._d_pos = torch.empty((n, 3), dtype=f64, device="cuda")
        self._d_q = torch.empty(n, dtype=f64, device="cuda")
        self._d_out7 = torch.empty(7, dtype=f64, device="cuda")
        self._d_F = torch.empty((n, 3), dtype=f64, device="cuda") if want_forces else None
        self.want_forces = want_forces
        self.h2d_bytes = (3 * n + n) * 8
        self.d2h_bytes = (3 * n * 8 if want_forces else 0) + 7 * 8

        # copies as stream-ordered cudaMemcpyAsync (copy-engine DMA once
        # captured in the graph)
        L = _lib.lib()

        def copy(dst, src):
            s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(L.esp_copy_async(C.c_void_p(dst.data_ptr()), C.c_void_p(src.data_ptr()),
                                        src.numel() * src.element_size(), s), "esp_copy_async")

        # the charge copy runs on a forked stream and overlaps the binning of
        # the positions (the step waits on it before its first charge read)
        qside = torch.cuda.Stream()
        qev = torch.cuda.Event()
        self._qside, self._qev = qside, qev

        # the force copy-out is issued by the step itself, range by range as
        # the gather finishes each original-index range (esp_set_host_forces)
        handle = solver.plan._handle
        chunks = host_force_chunks()

        # Large systems: positions first, alone on the link, so the binning
        # starts as soon as they are in; the charges follow on the side stream
        # while the positions are binned (two concurrent H2D copies share the
        # link and both finish late: config-4 e2e 15.5 -> 14.8 ms).  Small
        # systems are latency-bound and keep both copies in flight together
        # (config 1: 0.37 against 0.39 ms).
        serial = n >= 500_000

        def pre():
            main = torch.cuda.current_stream()
            if serial:
                copy(self._d_pos, self.positions)
            qside.wait_stream(main)
            with torch.cuda.stream(qside):
                copy(self._d_q, self.charges)
                qev.record(qside)
            if not serial:
                copy(self._d_pos, self.positions)
            _lib.check(L.esp_set_charges_event(handle, C.c_void_p(qev.cuda_event)),
                       "esp_set_charges_event")
            if want_forces:
                _lib.check(L.esp_set_host_forces(handle, C.c_void_p(self.forces.data_ptr()),
                                                 chunks), "esp_set_host_forces")

        def post():
            if want_forces:
                _lib.check(L.esp_set_host_forces(handle, None, 0), "esp_set_host_forces")
            copy(self.out7, self._d_out7)

        self.graph = solver.plan.graph(self._d_pos, self._d_q, want_forces, self._d_out7,
                                       self._d_F, pre=pre, post=post,
                                       analytic=solver.params.force_mode == "analytic")

    def launch(self):
        """Enqueue one step (no host synchronisation)."""
        self.graph.replay()

    def step(self):
        self.graph.replay()
        torch.cuda.current_stream().synchronize()
        return self.out7, (self.forces if self.want_forces else None)


@dataclass
class EnergyBreakdown:
    """Electrostatic outputs with per-term energies (evaluate.py:60-77)."""

    u_near: float
    u_far: float
    u_self: float
    u_background: float
    forces: np.ndarray | None = None
    pressure: np.ndarray | None = None
    pair_count: int = 0

    @property
    def energy(self) -> float:
        return self.u_near + self.u_far + self.u_self + self.u_background


class CoulombSolver:
    """evaluate.CoulombSolver (evaluate.py:81-152) on the B200.

    Near field (device cell list or a caller NeighborList + pair table,
    csrc/esp_near.cu), far field (the k-space pipeline), self energy and the
    uniform-background terms compose exactly as evaluate.py:114-144.  Host
    ``ParticleSystem`` inputs return numpy forces; CUDA-tensor systems keep
    them on the device."""

    def __init__(self, cell, params: EwaldParameters):
        self.params = params
        self.kspace = KSpaceSolver(cell, params)
        self.kern = self.kspace.kern
        self.cell = self.kspace.cell
        self.pair_table = build_pair_table(self.kern)
        self.near = NearFieldPlan(self.kern, self.pair_table)
        self.near.set_cell(self.cell)
        # transform counters (evaluate.py:92): evaluate() counts the forward
        # transform and the force / local-pressure inverse transforms here
        self.provider = TransformProvider()
        self._modes = None

    @property
    def spec(self):
        return self.kspace.spec

    @property
    def modes(self):
        """ModeWorkspace of the current spec and cell (evaluate.py:112)."""
        if self._modes is None or self._modes._spec is not self.spec:
            self._modes = ModeWorkspace(self.spec, self.kern, self.cell)
        return self._modes

    def rebind_cell(self, cell, fixed_M=None):
        """Re-plan for a new cell; bases and pair table persist
        (evaluate.py:99-112).  ``fixed_M=None`` re-plans the grid counts."""
        self.kspace.rebind_cell(cell, fixed_M)
        self.cell = self.kspace.cell
        self.near.set_cell(self.cell)

    def evaluate_device(self, positions: torch.Tensor, charges: torch.Tensor,
                        want_forces: bool = True, neighbors=None, stream=None):
        """Device step without synchronising: (out7_far, out7_near, stats, F)
        with F = far + near forces (prefactor 1) or None."""
        out7_far, F = self.kspace.evaluate_device(positions, charges, want_forces,
                                                  stream=stream)
        if neighbors is None:
            out7_near, Fn, stats = self.near.evaluate(positions, charges, forces=F,
                                                      accumulate=want_forces, stream=stream)
        else:
            out7_near, Fn, stats = self.near.evaluate_pairs(
                positions, charges, _to_device(neighbors.i, torch.int64),
                _to_device(neighbors.j, torch.int64), forces=F, accumulate=want_forces,
                stream=stream)
        return out7_far, out7_near, stats, (F if want_forces else None)

    def graphed(self, positions: torch.Tensor, charges: torch.Tensor,
                want_forces: bool = True):
        """Capture the whole device step (near and far field) into one CUDA
        graph on fixed buffers.  The near-field pair sum and the k-space
        pipeline run on two streams of the graph and their forces are summed
        at the end.  Returns (graph, outputs) with outputs = dict(out7_far,
        out7_near, stats, forces); ``graph.replay()`` recomputes them after
        the caller updates ``positions`` / ``charges`` in place.  Energies and
        forces are prefactor 1 (evaluate() applies the prefactor)."""
        n = positions.shape[0]
        dev = positions.device
        f64 = torch.float64
        out = {"out7_far": torch.empty(7, dtype=f64, device=dev),
               "out7_near": torch.empty(7, dtype=f64, device=dev),
               "stats": torch.empty(4, dtype=torch.int64, device=dev),
               "forces": torch.empty((n, 3), dtype=f64, device=dev) if want_forces else None}
        f_far = torch.empty((n, 3), dtype=f64, device=dev) if want_forces else None
        f_near = torch.empty((n, 3), dtype=f64, device=dev)
        self.near.reserve(n)
        self.kspace.plan.ensure_capacity(n)
        side = torch.cuda.Stream()

        def body():
            main = torch.cuda.current_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.near.evaluate(positions, charges, forces=f_near, out7=out["out7_near"],
                                   stats=out["stats"])
            self.kspace.evaluate_device(positions, charges, want_forces, out["out7_far"], f_far)
            main.wait_stream(side)
            if want_forces:
                torch.add(f_far, f_near, out=out["forces"])

        warm = torch.cuda.Stream()
        warm.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(warm):
            body()
        torch.cuda.current_stream().wait_stream(warm)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        kp = self.kspace.plan
        before = kp.counters()
        with torch.cuda.graph(g):
            body()
        torch.cuda.synchronize()
        after = kp.counters()
        return PlanGraph(g, [kp, self.near],
                         counted=(kp, after[0] - before[0], after[1] - before[1])), out

    def evaluate(self, sys, want_forces: bool = True, want_pressure: bool = True,
                 neighbors=None) -> EnergyBreakdown:
        if not np.allclose(np.asarray(sys.cell.h), self.cell.h):
            raise ParameterError("system cell differs from the solver's cell; "
                                 "call rebind_cell first")
        pref = self.params.prefactor
        host = not isinstance(sys.positions, torch.Tensor)
        pos = _to_device(sys.positions)
        q = _to_device(sys.charges)
        o_far, o_near, stats, F = self.evaluate_device(pos, q, want_forces, neighbors)
        self.provider.forward_count += 1
        if want_forces:
            self.provider.inverse_count += 1 if self.params.force_mode == "analytic" else 3
        st = stats.cpu().numpy()
        NearFieldPlan.check_stats(st)
        e_far, p_far = out7_to_tensor(o_far)
        e_near, p_near = out7_to_pressure(o_near)
        qh = q.cpu().numpy()
        u_self = self_energy(self.kern, qh)
        u_cb, u_bb, p_corr = background_correction(self.kern, float(qh.sum()), self.cell.volume)
        out = EnergyBreakdown(u_near=pref * e_near, u_far=pref * e_far, u_self=pref * u_self,
                              u_background=pref * (u_cb + u_bb), pair_count=int(st[0]))
        if want_forces:
            F = F * pref
            out.forces = F.cpu().numpy() if host else F
        if want_pressure:
            out.pressure = pref * (p_near + p_far + p_corr)
        return out


def _coulomb_local_pressure(self, sys):
    """Per-particle far-field pressure tensors, prefactored (evaluate.py:147-152):
    one forward and six inverse transforms."""
    self.provider.forward_count += 1
    self.provider.inverse_count += 6
    return self.kspace.local_pressure(sys.positions, sys.charges)


CoulombSolver.local_pressure = _coulomb_local_pressure


def evaluate_system(sys, params: EwaldParameters, want_forces=True, want_pressure=True):
    return CoulombSolver(sys.cell, params).evaluate(sys, want_forces, want_pressure)


def kinetic_pressure(sys) -> np.ndarray:
    """(1/V) sum_i p_i p_i^T / m_i (evaluate.py:163-166)."""
    p = np.asarray(sys.momenta, dtype=float)
    m = np.asarray(sys.masses, dtype=float)
    return np.einsum("ia,ib->ab", p / m[:, None], p) / sys.cell.volume
