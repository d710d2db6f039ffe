"""Near field (real-space pair sum) on the B200 — reference:
prolate_ewald/realspace.py and system.build_cell_list.

``short_range`` keeps the reference signature and result type.  The pair sum
runs in ``libesp_b200.so`` (csrc/esp_near.cu):

* ``neighbors=None``: the device cell list (system.py:144-222 semantics:
  every unordered pair within r_c under the minimum image), fused with the
  energy / force / pressure pass (realspace.py:115-157) — no pair list is
  materialised.
* a :class:`NeighborList`: the listed pairs exactly as the reference sums
  them (minimum image per pair, r <= r_c filter, SingularPairError).

Pair values come from the :class:`PairTable` (``table=``) or, without one,
from the exact Legendre series (kernel.py:41-97), both evaluated on the
device in the reference's operation order.  ``build_pair_table`` restates
realspace.py:70-112 on the host (setup).  There is no CPU fallback for the
pair sum: without the library or a GPU the entry points raise.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
from scipy.interpolate import CubicSpline, PPoly

from . import _lib
from .errors import RealspaceError, SingularPairError
from .kernel import SplitKernel, cumint_coeffs, far_field, fn_weight
from .system import Cell, NeighborList, check_cutoff


@dataclass(frozen=True)
class ShortRangeResult:
    """realspace.py:24-28."""

    energy: float
    forces: object          # (N,3) numpy array (host inputs) or CUDA tensor
    pressure: np.ndarray    # (3,3)
    pair_count: int


@dataclass(frozen=True)
class PairTable:
    """Smooth polynomial below r_in, cubic spline above (realspace.py:29-67).

    ``near_field`` / ``fn_weight`` evaluate the table on the host for
    inspection and tests, as the reference's methods do; the pair sum itself
    evaluates the same pieces on the device."""

    r_in: float
    r_c: float
    smooth_coeffs: np.ndarray
    fn_coeffs: np.ndarray
    smooth_spline: PPoly
    fn_spline: PPoly
    resolution: int

    def near_field(self, r):
        r = np.asarray(r, dtype=float)
        out = np.empty_like(r)
        lo = r <= self.r_in
        out[lo] = 1.0 / r[lo] - np.polynomial.polynomial.polyval(r[lo], self.smooth_coeffs)
        hi = ~lo
        out[hi] = 1.0 / r[hi] - self.smooth_spline(np.minimum(r[hi], self.r_c))
        out[r >= self.r_c] = 0.0
        return out

    def fn_weight(self, r):
        r = np.asarray(r, dtype=float)
        out = np.empty_like(r)
        lo = r <= self.r_in
        out[lo] = np.polynomial.polynomial.polyval(r[lo], self.fn_coeffs)
        hi = ~lo
        out[hi] = self.fn_spline(np.minimum(r[hi], self.r_c))
        out[r > self.r_c] = 0.0
        return out


def build_pair_table(kern: SplitKernel, r_in: float | None = None,
                     resolution: int = 4096, order: int = 8) -> PairTable:
    """Tabulate the near field and its force weight (realspace.py:70-112):
    degree-``order`` fits of the smooth pieces on Chebyshev nodes in
    [0, r_in], r_in halved until the fit reaches 1e-11 of far_field(0);
    not-a-knot cubic splines on ``resolution`` uniform knots in [r_in, r_c]."""
    r_c = kern.r_c
    if r_in is None:
        r_in = 0.1 * r_c
    if not (0.0 < r_in < r_c):
        raise RealspaceError(f"inner cutoff r_in={r_in} not in (0, r_c)")
    s = np.cos(np.pi * (2.0 * np.arange(order + 1) + 1.0) / (2.0 * (order + 1)))
    for _ in range(12):
        nodes = 0.5 * r_in * (s + 1.0)
        smooth = np.polynomial.Polynomial.fit(nodes, far_field(kern, nodes), order,
                                              domain=[0.0, r_in]).convert().coef
        fnc = np.polynomial.Polynomial.fit(nodes, fn_weight(kern, np.maximum(nodes, 1e-300)),
                                           order, domain=[0.0, r_in]).convert().coef
        probe = np.linspace(1e-6 * r_c, r_in, 512)
        err = np.max(np.abs(np.polynomial.polynomial.polyval(probe, smooth)
                            - far_field(kern, probe))) / far_field(kern, 0.0)
        if err <= 1e-11:
            break
        r_in *= 0.5
    else:
        raise RealspaceError("inner-cutoff polynomial fit did not converge")
    knots = np.linspace(r_in, r_c, resolution)
    sp = CubicSpline(knots, far_field(kern, knots))
    fsp = CubicSpline(knots, fn_weight(kern, knots))
    pad = np.zeros(order + 1)
    pad[: smooth.size] = smooth
    fpad = np.zeros(order + 1)
    fpad[: fnc.size] = fnc
    return PairTable(r_in=float(r_in), r_c=r_c, smooth_coeffs=pad, fn_coeffs=fpad,
                     smooth_spline=sp, fn_spline=fsp, resolution=int(resolution))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class NearFieldPlan:
    """Device near-field plan (``esp_near_*``) for one kernel / table / reach.

    ``evaluate`` (cell list) and ``evaluate_pairs`` (explicit list) run
    asynchronously on the current stream and return device tensors:
    out7 = [E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz] (prefactor 1), forces (N,3) in
    input order, stats = [pair count, first coincident pair or -1, first
    out-of-range pair or -1, directed pair count]."""

    def __init__(self, kern: SplitKernel | None, table: PairTable | None = None,
                 skin: float = 0.0, capacity: int = 1 << 16, cell_div: int = 0,
                 r_c: float | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("the near-field pair sum needs a CUDA device (no CPU fallback)")
        self.kern, self.table = kern, table
        self.r_c = float(kern.r_c if kern is not None else r_c)
        self.reach = self.r_c + float(skin)
        L = _lib.lib()
        if kern is not None:
            b = kern.basis
            leg = np.ascontiguousarray(b.legendre_coeffs, dtype=np.float64)
            cum = np.ascontiguousarray(cumint_coeffs(b), dtype=np.float64)
            C0 = float(b.C0)
        else:  # pair enumeration only (build_cell_list): no pair values
            leg, cum, C0 = np.ones(1), np.array([0.0, 1.0]), 1.0
        d = _lib.NearDesc()
        d.r_c = self.r_c
        d.reach = self.reach
        d.use_table = 1 if table is not None else 0
        keep = [leg, cum]
        if table is not None:
            if abs(table.r_c - self.r_c) > 0.0:
                raise RealspaceError("pair table cutoff differs from the kernel's r_c")
            sp, fsp = table.smooth_spline, table.fn_spline
            if sp.c.shape[0] != 4 or fsp.c.shape != sp.c.shape or not np.array_equal(sp.x, fsp.x):
                raise RealspaceError("pair table splines must be cubic on shared knots")
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                    (table.smooth_coeffs, table.fn_coeffs, sp.x, sp.c, fsp.c)]
            keep += arrs
            d.r_in = float(table.r_in)
            d.poly_order = int(arrs[0].size - 1)
            d.h_smooth_poly, d.h_fn_poly = _dp(arrs[0]), _dp(arrs[1])
            d.n_knots = int(arrs[2].size)
            d.h_knots, d.h_smooth_spline, d.h_fn_spline = _dp(arrs[2]), _dp(arrs[3]), _dp(arrs[4])
        d.n_legendre, d.h_legendre = int(leg.size), _dp(leg)
        d.n_cumint, d.h_cumint = int(cum.size), _dp(cum)
        d.C0 = C0
        d.max_particles = int(max(capacity, 1))
        d.cell_div = int(cell_div)
        h = C.c_void_p()
        _lib.check(L.esp_near_create(C.byref(d), C.byref(h)), "esp_near_create")
        self._h = h
        self._L = L
        self.cell: Cell | None = None
        self._n_pairs_cap = 0
        self._n_cap = int(max(capacity, 1))
        self.generation = 0       # bumps on set_cell / reserve (captured graphs go stale)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.esp_near_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def set_cell(self, cell) -> None:
        """Bind the cell (GeometryError as check_cutoff when reach is too large)."""
        cell = cell if isinstance(cell, Cell) else Cell(np.asarray(cell, dtype=float))
        check_cutoff(cell, self.reach)
        h = np.ascontiguousarray(cell.h, dtype=np.float64)
        hinv = np.ascontiguousarray(np.linalg.inv(cell.h), dtype=np.float64)
        _lib.check(self._L.esp_near_set_cell(self._h, _dp(h), _dp(hinv),
                                             1 if cell.is_orthorhombic else 0,
                                             float(cell.volume)), "esp_near_set_cell")
        self.cell = cell
        self.generation += 1

    def reserve(self, n: int, n_pairs: int = 0) -> None:
        if int(n) > self._n_cap or int(n_pairs) > self._n_pairs_cap:
            self.generation += 1  # buffers may be re-allocated
        _lib.check(self._L.esp_near_reserve(self._h, int(n), int(n_pairs)), "esp_near_reserve")
        self._n_pairs_cap = max(self._n_pairs_cap, int(n_pairs))
        self._n_cap = max(self._n_cap, int(n))

    def info(self) -> dict:
        a = (C.c_int64 * 8)()
        _lib.check(self._L.esp_near_info(self._h, a), "esp_near_info")
        return {"cells": (a[0], a[1], a[2]), "stencil": a[3], "capacity": a[4],
                "launches": a[5], "cells_per_reach": a[6], "table": bool(a[7])}

    @staticmethod
    def _outputs(n, dev, forces, out7, stats):
        if forces is None:
            forces = torch.empty((n, 3), dtype=torch.float64, device=dev)
        if out7 is None:
            out7 = torch.empty(7, dtype=torch.float64, device=dev)
        if stats is None:
            stats = torch.empty(4, dtype=torch.int64, device=dev)
        return forces, out7, stats

    @staticmethod
    def _check_particles(pos, q):
        if pos.dtype != torch.float64 or q.dtype != torch.float64 or not pos.is_cuda:
            raise RealspaceError("positions / charges must be float64 CUDA tensors")
        if pos.dim() != 2 or pos.shape[1] != 3 or q.shape != (pos.shape[0],):
            raise RealspaceError("positions must be (N,3) and charges (N,)")
        if not (pos.is_contiguous() and q.is_contiguous()):
            raise RealspaceError("positions / charges must be contiguous")

    def evaluate(self, pos: torch.Tensor, q: torch.Tensor, forces=None, accumulate=False,
                 out7=None, stats=None, stream=None):
        """Cell-list pair sum (no synchronisation)."""
        if self.cell is None:
            raise RealspaceError("set_cell first")
        self._check_particles(pos, q)
        n = pos.shape[0]
        self.reserve(n)
        forces, out7, stats = self._outputs(n, pos.device, forces, out7, stats)
        rc = self._L.esp_near_evaluate(
            self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()), n,
            _lib.ESP_NEAR_ACCUMULATE if accumulate else 0, C.c_void_p(out7.data_ptr()),
            C.c_void_p(forces.data_ptr()), C.c_void_p(stats.data_ptr()), _stream(stream))
        _lib.check(rc, "esp_near_evaluate")
        return out7, forces, stats

    def evaluate_local(self, pos: torch.Tensor, q: torch.Tensor, n_owned: int, forces=None,
                       out7=None, stats=None, stream=None):
        """Slab-local pair sum: rows [0, n_owned) are this rank's particles,
        the rest ghosts (partners only).  forces has n_owned rows."""
        if self.cell is None:
            raise RealspaceError("set_cell first")
        self._check_particles(pos, q)
        n = pos.shape[0]
        self.reserve(n)
        forces, out7, stats = self._outputs(n_owned, pos.device, forces, out7, stats)
        rc = self._L.esp_near_evaluate_local(
            self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()), n, int(n_owned), 0,
            C.c_void_p(out7.data_ptr()), C.c_void_p(forces.data_ptr()),
            C.c_void_p(stats.data_ptr()), _stream(stream))
        _lib.check(rc, "esp_near_evaluate_local")
        return out7, forces, stats

    def evaluate_pairs(self, pos: torch.Tensor, q: torch.Tensor, i: torch.Tensor,
                       j: torch.Tensor, forces=None, accumulate=False, out7=None, stats=None,
                       stream=None):
        """Explicit pair list (int64 device tensors of equal length)."""
        if self.cell is None:
            raise RealspaceError("set_cell first")
        self._check_particles(pos, q)
        if i.dtype != torch.int64 or j.dtype != torch.int64 or i.shape != j.shape or i.dim() != 1:
            raise RealspaceError("pair indices must be equal-length int64 vectors")
        i, j = i.contiguous(), j.contiguous()
        n, m = pos.shape[0], i.shape[0]
        self.reserve(n, m)
        forces, out7, stats = self._outputs(n, pos.device, forces, out7, stats)
        rc = self._L.esp_near_evaluate_pairs(
            self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()), n,
            C.c_void_p(i.data_ptr()), C.c_void_p(j.data_ptr()), m,
            _lib.ESP_NEAR_ACCUMULATE if accumulate else 0, C.c_void_p(out7.data_ptr()),
            C.c_void_p(forces.data_ptr()), C.c_void_p(stats.data_ptr()), _stream(stream))
        _lib.check(rc, "esp_near_evaluate_pairs")
        return out7, forces, stats

    def build_pairs(self, pos: torch.Tensor, stream=None):
        """All unordered pairs within reach (i < j, sorted by (i, j)) as two
        int64 device tensors (system.build_cell_list semantics).  Synchronises."""
        if self.cell is None:
            raise RealspaceError("set_cell first")
        if pos.dtype != torch.float64 or not pos.is_cuda or pos.dim() != 2 or pos.shape[1] != 3:
            raise RealspaceError("positions must be an (N,3) float64 CUDA tensor")
        pos = pos.contiguous()
        m = C.c_int64()
        _lib.check(self._L.esp_near_build_pairs(self._h, C.c_void_p(pos.data_ptr()),
                                                pos.shape[0], C.byref(m), _stream(stream)),
                   "esp_near_build_pairs")
        out = torch.empty((2, int(m.value)), dtype=torch.int64, device=pos.device)
        _lib.check(self._L.esp_near_copy_pairs(self._h, C.c_void_p(out[0].data_ptr()),
                                               C.c_void_p(out[1].data_ptr()), _stream(stream)),
                   "esp_near_copy_pairs")
        return out[0], out[1]

    @staticmethod
    def check_stats(stats_host) -> None:
        """Raise the reference's errors from a host copy of ``stats``."""
        if int(stats_host[2]) != -1:
            raise RealspaceError(f"pair {int(stats_host[2])} indexes outside the particle set")
        if int(stats_host[1]) != -1:
            code = int(stats_host[1]) & ((1 << 64) - 1)
            a, b = code >> 32, code & 0xFFFFFFFF
            raise SingularPairError(f"coincident particles {a} and {b}")


def out7_to_pressure(out7) -> tuple[float, np.ndarray]:
    o = out7.detach().cpu().numpy() if isinstance(out7, torch.Tensor) else np.asarray(out7)
    P = np.array([[o[1], o[2], o[3]], [o[2], o[4], o[5]], [o[3], o[5], o[6]]])
    return float(o[0]), P


_PLANS: dict = {}


def _plan_for(kern: SplitKernel, table, cell: Cell, reach_skin: float = 0.0) -> NearFieldPlan:
    key = (id(kern), id(table), float(reach_skin))
    ent = _PLANS.get(key)
    if ent is None or ent[0] is not kern or ent[1] is not table:
        if len(_PLANS) > 8:
            _PLANS.clear()
        ent = (kern, table, NearFieldPlan(kern, table, skin=reach_skin))
        _PLANS[key] = ent
    plan = ent[2]
    if plan.cell is None or not np.array_equal(plan.cell.h, cell.h):
        plan.set_cell(cell)
    return plan


def _as_device(x, dtype):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda").to(dtype).contiguous()


_ENUM: dict = {}


def build_cell_list(sys, r_c: float, skin: float = 0.0) -> NeighborList:
    """Cell-list pair enumeration under the minimum-image convention
    (system.py:144-222): each unordered pair within r_c + skin exactly once,
    as i < j sorted by (i, j).  Runs on the device; host systems get numpy
    index arrays, CUDA-tensor systems device tensors."""
    check_cutoff(sys.cell, r_c)
    host = not isinstance(sys.positions, torch.Tensor)
    pos = _as_device(sys.positions, torch.float64)
    key = (float(r_c), float(skin))
    plan = _ENUM.get(key)
    if plan is None:
        if len(_ENUM) > 8:
            _ENUM.clear()
        plan = _ENUM[key] = NearFieldPlan(None, None, skin=skin, r_c=r_c)
    if plan.cell is None or not np.array_equal(plan.cell.h, sys.cell.h):
        plan.set_cell(sys.cell)
    i, j = plan.build_pairs(pos)
    if host:
        i, j = i.cpu().numpy(), j.cpu().numpy()
    return NeighborList(i=i, j=j, r_c=float(r_c), skin=float(skin))


def short_range(sys, kern: SplitKernel, neighbors: NeighborList | None = None,
                table: PairTable | None = None) -> ShortRangeResult:
    """Fused near-field pass: energy, forces and pressure (realspace.py:115-157).

    energy = sum_pairs q_i q_j N(r); force_i = sum_j q_i q_j F_N(r) dr / r^3;
    P = (1/V) sum_pairs q_i q_j F_N(r) dr (x) dr / r^3.  ``neighbors=None``
    uses the device cell list (pairs within r_c)."""
    host = not isinstance(sys.positions, torch.Tensor)
    pos = _as_device(sys.positions, torch.float64)
    q = _as_device(sys.charges, torch.float64)
    n = pos.shape[0]
    if neighbors is not None and neighbors.n_pairs == 0:
        z = np.zeros((n, 3)) if host else torch.zeros((n, 3), dtype=torch.float64,
                                                       device=pos.device)
        return ShortRangeResult(0.0, z, np.zeros((3, 3)), 0)
    plan = _plan_for(kern, table, sys.cell)
    if neighbors is None:
        out7, F, stats = plan.evaluate(pos, q)
    else:
        out7, F, stats = plan.evaluate_pairs(pos, q, _as_device(neighbors.i, torch.int64),
                                             _as_device(neighbors.j, torch.int64))
    st = stats.cpu().numpy()
    NearFieldPlan.check_stats(st)
    E, P = out7_to_pressure(out7)
    return ShortRangeResult(energy=E, forces=F.cpu().numpy() if host else F, pressure=P,
                            pair_count=int(st[0]))
