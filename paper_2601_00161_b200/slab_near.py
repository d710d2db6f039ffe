"""Multi-GPU near field over z-slabs (SURVEY §8(e) applied to row f3).

One process per GPU.  Rank r owns the particles of its slab of the cell's
fractional z axis (the same ownership as the k-space slab solver when the
bounds come from its plane layout, ``SlabNearField.from_kspace``).  One step:

1. ghosts    - each rank sends every other rank the owned particles lying
               within reach of that rank's slab (periodic fractional
               distance along z, reach / perpendicular width); counts first,
               then positions and charges, with all-to-all
2. pair sum  - the rank's device cell list over owned + ghost particles,
               with sums only for the owned particles (esp_near_evaluate_local:
               each directed pair is summed on its i particle's rank)
3. reduce    - the per-rank [E, P_ab, directed count] are all-gathered and
               added in rank order (bit-stable at a fixed GPU count)

Forces come back for the owned particles in the caller's order.  The
collectives run on torch tensors, so the same orchestration runs on CPU with
gloo for the decomposition tests; the local pair-sum backend is pluggable for
that purpose only (the product backend is :class:`CudaNearOps`).

Reference: realspace.short_range (realspace.py:115-157) over
system.build_cell_list pairs (system.py:144-222).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .errors import ParameterError
from .system import Cell, check_cutoff


class CudaNearOps:
    """Product backend: the device cell list (NearFieldPlan.evaluate_local)."""

    def __init__(self, kern, table, cell: Cell):
        from .realspace import NearFieldPlan
        self.plan = NearFieldPlan(kern, table)
        self.plan.set_cell(cell)

    def evaluate(self, pos: torch.Tensor, q: torch.Tensor, n_owned: int):
        """-> (out8 float64 tensor [E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz, directed
        count], forces (n_owned, 3), stats)."""
        out7, F, st = self.plan.evaluate_local(pos, q, n_owned)
        out8 = torch.cat([out7, st[3:4].to(torch.float64)])
        return out8, F, st


class SlabNearField:
    """Distributed near field for R ranks of a process group.

    ``bounds``: R + 1 increasing fractional z boundaries of the slabs
    (periodic; bounds[R] - bounds[0] == 1).  Rank r owns fractional z in
    [bounds[r], bounds[r + 1]) modulo 1."""

    def __init__(self, h, r_c: float, bounds, ops, group=None, skin: float = 0.0):
        self.group = group
        self.R = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.cell = Cell(np.asarray(h, dtype=float))
        self.reach = float(r_c) + float(skin)
        check_cutoff(self.cell, self.reach)
        b = np.asarray(bounds, dtype=float)
        if b.size != self.R + 1 or np.any(np.diff(b) <= 0) or abs(b[-1] - b[0] - 1.0) > 1e-12:
            raise ParameterError("slab bounds must be R + 1 increasing values spanning 1")
        self.bounds = b
        self.hinv = np.linalg.inv(self.cell.h)
        wz = self.cell.perpendicular_widths()[2]
        # fractional reach along z, widened by a rounding margin (extra ghosts
        # are harmless: they are partners only)
        self.dz = self.reach / wz * (1.0 + 1e-9) + 1e-12
        self.ops = ops

    @classmethod
    def from_kspace(cls, kslab, r_c: float, ops, group=None):
        """Ownership of a SlabKSpaceSolver: z anchor plane in [z0, z0 + nz)
        (floor(u) for even P, rint(u) for odd P)."""
        Mz = kslab.M[2]
        off = -0.5 if kslab.P % 2 else 0.0
        starts = list(kslab.layout.zstart) + [Mz]
        bounds = [(z + off) / Mz for z in starts]
        return cls(kslab.h, r_c, bounds, ops, group)

    def frac_z(self, pos: np.ndarray) -> np.ndarray:
        s = np.asarray(pos, dtype=float) @ self.hinv[2]
        return s - np.floor(s)

    def owner(self, pos: np.ndarray) -> np.ndarray:
        """Rank owning each position (fractional z in the rank's slab, mod 1)."""
        s = self.frac_z(pos)
        s = np.where(s < self.bounds[0], s + 1.0, s)
        s = np.where(s >= self.bounds[-1], s - 1.0, s)
        return np.clip(np.searchsorted(self.bounds, s, side="right") - 1, 0, self.R - 1)

    def _ghost_mask(self, s, d: int):
        """Positions (fractional z ``s``, numpy or torch) within reach of rank
        d's slab, periodically."""
        lo, hi = float(self.bounds[d]), float(self.bounds[d + 1])
        mod = torch if isinstance(s, torch.Tensor) else np
        best = None
        for k in (-1.0, 0.0, 1.0):
            t = s + k
            gap = mod.maximum(mod.maximum(lo - t, t - hi), mod.zeros_like(t))
            best = gap if best is None else mod.minimum(best, gap)
        return best <= self.dz

    def evaluate(self, pos: torch.Tensor, q: torch.Tensor):
        """pos (n_own, 3), q (n_own,): this rank's particles (as owner()
        assigns them).  Returns (E, P (3,3), forces (n_own, 3), pair count),
        E / P / count summed over all ranks (prefactor 1)."""
        n_own = pos.shape[0]
        ghosts_pos, ghosts_q = self._exchange(pos, q)
        allp = torch.cat([pos, ghosts_pos]).contiguous()
        allq = torch.cat([q, ghosts_q]).contiguous()
        out8, F, st = self.ops.evaluate(allp, allq, n_own)
        st_h = st.cpu().numpy() if isinstance(st, torch.Tensor) else np.asarray(st)
        if int(st_h[1]) != -1:
            from .errors import SingularPairError
            raise SingularPairError("coincident particles")
        parts = self._gather8(out8.to(torch.float64).reshape(8))
        tot = np.zeros(8)
        for r in range(self.R):            # rank order: bit-stable at fixed R
            tot += parts[r]
        E = float(tot[0])
        P = np.array([[tot[1], tot[2], tot[3]], [tot[2], tot[4], tot[5]],
                      [tot[3], tot[5], tot[6]]])
        return E, P, F, int(round(0.5 * tot[7]))

    # -- communication -------------------------------------------------------
    def _exchange(self, pos: torch.Tensor, q: torch.Tensor):
        """Ghost selection on the particles' device (torch ops), then counts
        and [x, y, z, q] rows by all-to-all."""
        if self.R == 1:
            z3 = torch.zeros((0, 3), dtype=pos.dtype, device=pos.device)
            return z3, torch.zeros(0, dtype=q.dtype, device=q.device)
        hz = torch.as_tensor(self.hinv[2], dtype=pos.dtype, device=pos.device)
        s = pos @ hz
        s = s - torch.floor(s)
        sel = [torch.nonzero(self._ghost_mask(s, d)).reshape(-1) if d != self.rank else
               torch.zeros(0, dtype=torch.int64, device=pos.device) for d in range(self.R)]
        idx = torch.cat(sel)
        send = torch.cat([pos[idx], q[idx].reshape(-1, 1)], dim=1).contiguous()
        cnt_in = torch.stack([torch.tensor(x.numel(), dtype=torch.int64) for x in sel]).to(
            pos.device)
        in_splits = [int(x.numel()) for x in sel]
        cnt_out = torch.empty_like(cnt_in)
        dist.all_to_all_single(cnt_out, cnt_in, group=self.group)
        out_splits = [int(v) for v in cnt_out.cpu().tolist()]
        recv = torch.empty((sum(out_splits), 4), dtype=pos.dtype, device=pos.device)
        dist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)
        return recv[:, :3].contiguous(), recv[:, 3].contiguous()

    def _gather8(self, x: torch.Tensor):
        if self.R == 1:
            return [x.detach().cpu().numpy()]
        bufs = [torch.empty_like(x) for _ in range(self.R)]
        dist.all_gather(bufs, x.contiguous(), group=self.group)
        return [b.detach().cpu().numpy() for b in bufs]


class SlabCoulombSolver:
    """Multi-GPU ``CoulombSolver.evaluate`` (evaluate.py:114-144): the k-space
    slab solver and the slab near field on the same particle ownership
    (z anchor plane of the k-space layout), plus self and background terms.

    ``evaluate(pos, q)`` takes this rank's particles (``owned(pos_all)``) and
    returns an EnergyBreakdown with global energies / pressure / pair count
    and the forces of this rank's particles (prefactor applied).  ``kspace``
    / ``near_ops`` are pluggable for the CPU decomposition tests only."""

    def __init__(self, h, params, group=None, kspace=None, near_ops=None):
        from .kernel import SplitKernel
        from .mesh import plan_grid
        from .pswf import build_pswf, solve_bandwidth
        from .realspace import build_pair_table
        from .slab import SlabKSpaceSolver
        d_split, d_spread, P = params.resolved()
        if params.force_mode != "ik":
            raise ParameterError("the z-slab k-space solver computes ik forces only")
        self.params = params
        self.cell = Cell(np.asarray(h, dtype=float))
        check_cutoff(self.cell, params.r_c)
        basis = build_pswf(solve_bandwidth(d_split))
        spread = basis if abs(d_spread - d_split) <= 1e-300 else build_pswf(
            solve_bandwidth(d_spread))
        self.kern = SplitKernel(basis=basis, r_c=params.r_c)
        if kspace is None:
            ortho = self.cell.is_orthorhombic
            spec = plan_grid(self.cell, self.kern, delta_spread=d_spread, P=P,
                             oversampling=params.oversampling, spread_basis=spread,
                             fixed_M=params.fixed_M, allow_triclinic=not ortho)
            kspace = SlabKSpaceSolver(self.cell.h, spec.M, P, basis, spec.window, params.r_c,
                                      spread_basis=spread, group=group,
                                      precision=params.precision)
        self.kspace = kspace
        if near_ops is None:
            near_ops = CudaNearOps(self.kern, build_pair_table(self.kern), self.cell)
        self.near = SlabNearField.from_kspace(kspace, params.r_c, near_ops, group)
        self.group = group

    def owned(self, pos_all: np.ndarray) -> np.ndarray:
        return self.kspace.owned(pos_all)

    def _sum_ranks(self, x: float) -> float:
        t = torch.tensor([float(x)], dtype=torch.float64)
        if self.near.R == 1:
            return float(x)
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = t.to(dev)
        bufs = [torch.empty_like(t) for _ in range(self.near.R)]
        dist.all_gather(bufs, t, group=self.group)
        tot = 0.0
        for b in bufs:                      # rank order
            tot += float(b.item())
        return tot

    def evaluate(self, pos: torch.Tensor, q: torch.Tensor, want_forces: bool = True,
                 want_pressure: bool = True):
        from .kernel import background_correction
        from .solver import EnergyBreakdown
        pref = self.params.prefactor
        e_far, p_far, f_far = self.kspace.evaluate(pos, q, want_forces)
        e_near, p_near, f_near, npairs = self.near.evaluate(pos, q)
        qh = q.detach().cpu().numpy()
        q2 = self._sum_ranks(float(np.sum(qh * qh)))
        qt = self._sum_ranks(float(np.sum(qh)))
        b = self.kern.basis
        u_self = float(-(b.psi0_at_zero / (2.0 * b.C0 * self.kern.r_c)) * q2)
        u_cb, u_bb, p_corr = background_correction(self.kern, qt, self.cell.volume)
        out = EnergyBreakdown(u_near=pref * e_near, u_far=pref * e_far, u_self=pref * u_self,
                              u_background=pref * (u_cb + u_bb), pair_count=npairs)
        if want_forces:
            out.forces = pref * (f_far.to(f_near.dtype) + f_near.to(f_far.device))
        if want_pressure:
            out.pressure = pref * (np.asarray(p_near) + np.asarray(p_far) + p_corr)
        return out
