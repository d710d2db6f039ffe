"""Test-only per-rank spread/gather backend for the slab decomposition tests:
the CPU oracle's stencil arithmetic restricted to one z-slab (owned planes +
ghost planes, no periodic wrap in z).  Used with the gloo backend to check the
decomposition algebra (halo add, transposes, reductions) without GPUs."""

import numpy as np
import torch

from oracle import esp_oracle as O


class OracleSlabOps:
    def __init__(self, plan: "O.Plan", z0: int, nz: int):
        self.plan = plan
        self.z0, self.nz = z0, nz
        self.P = plan.P
        self.lo = -((plan.P - 1) // 2)
        self.nzl = nz + plan.P - 1

    def _stencils(self, pos):
        plan, P = self.plan, self.P
        u = O.grid_coordinates(plan, pos)
        ix, tx = O.stencil(u[:, 0], plan.M[0], P)
        iy, ty = O.stencil(u[:, 1], plan.M[1], P)
        base = np.round(u[:, 2]) if P % 2 else np.floor(u[:, 2])
        a = np.mod(base.astype(np.int64), plan.M[2]) - (self.z0 + self.lo)
        p = np.arange(self.lo, self.lo + P)
        iz = a[:, None] + p[None, :]
        tz = u[:, 2][:, None] - (base[:, None] + p[None, :])
        assert iz.min() >= 0 and iz.max() < self.nzl
        w = [plan.window(tx), plan.window(ty), plan.window(tz)]
        flat = ((iz[:, None, None, :] * plan.M[1] + iy[:, None, :, None]) * plan.M[0]
                + ix[:, :, None, None])
        wt = w[0][:, :, None, None] * w[1][:, None, :, None] * w[2][:, None, None, :]
        return flat.reshape(len(pos), -1), wt.reshape(len(pos), -1)

    def spread(self, pos, q):
        pos = np.asarray(pos.cpu() if isinstance(pos, torch.Tensor) else pos, dtype=float)
        q = np.asarray(q.cpu() if isinstance(q, torch.Tensor) else q, dtype=float)
        self._cache = self._stencils(pos) if len(pos) else None
        G = self.nzl * self.plan.M[1] * self.plan.M[0]
        if self._cache is None:
            return torch.zeros((self.nzl, self.plan.M[1], self.plan.M[0]), dtype=torch.float64)
        flat, wt = self._cache
        grid = np.bincount(flat.ravel(), weights=(wt * q[:, None]).ravel(), minlength=G)
        return torch.as_tensor(grid.reshape(self.nzl, self.plan.M[1], self.plan.M[0]))

    def gather(self, fields, pos, q):
        q = np.asarray(q.cpu() if isinstance(q, torch.Tensor) else q, dtype=float)
        if self._cache is None:
            return torch.zeros((0, 3), dtype=torch.float64)
        flat, wt = self._cache
        f = fields.detach().cpu().numpy().reshape(3, -1)
        F = np.stack([-q * np.einsum("np,np->n", f[d][flat], wt) for d in range(3)], axis=1)
        return torch.as_tensor(F)
