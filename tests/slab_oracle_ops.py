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


class OracleNearOps:
    """Test-only local pair sum for the distributed near field: the oracle's
    pair values (realspace.py restatement) over the rank's owned + ghost
    particles, sums for the owned particles' directed pairs only."""

    def __init__(self, h, basis, r_c, table=None):
        self.h = np.asarray(h, dtype=float)
        self.basis, self.r_c, self.table = basis, float(r_c), table

    def evaluate(self, pos, q, n_owned):
        P = pos.detach().cpu().numpy()
        Q = q.detach().cpu().numpy()
        F = np.zeros((n_owned, 3))
        out = np.zeros(8)
        npairs = 0
        if len(P) >= 2:
            i, j = O.pairs_within(self.h, P, self.r_c)
            oi, oj = i < n_owned, j < n_owned
            keep = oi | oj
            i, j, oi, oj = i[keep], j[keep], oi[keep], oj[keep]
            dr = O.minimum_image(self.h, P[i] - P[j])
            r = np.sqrt(np.einsum("ij,ij->i", dr, dr))
            m = r <= self.r_c
            i, j, oi, oj, dr, r = i[m], j[m], oi[m], oj[m], dr[m], r[m]
            qq = Q[i] * Q[j]
            nv, fv = (O.table_values(self.table, r) if self.table is not None else
                      (O.near_value(self.basis, self.r_c, r), O.fn_value(self.basis, self.r_c, r)))
            fmag = qq * fv / r ** 3
            w = 0.5 * (oi.astype(float) + oj.astype(float))
            out[0] = np.sum(w * qq * nv)
            W = (dr.T * (w * fmag)) @ dr / float(np.linalg.det(self.h))
            out[1:7] = [W[0, 0], W[0, 1], W[0, 2], W[1, 1], W[1, 2], W[2, 2]]
            out[7] = float(np.sum(oi) + np.sum(oj))
            pf = fmag[:, None] * dr
            np.add.at(F, i[oi], pf[oi])
            np.add.at(F, j[oj], -pf[oj])
            npairs = int(np.sum(oi & oj))
        stats = torch.tensor([npairs, -1, -1, int(out[7])], dtype=torch.int64)
        return torch.as_tensor(out), torch.as_tensor(F), stats
