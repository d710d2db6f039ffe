"""Multi-GPU z-slab decomposition of the k-space path.

One process per GPU (torch.distributed, NCCL over NVLink on a B200 box).
Rank r owns the global grid planes [z0_r, z1_r) of the [z][y][x] grid and the
charges whose z anchor falls in them.  One step:

1. spread      - the rank's charges into a local slab with P-1 ghost planes
                 (CUDA tile kernels through a z-slab EspPlan)
2. halo add    - ghost planes go to the neighbouring ranks (NCCL send/recv) and
                 are added to their owned planes
3. forward FFT - rfft2 over (y, x) per owned plane (cuFFT), all-to-all
                 transpose to ky chunks, fft along z (cuFFT)
4. scale/reduce- E and the six pressure components over the rank's in-band
                 modes; the 7 partial sums are all-gathered and added in
                 rank order (bit-stable at a fixed GPU count)
5. forces      - ik spectra, ifft along z, all-to-all back, irfft2, ghost
                 planes of the three fields from the neighbours, window gather

The per-rank mode tables (mask, Fhat What^-2, pressure kernel) are built on
the host once per cell with the reference's numpy expressions
(mesh.py:242-275), so the energy/pressure sums are those of the single-GPU
path up to summation order.

The collectives and FFT stages are written against torch tensors, so the same
orchestration runs on CPU with the gloo backend for the decomposition tests;
the per-rank spread/gather backend is pluggable for that purpose only (the
product backend is :class:`CudaSlabOps`).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist
from numpy.polynomial import legendre as L

from .errors import ParameterError, PlanningError
from .plan import EspPlan, cell_tables
from .pswf import PswfBasis, WindowTable


class SlabLayout:
    """Contiguous split of Mz planes (and My rows of the transposed
    spectrum) over R ranks."""

    def __init__(self, Mz: int, My: int, R: int, P: int):
        self.R = R
        zc = [Mz // R + (r < Mz % R) for r in range(R)]
        yc = [My // R + (r < My % R) for r in range(R)]
        if min(zc) < P:
            raise PlanningError(f"slab of {min(zc)} planes is thinner than the stencil P={P}; "
                                f"use fewer ranks")
        self.zcount = zc
        self.zstart = [int(v) for v in np.concatenate([[0], np.cumsum(zc)[:-1]])]
        self.ycount = yc
        self.ystart = [int(v) for v in np.concatenate([[0], np.cumsum(yc)[:-1]])]
        self.nlo = (P - 1) // 2          # ghost planes below the slab (= -lo)
        self.nup = P - 1 - self.nlo      # ghost planes above the slab

    def owner(self, zplane: np.ndarray) -> np.ndarray:
        return np.searchsorted(np.asarray(self.zstart), zplane, side="right") - 1


def anchor_plane(pos: np.ndarray, h: np.ndarray, M, P: int) -> np.ndarray:
    """Global z anchor plane of each charge with the kernels' arithmetic
    (grid_coords / anchor_base / wrap in esp_internal.cuh)."""
    pos = np.asarray(pos, dtype=float)
    h = np.asarray(h, dtype=float)
    off = h - np.diag(np.diag(h))
    if np.all(np.abs(off) <= 1e-12 * np.max(np.abs(h))):
        u = pos[:, 2] / (h[2, 2] / M[2])
    else:
        hi = np.linalg.inv(h)
        u = ((hi[2, 0] * pos[:, 0] + hi[2, 1] * pos[:, 1]) + hi[2, 2] * pos[:, 2]) * float(M[2])
    base = np.rint(u) if P % 2 else np.floor(u)
    return np.mod(base.astype(np.int64), M[2])


class CudaSlabOps:
    """Product backend: the CUDA tile kernels on a z-slab plan."""

    def __init__(self, M, P, window: WindowTable, split: PswfBasis, r_c: float, h,
                 z0: int, nz: int, precision="fp64", capacity=1 << 16):
        self.plan = EspPlan(M, P, window, split, r_c, precision=precision, capacity=capacity,
                            slab=(M[2], z0, nz))
        self.plan.set_cell(h)
        # full-grid plan whose band-pruned transforms run the distributed
        # transposes (esp_slab_*): only its mode tables and transform buffers
        # are used
        self.spectral = EspPlan(M, P, window, split, r_c, precision=precision, capacity=1)
        self.spectral.set_cell(h)
        self._n = 0

    def spread(self, pos: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
        self._n = pos.shape[0]
        return self.plan.spread(pos, q)           # (nz+P-1, My, Mx) view

    def gather(self, fields: torch.Tensor, pos, q) -> torch.Tensor:
        return self.plan.gather_fields(fields, self._n)


class SlabKSpaceSolver:
    """Far-field energy, pressure tensor and ik forces on R ranks."""

    def __init__(self, h, M, P: int, split: PswfBasis, window: WindowTable, r_c: float,
                 spread_basis: PswfBasis | None = None, group=None, ops=None,
                 precision="fp64", device=None, capacity=1 << 16):
        self.group = group
        self.R = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.h = np.asarray(h, dtype=float)
        self.M = tuple(int(m) for m in M)
        self.P = int(P)
        self.layout = SlabLayout(self.M[2], self.M[1], self.R, self.P)
        self.z0 = self.layout.zstart[self.rank]
        self.nz = self.layout.zcount[self.rank]
        self.y0 = self.layout.ystart[self.rank]
        self.ny = self.layout.ycount[self.rank]
        self.split = split
        self.spread_basis = spread_basis or split
        self.r_c = float(r_c)
        self.kmax = split.c / self.r_c
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self.ops = ops if ops is not None else CudaSlabOps(
            self.M, self.P, window, split, r_c, self.h, self.z0, self.nz, precision, capacity)
        self._build_modes()
        self._fused = self._setup_fused()

    # -- fused transposes over peer memory (esp_slab_*) ---------------------------
    def _setup_fused(self) -> bool:
        """Receive buffers for the distributed transforms: forward
        [Mz][ny_r][ldx] and backward [3][nz_r][nby][ldx] per rank, in one
        symmetric-memory allocation per rank whose peers' base pointers are
        the transpose targets.  False (torch/NCCL transposes) when the
        backend is not the CUDA one, the grid has no fused transforms, or
        peer memory is unavailable."""
        spec = getattr(self.ops, "spectral", None)
        if spec is None or spec.fft_path != "fused" or self.R > 8:
            return False
        R, lay = self.R, self.layout
        z_start = list(lay.zstart) + [self.M[2]]
        by, info = spec.slab_layout(R)
        cb, ldx, nby = info["cbytes"], info["ldx"], info["nby"]
        fwd_bytes = [self.M[2] * max(by[r + 1] - by[r], 1) * ldx * cb for r in range(R)]
        back_bytes = [3 * lay.zcount[r] * nby * ldx * cb for r in range(R)]
        off_back = (max(fwd_bytes) + 255) // 256 * 256
        total = off_back + max(back_bytes)
        try:
            if R == 1:
                raw = torch.zeros(total, dtype=torch.uint8, device=self.device)
                bases, self._symm = [raw.data_ptr()], None
            else:
                import torch.distributed._symmetric_memory as symm_mem
                group = self.group or dist.group.WORLD
                if not symm_mem.is_symm_mem_enabled_for_group(group.group_name):
                    symm_mem.enable_symm_mem_for_group(group.group_name)
                # same size on every rank (collective allocation)
                raw = symm_mem.empty(total, dtype=torch.uint8, device=self.device)
                raw.zero_()
                self._symm = symm_mem.rendezvous(raw, group)
                bases = list(self._symm.buffer_ptrs)
        except Exception:
            return False
        self._raw = raw
        ct = torch.complex128 if spec.precision == "fp64" else torch.complex64
        me = self.rank
        self._recv_fwd = raw[:fwd_bytes[me]].view(ct)
        self._recv_back = raw[off_back:off_back + back_bytes[me]].view(ct)
        d = _SlabPeers(R, me, z_start, [b for b in bases], [b + off_back for b in bases])
        self._desc = d.desc()
        return True

    def _rank_barrier(self):
        """Stream-ordered barrier between the transpose stages."""
        if self.R == 1:
            return
        self._symm.barrier()

    # -- per-cell mode tables for this rank's ky chunk -----------------------
    def _build_modes(self):
        M, P = self.M, self.P
        t = cell_tables(self.h, M, P, self.spread_basis, self.kmax)
        Hx = M[0] // 2 + 1
        kx_i = np.arange(Hx)
        ky_i = np.arange(self.y0, self.y0 + self.ny)
        kz_i = np.arange(M[2])
        K = t.axis_k
        shape = (self.ny, M[2], Hx)                  # local spectrum [ky][kz][kx]
        kv = []
        for a in range(3):
            kv.append(K[a][0][kx_i][None, None, :] + K[a][1][ky_i][:, None, None]
                      + K[a][2][kz_i][None, :, None])
        kx, ky, kz = [np.broadcast_to(k, shape) for k in kv]
        k2 = kx ** 2 + ky ** 2 + kz ** 2
        kmag = np.sqrt(k2)
        mask = (kmag <= self.kmax) & (k2 > 0.0)
        W = t.axis_what
        what = (W[0][kx_i][None, None, :] * W[1][ky_i][:, None, None]) * W[2][kz_i][None, :, None]
        what = np.broadcast_to(what, shape)[mask]
        if np.any(np.abs(what) < 1e-13 * abs(t.what_zero)):
            raise PlanningError("window transform underflow on a retained mode")
        winv2 = 1.0 / (what * what)
        b = self.split
        x = np.clip(kmag[mask] * self.r_c / b.c, 0.0, 1.0)
        pref = 2.0 * np.pi * b.lambda0 / b.C0
        k2m = k2[mask]
        fhat = pref * L.legval(x, b.legendre_coeffs) / k2m
        dterm = pref * x * L.legval(x, L.legder(b.legendre_coeffs)) / k2m ** 2
        A = fhat * winv2
        B = dterm * winv2 - 2.0 * A / k2m
        kxm = np.broadcast_to(kx_i[None, None, :], shape)[mask]
        wt = np.where((kxm == 0) | (2 * kxm == M[0]), 1.0, 2.0)
        dev = self.device
        f64 = torch.float64
        self._idx = torch.as_tensor(np.flatnonzero(mask), device=dev)
        self._A = torch.as_tensor(A, dtype=f64, device=dev)
        self._B = torch.as_tensor(B, dtype=f64, device=dev)
        self._wt = torch.as_tensor(wt, dtype=f64, device=dev)
        self._k = [torch.as_tensor(np.ascontiguousarray(k[mask]), dtype=f64, device=dev)
                   for k in (kx, ky, kz)]
        self._shape = shape
        self.volume = t.volume
        self.h3 = t.volume_element

    # -- ownership -------------------------------------------------------------
    def owned(self, pos_host: np.ndarray) -> np.ndarray:
        """Boolean mask of the charges this rank owns (z anchor in its slab)."""
        zp = anchor_plane(pos_host, self.h, self.M, self.P)
        return (zp >= self.z0) & (zp < self.z0 + self.nz)

    # -- communication helpers -------------------------------------------------
    def _neighbours(self):
        return (self.rank - 1) % self.R, (self.rank + 1) % self.R

    def _p2p(self, to_next: torch.Tensor, to_prev: torch.Tensor, from_prev_shape,
             from_next_shape):
        """Send to next/prev, receive from prev/next (same posting order on
        every rank, so R = 2 pairs match)."""
        if self.R == 1:
            return to_next.clone(), to_prev.clone()   # periodic: my own ghosts
        prev, nxt = self._neighbours()
        rp = torch.empty(from_prev_shape, dtype=to_next.dtype, device=to_next.device)
        rn = torch.empty(from_next_shape, dtype=to_next.dtype, device=to_next.device)
        ops = [dist.P2POp(dist.isend, to_next.contiguous(), nxt, self.group),
               dist.P2POp(dist.isend, to_prev.contiguous(), prev, self.group),
               dist.P2POp(dist.irecv, rp, prev, self.group),
               dist.P2POp(dist.irecv, rn, nxt, self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return rp, rn

    def _alltoall(self, x: torch.Tensor, in_splits, out_splits) -> torch.Tensor:
        """x split along dim 0 by in_splits -> pieces from every rank along
        dim 0 by out_splits."""
        if self.R == 1:
            return x.clone()
        out = torch.empty((sum(out_splits),) + tuple(x.shape[1:]), dtype=x.dtype,
                          device=x.device)
        dist.all_to_all_single(out, x.contiguous(), out_splits, in_splits, group=self.group)
        return out

    # -- the step ------------------------------------------------------------------
    def evaluate(self, pos: torch.Tensor, q: torch.Tensor, want_forces: bool = True):
        """pos/q: this rank's charges.  Returns (E, P (3x3 numpy), F (n,3) or
        None); E and P are global (identical on every rank).  One host
        synchronisation (the 7 reduced doubles); evaluate_device has none."""
        out7, F = self.evaluate_device(pos, q, want_forces)
        v = out7.cpu().numpy()
        pp = v[1:]
        Pt = np.array([[pp[0], pp[1], pp[2]], [pp[1], pp[3], pp[4]], [pp[2], pp[4], pp[5]]])
        return float(v[0]), Pt, F

    def evaluate_device(self, pos: torch.Tensor, q: torch.Tensor, want_forces: bool = True,
                        out7: torch.Tensor | None = None, forces: torch.Tensor | None = None):
        """The whole distributed step, stream-ordered with no host
        synchronisation (CUDA-graph capturable): returns (out7, F) with out7 =
        [E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz] on the device, the 7 per-rank sums
        added in rank order (bit-stable at a fixed GPU count)."""
        lay, P, M = self.layout, self.P, self.M
        nlo, nup, nz = lay.nlo, lay.nup, self.nz
        slab = self.ops.spread(pos, q)                     # (nz+P-1, My, Mx)
        own = slab[nlo:nlo + nz].clone()
        lower, upper = slab[:nlo], slab[nlo + nz:]
        from_prev, from_next = self._p2p(upper, lower, upper.shape, lower.shape)
        own[:nup] += from_prev                             # prev's upper ghosts
        own[nz - nlo:] += from_next                        # next's lower ghosts
        if self._fused:
            return self._evaluate_fused(own, pos, q, want_forces, out7, forces)
        # forward transform: (y, x) per plane, transpose, z
        X = torch.fft.rfft2(own, dim=(-2, -1))             # (nz, My, Hx)
        Hx = X.shape[-1]
        Xt = X.permute(1, 0, 2).contiguous()               # (My, nz, Hx)
        flat = Xt.reshape(M[1] * nz, Hx)
        in_splits = [c * nz for c in lay.ycount]
        out_splits = [self.ny * c for c in lay.zcount]
        recv = self._alltoall(flat, in_splits, out_splits)
        pieces = torch.split(recv, out_splits, dim=0)
        Y = torch.cat([p.reshape(self.ny, c, Hx) for p, c in zip(pieces, lay.zcount)], dim=1)
        Y = torch.fft.fft(Y, dim=1)                        # (ny, Mz, Hx): [ky][kz][kx]
        # fused scale/reduce over this rank's retained modes
        Xm = Y.reshape(-1)[self._idx]
        amp2 = (Xm.real ** 2 + Xm.imag ** 2).to(torch.float64)
        w = self._wt * amp2
        wa, tb = w * self._A, w * self._B
        kx, ky, kz = self._k
        part = torch.stack([wa.sum(), (tb * kx * kx + wa).sum(), (tb * kx * ky).sum(),
                            (tb * kx * kz).sum(), (tb * ky * ky + wa).sum(),
                            (tb * ky * kz).sum(), (tb * kz * kz + wa).sum()])
        tot = self._rank_ordered_sum(part)
        h3sq = self.h3 * self.h3
        scale = torch.tensor([h3sq / (2.0 * self.volume)] + [h3sq / (2.0 * self.volume ** 2)] * 6,
                             dtype=torch.float64, device=tot.device)
        out7 = self._out7(out7, tot * scale)
        if not want_forces:
            return out7, None
        # ik spectra (rho_hat = h3 X), inverse z, transpose back, inverse (y, x)
        c = self._A * self.h3
        spec = torch.zeros((3,) + tuple(self._shape), dtype=Y.dtype, device=Y.device)
        for d in range(3):
            val = (1j * (self._k[d] * c)).to(Y.dtype) * Xm
            spec[d].view(-1)[self._idx] = val
        spec = torch.fft.ifft(spec, dim=2)                 # along kz
        S = spec.permute(1, 0, 2, 3).contiguous()          # (ny, 3, Mz, Hx)
        back_in = [torch.split(S, lay.zcount, dim=2)[r].contiguous().reshape(-1, Hx)
                   for r in range(self.R)]
        flat_b = torch.cat(back_in, dim=0)
        in_b = [self.ny * 3 * c for c in lay.zcount]
        out_b = [c * 3 * nz for c in lay.ycount]
        recv_b = self._alltoall(flat_b, in_b, out_b)
        parts = torch.split(recv_b, out_b, dim=0)
        Z = torch.cat([p.reshape(c, 3, nz, Hx) for p, c in zip(parts, lay.ycount)], dim=0)
        Z = Z.permute(1, 2, 0, 3).contiguous()             # (3, nz, My, Hx)
        fields = torch.fft.irfft2(Z, s=(M[1], M[0]), dim=(-2, -1))   # (3, nz, My, Mx)
        # ghost planes of the fields: my bottom nup planes -> prev, top nlo -> next
        top, bottom = fields[:, nz - nlo:], fields[:, :nup]
        from_prev_f, from_next_f = self._p2p(top, bottom, (3, nlo) + tuple(fields.shape[2:]),
                                             (3, nup) + tuple(fields.shape[2:]))
        ext = torch.cat([from_prev_f, fields, from_next_f], dim=1)   # (3, nz+P-1, My, Mx)
        dt = torch.float64 if getattr(getattr(self.ops, "plan", None), "precision",
                                      "fp64") == "fp64" else torch.float32
        F = self.ops.gather(ext.to(dt).contiguous(), pos, q)
        if forces is not None:
            forces.copy_(F)
            F = forces
        return out7, F

    def _rank_ordered_sum(self, part: torch.Tensor) -> torch.Tensor:
        """All-gather the 7 per-rank partial sums and add them in rank order
        on the device (no host round trip; bit-stable at a fixed GPU count)."""
        if self.R == 1:
            return part
        flat = torch.empty(self.R * part.numel(), dtype=part.dtype, device=part.device)
        dist.all_gather_into_tensor(flat, part.contiguous(), group=self.group)
        allp = flat.view(self.R, -1)
        tot = allp[0].clone()
        for r in range(1, self.R):
            tot = tot + allp[r]
        return tot

    @staticmethod
    def _out7(out7, val):
        if out7 is None:
            return val
        out7.copy_(val)
        return out7

    def _evaluate_fused(self, own: torch.Tensor, pos, q, want_forces: bool, out7=None,
                        forces=None):
        """The spectral part on the band-pruned kernels with the transposes
        fused into them (peer stores), NCCL only for the 7-double reduction
        and the ghost planes."""
        spec = self.ops.spectral
        lay, M, nz, nlo, nup = self.layout, self.M, self.nz, self.layout.nlo, self.layout.nup
        spec.slab_forward(self._desc, own.to(spec.real_dtype))
        self._rank_barrier()
        part = spec.slab_reduce(self._desc, self._recv_fwd, want_forces)
        out7 = self._out7(out7, self._rank_ordered_sum(part))
        if not want_forces:
            return out7, None
        self._rank_barrier()
        fields = torch.empty((3, nz, M[1], M[0]), dtype=spec.real_dtype, device=own.device)
        spec.slab_inverse(self._desc, self._recv_back, fields)
        top, bottom = fields[:, nz - nlo:], fields[:, :nup]
        from_prev_f, from_next_f = self._p2p(top, bottom, (3, nlo) + tuple(fields.shape[2:]),
                                             (3, nup) + tuple(fields.shape[2:]))
        ext = torch.cat([from_prev_f, fields, from_next_f], dim=1)
        F = self.ops.gather(ext.contiguous(), pos, q)
        if forces is not None:
            forces.copy_(F)
            F = forces
        return out7, F

    def graphed(self, pos: torch.Tensor, q: torch.Tensor, want_forces: bool = True):
        """Capture evaluate_device on fixed buffers into one CUDA graph
        (spread, halo send/recv, fused transforms with peer-store transposes,
        device barriers, the rank-ordered reduction and the gather).  Returns
        (graph, out7, forces); ``graph.replay()`` re-runs the step after the
        caller updates pos / q in place.  Collective capture needs NCCL graph
        support; on failure the caller keeps the eager step."""
        dev = pos.device
        out7 = torch.empty(7, dtype=torch.float64, device=dev)
        F = torch.empty((pos.shape[0], 3), dtype=torch.float64, device=dev) if want_forces \
            else None
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.evaluate_device(pos, q, want_forces, out7, F)      # warm-up
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        if self.R > 1:
            dist.barrier(group=self.group)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.evaluate_device(pos, q, want_forces, out7, F)
        torch.cuda.synchronize()
        return g, out7, F

class _SlabPeers:
    """esp_slab_desc of one rank from raw peer base addresses."""

    def __init__(self, R, rank, z_start, fwd, back):
        self.R, self.rank, self.z_start, self.fwd, self.back = R, rank, z_start, fwd, back

    def desc(self):
        from . import _lib
        d = _lib.SlabDesc()
        d.nranks, d.rank = self.R, self.rank
        for i, v in enumerate(self.z_start):
            d.z_start[i] = int(v)
        for i in range(self.R):
            d.fwd_peers[i] = int(self.fwd[i])
            d.back_peers[i] = int(self.back[i])
        return d


def check_slab_geometry(M, R, P):
    if M[2] // R < P:
        raise ParameterError(f"{R} slabs of a {M[2]}-plane grid are thinner than P={P}")
