"""EspPlan: one device plan (grid, window, basis, buffers, cuFFT plans).

Python owner of the C-ABI ``esp_plan`` (include/esp_b200.h).  Setup-time
tables (per-axis wavenumbers and window transforms — the separable inputs of
the reference ModeWorkspace, mesh.py:237-275) are computed here on the host
with the reference's exact arithmetic and uploaded once per cell; the mask,
Fhat and dterm tables are then built on the device.  Every per-step
operation is a CUDA launch on the caller's torch stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ParameterError, PlanningError
from .pswf import PswfBasis, WindowTable

_DT = {"fp64": _lib.ESP_FP64, "fp32": _lib.ESP_FP32}


class _DevView:
    """__cuda_array_interface__ shim to alias plan-owned device memory."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class CellTables:
    """Per-cell inputs of the device mode setup."""
    h: np.ndarray
    hinv: np.ndarray
    orthorhombic: bool
    spacing: np.ndarray
    volume: float
    volume_element: float
    axis_k: list          # axis_k[a][d] : (M_d,) f64
    axis_what: list       # (M_d,) f64 per axis
    what_zero: float
    band: tuple
    grad_scale: np.ndarray


def cell_tables(h, M, P, spread: PswfBasis, kmax: float, orthorhombic=None) -> CellTables:
    """Separable mode-workspace inputs.

    Orthorhombic: k_d = 2 pi fftfreq(M_d, 1/M_d) / L_d (mesh.py:242) and
    What_d = omega_d lambda0 psi(clip(omega_d k_d / c)) (mesh.py:258-261) with
    omega_d = P h_d / 2 (mesh.py:109-110) — the same numpy expressions, so the
    mask and deconvolution agree bit-for-bit with the reference.
    Triclinic (fractional-coordinate lattice):
    k = 2 pi h^-T m and What(m) = V prod_d (P/2M_d) lambda0 psi(pi P m_d/(M_d c)).
    """
    h = np.asarray(h, dtype=float).reshape(3, 3)
    M = tuple(int(m) for m in M)
    if orthorhombic is None:
        off = h - np.diag(np.diag(h))
        orthorhombic = bool(np.all(np.abs(off) <= 1e-12 * np.max(np.abs(h))))
    volume = float(np.linalg.det(h))
    hinv = np.linalg.inv(h)
    freqs = [np.fft.fftfreq(M[d], d=1.0 / M[d]) for d in range(3)]
    zeros = [np.zeros(M[d]) for d in range(3)]
    axis_k = [[zeros[d] for d in range(3)] for _ in range(3)]
    sb = spread
    if orthorhombic:
        lengths = np.diag(h)
        spacing = lengths / np.asarray(M)
        omega = P * spacing / 2.0
        for d in range(3):
            axis_k[d][d] = 2.0 * np.pi * np.fft.fftfreq(M[d], d=1.0 / M[d]) / lengths[d]
        axis_what = [omega[d] * sb.lambda0 * sb.psi_series(
            np.clip(omega[d] * axis_k[d][d] / sb.c, -1, 1)) for d in range(3)]
        what_zero = float(np.prod([w * sb.lambda0 * sb.psi0_at_zero for w in omega]))
        volume_element = float(np.prod(spacing))
        band = []
        for d in range(3):
            inb = np.abs(axis_k[d][d]) <= kmax
            band.append(int(np.max(np.abs(np.round(freqs[d][inb])))) if inb.any() else 0)
        grad_scale = 1.0 / spacing
    else:
        norms = np.linalg.norm(h, axis=0)
        spacing = norms / np.asarray(M)
        B = 2.0 * np.pi * hinv.T
        for a in range(3):
            for d in range(3):
                axis_k[a][d] = B[a, d] * freqs[d]
        axis_what = []
        for d in range(3):
            arg = np.pi * P * freqs[d] / (M[d] * sb.c)
            w = (P / (2.0 * M[d])) * sb.lambda0 * sb.psi_series(np.clip(arg, -1, 1))
            axis_what.append(volume * w if d == 0 else w)
        what_zero = volume * float(np.prod([(P / (2.0 * m)) * sb.lambda0 * sb.psi0_at_zero
                                            for m in M]))
        volume_element = volume / float(np.prod(M))
        band = [min(M[d] // 2, int(np.floor(kmax * norms[d] / (2.0 * np.pi) * (1 + 1e-9))) + 1)
                for d in range(3)]
        grad_scale = np.zeros(3)
    return CellTables(h=h, hinv=hinv, orthorhombic=orthorhombic, spacing=np.asarray(spacing),
                      volume=volume, volume_element=volume_element,
                      axis_k=[[np.ascontiguousarray(x, dtype=float) for x in row] for row in axis_k],
                      axis_what=[np.ascontiguousarray(x, dtype=float) for x in axis_what],
                      what_zero=what_zero, band=tuple(band), grad_scale=np.asarray(grad_scale))


def _stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class EspPlan:
    """Device plan for one (M, P, window, splitting kernel, precision)."""

    def __init__(self, M, P: int, window: WindowTable, split: PswfBasis, r_c: float,
                 spread: PswfBasis | None = None, precision: str = "fp64",
                 deterministic: bool = True, capacity: int = 1 << 16, tile=(0, 0, 0),
                 slab: tuple | None = None):
        """``slab=(Mz_global, z0, nz)``: a z-slab plan for the multi-GPU slab
        decomposition — the local grid is (Mx, My, nz + P - 1) holding global
        planes z0 + lo ... (owned planes plus ghost planes)."""
        if not torch.cuda.is_available():
            raise RuntimeError("EspPlan needs a CUDA device (the B200 path has no CPU fallback)")
        if precision not in _DT:
            raise ParameterError(f"unknown precision {precision!r}")
        if window.P != P:
            raise PlanningError("supplied window table does not match P")
        torch.cuda.current_device()
        torch.empty(0, device="cuda")  # make torch's primary context current
        self.P = int(P)
        self.slab = tuple(int(v) for v in slab) if slab is not None else None
        if self.slab is not None:
            Mz_glob, z0, nz = self.slab
            self.M_global = (int(M[0]), int(M[1]), Mz_glob)
            M = (int(M[0]), int(M[1]), nz + self.P - 1)
        self.M = tuple(int(m) for m in M)
        if self.slab is None:
            self.M_global = self.M
        self.window = window
        self.split = split
        self.spread_basis = spread if spread is not None else split
        self.r_c = float(r_c)
        self.kmax = split.c / self.r_c
        self.precision = precision
        self.deterministic = bool(deterministic)
        self.tile = tuple(int(t) for t in tile)
        self.capacity = int(max(capacity, 1))
        self._handle = None
        self._cell = None
        self.version = 0          # bumps on every forward transform / spectrum change
        self.generation = 0       # bumps when device buffers or cell constants change
        self._create()

    # -- lifetime -----------------------------------------------------------
    def _create(self):
        L = _lib.lib()
        w = self.window
        self._coef = np.ascontiguousarray(w.coef, dtype=float)
        self._dcoef = np.ascontiguousarray(w.deriv_coef, dtype=float)
        self._breaks = np.ascontiguousarray(w.breaks, dtype=float)
        self._leg = np.ascontiguousarray(self.split.legendre_coeffs, dtype=float)
        self._legd = np.ascontiguousarray(self.split.derivative_coeffs, dtype=float)
        d = _lib.PlanDesc()
        d.M[:] = list(self.M)
        d.P = self.P
        d.precision = _DT[self.precision]
        d.deterministic = int(self.deterministic)
        d.max_particles = self.capacity
        d.n_pieces = w.coef.shape[0]
        d.degree = w.coef.shape[1] - 1
        d.h_window_coef = _ptr(self._coef)
        d.h_window_deriv_coef = _ptr(self._dcoef)
        d.h_window_breaks = _ptr(self._breaks)
        d.n_legendre = self._leg.size
        d.h_legendre = _ptr(self._leg)
        d.n_legendre_deriv = self._legd.size
        d.h_legendre_deriv = _ptr(self._legd)
        d.split_c = self.split.c
        d.split_lambda0 = self.split.lambda0
        d.split_C0 = self.split.C0
        d.r_c = self.r_c
        d.kmax = self.kmax
        d.tile[:] = list(self.tile)
        if self.slab is not None:
            d.slab_mz_global = self.slab[0]
            d.slab_z0 = self.slab[1]
        h = C.c_void_p()
        _lib.check(L.esp_plan_create(C.byref(d), C.byref(h)), "esp_plan_create")
        self._handle = h
        info = self.info()
        self.Hx = int(info[3])
        self.n_tiles = int(info[6])

    def close(self):
        if self._handle is not None and self._handle.value:
            torch.cuda.synchronize()
            _lib.lib().esp_plan_destroy(self._handle)
        self._handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def ensure_capacity(self, n: int):
        if n <= self.capacity:
            return
        cell = self._cell
        self.close()
        self.capacity = max(int(n), 2 * self.capacity)
        self._create()
        self.version += 1         # the recreated plan holds no spectrum
        self.generation += 1
        if cell is not None:
            self._cell = None
            self.set_cell(cell)

    # -- per cell -------------------------------------------------------------
    def set_cell(self, h, orthorhombic=None, stream=None):
        t = cell_tables(h, self.M_global, self.P, self.spread_basis, self.kmax, orthorhombic)
        if self.slab is not None:
            # slab plans spread/gather only: z axis arrays resized to the local
            # plane count (their mode tables are never used)
            nzl = self.M[2]
            for a in range(3):
                t.axis_k[a][2] = np.ascontiguousarray(np.resize(t.axis_k[a][2], nzl))
            t.axis_what[2] = np.ascontiguousarray(np.resize(t.axis_what[2], nzl))
            t.band = (t.band[0], t.band[1], min(t.band[2], nzl // 2))
        c = _lib.CellDesc()
        c.h[:] = list(t.h.reshape(-1))
        c.hinv[:] = list(t.hinv.reshape(-1))
        c.orthorhombic = int(t.orthorhombic)
        c.spacing[:] = list(t.spacing)
        c.volume = t.volume
        c.volume_element = t.volume_element
        for a in range(3):
            for dd in range(3):
                c.h_axis_k[3 * a + dd] = _ptr(t.axis_k[a][dd])
        for dd in range(3):
            c.h_axis_what[dd] = _ptr(t.axis_what[dd])
        c.what_zero = t.what_zero
        c.band[:] = list(t.band)
        c.grad_scale[:] = list(t.grad_scale)
        _lib.check(_lib.lib().esp_plan_set_cell(self._handle, C.byref(c), _stream_handle(stream)),
                   "esp_plan_set_cell")
        self._cell = t.h.copy()
        self.tables = t
        self.version += 1         # mode tables changed: cached reductions are stale
        self.generation += 1
        return t

    # -- introspection --------------------------------------------------------
    def info(self):
        buf = (C.c_int64 * 8)()
        _lib.check(_lib.lib().esp_grid_info(self._handle, buf), "esp_grid_info")
        return list(buf)

    def radix_binning(self, n: int) -> bool:
        """True when a step over n charges bins with the device radix sort
        (esp_binning_radix); False for the counting sort."""
        r = C.c_int32()
        _lib.check(_lib.lib().esp_binning_radix(self._handle, int(n), C.byref(r)),
                   "esp_binning_radix")
        return bool(r.value)

    # -- distributed z-slab transforms (esp_slab_*) -----------------------------
    def slab_layout(self, nranks: int):
        """(by_start, info): the in-band ky rows owned per rank and
        {ldx, nby, nbx, cbytes} of the fused transforms."""
        by = (C.c_int32 * (nranks + 1))()
        info = (C.c_int64 * 4)()
        _lib.check(_lib.lib().esp_slab_layout(self._handle, int(nranks), by, info),
                   "esp_slab_layout")
        return [int(v) for v in by], dict(ldx=int(info[0]), nby=int(info[1]),
                                           nbx=int(info[2]), cbytes=int(info[3]))

    def slab_buffers(self, nranks: int, rank: int, z_start):
        """Receive buffers of one rank: forward [Mz][ny_r][ldx] and backward
        [3][nz_r][nby][ldx], complex in the plan precision."""
        by, info = self.slab_layout(nranks)
        ct = torch.complex128 if self.precision == "fp64" else torch.complex64
        ny = by[rank + 1] - by[rank]
        nz = z_start[rank + 1] - z_start[rank]
        fwd = torch.zeros((self.M[2], max(ny, 1), info["ldx"]), dtype=ct, device="cuda")
        back = torch.zeros((3, nz, info["nby"], info["ldx"]), dtype=ct, device="cuda")
        return fwd, back

    @staticmethod
    def slab_desc(nranks: int, rank: int, z_start, fwd_peers, back_peers):
        d = _lib.SlabDesc()
        d.nranks, d.rank = int(nranks), int(rank)
        for i, v in enumerate(z_start):
            d.z_start[i] = int(v)
        for i in range(nranks):
            d.fwd_peers[i] = int(fwd_peers[i].data_ptr())
            d.back_peers[i] = int(back_peers[i].data_ptr())
        return d

    def slab_forward(self, desc, own: torch.Tensor, stream=None):
        own = own.contiguous()
        _lib.check(_lib.lib().esp_slab_forward(self._handle, C.byref(desc),
                                               C.c_void_p(own.data_ptr()),
                                               _stream_handle(stream)), "esp_slab_forward")

    def slab_reduce(self, desc, recv_fwd: torch.Tensor, want_ik: bool,
                    out7: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if out7 is None:
            out7 = torch.empty(7, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().esp_slab_reduce(self._handle, C.byref(desc),
                                              C.c_void_p(recv_fwd.data_ptr()),
                                              int(bool(want_ik)), C.c_void_p(out7.data_ptr()),
                                              _stream_handle(stream)), "esp_slab_reduce")
        return out7

    def slab_inverse(self, desc, recv_back: torch.Tensor, fields: torch.Tensor, stream=None):
        _lib.check(_lib.lib().esp_slab_inverse(self._handle, C.byref(desc),
                                               C.c_void_p(recv_back.data_ptr()),
                                               C.c_void_p(fields.data_ptr()),
                                               _stream_handle(stream)), "esp_slab_inverse")
        return fields

    @property
    def fft_path(self) -> str:
        """"fused" (band-pruned transforms, esp_fft.cu) or "cufft"."""
        return "fused" if _lib.lib().esp_fft_path(self._handle) else "cufft"

    @property
    def real_dtype(self):
        return torch.float64 if self.precision == "fp64" else torch.float32

    def counters(self):
        f, i = C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().esp_counters(self._handle, C.byref(f), C.byref(i)))
        return int(f.value), int(i.value)

    def reset_counters(self):
        _lib.lib().esp_reset_counters(self._handle)

    def grid_view(self) -> torch.Tensor:
        """Alias of the plan's real grid, shape (Mz, My, Mx) ([z][y][x])."""
        ts = "<f8" if self.precision == "fp64" else "<f4"
        ptr = _lib.lib().esp_grid_ptr(self._handle)
        return torch.as_tensor(_DevView(ptr, (self.M[2], self.M[1], self.M[0]), ts),
                               device="cuda")

    def fields_view(self) -> torch.Tensor:
        """Alias of the plan's three ik force fields (3, Mz, My, Mx) of the last
        force evaluation (diagnostics / slab tests); a strided view of the
        ghost-padded array when the TMA gather path wrote it."""
        ts = "<f8" if self.precision == "fp64" else "<f4"
        L = _lib.lib()
        lay = (C.c_int64 * 5)()
        _lib.check(L.esp_fields_layout(self._handle, lay), "esp_fields_layout")
        org, ex, ey, ez, cs = (int(v) for v in lay)
        ptr = L.esp_fields_ptr(self._handle)
        flat = torch.as_tensor(_DevView(ptr, (3 * cs,), ts), device="cuda")
        return flat.as_strided((3, self.M[2], self.M[1], self.M[0]), (cs, ex * ey, ex, 1), org)

    def spectrum_view(self) -> torch.Tensor:
        """Alias of the plan's half spectrum (Mz, My, Mx//2+1), unscaled."""
        ts = "<f8" if self.precision == "fp64" else "<f4"
        ptr = _lib.lib().esp_spectrum_ptr(self._handle)
        raw = torch.as_tensor(_DevView(ptr, (self.M[2], self.M[1], self.Hx, 2), ts),
                              device="cuda")
        return torch.view_as_complex(raw)

    # -- stages ---------------------------------------------------------------
    @staticmethod
    def _check_particles(pos, q):
        if not (isinstance(pos, torch.Tensor) and pos.is_cuda and pos.dtype == torch.float64):
            raise ParameterError("positions must be a CUDA float64 tensor of shape (N, 3)")
        if not (isinstance(q, torch.Tensor) and q.is_cuda and q.dtype == torch.float64):
            raise ParameterError("charges must be a CUDA float64 tensor of shape (N,)")
        if pos.dim() != 2 or pos.shape[1] != 3 or q.numel() != pos.shape[0]:
            raise ParameterError("positions (N,3) and charges (N,) shapes disagree")
        return pos.contiguous(), q.contiguous()

    def spread(self, pos: torch.Tensor, q: torch.Tensor, stream=None):
        pos, q = self._check_particles(pos, q)
        n = pos.shape[0]
        self.ensure_capacity(n)
        _lib.check(_lib.lib().esp_spread(self._handle, C.c_void_p(pos.data_ptr()),
                                         C.c_void_p(q.data_ptr()), n, None,
                                         _stream_handle(stream)), "esp_spread")
        return self.grid_view()

    def forward(self, grid: torch.Tensor | None = None, stream=None):
        ptr = None
        if grid is not None:
            g = grid.contiguous()
            if g.dtype != self.real_dtype or g.numel() != int(np.prod(self.M)):
                raise ParameterError("grid shape/dtype does not match the plan")
            ptr = C.c_void_p(g.data_ptr())
        _lib.check(_lib.lib().esp_forward(self._handle, ptr, _stream_handle(stream)),
                   "esp_forward")
        self.version += 1

    def set_spectrum(self, spec: torch.Tensor, stream=None):
        s = torch.view_as_real(spec.contiguous()).contiguous()
        _lib.check(_lib.lib().esp_set_spectrum(self._handle, C.c_void_p(s.data_ptr()),
                                               _stream_handle(stream)), "esp_set_spectrum")
        self.version += 1

    def scale_reduce(self, write_ik: bool = False, out7: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
        if out7 is None:
            out7 = torch.empty(7, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().esp_scale_reduce(self._handle, C.c_void_p(out7.data_ptr()),
                                               int(bool(write_ik)), _stream_handle(stream)),
                   "esp_scale_reduce")
        return out7

    def gather_fields(self, fields: torch.Tensor, n: int, forces: torch.Tensor | None = None,
                      stream=None):
        """ik forces from caller fields [3][M2][M1][M0] for the particles of the
        last spread (slab plans: the owned planes plus ghost planes)."""
        f = fields.contiguous()
        if f.dtype != self.real_dtype or f.numel() != 3 * int(np.prod(self.M)):
            raise ParameterError("fields shape/dtype does not match the plan")
        if forces is None:
            forces = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().esp_gather_fields(self._handle, C.c_void_p(f.data_ptr()),
                                                C.c_void_p(forces.data_ptr()),
                                                _stream_handle(stream)), "esp_gather_fields")
        return forces

    def forces_ik(self, n: int, forces: torch.Tensor | None = None, stream=None):
        if forces is None:
            forces = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().esp_forces_ik(self._handle, C.c_void_p(forces.data_ptr()),
                                            _stream_handle(stream)), "esp_forces_ik")
        return forces

    def forces_analytic(self, n: int, forces: torch.Tensor | None = None, stream=None):
        """One inverse transform + window-gradient gather (mesh.py:343-349)."""
        if forces is None:
            forces = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().esp_forces_analytic(self._handle, C.c_void_p(forces.data_ptr()),
                                                  _stream_handle(stream)), "esp_forces_analytic")
        return forces

    def local_pressure(self, n: int, out: torch.Tensor | None = None, stream=None):
        """Per-particle far-field pressure tensors (N,3,3) (mesh.py:353-379)."""
        if out is None:
            out = torch.empty((n, 3, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().esp_local_pressure(self._handle, C.c_void_p(out.data_ptr()),
                                                 _stream_handle(stream)), "esp_local_pressure")
        return out

    def evaluate(self, pos: torch.Tensor, q: torch.Tensor, want_forces: bool = True,
                 out7: torch.Tensor | None = None, forces: torch.Tensor | None = None,
                 stream=None, analytic: bool = False):
        """Whole step on the device: (out7[E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz], F)."""
        pos, q = self._check_particles(pos, q)
        n = pos.shape[0]
        self.ensure_capacity(n)
        if out7 is None:
            out7 = torch.empty(7, dtype=torch.float64, device="cuda")
        if want_forces and forces is None:
            forces = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        flags = _lib.ESP_WANT_ENERGY_PRESSURE | (_lib.ESP_WANT_FORCES if want_forces else 0)
        if analytic:
            flags |= _lib.ESP_FORCES_ANALYTIC
        _lib.check(_lib.lib().esp_evaluate(
            self._handle, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()), n, flags,
            C.c_void_p(out7.data_ptr()),
            C.c_void_p(forces.data_ptr()) if want_forces else None,
            _stream_handle(stream)), "esp_evaluate")
        self.version += 1
        return out7, forces

    def launches_last_step(self) -> int:
        return int(self.info()[5])

    # -- CUDA graphs ---------------------------------------------------------
    def graph(self, pos: torch.Tensor, q: torch.Tensor, want_forces: bool,
              out7: torch.Tensor, forces: torch.Tensor | None, pre=None, post=None,
              analytic: bool = False):
        """Capture one whole step (optionally with caller copies before/after)
        into a CUDA graph and return it; ``g.replay()`` re-runs the step on the
        same buffers with a single launch from the host."""
        pos, q = self._check_particles(pos, q)
        self.ensure_capacity(pos.shape[0])

        def body():
            if pre is not None:
                pre()
            self.evaluate(pos, q, want_forces, out7, forces, analytic=analytic)
            if post is not None:
                post()

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body()                      # warm-up: kernel attributes, cuFFT work areas
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        before = self.counters()
        with torch.cuda.graph(g):
            body()
        torch.cuda.synchronize()
        after = self.counters()
        # the capture counted the step's transforms once; replays add them
        return PlanGraph(g, [self], counted=(self, after[0] - before[0], after[1] - before[1]))

    def set_profiling(self, on: bool = True):
        _lib.check(_lib.lib().esp_set_profiling(self._handle, int(bool(on))), "esp_set_profiling")

    def profile(self):
        """[(kernel name, ms)] of the last profiled esp_evaluate (synchronises)."""
        names = C.create_string_buffer(2048)
        ms = (C.c_double * 48)()
        n = _lib.lib().esp_profile_read(self._handle, names, 2048, ms, 48)
        if n < 0:
            _lib.check(-n, "esp_profile_read")
        labels = names.value.decode().split(",") if n else []
        return list(zip(labels, [float(ms[i]) for i in range(n)]))


class PlanGraph:
    """A captured CUDA graph bound to the plans it was captured on.

    A graph bakes in device addresses (grids, scratch, mode tables) and
    by-value cell constants (spacing, volume).  ``set_cell`` (an NPT rebind)
    re-uploads the cell tables and ``ensure_capacity`` re-creates the plan, so
    a graph captured before either must not replay: ``replay()`` checks each
    plan's generation and raises instead of reading freed memory or the old
    geometry.  Graphs are tied to a fixed N and cell; re-capture after a
    rebind."""

    def __init__(self, graph, plans, counted=None):
        self.graph = graph
        self._deps = [(p, p.generation) for p in plans]
        # (plan, forward, inverse): transforms of one captured step, added to
        # the plan's counters at every replay (the C entries count at call
        # time, i.e. during capture only)
        self._counted = counted

    @property
    def valid(self) -> bool:
        return all(p.generation == g for p, g in self._deps)

    def replay(self):
        if not self.valid:
            raise ParameterError("CUDA graph captured before a cell rebind or capacity growth "
                                 "of its plan; capture it again")
        self.graph.replay()
        if self._counted is not None:
            plan, fwd, inv = self._counted
            if fwd or inv:
                _lib.lib().esp_add_counters(plan._handle, fwd, inv)


def probe_fp64_tflops(stream=None) -> float:
    """Measured FP64 FMA throughput of the current device (TFLOP/s)."""
    out = C.c_double()
    _lib.check(_lib.lib().esp_probe_fp64(C.byref(out), _stream_handle(stream)), "esp_probe_fp64")
    return float(out.value)


def out7_to_tensor(out7) -> np.ndarray:
    """[E, Pxx, Pxy, Pxz, Pyy, Pyz, Pzz] -> (E, 3x3 symmetric)."""
    v = out7.detach().cpu().numpy() if isinstance(out7, torch.Tensor) else np.asarray(out7)
    P = np.array([[v[1], v[2], v[3]], [v[2], v[4], v[5]], [v[3], v[5], v[6]]])
    return float(v[0]), P
