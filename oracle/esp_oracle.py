"""CPU ORACLE for the ESP k-space path — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's
long-range (k-space) pipeline, arXiv 2601.00161, ``prolate_ewald``
(``/root/reference/pkg/src/prolate_ewald``).  It is the parity checker for
the CUDA product path (k-space, and the near-field pair sum of
realspace.py / system.py, L3 below) and the timed CPU leg of ``bench.py``
(``cpu_baseline`` / ``--impl reference``, ``kind: "port"``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU leg may
import it; the product package never does.

Pinning: the orthorhombic functions are checked against golden vectors
produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``,
``tests/test_oracle_golden.py``).  The triclinic extension (the reference
mesh refuses non-orthorhombic cells, ``mesh.py:94-95``) is pinned two ways:
it reduces to the orthorhombic code path's numbers on orthorhombic cells,
and it matches the exact gridless mode sum (restated from
``oracle.py:60-106`` and checked against the reference's ``direct_ksum``
goldens) to Δ-level on small skewed cells.

Array conventions follow the reference: grids are C-order [x][y][z]
(z contiguous), positions (N,3) f64, charges (N,) f64.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numpy.polynomial import legendre as npleg
from scipy.interpolate import PPoly
from scipy.linalg import eigh_tridiagonal
from scipy.optimize import brentq

# --------------------------------------------------------------------------
# L0: order-zero prolate psi_0^c  (pswf.py)


def legendre_coefficients(c: float) -> np.ndarray:
    """psi_0^c as a Legendre series (pswf.py:41-84): smallest eigenvector of
    the even block of the prolate differential operator in the normalised
    Legendre basis, doubled until the tail decays below 1e-16."""
    n = max(int(np.ceil(c)) + 16, 40)
    for _ in range(8):
        k = 2.0 * np.arange(n)
        cc = c * c
        d = k * (k + 1.0) + cc * (2.0 * k * (k + 1.0) - 1.0) / (
            (2.0 * k + 3.0) * (2.0 * k - 1.0))
        kk = k[:-1]
        e = cc * (kk + 2.0) * (kk + 1.0) / (
            (2.0 * kk + 3.0) * np.sqrt((2.0 * kk + 1.0) * (2.0 * kk + 5.0)))
        _, v = eigh_tridiagonal(d, e, select="i", select_range=(0, 0))
        beta = v[:, 0]
        if np.max(np.abs(beta[-4:])) / np.max(np.abs(beta)) < 1e-16:
            break
        n *= 2
    else:
        raise ArithmeticError(f"prolate expansion did not converge for c={c}")
    coef = np.zeros(2 * n - 1)
    coef[::2] = beta * np.sqrt((2.0 * k + 1.0) / 2.0)
    big = np.max(np.abs(coef))
    last = np.nonzero(np.abs(coef) > 1e-17 * big)[0][-1]
    coef = coef[: last + 1]
    if npleg.legval(0.0, coef) < 0.0:
        coef = -coef
    return coef


def solve_bandwidth(delta: float) -> float:
    """c with psi_0^c(1) = delta (pswf.py:225-235)."""
    def g(c):
        return np.log(max(float(npleg.legval(1.0, legendre_coefficients(c))),
                          1e-290)) - np.log(delta)
    return float(brentq(g, 0.5, 80.0, xtol=1e-9, rtol=1e-10))


def _piecewise_table(fun, degree, n_int, lo, hi) -> PPoly:
    """Chebyshev-node interpolants per uniform piece, stored as monomials in
    (x - left) (pswf.py:87-107)."""
    edges = np.linspace(lo, hi, n_int + 1)
    width = edges[1] - edges[0]
    nodes = np.cos(np.pi * (2.0 * np.arange(degree + 1) + 1.0) / (2.0 * (degree + 1)))
    table = np.empty((degree + 1, n_int))
    to_local = np.polynomial.Polynomial([-1.0, 2.0 / width])
    for i in range(n_int):
        x = edges[i] + 0.5 * width * (nodes + 1.0)
        fit = np.polynomial.chebyshev.Chebyshev.fit(nodes, fun(x), degree, domain=[-1, 1])
        mono = fit.convert(kind=np.polynomial.Polynomial)(to_local)
        col = np.zeros(degree + 1)
        col[: mono.coef.size] = mono.coef
        table[:, i] = col[::-1]
    return PPoly(table, edges, extrapolate=False)


@dataclass(frozen=True)
class Basis:
    """Subset of ``PswfBasis`` (pswf.py:123-193) the k-space path consumes."""
    c: float
    coef: np.ndarray
    lambda0: float
    psi0_at_zero: float
    C0: float

    def psi(self, x, derivative=0):
        co = npleg.legder(self.coef, derivative) if derivative else self.coef
        return npleg.legval(np.asarray(x, dtype=float), co)


def build_basis(c: float) -> Basis:
    """pswf.py:155-193 (value quantities only; tables are built per window)."""
    coef = legendre_coefficients(c)
    psi00 = float(npleg.legval(0.0, coef))
    gx, gw = np.polynomial.legendre.leggauss(64)
    C0 = float(0.5 * np.sum(gw * npleg.legval(0.5 * (gx + 1.0), coef)))
    return Basis(c=float(c), coef=coef, lambda0=2.0 * C0 / psi00,
                 psi0_at_zero=psi00, C0=C0)


@dataclass(frozen=True)
class Window:
    """W(t) = psi_0^c(2t/P) on [-P/2, P/2] (pswf.py:238-293)."""
    P: int
    value: PPoly
    deriv: PPoly

    def __call__(self, t, derivative=0):
        out = (self.deriv if derivative else self.value)(np.asarray(t, dtype=float))
        return np.nan_to_num(out, nan=0.0, posinf=0.0, neginf=0.0)


def build_window(basis: Basis, P: int, tol: float = 1e-13, degree: int = 18) -> Window:
    half, scale = P / 2.0, 2.0 / P
    dco = npleg.legder(basis.coef)

    def w(x):
        return npleg.legval(np.clip(np.asarray(x) * scale, -1.0, 1.0), basis.coef)

    def wd(x):
        return npleg.legval(np.clip(np.asarray(x) * scale, -1.0, 1.0), dco) * scale

    pieces = 1
    for _ in range(8):
        val = _piecewise_table(w, degree, P * pieces, -half, half)
        der = _piecewise_table(wd, degree, P * pieces, -half, half)
        xs = np.linspace(-half, half, 4097)
        if np.max(np.abs(val(xs) - w(xs))) / basis.psi0_at_zero <= tol:
            return Window(P=int(P), value=val, deriv=der)
        pieces *= 2
    raise ArithmeticError("window table did not converge")


# --------------------------------------------------------------------------
# Geometry / plan  (mesh.py:58-142, generalised to triclinic lattices)


@dataclass(frozen=True)
class Plan:
    h: np.ndarray          # 3x3 columns = cell vectors
    M: tuple
    P: int
    split: Basis
    spread: Basis
    window: Window
    r_c: float

    @property
    def orthorhombic(self) -> bool:
        off = self.h - np.diag(np.diag(self.h))
        return bool(np.all(np.abs(off) <= 1e-12 * np.max(np.abs(self.h))))

    @property
    def kmax(self) -> float:
        return self.split.c / self.r_c              # kernel.py:28-39

    @property
    def volume(self) -> float:
        return float(np.linalg.det(self.h))

    @property
    def lengths(self):
        return np.diag(self.h)

    @property
    def spacing(self):
        return self.lengths / np.asarray(self.M)       # mesh.py:109

    @property
    def omega(self):
        return self.P * self.spacing / 2.0           # mesh.py:110

    @property
    def volume_element(self) -> float:
        """h_x h_y h_z (mesh.py:77-78); V/G on a triclinic lattice."""
        if self.orthorhombic:
            return float(np.prod(self.spacing))
        return self.volume / float(np.prod(self.M))


def make_plan(h, M, P, delta_split, r_c, delta_spread=None) -> Plan:
    h = np.asarray(h, dtype=float).reshape(3, 3)
    split = build_basis(solve_bandwidth(delta_split))
    spread = split if delta_spread is None or delta_spread == delta_split \
        else build_basis(solve_bandwidth(delta_spread))
    plan = Plan(h=h, M=tuple(int(m) for m in M), P=int(P), split=split,
                spread=spread, window=build_window(spread, P), r_c=float(r_c))
    check_plan(plan)
    return plan


def check_plan(plan: Plan) -> None:
    """Nyquist / band / support invariants (mesh.py:117-130); on a triclinic
    lattice |h_d| (column norm) replaces L_d."""
    norms = np.linalg.norm(plan.h, axis=0)
    kmax = plan.kmax
    for d in range(3):
        hd = norms[d] / plan.M[d]
        om = plan.P * hd / 2.0
        if np.pi / hd < kmax * (1.0 - 1e-12):
            raise ValueError(f"Nyquist coverage violated in dimension {d}")
        if plan.spread.c / om < kmax * (1.0 - 1e-12):
            raise ValueError(f"window band coverage violated in dimension {d}")
        if 2.0 * om >= norms[d]:
            raise ValueError(f"window support violated in dimension {d}")


def grid_coordinates(plan: Plan, pos: np.ndarray) -> np.ndarray:
    """u_d: particle position in grid units along lattice axis d.

    Orthorhombic: u = x / h_d exactly as mesh.py:160.  Triclinic: u_d =
    M_d * (h^{-1} r)_d, written out term by term (fixed operation order the
    CUDA kernel mirrors)."""
    pos = np.asarray(pos, dtype=float)
    if plan.orthorhombic:
        return pos / plan.spacing[None, :]
    hi = np.linalg.inv(plan.h)
    u = np.empty_like(pos)
    for d in range(3):
        s = (hi[d, 0] * pos[:, 0] + hi[d, 1] * pos[:, 1]) + hi[d, 2] * pos[:, 2]
        u[:, d] = s * float(plan.M[d])
    return u


# --------------------------------------------------------------------------
# Stencils, spreading, gathering (mesh.py:154-218)


def stencil(u_d: np.ndarray, M: int, P: int):
    """Nearest node (odd P, round-half-even) or left node (even P) anchors the
    P-point stencil; returns (N,P) wrapped indices and offsets t = u - node."""
    if P % 2:
        base = np.round(u_d)
        p = np.arange(-(P // 2), P // 2 + 1)
    else:
        base = np.floor(u_d)
        p = np.arange(-(P // 2 - 1), P // 2 + 1)
    nodes = base[:, None] + p[None, :]
    return np.mod(nodes.astype(np.int64), M), u_d[:, None] - nodes


def _weights(plan: Plan, u: np.ndarray, deriv_dim: int = -1):
    idx, wts = [], []
    for d in range(3):
        i, t = stencil(u[:, d], plan.M[d], plan.P)
        if d == deriv_dim:
            hd = plan.spacing[d] if plan.orthorhombic else None
            if hd is None:
                raise NotImplementedError("analytic gradient is orthorhombic only")
            w = plan.window(t, derivative=1) / hd
        else:
            w = plan.window(t)
        idx.append(i)
        wts.append(w)
    return idx, wts


def _flat(idx, M):
    ix, iy, iz = idx
    return ((ix[:, :, None, None] * M[1] + iy[:, None, :, None]) * M[2]
            + iz[:, None, None, :]).reshape(ix.shape[0], -1)


def _outer(w):
    wx, wy, wz = w
    return (wx[:, :, None, None] * wy[:, None, :, None]
            * wz[:, None, None, :]).reshape(wx.shape[0], -1)


def spread(plan: Plan, pos, q, chunk: int = 200_000) -> np.ndarray:
    """rho_grid = bincount(flat, q w) (mesh.py:204-210), chunked over
    particles (exact by linearity up to summation order)."""
    G = int(np.prod(plan.M))
    u = grid_coordinates(plan, pos)
    q = np.asarray(q, dtype=float)
    rho = np.zeros(G)
    for s in range(0, u.shape[0], chunk):
        idx, w = _weights(plan, u[s:s + chunk])
        vals = _outer(w) * q[s:s + chunk, None]
        part = np.bincount(_flat(idx, plan.M).ravel(), weights=vals.ravel(), minlength=G)
        rho = part if s == 0 else rho + part
    return rho.reshape(plan.M)


def gather(plan: Plan, field: np.ndarray, pos, deriv_dim: int = -1,
           chunk: int = 200_000) -> np.ndarray:
    """sum over the P^3 stencil of field x weight (mesh.py:213-218)."""
    u = grid_coordinates(plan, pos)
    flatf = np.asarray(field).reshape(-1)
    out = np.empty(u.shape[0])
    for s in range(0, u.shape[0], chunk):
        idx, w = _weights(plan, u[s:s + chunk], deriv_dim)
        out[s:s + chunk] = np.einsum("np,np->n", flatf[_flat(idx, plan.M)], _outer(w))
    return out


def forward_density(plan: Plan, pos, q) -> np.ndarray:
    """rho_hat = volume_element * fftn(rho_grid) (mesh.py:221-226)."""
    return np.fft.fftn(spread(plan, pos, q)) * plan.volume_element


# --------------------------------------------------------------------------
# Mode workspace (mesh.py:229-282, generalised)


def axis_wavenumbers(plan: Plan):
    """K[a][d]: Cartesian component a of the wavevector contributed by the
    index along lattice axis d, so k_a = K[a][0][mx] + K[a][1][my] +
    K[a][2][mz].  Orthorhombic: the reference's 2*pi*fftfreq(M, 1/M)/L
    (mesh.py:242) on the diagonal and exact zeros elsewhere."""
    freqs = [np.fft.fftfreq(plan.M[d], d=1.0 / plan.M[d]) for d in range(3)]
    K = [[np.zeros(plan.M[d]) for d in range(3)] for _ in range(3)]
    if plan.orthorhombic:
        for d in range(3):
            K[d][d] = 2.0 * np.pi * freqs[d] / plan.lengths[d]
    else:
        B = 2.0 * np.pi * np.linalg.inv(plan.h).T   # reciprocal columns (system.py:20-26)
        for a in range(3):
            for d in range(3):
                K[a][d] = B[a, d] * freqs[d]
    return K


def axis_window_factors(plan: Plan):
    """Per-axis window transforms whose product (a0*a1)*a2 is What(m).
    Orthorhombic: omega_d lambda0 psi(clip(omega_d k_d / c)) (mesh.py:258-261).
    Triclinic: V folded into axis 0 and omega_d k_d = pi P m_d / M_d."""
    sb = plan.spread
    K = axis_wavenumbers(plan)
    out = []
    if plan.orthorhombic:
        for d in range(3):
            arg = plan.omega[d] * K[d][d] / sb.c
            out.append(plan.omega[d] * sb.lambda0 * sb.psi(np.clip(arg, -1, 1)))
    else:
        for d in range(3):
            f = np.fft.fftfreq(plan.M[d], d=1.0 / plan.M[d])
            arg = np.pi * plan.P * f / (plan.M[d] * sb.c)
            a = (plan.P / (2.0 * plan.M[d])) * sb.lambda0 * sb.psi(np.clip(arg, -1, 1))
            out.append(plan.volume * a if d == 0 else a)
    return out


class Modes:
    """mask, kvec, k2, w_inv2, fhat, dterm over retained modes (mesh.py:237-275)."""

    def __init__(self, plan: Plan):
        self.volume = plan.volume
        K = axis_wavenumbers(plan)
        M = plan.M
        kv = []
        for a in range(3):
            kv.append(K[a][0][:, None, None] + K[a][1][None, :, None]
                      + K[a][2][None, None, :])
        kx, ky, kz = [np.broadcast_to(k, M) for k in kv]
        k2 = kx ** 2 + ky ** 2 + kz ** 2
        kmag = np.sqrt(k2)
        mask = (kmag <= plan.kmax) & (k2 > 0.0)
        self.mask = mask
        self.kvec = [kx[mask], ky[mask], kz[mask]]
        self.k2 = k2[mask]
        kmag = kmag[mask]
        A = axis_window_factors(plan)
        what = (A[0][:, None, None] * A[1][None, :, None]) * A[2][None, None, :]
        what = np.broadcast_to(what, M)[mask]
        sb = plan.spread
        if plan.orthorhombic:
            w0 = float(np.prod([w * sb.lambda0 * sb.psi0_at_zero for w in plan.omega]))
        else:
            w0 = plan.volume * float(np.prod([(plan.P / (2.0 * m)) * sb.lambda0
                                              * sb.psi0_at_zero for m in M]))
        if np.any(np.abs(what) < 1e-13 * abs(w0)):
            raise ValueError("window transform underflow on a retained mode")
        self.w_inv2 = 1.0 / (what * what)
        b = plan.split
        x = np.clip(kmag * plan.r_c / b.c, 0.0, 1.0)
        pref = 2.0 * np.pi * b.lambda0 / b.C0
        self.fhat = pref * b.psi(x) / self.k2
        self.dterm = pref * x * b.psi(x, derivative=1) / self.k2 ** 2

    def pressure_component(self, a, b):
        kk = self.kvec[a] * self.kvec[b]
        out = self.dterm * kk - 2.0 * self.fhat * kk / self.k2
        return out + self.fhat if a == b else out


# --------------------------------------------------------------------------
# Spectral reductions and forces (mesh.py:285-379)


def energy(modes: Modes, rho_hat) -> float:
    amp2 = np.abs(rho_hat[modes.mask]) ** 2
    return float(np.sum(modes.fhat * modes.w_inv2 * amp2) / (2.0 * modes.volume))


def pressure(modes: Modes, rho_hat) -> np.ndarray:
    amp2 = np.abs(rho_hat[modes.mask]) ** 2
    scaled = modes.w_inv2 * amp2 / (2.0 * modes.volume ** 2)
    out = np.empty((3, 3))
    for a in range(3):
        for b in range(a, 3):
            out[a, b] = out[b, a] = float(np.sum(modes.pressure_component(a, b) * scaled))
    return out


def forces_ik(plan: Plan, modes: Modes, rho_hat, pos, q) -> np.ndarray:
    h3 = plan.volume_element
    scale = modes.fhat * modes.w_inv2 * rho_hat[modes.mask]
    q = np.asarray(q, dtype=float)
    F = np.empty((q.size, 3))
    for d in range(3):
        spec = np.zeros(plan.M, dtype=complex)
        spec[modes.mask] = 1j * modes.kvec[d] * scale
        fld = np.fft.ifftn(spec).real / h3
        F[:, d] = -q * h3 * gather(plan, fld, pos)
    return F


def forces_analytic(plan: Plan, modes: Modes, rho_hat, pos, q) -> np.ndarray:
    h3 = plan.volume_element
    spec = np.zeros(plan.M, dtype=complex)
    spec[modes.mask] = modes.fhat * modes.w_inv2 * rho_hat[modes.mask]
    fld = np.fft.ifftn(spec).real / h3
    q = np.asarray(q, dtype=float)
    return np.stack([-q * h3 * gather(plan, fld, pos, deriv_dim=d) for d in range(3)], axis=1)


def local_pressure(plan: Plan, modes: Modes, rho_hat, pos, q) -> np.ndarray:
    h3 = plan.volume_element
    base = modes.w_inv2 * rho_hat[modes.mask]
    q = np.asarray(q, dtype=float)
    out = np.empty((q.size, 3, 3))
    for a in range(3):
        for b in range(a, 3):
            spec = np.zeros(plan.M, dtype=complex)
            spec[modes.mask] = modes.pressure_component(a, b) * base
            fld = np.fft.ifftn(spec).real / h3
            comp = q * h3 * gather(plan, fld, pos) / (2.0 * modes.volume)
            out[:, a, b] = out[:, b, a] = comp
    return out


def kspace(plan: Plan, pos, q, want_forces=True, modes: Modes | None = None):
    """(E, P[3,3], F or None) — the path the CUDA product computes."""
    modes = modes or Modes(plan)
    rh = forward_density(plan, pos, q)
    E = energy(modes, rh)
    Pt = pressure(modes, rh)
    F = forces_ik(plan, modes, rh, pos, q) if want_forces else None
    return E, Pt, F


# --------------------------------------------------------------------------
# Exact gridless mode sum (oracle.py:60-106): pins the triclinic extension.


def direct_ksum(h, kmax, split: Basis, r_c, pos, q):
    h = np.asarray(h, dtype=float)
    B = 2.0 * np.pi * np.linalg.inv(h).T
    mmax = np.ceil(kmax * np.linalg.norm(h, axis=0) / (2.0 * np.pi)).astype(int)
    g = np.meshgrid(*[np.arange(-m, m + 1) for m in mmax], indexing="ij")
    m = np.stack([x.ravel() for x in g], axis=1)
    m = m[np.any(m != 0, axis=1)]
    k = m @ B.T
    k = k[np.einsum("ij,ij->i", k, k) <= kmax * kmax]
    V = float(np.linalg.det(h))
    q = np.asarray(q, dtype=float)
    ekr = np.exp(1j * (k @ np.asarray(pos, dtype=float).T))
    rho = (q[None, :] * ekr).sum(axis=1)
    kmag = np.linalg.norm(k, axis=1)
    x = np.clip(kmag * r_c / split.c, 0.0, 1.0)
    pref = 2.0 * np.pi * split.lambda0 / split.C0
    fhat = pref * split.psi(x) / kmag ** 2
    amp2 = np.abs(rho) ** 2
    E = float(np.sum(fhat * amp2) / (2.0 * V))
    im = np.imag(np.conj(ekr) * rho[:, None])
    F = -((fhat[:, None] * im).T @ k) * q[:, None] / V
    dterm = pref * x * split.psi(x, derivative=1) / kmag ** 4
    w = amp2 / (2.0 * V ** 2)
    Pt = np.einsum("k,ka,kb->ab", (dterm - 2.0 * fhat / kmag ** 2) * w, k, k)
    Pt += np.sum(fhat * w) * np.eye(3)
    return E, F, 0.5 * (Pt + Pt.T)


# --------------------------------------------------------------------------
# L3: near field — pair table, pair enumeration, fused pair sum
# (realspace.py:29-157, kernel.py:41-97, system.py:75-222).  Pinned to the
# reference by tests/golden/near_*.npz (tests/test_oracle_golden.py).


def phi0(basis: Basis, r, r_c):
    """eval_phi0 (pswf.py:277-292): (1/C0) int_0^{min(r/r_c,1)} psi_0; 1 at r >= r_c."""
    r = np.asarray(r, dtype=float)
    x = np.minimum(r / r_c, 1.0)
    out = npleg.legval(x, npleg.legint(basis.coef, lbnd=0.0)) / basis.C0
    return np.where(r >= r_c, 1.0, out)


def near_value(basis: Basis, r_c, r):
    """near_field (kernel.py:41-50) for r > 0."""
    r = np.atleast_1d(np.asarray(r, dtype=float))
    out = np.zeros_like(r)
    inside = r < r_c
    out[inside] = (1.0 - phi0(basis, r[inside], r_c)) / r[inside]
    return out


def far_value(basis: Basis, r_c, r):
    """far_field (kernel.py:53-65)."""
    r = np.atleast_1d(np.asarray(r, dtype=float))
    out = np.empty_like(r)
    z = r == 0.0
    out[~z] = phi0(basis, r[~z], r_c) / r[~z]
    out[z] = basis.psi0_at_zero / (basis.C0 * r_c)
    return out


def fn_value(basis: Basis, r_c, r):
    """fn_weight (kernel.py:83-97)."""
    r = np.asarray(r, dtype=float)
    x = np.minimum(r / r_c, 1.0)
    val = 1.0 - phi0(basis, r, r_c) + (r / (basis.C0 * r_c)) * basis.psi(x)
    return np.where(r > r_c, 0.0, val)


@dataclass(frozen=True)
class PairTableO:
    r_in: float
    r_c: float
    smooth: np.ndarray
    fn: np.ndarray
    smooth_spline: object
    fn_spline: object


def pair_table(basis: Basis, r_c, r_in=None, resolution=4096, order=8) -> PairTableO:
    """build_pair_table (realspace.py:70-112)."""
    from scipy.interpolate import CubicSpline
    r_in = 0.1 * r_c if r_in is None else r_in
    s = np.cos(np.pi * (2.0 * np.arange(order + 1) + 1.0) / (2.0 * (order + 1)))
    for _ in range(12):
        nodes = 0.5 * r_in * (s + 1.0)
        smooth = np.polynomial.Polynomial.fit(nodes, far_value(basis, r_c, nodes), order,
                                              domain=[0.0, r_in]).convert().coef
        fnc = np.polynomial.Polynomial.fit(nodes, fn_value(basis, r_c, np.maximum(nodes, 1e-300)),
                                           order, domain=[0.0, r_in]).convert().coef
        probe = np.linspace(1e-6 * r_c, r_in, 512)
        err = np.max(np.abs(np.polynomial.polynomial.polyval(probe, smooth)
                            - far_value(basis, r_c, probe))) / far_value(basis, r_c, 0.0)[0]
        if err <= 1e-11:
            break
        r_in *= 0.5
    else:
        raise ArithmeticError("inner-cutoff polynomial fit did not converge")
    knots = np.linspace(r_in, r_c, resolution)
    pad = np.zeros(order + 1)
    pad[: smooth.size] = smooth
    fpad = np.zeros(order + 1)
    fpad[: fnc.size] = fnc
    return PairTableO(r_in=float(r_in), r_c=float(r_c), smooth=pad, fn=fpad,
                      smooth_spline=CubicSpline(knots, far_value(basis, r_c, knots)),
                      fn_spline=CubicSpline(knots, fn_value(basis, r_c, knots)))


def table_values(t: PairTableO, r):
    """PairTable.near_field / fn_weight (realspace.py:42-67)."""
    r = np.asarray(r, dtype=float)
    nv = np.empty_like(r)
    fv = np.empty_like(r)
    lo = r <= t.r_in
    hi = ~lo
    pv = np.polynomial.polynomial.polyval
    nv[lo] = 1.0 / r[lo] - pv(r[lo], t.smooth)
    nv[hi] = 1.0 / r[hi] - t.smooth_spline(np.minimum(r[hi], t.r_c))
    nv[r >= t.r_c] = 0.0
    fv[lo] = pv(r[lo], t.fn)
    fv[hi] = t.fn_spline(np.minimum(r[hi], t.r_c))
    fv[r > t.r_c] = 0.0
    return nv, fv


def minimum_image(h, dr):
    """system.py:75-79."""
    h = np.asarray(h, dtype=float)
    s = np.asarray(dr, dtype=float) @ np.linalg.inv(h).T
    s -= np.floor(s + 0.5)
    return s @ h.T


def pairs_within(h, pos, reach, chunk=2048):
    """All unordered pairs (i < j) with minimum-image distance <= reach, sorted
    by (i, j) — the pair set of build_cell_list (system.py:144-222), by brute
    force in row chunks (small N only)."""
    pos = np.asarray(pos, dtype=float)
    n = pos.shape[0]
    I, J = [], []
    for a in range(0, n, chunk):
        rows = np.arange(a, min(n, a + chunk))
        dr = minimum_image(h, pos[rows, None, :] - pos[None, :, :])
        r2 = np.einsum("abk,abk->ab", dr, dr)
        ii, jj = np.nonzero((r2 <= reach * reach) & (rows[:, None] < np.arange(n)[None, :]))
        I.append(rows[ii])
        J.append(jj)
    i = np.concatenate(I) if I else np.zeros(0, dtype=np.int64)
    j = np.concatenate(J) if J else np.zeros(0, dtype=np.int64)
    o = np.lexsort((j, i))
    return i[o].astype(np.int64), j[o].astype(np.int64)


def pairs_within_kdtree(L, pos, reach):
    """Orthorhombic pair set as the reference builds it (system.py:151-166,
    periodic cKDTree)."""
    from scipy.spatial import cKDTree
    L = np.asarray(L, dtype=float)
    p = np.maximum(np.minimum(np.asarray(pos, dtype=float), np.nextafter(L, 0.0)), 0.0)
    pairs = cKDTree(p, boxsize=L).query_pairs(reach, output_type="ndarray")
    if pairs.size == 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.int64)
    i = np.minimum(pairs[:, 0], pairs[:, 1])
    j = np.maximum(pairs[:, 0], pairs[:, 1])
    o = np.lexsort((j, i))
    return i[o].astype(np.int64), j[o].astype(np.int64)


def short_range(h, pos, q, i, j, basis: Basis, r_c, table: PairTableO | None = None,
                chunk=4_000_000):
    """realspace.short_range (realspace.py:115-157): returns (E, F, P, pairs)."""
    h = np.asarray(h, dtype=float)
    pos = np.asarray(pos, dtype=float)
    q = np.asarray(q, dtype=float)
    n = pos.shape[0]
    F = np.zeros((n, 3))
    E = 0.0
    V = float(np.linalg.det(h))
    W = np.zeros((3, 3))
    count = 0
    for a in range(0, len(i), chunk):
        ii, jj = i[a:a + chunk], j[a:a + chunk]
        dr = minimum_image(h, pos[ii] - pos[jj])
        r = np.sqrt(np.einsum("ij,ij->i", dr, dr))
        if np.any(r < 1e-12 * r_c):
            raise ZeroDivisionError("coincident particles")
        keep = r <= r_c
        ii, jj, dr, r = ii[keep], jj[keep], dr[keep], r[keep]
        qq = q[ii] * q[jj]
        if table is not None:
            nv, fv = table_values(table, r)
        else:
            nv, fv = near_value(basis, r_c, r), fn_value(basis, r_c, r)
        E += float(np.sum(qq * nv))
        fmag = qq * fv / r ** 3
        pf = fmag[:, None] * dr
        np.add.at(F, ii, pf)
        np.add.at(F, jj, -pf)
        W += (dr.T * fmag) @ dr
        count += int(r.size)
    P = W / V
    return E, F, 0.5 * (P + P.T), count


def short_range_rows(h, pos, q, rows, basis: Basis, r_c, table: PairTableO | None = None):
    """Near-field forces on the particles ``rows`` only, against every other
    particle by brute force (size-independent check at large N)."""
    pos = np.asarray(pos, dtype=float)
    q = np.asarray(q, dtype=float)
    out = np.zeros((len(rows), 3))
    for k, a in enumerate(rows):
        dr = minimum_image(h, pos[a] - pos)
        r = np.sqrt(np.einsum("ij,ij->i", dr, dr))
        m = (r <= r_c) & (np.arange(pos.shape[0]) != a)
        r, dr = r[m], dr[m]
        nv, fv = table_values(table, r) if table is not None else (
            near_value(basis, r_c, r), fn_value(basis, r_c, r))
        out[k] = np.sum((q[a] * q[m] * fv / r ** 3)[:, None] * dr, axis=0)
    return out


# --------------------------------------------------------------------------
# Parity metrics (oracle.py:43-48)


def rel_frobenius(a, b) -> float:
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = max(np.linalg.norm(a.ravel()), np.linalg.norm(b.ravel()), 1e-300)
    return float(np.linalg.norm((a - b).ravel()) / den)


def rms_rel_forces(F, Fref) -> float:
    F = np.asarray(F, dtype=float)
    Fref = np.asarray(Fref, dtype=float)
    num = np.sqrt(np.mean(np.sum((F - Fref) ** 2, axis=1)))
    den = np.sqrt(np.mean(np.sum(Fref ** 2, axis=1)))
    return float(num / max(den, 1e-300))


def rel_scalar(a, b) -> float:
    return abs(float(a) - float(b)) / max(abs(float(b)), 1e-300)
