"""Splitting-kernel constants used by the k-space path
(reference: prolate_ewald/kernel.py).

Host-side quantities: ``kmax = c / r_c`` (kernel.py:28-39), the far-field
transform Fhat (kernel.py:68-80, host diagnostics — the device computes it
per retained mode), the radial split functions near_field / far_field /
fn_weight (kernel.py:41-97; used to tabulate the pair table, the device pair
kernels evaluate them per pair), the self energy (kernel.py:117-123) and the
uniform-background correction (kernel.py:126-150).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numpy.polynomial import legendre as L

from .errors import DomainError
from .pswf import PswfBasis


class KernelError(Exception):
    pass


class ZeroModeError(KernelError):
    """The k = 0 mode is excluded under the conducting-boundary convention."""


@dataclass(frozen=True)
class SplitKernel:
    basis: PswfBasis
    r_c: float
    kmax: float = field(init=False)

    def __post_init__(self):
        if self.r_c <= 0.0:
            raise KernelError("cutoff r_c must be positive")
        object.__setattr__(self, "kmax", self.basis.c / self.r_c)


def far_field_hat(kern: SplitKernel, k):
    """2 pi lambda0 psi0(k r_c / c) / (C0 k^2) on |k| <= kmax, else 0."""
    ka = np.atleast_1d(np.asarray(k, dtype=float))
    if np.any(ka == 0.0):
        raise ZeroModeError("k = 0 is excluded (conducting boundary convention)")
    b = kern.basis
    x = ka * kern.r_c / b.c
    out = np.zeros_like(ka)
    band = x <= 1.0
    out[band] = 2.0 * np.pi * b.lambda0 / b.C0 * b.psi_series(x[band]) / ka[band] ** 2
    return float(out[0]) if np.ndim(k) == 0 else out


def phi0(basis: PswfBasis, r, r_c: float):
    """(1/C0) int_0^{r/r_c} psi_0 ; 1 beyond the cutoff."""
    if r_c <= 0.0:
        raise DomainError("cutoff r_c must be positive")
    ra = np.asarray(r, dtype=float)
    x = np.minimum(ra / r_c, 1.0)
    out = L.legval(x, L.legint(basis.legendre_coeffs, lbnd=0.0)) / basis.C0
    return np.where(ra >= r_c, 1.0, out)


def eval_phi0(basis: PswfBasis, r, r_c: float):
    """Normalized cumulative integral phi_0(r) (pswf.py:277-292): DomainError
    for r < 0 or r_c <= 0; 1 for r >= r_c."""
    if r_c <= 0.0:
        raise DomainError("cutoff r_c must be positive")
    ra = np.asarray(r, dtype=float)
    if np.any(ra < 0.0):
        raise DomainError("radius must be nonnegative")
    out = phi0(basis, ra, r_c)
    return out if out.ndim else float(out)


def pressure_kernel_hat(kern: SplitKernel, kvec) -> np.ndarray:
    """Mode-by-mode 3x3 pressure kernel of one wavevector (kernel.py:99-114;
    host reference for the per-mode table the device builds)."""
    kv = np.asarray(kvec, dtype=float)
    k2 = float(kv @ kv)
    if k2 == 0.0:
        raise ZeroModeError("k = 0 is excluded from the pressure kernel")
    k = np.sqrt(k2)
    if k > kern.kmax:
        return np.zeros((3, 3))
    b = kern.basis
    x = min(k * kern.r_c / b.c, 1.0)
    fhat = far_field_hat(kern, k)
    kk = np.outer(kv, kv)
    pref = 2.0 * np.pi * b.lambda0 / b.C0
    dterm = pref * x * b.psi_series(x, derivative=1) / k2 ** 2
    return fhat * (np.eye(3) - 2.0 * kk / k2) + dterm * kk


def background_integral(kern: SplitKernel, n_nodes: int = 128) -> float:
    """J = r_c^2/2 - int_0^{r_c} r phi_0(r) dr by fixed Gauss-Legendre
    (kernel.py:126-134)."""
    nodes, weights = np.polynomial.legendre.leggauss(n_nodes)
    r = 0.5 * kern.r_c * (nodes + 1.0)
    w = 0.5 * kern.r_c * weights
    return 0.5 * kern.r_c ** 2 - float(np.sum(w * r * phi0(kern.basis, r, kern.r_c)))


def cumint_coeffs(basis: PswfBasis) -> np.ndarray:
    """Legendre coefficients of int_0^x psi_0 (pswf.py:144-160, legint lbnd=0)."""
    return L.legint(basis.legendre_coeffs, lbnd=0.0)


def near_field(kern: SplitKernel, r):
    """(1 - phi_0(r)) / r on (0, r_c]; zero beyond (kernel.py:41-50)."""
    scalar = np.isscalar(r) or np.ndim(r) == 0
    ra = np.atleast_1d(np.asarray(r, dtype=float))
    if np.any(ra <= 0.0):
        raise DomainError("near_field requires r > 0 (self-pairs are excluded)")
    out = np.zeros_like(ra)
    inside = ra < kern.r_c
    out[inside] = (1.0 - phi0(kern.basis, ra[inside], kern.r_c)) / ra[inside]
    return float(out[0]) if scalar else out


def far_field(kern: SplitKernel, r):
    """phi_0(r) / r, psi_0(0) / (C0 r_c) at r = 0 (kernel.py:53-65)."""
    scalar = np.isscalar(r) or np.ndim(r) == 0
    ra = np.atleast_1d(np.asarray(r, dtype=float))
    if np.any(ra < 0.0):
        raise DomainError("far_field requires r >= 0")
    b = kern.basis
    out = np.empty_like(ra)
    zero = ra == 0.0
    out[~zero] = phi0(b, ra[~zero], kern.r_c) / ra[~zero]
    out[zero] = b.psi0_at_zero / (b.C0 * kern.r_c)
    return float(out[0]) if scalar else out


def fn_weight(kern: SplitKernel, r):
    """F_N(r) = 1 - phi_0(r) + (r / (C0 r_c)) psi_0(r / r_c); 0 beyond r_c
    (kernel.py:83-97)."""
    ra = np.asarray(r, dtype=float)
    if np.any(ra <= 0.0):
        raise DomainError("fn_weight requires r > 0")
    b = kern.basis
    x = np.minimum(ra / kern.r_c, 1.0)
    val = 1.0 - phi0(b, ra, kern.r_c) + (ra / (b.C0 * kern.r_c)) * b.psi_series(x)
    out = np.where(ra > kern.r_c, 0.0, val)
    return out if out.ndim else float(out)


def self_energy(kern: SplitKernel, charges) -> float:
    q = np.asarray(charges, dtype=float)
    if q.size == 0:
        return 0.0
    b = kern.basis
    return float(-(b.psi0_at_zero / (2.0 * b.C0 * kern.r_c)) * np.sum(q * q))


def background_correction(kern: SplitKernel, q_total: float, volume: float):
    """(U_cb, U_bb, P_corr) for a non-neutral cell; zeros when neutral."""
    if volume <= 0.0:
        raise KernelError("volume must be positive")
    if q_total == 0.0:
        return 0.0, 0.0, np.zeros((3, 3))
    nodes, weights = np.polynomial.legendre.leggauss(128)
    r = 0.5 * kern.r_c * (nodes + 1.0)
    w = 0.5 * kern.r_c * weights
    j = 0.5 * kern.r_c ** 2 - float(np.sum(w * r * phi0(kern.basis, r, kern.r_c)))
    u_cb = -4.0 * np.pi * q_total ** 2 / volume * j
    u_bb = 2.0 * np.pi * q_total ** 2 / volume * j
    p_corr = -2.0 * np.pi * q_total ** 2 * j / volume ** 2 * np.eye(3)
    return u_cb, u_bb, p_corr
