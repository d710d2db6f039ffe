"""Host-side construction of the order-zero prolate psi_0^c and the
spreading-window table (one-time plan setup; nothing here runs per step).

Restates the reference's published algorithm (``prolate_ewald/pswf.py``):

* psi_0^c is the lowest even eigenfunction of the prolate differential
  operator d/dx (1-x^2) d/dx - c^2 x^2; in the normalised Legendre basis the
  even block is symmetric tridiagonal (pswf.py:41-84).
* lambda0 = 2 C0 / psi_0(0) with C0 = int_0^1 psi_0 by 64-node Gauss-Legendre
  (pswf.py:166-170).
* c solves psi_0^c(1) = Delta (log-bracketed root, pswf.py:225-235).
* The window W(t) = psi_0^c(2t/P) on [-P/2, P/2] is tabulated as one
  degree-18 polynomial per unit interval (refined if 1e-13 is not met), each
  interpolating W at Chebyshev nodes and stored as monomials in
  (t - left end) (pswf.py:87-107, 261-293).

The device kernels read the table produced here; keeping the same numpy
operations makes the coefficients identical to the reference's, so the
GPU window weights differ from the reference only by evaluation rounding.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numpy.polynomial import Chebyshev, Polynomial
from numpy.polynomial import legendre as L
from scipy.linalg import eigh_tridiagonal
from scipy.optimize import brentq

from .errors import DomainError, PswfError

C_RANGE = (0.5, 80.0)
TABLE_TOL = 1e-13
TABLE_DEGREE = 18


def _even_block(c: float, n: int):
    """Diagonal / off-diagonal of the even-order block of the prolate operator
    in normalised Legendre polynomials of degree 0, 2, ..., 2n-2."""
    k = 2.0 * np.arange(n)
    c2 = c * c
    diag = k * (k + 1.0) + c2 * (2.0 * k * (k + 1.0) - 1.0) / (
        (2.0 * k + 3.0) * (2.0 * k - 1.0))
    kk = k[:-1]
    off = c2 * (kk + 2.0) * (kk + 1.0) / (
        (2.0 * kk + 3.0) * np.sqrt((2.0 * kk + 1.0) * (2.0 * kk + 5.0)))
    return k, diag, off


def prolate_legendre_series(c: float) -> np.ndarray:
    """Legendre-series coefficients of psi_0^c (unit L2 norm, psi(0) > 0)."""
    n = max(int(np.ceil(c)) + 16, 40)
    for _attempt in range(8):
        k, diag, off = _even_block(c, n)
        try:
            _, vec = eigh_tridiagonal(diag, off, select="i", select_range=(0, 0))
        except Exception as exc:  # pragma: no cover - LAPACK failure
            raise PswfError(f"prolate eigensolve failed for c={c}: {exc}") from exc
        v = vec[:, 0]
        if np.max(np.abs(v[-4:])) / np.max(np.abs(v)) < 1e-16:
            break
        n *= 2
    else:
        raise PswfError(f"prolate expansion did not converge for c={c}")
    series = np.zeros(2 * n - 1)
    series[::2] = v * np.sqrt((2.0 * k + 1.0) / 2.0)
    keep = np.nonzero(np.abs(series) > 1e-17 * np.max(np.abs(series)))[0][-1]
    series = series[: keep + 1]
    return -series if L.legval(0.0, series) < 0.0 else series


@dataclass(frozen=True)
class PswfBasis:
    """psi_0^c for one bandwidth: Legendre series and derived constants."""

    c: float
    legendre_coeffs: np.ndarray
    lambda0: float
    psi0_at_zero: float
    C0: float
    table_tol: float = TABLE_TOL
    table_degree: int = TABLE_DEGREE

    def psi_series(self, x, derivative: int = 0):
        co = L.legder(self.legendre_coeffs, derivative) if derivative else self.legendre_coeffs
        return L.legval(np.asarray(x, dtype=float), co)

    @property
    def derivative_coeffs(self) -> np.ndarray:
        return L.legder(self.legendre_coeffs)


def build_pswf(c: float, table_tol: float = TABLE_TOL,
               table_degree: int = TABLE_DEGREE) -> PswfBasis:
    if not (C_RANGE[0] <= c <= C_RANGE[1]):
        raise PswfError(f"bandwidth c={c} outside [{C_RANGE[0]}, {C_RANGE[1]}]")
    if not (1e-15 <= table_tol <= 1e-6):
        raise PswfError(f"table_tol={table_tol} outside [1e-15, 1e-6]")
    series = prolate_legendre_series(c)
    at0 = float(L.legval(0.0, series))
    nodes, weights = np.polynomial.legendre.leggauss(64)
    c0 = float(0.5 * np.sum(weights * L.legval(0.5 * (nodes + 1.0), series)))
    return PswfBasis(c=float(c), legendre_coeffs=series, lambda0=2.0 * c0 / at0,
                     psi0_at_zero=at0, C0=c0, table_tol=float(table_tol),
                     table_degree=int(table_degree))


def solve_bandwidth(delta: float) -> float:
    """Bandwidth c with psi_0^c(1) = delta (strictly decreasing in delta)."""
    if not (1e-14 <= delta <= 1e-1):
        raise PswfError(f"delta={delta} outside [1e-14, 1e-1]")
    target = np.log(delta)

    def resid(c):
        end = float(L.legval(1.0, prolate_legendre_series(c)))
        return np.log(max(end, 1e-290)) - target

    return float(brentq(resid, C_RANGE[0], C_RANGE[1], xtol=1e-9, rtol=1e-10))


def _chebyshev_pieces(fun, degree: int, n_int: int, lo: float, hi: float):
    """Monomial coefficients (highest power first, per piece) of Chebyshev-node
    interpolants on n_int uniform pieces of [lo, hi], in powers of
    (t - piece left end)."""
    edges = np.linspace(lo, hi, n_int + 1)
    width = edges[1] - edges[0]
    cheb_nodes = np.cos(np.pi * (2.0 * np.arange(degree + 1) + 1.0) / (2.0 * (degree + 1)))
    to_unit = Polynomial([-1.0, 2.0 / width])
    out = np.empty((n_int, degree + 1))
    for i in range(n_int):
        samples = fun(edges[i] + 0.5 * width * (cheb_nodes + 1.0))
        poly = Chebyshev.fit(cheb_nodes, samples, degree, domain=[-1, 1]).convert(
            kind=Polynomial)(to_unit)
        row = np.zeros(degree + 1)
        row[: poly.coef.size] = poly.coef
        out[i] = row[::-1]
    return out, edges


@dataclass(frozen=True)
class WindowTable:
    """W(t) = psi_0^c(2t/P) on [-P/2, P/2] in grid units, piecewise
    polynomial.  ``coef[j, m]`` multiplies (t - breaks[j])**(degree - m)."""

    P: int
    degree: int
    table_tol: float
    coef: np.ndarray
    deriv_coef: np.ndarray
    breaks: np.ndarray
    basis_c: float
    _cache: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def n_pieces(self) -> int:
        return self.coef.shape[0]

    def __call__(self, t, derivative: int = 0):
        """Host evaluation (diagnostics / tests); zero outside the support."""
        tab = self.deriv_coef if derivative else self.coef
        t = np.asarray(t, dtype=float)
        j = np.searchsorted(self.breaks, t, side="right") - 1
        j = np.where(t == self.breaks[-1], self.n_pieces - 1, j)
        inside = (t >= self.breaks[0]) & (t <= self.breaks[-1])
        jj = np.clip(j, 0, self.n_pieces - 1)
        s = t - self.breaks[jj]
        acc = tab[jj, 0]
        for m in range(1, tab.shape[1]):
            acc = acc * s + tab[jj, m]
        out = np.where(inside, acc, 0.0)
        return out if out.ndim else float(out)


def tabulate_window(basis: PswfBasis, P: int, table_tol: float = TABLE_TOL,
                    degree: int = TABLE_DEGREE) -> WindowTable:
    if P < 2:
        raise PswfError(f"spreading order P={P} must be >= 2")
    half, scale = P / 2.0, 2.0 / P
    series = basis.legendre_coeffs
    dseries = L.legder(series)

    def value(x):
        return L.legval(np.clip(np.asarray(x) * scale, -1.0, 1.0), series)

    def slope(x):
        return L.legval(np.clip(np.asarray(x) * scale, -1.0, 1.0), dseries) * scale

    probe = np.linspace(-half, half, 4097)
    per_unit = 1
    for _ in range(8):
        n_int = P * per_unit
        coef, edges = _chebyshev_pieces(value, degree, n_int, -half, half)
        dcoef, _ = _chebyshev_pieces(slope, degree, n_int, -half, half)
        table = WindowTable(P=int(P), degree=int(degree), table_tol=float(table_tol),
                            coef=coef, deriv_coef=dcoef, breaks=edges, basis_c=basis.c)
        err = np.max(np.abs(_power_sum(coef, edges, probe) - value(probe))) / basis.psi0_at_zero
        if err <= table_tol:
            return table
        per_unit *= 2
    raise PswfError(f"window table did not reach tolerance {table_tol}")


def _power_sum(coef, edges, t):
    """Evaluate the piecewise table as ascending power sums (scipy PPoly's
    evaluation order), used for the acceptance check of the fit."""
    j = np.clip(np.searchsorted(edges, t, side="right") - 1, 0, coef.shape[0] - 1)
    s = t - edges[j]
    deg = coef.shape[1] - 1
    res = np.zeros_like(t)
    z = np.ones_like(t)
    for kp in range(deg + 1):
        res = res + coef[j, deg - kp] * z
        z = z * s
    return res


def eval_psi0(basis: PswfBasis, x, derivative: int = 0):
    """psi_0^c or its derivative on [-1, 1] from the Legendre series."""
    if derivative not in (0, 1):
        raise PswfError(f"derivative order {derivative} not supported")
    xa = np.asarray(x, dtype=float)
    if np.any(np.abs(xa) > 1.0 + 1e-12):
        raise DomainError("eval_psi0 argument outside [-1, 1]")
    out = basis.psi_series(np.clip(xa, -1.0, 1.0), derivative)
    return out if np.ndim(out) else float(out)
