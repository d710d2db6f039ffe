"""Cell types of the north star (isotropic, semi-isotropic, anisotropic,
fully flexible triclinic) and the pressure quantity each one couples to.

The reference has a single ``Cell(h)`` and names the couplings only in its
finite-difference oracle (oracle.py:237-284) and the paper:
isotropic barostats use tr(P)/3, semi-isotropic ones the lateral
(Pxx+Pyy)/2 and normal Pzz, anisotropic ones diag(P), and a fully flexible
cell all six independent components.  The device always computes the
energy plus all six components; the cell type validates h and selects what
is reported.
"""

from __future__ import annotations

import enum

import numpy as np

from .errors import CellError


class CellType(str, enum.Enum):
    ISOTROPIC = "isotropic"
    SEMI_ISOTROPIC = "semi_isotropic"
    ANISOTROPIC = "anisotropic"
    TRICLINIC = "triclinic"

    def validate(self, h) -> None:
        h = np.asarray(h, dtype=float)
        off = h - np.diag(np.diag(h))
        ortho = bool(np.all(np.abs(off) <= 1e-12 * np.max(np.abs(h))))
        L = np.diag(h)
        if self is CellType.TRICLINIC:
            if np.linalg.det(h) <= 0:
                raise CellError("cell matrix must be right-handed with positive volume")
            return
        if not ortho:
            raise CellError(f"{self.value} cells must be orthorhombic")
        if self is CellType.ISOTROPIC and not np.allclose(L, L[0], rtol=1e-12, atol=0):
            raise CellError("isotropic cells must be cubic")
        if self is CellType.SEMI_ISOTROPIC and not np.isclose(L[0], L[1], rtol=1e-12, atol=0):
            raise CellError("semi-isotropic cells need L_x == L_y")

    def reduce(self, P):
        P = np.asarray(P, dtype=float)
        if self is CellType.ISOTROPIC:
            return float(np.trace(P) / 3.0)
        if self is CellType.SEMI_ISOTROPIC:
            return {"lateral": 0.5 * float(P[0, 0] + P[1, 1]), "normal": float(P[2, 2])}
        if self is CellType.ANISOTROPIC:
            return np.diag(P).copy()
        return {"xx": P[0, 0], "yy": P[1, 1], "zz": P[2, 2],
                "xy": P[0, 1], "xz": P[0, 2], "yz": P[1, 2]}


def infer_cell_type(h) -> CellType:
    h = np.asarray(h, dtype=float)
    off = h - np.diag(np.diag(h))
    if not np.all(np.abs(off) <= 1e-12 * np.max(np.abs(h))):
        return CellType.TRICLINIC
    L = np.diag(h)
    if np.allclose(L, L[0], rtol=1e-12, atol=0):
        return CellType.ISOTROPIC
    if np.isclose(L[0], L[1], rtol=1e-12, atol=0):
        return CellType.SEMI_ISOTROPIC
    return CellType.ANISOTROPIC
