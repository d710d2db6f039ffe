"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: every input is generated here from
``numpy.random.default_rng(seed)`` (PCG64, the reference's RNG convention,
``pkg/tests/conftest.py:24-36``) following the recipes of SURVEY.md §8(d.1).
Positions are wrapped into the cell with the same fractional round trip the
reference ``ParticleSystem`` applies (``system.py:64-72,105``), so the arrays
are bit-identical to what the reference sees after construction.  (The wrap
is not idempotent at the ulp level, so it is applied exactly once, to the raw
draw.)

Configs (index = seed):

====  ==========================  ==========  ==============  ===  =====  ====
cfg   cell                        N           M               P    Δ      r_c
====  ==========================  ==========  ==============  ===  =====  ====
0     cubic 31.04                 3,000       32³             6    1e-5   10
1     67×67×67.5 (semi-iso)       90,000      64³             8    1e-7   10
2     80×80×120 (aniso, ionic)    40,000      64×64×96        8    1e-7   12
3     triclinic membrane          1,000,000   192×192×256     8    1e-7   10
4     cubic 300                   8,100,000   384³            8    1e-7   10
====  ==========================  ==========  ==============  ===  =====  ====
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

O_CHARGE = -0.8476
H_CHARGE = 0.4238
OH_BOND = 1.0
HOH_ANGLE_DEG = 109.47


@dataclass(frozen=True)
class Workload:
    name: str
    index: int
    h: np.ndarray          # 3x3, columns are cell vectors
    M: tuple               # (Mx, My, Mz)
    P: int
    delta: float
    r_c: float
    n: int
    cell_type: str         # isotropic | semi_isotropic | anisotropic | triclinic

    @property
    def orthorhombic(self) -> bool:
        off = self.h - np.diag(np.diag(self.h))
        return bool(np.all(off == 0.0))


def _cube(L):
    return np.diag([float(L)] * 3)


CONFIGS = {
    0: dict(name="cfg0_water_cubic", h=_cube(31.04), M=(32, 32, 32), P=6,
            delta=1e-5, r_c=10.0, n=3000, cell_type="isotropic"),
    1: dict(name="cfg1_water_semiiso", h=np.diag([67.0, 67.0, 67.5]),
            M=(64, 64, 64), P=8, delta=1e-7, r_c=10.0, n=90000,
            cell_type="semi_isotropic"),
    2: dict(name="cfg2_ionic_aniso", h=np.diag([80.0, 80.0, 120.0]),
            M=(64, 64, 96), P=8, delta=1e-7, r_c=12.0, n=40000,
            cell_type="anisotropic"),
    3: dict(name="cfg3_membrane_triclinic",
            h=np.array([[200.0, 20.0, 10.0],
                        [0.0, 190.0, 15.0],
                        [0.0, 0.0, 250.0]]),
            M=(192, 192, 256), P=8, delta=1e-7, r_c=10.0, n=1_000_000,
            cell_type="triclinic"),
    4: dict(name="cfg4_water_cubic_large", h=_cube(300.0), M=(384, 384, 384),
            P=8, delta=1e-7, r_c=10.0, n=8_100_000, cell_type="isotropic"),
}


def workload(index: int) -> Workload:
    c = CONFIGS[index]
    return Workload(index=index, **c)


def wrap_positions(h: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """Fractional wrap with the reference's arithmetic (``system.py:64-72``)."""
    h = np.asarray(h, dtype=float)
    s = np.asarray(pos, dtype=float) @ np.linalg.inv(h).T
    return (s - np.floor(s)) @ h.T


def _rotations(rng, n):
    qv = rng.normal(size=(n, 4))
    qv /= np.linalg.norm(qv, axis=1, keepdims=True)
    w, x, y, z = qv.T
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _water_from_oxygens(rng, O):
    """Attach two H per oxygen with a uniformly random SO(3) orientation."""
    n = O.shape[0]
    R = _rotations(rng, n)
    half = np.deg2rad(HOH_ANGLE_DEG) / 2.0
    h1 = np.array([np.sin(half), 0.0, np.cos(half)]) * OH_BOND
    h2 = np.array([-np.sin(half), 0.0, np.cos(half)]) * OH_BOND
    H1 = O + R @ h1
    H2 = O + R @ h2
    pos = np.stack([O, H1, H2], axis=1).reshape(-1, 3)
    q = np.tile([O_CHARGE, H_CHARGE, H_CHARGE], n)
    return pos, q


def water_box(h, n_mol, seed):
    """Config 0/1/4 recipe: O uniform in the cell, then rigid 3-site water."""
    rng = np.random.default_rng(seed)
    h = np.asarray(h, dtype=float)
    O = rng.uniform(0.0, 1.0, (n_mol, 3)) @ h.T
    return _water_from_oxygens(rng, O)


def ionic_box(lengths, n, seed, min_sep=1.5, charge=0.8):
    """Config 2 recipe: random sequential addition with a minimum
    minimum-image separation, cell-list accelerated; +q even, -q odd."""
    rng = np.random.default_rng(seed)
    L = np.asarray(lengths, dtype=float)
    nb = np.maximum((L // min_sep).astype(int), 1)
    width = L / nb
    cells: dict = {}
    out = np.empty((n, 3))
    m2 = min_sep * min_sep
    k = 0
    while k < n:
        cand = rng.uniform(size=3) * L
        ci = np.minimum((cand // width).astype(int), nb - 1)
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    key = ((ci[0] + dx) % nb[0], (ci[1] + dy) % nb[1],
                           (ci[2] + dz) % nb[2])
                    for j in cells.get(key, ()):
                        d = cand - out[j]
                        d -= L * np.round(d / L)
                        if d @ d < m2:
                            ok = False
                            break
                    if not ok:
                        break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            out[k] = cand
            cells.setdefault((ci[0], ci[1], ci[2]), []).append(k)
            k += 1
    q = np.where(np.arange(n) % 2 == 0, charge, -charge)
    return out, q


def membrane_box(h, n_total, seed, slab=(0.42, 0.58), dipole_density=0.05,
                 dipole_sep=1.5, dipole_q=0.5):
    """Config 3 recipe: ±0.5 e dipoles in the slab
    |z-125|<20 Å at 0.05 charges/Å³, water-like triplets elsewhere, so that
    N = n_total exactly.  Draw order: dipole centres, dipole directions,
    then water oxygens (fractional) and orientations."""
    rng = np.random.default_rng(seed)
    h = np.asarray(h, dtype=float)
    vol = float(np.linalg.det(h))
    slab_vol = vol * (slab[1] - slab[0])
    n_dip_charges = int(round(dipole_density * slab_vol))
    n_dip_charges -= n_dip_charges % 2
    n_water = (n_total - n_dip_charges) // 3
    n_dip_charges = n_total - 3 * n_water
    n_dip = n_dip_charges // 2
    s = rng.uniform(0.0, 1.0, (n_dip, 3))
    s[:, 2] = slab[0] + (slab[1] - slab[0]) * s[:, 2]
    centre = s @ h.T
    u = rng.normal(size=(n_dip, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    half = 0.5 * dipole_sep
    dpos = np.stack([centre + half * u, centre - half * u], axis=1).reshape(-1, 3)
    dq = np.tile([dipole_q, -dipole_q], n_dip)
    so = rng.uniform(0.0, 1.0, (n_water, 3))
    outside = 1.0 - (slab[1] - slab[0])
    so[:, 2] = np.mod(slab[1] + outside * so[:, 2], 1.0)
    wpos, wq = _water_from_oxygens(rng, so @ h.T)
    pos = np.concatenate([dpos, wpos])
    q = np.concatenate([dq, wq])
    return pos, q


def generate(index: int, wrap: bool = True):
    """(workload, positions (N,3) f64, charges (N,) f64) for config ``index``.

    With ``wrap`` (default) positions are wrapped once into the cell exactly
    as the reference ``ParticleSystem`` constructor does; ``wrap=False``
    returns the raw draw (what a caller would hand to that constructor)."""
    w = workload(index)
    if index in (0, 1, 4):
        pos, q = water_box(w.h, w.n // 3, seed=index)
    elif index == 2:
        pos, q = ionic_box(np.diag(w.h), w.n, seed=index)
    elif index == 3:
        pos, q = membrane_box(w.h, w.n, seed=index)
    else:  # pragma: no cover
        raise KeyError(index)
    assert pos.shape == (w.n, 3)
    return w, (wrap_positions(w.h, pos) if wrap else pos), q


def random_neutral_system(n, lengths, seed, charge_style="alternating", wrap=True):
    """The reference test-suite ensemble generator (``tests/conftest.py:24-36``)."""
    rng = np.random.default_rng(seed)
    lengths = np.asarray(lengths, dtype=float)
    pos = rng.uniform(0.0, 1.0, (n, 3)) * lengths
    if charge_style == "alternating":
        q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
        if n % 2:
            q = q - q.sum() / n
    else:
        q = rng.normal(size=n)
        q -= q.mean()
    return (wrap_positions(np.diag(lengths), pos) if wrap else pos), q
