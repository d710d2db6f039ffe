"""Generate the golden fixtures by running the REFERENCE implementation.

Run once in the build container (the reference tree exists only there):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

It imports ``prolate_ewald`` from ``/root/reference/pkg/src`` and calls the
reference API exactly as SURVEY.md §8(c) "Oracle call sequence" lists
(``plan_grid(..., fixed_M=...)``, ``ModeWorkspace``, ``forward_density``,
``long_range_energy``, ``long_range_pressure``, ``long_range_forces(mode=
"ik")``), plus ``direct_ksum`` on small triclinic cells.  Outputs go to
``tests/golden/*.npz`` together with the numpy/scipy versions used.
Nothing under ``tests/`` reads ``/root/reference`` at run time; only these
committed fixtures travel.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from prolate_ewald import (Cell, ParticleSystem, SplitKernel, build_pswf,  # noqa: E402
                           solve_bandwidth, tabulate_window)
from prolate_ewald.mesh import (ModeWorkspace, TransformProvider,  # noqa: E402
                                forward_density, local_pressure,
                                long_range_energy, long_range_forces,
                                long_range_pressure, plan_grid,
                                spread_charges)
from prolate_ewald.oracle import direct_ksum  # noqa: E402
from prolate_ewald.evaluate import CoulombSolver, EwaldParameters  # noqa: E402
from prolate_ewald.realspace import build_pair_table, short_range  # noqa: E402
from prolate_ewald.system import build_cell_list  # noqa: E402

from paper_2601_00161_b200 import workloads  # noqa: E402

VERSIONS = np.array([np.__version__, scipy.__version__])


def run_reference(h, raw, q, M, P, delta, r_c, with_grid=False, with_local=False,
                  with_analytic=False):
    basis = build_pswf(solve_bandwidth(delta))
    kern = SplitKernel(basis=basis, r_c=r_c)
    cell = Cell(np.asarray(h, dtype=float))
    sys_ = ParticleSystem(cell=cell, positions=raw, charges=q)
    assert np.array_equal(sys_.positions, workloads.wrap_positions(h, raw))
    spec = plan_grid(cell, kern, delta_spread=delta, P=P, spread_basis=basis,
                     fixed_M=tuple(M))
    modes = ModeWorkspace(spec, kern, cell)
    prov = TransformProvider()
    rho_hat = forward_density(sys_, spec, prov)
    E = long_range_energy(rho_hat, kern, spec, cell, modes)
    Pt = long_range_pressure(rho_hat, kern, spec, cell, modes)
    assert prov.forward_count == 1 and prov.inverse_count == 0
    F = long_range_forces(rho_hat, sys_, kern, spec, cell, "ik", prov, modes)
    out = dict(E=E, Pt=Pt, F=F, c=basis.c, lambda0=basis.lambda0, C0=basis.C0,
               psi0_at_zero=basis.psi0_at_zero, legendre=basis.legendre_coeffs,
               window_c=spec.window.value.c, window_x=spec.window.value.x,
               window_dc=spec.window.deriv.c, n_modes=int(modes.mask.sum()),
               versions=VERSIONS)
    if with_grid:
        out["grid"] = spread_charges(sys_, spec).values
        out["rho_hat_masked"] = rho_hat.values[modes.mask]
    if with_local:
        out["local"] = local_pressure(rho_hat, sys_, kern, spec, cell, prov, modes)
    if with_analytic:
        out["F_analytic"] = long_range_forces(rho_hat, sys_, kern, spec, cell,
                                              "analytic", prov, modes)
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def configs():
    for idx in (0, 1, 2):
        w, raw, q = workloads.generate(idx, wrap=False)
        pos = workloads.wrap_positions(w.h, raw)
        r = run_reference(w.h, raw, q, w.M, w.P, w.delta, w.r_c,
                          with_grid=(idx == 0))
        F = r.pop("F")
        sel = np.arange(w.n)          # every atom's force (full parity, not a sample)
        save(f"cfg{idx}", pos_head=pos[:4], pos_sum=pos.sum(axis=0),
             F_idx=sel, F_sel=F[sel], F_rms=np.sqrt(np.mean(np.sum(F * F, axis=1))),
             F_sum=F.sum(axis=0), **r)


SMALL = [
    # (name, n, lengths, seed, delta, P, r_c, oversampling)
    ("small_cube_p5", 32, (6.0, 6.0, 6.0), 0, 1e-4, 5, 1.0, 2.0),
    ("small_cube_p6", 32, (6.0, 6.0, 6.0), 1, 1e-5, 6, 1.2, 2.0),
    ("small_brick_p6", 48, (5.0, 6.0, 7.0), 4, 1e-5, 6, 1.2, 2.0),
    ("small_brick_p8", 64, (6.2, 6.0, 6.4), 523, 1e-7, 8, 2.94, 2.0),
    ("small_brick_p7", 40, (6.0, 7.0, 8.0), 9, 1e-6, 7, 1.2, 2.0),
    ("small_cube_p4", 16, (6.0, 6.0, 6.0), 10, 1e-3, 4, 1.1, 2.0),
    ("small_single", 1, (6.0, 6.0, 6.0), 3, 1e-4, 5, 1.0, 2.0),
]


def small_cases():
    for (name, n, lengths, seed, delta, P, r_c, ovs) in SMALL:
        raw, q = workloads.random_neutral_system(n, lengths, seed, wrap=False)
        pos = workloads.wrap_positions(np.diag(lengths), raw)
        if n == 1:
            q = np.array([1.0])
        basis = build_pswf(solve_bandwidth(delta))
        kern = SplitKernel(basis=basis, r_c=r_c)
        cell = Cell.orthorhombic(lengths)
        spec = plan_grid(cell, kern, delta_spread=delta, P=P, oversampling=ovs,
                         spread_basis=basis)
        r = run_reference(np.diag(lengths), raw, q, spec.M, P, delta, r_c,
                          with_grid=True, with_local=True, with_analytic=True)
        e_d, f_d, p_d = direct_ksum(ParticleSystem(cell=cell, positions=raw, charges=q), kern)
        save(name, pos=pos, q=q, h=np.diag(lengths), M=np.array(spec.M), P=P,
             delta=delta, r_c=r_c, E_direct=e_d, F_direct=f_d, Pt_direct=p_d, **r)


TRICLINIC = [
    # (name, h columns, n, seed, delta, P, r_c, M)
    ("tri_skew_p8", np.array([[20.0, 2.0, 1.0], [0.0, 19.0, 1.5], [0.0, 0.0, 25.0]]),
     400, 11, 1e-7, 8, 4.0, (64, 64, 80)),
    ("tri_skew_p6", np.array([[20.0, 2.0, 1.0], [0.0, 19.0, 1.5], [0.0, 0.0, 25.0]]),
     400, 12, 1e-5, 6, 4.0, (48, 48, 60)),
    ("tri_flex_p7", np.array([[6.0, 1.2, -0.8], [0.0, 6.5, 0.9], [0.0, 0.0, 7.0]]),
     32, 13, 1e-6, 7, 1.5, (44, 48, 52)),
]


def triclinic_cases():
    """Exact mode sums (reference direct_ksum, any cell) that pin the
    triclinic mesh extension at the Delta level."""
    for (name, h, n, seed, delta, P, r_c, M) in TRICLINIC:
        rng = np.random.default_rng(seed)
        raw = rng.uniform(0.0, 1.0, (n, 3)) @ h.T
        pos = workloads.wrap_positions(h, raw)
        q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
        basis = build_pswf(solve_bandwidth(delta))
        kern = SplitKernel(basis=basis, r_c=r_c)
        cell = Cell(h)
        sys_ = ParticleSystem(cell=cell, positions=raw, charges=q)
        assert np.array_equal(sys_.positions, pos)
        e_d, f_d, p_d = direct_ksum(sys_, kern)
        save(name, pos=pos, q=q, h=h, M=np.array(M), P=P, delta=delta, r_c=r_c,
             E_direct=e_d, F_direct=f_d, Pt_direct=p_d, versions=VERSIONS)


def window_tables():
    """Reference window tables for P in 2..12 at a few tolerances."""
    rows = {}
    for delta in (1e-3, 1e-5, 1e-7, 1e-9):
        basis = build_pswf(solve_bandwidth(delta))
        for P in (2, 3, 4, 5, 6, 7, 8, 10, 12):
            w = tabulate_window(basis, P)
            rows[f"d{delta:g}_P{P}_c"] = w.value.c
            rows[f"d{delta:g}_P{P}_x"] = w.value.x
            rows[f"d{delta:g}_P{P}_dc"] = w.deriv.c
        rows[f"d{delta:g}_legendre"] = basis.legendre_coeffs
        rows[f"d{delta:g}_consts"] = np.array([basis.c, basis.lambda0, basis.C0,
                                               basis.psi0_at_zero])
    save("window_tables", versions=VERSIONS, **rows)


NEAR_SMALL = [
    # (name, h (columns = cell vectors), n, seed, delta, r_c, skin)
    ("near_brick", np.diag([5.0, 6.0, 7.0]), 64, 21, 1e-5, 1.4, 0.0),
    ("near_cube_skin", np.diag([7.0, 7.0, 7.0]), 128, 22, 1e-6, 1.5, 0.3),
    ("near_tri", np.array([[6.0, 1.2, -0.8], [0.0, 6.5, 0.9], [0.0, 0.0, 7.0]]),
     96, 23, 1e-6, 1.5, 0.0),
    ("near_tight", np.diag([5.0, 5.0, 5.0]), 64, 24, 1e-8, 1.0, 0.0),
]


def near_cases():
    """Near field (realspace.py): pair tables, short_range with the table and
    with exact values, over the reference's own cell lists; CoulombSolver
    totals for config 0; the near field of configs 0-2."""
    tabs = {}
    for (tag, delta, r_c) in (("d1e-5_rc10", 1e-5, 10.0), ("d1e-7_rc10", 1e-7, 10.0),
                              ("d1e-8_rc1", 1e-8, 1.0), ("d1e-7_rc12", 1e-7, 12.0)):
        kern = SplitKernel(basis=build_pswf(solve_bandwidth(delta)), r_c=r_c)
        t = build_pair_table(kern)
        tabs[f"{tag}_rin"] = np.array(t.r_in)
        tabs[f"{tag}_smooth"] = t.smooth_coeffs
        tabs[f"{tag}_fn"] = t.fn_coeffs
        tabs[f"{tag}_sc"] = t.smooth_spline.c
        tabs[f"{tag}_fc"] = t.fn_spline.c
        tabs[f"{tag}_x"] = t.smooth_spline.x
        r = np.exp(np.linspace(np.log(1e-3 * r_c), np.log(1.2 * r_c), 2001))
        tabs[f"{tag}_probe_r"] = r
        tabs[f"{tag}_probe_nv"] = t.near_field(r)
        tabs[f"{tag}_probe_fv"] = t.fn_weight(r)
    save("near_tables", versions=VERSIONS, **tabs)
    for (name, h, n, seed, delta, r_c, skin) in NEAR_SMALL:
        rng = np.random.default_rng(seed)
        raw = rng.uniform(0.0, 1.0, (n, 3)) @ h.T
        q = rng.normal(size=n)
        q -= q.mean()
        kern = SplitKernel(basis=build_pswf(solve_bandwidth(delta)), r_c=r_c)
        sys_ = ParticleSystem(cell=Cell(h), positions=raw, charges=q)
        nb = build_cell_list(sys_, r_c, skin=skin)
        t = build_pair_table(kern)
        a = short_range(sys_, kern, nb, table=t)
        b = short_range(sys_, kern, nb)
        save(name, h=h, pos=sys_.positions, q=q, delta=delta, r_c=r_c, skin=skin,
             pi=nb.i, pj=nb.j, E_tab=a.energy, F_tab=a.forces, P_tab=a.pressure,
             count=a.pair_count, E_exact=b.energy, F_exact=b.forces, P_exact=b.pressure,
             versions=VERSIONS)
    for idx in (0, 1, 2):
        w, raw, q = workloads.generate(idx, wrap=False)
        kern = SplitKernel(basis=build_pswf(solve_bandwidth(w.delta)), r_c=w.r_c)
        cell = Cell(np.asarray(w.h, dtype=float))
        sys_ = ParticleSystem(cell=cell, positions=raw, charges=q)
        nb = build_cell_list(sys_, w.r_c)
        a = short_range(sys_, kern, nb, table=build_pair_table(kern))
        F = a.forces
        stride = 1 if idx == 0 else 97
        sel = np.arange(0, w.n, stride)
        extra = {}
        if idx == 0:
            params = EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P)
            solver = CoulombSolver(cell, params)
            solver.rebind_cell(cell, fixed_M=tuple(w.M))
            tot = solver.evaluate(sys_)
            extra = dict(tot_u=np.array([tot.u_near, tot.u_far, tot.u_self, tot.u_background]),
                         tot_F=tot.forces, tot_P=tot.pressure, tot_count=tot.pair_count)
        save(f"near_cfg{idx}", E=a.energy, P=a.pressure, count=a.pair_count, F_idx=sel,
             F_sel=F[sel], F_sum=F.sum(axis=0),
             F_rms=np.sqrt(np.mean(np.sum(F * F, axis=1))), versions=VERSIONS, **extra)
        del nb, a, F


def host_helpers():
    """Host-side kernel / solver helpers of the reference (kernel.py,
    pswf.eval_phi0, evaluate.kinetic_pressure) at fixed arguments."""
    from prolate_ewald.evaluate import kinetic_pressure
    from prolate_ewald.kernel import (background_correction, background_integral, far_field,
                                      far_field_hat, fn_weight, near_field,
                                      pressure_kernel_hat, self_energy)
    from prolate_ewald.pswf import eval_phi0
    out = {}
    for tag, delta, r_c in (("a", 1e-5, 10.0), ("b", 1e-7, 1.3)):
        kern = SplitKernel(basis=build_pswf(solve_bandwidth(delta)), r_c=r_c)
        r = np.linspace(0.01, 1.2, 97) * r_c
        out[f"{tag}_r"] = r
        out[f"{tag}_phi0"] = eval_phi0(kern.basis, r, r_c)
        out[f"{tag}_near"] = near_field(kern, r)
        out[f"{tag}_far"] = far_field(kern, np.concatenate([[0.0], r]))
        out[f"{tag}_fn"] = fn_weight(kern, r)
        ks = np.array([[0.1, 0.2, 0.3], [0.5, -0.4, 0.2], [1.2, 0.0, 0.0]]) * kern.kmax
        out[f"{tag}_k"] = ks
        out[f"{tag}_pk"] = np.stack([pressure_kernel_hat(kern, k) for k in ks])
        out[f"{tag}_fhat"] = far_field_hat(kern, np.linalg.norm(ks, axis=1))
        out[f"{tag}_J"] = np.array(background_integral(kern))
        q = np.array([0.5, -0.2, 0.9, 0.1])
        out[f"{tag}_self"] = np.array(self_energy(kern, q))
        u_cb, u_bb, pc = background_correction(kern, float(q.sum()), 1234.5)
        out[f"{tag}_bg"] = np.array([u_cb, u_bb])
        out[f"{tag}_pcorr"] = pc
    rng = np.random.default_rng(5)
    sys_ = ParticleSystem(cell=Cell(np.array([[5.0, 0.4, 0.1], [0.0, 6.0, -0.3], [0.0, 0.0, 7.0]])),
                          positions=rng.uniform(0, 5, (9, 3)), charges=rng.normal(size=9),
                          masses=rng.uniform(0.5, 2.0, 9), momenta=rng.normal(size=(9, 3)))
    out["kin_h"] = sys_.cell.h
    out["kin_p"] = sys_.momenta
    out["kin_m"] = sys_.masses
    out["kin_P"] = kinetic_pressure(sys_)
    save("host_helpers", versions=VERSIONS, **out)


def particle_files():
    """Reference-written particle files (cli.write_particles) and what the
    reference reads back from them (cli.read_particles)."""
    from prolate_ewald.cli import read_particles, write_particles
    rng = np.random.default_rng(31)
    cases = {
        "particles_ortho": ParticleSystem(cell=Cell.orthorhombic([5.0, 6.0, 7.0]),
                                          positions=rng.uniform(-2, 9, (12, 3)),
                                          charges=rng.standard_normal(12),
                                          masses=rng.uniform(0.5, 2.0, 12)),
        "particles_tri": ParticleSystem(
            cell=Cell(np.array([[5.0, 0.4, 0.1], [0.0, 6.0, -0.3], [0.0, 0.0, 7.0]])),
            positions=rng.uniform(-2, 9, (7, 3)), charges=rng.standard_normal(7),
            masses=rng.uniform(0.5, 2.0, 7)),
    }
    for name, s_ in cases.items():
        path = os.path.join(HERE, name + ".txt")
        write_particles(path, s_)
        back = read_particles(path)
        write_particles(os.path.join(HERE, name + "_2.txt"), back)
        save(name, h=back.cell.h, pos=back.positions, q=back.charges, m=back.masses,
             versions=VERSIONS)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["window", "small", "triclinic", "configs", "near", "particles",
                                 "helpers"]
    if "particles" in parts:
        particle_files()
    if "helpers" in parts:
        host_helpers()
    if "window" in parts:
        window_tables()
    if "small" in parts:
        small_cases()
    if "triclinic" in parts:
        triclinic_cases()
    if "configs" in parts:
        configs()
    if "near" in parts:
        near_cases()
