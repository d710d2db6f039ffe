"""CPU-side tests: host setup parity, the C ABI surface, cell types, inputs."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, SMALL_CASES, golden
from oracle import esp_oracle as O
from paper_2601_00161_b200 import (CellType, PlanningError, build_pswf, cell_tables,
                                   infer_cell_type, solve_bandwidth, tabulate_window,
                                   workloads)
from paper_2601_00161_b200 import _lib
from paper_2601_00161_b200.errors import CellError


@pytest.mark.parametrize("delta", [1e-3, 1e-5, 1e-7, 1e-9])
def test_pswf_and_window_tables_bit_identical_to_reference(delta):
    g = golden("window_tables")
    b = build_pswf(solve_bandwidth(delta))
    consts = g[f"d{delta:g}_consts"]
    assert b.c == consts[0] and b.lambda0 == consts[1] and b.C0 == consts[2]
    assert b.psi0_at_zero == consts[3]
    np.testing.assert_array_equal(b.legendre_coeffs, g[f"d{delta:g}_legendre"])
    for P in (2, 3, 4, 5, 6, 7, 8, 10, 12):
        w = tabulate_window(b, P)
        np.testing.assert_array_equal(w.coef, g[f"d{delta:g}_P{P}_c"].T)
        np.testing.assert_array_equal(w.deriv_coef, g[f"d{delta:g}_P{P}_dc"].T)
        np.testing.assert_array_equal(w.breaks, g[f"d{delta:g}_P{P}_x"])


def test_window_host_eval_matches_oracle():
    b = build_pswf(solve_bandwidth(1e-7))
    w = tabulate_window(b, 8)
    ow = O.build_window(O.build_basis(b.c), 8)
    t = np.linspace(-4.2, 4.2, 2001)
    assert np.max(np.abs(w(t) - ow(t))) <= 1e-14


@pytest.mark.parametrize("name", SMALL_CASES[:4])
def test_cell_tables_reproduce_reference_mode_workspace(name):
    """The per-axis arrays uploaded to the device rebuild exactly the
    reference's mask and What^-2 (mesh.py:242-267)."""
    g = golden(name)
    plan = O.make_plan(g["h"], tuple(g["M"]), int(g["P"]), float(g["delta"]), float(g["r_c"]))
    m = O.Modes(plan)
    b = build_pswf(float(g["c"]))
    t = cell_tables(g["h"], tuple(g["M"]), int(g["P"]), b, plan.kmax)
    M = tuple(g["M"])
    kv = [t.axis_k[a][0][:, None, None] + t.axis_k[a][1][None, :, None]
          + t.axis_k[a][2][None, None, :] for a in range(3)]
    kx, ky, kz = [np.broadcast_to(k, M) for k in kv]
    k2 = kx ** 2 + ky ** 2 + kz ** 2
    mask = (np.sqrt(k2) <= plan.kmax) & (k2 > 0)
    np.testing.assert_array_equal(mask, m.mask)
    what = (t.axis_what[0][:, None, None] * t.axis_what[1][None, :, None]) \
        * t.axis_what[2][None, None, :]
    np.testing.assert_array_equal(1.0 / (np.broadcast_to(what, M)[mask] ** 2), m.w_inv2)
    # the in-band box covers every retained mode
    idx = np.nonzero(mask)
    for d in range(3):
        f = np.fft.fftfreq(M[d], 1.0 / M[d])[idx[d]]
        assert np.max(np.abs(f)) <= t.band[d]


def test_header_symbols_exported():
    """libesp_b200.so loads without a GPU and exports every symbol that
    include/esp_b200.h declares."""
    hdr = open(os.path.join(REPO, "include", "esp_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*|void\*)\s+(esp_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED)
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert lib.esp_version() == 100


def test_cell_types():
    assert infer_cell_type(np.diag([5.0, 5.0, 5.0])) is CellType.ISOTROPIC
    assert infer_cell_type(np.diag([67.0, 67.0, 67.5])) is CellType.SEMI_ISOTROPIC
    assert infer_cell_type(np.diag([80.0, 90.0, 120.0])) is CellType.ANISOTROPIC
    CellType.ANISOTROPIC.validate(np.diag([80.0, 80.0, 120.0]))  # cfg2: coupling is a choice
    assert infer_cell_type(workloads.workload(3).h) is CellType.TRICLINIC
    with pytest.raises(CellError):
        CellType.ISOTROPIC.validate(np.diag([5.0, 5.0, 6.0]))
    with pytest.raises(CellError):
        CellType.SEMI_ISOTROPIC.validate(np.diag([5.0, 6.0, 6.0]))
    with pytest.raises(CellError):
        CellType.ANISOTROPIC.validate(workloads.workload(3).h)
    P = np.array([[1.0, 0.1, 0.2], [0.1, 2.0, 0.3], [0.2, 0.3, 3.0]])
    assert CellType.ISOTROPIC.reduce(P) == pytest.approx(2.0)
    assert CellType.SEMI_ISOTROPIC.reduce(P) == {"lateral": 1.5, "normal": 3.0}
    np.testing.assert_array_equal(CellType.ANISOTROPIC.reduce(P), [1.0, 2.0, 3.0])
    assert CellType.TRICLINIC.reduce(P)["yz"] == 0.3


def test_plan_grid_rejects_like_reference():
    from paper_2601_00161_b200 import Cell, SplitKernel, plan_grid
    b = build_pswf(solve_bandwidth(1e-4))
    kern = SplitKernel(basis=b, r_c=1.0)
    cell = Cell.orthorhombic([6.0, 6.0, 6.0])
    with pytest.raises(PlanningError):
        plan_grid(cell, kern, delta_spread=1e-4, P=5, oversampling=0.5)
    with pytest.raises(PlanningError):
        plan_grid(cell, kern, delta_spread=1e-4, P=1)
    h = np.array([[6.0, 0.5, 0.0], [0.0, 6.0, 0.0], [0.0, 0.0, 6.0]])
    with pytest.raises(PlanningError):
        plan_grid(Cell(h=h), kern, delta_spread=1e-4, P=5)
    spec = plan_grid(Cell(h=h), kern, delta_spread=1e-4, P=5, allow_triclinic=True)
    assert all(m % 2 == 0 for m in spec.M)
    with pytest.raises(PlanningError, match="support|band|Nyquist"):
        plan_grid(Cell.orthorhombic([0.9] * 3), SplitKernel(basis=b, r_c=0.4),
                  delta_spread=1e-4, P=12)


def test_workloads_shapes_and_neutrality():
    for idx in (0, 1, 2):
        w, pos, q = workloads.generate(idx)
        assert pos.shape == (w.n, 3) and q.shape == (w.n,)
        assert abs(q.sum()) < 1e-9
        L = np.diag(w.h)
        assert np.all(pos >= 0) and np.all(pos <= L)
    # config 2 honours the minimum separation (spot-check a sample)
    w, pos, q = workloads.generate(2)
    sub = pos[:2000]
    d = sub[:, None, :] - sub[None, :, :]
    L = np.diag(w.h)
    d -= L * np.round(d / L)
    r = np.sqrt((d ** 2).sum(-1)) + np.eye(len(sub)) * 10
    assert r.min() >= 1.5


def test_membrane_recipe_small():
    h = workloads.workload(3).h
    pos, q = workloads.membrane_box(h, 30_000, seed=3, dipole_density=0.05 * 0.03)
    assert pos.shape == (30_000, 3) and abs(q.sum()) < 1e-9
    s = workloads.wrap_positions(h, pos) @ np.linalg.inv(h).T
    in_slab = (s[:, 2] > 0.41) & (s[:, 2] < 0.59)
    assert np.all(np.isin(q[in_slab & (np.abs(q) == 0.5)], [0.5, -0.5]))


@pytest.mark.parametrize("tag,delta,r_c", [("a", 1e-5, 10.0), ("b", 1e-7, 1.3)])
def test_host_kernel_helpers_match_reference(tag, delta, r_c):
    """kernel.py / pswf.eval_phi0 host helpers against the reference's values
    (tests/golden/host_helpers.npz)."""
    from conftest import golden
    from paper_2601_00161_b200 import (SplitKernel, background_correction, background_integral,
                                       build_pswf, eval_phi0, far_field, far_field_hat,
                                       fn_weight, near_field, pressure_kernel_hat, self_energy,
                                       solve_bandwidth)
    g = golden("host_helpers")
    kern = SplitKernel(basis=build_pswf(solve_bandwidth(delta)), r_c=r_c)
    r = g[f"{tag}_r"]
    np.testing.assert_allclose(eval_phi0(kern.basis, r, r_c), g[f"{tag}_phi0"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(near_field(kern, r), g[f"{tag}_near"], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(far_field(kern, np.concatenate([[0.0], r])), g[f"{tag}_far"],
                               rtol=1e-14)
    np.testing.assert_allclose(fn_weight(kern, r), g[f"{tag}_fn"], rtol=1e-13, atol=1e-300)
    pk = np.stack([pressure_kernel_hat(kern, k) for k in g[f"{tag}_k"]])
    np.testing.assert_allclose(pk, g[f"{tag}_pk"], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(far_field_hat(kern, np.linalg.norm(g[f"{tag}_k"], axis=1)),
                               g[f"{tag}_fhat"], rtol=1e-14)
    assert background_integral(kern) == pytest.approx(float(g[f"{tag}_J"]), rel=1e-14)
    q = np.array([0.5, -0.2, 0.9, 0.1])
    assert self_energy(kern, q) == pytest.approx(float(g[f"{tag}_self"]), rel=1e-14)
    u_cb, u_bb, pc = background_correction(kern, float(q.sum()), 1234.5)
    np.testing.assert_allclose([u_cb, u_bb], g[f"{tag}_bg"], rtol=1e-14)
    np.testing.assert_allclose(pc, g[f"{tag}_pcorr"], rtol=1e-14)


def test_kinetic_pressure_matches_reference():
    from conftest import golden
    from paper_2601_00161_b200 import Cell, ParticleSystem, kinetic_pressure
    g = golden("host_helpers")
    s = ParticleSystem(cell=Cell(g["kin_h"]), positions=np.zeros((len(g["kin_m"]), 3)),
                       charges=np.zeros(len(g["kin_m"])), masses=g["kin_m"], momenta=g["kin_p"])
    np.testing.assert_allclose(kinetic_pressure(s), g["kin_P"], rtol=1e-14)
