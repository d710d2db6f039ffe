"""Near field: realspace.short_range / build_cell_list on
the B200 (csrc/esp_near.cu) against the reference goldens
(tests/golden/near_*.npz, made by running the reference) and the CPU oracle.

CPU tests pin the oracle restatement and the host pair-table construction
to the reference.  GPU tests (``-m gpu``) run the CUDA pair sum through the
C ABI.  Tolerances: fp64 energy and pressure (Frobenius) within 1e-10
relative, forces within 1e-10 rms-relative, pair counts exact.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import esp_oracle as O
from paper_2601_00161_b200 import workloads

TOL = 1e-10
TABLES = [("d1e-5_rc10", 1e-5, 10.0), ("d1e-7_rc10", 1e-7, 10.0),
          ("d1e-8_rc1", 1e-8, 1.0), ("d1e-7_rc12", 1e-7, 12.0)]
SMALL = ["near_brick", "near_cube_skin", "near_tri", "near_tight"]


def _basis(delta):
    return O.build_basis(O.solve_bandwidth(delta))


# ---------------------------------------------------------------- CPU: pins


@pytest.mark.parametrize("tag,delta,r_c", TABLES)
def test_oracle_pair_table_matches_reference(tag, delta, r_c):
    g = golden("near_tables")
    t = O.pair_table(_basis(delta), r_c)
    assert t.r_in == float(g[f"{tag}_rin"])
    np.testing.assert_array_equal(t.smooth, g[f"{tag}_smooth"])
    np.testing.assert_array_equal(t.fn, g[f"{tag}_fn"])
    np.testing.assert_array_equal(t.smooth_spline.c, g[f"{tag}_sc"])
    np.testing.assert_array_equal(t.fn_spline.c, g[f"{tag}_fc"])
    nv, fv = O.table_values(t, g[f"{tag}_probe_r"])
    np.testing.assert_array_equal(nv, g[f"{tag}_probe_nv"])
    np.testing.assert_array_equal(fv, g[f"{tag}_probe_fv"])


@pytest.mark.parametrize("tag,delta,r_c", TABLES)
def test_package_pair_table_bit_identical(tag, delta, r_c):
    """The host setup of the product (realspace.build_pair_table) builds the
    reference's table bit for bit."""
    from paper_2601_00161_b200 import SplitKernel, build_pswf, solve_bandwidth
    from paper_2601_00161_b200.realspace import build_pair_table
    g = golden("near_tables")
    t = build_pair_table(SplitKernel(basis=build_pswf(solve_bandwidth(delta)), r_c=r_c))
    assert t.r_in == float(g[f"{tag}_rin"])
    np.testing.assert_array_equal(t.smooth_coeffs, g[f"{tag}_smooth"])
    np.testing.assert_array_equal(t.fn_coeffs, g[f"{tag}_fn"])
    np.testing.assert_array_equal(t.smooth_spline.c, g[f"{tag}_sc"])
    np.testing.assert_array_equal(t.fn_spline.c, g[f"{tag}_fc"])
    np.testing.assert_array_equal(t.smooth_spline.x, g[f"{tag}_x"])
    np.testing.assert_array_equal(t.near_field(g[f"{tag}_probe_r"]), g[f"{tag}_probe_nv"])


@pytest.mark.parametrize("name", SMALL)
def test_oracle_short_range_matches_reference(name):
    g = golden(name)
    b = _basis(float(g["delta"]))
    r_c = float(g["r_c"])
    i, j = O.pairs_within(g["h"], g["pos"], r_c + float(g["skin"]))
    np.testing.assert_array_equal(i, g["pi"])
    np.testing.assert_array_equal(j, g["pj"])
    t = O.pair_table(b, r_c)
    E, F, P, cnt = O.short_range(g["h"], g["pos"], g["q"], i, j, b, r_c, t)
    assert cnt == int(g["count"])
    assert O.rel_scalar(E, g["E_tab"]) <= 1e-13
    assert O.rel_frobenius(P, g["P_tab"]) <= 1e-13
    assert O.rms_rel_forces(F, g["F_tab"]) <= 1e-13
    E, F, P, _ = O.short_range(g["h"], g["pos"], g["q"], i, j, b, r_c, None)
    assert O.rel_scalar(E, g["E_exact"]) <= 1e-13
    assert O.rel_frobenius(P, g["P_exact"]) <= 1e-13
    assert O.rms_rel_forces(F, g["F_exact"]) <= 1e-13


def test_oracle_config0_near_matches_reference():
    g = golden("near_cfg0")
    w, pos, q = workloads.generate(0)
    b = _basis(w.delta)
    i, j = O.pairs_within_kdtree(np.diag(w.h), pos, w.r_c)
    E, F, P, cnt = O.short_range(w.h, pos, q, i, j, b, w.r_c, O.pair_table(b, w.r_c))
    assert cnt == int(g["count"])
    assert O.rel_scalar(E, g["E"]) <= 1e-13
    assert O.rel_frobenius(P, g["P"]) <= 1e-13
    assert O.rms_rel_forces(F, g["F_sel"]) <= 1e-13


def test_geometry_error_and_neighbor_list_host():
    from paper_2601_00161_b200 import Cell
    from paper_2601_00161_b200.errors import CellError, GeometryError
    from paper_2601_00161_b200.system import NeighborList, check_cutoff, minimum_image
    with pytest.raises(GeometryError):
        check_cutoff(Cell.orthorhombic([10.0, 10.0, 10.0]), 5.0)
    assert issubclass(GeometryError, CellError)
    nb = NeighborList(i=np.array([0, 1]), j=np.array([1, 2]), r_c=1.0, skin=0.0)
    assert nb.n_pairs == 2
    c = Cell.orthorhombic([4.0, 5.0, 6.0])
    np.testing.assert_allclose(minimum_image(c, np.array([[3.5, -4.0, 2.9]])),
                               [[-0.5, 1.0, 2.9]])


# ------------------------------------------------------------- GPU: parity


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _kern(delta, r_c):
    from paper_2601_00161_b200 import SplitKernel, build_pswf, solve_bandwidth
    return SplitKernel(basis=build_pswf(solve_bandwidth(delta)), r_c=r_c)


def _sys(h, pos, q):
    from paper_2601_00161_b200 import Cell, ParticleSystem
    return ParticleSystem(cell=Cell(np.asarray(h, dtype=float)), positions=pos, charges=q)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("use_table", [True, False])
@pytest.mark.parametrize("listed", [False, True])
def test_short_range_small_against_reference(name, use_table, listed):
    _torch()
    from paper_2601_00161_b200.realspace import build_pair_table, short_range
    from paper_2601_00161_b200.system import NeighborList
    g = golden(name)
    r_c = float(g["r_c"])
    if not listed and float(g["skin"]) > 0.0:
        pytest.skip("cell-list path enumerates pairs within r_c (no skin)")
    kern = _kern(float(g["delta"]), r_c)
    table = build_pair_table(kern) if use_table else None
    sys_ = _sys(g["h"], g["pos"], g["q"])
    nb = NeighborList(i=g["pi"], j=g["pj"], r_c=r_c, skin=float(g["skin"])) if listed else None
    res = short_range(sys_, kern, nb, table=table)
    sfx = "tab" if use_table else "exact"
    assert res.pair_count == int(g["count"])
    assert O.rel_scalar(res.energy, g[f"E_{sfx}"]) <= TOL
    assert O.rel_frobenius(res.pressure, g[f"P_{sfx}"]) <= TOL
    assert O.rms_rel_forces(res.forces, g[f"F_{sfx}"]) <= TOL
    np.testing.assert_array_equal(res.pressure, res.pressure.T)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [0, 1, 2])
@pytest.mark.parametrize("div", [1, 2, 3])
def test_short_range_configs_against_reference(idx, div):
    torch = _torch()
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table, out7_to_pressure
    g = golden(f"near_cfg{idx}")
    w, pos, q = workloads.generate(idx)
    kern = _kern(w.delta, w.r_c)
    plan = NearFieldPlan(kern, build_pair_table(kern), capacity=w.n, cell_div=div)
    plan.set_cell(w.h)
    out7, F, st = plan.evaluate(torch.as_tensor(pos, device="cuda"),
                                torch.as_tensor(q, device="cuda"))
    st = st.cpu().numpy()
    assert int(st[0]) == int(g["count"]) and int(st[1]) == -1
    E, P = out7_to_pressure(out7)
    F = F.cpu().numpy()
    assert O.rel_scalar(E, g["E"]) <= TOL
    assert O.rel_frobenius(P, g["P"]) <= TOL
    assert O.rms_rel_forces(F[g["F_idx"]], g["F_sel"]) <= TOL
    assert np.abs(F.sum(axis=0)).max() <= 1e-9 * float(g["F_rms"]) * w.n ** 0.5


@pytest.mark.gpu
def test_coulomb_solver_totals_config0_against_reference():
    """CoulombSolver.evaluate (evaluate.py:114-144): near + far + self +
    background on the device, against the reference's totals."""
    _torch()
    from paper_2601_00161_b200 import CoulombSolver, EwaldParameters
    g = golden("near_cfg0")
    w, pos, q = workloads.generate(0)
    solver = CoulombSolver(_sys(w.h, pos, q).cell,
                           EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                           fixed_M=w.M))
    out = solver.evaluate(_sys(w.h, pos, q))
    u = g["tot_u"]
    for got, want in zip((out.u_near, out.u_far, out.u_self, out.u_background), u):
        assert abs(got - want) <= TOL * max(abs(want), 1.0)
    assert O.rel_scalar(out.energy, float(np.sum(u))) <= TOL
    assert out.pair_count == int(g["tot_count"])
    assert O.rel_frobenius(out.pressure, g["tot_P"]) <= TOL
    assert O.rms_rel_forces(out.forces, g["tot_F"]) <= TOL


@pytest.mark.gpu
def test_near_config3_triclinic_rows_against_oracle():
    """Config 3 (1M charges, triclinic): forces on 64 particles against the
    oracle's brute-force rows; momentum and pressure symmetry globally."""
    torch = _torch()
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table, out7_to_pressure
    w, pos, q = workloads.generate(3)
    kern = _kern(w.delta, w.r_c)
    table = build_pair_table(kern)
    plan = NearFieldPlan(kern, table, capacity=w.n)
    plan.set_cell(w.h)
    out7, F, st = plan.evaluate(torch.as_tensor(pos, device="cuda"),
                                torch.as_tensor(q, device="cuda"))
    F = F.cpu().numpy()
    rows = np.random.default_rng(5).choice(w.n, 64, replace=False)
    b = _basis(w.delta)
    ref = O.short_range_rows(w.h, pos, q, rows, b, w.r_c, O.pair_table(b, w.r_c))
    assert O.rms_rel_forces(F[rows], ref) <= TOL
    assert np.abs(F.sum(axis=0)).max() <= 1e-8 * np.sqrt(np.mean(np.sum(F * F, 1))) * w.n ** 0.5
    E, P = out7_to_pressure(out7)
    assert np.isfinite(E) and int(st.cpu()[0]) > 0


@pytest.mark.gpu
def test_near_deterministic_and_permutation_invariant():
    torch = _torch()
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table
    w, pos, q = workloads.generate(1)
    kern = _kern(w.delta, w.r_c)
    plan = NearFieldPlan(kern, build_pair_table(kern), capacity=w.n)
    plan.set_cell(w.h)
    P = torch.as_tensor(pos, device="cuda")
    Q = torch.as_tensor(q, device="cuda")
    a7, aF, _ = plan.evaluate(P, Q)
    a7, aF = a7.clone(), aF.clone()
    b7, bF, _ = plan.evaluate(P, Q)
    assert torch.equal(a7, b7) and torch.equal(aF, bF)
    perm = np.random.default_rng(0).permutation(w.n)
    c7, cF, _ = plan.evaluate(P[perm].contiguous(), Q[perm].contiguous())
    assert O.rel_scalar(c7[0].item(), a7[0].item()) <= 1e-13
    assert O.rms_rel_forces(cF.cpu().numpy(), aF.cpu().numpy()[perm]) <= 1e-13


@pytest.mark.gpu
def test_near_edge_cases():
    torch = _torch()
    from paper_2601_00161_b200 import Cell, ParticleSystem
    from paper_2601_00161_b200.errors import GeometryError, SingularPairError
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table, short_range
    from paper_2601_00161_b200.system import NeighborList
    kern = _kern(1e-5, 1.5)
    table = build_pair_table(kern)
    cell = Cell.orthorhombic([10.0, 10.0, 10.0])
    # coincident particles raise, through both paths
    s = ParticleSystem(cell=cell, positions=np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 1.0]]),
                       charges=np.array([1.0, -1.0]))
    with pytest.raises(SingularPairError):
        short_range(s, kern, None, table)
    with pytest.raises(SingularPairError):
        short_range(s, kern, NeighborList(i=np.array([0]), j=np.array([1]), r_c=1.5, skin=0.0),
                    table)
    # beyond the cutoff: exact zeros; single pair across the periodic face
    s = ParticleSystem(cell=cell, positions=np.array([[0.2, 5.0, 5.0], [9.6, 5.0, 5.0]]),
                       charges=np.array([1.0, -1.0]))
    r = short_range(s, kern, None, table)
    d = 0.6
    assert r.pair_count == 1
    assert r.energy == pytest.approx(-float(table.near_field(np.array([d]))[0]), rel=1e-12)
    assert r.forces[0, 0] == pytest.approx(-float(table.fn_weight(np.array([d]))[0]) / d ** 2,
                                           rel=1e-12)
    s = ParticleSystem(cell=cell, positions=np.array([[1.0, 1.0, 1.0], [5.0, 1.0, 1.0]]),
                       charges=np.array([1.0, -1.0]))
    r = short_range(s, kern, None, table)
    assert r.energy == 0.0 and r.pair_count == 0 and not np.any(r.forces)
    assert not np.any(r.pressure)
    # one particle, and a cutoff too large for the cell
    s = ParticleSystem(cell=cell, positions=np.array([[1.0, 2.0, 3.0]]), charges=np.array([1.0]))
    r = short_range(s, kern, None, table)
    assert r.energy == 0.0 and r.pair_count == 0
    plan = NearFieldPlan(_kern(1e-5, 6.0), None)
    with pytest.raises(GeometryError):
        plan.set_cell(cell)
    # empty device system
    plan = NearFieldPlan(kern, table)
    plan.set_cell(cell)
    out7, F, st = plan.evaluate(torch.zeros((0, 3), dtype=torch.float64, device="cuda"),
                                torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert not torch.any(out7) and int(st[0]) == 0
    # unwrapped positions (outside the cell) give the wrapped result
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 10, (200, 3))
    qq = rng.normal(size=200)
    base = plan.evaluate(torch.as_tensor(pos, device="cuda"), torch.as_tensor(qq, device="cuda"))
    shifted = pos + np.array([10.0, -20.0, 30.0]) * (rng.integers(0, 2, (200, 1)))
    moved = plan.evaluate(torch.as_tensor(shifted, device="cuda"),
                          torch.as_tensor(qq, device="cuda"))
    assert O.rel_scalar(moved[0][0].item(), base[0][0].item()) <= 1e-12
    assert O.rms_rel_forces(moved[1].cpu().numpy(), base[1].cpu().numpy()) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", SMALL)
def test_build_cell_list_small_against_reference(name):
    """Device pair enumeration = the reference's build_cell_list output
    (same pairs, same (i, j) order), including skin and a triclinic cell."""
    _torch()
    from paper_2601_00161_b200.realspace import build_cell_list
    g = golden(name)
    nb = build_cell_list(_sys(g["h"], g["pos"], g["q"]), float(g["r_c"]), skin=float(g["skin"]))
    np.testing.assert_array_equal(nb.i, g["pi"])
    np.testing.assert_array_equal(nb.j, g["pj"])


@pytest.mark.gpu
def test_build_cell_list_config0_and_short_range_through_list():
    _torch()
    from paper_2601_00161_b200.realspace import build_cell_list, build_pair_table, short_range
    g = golden("near_cfg0")
    w, pos, q = workloads.generate(0)
    nb = build_cell_list(_sys(w.h, pos, q), w.r_c)
    i, j = O.pairs_within_kdtree(np.diag(w.h), pos, w.r_c)
    np.testing.assert_array_equal(nb.i, i)
    np.testing.assert_array_equal(nb.j, j)
    kern = _kern(w.delta, w.r_c)
    res = short_range(_sys(w.h, pos, q), kern, nb, build_pair_table(kern))
    assert res.pair_count == int(g["count"])
    assert O.rel_scalar(res.energy, g["E"]) <= TOL
    assert O.rms_rel_forces(res.forces, g["F_sel"]) <= TOL


@pytest.mark.gpu
def test_coulomb_solver_explicit_list_and_rebind():
    """CoulombSolver.evaluate with a caller NeighborList equals the cell-list
    path; after an NPT-style rebind (M pinned) the near plan follows the new
    cell (evaluate.py:99-112)."""
    _torch()
    from paper_2601_00161_b200 import Cell, CoulombSolver, EwaldParameters, ParticleSystem
    from paper_2601_00161_b200.realspace import build_cell_list
    w, pos, q = workloads.generate(0)
    cell = Cell(np.asarray(w.h, dtype=float))
    s = ParticleSystem(cell=cell, positions=pos, charges=q)
    solver = CoulombSolver(cell, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                                 fixed_M=w.M))
    a = solver.evaluate(s)
    b = solver.evaluate(s, neighbors=build_cell_list(s, w.r_c))
    assert a.pair_count == b.pair_count
    assert O.rel_scalar(b.u_near, a.u_near) <= 1e-13
    assert O.rms_rel_forces(b.forces, a.forces) <= 1e-13
    cell2 = Cell(np.asarray(w.h, dtype=float) * 1.01)
    solver.rebind_cell(cell2, fixed_M=w.M)
    s2 = ParticleSystem(cell=cell2, positions=pos * 1.01, charges=q)
    c = solver.evaluate(s2)
    fresh = CoulombSolver(cell2, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                                 fixed_M=w.M)).evaluate(s2)
    assert c.pair_count == fresh.pair_count
    assert O.rel_scalar(c.energy, fresh.energy) <= 1e-12
    assert O.rms_rel_forces(c.forces, fresh.forces) <= 1e-12
    from paper_2601_00161_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        solver.evaluate(s)


@pytest.mark.gpu
def test_coulomb_graphed_step_matches_evaluate():
    """CoulombSolver.graphed: near and far field on two streams of one CUDA
    graph give the evaluate() totals; replays after an in-place update follow
    the new positions."""
    torch = _torch()
    from paper_2601_00161_b200 import Cell, CoulombSolver, EwaldParameters, ParticleSystem
    from paper_2601_00161_b200.realspace import out7_to_pressure
    w, pos, q = workloads.generate(0)
    cell = Cell(np.asarray(w.h, dtype=float))
    solver = CoulombSolver(cell, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                                 fixed_M=w.M))
    P = torch.as_tensor(pos, device="cuda")
    Q = torch.as_tensor(q, device="cuda")
    g, out = solver.graphed(P, Q)
    rng = np.random.default_rng(1)
    for step in range(2):
        pos2 = (pos + 0.01 * step * rng.normal(size=pos.shape)) % np.diag(w.h)
        P.copy_(torch.as_tensor(pos2))
        g.replay()
        torch.cuda.synchronize()
        ref = solver.evaluate(ParticleSystem(cell=cell, positions=pos2, charges=q))
        En, Pn = out7_to_pressure(out["out7_near"])
        Ef, Pf = out7_to_pressure(out["out7_far"])
        assert O.rel_scalar(En, ref.u_near) <= 1e-13
        assert O.rel_scalar(Ef, ref.u_far) <= 1e-13
        assert int(out["stats"][0]) == ref.pair_count
        assert O.rms_rel_forces(out["forces"].cpu().numpy(), ref.forces) <= 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("idx,R", [(1, 1), (1, 2), (1, 4), (3, 3)])
def test_slab_local_near_field_emulated_on_one_gpu(idx, R):
    """esp_near_evaluate_local for R slab ranks run one after another on one
    device (owned particles + ghosts within reach of the slab, chosen as
    SlabNearField chooses them): the summed energy / pressure / pair count
    and every rank's forces equal the single-plan pair sum."""
    torch = _torch()
    from paper_2601_00161_b200 import Cell
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table, out7_to_pressure
    from paper_2601_00161_b200.slab_near import CudaNearOps, SlabNearField
    w, pos, q = workloads.generate(idx)
    kern = _kern(w.delta, w.r_c)
    table = build_pair_table(kern)
    full = NearFieldPlan(kern, table, capacity=w.n)
    full.set_cell(w.h)
    o7, F0, st0 = full.evaluate(torch.as_tensor(pos, device="cuda"),
                                torch.as_tensor(q, device="cuda"))
    E0, P0 = out7_to_pressure(o7)
    F0 = F0.cpu().numpy()
    ops = CudaNearOps(kern, table, Cell(np.asarray(w.h, dtype=float)))
    bounds = np.linspace(0.0, 1.0, R + 1) + 0.01
    sl = SlabNearField.__new__(SlabNearField)   # geometry only, no process group
    sl.R, sl.rank, sl.group = R, 0, None
    sl.cell = Cell(np.asarray(w.h, dtype=float))
    sl.reach = w.r_c
    sl.bounds = bounds
    sl.hinv = np.linalg.inv(sl.cell.h)
    sl.dz = w.r_c / sl.cell.perpendicular_widths()[2] * (1 + 1e-9) + 1e-12
    owner = sl.owner(pos)
    s = sl.frac_z(pos)
    tot = np.zeros(8)
    F = np.zeros_like(F0)
    for r in range(R):
        own = np.nonzero(owner == r)[0]
        gh = np.nonzero((owner != r) & sl._ghost_mask(s, r))[0]
        idx_all = np.concatenate([own, gh])
        out8, Fr, st = ops.evaluate(torch.as_tensor(pos[idx_all], device="cuda"),
                                    torch.as_tensor(q[idx_all], device="cuda"), len(own))
        tot += out8.cpu().numpy()
        F[own] = Fr.cpu().numpy()
    assert abs(tot[0] - E0) <= 1e-12 * abs(E0)
    P = np.array([[tot[1], tot[2], tot[3]], [tot[2], tot[4], tot[5]], [tot[3], tot[5], tot[6]]])
    assert O.rel_frobenius(P, P0) <= 1e-12
    assert int(round(0.5 * tot[7])) == int(st0[0])
    assert O.rms_rel_forces(F, F0) <= 1e-12


@pytest.mark.gpu
def test_slab_coulomb_solver_single_rank_equals_coulomb_solver():
    """SlabCoulombSolver at R = 1 on the GPU (slab k-space plan + slab near
    field) equals CoulombSolver.evaluate."""
    torch = _torch()
    from paper_2601_00161_b200 import Cell, CoulombSolver, EwaldParameters, ParticleSystem
    from paper_2601_00161_b200.slab_near import SlabCoulombSolver
    w, pos, q = workloads.generate(1)
    params = EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                             prefactor=0.5)
    cell = Cell(np.asarray(w.h, dtype=float))
    ref = CoulombSolver(cell, params).evaluate(ParticleSystem(cell=cell, positions=pos, charges=q))
    sc = SlabCoulombSolver(w.h, params)
    mine = sc.owned(pos)
    assert mine.all()
    r = sc.evaluate(torch.as_tensor(pos, device="cuda"), torch.as_tensor(q, device="cuda"))
    assert O.rel_scalar(r.u_near, ref.u_near) <= 1e-12
    assert O.rel_scalar(r.u_far, ref.u_far) <= 1e-10
    assert O.rel_scalar(r.energy, ref.energy) <= 1e-10
    assert O.rel_frobenius(r.pressure, ref.pressure) <= 1e-10
    assert O.rms_rel_forces(r.forces.cpu().numpy(), ref.forces) <= 1e-10
    assert r.pair_count == ref.pair_count


def test_pair_table_argument_errors_and_cutoff_zero():
    """realspace.py:81-82 (bad r_in) and :60-61/:66-67 (zero beyond r_c)."""
    from paper_2601_00161_b200.errors import RealspaceError
    from paper_2601_00161_b200.realspace import build_pair_table
    kern = _kern(1e-5, 0.9)
    with pytest.raises(RealspaceError):
        build_pair_table(kern, r_in=kern.r_c)
    with pytest.raises(RealspaceError):
        build_pair_table(kern, r_in=-0.1)
    t = build_pair_table(kern)
    r = np.array([kern.r_c, 1.1 * kern.r_c, 5.0 * kern.r_c])
    assert np.all(t.near_field(r) == 0.0)
    assert np.all(t.fn_weight(r)[1:] == 0.0)
    assert build_pair_table(_kern(1e-8, 1.0)).r_in <= 0.1


@pytest.mark.gpu
def test_near_forces_are_energy_gradient_and_pressure_is_box_derivative():
    """test_realspace.py:235-282 analogues on the device: forces against a
    4-point finite difference of the pair-sum energy, diagonal pressure
    against -(L_a/V) dE/dL_a at fixed fractional coordinates."""
    _torch()
    from paper_2601_00161_b200 import Cell, ParticleSystem
    from paper_2601_00161_b200.realspace import short_range
    kern = _kern(1e-6, 1.3)
    rng = np.random.default_rng(15)
    L = np.array([5.0, 5.5, 6.0])
    pos = rng.uniform(0, 1, (24, 3)) * L
    q = rng.normal(size=24)
    q -= q.mean()
    cell = Cell.orthorhombic(L)
    base = short_range(ParticleSystem(cell=cell, positions=pos, charges=q), kern)
    step = 1e-5
    for idx in (0, 7, 13):
        for axis in range(3):
            num = 0.0
            for sgn, coef in ((1, 8.0), (-1, -8.0), (2, -1.0), (-2, 1.0)):
                p2 = pos.copy()
                p2[idx, axis] += sgn * step
                num += coef * short_range(ParticleSystem(cell=cell, positions=p2, charges=q),
                                          kern).energy
            num /= 12.0 * step
            assert base.forces[idx, axis] == pytest.approx(-num, abs=2e-6)
    frac = pos / L
    for axis in range(3):
        num = 0.0
        for sgn, coef in ((1, 8.0), (-1, -8.0), (2, -1.0), (-2, 1.0)):
            L2 = L.copy()
            L2[axis] += sgn * step
            c2 = Cell.orthorhombic(L2)
            num += coef * short_range(ParticleSystem(cell=c2, positions=frac * L2, charges=q),
                                      kern).energy
        num /= 12.0 * step
        assert base.pressure[axis, axis] == pytest.approx(-L[axis] / cell.volume * num, abs=2e-6)


@pytest.mark.gpu
def test_near_translation_invariance():
    torch = _torch()
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table
    w, pos, q = workloads.generate(2)
    kern = _kern(w.delta, w.r_c)
    plan = NearFieldPlan(kern, build_pair_table(kern), capacity=w.n)
    plan.set_cell(w.h)
    a7, aF, _ = plan.evaluate(torch.as_tensor(pos, device="cuda"), torch.as_tensor(q, device="cuda"))
    a7, aF = a7.clone(), aF.clone()
    shifted = (pos + np.array([1.7, -2.3, 0.9])) % np.diag(w.h)
    b7, bF, _ = plan.evaluate(torch.as_tensor(shifted, device="cuda"),
                              torch.as_tensor(q, device="cuda"))
    assert O.rel_scalar(b7[0].item(), a7[0].item()) <= 1e-11
    assert O.rms_rel_forces(bF.cpu().numpy(), aF.cpu().numpy()) <= 1e-11
    assert O.rel_frobenius(b7[1:].cpu().numpy(), a7[1:].cpu().numpy()) <= 1e-11


@pytest.mark.gpu
def test_near_orderings_agree():
    """Cell-octant sub-order (default), plain cell order (ESP_NEAR_OCT=0) and
    the per-particle row kernel (ESP_NEAR_KERNEL=rows) sum the same pairs:
    equal pair counts, energies / forces to round-off."""
    import os
    torch = _torch()
    from paper_2601_00161_b200.realspace import NearFieldPlan, build_pair_table
    w, pos, q = workloads.generate(1)
    kern = _kern(w.delta, w.r_c)
    table = build_pair_table(kern)
    P = torch.as_tensor(pos, device="cuda")
    Q = torch.as_tensor(q, device="cuda")
    res = []
    for env in ({}, {"ESP_NEAR_OCT": "0"}, {"ESP_NEAR_KERNEL": "rows"}):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            plan = NearFieldPlan(kern, table, capacity=w.n)
            plan.set_cell(w.h)
            o7, F, st = plan.evaluate(P, Q)
            res.append((o7.cpu().numpy(), F.cpu().numpy(), int(st[0])))
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    for o7, F, cnt in res[1:]:
        assert cnt == res[0][2]
        assert O.rel_scalar(o7[0], res[0][0][0]) <= 1e-12
        assert O.rms_rel_forces(F, res[0][1]) <= 1e-12
