"""GPU parity: the CUDA path (through the C ABI) against the reference
goldens and the CPU oracle.

Tolerances (north star): fp64 energy / pressure (Frobenius) / forces (rms
relative over atoms) within 1e-10; fp32 mode within 1e-5.  Spread grids
are compared at 1e-13 of the grid's max.
"""

import numpy as np
import pytest

from conftest import SMALL_CASES, TRI_CASES, golden
from oracle import esp_oracle as O
from paper_2601_00161_b200 import workloads

pytestmark = pytest.mark.gpu

F64_TOL = 1e-10
F32_TOL = 1e-5


def _torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _plan_for(g, M=None, precision="fp64", deterministic=True, capacity=1 << 12):
    from paper_2601_00161_b200 import EspPlan, build_pswf, tabulate_window
    b = build_pswf(float(g["c"])) if "c" in g else None
    if b is None:
        from paper_2601_00161_b200 import solve_bandwidth
        b = build_pswf(solve_bandwidth(float(g["delta"])))
    P = int(g["P"])
    w = tabulate_window(b, P)
    plan = EspPlan(tuple(M if M is not None else g["M"]), P, w, b, float(g["r_c"]),
                   precision=precision, deterministic=deterministic, capacity=capacity)
    plan.set_cell(g["h"])
    return plan


def _dev(torch, a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def _run(plan, pos, q, want_forces=True):
    torch = _torch()
    from paper_2601_00161_b200.plan import out7_to_tensor
    out7, F = plan.evaluate(_dev(torch, pos), _dev(torch, q), want_forces)
    E, Pt = out7_to_tensor(out7)
    return E, Pt, (F.cpu().numpy() if F is not None else None)


@pytest.mark.parametrize("name", SMALL_CASES)
def test_spread_grid_matches_reference(name):
    torch = _torch()
    g = golden(name)
    plan = _plan_for(g)
    grid = plan.spread(_dev(torch, g["pos"]), _dev(torch, g["q"]))
    got = grid.permute(2, 1, 0).cpu().numpy()           # device [z][y][x] -> [x][y][z]
    ref = g["grid"]
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", SMALL_CASES)
def test_small_cases_energy_pressure_forces(name):
    g = golden(name)
    plan = _plan_for(g)
    E, Pt, F = _run(plan, g["pos"], g["q"])
    assert O.rel_scalar(E, g["E"]) <= F64_TOL
    assert O.rel_frobenius(Pt, g["Pt"]) <= F64_TOL
    scale = np.sqrt(np.mean(np.sum(g["F"] ** 2, axis=1)))
    if scale > 1e-12:
        assert O.rms_rel_forces(F, g["F"]) <= F64_TOL
    else:  # a lone charge feels no self force: both are round-off zero
        assert np.max(np.abs(F)) <= 1e-12


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_configs_match_reference_goldens(idx):
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    g = golden(f"cfg{idx}")
    w, pos, q = workloads.generate(idx)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                          fixed_M=w.M, cell_type=w.cell_type))
    r = s.evaluate(pos, q)
    assert O.rel_scalar(r.energy, g["E"]) <= F64_TOL
    assert O.rel_frobenius(r.pressure, g["Pt"]) <= F64_TOL
    assert O.rms_rel_forces(r.forces[g["F_idx"]], g["F_sel"]) <= F64_TOL
    if idx == 0:
        plan = s.plan
        torch = _torch()
        grid = plan.spread(_dev(torch, pos), _dev(torch, q)).permute(2, 1, 0).cpu().numpy()
        assert np.max(np.abs(grid - g["grid"])) <= 1e-13 * np.max(np.abs(g["grid"]))


def test_pressure_only_path_is_one_forward_fft():
    """Energy + full pressure tensor ride on one forward transform and no
    inverse (test_mesh.py:163-172), through the drop-in mesh API."""
    _torch()
    from paper_2601_00161_b200 import (Cell, ParticleSystem, SplitKernel, TransformProvider,
                                       build_pswf, forward_density, long_range_energy,
                                       long_range_forces, long_range_pressure, plan_grid,
                                       solve_bandwidth)
    g = golden("small_brick_p6")
    b = build_pswf(solve_bandwidth(float(g["delta"])))
    kern = SplitKernel(basis=b, r_c=float(g["r_c"]))
    cell = Cell(g["h"])
    spec = plan_grid(cell, kern, delta_spread=float(g["delta"]), P=int(g["P"]),
                     spread_basis=b, fixed_M=tuple(g["M"]))
    sys = ParticleSystem(cell=cell, positions=g["pos"], charges=g["q"])
    prov = TransformProvider()
    rho_hat = forward_density(sys, spec, prov)
    E = long_range_energy(rho_hat, kern, spec, cell)
    Pt = long_range_pressure(rho_hat, kern, spec, cell)
    assert prov.forward_count == 1 and prov.inverse_count == 0
    assert O.rel_scalar(E, g["E"]) <= F64_TOL
    assert O.rel_frobenius(Pt, g["Pt"]) <= F64_TOL
    F = long_range_forces(rho_hat, sys, kern, spec, cell, provider=prov)
    assert prov.forward_count == 1 and prov.inverse_count == 3
    assert O.rms_rel_forces(F, g["F"]) <= F64_TOL
    # the spectrum itself: masked full-spectrum values vs the reference
    full = rho_hat.full()
    plan = O.make_plan(g["h"], tuple(g["M"]), int(g["P"]), float(g["delta"]), float(g["r_c"]))
    m = O.Modes(plan)
    ref = g["rho_hat_masked"]
    assert np.max(np.abs(full[m.mask] - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_wrong_space_rejected():
    _torch()
    from paper_2601_00161_b200 import (Cell, MeshError, ParticleSystem, SplitKernel,
                                       build_pswf, long_range_energy, long_range_forces,
                                       long_range_pressure, plan_grid, solve_bandwidth,
                                       spread_charges)
    b = build_pswf(solve_bandwidth(1e-4))
    kern = SplitKernel(basis=b, r_c=1.0)
    cell = Cell.orthorhombic([6.0, 6.0, 6.0])
    spec = plan_grid(cell, kern, delta_spread=1e-4, P=5, oversampling=2.0, spread_basis=b)
    pos, q = workloads.random_neutral_system(8, [6.0] * 3, seed=2)
    sys = ParticleSystem(cell=cell, positions=pos, charges=q)
    rho = spread_charges(sys, spec)
    for fn in (long_range_energy, long_range_pressure):
        with pytest.raises(MeshError):
            fn(rho, kern, spec, cell)
    with pytest.raises(MeshError):
        long_range_forces(rho, sys, kern, spec, cell)


def test_ik_forces_conserve_momentum():
    g = golden("small_brick_p8")
    plan = _plan_for(g)
    _, _, F = _run(plan, g["pos"], g["q"])
    assert np.linalg.norm(F.sum(axis=0)) < 1e-10 * np.linalg.norm(F, axis=1).max()
    w, pos, q = workloads.generate(1)
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M))
    F = s.evaluate(pos, q).forces
    assert np.linalg.norm(F.sum(axis=0)) < 1e-10 * np.linalg.norm(F, axis=1).max()


def test_deterministic_bitwise():
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w, pos, q = workloads.generate(1)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M))
    P_, Q_ = _dev(torch, pos), _dev(torch, q)
    a7, aF = s.evaluate_device(P_, Q_)
    a7, aF = a7.clone(), aF.clone()
    perm = torch.randperm(P_.shape[0], device="cuda")
    for _ in range(3):
        b7, bF = s.evaluate_device(P_, Q_)
        assert torch.equal(a7, b7) and torch.equal(aF, bF)
    # a permuted particle order gives the same physics to round-off
    c7, cF = s.evaluate_device(P_[perm].contiguous(), Q_[perm].contiguous())
    assert torch.allclose(c7, a7, rtol=1e-13, atol=0)
    assert torch.allclose(cF, aF[perm], rtol=1e-11, atol=1e-15)


def test_fp32_mode_within_1e5():
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    for idx in (0, 1):
        g = golden(f"cfg{idx}")
        w, pos, q = workloads.generate(idx)
        s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                              fixed_M=w.M, precision="fp32"))
        r = s.evaluate(pos, q)
        assert O.rel_scalar(r.energy, g["E"]) <= F32_TOL
        assert O.rel_frobenius(r.pressure, g["Pt"]) <= F32_TOL
        assert O.rms_rel_forces(r.forces[g["F_idx"]], g["F_sel"]) <= F32_TOL


@pytest.mark.parametrize("name,M", TRI_CASES)
def test_triclinic_matches_oracle(name, M):
    g = golden(name)
    plan = _plan_for(g, M=M)
    E, Pt, F = _run(plan, g["pos"], g["q"])
    op = O.make_plan(g["h"], M, int(g["P"]), float(g["delta"]), float(g["r_c"]))
    oE, oP, oF = O.kspace(op, g["pos"], g["q"])
    assert O.rel_scalar(E, oE) <= F64_TOL
    assert O.rel_frobenius(Pt, oP) <= F64_TOL
    assert O.rms_rel_forces(F, oF) <= F64_TOL
    tol = 50 * float(g["delta"])
    assert O.rel_scalar(E, g["E_direct"]) <= tol
    assert O.rms_rel_forces(F, g["F_direct"]) <= tol


def test_edge_particles_on_faces_and_capacity_growth():
    torch = _torch()
    g = golden("small_brick_p7")           # odd P: round-half-even anchors
    plan = _plan_for(g, capacity=4)
    L = np.diag(g["h"])
    h = L / np.asarray(g["M"])
    pos = np.array([[0.0, 0.0, 0.0], [np.nextafter(L[0], 0), 1.0, 2.0],
                    [2.5 * h[0], 3.5 * h[1], 0.5 * h[2]],      # exact .5: ties to even
                    [L[0] / 2, L[1] / 2, np.nextafter(L[2], 0)]])
    q = np.array([1.0, -0.5, 0.75, -1.25])
    pos = workloads.wrap_positions(g["h"], pos)
    E, Pt, F = _run(plan, pos, q)
    op = O.make_plan(g["h"], tuple(g["M"]), int(g["P"]), float(g["delta"]), float(g["r_c"]))
    oE, oP, oF = O.kspace(op, pos, q)
    assert O.rel_scalar(E, oE) <= F64_TOL
    assert O.rel_frobenius(Pt, oP) <= F64_TOL
    assert O.rms_rel_forces(F, oF) <= F64_TOL
    # grow past the initial capacity of 4
    E2, P2, F2 = _run(plan, g["pos"], g["q"])
    assert O.rel_scalar(E2, g["E"]) <= F64_TOL
    # empty system: zero energy, pressure
    empty = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    out7, _ = plan.evaluate(empty, torch.zeros(0, dtype=torch.float64, device="cuda"),
                            want_forces=True)
    assert torch.count_nonzero(out7).item() == 0


def test_counters_and_launch_count():
    g = golden("small_cube_p6")
    plan = _plan_for(g)
    plan.reset_counters()
    _run(plan, g["pos"], g["q"], want_forces=False)
    assert plan.counters() == (1, 0)
    _run(plan, g["pos"], g["q"], want_forces=True)
    assert plan.counters() == (2, 3)
    assert plan.launches_last_step() >= 7


@pytest.mark.slow
def test_config4_geometry_subset_against_oracle():
    """384^3 grid, P=8 (config 4 geometry) with a 60k-charge subset: the full
    CUDA pipeline against the oracle at the north-star tolerances."""
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w = workloads.workload(4)
    rng = np.random.default_rng(44)
    n = 60_000
    pos = workloads.wrap_positions(w.h, rng.uniform(0, 300.0, (n, 3)))
    q = np.where(np.arange(n) % 2 == 0, 0.7, -0.7)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M))
    r = s.evaluate(pos, q)
    op = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    oE, oP, oF = O.kspace(op, pos, q)
    assert O.rel_scalar(r.energy, oE) <= F64_TOL
    assert O.rel_frobenius(r.pressure, oP) <= F64_TOL
    assert O.rms_rel_forces(r.forces, oF) <= F64_TOL


def test_cuda_graph_replay_matches_eager():
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w, pos, q = workloads.generate(0)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M))
    P_, Q_ = _dev(torch, pos), _dev(torch, q)
    e7, eF = s.evaluate_device(P_, Q_)
    e7, eF = e7.clone(), eF.clone()
    g, o7, oF = s.graphed(P_, Q_)
    o7.zero_()
    oF.zero_()
    s.plan.reset_counters()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o7, e7) and torch.equal(oF, eF)
    # replays count their transforms (1 forward + 3 inverse per ik step)
    assert s.plan.counters() == (1, 3)
    g.replay()
    assert s.plan.counters() == (2, 6)
    # new positions in place -> replay recomputes
    P_.add_(0.37)
    g.replay()
    f7, fF = s.evaluate_device(P_, Q_)
    torch.cuda.synchronize()
    assert torch.equal(o7, f7) and torch.equal(oF, fF)
    hs = s.host_stepper(w.n)
    hs.positions.copy_(torch.as_tensor(pos))
    hs.charges.copy_(torch.as_tensor(q))
    h7, hF = hs.step()
    assert torch.equal(h7, e7.cpu()) and torch.equal(hF, eF.cpu())
    # new charges through the host buffers (copied on the forked stream):
    # the step must use them
    q2 = q * np.linspace(0.5, 1.5, len(q))
    hs.charges.copy_(torch.as_tensor(q2))
    h7, hF = hs.step()
    r7, rF = s.evaluate_device(torch.as_tensor(pos, device="cuda"),
                               torch.as_tensor(q2, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(h7, r7.cpu()) and torch.equal(hF, rF.cpu())


@pytest.mark.slow
def test_config3_triclinic_against_oracle():
    """Config 3 (1e6 charges, triclinic 192x192x256, P=8): E and the full
    pressure tensor against the oracle; forces on a 20k-atom sample."""
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w, pos, q = workloads.generate(3)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          cell_type="triclinic"), capacity=w.n)
    r = s.evaluate(pos, q)
    op = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    m = O.Modes(op)
    rh = O.forward_density(op, pos, q)
    assert O.rel_scalar(r.energy, O.energy(m, rh)) <= F64_TOL
    assert O.rel_frobenius(r.pressure, O.pressure(m, rh)) <= F64_TOL
    sel = np.random.default_rng(3).choice(w.n, 20_000, replace=False)
    h3 = op.volume_element
    scale = m.fhat * m.w_inv2 * rh[m.mask]
    Fo = np.empty((sel.size, 3))
    for d in range(3):
        spec = np.zeros(op.M, dtype=complex)
        spec[m.mask] = 1j * m.kvec[d] * scale
        fld = np.fft.ifftn(spec).real / h3
        Fo[:, d] = -q[sel] * h3 * O.gather(op, fld, pos[sel])
    assert O.rms_rel_forces(r.forces[sel], Fo) <= F64_TOL
    assert np.linalg.norm(r.forces.sum(axis=0)) < 1e-10 * np.linalg.norm(r.forces, axis=1).max() * 1e3


@pytest.mark.slow
def test_config4_size_independent_properties():
    """Config 4 (8.1e6 charges, 384^3): momentum conservation, bitwise
    determinism, invariance under a one-grid-spacing translation, charge
    scaling (E, P ~ q^2; F ~ q^2), and fp32 mode within 1e-5."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w, pos, q = workloads.generate(4)
    prm = dict(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M)
    s = KSpaceSolver(w.h, EwaldParameters(**prm), capacity=w.n)
    P_, Q_ = _dev(torch, pos), _dev(torch, q)
    a7, aF = s.evaluate_device(P_, Q_)
    a7, aF = a7.clone(), aF.clone()
    b7, bF = s.evaluate_device(P_, Q_)
    assert torch.equal(a7, b7) and torch.equal(aF, bF)
    F = aF.cpu().numpy()
    assert np.linalg.norm(F.sum(axis=0)) < 1e-9 * np.linalg.norm(F, axis=1).max()
    hx = 300.0 / 384
    shifted = workloads.wrap_positions(w.h, pos + np.array([hx, 0.0, 0.0]))
    c7, cF = s.evaluate_device(_dev(torch, shifted), Q_)
    assert O.rel_scalar(c7[0].item(), a7[0].item()) <= F64_TOL
    assert torch.allclose(c7, a7, rtol=1e-9, atol=1e-12 * a7.abs().max().item())
    assert O.rms_rel_forces(cF.cpu().numpy(), F) <= F64_TOL
    d7, dF = s.evaluate_device(P_, 2.0 * Q_)
    assert torch.allclose(d7, 4.0 * a7, rtol=1e-12, atol=0)
    assert O.rms_rel_forces(dF.cpu().numpy(), 4.0 * F) <= 1e-13
    s32 = KSpaceSolver(w.h, EwaldParameters(precision="fp32", **prm), capacity=w.n)
    e7, eF = s32.evaluate_device(P_, Q_)
    assert O.rel_scalar(e7[0].item(), a7[0].item()) <= F32_TOL
    assert O.rms_rel_forces(eF.cpu().numpy(), F) <= F32_TOL


def test_cuda_slab_plans_reassemble_whole_grid():
    """Emulate R = 3 slab ranks on one GPU (sequentially, no collectives):
    per-slab CUDA spreads + halo adds reassemble the whole-grid spread, and
    per-slab gathers from ghosted field slabs reproduce the whole-grid forces."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    from paper_2601_00161_b200.slab import CudaSlabOps, SlabLayout, anchor_plane
    for idx in (1, 3):
        w, pos, q = workloads.generate(idx)
        if idx == 3:                      # a 200k-charge subset keeps it quick
            pos, q = pos[::5], q[::5]
        s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                              fixed_M=w.M, cell_type=w.cell_type),
                         capacity=len(q))
        P_, Q_ = _dev(torch, pos), _dev(torch, q)
        out7, F = s.evaluate_device(P_, Q_)
        F = F.cpu().numpy()
        fields = s.plan.fields_view().clone()                  # (3, Mz, My, Mx)
        whole = s.plan.spread(P_, Q_).clone()                  # (Mz, My, Mx)
        R = 3
        lay = SlabLayout(w.M[2], w.M[1], R, w.P)
        zp = anchor_plane(pos, w.h, w.M, w.P)
        acc = torch.zeros_like(whole)
        for r in range(R):
            z0, nz = lay.zstart[r], lay.zcount[r]
            mine = (zp >= z0) & (zp < z0 + nz)
            ops = CudaSlabOps(w.M, w.P, s.spec.window, s.kern.basis, w.r_c, w.h, z0, nz,
                              capacity=int(mine.sum()) + 1)
            slab = ops.spread(_dev(torch, pos[mine]), _dev(torch, q[mine]))
            planes = (z0 - lay.nlo + torch.arange(slab.shape[0], device="cuda")) % w.M[2]
            acc.index_add_(0, planes, slab)
            ext = fields.index_select(1, planes).contiguous()
            Fr = ops.gather(ext, None, None).cpu().numpy()
            assert O.rms_rel_forces(Fr, F[mine]) <= 1e-13
        assert torch.allclose(acc, whole, rtol=0, atol=1e-13 * whole.abs().max().item())


def test_slab_solver_single_rank_on_gpu():
    """The full slab orchestration (CUDA slab plan, torch cuFFT stages, host
    mode tables) on one rank equals the single-plan path."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    from paper_2601_00161_b200.slab import SlabKSpaceSolver
    w, pos, q = workloads.generate(1)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M))
    r = s.evaluate(pos, q)
    sl = SlabKSpaceSolver(w.h, w.M, w.P, s.kern.basis, s.spec.window, w.r_c, capacity=w.n)
    E, Pt, F = sl.evaluate(_dev(torch, pos), _dev(torch, q))
    assert O.rel_scalar(E, r.energy) <= 1e-12
    assert O.rel_frobenius(Pt, r.pressure) <= 1e-12
    assert O.rms_rel_forces(F.cpu().numpy(), r.forces) <= 1e-12


@pytest.mark.parametrize("idx", [1, 4])
def test_slab_step_graph_captured_matches_single_plan(idx):
    """The multi-GPU step (SlabKSpaceSolver.evaluate_device: spread, halo
    exchange, fused transforms with the peer-store transposes, device-side
    rank-ordered reduction, gather) captured in one CUDA graph at R = 1 —
    the run bench.py --gpus N makes on every rank — equals the single-plan
    step to 1e-12 (config 1, and config 4 at full size), also after the
    positions are updated in place."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    from paper_2601_00161_b200.plan import out7_to_tensor
    from paper_2601_00161_b200.slab import SlabKSpaceSolver
    w, pos, q = workloads.generate(idx)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M),
                     capacity=w.n)
    sl = SlabKSpaceSolver(w.h, w.M, w.P, s.kern.basis, s.spec.window, w.r_c, capacity=w.n)
    P_, Q_ = _dev(torch, pos), _dev(torch, q)
    g, o7, F = sl.graphed(P_, Q_, True)
    for shift in (0.0, 0.37):
        if shift:
            P_.copy_(_dev(torch, workloads.wrap_positions(w.h, pos + shift)))
        g.replay()
        r7, rF = s.evaluate_device(P_, Q_)
        torch.cuda.synchronize()
        E, Pt = out7_to_tensor(o7)
        Er, Ptr = out7_to_tensor(r7)
        assert O.rel_scalar(E, Er) <= 1e-12
        assert O.rel_frobenius(Pt, Ptr) <= 1e-12
        assert O.rms_rel_forces(F.cpu().numpy(), rF.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("name", ["small_cube_p5", "small_brick_p6", "small_brick_p8",
                                  "small_brick_p7", "small_cube_p4"])
def test_analytic_forces_and_local_pressure_match_reference(name):
    """f1 / f2 of SURVEY §8(f): analytic-differentiation forces
    (mesh.py:343-349) and per-particle pressure tensors (mesh.py:353-379)."""
    torch = _torch()
    g = golden(name)
    plan = _plan_for(g)
    pos, q = _dev(torch, g["pos"]), _dev(torch, g["q"])
    plan.evaluate(pos, q, want_forces=True, analytic=True)
    Fa = plan.forces_analytic(pos.shape[0]).cpu().numpy()
    assert O.rms_rel_forces(Fa, g["F_analytic"]) <= F64_TOL
    plan.reset_counters()
    plan.evaluate(pos, q, want_forces=False)
    lp = plan.local_pressure(pos.shape[0]).cpu().numpy()
    assert plan.counters() == (1, 6)
    ref = g["local"]
    assert np.max(np.abs(lp - ref)) <= F64_TOL * np.max(np.abs(ref))
    np.testing.assert_array_equal(lp, np.swapaxes(lp, 1, 2))
    # sum of local tensors ~ global pressure (test_mesh.py:279-287)
    assert np.linalg.norm(lp.sum(0) - g["Pt"]) <= 1e-8 * np.linalg.norm(g["Pt"])


def test_analytic_forces_through_mesh_api_and_triclinic():
    torch = _torch()
    from paper_2601_00161_b200 import (Cell, ParticleSystem, SplitKernel, TransformProvider,
                                       build_pswf, forward_density, long_range_forces,
                                       local_pressure, plan_grid, solve_bandwidth)
    g = golden("small_brick_p8")
    b = build_pswf(solve_bandwidth(float(g["delta"])))
    kern = SplitKernel(basis=b, r_c=float(g["r_c"]))
    cell = Cell(g["h"])
    spec = plan_grid(cell, kern, delta_spread=float(g["delta"]), P=int(g["P"]),
                     spread_basis=b, fixed_M=tuple(g["M"]))
    sys = ParticleSystem(cell=cell, positions=g["pos"], charges=g["q"])
    prov = TransformProvider()
    rho_hat = forward_density(sys, spec, prov)
    Fa = long_range_forces(rho_hat, sys, kern, spec, cell, mode="analytic", provider=prov)
    assert prov.inverse_count == 1
    assert O.rms_rel_forces(Fa, g["F_analytic"]) <= F64_TOL
    lp = local_pressure(rho_hat, sys, kern, spec, cell, provider=prov)
    assert prov.inverse_count == 7
    assert np.max(np.abs(lp - g["local"])) <= F64_TOL * np.max(np.abs(g["local"]))
    # triclinic: analytic and ik forces agree at the Delta level
    gt = golden("tri_skew_p8")
    plan = _plan_for(gt, M=(64, 64, 80))
    pos, q = _dev(torch, gt["pos"]), _dev(torch, gt["q"])
    _, Fik = plan.evaluate(pos, q, want_forces=True)
    Fik = Fik.cpu().numpy()
    _, Fan = plan.evaluate(pos, q, want_forces=True, analytic=True)
    assert O.rms_rel_forces(Fan.cpu().numpy(), Fik) <= 50 * float(gt["delta"])
    assert O.rms_rel_forces(Fan.cpu().numpy(), gt["F_direct"]) <= 50 * float(gt["delta"])


# --- band-pruned fused transforms (esp_fft.cu) ---------------------------------
# Grids whose lengths are all in {32,48,64,96,128,192,256,384} run esp_evaluate
# through the fused transform pipeline; others (and ESP_FFT=cufft) use cuFFT.
FUSED_CASES = [
    ("tri_skew_p8", (64, 64, 96)),     # triclinic, P=8
    ("tri_flex_p7", (48, 48, 64)),     # triclinic, odd P
    ("small_brick_p6", (48, 64, 64)),  # orthorhombic (x != y: k_x_c2r + TMA gather)
    ("small_brick_p7", (64, 64, 96)),  # orthorhombic, odd P
    ("small_cube_p5", (48, 48, 48)),   # odd P, cubic
    # grids whose inverse x pass is k_x_c2r (x != y or x > 64): the ghost-padded
    # fields and the TMA gathers (fp64 and fp32), every P and odd/even anchoring
    ("small_cube_p4", (48, 64, 48)),
    ("small_cube_p5", (64, 48, 96)),
    ("small_brick_p7", (96, 64, 96)),
    ("small_brick_p8", (32, 48, 32)),
    ("tri_flex_p7", (64, 48, 64)),     # triclinic, odd P
    ("small_single", (48, 64, 48)),    # one charge
    # long rows: the forward x pass stages the spread's scratch rows with
    # cp.async.bulk (k_x_bulk_r2c, Mx = 256 / 384), odd and even P
    ("small_brick_p8", (256, 48, 32)),
    ("small_brick_p7", (384, 32, 48)),
    ("tri_flex_p7", (256, 32, 32)),
    ("small_brick_p6", (192, 48, 32)),   # 64-thread CTAs
]


@pytest.mark.parametrize("name,M", FUSED_CASES)
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fused_fft_path_matches_oracle(name, M, precision):
    g = golden(name)
    plan = _plan_for(g, M=M, precision=precision)
    assert plan.fft_path == "fused"
    E, Pt, F = _run(plan, g["pos"], g["q"])
    op = O.make_plan(g["h"], M, int(g["P"]), float(g["delta"]), float(g["r_c"]))
    oE, oP, oF = O.kspace(op, g["pos"], g["q"])
    tol = F64_TOL if precision == "fp64" else F32_TOL
    assert O.rel_scalar(E, oE) <= tol
    assert O.rel_frobenius(Pt, oP) <= tol
    if np.sqrt(np.mean(np.sum(oF ** 2, axis=1))) > 1e-12:
        assert O.rms_rel_forces(F, oF) <= tol
    else:   # a lone charge feels no self force: both are round-off zero
        assert np.max(np.abs(F)) <= (1e-12 if precision == "fp64" else 1e-6)
    # pressure-only step: one forward transform, no inverse, same E and P
    plan.reset_counters()
    E2, P2, _ = _run(plan, g["pos"], g["q"], want_forces=False)
    assert plan.counters() == (1, 0)
    assert O.rel_scalar(E2, oE) <= tol and O.rel_frobenius(P2, oP) <= tol


def test_fused_and_cufft_paths_agree(monkeypatch):
    g = golden("tri_skew_p8")
    M = (64, 64, 96)
    fused = _plan_for(g, M=M)
    monkeypatch.setenv("ESP_FFT", "cufft")
    ref = _plan_for(g, M=M)
    assert fused.fft_path == "fused" and ref.fft_path == "cufft"
    Ea, Pa, Fa = _run(fused, g["pos"], g["q"])
    Eb, Pb, Fb = _run(ref, g["pos"], g["q"])
    assert O.rel_scalar(Ea, Eb) <= 1e-13
    assert O.rel_frobenius(Pa, Pb) <= 1e-13
    assert O.rms_rel_forces(Fa, Fb) <= 1e-13
    # the in-band spectrum box the fused forward pass leaves in the plan
    # feeds the stage-level API (scale/reduce on the same spectrum)
    torch = _torch()
    out7 = torch.empty(7, dtype=torch.float64, device="cuda")
    fused.scale_reduce(False, out7)
    from paper_2601_00161_b200.plan import out7_to_tensor
    E3, P3 = out7_to_tensor(out7)
    assert O.rel_scalar(E3, Ea) <= 1e-14 and O.rel_frobenius(P3, Pa) <= 1e-14


@pytest.mark.parametrize("name,M", [("small_brick_p8", (32, 48, 32)), ("small_brick_p7", (96, 64, 96)),
                                    ("small_cube_p4", (48, 64, 48)), ("tri_flex_p7", (64, 48, 64)),
                                    ("small_brick_p6", (128, 96, 64)),
                                    ("small_brick_p8", (256, 48, 32)), ("small_cube_p5", (384, 32, 48)),
                                    ("tri_flex_p7", (192, 32, 48))])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_x_pass_combine_bitwise_equals_separate_combine(name, M, precision, monkeypatch):
    """esp_evaluate sums the spread's tile blocks inside the forward x pass
    (k_x_comb_r2c); ESP_NO_XCOMBINE keeps k_combine + k_x_r2c.  Same sums in
    the same order: bitwise-identical energy, pressure and forces, also where
    the periodic wrap puts more than two tiles on a coordinate."""
    g = golden(name)
    plan = _plan_for(g, M=M, precision=precision)
    assert plan.fft_path == "fused"
    Ea, Pa, Fa = _run(plan, g["pos"], g["q"])
    la = plan.launches_last_step()
    monkeypatch.setenv("ESP_NO_XCOMBINE", "1")
    Eb, Pb, Fb = _run(plan, g["pos"], g["q"])
    assert plan.launches_last_step() == la + 1
    assert Ea == Eb and np.array_equal(Pa, Pb) and np.array_equal(Fa, Fb)


def test_unsupported_lengths_fall_back_to_cufft():
    g = golden("tri_skew_p8")                  # M = (64, 64, 80): 80 not a fused length
    plan = _plan_for(g)
    assert plan.fft_path == "cufft"
    E, Pt, F = _run(plan, g["pos"], g["q"])
    op = O.make_plan(g["h"], tuple(g["M"]), int(g["P"]), float(g["delta"]), float(g["r_c"]))
    oE, oP, oF = O.kspace(op, g["pos"], g["q"])
    assert O.rel_scalar(E, oE) <= F64_TOL
    assert O.rms_rel_forces(F, oF) <= F64_TOL


def test_non_finite_and_huge_positions_do_not_fault():
    """Garbage coordinates (NaN, inf, 1e300, random bit patterns) must not
    fault the device path: every pass clamps the anchor base the same way,
    so packed tile-local anchors stay inside their tile.  Finite charges
    elsewhere keep finite outputs."""
    torch = _torch()
    g = golden("small_cube_p6")
    plan = _plan_for(g, capacity=256)
    pos = np.ascontiguousarray(g["pos"], dtype=np.float64)
    for val in (np.nan, np.inf, -np.inf, 1e300, -1e300, 3e15, 1e-310):
        p2 = pos.copy()
        p2[::5, 0] = val
        p2[::7, 2] = val
        E, Pt, F = _run(plan, p2, g["q"])
        torch.cuda.synchronize()
        if not np.isnan(val):
            assert np.isfinite(E)
    bits = np.random.default_rng(3).integers(0, 2 ** 63, size=pos.shape, dtype=np.int64)
    _run(plan, bits.view(np.float64), g["q"])
    torch.cuda.synchronize()
    # the plan is still healthy afterwards
    E, Pt, F = _run(plan, g["pos"], g["q"])
    assert O.rel_scalar(E, g["E"]) <= F64_TOL


def test_fused_path_empty_system_and_cell_rebind():
    """Fused / plane transform path (48^3): an empty system gives zeros, and
    NPT-style rebinds (same band: buffers kept; new band: rebuilt) match the
    oracle for each new cell."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    g = golden("small_cube_p6")
    M = tuple(int(m) for m in g["M"])
    s = KSpaceSolver(g["h"], EwaldParameters(r_c=float(g["r_c"]), delta_split=float(g["delta"]),
                                             P=int(g["P"]), fixed_M=M), capacity=256)
    assert s.plan.fft_path == "fused"
    empty = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    out7, _ = s.plan.evaluate(empty, torch.zeros(0, dtype=torch.float64, device="cuda"),
                              want_forces=True)
    assert torch.count_nonzero(out7).item() == 0
    for scale in (1.0, 1.002, 0.97, 1.05):
        h = np.asarray(g["h"]) * scale
        s.rebind_cell(h)
        pos = np.asarray(g["pos"]) * scale
        r = s.evaluate(pos, g["q"])
        op = O.make_plan(h, M, int(g["P"]), float(g["delta"]), float(g["r_c"]))
        oE, oP, oF = O.kspace(op, pos, g["q"])
        assert O.rel_scalar(r.energy, oE) <= F64_TOL
        assert O.rel_frobenius(r.pressure, oP) <= F64_TOL
        assert O.rms_rel_forces(r.forces, oF) <= F64_TOL


@pytest.mark.parametrize("R,precision", [(1, "fp64"), (2, "fp64"), (3, "fp64"), (3, "fp32")])
def test_fused_slab_transforms_emulated_on_one_gpu(R, precision):
    """Distributed z-slab transforms (esp_slab_*): R ranks run one after
    another on one device, each storing its transpose output straight into
    the other ranks' receive buffers (what NVLink peer stores do on a box).
    The ranks' energy/pressure shares add up to the single-plan result and
    each rank's field slab equals the single-plan fields on its planes."""
    torch = _torch()
    g = golden("tri_skew_p8")
    M = (64, 64, 96)
    plan = _plan_for(g, M=M, precision=precision)
    assert plan.fft_path == "fused"
    tol = 1e-12 if precision == "fp64" else 2e-6
    pos, q = _dev(torch, g["pos"]), _dev(torch, g["q"])
    out7, _ = plan.evaluate(pos, q, True)
    ref7 = out7.cpu().numpy().copy()
    ref_fields = plan.fields_view().clone()
    grid = plan.spread(pos, q).clone()                   # (Mz, My, Mx)
    zc = [M[2] // R + (r < M[2] % R) for r in range(R)]
    z_start = [0] + list(np.cumsum(zc))
    bufs = [plan.slab_buffers(R, r, z_start) for r in range(R)]
    fwd = [b[0] for b in bufs]
    back = [b[1] for b in bufs]
    descs = [plan.slab_desc(R, r, z_start, fwd, back) for r in range(R)]
    for r in range(R):
        plan.slab_forward(descs[r], grid[z_start[r]:z_start[r + 1]])
    torch.cuda.synchronize()
    parts = [plan.slab_reduce(descs[r], fwd[r], True).cpu().numpy().copy() for r in range(R)]
    torch.cuda.synchronize()
    tot = parts[0]
    for r in range(1, R):
        tot = tot + parts[r]
    assert abs(tot[0] - ref7[0]) <= tol * abs(ref7[0])
    assert np.linalg.norm(tot[1:] - ref7[1:]) <= tol * np.linalg.norm(ref7[1:])
    for r in range(R):
        nz = z_start[r + 1] - z_start[r]
        f = torch.empty((3, nz, M[1], M[0]), dtype=plan.real_dtype, device="cuda")
        plan.slab_inverse(descs[r], back[r], f)
        refp = ref_fields[:, z_start[r]:z_start[r + 1]]
        err = (f - refp).abs().max().item()
        assert err <= tol * refp.abs().max().item()


def test_fused_analytic_forces_config1_against_oracle():
    """Analytic-differentiation forces on the band-pruned fused transforms
    (one potential spectrum, one inverse transform, window-gradient gather)
    at config 1, against the oracle's analytic forces (mesh.py:343-349)."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w, pos, q = workloads.generate(1)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          force_mode="analytic"), capacity=w.n)
    assert s.plan.fft_path == "fused"
    s.plan.reset_counters()
    r = s.evaluate(pos, q)
    assert s.plan.counters() == (1, 1)
    plan = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    modes = O.Modes(plan)
    rh = O.forward_density(plan, pos, q)
    Fa = O.forces_analytic(plan, modes, rh, pos, q)
    assert O.rel_scalar(r.energy, O.energy(modes, rh)) <= F64_TOL
    assert O.rel_frobenius(r.pressure, O.pressure(modes, rh)) <= F64_TOL
    assert O.rms_rel_forces(r.forces, Fa) <= F64_TOL
    # the CUDA-graph and host-buffer paths run the same analytic step
    P_ = torch.as_tensor(pos, device="cuda")
    Q_ = torch.as_tensor(q, device="cuda")
    g, o7, oF = s.graphed(P_, Q_)
    g.replay()
    torch.cuda.synchronize()
    assert O.rms_rel_forces(oF.cpu().numpy(), Fa) <= F64_TOL
    hs = s.host_stepper(w.n)
    hs.positions.copy_(torch.as_tensor(pos))
    hs.charges.copy_(torch.as_tensor(q))
    _, hF = hs.step()
    assert torch.equal(hF, oF.cpu())


def test_spread_row_layouts_bitwise_identical():
    """Every rows-per-thread layout of the tile spread (ESP_SPREAD_ROWS, read
    once per process) owns each grid column with one thread that adds the
    charges in the same order, so the step's results are bitwise equal."""
    import os
    import subprocess
    import sys
    _torch()
    code = (
        "import sys, hashlib, numpy as np, torch\n"
        "sys.path.insert(0, '.')\n"
        "from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver, workloads\n"
        "w, pos, q = workloads.generate(1)\n"
        "s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,"
        " fixed_M=w.M, cell_type=w.cell_type), capacity=w.n)\n"
        "r = s.evaluate(pos, q)\n"
        "h = hashlib.sha1(np.float64(r.energy).tobytes() + np.asarray(r.pressure).tobytes()"
        " + np.asarray(r.forces).tobytes()).hexdigest()\n"
        "print('HASH', h)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hashes = {}
    for rows in ("1", "2", "4", "8"):
        env = dict(os.environ, ESP_SPREAD_ROWS=rows)
        out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env,
                             capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        hashes[rows] = [ln for ln in out.stdout.splitlines() if ln.startswith("HASH")][0]
    assert len(set(hashes.values())) == 1, hashes


@pytest.mark.parametrize("cfg,radix", [(1, False), (2, False), (1, True), (2, True)])
@pytest.mark.parametrize("chunks", [1, 2, 3, 8])
def test_host_stepper_chunked_force_copy_bitwise(cfg, radix, chunks, monkeypatch):
    """The host-buffer step copies its forces out in original-index ranges
    as the gather finishes each one (esp_set_host_forces); every range count
    gives the device step's forces bit for bit.  ``radix``: the large-N
    binning path, where the step bins the late charges after the records
    pass (k_bin_charges) so their copy hides behind the binning."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    monkeypatch.setenv("ESP_HOST_CHUNKS", str(chunks))
    if radix:
        monkeypatch.setenv("ESP_SORT_THRESHOLD", "0")
    w, pos, q = workloads.generate(cfg)
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          cell_type=w.cell_type), capacity=w.n)
    e7, eF = s.evaluate_device(torch.as_tensor(pos, device="cuda"),
                               torch.as_tensor(q, device="cuda"))
    e7, eF = e7.cpu(), eF.cpu()
    hs = s.host_stepper(w.n)
    hs.positions.copy_(torch.as_tensor(pos))
    hs.charges.copy_(torch.as_tensor(q))
    for _ in range(2):
        hs.forces.fill_(float("nan"))
        h7, hF = hs.step()
        assert torch.equal(h7, e7) and torch.equal(hF, eF)
    # eager steps after the capture do not write the host buffer
    hs.forces.zero_()
    s.evaluate_device(torch.as_tensor(pos, device="cuda"), torch.as_tensor(q, device="cuda"))
    torch.cuda.synchronize()
    assert not hs.forces.any()
