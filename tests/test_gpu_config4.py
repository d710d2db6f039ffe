"""Config 4 at full size against the reference, and the radix-sort binning
path on orthorhombic cells.

``tests/golden/cfg4.npz`` was produced by running the reference package
itself on the full 8,100,000-charge system (``make_golden_cfg4.py``: chunked
reference ``spread_charges``, reference ``forward_density`` arithmetic,
``long_range_energy`` / ``long_range_pressure`` on the whole spectrum and
``long_range_forces(mode="ik")`` on a seeded 20,000-charge sample).  The
CUDA path runs the whole system (the radix-sort binning, 32-plane tile
spread, 384^3 band-pruned transforms and the tile gather) and is compared
at the north-star tolerances: fp64 1e-10, fp32 1e-5 (energy relative,
pressure Frobenius relative, forces rms relative over the sampled atoms).

Radix path: plans with at least ``sort_threshold`` charges (5e5 by default,
esp_internal.cuh) bin with a device radix sort instead of the counting sort
(esp_bin.cu).  ``ESP_SORT_THRESHOLD`` (read at plan creation) forces it on
small systems, so the same cases run through both binnings: bitwise equal
results, and parity with the reference goldens for ik and analytic forces.
"""

import numpy as np
import pytest

from conftest import SMALL_CASES, golden
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


@pytest.fixture(scope="module")
def cfg4():
    torch = _torch()
    w, pos, q = workloads.generate(4)
    g = golden("cfg4")
    assert np.array_equal(pos[:4], g["pos_head"]) and np.allclose(pos.sum(axis=0), g["pos_sum"],
                                                                  rtol=1e-15, atol=0)
    P_ = torch.as_tensor(pos, device="cuda")
    Q_ = torch.as_tensor(q, device="cuda")
    yield w, P_, Q_, g
    del P_, Q_
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("precision,tol", [("fp64", F64_TOL), ("fp32", F32_TOL)])
def test_config4_full_size_against_reference(cfg4, precision, tol):
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    torch = _torch()
    w, P_, Q_, g = cfg4
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          precision=precision, cell_type=w.cell_type),
                     capacity=w.n)
    assert s.plan.radix_binning(w.n), "config 4 must take the radix-sort binning path"
    out7, F = s.evaluate_device(P_, Q_)
    torch.cuda.synchronize()
    from paper_2601_00161_b200.plan import out7_to_tensor
    E, Pt = out7_to_tensor(out7)
    idx = torch.as_tensor(g["F_idx"], device="cuda")
    Fs = F.index_select(0, idx).cpu().numpy()
    assert O.rel_scalar(E, float(g["E"])) <= tol
    assert O.rel_frobenius(Pt, g["Pt"]) <= tol
    assert O.rms_rel_forces(Fs, g["F_sel"]) <= tol
    # momentum over all 8.1M charges (ik forces conserve it, test_mesh.py:218-222);
    # fp32 fields: the residual is a random walk of fp32 roundings, so it is
    # bounded against sqrt(N) x rms|F|
    Fn = F.cpu().numpy()
    net = np.linalg.norm(Fn.sum(axis=0))
    if precision == "fp64":
        assert net < 1e-9 * np.linalg.norm(Fn, axis=1).max()
    else:
        assert net < 1e-5 * np.sqrt(w.n) * np.sqrt(np.mean(np.sum(Fn * Fn, axis=1)))
    del s, F


@pytest.mark.slow
def test_config4_host_buffer_step_equals_device_step(cfg4):
    """The host-buffer step at full size (positions copied first, charges
    behind them on the side stream and binned after the records pass, forces
    copied out in two index ranges) gives the device step's numbers bit for
    bit, also after the host buffers change."""
    torch = _torch()
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    w, P_, Q_, g = cfg4
    s = KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P, fixed_M=w.M,
                                          cell_type=w.cell_type), capacity=w.n)
    e7, eF = s.evaluate_device(P_, Q_)
    e7, eF = e7.cpu(), eF.cpu()
    hs = s.host_stepper(w.n)
    hs.positions.copy_(P_.cpu())
    hs.charges.copy_(Q_.cpu())
    h7, hF = hs.step()
    assert torch.equal(h7, e7) and torch.equal(hF, eF)
    # new charges and shifted positions through the host buffers
    q2 = Q_.cpu() * torch.linspace(0.5, 1.5, w.n, dtype=torch.float64)
    p2 = P_.cpu() + 0.37
    hs.charges.copy_(q2)
    hs.positions.copy_(p2)
    hs.forces.fill_(float("nan"))
    h7, hF = hs.step()
    r7, rF = s.evaluate_device(p2.cuda(), q2.cuda())
    torch.cuda.synchronize()
    assert torch.equal(h7, r7.cpu()) and torch.equal(hF, rF.cpu())
    del s, hs


def _solver(w, force_mode="ik", precision="fp64"):
    from paper_2601_00161_b200 import EwaldParameters, KSpaceSolver
    return KSpaceSolver(w.h, EwaldParameters(r_c=w.r_c, delta_split=w.delta, P=w.P,
                                             fixed_M=w.M, precision=precision,
                                             cell_type=w.cell_type, force_mode=force_mode),
                        capacity=w.n)


def _bits(r):
    return (np.float64(r.energy).tobytes(), np.asarray(r.pressure).tobytes(),
            np.asarray(r.forces).tobytes())


@pytest.mark.parametrize("idx", [0, 1, 2])
@pytest.mark.parametrize("force_mode", ["ik", "analytic"])
def test_radix_binning_orthorhombic_matches_counting_sort(monkeypatch, idx, force_mode):
    """Configs 0-2 (orthorhombic; the fused transform path) binned by the
    radix sort: bitwise equal to the counting-sort binning, and ik forces
    within 1e-10 of the reference goldens."""
    _torch()
    w, pos, q = workloads.generate(idx)
    monkeypatch.delenv("ESP_SORT_THRESHOLD", raising=False)
    s_count = _solver(w, force_mode)
    assert not s_count.plan.radix_binning(w.n)
    monkeypatch.setenv("ESP_SORT_THRESHOLD", "0")
    s_radix = _solver(w, force_mode)
    assert s_radix.plan.radix_binning(w.n)
    a = s_count.evaluate(pos, q)
    b = s_radix.evaluate(pos, q)
    assert _bits(a) == _bits(b)
    if force_mode == "ik":
        g = golden(f"cfg{idx}")
        assert O.rel_scalar(b.energy, g["E"]) <= F64_TOL
        assert O.rel_frobenius(b.pressure, g["Pt"]) <= F64_TOL
        assert O.rms_rel_forces(b.forces[g["F_idx"]], g["F_sel"]) <= F64_TOL


@pytest.mark.parametrize("name", SMALL_CASES)
def test_radix_binning_small_cases_against_reference(monkeypatch, name):
    """Every small golden (odd and even P, N = 1, cubes and bricks) through
    the radix binning: E, P and ik / analytic forces and the local pressure
    against the reference at 1e-10."""
    torch = _torch()
    from paper_2601_00161_b200 import EspPlan, build_pswf, solve_bandwidth, tabulate_window
    g = golden(name)
    monkeypatch.setenv("ESP_SORT_THRESHOLD", "0")
    b = build_pswf(solve_bandwidth(float(g["delta"])))
    plan = EspPlan(tuple(g["M"]), int(g["P"]), tabulate_window(b, int(g["P"])), b,
                   float(g["r_c"]), capacity=1 << 12)
    plan.set_cell(g["h"])
    assert plan.radix_binning(len(g["q"]))
    from paper_2601_00161_b200.plan import out7_to_tensor
    P_ = torch.as_tensor(g["pos"], device="cuda")
    Q_ = torch.as_tensor(g["q"], device="cuda")
    out7, F = plan.evaluate(P_, Q_, True)
    E, Pt = out7_to_tensor(out7)
    assert O.rel_scalar(E, g["E"]) <= F64_TOL
    assert O.rel_frobenius(Pt, g["Pt"]) <= F64_TOL
    ref = g["F"]
    Fn = F.cpu().numpy()
    if np.sqrt(np.mean(np.sum(ref ** 2, axis=1))) > 1e-12:
        assert O.rms_rel_forces(Fn, ref) <= F64_TOL
        Fa = plan.forces_analytic(len(g["q"])).cpu().numpy()
        assert O.rms_rel_forces(Fa, g["F_analytic"]) <= F64_TOL
    else:
        assert np.max(np.abs(Fn)) <= 1e-12
