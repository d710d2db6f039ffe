"""Pin the CPU oracle (oracle/esp_oracle.py) to the reference.

Golden vectors were produced by running the reference package itself
(tests/golden/make_golden.py).  The oracle is a restatement, so on the same
numpy/scipy it reproduces the reference bit-for-bit; the tolerances below
(1e-13) only leave room for a different BLAS/pocketfft build.
"""

import numpy as np
import pytest

from conftest import SMALL_CASES, TRI_CASES, golden
from oracle import esp_oracle as O
from paper_2601_00161_b200 import workloads

TIGHT = 1e-13


def plan_from(g, M=None):
    return O.make_plan(g["h"], tuple(M if M is not None else g["M"]), int(g["P"]),
                       float(g["delta"]), float(g["r_c"]))


@pytest.mark.parametrize("name", SMALL_CASES)
def test_small_cases_match_reference(name):
    g = golden(name)
    plan = plan_from(g)
    assert plan.split.c == pytest.approx(float(g["c"]), rel=1e-15)
    assert plan.split.lambda0 == pytest.approx(float(g["lambda0"]), rel=1e-14)
    np.testing.assert_allclose(plan.window.value.c, g["window_c"], rtol=0, atol=1e-15)
    modes = O.Modes(plan)
    assert int(modes.mask.sum()) == int(g["n_modes"])
    grid = O.spread(plan, g["pos"], g["q"])
    assert np.max(np.abs(grid - g["grid"])) <= TIGHT * np.max(np.abs(g["grid"]))
    rh = np.fft.fftn(grid) * plan.volume_element
    assert O.rel_scalar(O.energy(modes, rh), g["E"]) <= TIGHT
    assert O.rel_frobenius(O.pressure(modes, rh), g["Pt"]) <= TIGHT
    if np.any(g["F"]):
        assert O.rms_rel_forces(O.forces_ik(plan, modes, rh, g["pos"], g["q"]), g["F"]) <= TIGHT
        assert O.rms_rel_forces(O.forces_analytic(plan, modes, rh, g["pos"], g["q"]),
                                g["F_analytic"]) <= TIGHT
    lp = O.local_pressure(plan, modes, rh, g["pos"], g["q"])
    assert np.max(np.abs(lp - g["local"])) <= TIGHT * max(np.max(np.abs(g["local"])), 1e-300)


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_configs_match_reference(idx):
    g = golden(f"cfg{idx}")
    w, pos, q = workloads.generate(idx)
    np.testing.assert_array_equal(pos[:4], g["pos_head"])
    plan = O.make_plan(w.h, w.M, w.P, w.delta, w.r_c)
    E, Pt, F = O.kspace(plan, pos, q)
    assert O.rel_scalar(E, g["E"]) <= TIGHT
    assert O.rel_frobenius(Pt, g["Pt"]) <= TIGHT
    assert O.rms_rel_forces(F[g["F_idx"]], g["F_sel"]) <= TIGHT
    if idx == 0:
        grid = O.spread(plan, pos, q)
        assert np.max(np.abs(grid - g["grid"])) <= TIGHT * np.max(np.abs(g["grid"]))


def test_survey_spot_values():
    """SURVEY §8(c) known-answer values (config 0 / 1 generator + outputs)."""
    _, p0, _ = workloads.generate(0)
    assert tuple(p0[1]) == (19.420929525854891, 9.2614251285024594, 1.5718887732850522)
    _, p1, _ = workloads.generate(1)
    assert tuple(p1[1]) == (35.223538188692849, 63.444389048414656, 9.4545296571932145)
    g0, g1 = golden("cfg0"), golden("cfg1")
    assert float(g0["E"]) == pytest.approx(1.7409503392262431, rel=1e-14)
    assert float(g1["E"]) == pytest.approx(82.563381130618652, rel=1e-14)
    assert float(g1["F_rms"]) == pytest.approx(0.030202267446825103, rel=1e-12)


@pytest.mark.parametrize("name,M", TRI_CASES)
def test_triclinic_extension_matches_exact_mode_sum(name, M):
    """The triclinic lattice (no reference mesh path) agrees with the
    reference's exact gridless mode sum at the Delta level."""
    g = golden(name)
    plan = plan_from(g, M)
    assert not plan.orthorhombic
    E, Pt, F = O.kspace(plan, g["pos"], g["q"])
    tol = 50 * float(g["delta"])
    assert O.rel_scalar(E, g["E_direct"]) <= tol
    assert O.rel_frobenius(Pt, g["Pt_direct"]) <= tol
    assert O.rms_rel_forces(F, g["F_direct"]) <= tol
    # the oracle's own exact sum restates the reference's direct_ksum exactly
    Ed, Fd, Pd = O.direct_ksum(g["h"], plan.kmax, plan.split, plan.r_c, g["pos"], g["q"])
    assert O.rel_scalar(Ed, g["E_direct"]) <= 1e-12
    assert O.rel_frobenius(Pd, g["Pt_direct"]) <= 1e-12


def test_triclinic_code_path_reduces_to_orthorhombic():
    import dataclasses

    g = golden("small_brick_p8")
    plan = plan_from(g)

    class Tri(O.Plan):
        @property
        def orthorhombic(self):
            return False

    tri = Tri(**{f.name: getattr(plan, f.name) for f in dataclasses.fields(plan)})
    E, Pt, F = O.kspace(tri, g["pos"], g["q"])
    assert O.rel_scalar(E, g["E"]) <= 1e-13
    assert O.rel_frobenius(Pt, g["Pt"]) <= 1e-13
    assert O.rms_rel_forces(F, g["F"]) <= 1e-13


def test_mesh_matches_direct_sum_at_delta():
    """Reference acceptance criterion (test_acceptance.py:153-159) on the goldens."""
    for name in ("small_brick_p8", "small_brick_p7", "small_cube_p6"):
        g = golden(name)
        tol = 50 * float(g["delta"])
        assert O.rel_scalar(g["E"], g["E_direct"]) <= tol
        assert O.rel_frobenius(g["Pt"], g["Pt_direct"]) <= tol
