"""Multi-rank slab decomposition on CPU (gloo, world_size 2 and 3).

Each rank owns a z-slab and the charges anchored in it; the orchestration of
paper_2601_00161_b200.slab (halo add over send/recv, all-to-all transposes,
rank-ordered reduction, field ghost exchange) runs unchanged, with the CPU
oracle's stencil arithmetic as the per-rank spread/gather (test-only).  The
result must equal the single-process oracle to round-off.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import esp_oracle as O
from paper_2601_00161_b200 import build_pswf, solve_bandwidth, tabulate_window, workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "ortho": dict(h=np.diag([12.0, 13.0, 14.0]), M=(24, 24, 36), P=6, delta=1e-5, r_c=3.0, n=300),
    "tri": dict(h=np.array([[12.0, 1.5, 0.5], [0.0, 12.5, 1.0], [0.0, 0.0, 14.0]]),
                M=(28, 28, 36), P=7, delta=1e-6, r_c=3.0, n=240),
}


def _system(c):
    rng = np.random.default_rng(7)
    pos = workloads.wrap_positions(c["h"], rng.uniform(0, 1, (c["n"], 3)) @ c["h"].T)
    q = np.where(np.arange(c["n"]) % 2 == 0, 1.0, -1.0)
    return pos, q


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from slab_oracle_ops import OracleSlabOps
        from paper_2601_00161_b200.slab import SlabKSpaceSolver

        c = CASES[case]
        pos, q = _system(c)
        basis = build_pswf(solve_bandwidth(c["delta"]))
        window = tabulate_window(basis, c["P"])
        oplan = O.make_plan(c["h"], c["M"], c["P"], c["delta"], c["r_c"])
        # layout first, to know this rank's slab
        from paper_2601_00161_b200.slab import SlabLayout
        lay = SlabLayout(c["M"][2], c["M"][1], world, c["P"])
        ops = OracleSlabOps(oplan, lay.zstart[rank], lay.zcount[rank])
        s = SlabKSpaceSolver(c["h"], c["M"], c["P"], basis, window, c["r_c"], ops=ops,
                             device=torch.device("cpu"))
        mine = s.owned(pos)
        E, Pt, F = s.evaluate(torch.as_tensor(pos[mine]), torch.as_tensor(q[mine]))
        Fg = np.zeros((len(q), 3))
        Fg[mine] = F.numpy()
        t = torch.as_tensor(Fg)
        dist.all_reduce(t)
        if rank == 0:
            out.put((E, Pt, t.numpy(), int(mine.sum())))
        else:
            out.put((None, None, None, int(mine.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("ortho", 2), ("ortho", 3), ("tri", 2)])
def test_slab_decomposition_matches_single_process(case, world):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = [out.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    E, Pt, F = next((r[0], r[1], r[2]) for r in res if r[0] is not None)
    assert sum(r[3] for r in res) == CASES[case]["n"]      # every charge owned once
    c = CASES[case]
    pos, q = _system(c)
    oplan = O.make_plan(c["h"], c["M"], c["P"], c["delta"], c["r_c"])
    oE, oP, oF = O.kspace(oplan, pos, q)
    assert O.rel_scalar(E, oE) <= 1e-12
    assert O.rel_frobenius(Pt, oP) <= 1e-12
    assert O.rms_rel_forces(F, oF) <= 1e-12


def test_single_rank_slab_equals_whole_grid():
    """R = 1: the ghost planes wrap onto the rank itself (periodic)."""
    from slab_oracle_ops import OracleSlabOps
    from paper_2601_00161_b200.slab import SlabKSpaceSolver
    c = CASES["ortho"]
    pos, q = _system(c)
    basis = build_pswf(solve_bandwidth(c["delta"]))
    oplan = O.make_plan(c["h"], c["M"], c["P"], c["delta"], c["r_c"])
    s = SlabKSpaceSolver(c["h"], c["M"], c["P"], basis, tabulate_window(basis, c["P"]),
                         c["r_c"], ops=OracleSlabOps(oplan, 0, c["M"][2]),
                         device=torch.device("cpu"))
    E, Pt, F = s.evaluate(torch.as_tensor(pos), torch.as_tensor(q))
    oE, oP, oF = O.kspace(oplan, pos, q)
    assert O.rel_scalar(E, oE) <= 1e-12
    assert O.rel_frobenius(Pt, oP) <= 1e-12
    assert O.rms_rel_forces(F.numpy(), oF) <= 1e-12


def _coulomb_worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from slab_oracle_ops import OracleNearOps, OracleSlabOps
        from paper_2601_00161_b200 import EwaldParameters
        from paper_2601_00161_b200.slab import SlabKSpaceSolver, SlabLayout
        from paper_2601_00161_b200.slab_near import SlabCoulombSolver
        c = CASES[case]
        pos, q = _system(c)
        basis = build_pswf(solve_bandwidth(c["delta"]))
        oplan = O.make_plan(c["h"], c["M"], c["P"], c["delta"], c["r_c"])
        lay = SlabLayout(c["M"][2], c["M"][1], world, c["P"])
        ks = SlabKSpaceSolver(c["h"], c["M"], c["P"], basis, tabulate_window(basis, c["P"]),
                              c["r_c"], ops=OracleSlabOps(oplan, lay.zstart[rank],
                                                          lay.zcount[rank]),
                              device=torch.device("cpu"))
        ob = O.build_basis(O.solve_bandwidth(c["delta"]))
        near_ops = OracleNearOps(c["h"], ob, c["r_c"], O.pair_table(ob, c["r_c"]))
        params = EwaldParameters(r_c=c["r_c"], delta_split=c["delta"], P=c["P"],
                                 fixed_M=c["M"], prefactor=1.5)
        sc = SlabCoulombSolver(c["h"], params, kspace=ks, near_ops=near_ops)
        mine = sc.owned(pos)
        r = sc.evaluate(torch.as_tensor(pos[mine]), torch.as_tensor(q[mine]))
        Fg = np.zeros((len(q), 3))
        Fg[mine] = np.asarray(r.forces)
        t = torch.as_tensor(Fg)
        dist.all_reduce(t)
        out.put((rank, r.u_near, r.u_far, r.u_self, r.u_background, r.pressure, t.numpy(),
                 r.pair_count))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("ortho", 2), ("tri", 3)])
def test_slab_coulomb_solver_matches_single_process(case, world):
    """SlabCoulombSolver (k-space slabs + slab near field + self/background)
    on gloo ranks equals the single-process oracle composition of
    evaluate.py:114-144 (prefactor 1.5)."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coulomb_worker, args=(r, world, port, case, out))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([out.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = CASES[case]
    pos, q = _system(c)
    pref = 1.5
    oplan = O.make_plan(c["h"], c["M"], c["P"], c["delta"], c["r_c"])
    oE, oP, oF = O.kspace(oplan, pos, q)
    b = O.build_basis(O.solve_bandwidth(c["delta"]))
    i, j = O.pairs_within(c["h"], pos, c["r_c"])
    nE, nF, nP, npairs = O.short_range(c["h"], pos, q, i, j, b, c["r_c"], O.pair_table(b, c["r_c"]))
    u_self = -(b.psi0_at_zero / (2.0 * b.C0 * c["r_c"])) * float(np.sum(q * q))
    for (_, u_near, u_far, us, ub, P, F, cnt) in res:
        assert O.rel_scalar(u_near, pref * nE) <= 1e-12
        assert O.rel_scalar(u_far, pref * oE) <= 1e-12
        assert O.rel_scalar(us, pref * u_self) <= 1e-12
        assert abs(ub) <= 1e-12                      # neutral system
        assert O.rel_frobenius(P, pref * (nP + oP)) <= 1e-12
        assert O.rms_rel_forces(F, pref * (nF + oF)) <= 1e-12
        assert cnt == npairs
