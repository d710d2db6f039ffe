"""Distributed near field (paper_2601_00161_b200.slab_near) on CPU with gloo at
world sizes 2 and 3: ghost exchange over all-to-all, slab-local sums for the
owned particles, rank-ordered reduction.  The oracle's pair values are the
test-only local backend; the result must equal the single-process oracle
short_range (realspace.py:115-157) to round-off."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import esp_oracle as O

CASES = {
    "ortho": dict(h=np.diag([7.0, 7.5, 8.0]), n=160, delta=1e-5, r_c=1.6, seed=3),
    "tri": dict(h=np.array([[6.0, 1.2, -0.8], [0.0, 6.5, 0.9], [0.0, 0.0, 7.0]]), n=120,
                delta=1e-6, r_c=1.5, seed=4),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _system(c):
    rng = np.random.default_rng(c["seed"])
    pos = rng.uniform(0, 1, (c["n"], 3)) @ c["h"].T
    s = pos @ np.linalg.inv(c["h"]).T
    pos = (s - np.floor(s)) @ c["h"].T
    q = rng.normal(size=c["n"])
    return pos, q - q.mean()


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from slab_oracle_ops import OracleNearOps
        from paper_2601_00161_b200.slab_near import SlabNearField
        c = CASES[case]
        pos, q = _system(c)
        b = O.build_basis(O.solve_bandwidth(c["delta"]))
        table = O.pair_table(b, c["r_c"])
        bounds = np.linspace(0.0, 1.0, world + 1) - 0.013   # slabs not aligned with 0
        sl = SlabNearField(c["h"], c["r_c"], bounds, OracleNearOps(c["h"], b, c["r_c"], table))
        own = np.nonzero(sl.owner(pos) == rank)[0]
        E, P, F, cnt = sl.evaluate(torch.as_tensor(pos[own]), torch.as_tensor(q[own]))
        out.put((rank, own, E, P, np.asarray(F), cnt))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["ortho", "tri"])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_near_field_matches_single_process(case, world):
    c = CASES[case]
    pos, q = _system(c)
    b = O.build_basis(O.solve_bandwidth(c["delta"]))
    table = O.pair_table(b, c["r_c"])
    i, j = O.pairs_within(c["h"], pos, c["r_c"])
    E0, F0, P0, n0 = O.short_range(c["h"], pos, q, i, j, b, c["r_c"], table)
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
    F = np.zeros_like(F0)
    seen = np.zeros(len(pos), dtype=int)
    for (_, own, E, P, Fr, cnt) in res:
        F[own] = Fr
        seen[own] += 1
        assert abs(E - E0) <= 1e-12 * abs(E0)
        assert O.rel_frobenius(P, P0) <= 1e-12
        assert cnt == n0
    assert np.all(seen == 1)
    assert O.rms_rel_forces(F, F0) <= 1e-12
