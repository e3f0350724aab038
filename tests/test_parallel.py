"""Multi-rank (slab-sharded) integrators: world size 2 over gloo on CPU.

The orchestration (layouts, pencil transposes through all_to_all, the
operation order of every method) runs with a CPU test backend whose mode
products are the oracle's (sequential-k, shape-independent rounding), so the
sharded run must equal the unsharded one BIT FOR BIT -- the property the GPU
backend has with the single-GPU kernels -- and match the oracle's integrate."""
import os

import pytest

from conftest import ROOT, run_torchrun

WORKER = os.path.join(ROOT, "tests", "parallel_worker.py")


@pytest.mark.parametrize("case,method", [("ac2d", "exp_euler"), ("ac3d", "etd2rk"),
                                         ("bru", "etd2rk"), ("bru", "lawson2b"),
                                         ("nls", "exp_euler"), ("ac3d", "lawson_euler")])
def test_sharded_equals_unsharded_world2(case, method):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    rc, out = run_torchrun(WORKER, [case, method], env=env)
    assert rc == 0, out[-4000:]
    assert "SHARDED-OK" in out, out[-4000:]


@pytest.mark.parametrize("P,species,spatial", [(2, 1, [6, 4, 8]), (3, 2, [5, 6, 9]),
                                               (4, 1, [8, 12])])
def test_scatter_map_equals_all_to_all(P, species, spatial):
    """The device exchange's index map (parallel.scatter_destinations, the
    host restatement of kp_scatter) places every entry exactly where the
    all-to-all pencil transposes put it, in both directions."""
    import numpy as np
    import torch
    from paper_2304_02327_b200 import parallel

    lay = parallel.Layout.of(spatial, species, P)
    rng = np.random.default_rng(5)
    glob = rng.standard_normal(list(spatial) + ([species] if species > 1 else []))

    def all_to_all_sim(sends):  # P in-process ranks
        chunks = [s.view(P, -1) for s in sends]
        return [torch.cat([chunks[src][dst] for src in range(P)]) for dst in range(P)]

    slabs = []
    for r in range(P):
        sl = parallel.local_slab(glob, P, r, species)
        slabs.append(torch.from_numpy(np.asfortranarray(sl).reshape(-1, order="F").copy()))

    # reference: the collective path (slab_to_pencil's permutes + all_to_all)
    A, B, C, S = lay.A, lay.B, lay.C, lay.S
    Cl, Bp = C // P, B // P
    sends = [x.view(S, Cl, P, Bp, A).permute(2, 0, 1, 3, 4).contiguous().view(-1) for x in slabs]
    recvs = all_to_all_sim(sends)
    pencils = [rv.view(P, S, Cl, Bp, A).permute(1, 0, 2, 3, 4).contiguous().view(-1)
               for rv in recvs]
    # the scatter map
    got = [np.full(pencils[0].numel(), np.nan) for _ in range(P)]
    for r in range(P):
        dst, idx = parallel.scatter_destinations(lay, 1, r)
        for s in range(P):
            m = dst == s
            got[s][idx[m]] = slabs[r].numpy()[m]
    for s in range(P):
        assert np.array_equal(got[s], pencils[s].numpy())
    # and back
    back = [np.full(slabs[0].numel(), np.nan) for _ in range(P)]
    for r in range(P):
        dst, idx = parallel.scatter_destinations(lay, 2, r)
        for s in range(P):
            m = dst == s
            back[s][idx[m]] = pencils[r].numpy()[m]
    for s in range(P):
        assert np.array_equal(back[s], slabs[s].numpy())

