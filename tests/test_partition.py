"""Leaf partition + halo exchange (the multi-GPU path) on CPU:
partition invariants, and a world_size-2 gloo run of the emulated stage
kernel that must reproduce the single-rank golden step bitwise."""

import os
import socket

import numpy as np
import pytest

import octomini_host as mesh
from paper_2107_10987_b200.batch import OFFS, neighbor_table
from paper_2107_10987_b200.partition import Partition


@pytest.mark.parametrize("bnd", ["reflecting", "periodic"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_invariants(bnd, world):
    t = mesh.build_uniform_tree(2, 8, boundary=bnd)
    parts = [Partition(t, world, r) for r in range(world)]
    G = len(t.leaves())
    assert sum(p.nown for p in parts) == G
    for r, p in enumerate(parts):
        local = set(int(g) for g in p.gids)
        for g in range(p.bounds[r], p.bounds[r + 1]):
            for j in p.gnbr[g]:
                if j >= 0:
                    assert int(j) in local  # every neighbour is owned or in the halo
        for s in range(world):
            assert p.recv_counts[s] == parts[s].send_counts[r]
            if s != r:
                # what s sends to r is exactly r's halo block from s, same order
                blk = p.halo[parts[0].owner[p.halo] == s]
                assert np.array_equal(blk, parts[s].send[r])
        b = p.batch(t)
        assert sorted(b.run_leaf.tolist()) == list(range(p.nown))


def test_runs_respect_the_kernel_run_cap():
    from paper_2107_10987_b200.batch import MAX_RUN, LeafBatch

    t = mesh.build_uniform_tree(2, 8, boundary="reflecting")
    for m in range(1, MAX_RUN + 1):
        b = LeafBatch(t, max_run=m)
        assert np.diff(b.run_off).max() <= m and b.run_off[-1] == b.ncompute
    for m in (0, MAX_RUN + 1, 8):
        with pytest.raises(ValueError):
            LeafBatch(t, max_run=m)


def test_split_tail_keeps_every_leaf_once():
    from paper_2107_10987_b200.batch import LeafBatch

    t = mesh.build_uniform_tree(3, 8, boundary="reflecting")  # 512 leaves, 128 runs of 4
    b = LeafBatch(t)
    b.split_tail([148])  # not below the run count: unchanged
    assert b.nruns == 128
    b.split_tail([20, 10])
    lens = np.diff(b.run_off)
    assert b.nruns == 128 + 20 + 10 and list(lens[:108]) == [4] * 108
    assert list(lens[108:]) == [2] * 30 + [1] * 20
    assert sorted(b.run_leaf.tolist()) == list(range(b.ncompute))
    for r in b.runs:  # still consecutive along +x
        for a, c in zip(r, r[1:]):
            assert b.info[a]["nbr"][OFFS.index((1, 0, 0))] == c


def test_neighbor_table_fast_path_matches_generic():
    for bnd in ("reflecting", "periodic", "outflow"):
        t = mesh.build_uniform_tree(2, 8, boundary=bnd)
        leaves = t.sorted_leaves()
        fast = neighbor_table(t, leaves)
        for i, lf in enumerate(leaves):
            for q, o in enumerate(OFFS):
                pos = t.neighbor_ipos(lf, o)
                want = -1 if pos is None else leaves.index(t.find_leaf_region(lf.level, pos)[0][0])
                assert fast[i, q] == want


def _worker(rank, world, port, out, case="sedov_c1"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _cases import case_tree, state_of
        from emu import EmuDistStepper

        t, g = case_tree(case)
        st = EmuDistStepper(t, 1.4, world, rank, max_run=2)
        st.rk3_step(float(g["dts"][0]))
        mine = state_of(t)[st.part.bounds[rank]:st.part.bounds[rank + 1]]
        ref = g["state1"][st.part.bounds[rank]:st.part.bounds[rank + 1]]
        np.save(os.path.join(out, f"r{rank}.npy"), np.array([np.count_nonzero(mine != ref)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("sedov_c1", 2), ("amr_reflux", 2), ("amr_reflux", 3),
                                        ("amr_sedov_small", 3)])
def test_multi_rank_gloo_step_bitwise(tmp_path, case, world):
    """World 2/3 on CPU (gloo): halo exchange, AMR ghost sources across ranks and the
    second (flux-slot) exchange for reflux must reproduce the single-rank golden step."""
    import sys

    import torch.multiprocessing as mp

    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    if case != "sedov_c1":
        from _cases import case_tree

        t, _ = case_tree(case)
        assert sum(sum(Partition(t, world, r).flux_send_counts) for r in range(world)) > 0
    mp.spawn(_worker, args=(world, port, str(tmp_path), case), nprocs=world, join=True)
    for r in range(world):
        assert int(np.load(tmp_path / f"r{r}.npy")[0]) == 0
