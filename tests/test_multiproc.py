"""World-size-2 gloo test of the multi-GPU host logic (paper_2301_00806_b200.dist):
each rank computes its root-task shard (here with the CPU restatement of the
device search, standing in for Plan.run(rank, world)), the shards are gathered
with torch.distributed and merged canonically; rank 0 checks the union equals
the single-process result, with no duplicates and the node counts adding up."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, results):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    from oracle_bind import Oracle
    from paper_2301_00806_b200 import dist as wdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        rows = orc.idcm_orbits(n)
        maps_out, bits_out, node_sum = [], [], 0
        per_map = []
        for i, r in enumerate(rows[:4]):
            u = orc.matroid_universe(r)
            cnt, nodes, bits = orc.dfs_shard(n, u, orc.cyclic_facet_bound(n), rank, world)
            node_sum += nodes
            per_map.append(cnt)
            maps_out.append(np.full(cnt, i, dtype=np.int64))
            w = 4
            pad = np.zeros((cnt, w), dtype=np.uint64)
            pad[:, : bits.shape[1]] = bits
            bits_out.append(pad)
        maps = np.concatenate(maps_out)
        bits = np.concatenate(bits_out)
        parts = wdist.gather_rows(dist, maps, bits)
        counts, nodes = wdist.reduce_counts(dist, per_map, node_sum)
        if rank == 0:
            m, b, dups = wdist.merge_host(parts)
            results.put((counts, nodes, m.tolist(), b.tolist(), dups))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_gather_merge(oracle, world):
    import torch.multiprocessing as mp

    n = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    counts, nodes, maps, bits, dups = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference
    rows = oracle.idcm_orbits(n)
    exp_maps, exp_bits, exp_nodes, exp_counts = [], [], 0, []
    for i, r in enumerate(rows[:4]):
        u = oracle.matroid_universe(r)
        cnt, nd, b = oracle.dfs(n, u, oracle.cyclic_facet_bound(n))
        exp_counts.append(cnt)
        exp_nodes += nd
        pad = np.zeros((cnt, 4), dtype=np.uint64)
        pad[:, : b.shape[1]] = b
        exp_maps += [i] * cnt
        exp_bits += pad.tolist()
    assert dups == 0
    assert counts == exp_counts
    assert nodes == exp_nodes
    assert maps == exp_maps
    assert bits == exp_bits


def test_shard_roots_partition():
    from paper_2301_00806_b200 import dist as wdist

    for world in (1, 2, 3, 8):
        got = sorted(t for r in range(world) for t in wdist.shard_roots(100, r, world))
        assert got == list(range(100))
