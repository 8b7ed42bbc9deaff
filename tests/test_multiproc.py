"""World-size-2 gloo tests of the multi-GPU host logic (paper_2301_00806_b200.dist):
the static root-task shard (Plan.run(rank, world)) and the shared-frontier
claim protocol of dist.run_job (broadcast frontier, one atomic claim counter,
point-to-point gather to rank 0, canonical merge), with the CPU restatement of
the device search standing in for the GPU; rank 0 checks the union equals
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
        import torch

        maps = np.concatenate(maps_out)
        bits = np.concatenate(bits_out)
        got = wdist.gather_to_rank0(dist, rank, world, [torch.from_numpy(maps),
                                                        torch.from_numpy(bits.view(np.int64).reshape(-1))])
        counts, nodes = wdist.reduce_counts(dist, per_map, node_sum)
        if rank == 0:
            parts = [(g[0].numpy(), g[1].numpy().view(np.uint64).reshape(-1, 4)) for g in got]
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


def _claim_worker(rank, world, port, port2, n, results):
    """The shared-frontier protocol of dist.run_job over gloo: every rank makes
    its share of the frontier (here: its share of the root tasks (map, minimum
    facet f) of four maps), the shares are all-gathered, every rank claims
    items through one shared atomic
    counter (a Store counter standing in for the device counter) and runs
    them (the CPU restatement of the device search over root f only), the
    rows go to rank 0 by point-to-point gather and are merged canonically."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch
    import torch.distributed as dist

    from oracle_bind import Oracle
    from paper_2301_00806_b200 import dist as wdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.TCPStore("127.0.0.1", port2, world, rank == 0)
    try:
        orc = Oracle()
        rows = orc.idcm_orbits(n)[:4]
        unis = [orc.matroid_universe(r) for r in rows]
        cap = orc.cyclic_facet_bound(n)
        recw = 2
        # each rank's share of the root tasks (t % world == rank) is its
        # "frontier"; the frontiers are all-gathered in rank order
        items = [(i, f) for i, u in enumerate(unis) for f in range(len(u))]
        share = [it for t, it in enumerate(items) if t % world == rank]
        mine = torch.tensor([x for it in share for x in it] or [0], dtype=torch.int32)
        recs, count = wdist.all_gather_records(dist, mine, len(share), recw, "cpu")
        assert count == len(items)
        dist.barrier()
        maps_out, bits_out, node_sum, mine = [], [], 0, []

        def work(i):
            nonlocal node_sum
            m, f = int(recs[2 * i]), int(recs[2 * i + 1])
            cnt, nodes, bits = orc.dfs(n, unis[m], cap, root_lo=f, root_hi=f + 1)
            node_sum += nodes
            mine.append(i)
            maps_out.append(np.full(cnt, m, dtype=np.int64))
            pad = np.zeros((cnt, 4), dtype=np.uint64)
            pad[:, : bits.shape[1]] = bits
            bits_out.append(pad)

        done = wdist.claim_loop(wdist.StoreCounter(store), count, work)
        maps = np.concatenate(maps_out) if maps_out else np.zeros(0, dtype=np.int64)
        bits = np.concatenate(bits_out) if bits_out else np.zeros((0, 4), dtype=np.uint64)
        got = wdist.gather_to_rank0(dist, rank, world, [torch.from_numpy(maps), torch.from_numpy(bits.view(np.int64).reshape(-1)),
                                                        torch.tensor(mine, dtype=torch.int64)])
        _, nodes = wdist.reduce_counts(dist, [done], node_sum)
        if rank == 0:
            parts = [(g[0].numpy(), g[1].numpy().view(np.uint64).reshape(-1, 4)) for g in got]
            claimed = sorted(int(x) for g in got for x in g[2].tolist())
            m, b, dups = wdist.merge_host(parts)
            results.put((nodes, m.tolist(), b.tolist(), dups, claimed, count, [len(g[2]) for g in got]))
    finally:
        dist.destroy_process_group()


def test_gloo_shared_frontier_claims(oracle):
    import torch.multiprocessing as mp

    n, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port, port2 = _free_port(), _free_port()
    procs = [ctx.Process(target=_claim_worker, args=(r, world, port, port2, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    nodes, maps, bits, dups, claimed, count, per_rank = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert claimed == list(range(count)) and sum(per_rank) == count  # every item exactly once
    exp_maps, exp_bits, exp_nodes = [], [], 0
    for i, r in enumerate(oracle.idcm_orbits(n)[:4]):
        u = oracle.matroid_universe(r)
        cnt, nd, b = oracle.dfs(n, u, oracle.cyclic_facet_bound(n))
        exp_nodes += nd
        pad = np.zeros((cnt, 4), dtype=np.uint64)
        pad[:, : b.shape[1]] = b
        exp_maps += [i] * cnt
        exp_bits += pad.tolist()
    assert dups == 0 and nodes == exp_nodes
    assert maps == exp_maps and bits == exp_bits
