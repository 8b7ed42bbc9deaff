"""Multi-GPU plumbing for the enumeration (one process per GPU).

The job (parallel_for_index, parallel.hpp:27-54, across GPUs):

  1. every rank splits its share of the root tasks below the root
     (Plan.split(rank, world): split-mode kernel-3 launches until the
     frontiers hold >= 640 records per GPU; the rows and nodes above a rank's
     frontier stay on that rank);
  2. the frontier records are all-gathered (NCCL) and a claim counter in
     rank 0's HBM is shared through a CUDA IPC handle;
  3. every rank runs the claim phase (Plan.run_claim): its kernel pulls
     frontier records through the one counter (system-scope atomics over
     NVLink) into its own work queue and shares them by donation -- no GPU
     ever waits for another, the records go to whichever GPU is free;
  4. the canonical rows are gathered to rank 0 only (point-to-point
     send/recv, not an all-gather) and sorted there once
     (wpm_canonical_sort_device); the union is disjoint, so the sort finds no
     duplicate, which is checked.

The same host logic runs over gloo with CPU tensors in the CPU tests, with a
torch.distributed Store counter standing in for the device counter
(StoreCounter) and the CPU restatement standing in for the device search.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np


def shard_roots(num_tasks: int, rank: int, world: int) -> List[int]:
    """Static root-task shard of `rank` (wpm_plan_run(plan, rank, world);
    the fallback without a shared counter)."""
    return [t for t in range(num_tasks) if t % world == rank]


def canonical_key(map_id: int, row: np.ndarray) -> Tuple[int, Tuple[int, ...]]:
    """(map, ascending facet indices): Python tuple order is exactly the
    reference's complex order (search.hpp:254-255, a proper prefix first)."""
    idx = []
    for w, word in enumerate(row.tolist()):
        x = int(word)
        while x:
            b = (x & -x).bit_length() - 1
            idx.append(w * 64 + b)
            x &= x - 1
    return map_id, tuple(idx)


def merge_host(parts: Sequence[Tuple[np.ndarray, np.ndarray]]) -> Tuple[np.ndarray, np.ndarray, int]:
    """Canonical merge of per-rank (map_ids, rows) on the host.  Returns
    (map_ids, rows, duplicates)."""
    items = []
    for maps, rows in parts:
        for i in range(rows.shape[0]):
            items.append((canonical_key(int(maps[i]), rows[i]), int(maps[i]), rows[i]))
    items.sort(key=lambda t: t[0])
    dups = sum(1 for a, b in zip(items, items[1:]) if a[0] == b[0])
    words = parts[0][1].shape[1] if parts else 1
    rows = np.array([t[2] for t in items], dtype=np.uint64).reshape(-1, words)
    maps = np.array([t[1] for t in items], dtype=np.int64)
    return maps, rows, dups


# ---------------------------------------------------------------- collectives

def gather_to_rank0(dist, rank: int, world: int, parts: Sequence, device=None) -> List[List]:
    """Point-to-point gather of per-rank tensors to rank 0 (each rank sends
    its tensors' lengths, then the tensors; rank 0 receives them in rank
    order).  parts: a list of 1-D tensors of fixed dtypes; returns, on rank 0,
    [[rank r's tensors] for r in ranks], [] elsewhere.  NCCL and gloo."""
    import torch

    lens = torch.tensor([p.numel() for p in parts], dtype=torch.int64, device=device)
    if rank != 0:
        dist.send(lens, 0)
        for p in parts:
            if p.numel():
                dist.send(p.contiguous(), 0)
        return []
    out = [list(parts)]
    for r in range(1, world):
        ln = torch.zeros_like(lens)
        dist.recv(ln, r)
        got = []
        for p, k in zip(parts, ln.tolist()):
            buf = torch.empty(int(k), dtype=p.dtype, device=p.device)
            if k:
                dist.recv(buf, r)
            got.append(buf)
        out.append(got)
    return out


def reduce_counts(dist, per_map: Sequence[int], nodes: int, device=None) -> Tuple[List[int], int]:
    """all_reduce(sum) of per-map WPM counts and the node count."""
    import torch

    t = torch.tensor(list(per_map) + [nodes], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    v = [int(x) for x in t.tolist()]
    return v[:-1], v[-1]


# ---------------------------------------------------------------- the shared frontier

class StoreCounter:
    """A claim counter over a torch.distributed Store (atomic add): the host
    stand-in for the device claim counter in CPU tests."""

    def __init__(self, store, key: str = "wpm_claim"):
        self.store, self.key = store, key

    def claim(self) -> int:
        return int(self.store.add(self.key, 1)) - 1


def claim_loop(counter, count: int, work: Callable[[int], None]) -> int:
    """Host form of a GPU's claim phase: pull item indices from the shared
    counter until it passes `count`; returns the items this rank processed."""
    done = 0
    while True:
        i = counter.claim()
        if i >= count:
            return done
        work(i)
        done += 1


def share_frontier(dist, rank: int, recs, count: int, recw: int, device):
    """Broadcast rank 0's frontier records (count x recw uint32 words, shipped
    as int32) to every rank; returns (recs tensor on this rank's device, count, recw)."""
    import torch

    hdr = torch.tensor([count, recw] if rank == 0 else [0, 0], dtype=torch.int64, device=device)
    dist.broadcast(hdr, 0)
    count, recw = (int(x) for x in hdr.tolist())
    if rank != 0:
        recs = torch.empty(max(count * recw, 1), dtype=torch.int32, device=device)
    if count:
        dist.broadcast(recs[: count * recw], 0)
    return recs, count, recw


def all_gather_records(dist, mine, count: int, recw: int, device):
    """Concatenate every rank's `count` records (recw int32 words each) in rank
    order on every rank (padded all_gather); returns (tensor, total count)."""
    import torch

    counts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(dist.get_world_size())]
    dist.all_gather(counts, torch.tensor([count], dtype=torch.int64, device=device))
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)
    pad = torch.zeros(cap * recw, dtype=torch.int32, device=device)
    pad[: count * recw] = mine[: count * recw]
    parts = [torch.empty_like(pad) for _ in counts]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: counts[r] * recw] for r in range(len(counts))]), sum(counts)


def share_claim_counter(dist, rank: int, device: int):
    """Rank 0 creates the device claim counter and broadcasts its 64-byte CUDA
    IPC handle; the other ranks open it.  Returns (pointer, opened)."""
    import torch

    import paper_2301_00806_b200 as wpm

    dev = torch.device("cuda", device)
    if rank == 0:
        ptr, handle = wpm.claim_counter_create(device)
        h = torch.tensor(list(handle), dtype=torch.uint8, device=dev)
    else:
        h = torch.zeros(64, dtype=torch.uint8, device=dev)
    dist.broadcast(h, 0)
    if rank == 0:
        return ptr, False
    return wpm.claim_counter_open(device, bytes(h.cpu().tolist())), True


def run_job(dist, plan, rank: int, world: int, device: int, counter=None, target: int = 0) -> int:
    """One multi-GPU enumeration across the ranks (the module docstring's steps
    1-3) on the ranks' resident plans (same maps).  `counter` = (pointer,
    opened) from share_claim_counter, reused across runs (reset by rank 0).
    Returns this rank's row count; its canonical rows stay on its device."""
    import torch

    import paper_2301_00806_b200 as wpm

    dev = torch.device("cuda", device)
    if world == 1:
        plan.split(0, target or 2048)
        own = counter is None
        ctr = wpm.claim_counter_create(device)[0] if own else counter[0]
        if not own:
            wpm.claim_counter_reset(device, ctr)
        try:
            return plan.run_claim(ctr)
        finally:
            if own:
                wpm.claim_counter_close(device, ctr, False)
    # every rank splits its share of the root tasks; the frontiers are all-gathered
    plan.split(0, target or 640, rank, world)  # depth 0: the library's per-shard first depth
    ptr, count, recw = plan.frontier()
    recs, total_recs = all_gather_records(dist, _wrap_device(ptr, count * recw, torch.int32, dev), count, recw, dev)
    torch.cuda.synchronize(dev)
    plan.load_frontier(recs.data_ptr(), total_recs)  # a copy: `recs` may go after this
    if rank == 0:
        wpm.claim_counter_reset(device, counter[0])
    dist.barrier()  # the counter is reset before any rank claims
    total = plan.run_claim(counter[0])
    dist.barrier()  # every claim is done before the counter is reused
    return total


def gather_to_rank0_device(dist, plan, rank: int, device: int, return_rows: bool = False):
    """Every rank's resident canonical rows go to rank 0 only (send/recv),
    then one canonical sort there.  Returns (count, duplicates) on rank 0,
    (local count, 0) elsewhere; with return_rows also the sorted rows / map
    ids (rank 0) as device tensors."""
    import torch

    import paper_2301_00806_b200 as wpm

    bits_ptr, map_ptr, count, w32 = plan.device_result()
    dev = torch.device("cuda", device)
    rows = _wrap_device(bits_ptr, count * w32, torch.int32, dev)
    maps = _wrap_device(map_ptr, count, torch.int16, dev).view(torch.uint8)  # NCCL has no int16: bytes
    world = dist.get_world_size()
    got = gather_to_rank0(dist, rank, world, [rows, maps], dev)
    if rank != 0:
        return (count, 0, None, None) if return_rows else (count, 0)
    all_rows = torch.cat([g[0] for g in got])
    all_maps = torch.cat([g[1] for g in got]).view(torch.int16)
    total = all_maps.numel()
    out_rows = torch.empty_like(all_rows)
    out_maps = torch.empty_like(all_maps)
    torch.cuda.synchronize(dev)
    dups = wpm.canonical_sort_device(device, all_rows.data_ptr(), all_maps.data_ptr(), total, w32,
                                     out_rows.data_ptr(), out_maps.data_ptr())
    if return_rows:
        return total, dups, out_rows, out_maps
    return total, dups


def _wrap_device(ptr: int, numel: int, dtype, device):
    """A torch view (CUDA array interface, no copy) of library-owned device
    memory; valid until the plan's next run."""
    import torch

    if numel == 0:
        return torch.zeros(0, dtype=dtype, device=device)
    typestr = {torch.int32: "<i4", torch.int16: "<i2", torch.int64: "<i8"}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_CAI(), device=device)
