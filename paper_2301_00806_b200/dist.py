"""Multi-GPU plumbing for the enumeration (one process per GPU).

The search shards with no data-path collective: rank r of W takes the root
tasks t with t % W == r (Plan.run(r, W); the root tasks are the
"minimum facet" branches of every map, disjoint and exhaustive).  The only
collectives are at the end:

  1. all_reduce of the per-map WPM counts and the node count,
  2. all_gather of the per-rank row counts, then of the (padded) rows,
  3. one canonical sort on rank 0 (wpm_canonical_sort_device on the GPU;
     merge_host for CPU/gloo runs) -- the union is disjoint, so the sort
     finds no duplicate, which is checked.

Backend-agnostic over torch.distributed: NCCL with CUDA tensors on the GPU
box, gloo with CPU tensors in the CPU tests.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def shard_roots(num_tasks: int, rank: int, world: int) -> List[int]:
    """Root-task indices owned by `rank` (mirrors plan_search in api.cu)."""
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


def gather_rows(dist, maps: np.ndarray, rows: np.ndarray, device=None):
    """all_gather per-rank (map_ids, rows) to every rank; returns the list of
    per-rank parts.  Rows are uint64 words shipped as int64 tensors."""
    import torch

    words = rows.shape[1]
    world = dist.get_world_size()
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=device)
    counts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    cap = max(counts) if counts else 0
    pad_rows = np.zeros((cap, words), dtype=np.uint64)
    pad_rows[: rows.shape[0]] = rows
    pad_maps = np.zeros(cap, dtype=np.int64)
    pad_maps[: maps.shape[0]] = maps
    t_rows = torch.from_numpy(pad_rows.view(np.int64).copy()).to(device)
    t_maps = torch.from_numpy(pad_maps).to(device)
    g_rows = [torch.zeros_like(t_rows) for _ in range(world)]
    g_maps = [torch.zeros_like(t_maps) for _ in range(world)]
    dist.all_gather(g_rows, t_rows)
    dist.all_gather(g_maps, t_maps)
    parts = []
    for r in range(world):
        c = counts[r]
        parts.append((g_maps[r][:c].cpu().numpy(), g_rows[r][:c].cpu().numpy().view(np.uint64)))
    return parts


def reduce_counts(dist, per_map: Sequence[int], nodes: int, device=None) -> Tuple[List[int], int]:
    """all_reduce(sum) of per-map WPM counts and the node count."""
    import torch

    t = torch.tensor(list(per_map) + [nodes], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    v = [int(x) for x in t.tolist()]
    return v[:-1], v[-1]


def gather_to_rank0_device(dist, plan, rank: int, device: int, return_rows: bool = False):
    """GPU path: NCCL all_gather of every rank's resident canonical rows into
    rank 0's HBM, then one canonical sort there.  Returns (count, duplicates)
    on rank 0, (local count, 0) elsewhere; with return_rows also the sorted
    rows / map ids (rank 0) as device tensors."""
    import torch

    import paper_2301_00806_b200 as wpm

    bits_ptr, map_ptr, count, w32 = plan.device_result()
    dev = torch.device("cuda", device)
    # wrap the resident rows (uint32 words) and map ids without a copy
    rows = _wrap_device(bits_ptr, count * w32, torch.int32, dev)
    maps = _wrap_device(map_ptr, count, torch.int16, dev)
    world = dist.get_world_size()
    n = torch.tensor([count], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)
    pr = torch.zeros(cap * w32, dtype=torch.int32, device=dev)
    pm = torch.zeros(cap, dtype=torch.int16, device=dev)
    pr[: count * w32] = rows
    pm[:count] = maps
    g_rows = [torch.zeros_like(pr) for _ in range(world)]
    g_maps = [torch.zeros(cap * 2, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(g_rows, pr)
    dist.all_gather(g_maps, pm.view(torch.uint8))  # NCCL has no int16: ship the ids as bytes
    if rank != 0:
        return (count, 0, None, None) if return_rows else (count, 0)
    all_rows = torch.cat([g_rows[r][: counts[r] * w32] for r in range(world)])
    all_maps = torch.cat([g_maps[r].view(torch.int16)[: counts[r]] for r in range(world)])
    total = sum(counts)
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
