"""The reference's Algorithm 1 run EXHAUSTIVELY on the device for one n, in
resumable chunks -- the optional SURVEY 8(c) pin.

For every map of idcm_orbits(n, 4): the reference's combination space
(search.hpp:81-104, every leaf) is cut by the candidate of its outermost
(widest) blocks; each chunk runs the reference's inner odometer over the rest
on the device (Plan.run_kernel_basis_prefix, k6_odometer.cu) and its
accepted WPMs are compared, as sets, with the DFS rows whose reference
coordinates (kernel 8) share that prefix.  Over all chunks of a map this is
the full Algorithm 1 against the full DFS, both ways.

usage: python tools/alg1_full.py N OUT.jsonl [DONE.jsonl ...] [--budget-s S] [--chunk-leaves L]
  one JSON line per finished chunk is appended to OUT.jsonl; chunks already
  in a DONE file are skipped (resume across calls); stops after S seconds.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))

import paper_2301_00806_b200 as wpm  # noqa: E402
from reach_protocol import block_candidates, ncand  # noqa: E402


def chunks_of(widths, chunk_leaves):
    """Prefix length j and the prefixes (candidate tuples of the first j
    blocks) that cut the map's space into chunks of <= chunk_leaves leaves."""
    sizes = [ncand(w) for w in widths]
    j = 0
    rest = int(np.prod([float(c) for c in sizes]))
    while j < len(sizes) and rest > chunk_leaves:
        rest //= sizes[j]
        j += 1
    idx = np.indices(sizes[:j]).reshape(j, -1).T if j else np.zeros((1, 0), dtype=np.int64)
    return j, [tuple(int(x) for x in row) for row in idx]


def main():
    args = [a for a in sys.argv[1:]]
    budget = float(args[args.index("--budget-s") + 1]) if "--budget-s" in args else 1e18
    chunk_leaves = float(args[args.index("--chunk-leaves") + 1]) if "--chunk-leaves" in args else 2e13
    pos = [a for i, a in enumerate(args) if not a.startswith("--") and (i == 0 or not args[i - 1].startswith("--"))]
    n, out_path, done_paths = int(pos[0]), pos[1], pos[2:]
    done = set()
    for dp in done_paths + [out_path]:
        if os.path.exists(dp):
            for ln in open(dp):
                if ln.strip():
                    r = json.loads(ln)
                    done.add((r["map"], tuple(r["prefix"])))
    t0 = time.time()
    with wpm.Plan.orbits(n) as p, open(out_path, "a") as out:
        p.run()
        res = p.fetch()
        unsound, unreach, coords = p.verify(reach=True, coords=True)
        assert unsound == 0 and unreach == 0, (unsound, unreach)
        for i in range(p.num_maps):
            widths = p.space_blocks(i)
            j, prefixes = chunks_of(widths, chunk_leaves)
            lo, hi = res.offsets[i], res.offsets[i + 1]
            cands = block_candidates(coords[lo:hi], widths, j)
            dfs_all = res.map_bits(i)
            for pre in prefixes:
                if (i, pre) in done:
                    continue
                if time.time() - t0 > budget:
                    print("budget spent", flush=True)
                    return
                share = np.all(cands == np.array(pre, dtype=np.int64)[None, :], axis=1) if j else np.ones(hi - lo, bool)
                dfs_rows = dfs_all[share]
                t1 = time.time()
                got_total = p.run_kernel_basis_prefix(i, list(pre))
                st = p.kernel_basis_stats()
                got = p.fetch().map_bits(i)
                equal = got.shape == dfs_rows.shape and bool(np.array_equal(got, dfs_rows))
                rec = {"n": n, "map": i, "nfixed": j, "prefix": list(pre), "leaves": st["leaves"],
                       "odometer": int(got_total), "dfs": int(dfs_rows.shape[0]), "equal": equal,
                       "s": round(time.time() - t1, 3)}
                out.write(json.dumps(rec) + "\n")
                out.flush()
                if not equal:
                    print("MISMATCH", rec, flush=True)
    print("complete", flush=True)


if __name__ == "__main__":
    main()
