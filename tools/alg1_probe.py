"""Dev probe: Algorithm 1 (kernel-basis odometer) on the device vs the golden
reference counts/spaces; prints leaves/s per n."""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_00806_b200 as wpm  # noqa: E402

g = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                "golden.json")))
for n in [int(x) for x in sys.argv[1:]] or [2, 3, 4, 5, 6]:
    with wpm.Plan.orbits(n) as p:
        t0 = time.time()
        tot = p.run_kernel_basis()
        wall = time.time() - t0
        st = p.kernel_basis_stats()
        res = p.fetch()
        ref = g["ubt"].get(str(n))
        ok_counts = ok_space = None
        if ref:
            ok_counts = res.counts == [m["wpms"] for m in ref["maps"]]
            ok_space = [p.combination_space(i)["space"] for i in range(res.num_maps)] == [m["space"] for m in ref["maps"]]
        tot2 = p.run_kernel_basis()
        st2 = p.kernel_basis_stats()
        print(json.dumps({"n": n, "wpms": tot, "counts_ok": ok_counts, "space_ok": ok_space, "leaves": st2["leaves"],
                          "checked": st2["checked"], "ms_prep": round(st2["ms_prep"], 2),
                          "ms_leaves": round(st2["ms_leaves"], 3), "wall_s": round(wall, 3),
                          "leaves_per_s": st2["leaves"] / (st2["ms_leaves"] * 1e-3) if st2["ms_leaves"] else None,
                          "dups": res.duplicates}), flush=True)
