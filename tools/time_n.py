"""Per-n timing sweep of the device path (dev tool): search / sort / step ms,
nodes, WPMs, nodes/s, for n in argv (default 2..11)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_00806_b200 as wpm  # noqa: E402

ns = [int(x) for x in sys.argv[1:]] or list(range(2, 12))
peak = wpm.int_peak(0)
print(f"int peak {peak / 1e12:.2f} Tops/s", flush=True)
for n in ns:
    t0 = time.time()
    with wpm.Plan.orbits(n) as p:
        tc = time.time() - t0
        best = None
        for _ in range(4):
            p.run()
            st = p.stats()
            tm = p.timing()
            if best is None or tm["ms_total"] < best[2]:
                best = (st["ms_search"], st["ms_sort"], tm["ms_total"], st["nodes"], st["tasks"], tm["warps"])
        r = p.fetch()
    s, so, tot, nodes, tasks, warps = best
    print(json.dumps({"n": n, "maps": r.num_maps, "wpms": r.total, "dups": r.duplicates, "nodes": nodes,
                      "tasks": tasks, "warps": warps, "ms_search": round(s, 3), "ms_sort": round(so, 3),
                      "ms_total": round(tot, 3), "Gnodes_per_s_search": round(nodes / s / 1e6, 3),
                      "create_s": round(tc, 3)}), flush=True)
