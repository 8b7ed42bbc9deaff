"""Median search / sort ms per n (Plan.orbits, 8 runs)."""
import os, statistics, sys
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
for n in [int(x) for x in sys.argv[1:]] or [8]:
    with wpm.Plan.orbits(n) as p:
        s, t = [], []
        for _ in range(8):
            p.run()
            st = p.stats()
            s.append(st["ms_search"])
            t.append(st["ms_sort"])
        print("n", n, "search", round(statistics.median(s[1:]), 3), "sort", round(statistics.median(t[1:]), 3), flush=True)
