"""Single-GPU split-then-search vs root seeding at small n (ms_search median)."""
import os, statistics, sys, time
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
for n in [int(x) for x in sys.argv[1:]] or [5]:
    for d in (0, 1, 2, 3, 4, 5, 6):
        with wpm.Plan.orbits(n) as p:
            p.set_split(d)
            s, w = [], []
            for _ in range(8):
                t0 = time.perf_counter()
                p.run()
                w.append((time.perf_counter() - t0) * 1e3)
                s.append(p.stats()["ms_search"])
            print("n", n, "split", d, "search", round(statistics.median(s[1:]), 3), "wall", round(statistics.median(w[1:]), 3), "tasks", p.stats()["tasks"], flush=True)
