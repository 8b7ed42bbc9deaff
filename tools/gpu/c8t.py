import os, sys, statistics
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm
for n in (7, 8):
    ds = wpm.idcm_orbits(n)
    for i in (0, 3, 7):
        cols = wpm.charmap_of_dcm(ds[i])
        with wpm.Plan.charmaps(n, n + 4, [cols]) as p:
            ms = []
            for _ in range(6):
                p.run(); ms.append(p.stats()["ms_search"])
            st = p.stats()
            print(os.environ.get("WPM_DEBUG_LIB", "main"), os.environ.get("WPM_TS", "1"), n, i, p.timing()["warps"], round(statistics.median(ms[1:]), 3), st["nodes"], round(st["nodes"] / statistics.median(ms[1:]) / 1e6, 3), flush=True)
